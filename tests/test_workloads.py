"""CPU: the synthetic block selections are the reference's own.  Config 1/2
(and the Config 5 block sizes) draw every request's hash_ids the way
kvcsim::generate_workload does (proj/src/trace.cpp:188-218: the first
floor(cache_ratio * blocks) ids from one shared hot chain grown on demand,
the rest globally fresh); tests/golden/workload_ids.npz holds the
reference's outputs (tests/golden/make_workload_golden.sh)."""
import numpy as np
import pytest

from conftest import golden
from paper_2407_00079_b200.workloads import TransferWorkload


@pytest.mark.parametrize("name", ["c2_bs16", "c1_bs16", "c2_bs64", "c2_bs512", "c2_r03"])
def test_transfer_workload_ids_equal_generate_workload(name):
    g = golden("workload_ids.npz")
    n_req, tokens, ratio, bs = g[name + "_args"]
    wl = TransferWorkload(n_req=int(n_req), wave=1, tokens=int(tokens), block_size=int(bs),
                          cache_ratio=float(ratio))
    got = np.stack(wl.hash_ids)
    assert got.shape == g[name].shape
    assert np.array_equal(got, g[name])


def test_config2_selection_shape():
    wl = TransferWorkload()
    assert wl.blocks == 512 and wl.src_slots == 256 + 64 * 256  # shared prefix stored once
    assert wl.payload_bytes() == 64 * 2_684_354_560
    # the source table maps every id to one slot: shared ids to the same slots
    assert all(np.array_equal(t[:256], wl.src_tables[0][:256]) for t in wl.src_tables)
    assert len(np.unique(np.concatenate(wl.src_tables))) == wl.src_slots
