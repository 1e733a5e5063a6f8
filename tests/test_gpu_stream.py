"""GPU parity of the C++ layer-wise streamer (kvx_streamer_*): local modes on
one GPU against the C restatement (memcmp), and -- when the box has 2+ GPUs --
the peer modes through bench.py under torchrun (every destination word is
verified inside bench.py; a mismatch exits non-zero)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int32, device=DEV)


@pytest.mark.parametrize("mode", ["local_fused", "local_staged"])
@pytest.mark.parametrize("chunk,lpc", [(0, 1), (5, 1), (7, 3), (64, 80)])
def test_local_streamer_vs_oracle(kvx, oracle_lib, mode, chunk, lpc):
    from paper_2407_00079_b200.streamer import Streamer
    L, bs, n = 6, 16, 23
    src = kvx.KVPool(L, bs, 8, 128, 2, 40, 0)
    dst = kvx.KVPool(L, bs, 8, 128, 2, 50, 0)
    src.fill_synthetic(4)
    dst.tensor_view().zero_()
    rng = np.random.default_rng(chunk * 10 + lpc)
    st_tab = rng.integers(0, 40, size=n).astype(np.int32)
    dt_tab = rng.permutation(50)[:n].astype(np.int32)
    cb = chunk or n
    slot = min(lpc, L) * 2 * min(cb, n) * src.slab
    s = Streamer(mode, "local", src, dst, ring=2, slot_bytes=slot)
    s.send(_t(st_tab), _t(dt_tab), 1, L, chunk, lpc)
    s.finish()
    s.finish(torch.cuda.current_stream())
    torch.cuda.synchronize()
    want = np.zeros(dst.nbytes, dtype=np.uint8)
    o = oracle_lib
    o.copy_paged(src.tensor_view().cpu().numpy(), 40, st_tab, want, 50, dt_tab, src.slab, 1, L)
    assert np.array_equal(dst.tensor_view().cpu().numpy(), want)
    units = -(-n // cb) * -(-(L - 1) // lpc)
    assert s.units == units


def test_local_streamer_graph_replay(kvx, oracle_lib):
    """Record one step of many small units (programmatic-dependent launches)
    as a CUDA graph, replay it: bit-exact, and the tables are read at replay
    time (new contents, same pointers)."""
    from paper_2407_00079_b200.streamer import Streamer
    L, bs, n = 6, 16, 23
    src = kvx.KVPool(L, bs, 8, 128, 2, 40, 0)
    dst = kvx.KVPool(L, bs, 8, 128, 2, 50, 0)
    src.fill_synthetic(4)
    rng = np.random.default_rng(3)
    st_d = _t(rng.integers(0, 40, size=n).astype(np.int32))
    dt_d = _t(rng.permutation(50)[:n].astype(np.int32))
    s = Streamer("local_fused", "local", src, dst)
    s.send(st_d, dt_d, 0, L, 2, 1)  # eager warm-up: 12 chunks x 6 layers
    s.finish(torch.cuda.current_stream())
    torch.cuda.synchronize()
    u0 = s.units
    launches0 = kvx.launch_count()
    s.record_begin()
    s.send(st_d, dt_d, 0, L, 2, 1)
    s.record_end()
    assert s.units == u0 and kvx.launch_count() == launches0  # recorded, not run
    o = oracle_lib
    for trial in range(2):
        st_tab = rng.integers(0, 40, size=n).astype(np.int32)
        dt_tab = rng.permutation(50)[:n].astype(np.int32)
        st_d.copy_(_t(st_tab))
        dt_d.copy_(_t(dt_tab))
        dst.tensor_view().zero_()
        torch.cuda.synchronize()
        s.replay()
        s.finish(torch.cuda.current_stream())
        torch.cuda.synchronize()
        want = np.zeros(dst.nbytes, dtype=np.uint8)
        o.copy_paged(src.tensor_view().cpu().numpy(), 40, st_tab, want, 50, dt_tab, src.slab,
                     0, L)
        assert np.array_equal(dst.tensor_view().cpu().numpy(), want), trial
    assert s.units == u0 + 2 * 12 * 6
    assert kvx.launch_count() == launches0 + 2 * 12 * 6


def test_local_streamer_calls_stay_ordered(kvx, oracle_lib):
    """Units inside one send overlap (programmatic dependent launch); a later
    send that rewrites the same decode slots must still land after it."""
    from paper_2407_00079_b200.streamer import Streamer
    L, bs, n = 8, 16, 64
    src = kvx.KVPool(L, bs, 8, 128, 2, 200, 0)
    dst = kvx.KVPool(L, bs, 8, 128, 2, 64, 0)
    src.fill_synthetic(9)
    s = Streamer("local_fused", "local", src, dst)
    dt_tab = np.arange(n, dtype=np.int32)
    rng = np.random.default_rng(8)
    tabs = [rng.permutation(200)[:n].astype(np.int32) for _ in range(6)]
    for t in tabs:  # six waves into the same 64 slots, one layer per unit
        s.send(_t(t), _t(dt_tab), 0, L, 16, 1)
    s.finish(torch.cuda.current_stream())
    torch.cuda.synchronize()
    want = np.zeros(dst.nbytes, dtype=np.uint8)
    oracle_lib.copy_paged(src.tensor_view().cpu().numpy(), 200, tabs[-1], want, 64, dt_tab,
                          src.slab, 0, L)
    assert np.array_equal(dst.tensor_view().cpu().numpy(), want)


def test_streamer_rejects_bad_shapes(kvx):
    from paper_2407_00079_b200.streamer import Streamer
    src = kvx.KVPool(2, 16, 8, 128, 2, 8, 0)
    with pytest.raises(kvx.ValidationError):
        Streamer("local_fused", "sender", src, None)
    with pytest.raises(kvx.ValidationError):
        Streamer("peer_ce", "sender", src, None, ring=0, slot_bytes=0)


_PORT = [29531]


def _torchrun(n, *args, timeout=900):
    _PORT[0] += 1  # a fresh rendezvous port per launch (no TIME_WAIT collisions)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_PORT[0]), "bench.py", "--gpus",
           str(n), *args]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", ["peer_ce", "peer_fused", "peer_pull", "peer_nccl"])
def test_two_gpu_modes_bit_exact(mode):
    d = _torchrun(2, "--mode", mode, "--requests", "4", "--wave", "2", "--steps", "2",
                  "--warmup", "3", "--no-match", "--no-e2e", "--no-cpu-baseline")
    assert d["parity"]["mismatched_words"] == 0 and d["parity"]["checked_bytes"] > 0
    assert d["value"] > 0 and d["link"]["peak_per_direction"] > 0


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_gpu_long_context_chunked():
    d = _torchrun(2, "--config", "3", "--block-size", "64", "--steps", "2", "--warmup", "3",
                  "--no-match", "--no-e2e", "--no-cpu-baseline")
    assert d["parity"]["mismatched_words"] == 0 and d["scaling"] == "strong"


# ---- the peer protocol on a 1-GPU box: two processes sharing cuda:0 --------
# Prefill and decode ranks are separate processes (CUDA IPC mappings of the
# other's pool / ring / flags, gloo handshake) on the same GPU.  No kernel ever
# waits for the other process there (the pull units are released by stream
# waits), so the ranks need not run concurrently.  Every destination word is
# checked by bench.py's verify kernel (a mismatch exits non-zero).

@pytest.mark.parametrize("mode", ["peer_ce", "peer_fused", "peer_pull"])
def test_shared_gpu_peer_modes_bit_exact(kvx, mode):
    d = _torchrun(2, "--share-gpu", "--mode", mode, "--requests", "4", "--wave", "2", "--steps",
                  "2", "--warmup", "3", "--no-match", "--no-e2e", "--no-cpu-baseline",
                  timeout=600)
    assert d["parity"]["mismatched_words"] == 0 and d["parity"]["checked_bytes"] > 0
    assert d["config"]["share_gpu"] and d["config"]["mode"] == mode and d["value"] > 0


@pytest.mark.parametrize("mode", ["peer_ce", "peer_pull"])
def test_shared_gpu_long_context_chunked(kvx, mode):
    d = _torchrun(2, "--share-gpu", "--mode", mode, "--config", "3", "--block-size", "64",
                  "--layers-per-chunk", "5", "--steps", "2", "--warmup", "3", "--no-match",
                  "--no-e2e", "--no-cpu-baseline", timeout=600)
    assert d["parity"]["mismatched_words"] == 0 and d["scaling"] == "strong"
    assert d["parity"]["checked_bytes"] == 42949672960  # the whole 128K request, every word


def test_shared_gpu_match_exchange(kvx):
    """Stage 1 at world 2 on one GPU.  Headline: each process its own batch
    against its own 1M-key index, every (best_len, best_id) checked against
    the oracle.  "sharded": ONE batch, each process hashes its shard of the
    requests and pushes the keys into the other's key buffer
    (kvx_xmatch_share_keys), each holds one prefill instance and kvx_xmatch
    combines them in the match kernel (remote atomics + stream flags); the
    keys and the global best are checked against the oracle."""
    d = _torchrun(2, "--share-gpu", "--mode", "peer_ce", "--requests", "2", "--wave", "2",
                  "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
                  timeout=900)
    m = d["match"]
    assert m["value"] > 0 and m["scaling"] == "weak"
    assert m["parity"]["best_match"]["requests"] == 2 * 4096
    assert m["parity"]["best_match"]["mismatched"] == 0
    assert m["sharded"]["parity"]["mismatched"] == 0 and m["sharded"]["value"] > 0
