"""GPU parity of the KV store and the migration data path (hot-spot
replication): put/get/evict semantics, bytes landed bit-exact, landing skips
resident blocks (insert_replicated, proj/src/kvcache.cpp:140), and the abort
rule (proj/src/sim_engine.cpp:605-639): any source block evicted -> the whole
migration is refused and nothing changes."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int32, device="cuda:0")


@pytest.fixture
def stores(kvx):
    from paper_2407_00079_b200.store import KVStore
    a = KVStore(4, 16, 8, 128, 2, 64, 0)
    b = KVStore(4, 16, 8, 128, 2, 80, 0)
    a.pool.fill_synthetic(7)
    b.pool.tensor_view().zero_()
    return a, b


def test_put_get_evict(stores):
    a, _ = stores
    keys = np.arange(100, 130, dtype=np.int64) * 7919
    slots = a.put(keys)
    assert slots.tolist() == list(range(30))  # lowest free slots, in order
    assert a.put(keys[:5]).tolist() == list(range(5))  # re-put keeps slots
    assert np.array_equal(a.get(keys), slots)
    a.evict(keys[3:6])
    got = a.get(keys)
    assert (got[3:6] == -1).all() and np.array_equal(got[6:], slots[6:])
    assert a.put([42]).tolist() == [3]  # freed slots are reused lowest-first


def test_migrate_bytes_and_landing(stores, kvx):
    from paper_2407_00079_b200.kvx import TransferAborted
    a, b = stores
    chain = (np.arange(40, dtype=np.int64) + 1) << 20
    a_slots = a.put(chain)
    b.put(chain[10:15])  # destination already holds part of the range
    before = b.get(chain)
    n = a.migrate_to(b, chain[5:30])
    assert n == 20  # 25 requested, 5 already resident at b
    b_slots = b.get(chain[5:30])
    assert (b_slots >= 0).all()
    assert np.array_equal(b_slots[5:10], before[10:15])  # resident ones untouched
    fresh = np.r_[0:5, 10:25]
    ctr = b.pool.verify(_t(b_slots[fresh]), 7, _t(a_slots[5:30][fresh]), 0, 4)
    assert ctr.item() == 0
    # abort: one source block evicted -> refused, destination unchanged
    a.evict(chain[33:34])
    snapshot = b.get(chain)
    with pytest.raises(TransferAborted):
        a.migrate_to(b, chain[30:40])
    assert np.array_equal(b.get(chain), snapshot)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_migrate_across_gpus(kvx):
    from paper_2407_00079_b200.store import KVStore
    a = KVStore(3, 16, 8, 128, 2, 32, 0)
    b = KVStore(3, 16, 8, 128, 2, 32, 1)
    a.pool.fill_synthetic(2)
    chain = np.arange(12, dtype=np.int64) + 900
    a_slots = a.put(chain)
    assert a.migrate_to(b, chain) == 12
    b_slots = b.get(chain)
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda:1")
    with torch.cuda.device(1):
        b.pool.verify(torch.as_tensor(b_slots, device="cuda:1"), 2,
                      torch.as_tensor(a_slots, device="cuda:1"), 0, 3, counter=ctr,
                      stream=torch.cuda.current_stream(1))
        torch.cuda.synchronize(1)
    assert ctr.item() == 0


def test_repeated_keys_take_one_slot(stores):
    a, b = stores
    slots = a.put([5, 6, 5, 7, 6, 5])
    assert slots.tolist() == [0, 1, 0, 2, 1, 0]
    a.evict([6, 6, 5])  # a key repeated in one evict frees its slot once
    assert a.put([8, 9, 10]).tolist() == [0, 1, 3]
    a_slots = a.put([11, 12])
    assert b.put([]).tolist() == []
    assert a.migrate_to(b, [11, 12, 11]) == 2  # duplicates land once
    assert b.get([11, 12]).tolist() == [0, 1]
    ctr = b.pool.verify(_t([0, 1]), 7, _t(a_slots), 0, 4)
    assert ctr.item() == 0
