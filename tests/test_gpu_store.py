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


# ---- asynchronous, engine-driven migration (kvx_store_migrate_submit/wait) ----
# The reference engine's two migration KATs (proj/tests/test_engine.cpp:170-231)
# replayed with real bytes: a per-sender FIFO of transfers
# (sim_engine.cpp:409-411), the residency check at BEGIN (:605-639) and the
# landing at DONE (:641-650).

def test_async_migration_replicates_prefix(kvx):
    """test_engine.cpp:170-189: instance 0 holds the chain {1,2,3,4}; the
    migration replicates it onto instance 1 with the bytes; afterwards the
    whole prefix is reusable there, so replicating it again copies nothing."""
    from paper_2407_00079_b200.store import KVStore
    a = KVStore(4, 16, 8, 128, 2, 8, 0)
    b = KVStore(4, 16, 8, 128, 2, 8, 0)
    a.pool.fill_synthetic(3)
    chain = [1, 2, 3, 4]
    a_slots = a.put(chain)
    t = a.migrate_submit(b, chain)
    assert a.migrate_wait(t) == 4
    b_slots = b.get(chain)
    assert (b_slots >= 0).all()
    assert b.pool.verify(_t(b_slots), 3, _t(a_slots), 0, 4).item() == 0
    t2 = a.migrate_submit(b, chain)  # replication growth: already resident at b
    assert a.migrate_wait(t2) == 0
    assert np.array_equal(b.get(chain), b_slots)


def test_async_migration_fifo_abort(kvx):
    """test_engine.cpp:191-231: two migrations of the hot prefix {1,2,3,4}
    queue on instance 0's sender FIFO; a fresh chain {11,...,14} arriving at
    instance 0 evicts the hot blocks before the SECOND begins.  The first
    (already begun) completes with the right bytes, the second aborts and
    lands nothing: migrations_completed == 1, migrations_aborted == 1.  The
    evicted slots the first copy still reads are not handed to the fresh
    chain until that copy is done."""
    from paper_2407_00079_b200.kvx import TransferAborted
    from paper_2407_00079_b200.store import KVStore
    L = 4
    a = KVStore(L, 16, 8, 128, 2, 8, 0)
    b = KVStore(L, 16, 8, 128, 2, 16, 0)
    other = kvx.KVPool(L, 16, 8, 128, 2, 8, 0)
    a.pool.fill_synthetic(3)
    other.fill_synthetic(9)
    torch.cuda.synchronize()
    hot = [1, 2, 3, 4]
    a_slots = a.put(hot)
    gate = torch.cuda.Stream(0)  # holds the first transfer on the link (~0.2 s)
    with torch.cuda.stream(gate):
        torch.cuda._sleep(400_000_000)
    t1 = a.migrate_submit(b, hot, after_stream=gate)  # begins now, copy behind the gate
    t2 = a.migrate_submit(b, hot)                     # queued behind t1 on the FIFO
    assert a.migrate_query(t1) == "pending" and a.migrate_query(t2) == "pending"
    # r3 at instance 0: the hot blocks are evicted, the fresh chain's KV is written
    a.evict(hot)
    fresh = a.put([11, 12, 13, 14])
    assert not set(fresh.tolist()) & set(a_slots.tolist())  # pinned slots not reused yet
    other.copy_to(a.pool, _t(np.arange(4)), _t(fresh), 0, L)  # r3's prefill writes its KV
    assert a.migrate_wait(t1) == 4
    b_slots = b.get(hot)
    assert b.pool.verify(_t(b_slots), 3, _t(a_slots), 0, L).item() == 0  # the hot KV, intact
    with pytest.raises(TransferAborted):
        a.migrate_wait(t2)
    assert np.array_equal(b.get(hot), b_slots)  # the aborted one landed nothing
    # the deferred slots are free again once the first copy is done
    assert sorted(a.put([100, 101, 102, 103]).tolist()) == sorted(a_slots.tolist())
    with pytest.raises(kvx.ValidationError):
        a.migrate_wait(t1)  # collected
