"""GPU parity: paged pool generator, K3 gather, K5 scatter, fused paged copy
and the transfer engine (through the C ABI) against the C restatement
(oracle/kvx_oracle.c).  Bytes must be identical (memcmp)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
IMPLS = ["lsu", "tma"]


def _t(a, dtype=torch.int32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def _host(pool):
    torch.cuda.synchronize()
    return pool.tensor_view().cpu().numpy()


@pytest.fixture(autouse=True)
def _reset_impl(kvx):
    yield
    kvx.set_copy_impl("lsu")


@pytest.mark.parametrize("bs,heads,dim,dtype_bytes", [(16, 8, 128, 2), (5, 2, 16, 1),
                                                      (3, 1, 8, 2), (64, 8, 128, 1)])
def test_fill_synthetic_matches_oracle(kvx, oracle_lib, bs, heads, dim, dtype_bytes):
    L, slots = 3, 7
    pool = kvx.KVPool(L, bs, heads, dim, dtype_bytes, slots, 0)
    pool.fill_synthetic(11)
    want = np.zeros(pool.nbytes, dtype=np.uint8)
    oracle_lib.fill_pool(want, 11, L, slots, pool.slab)
    assert np.array_equal(_host(pool), want)


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("bs,dtype_bytes", [(16, 2), (16, 1), (32, 2), (5, 2), (128, 2), (512, 1)])
def test_gather_scatter_copy_vs_oracle(kvx, oracle_lib, impl, bs, dtype_bytes):
    kvx.set_copy_impl(impl)
    rng = np.random.default_rng(bs * 7 + dtype_bytes)
    L, heads, dim = 4, 8, 128 if bs < 256 else 16
    src_slots, dst_slots, n = 23, 31, 13
    src = kvx.KVPool(L, bs, heads, dim, dtype_bytes, src_slots, 0)
    dst = kvx.KVPool(L, bs, heads, dim, dtype_bytes, dst_slots, 0)
    src.fill_synthetic(1)
    dst.tensor_view().zero_()
    src_table = rng.integers(0, src_slots, size=n).astype(np.int32)  # repeats allowed (shared prefix)
    used = np.zeros(dst_slots, dtype=np.uint8)
    used[rng.choice(dst_slots, 6, replace=False)] = 1
    got_n, dst_table = oracle_lib.alloc_lowest_free(used, n)
    assert got_n == n
    lo, hi = 1, 4
    buf = torch.zeros(src.buffer_bytes(n, lo, hi), dtype=torch.uint8, device=DEV)
    src.gather(_t(src_table), lo, hi, buf.data_ptr())
    src_h = _host(src)
    want_buf = np.zeros(buf.numel(), dtype=np.uint8)
    oracle_lib.gather(src_h, src_slots, src.slab, src_table, lo, hi, want_buf)
    torch.cuda.synchronize()
    assert np.array_equal(buf.cpu().numpy(), want_buf)

    dst.scatter(_t(dst_table), lo, hi, buf.data_ptr())
    want_dst = np.zeros(dst.nbytes, dtype=np.uint8)
    oracle_lib.scatter(want_dst, dst_slots, dst.slab, dst_table, lo, hi, want_buf)
    assert np.array_equal(_host(dst), want_dst)

    dst2 = kvx.KVPool(L, bs, heads, dim, dtype_bytes, dst_slots, 0)
    dst2.tensor_view().zero_()
    src.copy_to(dst2, _t(src_table), _t(dst_table), lo, hi)
    assert np.array_equal(_host(dst2), want_dst)

    ctr = dst2.verify(_t(dst_table), 1, _t(src_table), lo, hi)
    assert ctr.item() == 0
    ctr = dst2.verify(_t(dst_table), 2, _t(src_table), lo, hi)  # wrong source id -> all differ
    assert ctr.item() == (hi - lo) * 2 * n * src.slab // 8


def test_empty_and_bad_ranges(kvx):
    pool = kvx.KVPool(2, 16, 8, 128, 2, 4, 0)
    empty = torch.zeros(0, dtype=torch.int32, device=DEV)
    pool.gather(empty, 0, 2, 16)  # n == 0 is a no-op
    with pytest.raises(kvx.ValidationError):
        pool.gather(_t([0]), 1, 3, 16)
    with pytest.raises(kvx.ValidationError):
        kvx.KVPool(2, 16, 8, 128, 3, 4, 0)


@pytest.mark.parametrize("impl", IMPLS)
def test_out_of_range_table_entries_are_skipped(kvx, impl):
    """Entries outside [0, slots) (incl. negative) never write outside a pool:
    those units are skipped, the rest copied, and kvx_copy_check reports it."""
    kvx.set_copy_impl(impl)
    src = kvx.KVPool(2, 16, 8, 128, 2, 6, 0)
    dst = kvx.KVPool(2, 16, 8, 128, 2, 6, 0)
    src.fill_synthetic(5)
    guard = dst.tensor_view()
    guard.fill_(0xAB)
    kvx.copy_check()  # clean slate
    src.copy_to(dst, _t([0, 9, 2, -1]), _t([1, 2, 6, 3]), 0, 2)
    with pytest.raises(kvx.ValidationError):
        kvx.copy_check()
    kvx.copy_check()  # the flag was cleared
    ctr = dst.verify(_t([1]), 5, _t([0]), 0, 2)  # the valid unit landed
    assert ctr.item() == 0
    host = _host(dst).reshape(2, 2, 6, -1)
    assert (host[:, :, [0, 2, 3, 4, 5]] == 0xAB).all()  # skipped units wrote nothing
    buf = torch.zeros(3 * 2 * 2 * src.slab, dtype=torch.uint8, device=DEV)
    src.gather(_t([0, 6, 1]), 0, 2, buf.data_ptr())
    with pytest.raises(kvx.ValidationError):
        kvx.copy_check()


def test_transfer_engine_local(kvx):
    eng = kvx.TransferEngine(0)
    a = torch.arange(1 << 20, dtype=torch.int64, device=DEV)
    b = torch.zeros_like(a)
    c = torch.zeros_like(a)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a.mul_(3)
    t1 = eng.submit(b.data_ptr(), a.data_ptr(), a.numel() * 8, after_stream=s)
    t2 = eng.submit(c.data_ptr(), b.data_ptr(), a.numel() * 8)  # FIFO: runs after t1
    eng.wait(t2)
    assert eng.done(t1) and eng.done(t2)
    assert torch.equal(c, torch.arange(1 << 20, dtype=torch.int64, device=DEV) * 3)
    flag = torch.zeros(1, dtype=torch.int64, device=DEV)
    eng.signal(flag.data_ptr(), 5)
    s2 = torch.cuda.Stream()
    kvx.kvx.signal_wait(flag.data_ptr(), 5, stream=s2)
    with torch.cuda.stream(s2):
        d = c + 1
    s2.synchronize()
    assert flag.item() == 5 and d[1].item() == 4
    with pytest.raises(kvx.ValidationError):
        eng.wait(10**9)


@pytest.mark.parametrize("impl", IMPLS)
def test_config1_full_size_roundtrip(kvx, impl):
    """Config 1 at full size: one 8K-token request, 512 blocks x 80 layers,
    fp16, bs=16 (2,684,354,560 B).  Staged gather -> buffer -> scatter and the
    fused paged copy; every destination word is checked by the verify kernel."""
    kvx.set_copy_impl(impl)
    L, bs, n = 80, 16, 512
    rng = np.random.default_rng(1)
    src = kvx.KVPool(L, bs, 8, 128, 2, 1024, 0)
    dst = kvx.KVPool(L, bs, 8, 128, 2, 600, 0)
    src.fill_synthetic(0)
    st = _t(rng.permutation(1024)[:n])
    dt = _t(np.arange(n))
    buf = torch.empty(src.buffer_bytes(n, 0, L), dtype=torch.uint8, device=DEV)
    assert buf.numel() == 2684354560
    src.gather(st, 0, L, buf.data_ptr())
    dst.scatter(dt, 0, L, buf.data_ptr())
    assert dst.verify(dt, 0, st, 0, L).item() == 0
    dst.tensor_view().zero_()
    src.copy_to(dst, st, dt, 0, L)
    assert dst.verify(dt, 0, st, 0, L).item() == 0
