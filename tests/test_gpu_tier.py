"""GPU parity of the CPU-DRAM KVCache tier (kvx_pool_create_host) and the
layer-wise load / store with launch / wait per layer (kvx_layer_*; PAPER.md:270,
the byte path behind proj/src/perf_model.cpp:73-85): memcmp against the C
restatement's paged copy (oracle kvo_copy_paged) on the same seeded inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int32, device=DEV)


def _pools(kvx, L, bs, db, host_slots, dev_slots):
    host = kvx.KVPool(L, bs, 8, 128, db, host_slots, 0, host=True)
    dev = kvx.KVPool(L, bs, 8, 128, db, dev_slots, 0)
    return host, dev


def test_host_pool_fill_matches_oracle(kvx, oracle_lib):
    host = kvx.KVPool(3, 16, 8, 128, 2, 20, 0, host=True)
    host.fill_synthetic(4)  # a GPU kernel writing DRAM over PCIe
    torch.cuda.synchronize()
    want = np.zeros(host.nbytes, dtype=np.uint8)
    oracle_lib.fill_pool(want, 4, 3, 20, host.slab)
    assert np.array_equal(host.host_array(), want)


@pytest.mark.parametrize("bs,db", [(16, 2), (5, 2), (64, 1)])
def test_layerwise_load_store_vs_oracle(kvx, oracle_lib, bs, db):
    L, hs, ds, n = 6, 90, 70, 37
    host, dev = _pools(kvx, L, bs, db, hs, ds)
    host.fill_synthetic(2)
    dev.tensor_view().zero_()
    torch.cuda.synchronize()  # the fill / zero run on the current stream, the loads on io's
    rng = np.random.default_rng(bs)
    ht = rng.permutation(hs)[:n].astype(np.int32)
    dt = rng.permutation(ds)[:n].astype(np.int32)
    io = kvx.LayerIO(0, L)
    s = torch.cuda.Stream(0)
    io.load(host, _t(ht), dev, _t(dt), 0, L, after=s)
    for layer in range(L):  # "wait before each layer's attention"
        io.wait_layer(layer, s)
    s.synchronize()
    torch.cuda.synchronize()
    want = np.zeros(dev.nbytes, dtype=np.uint8)
    oracle_lib.copy_paged(host.host_array().copy(), hs, ht, want, ds, dt, dev.slab, 0, L)
    assert np.array_equal(dev.tensor_view().cpu().numpy(), want)
    # store back layer by layer into other DRAM slots
    back = kvx.KVPool(L, bs, 8, 128, db, hs, 0, host=True)
    back.host_array()[:] = 0
    ht2 = rng.permutation(hs)[:n].astype(np.int32)
    for layer in range(L):
        io.store(dev, _t(dt), back, _t(ht2), layer, layer + 1, after=s)
    io.wait_stores()  # host-blocking
    want2 = np.zeros(back.nbytes, dtype=np.uint8)
    oracle_lib.copy_paged(want, ds, dt, want2, hs, ht2, dev.slab, 0, L)
    assert np.array_equal(back.host_array(), want2)
    assert back.verify(_t(ht2), 2, _t(ht), 0, L).item() == 0


def test_layer_wait_orders_consumer(kvx):
    """A consumer on another stream that waits for layer l sees layer l's KV
    (verify kernel reads the device pool right after the wait)."""
    L, hs, ds, n = 8, 600, 600, 512
    host, dev = _pools(kvx, L, 16, 2, hs, ds)
    host.fill_synthetic(9)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    ht, dt = _t(rng.permutation(hs)[:n]), _t(rng.permutation(ds)[:n])
    io = kvx.LayerIO(0, L)
    for rep in range(3):
        dev.tensor_view().zero_()
        torch.cuda.synchronize()
        s = torch.cuda.Stream(0)
        bad = torch.zeros(1, dtype=torch.int64, device=DEV)
        io.load(host, ht, dev, dt, 0, L, after=s)
        for layer in range(L):
            io.wait_layer(layer, s)
            dev.verify(dt, 9, ht, layer, layer + 1, counter=bad, stream=s)
        s.synchronize()
        assert bad.item() == 0


def test_layer_io_validation(kvx):
    host, dev = _pools(kvx, 2, 16, 2, 8, 8)
    io = kvx.LayerIO(0, 2)
    t = _t(np.arange(4))
    with pytest.raises(kvx.ValidationError):
        io.load(dev, t, host, t, 0, 2)  # wrong direction
    with pytest.raises(kvx.ValidationError):
        io.load(host, t, dev, t, 0, 3)  # past max_layers
    with pytest.raises(kvx.ValidationError):
        io.store(host, t, dev, t, 0, 1)


def test_contiguous_range_load_store_vs_oracle(kvx, oracle_lib):
    """Contiguous block runs move by copy engine (kvx_layer_*_range): the
    same bytes as the paged copy of the equivalent ascending tables."""
    L, hs, ds, n = 5, 60, 50, 17
    host, dev = _pools(kvx, L, 16, 2, hs, ds)
    host.fill_synthetic(6)
    dev.tensor_view().zero_()
    torch.cuda.synchronize()
    io = kvx.LayerIO(0, L)
    s = torch.cuda.Stream(0)
    io.load_range(host, 31, dev, 9, n, 1, L, after=s)  # layers [1, L)
    io.wait_layer(L - 1, s)
    s.synchronize()
    torch.cuda.synchronize()
    want = np.zeros(dev.nbytes, dtype=np.uint8)
    oracle_lib.copy_paged(host.host_array().copy(), hs, np.arange(31, 31 + n, dtype=np.int32),
                          want, ds, np.arange(9, 9 + n, dtype=np.int32), dev.slab, 1, L)
    assert np.array_equal(dev.tensor_view().cpu().numpy(), want)
    back = kvx.KVPool(L, 16, 8, 128, 2, hs, 0, host=True)
    back.host_array()[:] = 0
    io.store_range(dev, 9, back, 0, n, 0, L, after=s)
    io.wait_stores()
    want2 = np.zeros(back.nbytes, dtype=np.uint8)
    oracle_lib.copy_paged(want, ds, np.arange(9, 9 + n, dtype=np.int32), want2, hs,
                          np.arange(0, n, dtype=np.int32), dev.slab, 0, L)
    assert np.array_equal(back.host_array(), want2)
    with pytest.raises(kvx.ValidationError):
        io.load_range(host, hs - 3, dev, 0, 4, 0, 1)  # past the DRAM pool
