"""Cross-GPU best prefix match without a collective (kvx_xmatch_*): bit-exact
against find_best_prefix_match over all instances on one GPU, 2 GPUs under
torchrun (SURVEY 8(e) case ii; proj/src/conductor.cpp:57-73 tie-break)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_xmatch_two_gpus_bit_exact():
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29537", "tests/xmatch_worker.py"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "XMATCH OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_xmatch_shared_gpu_bit_exact(kvx):
    """The same worker as two processes sharing cuda:0 (gloo handshake): the
    remote atomics and flags go through CUDA IPC mappings of the other
    process's buffers on the same device."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "tests/xmatch_worker.py"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "KVX_SHARE_GPU": "1"})
    assert r.returncode == 0 and "XMATCH OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_xmatch_fused_stage1_two_gpus():
    """Request-sharded hash with the keys stored into every GPU's buffer from
    the hash kernel, and each GPU's match kernel following them."""
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29557",
           "tests/xmatch_stage1_worker.py"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "XMATCH STAGE1 OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_xmatch_fused_stage1_refuses_shared_gpu(kvx):
    """Two processes on one GPU: the fused call must refuse (its match kernel
    would wait on the other process's hash kernel on the same GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29567",
           "tests/xmatch_stage1_worker.py"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "KVX_SHARE_GPU": "1"})
    assert r.returncode == 0 and "XMATCH STAGE1 OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_xmatch_validation(kvx):
    with pytest.raises(kvx.ValidationError):
        kvx.XMatch(0, 2, 2, 16)  # rank out of range
    x = kvx.XMatch(0, 0, 2, 16)
    with pytest.raises(kvx.ValidationError):
        x.connect(b"\\0" * 8)  # truncated blob
    idx = kvx.BlockIndex(0, 16)
    keys = torch.zeros(4, dtype=torch.int64, device="cuda:0")
    off = torch.tensor([0, 4], dtype=torch.int64, device="cuda:0")
    with pytest.raises(kvx.ValidationError):
        x.run([idx], [0], keys, off)  # rank 1 never connected
