"""Layer-wise KVCache streaming from a prefill instance to a decode instance
(stages 2 -> 3 -> 4), the real data plane behind the reference's analytic
model:

* the stream envelope and per-layer overlap -- ``on_prefill_done``
  (proj/src/sim_engine.cpp:455-470; layer-wise launch/wait per layer,
  PAPER.md:270; ``layerwise_effective_prefill``, proj/src/perf_model.cpp:73-78);
* the per-sender FIFO -- ``sender_busy_until_ms`` (proj/src/sim_engine.cpp:409-411):
  one in-order transfer queue per source GPU (``TransferEngine``).

A *chunk* is ``layers_per_chunk`` layers (K and V) of one decode wave's
blocks.  Modes:

``local_fused``  one GPU: paged -> paged copy kernel per chunk (2x payload HBM)
``local_staged`` one GPU: gather -> contiguous ring -> scatter on two streams
``peer_fused``   prefill GPU: copy kernel reads local slabs and stores straight
                 into the decode GPU's pool (CUDA IPC view) over NVLink
``peer_ce``      gather -> copy-engine P2P copy into the decode GPU's receive
                 ring -> scatter on the decode GPU; cross-process ordering by
                 stream-ordered 64-bit flags (no kernel spins)
``peer_nccl``    gather -> NCCL send/recv (torch.distributed) -> scatter

All byte movement is libkvx (sm_100a kernels / copy engines); this module only
sequences launches on CUDA streams.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import kvx


class KernelTimer:
    """CUDA-event pairs around launches of the dominant kernel (roofline)."""

    def __init__(self, enabled: bool = False):
        self.enabled = enabled
        self.pairs = []

    def start(self, stream):
        if not self.enabled:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def stop(self, stream, e0, nbytes: int):
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        self.pairs.append((e0, e1, nbytes))

    def summary(self):
        if not self.pairs:
            return None
        ms = [a.elapsed_time(b) for a, b, _ in self.pairs]
        nbytes = [n for _, _, n in self.pairs]
        return {"launches": len(ms), "avg_ms": sum(ms) / len(ms),
                "avg_algorithmic_bytes": sum(nbytes) / len(nbytes)}


def _chunks(layers: int, per: int):
    for lo in range(0, layers, per):
        yield lo, min(layers, lo + per)


class LocalStream:
    """Prefill and decode instance share one GPU (N = 1)."""

    def __init__(self, src: kvx.KVPool, dst: kvx.KVPool, mode: str = "local_fused",
                 layers_per_chunk: int = 1, ring: int = 3, max_blocks: int = 0):
        assert mode in ("local_fused", "local_staged")
        self.src, self.dst, self.mode = src, dst, mode
        self.per = layers_per_chunk
        self.dev = src.device
        self.s_main = torch.cuda.Stream(self.dev)
        self.s_scatter = torch.cuda.Stream(self.dev)
        self.ring = []
        if mode == "local_staged":
            nbytes = src.buffer_bytes(max_blocks, 0, layers_per_chunk)
            self.ring = [kvx.DeviceBuffer(nbytes, self.dev) for _ in range(ring)]
            self.ev_gather = [torch.cuda.Event() for _ in range(ring)]
            self.ev_scatter = [torch.cuda.Event() for _ in range(ring)]
            self.c = 0

    def streams(self):
        return [self.s_main, self.s_scatter]

    def send_wave(self, src_table: torch.Tensor, dst_table: torch.Tensor, timer: KernelTimer):
        n = src_table.numel()
        for lo, hi in _chunks(self.src.layers, self.per):
            nbytes = 2 * (hi - lo) * 2 * n * self.src.slab  # read + write
            if self.mode == "local_fused":
                e0 = timer.start(self.s_main)
                self.src.copy_to(self.dst, src_table, dst_table, lo, hi, stream=self.s_main)
                timer.stop(self.s_main, e0, nbytes)
                continue
            slot = self.c % len(self.ring)
            if self.c >= len(self.ring):
                self.s_main.wait_event(self.ev_scatter[slot])  # ring slot drained
            e0 = timer.start(self.s_main)
            self.src.gather(src_table, lo, hi, self.ring[slot].ptr, stream=self.s_main)
            timer.stop(self.s_main, e0, nbytes)
            self.ev_gather[slot].record(self.s_main)
            self.s_scatter.wait_event(self.ev_gather[slot])
            self.dst.scatter(dst_table, lo, hi, self.ring[slot].ptr, stream=self.s_scatter)
            self.ev_scatter[slot].record(self.s_scatter)
            self.c += 1


class PeerSender:
    """Prefill side of a prefill -> decode pair (separate processes/GPUs)."""

    def __init__(self, src: kvx.KVPool, mode: str, layers_per_chunk: int, ring: int,
                 max_blocks: int, peer_rank: int):
        assert mode in ("peer_fused", "peer_ce", "peer_nccl")
        self.src, self.mode, self.per, self.peer = src, mode, layers_per_chunk, peer_rank
        self.dev = src.device
        self.s_main = torch.cuda.Stream(self.dev)
        self.nring = ring
        self.c = 0
        self.flags = kvx.DeviceBuffer(64, self.dev)  # [0]: chunks the peer has drained
        self.flags.tensor(torch.int64).zero_()
        if mode in ("peer_ce", "peer_nccl"):
            nbytes = src.buffer_bytes(max_blocks, 0, layers_per_chunk)
            self.chunk_bytes = nbytes
            self.ring = [kvx.DeviceBuffer(nbytes, self.dev) for _ in range(ring)]
        if mode == "peer_ce":
            self.eng = kvx.TransferEngine(self.dev)
            self.tickets: List[Optional[int]] = [None] * ring
        if mode == "peer_nccl":
            self.works = [None] * ring
            self.s_comm = torch.cuda.Stream(self.dev)
            self.ev = [torch.cuda.Event() for _ in range(ring)]
        self.peer_dst: Optional[kvx.KVPool] = None

    # handshake payloads ------------------------------------------------------
    def export(self) -> dict:
        return {"flags": kvx.ipc_export(self.flags.ptr)}

    def connect(self, peer: dict, dst_desc: dict):
        self.peer_flags = kvx.ipc_open(peer["flags"], self.dev)
        if self.mode == "peer_fused":
            base = kvx.ipc_open(peer["pool"], self.dev)
            self.peer_dst = kvx.KVPool(**dst_desc, device=self.dev, base_ptr=base)
        if self.mode == "peer_ce":
            self.peer_ring = [kvx.ipc_open(h, self.dev) for h in peer["ring"]]

    def streams(self):
        s = [self.s_main]
        if self.mode == "peer_ce":
            s.append(torch.cuda.ExternalStream(self.eng.stream_handle, device=self.dev))
        if self.mode == "peer_nccl":
            s.append(self.s_comm)
        return s

    def send_wave(self, src_table: torch.Tensor, dst_table: Optional[torch.Tensor],
                  timer: KernelTimer):
        n = src_table.numel()
        for lo, hi in _chunks(self.src.layers, self.per):
            slot = self.c % self.nring
            payload = (hi - lo) * 2 * n * self.src.slab
            if self.mode == "peer_fused":
                e0 = timer.start(self.s_main)
                self.src.copy_to(self.peer_dst, src_table, dst_table, lo, hi, stream=self.s_main)
                timer.stop(self.s_main, e0, payload)  # NVLink-bound: 1x payload crosses
            elif self.mode == "peer_ce":
                if self.tickets[slot] is not None:  # gather slot free once its copy finished
                    self.eng.wait_stream(self.tickets[slot], self.s_main)
                e0 = timer.start(self.s_main)
                self.src.gather(src_table, lo, hi, self.ring[slot].ptr, stream=self.s_main)
                timer.stop(self.s_main, e0, 2 * payload)
                if self.c >= self.nring:  # receive slot free once the peer scattered c-ring
                    kvx.signal_wait(self.flags.ptr, self.c - self.nring + 1,
                                    stream=self.eng.stream_handle)
                self.tickets[slot] = self.eng.submit(self.peer_ring[slot], self.ring[slot].ptr,
                                                     payload, after_stream=self.s_main)
                self.eng.signal(self.peer_flags, self.c + 1)  # peer: chunk c landed
            else:  # peer_nccl
                if self.works[slot] is not None:
                    with torch.cuda.stream(self.s_main):
                        self.works[slot].wait()
                e0 = timer.start(self.s_main)
                self.src.gather(src_table, lo, hi, self.ring[slot].ptr, stream=self.s_main)
                timer.stop(self.s_main, e0, 2 * payload)
                self.ev[slot].record(self.s_main)
                self.s_comm.wait_event(self.ev[slot])
                with torch.cuda.stream(self.s_comm):
                    t = self.ring[slot].tensor()[:payload]
                    self.works[slot] = torch.distributed.isend(t, self.peer)
            self.c += 1

    def end_step(self):
        """peer_fused: tell the decode side everything up to chunk c landed."""
        if self.mode == "peer_fused":
            kvx.signal_write(self.peer_flags, self.c, stream=self.s_main)


class PeerReceiver:
    """Decode side of a pair: owns the decode pool, receive ring and flags."""

    def __init__(self, dst: kvx.KVPool, mode: str, layers_per_chunk: int, ring: int,
                 max_blocks: int, peer_rank: int):
        self.dst, self.mode, self.per, self.peer = dst, mode, layers_per_chunk, peer_rank
        self.dev = dst.device
        self.s_main = torch.cuda.Stream(self.dev)
        self.nring = ring
        self.c = 0
        self.flags = kvx.DeviceBuffer(64, self.dev)  # [0]: chunks landed here
        self.flags.tensor(torch.int64).zero_()
        if mode in ("peer_ce", "peer_nccl"):
            nbytes = dst.buffer_bytes(max_blocks, 0, layers_per_chunk)
            self.ring = [kvx.DeviceBuffer(nbytes, self.dev) for _ in range(ring)]
        if mode == "peer_nccl":
            self.works = [None] * ring

    def export(self) -> dict:
        out = {"flags": kvx.ipc_export(self.flags.ptr)}
        if self.mode == "peer_fused":
            out["pool"] = kvx.ipc_export(self.dst.base)
        if self.mode == "peer_ce":
            out["ring"] = [kvx.ipc_export(b.ptr) for b in self.ring]
        return out

    def connect(self, peer: dict):
        self.peer_flags = kvx.ipc_open(peer["flags"], self.dev)

    def streams(self):
        return [self.s_main]

    def recv_wave(self, dst_table: torch.Tensor, n_src: int, timer: KernelTimer):
        n = dst_table.numel()
        for lo, hi in _chunks(self.dst.layers, self.per):
            slot = self.c % self.nring
            payload = (hi - lo) * 2 * n * self.dst.slab
            if self.mode == "peer_ce":
                kvx.signal_wait(self.flags.ptr, self.c + 1, stream=self.s_main)
                e0 = timer.start(self.s_main)
                self.dst.scatter(dst_table, lo, hi, self.ring[slot].ptr, stream=self.s_main)
                timer.stop(self.s_main, e0, 2 * payload)
                kvx.signal_write(self.peer_flags, self.c + 1, stream=self.s_main)
            elif self.mode == "peer_nccl":
                with torch.cuda.stream(self.s_main):
                    t = self.ring[slot].tensor()[:payload]
                    torch.distributed.irecv(t, self.peer).wait()
                e0 = timer.start(self.s_main)
                self.dst.scatter(dst_table, lo, hi, self.ring[slot].ptr, stream=self.s_main)
                timer.stop(self.s_main, e0, 2 * payload)
            self.c += 1

    def end_step(self):
        if self.mode == "peer_fused":
            # everything the sender issued so far has landed in our pool
            kvx.signal_wait(self.flags.ptr, self.c, stream=self.s_main)

    def count_fused_chunks(self, n_chunks: int):
        self.c += n_chunks
