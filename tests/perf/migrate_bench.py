"""Throughput of the migration data path (hot-spot replication, SURVEY 8(f)
row 2): kvx_store_migrate of a 1,024-block chain (16K tokens of LLaMA2-70B
KV, 5.37 GB) from one KV store to another -- on the same GPU and, when there
are two, across NVLink -- through the public API (residency check, slot
allocation, index insert, paged->paged copy), destination evicted between
repetitions.  Every copied word is verified once before timing."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00079_b200 import kvx  # noqa: E402
from paper_2407_00079_b200.store import KVStore  # noqa: E402

L, BS, H, D, DT = 80, 16, 8, 128, 2
SLOTS, N, REPS = 1536, 1024, 10
payload = N * L * 2 * BS * H * D * DT


def run(dev_b: int):
    a = KVStore(L, BS, H, D, DT, SLOTS, 0)
    b = KVStore(L, BS, H, D, DT, SLOTS, dev_b)
    a.pool.fill_synthetic(5)
    torch.cuda.synchronize(0)
    chain = (np.arange(N, dtype=np.int64) + 7) << 16
    a_slots = a.put(chain)
    assert a.migrate_to(b, chain) == N
    b_slots = b.get(chain)
    ctr = torch.zeros(1, dtype=torch.int64, device=f"cuda:{dev_b}")
    with torch.cuda.device(dev_b):
        b.pool.verify(torch.as_tensor(b_slots, device=f"cuda:{dev_b}"), 5,
                      torch.as_tensor(a_slots, device=f"cuda:{dev_b}"), 0, L, counter=ctr,
                      stream=torch.cuda.current_stream(dev_b))
        torch.cuda.synchronize(dev_b)
    assert ctr.item() == 0, "migration parity"
    times = []
    for _ in range(REPS + 2):
        b.evict(chain)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(dev_b)
        t0 = time.perf_counter()
        n = a.migrate_to(b, chain)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(dev_b)
        times.append(time.perf_counter() - t0)
        assert n == N
    ms = float(np.median(times[2:])) * 1e3
    return {"dst_gpu": dev_b, "blocks": N, "payload_bytes": payload, "ms_median": ms,
            "gb_per_s": payload / (ms / 1e3) / 1e9}


res = [run(0)]
if torch.cuda.device_count() > 1:
    res.append(run(1))
print(json.dumps({"metric": "migration (hot-spot replication) payload GB/s", "runs": res}))
