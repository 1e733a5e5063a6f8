#!/bin/bash
# Config 5 at N=4 (2P->2D, copy engine): block size 16..512 x KV dtype (2 / 1 bytes).
mkdir -p gpurun_out/c5
for bs in 16 32 64 128 256 512; do
  for dt in 2 1; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
      bench.py --gpus 4 --block-size $bs --dtype-bytes $dt --steps 3 --no-match --no-e2e \
      > gpurun_out/c5/n4_bs${bs}_dt${dt}.json 2>/dev/null; echo "n4 bs=$bs dt=$dt rc=$?"
  done
done
