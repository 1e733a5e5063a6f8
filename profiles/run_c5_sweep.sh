#!/bin/bash
# Config 5: block size 16..512 x KV dtype (fp16/bf16 = 2 bytes, fp8 = 1 byte), Config-2 request
# structure, N=1 (local fused) and N=2 (1P->1D copy engine).  One JSON line per run.
mkdir -p gpurun_out/c5
for bs in 16 32 64 128 256 512; do
  for dt in 2 1; do
    timeout 300 python bench.py --block-size $bs --dtype-bytes $dt --steps 3 --no-match --no-cpu-baseline --no-e2e \
      > gpurun_out/c5/n1_bs${bs}_dt${dt}.json 2>/dev/null; echo "n1 bs=$bs dt=$dt rc=$?"
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus 2 --block-size $bs --dtype-bytes $dt --steps 3 --no-match --no-e2e \
      > gpurun_out/c5/n2_bs${bs}_dt${dt}.json 2>/dev/null; echo "n2 bs=$bs dt=$dt rc=$?"
  done
done
