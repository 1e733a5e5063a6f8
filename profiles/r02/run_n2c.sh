#!/bin/bash
# r02: C-ABI NCCL streamer mode + 2-GPU stream tests; hash warps sweep (GPU 0)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29901 bench.py --gpus 2 --mode peer_nccl --steps 5 --warmup 3 --no-match --no-cpu-baseline > gpurun_out/n2_c2_nccl_r02g.json 2> gpurun_out/n2_c2_nccl_r02g.err
echo "nccl c2 rc=$? $(tail -c 300 gpurun_out/n2_c2_nccl_r02g.err | tr '\n' ' ')"
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_tier.py -x -q > gpurun_out/gputests_r02g.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gputests_r02g.log
for W in 10 11 12 13 14; do KVX_HASH_HW_WARPS=$W timeout 300 python tests/perf/hash_phase.py 2>&1 | tail -1; done | tee gpurun_out/hash_warps_r02g.txt
