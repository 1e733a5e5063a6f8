#!/bin/bash
# r02: request-sharded stage 1 with the key exchange inside the kernels (kvx_xmatch_hash_match)
# on a 2-GPU box: parity tests, then the N=2 bench (Config 2 + stage 1, sharded and weak).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=${TAG:-r02x}
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_xmatch.py tests/test_gpu_hash_match.py -x -q > gpurun_out/xstage1_tests_$TAG.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/xstage1_tests_$TAG.log
timeout 900 $TR --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-tier > gpurun_out/n2_c2_$TAG.json 2> gpurun_out/n2_c2_$TAG.err
echo "n2 rc=$?"; tail -c 600 gpurun_out/n2_c2_$TAG.err
