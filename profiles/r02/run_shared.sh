#!/bin/bash
# r02: peer protocol as two processes sharing one GPU, then the full GPU suite.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpus.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_xmatch.py -k shared -x -q \
  > gpurun_out/shared.log 2>&1
echo "shared rc=$?" >> gpurun_out/shared.log
tail -3 gpurun_out/shared.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
echo "gpu suite rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
