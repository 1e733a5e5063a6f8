#!/bin/bash
# r02: N=1 bench (default config) + stage-1 parity at Config 4 scale + GPU suite.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=${TAG:-r02a}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1_$TAG.json 2> gpurun_out/bench_n1_$TAG.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench_n1_$TAG.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$TAG.log 2>&1
echo "gpu suite rc=$?"; tail -5 gpurun_out/gputests_$TAG.log
