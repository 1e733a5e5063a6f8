#!/bin/bash
# ncu --set full on the stage-1 kernels (Config 4 batch); 1 GPU.
set -e
mkdir -p gpurun_out
TAG=${TAG:-r01b}
MATCH="--requests 4 --wave 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
python bench.py $MATCH > gpurun_out/ncu_plain_match.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_hash|match_kernel" \
    -s 3 -c 3 -o gpurun_out/prof_match_${TAG} python bench.py $MATCH > gpurun_out/ncu_match.log 2>&1
echo done
