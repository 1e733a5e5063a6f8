#!/bin/bash
# ncu evidence for the bench kernels (run on the B200 box via gpurun; 1 GPU).
# Each ncu command is preceded by the same command run plainly (must exit 0).
# Outputs land in gpurun_out/; summaries go to profiles/ via summarize_ncu.py.
set -e
mkdir -p gpurun_out
SMALL="--requests 16 --wave 16 --steps 2 --warmup 3 --no-match --no-cpu-baseline --no-e2e --no-tier"
MATCH="--requests 4 --wave 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tier"
TAG=${TAG:-r01}

# 1. launch list of the transfer step (every kernel with its device time)
python bench.py $SMALL > gpurun_out/ncu_plain_small.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py $SMALL > gpurun_out/ncu_launches.log 2>&1

# 2. full set on one launch of the dominant kernel (fused paged copy)
ncu --set full --clock-control none --import-source on -k regex:copy_lsu -s 250 -c 1 \
    -o gpurun_out/prof_copy_${TAG} python bench.py $SMALL > gpurun_out/ncu_copy.log 2>&1

# 3. full set on the stage-1 kernels (block hash + prefix match, Config 4 batch)
python bench.py $MATCH > gpurun_out/ncu_plain_match.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hash_kernel|match_group|match_kernel|match_follow" \
    -s 3 -c 4 -o gpurun_out/prof_match_${TAG} python bench.py $MATCH > gpurun_out/ncu_match.log 2>&1
echo done
