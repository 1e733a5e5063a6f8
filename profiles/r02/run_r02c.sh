#!/bin/bash
cd "$(dirname "$0")/../.."
bash profiles/r02/run_match.sh
bash profiles/r02/run_dropin.sh 2>&1 | tee gpurun_out/dropin_latency.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r02c.log 2>&1
echo "gpu suite rc=$?"; tail -5 gpurun_out/gputests_r02c.log
