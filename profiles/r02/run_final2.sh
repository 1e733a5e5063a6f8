#!/bin/bash
# r02 final code: N=1 default line, GPU suite, ncu evidence (launch list + full set)
cd "$(dirname "$0")/../.."
T=${TAG:-r02h}
mkdir -p gpurun_out/$T
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/n1_c2.json 2> gpurun_out/$T/n1_c2.err; echo "n1 c2 rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$T/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/$T/gputests.log
TAG=$T bash profiles/run_ncu.sh; echo "ncu rc=$?"
