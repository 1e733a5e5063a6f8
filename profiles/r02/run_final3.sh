#!/bin/bash
# Final r02 numbers on 1 GPU: default line, reference arm, Configs 1 / 3, the GPU
# suite, then the ncu evidence (profiles/run_ncu.sh).
cd "$(dirname "$0")/../.."
T=${TAG:-r02m}
mkdir -p gpurun_out/$T
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/n1_c2.json 2> gpurun_out/$T/n1_c2.err; echo "n1 c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/$T/n1_ref.json 2> gpurun_out/$T/n1_ref.err; echo "n1 ref rc=$?"
timeout 400 python bench.py --config 3 --no-match --no-cpu-baseline --no-tier > gpurun_out/$T/n1_c3.json 2> gpurun_out/$T/n1_c3.err; echo "n1 c3 rc=$?"
timeout 400 python bench.py --config 1 --no-match --no-cpu-baseline --no-tier > gpurun_out/$T/n1_c1.json 2> gpurun_out/$T/n1_c1.err; echo "n1 c1 rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/$T/gputests.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/$T/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$T/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/$T/smoke.log
TAG=$T bash profiles/run_ncu.sh; echo "ncu rc=$?"
