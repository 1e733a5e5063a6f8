#!/bin/bash
# End-of-round numbers, 1 GPU: default line (Config 2 + stage 1 + DRAM tier), the
# reference arm, Config 1 / Config 3, then the ncu evidence (profiles/run_ncu.sh).
cd "$(dirname "$0")/../.."
T=${TAG:-r02f}
mkdir -p gpurun_out/$T
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/$T/n1_c2.json 2> gpurun_out/$T/n1_c2.err; echo "n1 c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/$T/n1_ref.json 2> gpurun_out/$T/n1_ref.err; echo "n1 ref rc=$?"
timeout 400 python bench.py --config 3 --no-match --no-cpu-baseline --no-tier > gpurun_out/$T/n1_c3.json 2> gpurun_out/$T/n1_c3.err; echo "n1 c3 rc=$?"
timeout 400 python bench.py --config 1 --no-match --no-cpu-baseline --no-tier > gpurun_out/$T/n1_c1.json 2> gpurun_out/$T/n1_c1.err; echo "n1 c1 rc=$?"
TAG=$T bash profiles/run_ncu.sh; echo "ncu rc=$?"
