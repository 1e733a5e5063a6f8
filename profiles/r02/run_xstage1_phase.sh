#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
make -C paper_2407_00079_b200/csrc -j8 > /dev/null 2>&1 || echo "build failed"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_xmatch.py -x -q 2>&1 | tail -2
timeout 300 $TR --master-port 29711 tests/perf/xstage1_phase.py 2>&1 | grep world= | tee gpurun_out/xstage1_phase_n${NG:-2}.txt
