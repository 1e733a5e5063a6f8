#!/bin/bash
# Multi-GPU bench runs: bash profiles/run_multi.sh <N> <mode...>
N=$1; shift
for m in "$@"; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus $N --mode $m --steps 5 --warmup 3 --no-match \
      > gpurun_out/m${N}_$m.json 2> gpurun_out/m${N}_$m.err
  echo "N=$N $m rc=$?"
  grep -E "PARITY|Error" gpurun_out/m${N}_$m.err | head -3
done
