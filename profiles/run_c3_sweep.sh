#!/bin/bash
# Config 3 (128K request) units: layers per unit sweep, N=1 and N=2.
for l in 1 2 4 8 16; do
  timeout 300 python bench.py --config 3 --layers-per-chunk $l --no-match --no-cpu-baseline --steps 5 > gpurun_out/c3_n1_l$l.json 2>/dev/null
  echo "n1 lpc=$l $(python profiles/show.py gpurun_out/c3_n1_l$l.json | head -1)"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus 2 --config 3 --layers-per-chunk $l --no-match --steps 5 > gpurun_out/c3_n2_l$l.json 2>/dev/null
  echo "n2 lpc=$l $(python profiles/show.py gpurun_out/c3_n2_l$l.json | head -1)"
done
