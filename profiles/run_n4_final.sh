#!/bin/bash
# 4-GPU (2P->2D) final runs: Config 2 (default copy engine) and Config 3 (default pull).
for c in 2 3; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 4 --config $c --steps 5 > gpurun_out/final_n4_c$c.json 2> gpurun_out/final_n4_c$c.err
  echo "n4 c$c rc=$? $(python profiles/show.py gpurun_out/final_n4_c$c.json | head -1)"
  python profiles/show.py gpurun_out/final_n4_c$c.json | grep match
done
