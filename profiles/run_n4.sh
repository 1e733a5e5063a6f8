#!/bin/bash
# 4-GPU (2P->2D) runs: Config 2 (copy engine, fused) and Config 3 (layer-range shards).
for spec in "2 peer_ce" "2 peer_fused" "3 peer_ce"; do
  set -- $spec
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 4 --config $1 --mode $2 --steps 5 > gpurun_out/n4_c$1_$2.json 2> gpurun_out/n4_c$1_$2.err
  echo "n4 c$1 $2 rc=$? $(python profiles/show.py gpurun_out/n4_c$1_$2.json | head -1)"
done
