#!/bin/bash
# Round-1 measurement suite on a 2-GPU box: N=1 (Config 2 default, Config 3) and N=2 modes.
T=${TAG:-r01}
timeout 400 python bench.py > gpurun_out/${T}_n1_c2.json 2> gpurun_out/${T}_n1_c2.err; echo "n1 c2 rc=$?"
timeout 400 python bench.py --config 3 --no-match --no-cpu-baseline > gpurun_out/${T}_n1_c3.json 2> gpurun_out/${T}_n1_c3.err; echo "n1 c3 rc=$?"
for m in peer_ce peer_fused; do
  for c in 2 3; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus 2 --mode $m --config $c --steps 5 --no-match \
      > gpurun_out/${T}_n2_c${c}_$m.json 2> gpurun_out/${T}_n2_c${c}_$m.err
    echo "n2 c$c $m rc=$?"
  done
done
