#!/bin/bash
# Config 3 with one / sixteen layers per unit: copy-engine vs pull, N=2.
for m in peer_ce peer_pull; do for l in 1 4 16; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --config 3 --mode $m --layers-per-chunk $l --steps 5 --no-match > gpurun_out/c3_${m}_l$l.json 2>/dev/null
  echo "$m lpc$l $(python profiles/show.py gpurun_out/c3_${m}_l$l.json | head -1)"
done; done
