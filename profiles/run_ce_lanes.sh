#!/bin/bash
# PEER_CE lanes: Config 2 and Config 3 at 1 and 16 layers per unit, N=2.
for spec in "2 1" "3 1" "3 16"; do
  set -- $spec
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --config $1 --layers-per-chunk $2 --steps 5 --no-match > gpurun_out/ce_c$1_l$2.json 2> gpurun_out/ce_c$1_l$2.err
  echo "c$1 lpc$2 rc=$? $(python profiles/show.py gpurun_out/ce_c$1_l$2.json | head -1)"
done
timeout 600 python -m pytest tests/test_gpu_stream.py -q 2>&1 | tail -1
