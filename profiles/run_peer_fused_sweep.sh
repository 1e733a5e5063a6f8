#!/bin/bash
# peer_fused (SM stores into the peer pool over NVLink): copy kernel variants, N=2.
run() {
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --mode peer_fused --steps 5 --no-match --no-e2e "$@" > gpurun_out/pf.json 2>/dev/null
  python profiles/show.py gpurun_out/pf.json | sed -n 2p
}
echo "lsu 4/SM: $(run)"
echo "lsu 2/SM: $(KVX_LSU_CTAS=2 run)"
echo "lsu 1/SM: $(KVX_LSU_CTAS=1 run)"
echo "tma 2/SM: $(run --copy-impl tma)"
echo "tma 1/SM 6-stage: $(KVX_TMA_CFG=1 run --copy-impl tma)"
