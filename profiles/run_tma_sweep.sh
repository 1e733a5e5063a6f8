#!/bin/bash
# TMA bulk-copy pipeline shapes (KVX_TMA_CFG) vs the LSU copy kernel, N=1 Config 2.
for cfg in 0 4 5; do
  KVX_TMA_CFG=$cfg timeout 300 python bench.py --copy-impl tma --requests 16 --steps 5 --no-match --no-cpu-baseline --no-e2e > gpurun_out/tma_$cfg.json 2>/dev/null
  echo "tma cfg=$cfg $(python profiles/show.py gpurun_out/tma_$cfg.json | sed -n 2p)"
done
timeout 300 python bench.py --copy-impl lsu --requests 16 --steps 5 --no-match --no-cpu-baseline --no-e2e > gpurun_out/lsu.json 2>/dev/null
echo "lsu $(python profiles/show.py gpurun_out/lsu.json | sed -n 2p)"
