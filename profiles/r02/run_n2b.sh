#!/bin/bash
# r02: 2-GPU box -- pull receiver wait modes (throughput + decode starvation), 2-GPU tests
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=${TAG:-r02e}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29700
for G in gate inline stream; do
  for LPC in 16 1; do
    P=$((P+1))
    KVX_PULL_GATE=$G timeout 600 $TR --master-port $P bench.py --gpus 2 --config 3 --layers-per-chunk $LPC --steps 5 --warmup 3 --no-match --no-cpu-baseline --no-e2e > gpurun_out/n2_c3_${G}_l${LPC}_$TAG.json 2> gpurun_out/n2_c3_${G}_l${LPC}_$TAG.err
    echo "c3 wait=$G lpc=$LPC rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/n2_c3_${G}_l${LPC}_$TAG.json').read().strip().splitlines()[-1]); print(round(d['value'],1), d['parity']['mismatched_words'])" 2>&1 | tail -1)"
  done
  P=$((P+1))
  KVX_PULL_GATE=$G timeout 300 $TR --master-port $P tests/perf/pull_starvation.py 2>&1 | grep '^{' | tee -a gpurun_out/pull_starvation_$TAG.txt
done
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_xmatch.py tests/test_gpu_store.py -x -q > gpurun_out/gputests_n2_$TAG.log 2>&1
echo "2-gpu tests rc=$?"; tail -3 gpurun_out/gputests_n2_$TAG.log
