#!/bin/bash
# End-of-round numbers, N = 2 and 4 (Configs 2 and 3, stage 1 weak + sharded).
cd "$(dirname "$0")/../.."
T=${TAG:-r02f}
mkdir -p gpurun_out/$T
G=$(nvidia-smi -L | wc -l)
P=29800
for N in 2 4; do
  [ "$G" -ge "$N" ] || continue
  for c in 2 3; do
    P=$((P+1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $P bench.py --gpus $N --config $c $( [ $c = 3 ] && echo --no-match ) \
      > gpurun_out/$T/n${N}_c$c.json 2> gpurun_out/$T/n${N}_c$c.err
    echo "n$N c$c rc=$?"
  done
done
# decode-GPU starvation while a pull receiver waits for a slow prefill (2 of the GPUs)
for M in gate inline stream; do
  P=$((P+1))
  KVX_PULL_GATE=$M timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $P tests/perf/pull_starvation.py 2>&1 | grep '^{' \
    | tee -a gpurun_out/$T/pull_starvation.txt
done
