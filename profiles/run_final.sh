#!/bin/bash
# Final round numbers on one box: N=1 (Config 2 default line, Config 3, Config 5 sweep)
# and, when the box has >= 2 / 4 GPUs, the default N=2 / N=4 lines for Configs 2 and 3.
T=${TAG:-r01g}
mkdir -p gpurun_out/$T gpurun_out/c5_$T
G=$(nvidia-smi -L | wc -l)
timeout 400 python bench.py > gpurun_out/$T/n1_c2.json 2> gpurun_out/$T/n1_c2.err; echo "n1 c2 rc=$?"
timeout 400 python bench.py --config 3 --no-match --no-cpu-baseline > gpurun_out/$T/n1_c3.json 2> gpurun_out/$T/n1_c3.err; echo "n1 c3 rc=$?"
for N in 2 4; do
  [ "$G" -ge "$N" ] || continue
  for c in 2 3; do
    timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus $N --config $c \
      > gpurun_out/$T/n${N}_c$c.json 2> gpurun_out/$T/n${N}_c$c.err
    echo "n$N c$c rc=$?"
  done
done
for bs in 16 32 64 128 256 512; do
  for dt in 2 1; do
    timeout 300 python bench.py --block-size $bs --dtype-bytes $dt --steps 3 --no-match --no-cpu-baseline --no-e2e \
      > gpurun_out/c5_$T/n1_bs${bs}_dt${dt}.json 2>/dev/null; echo "c5 n1 bs=$bs dt=$dt rc=$?"
  done
done
