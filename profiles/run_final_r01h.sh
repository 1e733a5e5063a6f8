#!/bin/bash
# End-of-round numbers (r01h, half-warp hash kernel): N=1 default line (Config 2 + stage 1),
# Config 3, and the N=2 / N=4 default lines when the box has the GPUs; then the ncu evidence
# (1 GPU) through profiles/run_ncu.sh.
T=${TAG:-r01h}
mkdir -p gpurun_out/$T
G=$(nvidia-smi -L | wc -l)
timeout 400 python bench.py > gpurun_out/$T/n1_c2.json 2> gpurun_out/$T/n1_c2.err; echo "n1 c2 rc=$?"
timeout 400 python bench.py --config 3 --no-match --no-cpu-baseline > gpurun_out/$T/n1_c3.json 2> gpurun_out/$T/n1_c3.err; echo "n1 c3 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/$T/n1_ref.json 2> gpurun_out/$T/n1_ref.err; echo "n1 ref rc=$?"
for N in 2 4; do
  [ "$G" -ge "$N" ] || continue
  for c in 2 3; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus $N --config $c \
      > gpurun_out/$T/n${N}_c$c.json 2> gpurun_out/$T/n${N}_c$c.err
    echo "n$N c$c rc=$?"
  done
done
TAG=$T bash profiles/run_ncu.sh; echo "ncu rc=$?"
