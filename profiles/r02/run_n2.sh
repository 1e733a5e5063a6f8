#!/bin/bash
# r02: 2-GPU box -- GPU suite (2-GPU tests included), N=2 benches, NVLink counters.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=${TAG:-r02b}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests2_$TAG.log 2>&1
echo "gpu suite rc=$?"; tail -4 gpurun_out/gputests2_$TAG.log
timeout 900 $TR --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/n2_c2_$TAG.json 2> gpurun_out/n2_c2_$TAG.err
echo "n2 c2 rc=$?"; tail -c 400 gpurun_out/n2_c2_$TAG.err
for G in kernel stream; do
  for LPC in 16 1; do
    KVX_PULL_GATE=$G timeout 600 $TR --master-port $((29620 + LPC)) bench.py --gpus 2 --config 3 --layers-per-chunk $LPC --steps 5 --warmup 3 --no-match --no-cpu-baseline --no-e2e > gpurun_out/n2_c3_${G}_l${LPC}_$TAG.json 2> gpurun_out/n2_c3_${G}_l${LPC}_$TAG.err
    echo "c3 gate=$G lpc=$LPC rc=$?"
  done
done
timeout 300 python tests/perf/nvlink_counters.py > gpurun_out/nvl_plain_$TAG.json 2>&1
echo "nvl plain rc=$?"; cat gpurun_out/nvl_plain_$TAG.json | tail -5
timeout 300 python tests/perf/nvlink_counters.py --modes pull,push --reps 1 > gpurun_out/nvl_plain1_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:copy_lsu --csv --log-file gpurun_out/nvl_ncu_$TAG.csv \
  python tests/perf/nvlink_counters.py --modes pull,push --reps 1 > gpurun_out/nvl_ncu_$TAG.log 2>&1
echo "nvl ncu rc=$?"; tail -5 gpurun_out/nvl_ncu_$TAG.csv
