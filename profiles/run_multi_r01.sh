set -x
export NCCL_DEBUG=WARN
for m in peer_fused peer_ce peer_nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --mode $m --steps 5 --warmup 3 --no-match --no-e2e > gpurun_out/m2_$m.json 2> gpurun_out/m2_$m.err
  echo "$m rc=$?"
  tail -3 gpurun_out/m2_$m.err
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/b2_match.json 2> gpurun_out/b2_match.err; echo rc=$?; tail -3 gpurun_out/b2_match.err
