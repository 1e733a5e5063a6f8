# peer_pull (Config 3, N=2): in-kernel readiness wait + programmatic dependent launch
# vs stream waits (KVX_STREAM_PDL=0), at 16 / 4 / 1 layers per unit
mkdir -p gpurun_out/pull
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x 2>&1 | tail -1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --config 3 --no-match --steps 5"
for lpc in 16 4 1; do
  for pdl in 1 0; do
    KVX_STREAM_PDL=$pdl timeout 600 $R --layers-per-chunk $lpc > gpurun_out/pull/l${lpc}_p$pdl.json 2> gpurun_out/pull/l${lpc}_p$pdl.err
    echo "lpc=$lpc pdl=$pdl rc=$? $(python -c "
import json; d=json.loads([l for l in open('gpurun_out/pull/l${lpc}_p$pdl.json') if l.startswith('{')][-1]); print(round(d['value'],1), 'link', round(d['link']['frac'],3), 'wall', round(d['host_wall_ms_per_step'],2), 'ms', round(d['ms_per_step'],2))" 2>&1 | tail -1)"
  done
done
