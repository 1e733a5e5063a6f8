# N=2 streamer modes after programmatic dependent launch (Config 2 and Config 3), PDL on vs off
mkdir -p gpurun_out/modes
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --no-match --steps 5"
for c in 2 3; do for m in peer_ce peer_fused peer_pull; do for pdl in 1 0; do
  KVX_STREAM_PDL=$pdl timeout 600 $R --config $c --mode $m > gpurun_out/modes/c${c}_${m}_p$pdl.json 2>/dev/null
  echo "c$c $m pdl=$pdl rc=$? $(python -c "
import json; d=json.loads([l for l in open('gpurun_out/modes/c${c}_${m}_p$pdl.json') if l.startswith('{')][-1]); print(round(d['value'],1), 'link', round(d['link']['frac'],3))" 2>&1 | tail -1)"
done; done; done
