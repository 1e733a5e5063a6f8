#!/bin/bash
# r02: match -- task order (longest first), full residency, request-count scaling
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for cfg in "0 0" "1 0" "0 1" "1 1"; do set -- $cfg
  KVX_MATCH_ORDER=$1 KVX_MATCH_OCC=$2 MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1
done | tee gpurun_out/match_sweep3.txt
for N in 148 592 1184 2048 4096; do MP_NREQ=$N MP_PIN=0 timeout 300 python tests/perf/match_phase.py 2>&1 | grep after_hash=1; done | tee -a gpurun_out/match_sweep3.txt
# in-situ DRAM bytes of the match right after the hash (no cache flush between kernels)
python bench.py --requests 4 --wave 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tier > gpurun_out/plain_m.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --cache-control none \
  --clock-control none -k regex:"match_group|hash_kernel" --csv --log-file gpurun_out/match_insitu.csv \
  python bench.py --requests 4 --wave 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tier > gpurun_out/ncu_m.log 2>&1
echo "ncu rc=$?"
