#!/bin/bash
# r02: drop-in latency -- the reference engine relinked on libkvcsim_gpu.so vs the pure reference
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for b in ref_replay dropin_replay; do
  /usr/bin/time -f "$b wall %e s" env KVCSIM_GPU_STATS=1 oracle/_ref/$b > gpurun_out/$b.out 2> gpurun_out/$b.err
  tail -2 gpurun_out/$b.err
done
cmp gpurun_out/ref_replay.out gpurun_out/dropin_replay.out && echo "reports byte-identical"
for b in ref_acceptance dropin_acceptance; do
  /usr/bin/time -f "$b wall %e s" env KVCSIM_GPU_STATS=1 oracle/_ref/$b > gpurun_out/$b.out 2> gpurun_out/$b.err
  tail -2 gpurun_out/$b.err
done
