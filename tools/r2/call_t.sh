#!/usr/bin/env bash
# hub-row threshold sweep on the twin (KPM_HEAVY_DEGREE)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_t_heavy.log
: > $out
for spec in "c5 128 6" "c5 64 6" "c5 32 8" "c3 128 10" "c3 32 10"; do
  set -- $spec
  for hd in 65536 131072 262144 524288 2000000; do
    KPM_HEAVY_DEGREE=$hd timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag heavy$hd >> $out 2>&1
  done
done
