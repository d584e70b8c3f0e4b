#!/usr/bin/env bash
# Round 2 GPU call G: hot-ordered waves with the evict_first-only policy
# (cold gather4 groups, own rows, col ids, T_{k+1} stores) vs the default order.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2_g_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2_g_parity.log
out=gpurun_out/r2_g_hot.log
: > $out
run() {  # cfg P steps hot mb
  KPM_G4_HOT=$4 KPM_HOT_MB_G4=$5 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag "hot$4-mb$5" >> $out 2>&1
}
for spec in "c3 128 10" "c3 64 10" "c3 32 10" "c5 128 6" "c5 32 8"; do
  set -- $spec
  run $1 $2 $3 0 64
  for mb in 32 48 64 96; do run $1 $2 $3 1 $mb; done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum
for spec in "c3 128" "c5 128" "c5 32"; do
  set -- $spec
  for hot in 0 1; do
    echo "== ncu $1 P=$2 hot=$hot mb=48" >> $out
    KPM_G4_HOT=$hot KPM_HOT_MB_G4=48 timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
