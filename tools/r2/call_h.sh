#!/usr/bin/env bash
# Round 2 GPU call H: hot rule with a fractional boundary degree bucket.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "light_paths or hub or determin" > gpurun_out/r2_h_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2_h_parity.log
out=gpurun_out/r2_h_hot.log
: > $out
run() {  # cfg P steps hot mb frac
  KPM_G4_HOT=$4 KPM_HOT_MB_G4=$5 KPM_HOT_FRAC=$6 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag "hot$4-mb$5-frac$6" >> $out 2>&1
}
for spec in "c5 128 6" "c3 128 10" "c5 32 8"; do
  set -- $spec
  run $1 $2 $3 0 64 1
  run $1 $2 $3 1 64 0
  for mb in 40 56 72; do run $1 $2 $3 1 $mb 1; done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum
for spec in "c5 128 56" "c5 128 72" "c3 128 56"; do
  set -- $spec
  echo "== ncu $1 P=$2 hot=1 mb=$3 frac=1" >> $out
  KPM_G4_HOT=1 KPM_HOT_MB_G4=$3 timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
