#!/usr/bin/env bash
# Round 2 GPU call Z: dinv_j of cold ids from the twin's degree-step table in
# shared memory (kpm_graph::dstep_id) instead of an 8-byte gather per nonzero.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_twin_order.py tests/test_gpu_race_stress.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2_z_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_z_tests.log
out=gpurun_out/r2_z_dinv_table.log
: > $out
for spec in "c5 128 6" "c5 32 8" "c5 64 6" "c3 128 10" "c3 32 10" "c3 64 10"; do
  set -- $spec
  for rep in 1 2; do
    KPM_DINV_TABLE=0 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag gather >> $out 2>&1
    timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag table >> $out 2>&1
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for spec in "c5 128" "c5 32" "c3 128"; do
  set -- $spec
  for tab in 0 1; do
    echo "== ncu table=$tab $1 P=$2" >> $out
    KPM_DINV_TABLE=$tab timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
