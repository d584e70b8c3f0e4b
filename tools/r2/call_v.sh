#!/usr/bin/env bash
# Round 2 GPU call V: streamed empty-chunk path: parity + A/B vs the previous build.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twin_order.py tests/test_gpu_race_stress.py tests/test_gpu_partition.py -m gpu -q -x > gpurun_out/r2_v_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_v_tests.log
out=gpurun_out/r2_v_ab.log
: > $out
for spec in "c5 128 6" "c5 32 8" "c3 128 10" "c3 32 10" "c5 64 6"; do
  set -- $spec
  for rep in 1 2; do
    KPM_LIB=$PWD/tools/exp/libkpm_base.so timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag base >> $out 2>&1
    timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag emptypath >> $out 2>&1
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum
for lib in tools/exp/libkpm_base.so paper_1905_09758_b200/libkpm.so; do
  echo "== ncu $lib c5 P=32" >> $out
  KPM_LIB=$PWD/$lib timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config c5 --probes 32 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
