#!/usr/bin/env bash
# Round 2 GPU call AB: cold-group test from one ballot per wave + constant
# tile width (immediate shared-memory offsets in the consumer) for full-width
# single-tile launches; A/B against the previous commit's build.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_twin_order.py tests/test_gpu_race_stress.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2_ab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ab_tests.log
out=gpurun_out/r2_ab_ballot_constw.log
: > $out
for spec in "c5 32 8" "c5 128 6" "c5 64 6" "c3 32 10" "c3 128 10" "c3 64 10" "c2 64 20" "c4 64 20"; do
  set -- $spec
  for rep in 1 2; do
    KPM_LIB=$PWD/tools/exp/libkpm_base.so timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag base >> $out 2>&1
    timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag new >> $out 2>&1
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum
for spec in "c5 32" "c5 128"; do
  set -- $spec
  for tag in base new; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = new ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    echo "== ncu $tag $1 P=$2" >> $out
    KPM_LIB=$lib timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
