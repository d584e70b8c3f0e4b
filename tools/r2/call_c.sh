#!/usr/bin/env bash
# Round 2 GPU call C: A/B of the leaner gather4 wave (elect.sync issue, fix-ups
# only on the last wave, one h_ij product per neighbour in full-row waves)
# against the previous build (tools/exp/libkpm_base.so).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -m gpu -q -x > gpurun_out/r2_c_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2_c_parity.log
out=gpurun_out/r2_c_ab.log
: > $out
for spec in "c3 128 10" "c3 64 10" "c3 32 10" "c5 128 6" "c5 32 10" "c2 64 20" "c4 64 20"; do
  set -- $spec
  for rep in 1 2; do
    KPM_LIB=$PWD/tools/exp/libkpm_base.so timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag base >> $out 2>&1
    timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag new >> $out 2>&1
  done
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__cycles_elapsed.avg.per_second
for lib in tools/exp/libkpm_base.so paper_1905_09758_b200/libkpm.so; do
  for spec in "c3 128" "c3 32"; do
    set -- $spec
    echo "== ncu $lib $1 P=$2" >> $out
    KPM_LIB=$PWD/$lib timeout 900 ncu --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
