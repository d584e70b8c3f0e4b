#!/usr/bin/env bash
# Round 2 GPU call Y: (a) branchless L2-policy select per gather4 (KPM_G4_POLSEL),
# (b) upper bound of what the per-nonzero dinv_j gathers cost (KPM_EXP_DINV_HOT:
# every dinv_j an L2 hit; wrong results, timing only).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_y_polsel.log
: > $out
for spec in "c5 32 8" "c5 128 6" "c3 32 10" "c3 128 10" "c5 64 6"; do
  set -- $spec
  for rep in 1 2; do
  for tag in default polsel dinvhot; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum
for spec in "c5 32" "c5 128"; do
  set -- $spec
  for tag in default polsel dinvhot; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    echo "== ncu $tag $1 P=$2" >> $out
    KPM_LIB=$lib timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
