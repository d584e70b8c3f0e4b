#!/usr/bin/env bash
# Round 2 GPU call AF: the final kernel's C5 P=128 launch spends 43% of its
# warp time in the wave's mbarrier wait (profiles/r02_prof_c5_final2_*):
# several smaller waves in flight per warp for the 64-column layout.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_af_c2_depth.log
: > $out
for spec in "c5 128 6" "c3 128 10" "c5 64 6"; do
  set -- $spec
  for rep in 1 2; do
  for tag in default w8d2 w8d3 w12d2; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
  done
done
for hr in 100000 500000 1000000; do
  KPM_HOT_ROWS=$hr timeout 600 python tools/step_timer.py --config c5 --probes 128 --steps 6 --warmup 3 --tag hot$hr >> $out 2>&1
  KPM_HOT_ROWS=$hr timeout 600 python tools/step_timer.py --config c5 --probes 32 --steps 8 --warmup 3 --tag hot$hr >> $out 2>&1
done
