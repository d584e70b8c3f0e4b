#!/usr/bin/env bash
# Round 2 GPU call I: occupancy / wave-shape variants of the gather4 kernel.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_i_variants.log
: > $out
for spec in "c5 128 6" "c3 128 10" "c5 32 8" "c3 32 10"; do
  set -- $spec
  for lib in paper_1905_09758_b200/libkpm.so tools/exp/libkpm_t320.so tools/exp/libkpm_w8d2.so tools/exp/libkpm_t320w12.so; do
    for hot in default 0; do
      if [ $hot = default ]; then unset KPM_G4_HOT; else export KPM_G4_HOT=0; fi
      KPM_LIB=$PWD/$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag "$(basename $lib)-hot$hot" >> $out 2>&1
    done
  done
done
