#!/usr/bin/env bash
# Round 2 GPU call AI: own-row prefetch ring depth (KPM_G4_OWN = 2 / 4 / 8).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_ai_own_ring.log
: > $out
for spec in "c5 128 6" "c5 32 8" "c3 128 10" "c2 64 20"; do
  set -- $spec
  for rep in 1 2; do
  for tag in default own8 own2; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
  done
done
