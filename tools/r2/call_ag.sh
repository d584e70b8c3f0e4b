#!/usr/bin/env bash
# Round 2 GPU call AG: 18 warps per SM (2 CTAs x 9 warps, <= 112 registers)
# for the gather4 kernels; shared memory has room for 18 x 10.9 KB.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_ag_t288.log
: > $out
for spec in "c5 128 6" "c5 32 8" "c3 128 10" "c3 32 10" "c5 64 6" "c2 64 20"; do
  set -- $spec
  for rep in 1 2; do
  for tag in default t288; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
  done
done
