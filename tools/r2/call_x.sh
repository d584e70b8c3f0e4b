#!/usr/bin/env bash
# Round 2 GPU call X: two waves in flight per warp (D=2) at fewer warps per SM,
# after tools/exp/gather_bw.cu showed 8 warps x 2 x 8 KB reach 7.2 TB/s on
# cold 256-byte gathers where 24 warps x 1 x 8 KB reach 6.7.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_x_d2.log
: > $out
for spec in "c5 32 8" "c5 128 6" "c3 32 10" "c3 128 10" "c5 64 6"; do
  set -- $spec
  for tag in default d2w8 d2t160 d2w16; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
done
