#!/usr/bin/env bash
# Round 2 GPU call AC: (a) row-segment consume for waves that span row ends
# (KPM_G4_SEG), (b) two smaller waves in flight per warp at the full 14-16
# warps per SM for the 32-column layout (20 / 24 rows per wave).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_ac_seg_d2.log
: > $out
for tag in seg d2w20 d2w24 segd2w20; do
  KPM_LIB=$PWD/tools/exp/libkpm_$tag.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "light_paths or bitexact or race" > gpurun_out/r2_ac_tests_$tag.log 2>&1
  echo "$tag tests rc=$?" >> $out
done
for spec in "c5 32 8" "c3 32 10" "c5 128 6" "c3 128 10" "c2 64 20"; do
  set -- $spec
  for rep in 1 2; do
  for tag in default seg d2w20 d2w24 segd2w20; do
    lib=$PWD/tools/exp/libkpm_$tag.so
    [ $tag = default ] && lib=$PWD/paper_1905_09758_b200/libkpm.so
    case "$2-$tag" in 128-d2w20|128-d2w24|128-segd2w20) continue;; esac
    KPM_LIB=$lib timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag $tag >> $out 2>&1
  done
  done
done
