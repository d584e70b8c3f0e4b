#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_l2exp_tma2.log
: > $out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for spec in "32 0.45" "64 0.55"; do
  for v in 14 15 16; do
    ./tools/exp/l2policy $spec $v >> $out 2>&1
    echo "== ncu variant $v hot/p $spec" >> $out
    ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv ./tools/exp/l2policy $spec $v 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
