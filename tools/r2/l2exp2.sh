#!/usr/bin/env bash
# L2 residency microbenchmark, TMA variants (10-13) next to the LSU ones (0-2).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_l2exp_tma.log
: > $out
./tools/exp/l2policy 64 0.55 >> $out 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for spec in "32 0.45" "64 0.55"; do
  for v in 0 1 2 10 11 12 13; do
    echo "== ncu variant $v hot/p $spec" >> $out
    ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv ./tools/exp/l2policy $spec $v 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
