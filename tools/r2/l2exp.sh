#!/usr/bin/env bash
# L2 residency microbenchmark (tools/exp/l2policy.cu): times of every policy
# variant for several (hot MB, hot share) points, then ncu DRAM bytes / L2 hit
# rate per variant.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_l2exp.log
: > $out
for spec in "32 0.45" "48 0.5" "64 0.55" "96 0.62"; do
  ./tools/exp/l2policy $spec >> $out 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for spec in "32 0.45" "64 0.55" "96 0.62"; do
  for v in 0 1 2 3 4 6 7; do
    echo "== ncu variant $v hot/p $spec" >> $out
    ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv ./tools/exp/l2policy $spec $v 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
  done
done
