#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_l2exp2.log
: > $out
for spec in "96 0.3" "64 0.2" "64 0.3" "48 0.3"; do
  ./tools/exp/l2policy $spec >> $out 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
for v in 0 1 2 3 4; do
  echo "== ncu variant $v hot 96 p 0.3" >> $out
  ncu --metrics $M --clock-control none -k regex:gather -s 1 -c 1 --csv ./tools/exp/l2policy 96 0.3 $v 2>&1 | grep -E '^"0"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
