#!/usr/bin/env bash
# Round 2 GPU call D: degree-relabelled graph + persisting L2 window over the
# hot rows of the gathered block (experiment; sums not in reference order).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_d_relabel.log
: > $out
for scale in 24 26; do
  for win in 0 79 48; do
    KPM_WINDOW_MB=$win timeout 900 python tools/r2/relabel_exp.py --scale $scale --probes 64 32 --steps 8 >> $out 2>&1
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for win in 0 79; do
  echo "== ncu scale 24 relab window $win P=64" >> $out
  KPM_WINDOW_MB=$win timeout 900 ncu --metrics $M --clock-control none -k regex:kpm_step -s 6 -c 1 --csv python tools/r2/relabel_exp.py --scale 24 --probes 64 --only relab --steps 4 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
