#!/usr/bin/env bash
# Round 2 GPU call L (experiment): hot-first neighbour order (degree-relabelled
# canonical CSR) + evict_first on all-cold gather4 groups and on the streams,
# in the default (unpartitioned) wave order.  libkpm_exp.so = -DKPM_EXP_HOTK.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_l_hotfirst.log
: > $out
export KPM_LIB=$PWD/tools/exp/libkpm_exp.so KPM_G4_HOT=0
timeout 1500 python tools/r2/relabel_exp.py --scale 24 --probes 128 64 32 --hotk 0 50000 100000 150000 200000 --steps 8 >> $out 2>&1
timeout 2400 python tools/r2/relabel_exp.py --scale 26 --probes 128 32 --hotk 0 80000 130000 200000 --steps 5 >> $out 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum
for hotk in 0 100000; do
  echo "== ncu scale 24 relab P=128 hotk=$hotk" >> $out
  timeout 900 ncu --metrics $M --clock-control none -k regex:kpm_step_g4 -s 6 -c 1 --csv python tools/r2/relabel_exp.py --scale 24 --probes 128 --only relab --hotk $hotk --steps 4 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
for hotk in 0 130000; do
  echo "== ncu scale 26 relab P=128 hotk=$hotk" >> $out
  timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 4 -c 1 --csv python tools/r2/relabel_exp.py --scale 26 --probes 128 --only relab --hotk $hotk --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> $out
done
