#!/usr/bin/env bash
# Round 2, GPU call 1: steady-state step times and limiter metrics of the
# round-1 kernel on C5 (P=128, P=32) and C3 (P=128, P=32).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
out=gpurun_out/r2_prof1.log
: > $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $out
for spec in "c5 128 6" "c5 32 10" "c3 128 10" "c3 32 10"; do
  set -- $spec
  timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 >> $out 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_requests.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,lts__cycles_elapsed.avg.per_second,dram__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
for spec in "c3 128" "c3 32" "c5 32"; do
  set -- $spec
  echo "== ncu $1 P=$2" >> $out
  timeout 900 ncu --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 >> $out 2>&1
done
echo "== ncu c5 P=128 (application replay)" >> $out
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config c5 --probes 128 --steps 3 >> $out 2>&1
echo done >> $out
