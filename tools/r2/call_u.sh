#!/usr/bin/env bash
# Round 2 GPU call U: adaptive hub threshold (nnz/2048): full suite, smoke,
# traffic, limiter metrics, bench arms, shard emulation.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r2_u_gpu_tests_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_u_gpu_tests_full.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_u_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_u_smoke.log
rm -f gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_u_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_u_traffic.log
( time timeout 1500 python bench.py ) > gpurun_out/r2_u_bench.log 2>&1
( time timeout 900 python bench.py --config c3 ) > gpurun_out/r2_u_bench_c3.log 2>&1
for n in 1 2 4 8; do
  timeout 900 python bench.py --shard-of $n --no-cpu --no-e2e > gpurun_out/r2_u_shard_of_$n.log 2>&1
done
for spec in "c3 128 10" "c3 64 10" "c3 32 10" "c5 128 6" "c5 64 6" "c5 32 8" "c2 64 20" "c4 64 20"; do
  set -- $spec
  timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag final >> gpurun_out/r2_u_steps.log 2>&1
  KPM_REORDER=0 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag final-reference-order >> gpurun_out/r2_u_steps.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for spec in "c3 128" "c5 128" "c5 32"; do
  set -- $spec
  echo "== ncu $1 P=$2" >> gpurun_out/r2_u_ncu.log
  timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/r2_u_ncu.log
done
