#!/usr/bin/env bash
# Round 2 GPU call AD: the final kernel of the round (dinv step table, ballot
# cold test, constant-width light path, row-segment consume): full GPU suite,
# smoke, DRAM traffic per batch width (-> profiles/traffic.json), both bench
# arms, C3 bench, shard emulation, steady-state steps, limiter metrics, the
# bench command's launch list, every config end to end.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/r2_ad_gpu_tests_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ad_gpu_tests_full.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_ad_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ad_smoke.log
cp profiles/traffic.json gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_ad_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ad_traffic.log
cp gpurun_out/traffic.json profiles/traffic.json
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2_ad_bench_ref.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/r2_ad_bench.log 2>&1
( time timeout 900 python bench.py --config c3 ) > gpurun_out/r2_ad_bench_c3.log 2>&1
for n in 1 2 4 8; do
  timeout 900 python bench.py --shard-of $n --no-cpu --no-e2e > gpurun_out/r2_ad_shard_of_$n.log 2>&1
done
for spec in "c3 128 10" "c3 64 10" "c3 32 10" "c5 128 6" "c5 64 6" "c5 32 8" "c2 64 20" "c4 64 20" "c1 20 50"; do
  set -- $spec
  timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag final >> gpurun_out/r2_ad_steps.log 2>&1
done
KPM_REORDER=0 timeout 600 python tools/step_timer.py --config c5 --probes 128 --steps 6 --warmup 3 --tag final-reference-order >> gpurun_out/r2_ad_steps.log 2>&1
KPM_REORDER=0 timeout 600 python tools/step_timer.py --config c3 --probes 128 --steps 10 --warmup 3 --tag final-reference-order >> gpurun_out/r2_ad_steps.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for spec in "c3 128" "c5 128" "c5 32"; do
  set -- $spec
  echo "== ncu $1 P=$2" >> gpurun_out/r2_ad_ncu.log
  timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/r2_ad_ncu.log
done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_ad_launches_c5_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_ad_launches.log 2>&1
timeout 1500 python tools/config_report.py > gpurun_out/r2_ad_config_report.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ad_config_report.log
