#!/usr/bin/env bash
# Round 2 GPU call N: full GPU suite on the twin build, DRAM traffic per batch
# width (profiles/traffic.json), limiter metrics of the twin step, both bench
# arms, the one-GPU shard emulation of the strong-scaling run.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/r2_n_gpu_tests_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_n_gpu_tests_full.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_n_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_n_smoke.log
rm -f gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_n_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_n_traffic.log
( time timeout 1500 python bench.py ) > gpurun_out/r2_n_bench.log 2>&1
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2_n_bench_ref.log 2>&1
( time timeout 900 python bench.py --config c3 ) > gpurun_out/r2_n_bench_c3.log 2>&1
for n in 2 4 8; do
  timeout 900 python bench.py --shard-of $n --no-cpu --no-e2e > gpurun_out/r2_n_shard_of_$n.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed
for spec in "c3 128" "c5 128" "c5 32"; do
  set -- $spec
  for ro in 0 1; do
    echo "== ncu $1 P=$2 KPM_REORDER=$ro" >> gpurun_out/r2_n_twin_ncu.log
    KPM_REORDER=$ro timeout 900 ncu --replay-mode application --metrics $M --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>&1 | grep -E '^"[0-9]+"' | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/r2_n_twin_ncu.log
  done
done
