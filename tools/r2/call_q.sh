#!/usr/bin/env bash
# Round 2 GPU call Q: the new twin cases, the driver's own sequence (bench both
# arms with default flags), and the twin on the small configs.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_twin_order.py tests/test_gpu_race_stress.py -m gpu -q -x > gpurun_out/r2_q_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_q_tests.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2_q_bench_ref.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/r2_q_bench.log 2>&1
( time timeout 900 python bench.py --config c3 ) > gpurun_out/r2_q_bench_c3.log 2>&1
for spec in "c2 64 0" "c2 64 2" "c4 64 0"; do
  set -- $spec
  for ro in 0 1; do
    KPM_REORDER=$ro timeout 600 python tools/step_timer.py --config $1 --probes $2 --mode $3 --steps 20 --warmup 3 --tag reorder$ro >> gpurun_out/r2_q_small.log 2>&1
  done
done
