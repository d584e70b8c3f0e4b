#!/usr/bin/env bash
# Round 2 GPU call M: the gather-ordered twin in production: tests, A/B of
# KPM_REORDER=0 vs the default, hot-row count sweep, bench.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_twin_order.py tests/test_gpu_parity.py tests/test_gpu_race_stress.py tests/test_gpu_multidevice.py tests/test_gpu_partition.py tests/test_density_device.py -m gpu -q -x > gpurun_out/r2_m_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_m_tests.log
timeout 2400 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -s --durations=10 > gpurun_out/r2_m_config_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_m_config_tests.log
out=gpurun_out/r2_m_twin_ab.log
: > $out
for spec in "c3 128 10" "c3 64 10" "c3 32 10" "c5 128 6" "c5 64 6" "c5 32 8"; do
  set -- $spec
  KPM_REORDER=0 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag reference-order >> $out 2>&1
  for hr in 100000 160000 250000 400000; do
    KPM_HOT_ROWS=$hr timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag twin-hot$hr >> $out 2>&1
  done
done
( time timeout 1500 python bench.py --no-cpu ) > gpurun_out/r2_m_bench.log 2>&1
( time timeout 900 python bench.py --config c3 --no-cpu ) > gpurun_out/r2_m_bench_c3.log 2>&1
