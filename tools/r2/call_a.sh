#!/usr/bin/env bash
# Round 2 GPU call A: C5 fixture on the box host (background), the GPU suite
# minus the fixture-based config cases, the reference's own test files through
# the drop-in, then (host idle again) both bench arms on the default config.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > gpurun_out/r2_a_env.log
nproc >> gpurun_out/r2_a_env.log; free -g >> gpurun_out/r2_a_env.log
(python tests/golden/make_config_golden.py c5 --out gpurun_out > gpurun_out/r2_c5_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r2_c5_golden.log) &
gold=$!
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 -k "not full_length and not full_vs and not full_config and not reference_suite" > gpurun_out/r2_a_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_a_gpu_tests.log
timeout 1800 python -m pytest tests/test_reference_suite_gpu.py -m gpu -q -s > gpurun_out/r2_a_refsuite.log 2>&1
echo "rc=$?" >> gpurun_out/r2_a_refsuite.log
wait $gold
( time timeout 1500 python bench.py ) > gpurun_out/r2_a_bench.log 2>&1
echo "rc=$?" >> gpurun_out/r2_a_bench.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2_a_bench_ref.log 2>&1
echo "rc=$?" >> gpurun_out/r2_a_bench_ref.log
( time timeout 900 python bench.py --config c3 ) > gpurun_out/r2_a_bench_c3.log 2>&1
echo "rc=$?" >> gpurun_out/r2_a_bench_c3.log
