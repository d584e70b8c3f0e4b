#!/usr/bin/env bash
# Round 2 GPU call B: fixture-based config cases (C2/C4/C5), the L2 residency
# microbenchmark, and the ncu DRAM traffic of the step launch per batch width.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -s --durations=8 -k "full_vs or full_config or c5_probe_subset" > gpurun_out/r2_b_fixture_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_b_fixture_tests.log
bash tools/r2/l2exp.sh
timeout 2400 python tools/r2/traffic.py c3:128 c5:128 c5:32 c3:32 > gpurun_out/r2_b_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_b_traffic.log
