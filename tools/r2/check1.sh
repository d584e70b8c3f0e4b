#!/usr/bin/env bash
# Round 2 GPU call: new multi-context / accumulate paths + parity + the new bench.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multidevice.py tests/test_gpu_parity.py tests/test_density_device.py tests/test_fileio.py -m gpu -x -q > gpurun_out/r2_check1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2_check1_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_check1_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_check1_bench.log
