#!/usr/bin/env bash
# Round 2 GPU call AH: the driver's own round-end sequence on the committed
# tree after a clean rebuild: GPU suite, smoke, reference arm, bench.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/r2_ah_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ah_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_ah_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ah_smoke.log
( time timeout 1500 python bench.py --impl reference --gpus 1 --steps 10 --warmup 3 ) > gpurun_out/r2_ah_bench_ref.log 2>&1
( time timeout 1500 python bench.py --gpus 1 --steps 10 --warmup 3 ) > gpurun_out/r2_ah_bench.log 2>&1
