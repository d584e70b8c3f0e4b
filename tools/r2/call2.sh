#!/usr/bin/env bash
# GPU call: C5 fixture on the box host (background), GPU suite, reference suite,
# sanitizers, traffic of the C5 batch widths.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
(python tests/golden/make_config_golden.py c5 --out gpurun_out > gpurun_out/r2_c5_golden.log 2>&1; echo "rc=$?" >> gpurun_out/r2_c5_golden.log) &
gold=$!
timeout 2400 python -m pytest tests -m gpu -q -x -k "not full_length and not full_vs and not reference_suite" > gpurun_out/r2_gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_gpu_tests.log
timeout 1800 python -m pytest tests/test_reference_suite_gpu.py -m gpu -q -s > gpurun_out/r2_refsuite.log 2>&1
echo "rc=$?" >> gpurun_out/r2_refsuite.log
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/r2_sanitizer.log
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/r2/sanitize_paths.py >> gpurun_out/r2_sanitizer.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_sanitizer.log
  echo "== $tool (hub pipeline)" >> gpurun_out/r2_sanitizer.log
  KPM_HEAVY_DEGREE=48 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/r2/sanitize_paths.py g4 bulk register >> gpurun_out/r2_sanitizer.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_sanitizer.log
done
timeout 1500 python tools/r2/traffic.py c5:128 c5:64 c5:32 c3:128 > gpurun_out/r2_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_traffic.log
wait $gold
