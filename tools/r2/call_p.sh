#!/usr/bin/env bash
# Round 2 GPU call P: after deleting the hot-ordered-wave template and fixing
# the bulk path's policy: full suite, smoke, traffic, bench arms, shard runs.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/r2_p_gpu_tests_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p_gpu_tests_full.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_p_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p_smoke.log
rm -f gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_p_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_p_traffic.log
for spec in "c3 128 10" "c5 128 6" "c5 32 8"; do
  set -- $spec
  timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag final >> gpurun_out/r2_p_steps.log 2>&1
  KPM_REORDER=0 timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps $3 --warmup 3 --tag final-reference-order >> gpurun_out/r2_p_steps.log 2>&1
done
# LDOS on the big graph (bulk path, 4-column layout) in both orders
for ro in 0 1; do
  KPM_REORDER=$ro timeout 600 python tools/step_timer.py --config c3 --probes 128 --mode 2 --steps 6 --warmup 3 --tag ldos-reorder$ro >> gpurun_out/r2_p_steps.log 2>&1
  KPM_REORDER=$ro timeout 600 python tools/step_timer.py --config c3 --probes 64 --mode 2 --steps 6 --warmup 3 --tag ldos-reorder$ro >> gpurun_out/r2_p_steps.log 2>&1
done
