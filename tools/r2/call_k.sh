#!/usr/bin/env bash
# Round 2 GPU call K: compute-sanitizer (memcheck / racecheck / synccheck) over
# every light path of the fused step kernel, with and without forced hub rows,
# plus the cross-process IPC test.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
log=gpurun_out/r2_k_sanitizer.log
: > $log
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $log
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/r2/sanitize_paths.py >> $log 2>&1
  echo "rc=$?" >> $log
  echo "== $tool (hub pipeline, KPM_HEAVY_DEGREE=48)" >> $log
  KPM_HEAVY_DEGREE=48 timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/r2/sanitize_paths.py g4 bulk register >> $log 2>&1
  echo "rc=$?" >> $log
done
# work-item trace of one C5 step (load balance / tail)
for spec in "c5 128" "c5 32" "c3 128"; do
  set -- $spec
  KPM_TRACE=/tmp/trace_$1_$2.bin KPM_TRACE_STEP=3 timeout 600 python tools/prof_step.py --config $1 --probes $2 --steps 5 > /dev/null 2>&1
  echo "== trace $1 P=$2" >> gpurun_out/r2_k_trace.log
  python tools/trace_report.py /tmp/trace_$1_$2.bin >> gpurun_out/r2_k_trace.log 2>&1
done
