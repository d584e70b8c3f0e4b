#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for spec in "c3 64 512" "c5 64 512" "c5 32 256"; do
  set -- $spec
  for ro in 1 0; do
    KPM_REORDER=$ro KPM_TRACE=/tmp/trace_$1_$2_$ro.bin KPM_TRACE_STEP=3 timeout 600 python tools/prof_step.py --config $1 --probes $2 --steps 5 > /dev/null 2>&1
    echo "== trace $1 P=$2 KPM_REORDER=$ro" >> gpurun_out/r2_s_trace_bw.log
    python tools/r2/trace_bw.py /tmp/trace_$1_$2_$ro.bin $3 >> gpurun_out/r2_s_trace_bw.log 2>&1
    python tools/trace_report.py /tmp/trace_$1_$2_$ro.bin 2>&1 | cut -c1-700 >> gpurun_out/r2_s_trace_bw.log
  done
done
