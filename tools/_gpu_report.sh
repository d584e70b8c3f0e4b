# Fresh per-config numbers: step-kernel timings and end-to-end time-to-solution.
mkdir -p gpurun_out
for spec in "c1 0" "c2 0" "c3 32" "c3 64" "c3 128" "c4 0" "c5 32" "c5 128"; do
  set -- $spec
  timeout 600 python tools/step_timer.py --config $1 --probes $2 --steps 10 --warmup 3 >> gpurun_out/steps.log 2>&1
done
timeout 300 python tools/step_timer.py --config c2 --mode 2 --steps 10 --warmup 3 >> gpurun_out/steps.log 2>&1
cat gpurun_out/steps.log | grep '^{'
timeout 1500 python tools/config_report.py > gpurun_out/config_report.log 2>&1; echo report_rc=$?
cat gpurun_out/config_report.log | grep '^{'
