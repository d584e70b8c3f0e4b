mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -1 gpurun_out/bench.json
timeout 300 python tools/step_timer.py --config c5 --probes 128 --steps 6 --warmup 2 --tag default > gpurun_out/c5step.log 2>&1; grep '^{' gpurun_out/c5step.log
timeout 1500 python tools/config_report.py > gpurun_out/config_report.log 2>&1; echo report_rc=$?
grep '^{' gpurun_out/config_report.log
