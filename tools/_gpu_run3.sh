mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "motif or c4" > gpurun_out/gpu_motif_tests.log 2>&1; echo motif_tests_rc=$?; tail -2 gpurun_out/gpu_motif_tests.log
timeout 600 python tools/config_report.py --configs c4 > gpurun_out/config_report_c4.log 2>&1; grep '^{' gpurun_out/config_report_c4.log
for lib in default w16 w16m3; do
  if [ $lib = default ]; then L=""; else L="KPM_LIB=build/variants/libkpm_$lib.so"; fi
  for spec in "c3 128 0" "c3 64 0" "c2 64 2" "c4 64 0"; do
    set -- $spec
    env $L timeout 300 python tools/step_timer.py --config $1 --probes $2 --mode $3 --steps 10 --warmup 3 --tag $lib >> gpurun_out/w16.log 2>&1
  done
done
grep '^{' gpurun_out/w16.log
