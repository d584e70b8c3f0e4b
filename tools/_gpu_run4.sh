mkdir -p gpurun_out
free -g | head -2; nproc
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
python -m pytest tests -m gpu -q -s -k "subset_vs_oracle" 2>&1 | grep -E "subset normwise|passed|failed|skipped"
for lib in default c1w32 c2w32 c1m2; do
  if [ $lib = default ]; then L=""; else L="KPM_LIB=build/variants/libkpm_$lib.so"; fi
  for spec in "c3 128 0" "c3 64 0" "c3 32 0" "c5 32 0" "c2 64 2"; do
    set -- $spec
    env $L timeout 300 python tools/step_timer.py --config $1 --probes $2 --mode $3 --steps 10 --warmup 3 --tag $lib >> gpurun_out/v4.log 2>&1
  done
done
grep '^{' gpurun_out/v4.log
