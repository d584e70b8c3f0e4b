mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "light_paths or bitexact or deterministic or batch or c3_full" > gpurun_out/gpu_tests_fuse.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_fuse.log
for rep in 1 2; do
for f in 1 0; do
  KPM_FUSE_TILES=$f timeout 300 python tools/step_timer.py --config c3 --probes 128 --steps 10 --warmup 3 --tag fuse$f >> gpurun_out/v8.log 2>&1
  KPM_FUSE_TILES=$f timeout 300 python tools/step_timer.py --config c5 --probes 128 --steps 6 --warmup 2 --tag fuse$f >> gpurun_out/v8.log 2>&1
done
done
grep '^{' gpurun_out/v8.log
