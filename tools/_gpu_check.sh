# One GPU verification pass: parity suite, smoke, bench, launch list, one ncu --set full capture.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -1 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --import-source on --clock-control none -k regex:kpm_step -s 4 -c 1 -o gpurun_out/prof_c3 -f python tools/prof_step.py --steps 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
tail -2 gpurun_out/ncu_full.log
