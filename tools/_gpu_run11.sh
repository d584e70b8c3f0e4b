# Round-1 final-state verification: full GPU suite, smoke, bench (both arms), launch list, ncu --set full.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_v11.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_v11.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench_v12.json 2> gpurun_out/bench_v12.err; echo bench_rc=$?; tail -1 gpurun_out/bench_v12.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?; tail -1 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_v12.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_v12.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --import-source on --clock-control none -k regex:kpm_step -s 4 -c 1 -o gpurun_out/prof_c3_v12 -f python tools/prof_step.py --steps 4 > gpurun_out/ncu_full_v12.log 2>&1; echo ncu_full_rc=$?
tail -2 gpurun_out/ncu_full_v12.log
