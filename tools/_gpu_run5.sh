mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "light_paths or bitexact or motif" > gpurun_out/gpu_tests_quick.log 2>&1; echo quick_rc=$?; tail -1 gpurun_out/gpu_tests_quick.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -1 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
ncu --set full --import-source on --clock-control none -k regex:kpm_step -s 4 -c 1 -o gpurun_out/prof_c3_w16 -f python tools/prof_step.py --steps 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
KPM_FULL_SUBSET=1 timeout 3000 python -m pytest tests -m gpu -q -s -k "subset_vs_oracle" > gpurun_out/subset_full.log 2>&1; echo subset_rc=$?
grep -E "subset normwise|passed|failed" gpurun_out/subset_full.log
