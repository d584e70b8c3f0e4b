python bench.py > gpurun_out/bench_r01_bulk.json 2> gpurun_out/bench_r01_bulk.err; tail -1 gpurun_out/bench_r01_bulk.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_bulk.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch_bulk.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:kpm_step_bulk -s 2 -c 1 -o gpurun_out/prof_c3_bulk_default -f python tools/prof_step.py --steps 3 > gpurun_out/ncu_bulk_default.log 2>&1
tail -2 gpurun_out/ncu_bulk_default.log
