#!/usr/bin/env bash
# Round 2 GPU call O: one-GPU emulation of the strong-scaling shards, launch
# list of the bench command and ncu --set full of the final (twin) kernel.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for n in 1 2 4 8; do
  timeout 900 python bench.py --shard-of $n --no-cpu --no-e2e > gpurun_out/r2_o_shard_of_$n.log 2>&1
done
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_o_bench_short.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_o_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_o_ncu_launch.log 2>&1
export_rep() {  # name
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/$1_source.csv.gz
}
timeout 600 python tools/prof_step.py --config c3 --steps 4 > /dev/null 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:kpm_step_g4 -s 3 -c 1 -f -o /tmp/r2_prof_c3_twin python tools/prof_step.py --config c3 --steps 4 > gpurun_out/r2_o_ncu_c3.log 2>&1
export_rep r2_prof_c3_twin
timeout 600 python tools/prof_step.py --config c5 --probes 128 --steps 3 > /dev/null 2>&1 && \
timeout 3000 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:kpm_step_g4 -s 2 -c 1 -f -o /tmp/r2_prof_c5_twin python tools/prof_step.py --config c5 --probes 128 --steps 3 > gpurun_out/r2_o_ncu_c5.log 2>&1
export_rep r2_prof_c5_twin
