#!/usr/bin/env bash
# Round 2 GPU call J: full GPU suite (fixtures + the reference's own tests),
# smoke, DRAM traffic per batch width, launch list of the bench command, and
# ncu --set full captures of the step kernel (C5 application replay, C3);
# the .ncu-rep files stay on the box (size), their raw/details/source pages
# come back as CSV.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=12 > gpurun_out/r2_j_gpu_tests_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2_j_gpu_tests_full.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_j_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2_j_smoke.log
rm -f gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_j_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_j_traffic.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_j_bench_short.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_j_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_j_ncu_launch.log 2>&1
export_rep() {  # name
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/$1_source.csv.gz
  ls -la /tmp/$1.ncu-rep >> gpurun_out/r2_j_ncu_sizes.log
  sz=$(stat -c %s /tmp/$1.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 0 ] && [ "$sz" -lt 12000000 ]; then cp /tmp/$1.ncu-rep gpurun_out/; fi
}
timeout 600 python tools/prof_step.py --config c3 --steps 4 > /dev/null 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:kpm_step -s 3 -c 1 -f -o /tmp/r2_prof_c3 python tools/prof_step.py --config c3 --steps 4 > gpurun_out/r2_j_ncu_c3.log 2>&1
export_rep r2_prof_c3
timeout 600 python tools/prof_step.py --config c5 --probes 128 --steps 3 > /dev/null 2>&1 && \
timeout 3000 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:kpm_step -s 2 -c 1 -f -o /tmp/r2_prof_c5 python tools/prof_step.py --config c5 --probes 128 --steps 3 > gpurun_out/r2_j_ncu_c5.log 2>&1
export_rep r2_prof_c5
du -sh gpurun_out >> gpurun_out/r2_j_ncu_sizes.log
