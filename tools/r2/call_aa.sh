#!/usr/bin/env bash
# Round 2 GPU call AA: ncu --set full of the C5 P=32 step (the 8-GPU shard) on
# the dinv-table kernel, and traffic.json for this kernel hash.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --config c5 --probes 32 --steps 3 > gpurun_out/r2_aa_prof.log 2>&1
timeout 1500 ncu --set full --import-source on --replay-mode application --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 -f -o gpurun_out/r2_aa_c5_p32 python tools/prof_step.py --config c5 --probes 32 --steps 3 >> gpurun_out/r2_aa_prof.log 2>&1
echo "rc=$?" >> gpurun_out/r2_aa_prof.log
ncu -i gpurun_out/r2_aa_c5_p32.ncu-rep --page raw --csv > gpurun_out/r2_aa_c5_p32_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_aa_c5_p32.ncu-rep --page details --csv > gpurun_out/r2_aa_c5_p32_details.csv 2>/dev/null
ncu -i gpurun_out/r2_aa_c5_p32.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/r2_aa_c5_p32_source.csv.gz
rm -f gpurun_out/r2_aa_c5_p32.ncu-rep
cp profiles/traffic.json gpurun_out/traffic.json
timeout 2400 python tools/r2/traffic.py c5:128 c3:128 c5:64 c5:32 > gpurun_out/r2_aa_traffic.log 2>&1
echo "rc=$?" >> gpurun_out/r2_aa_traffic.log
