#!/usr/bin/env bash
# Round 2 GPU call AE: ncu --set full (source page) of the final kernel's C5
# and C3 128-probe step launches.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for cfg in c5 c3; do
  timeout 600 python tools/prof_step.py --config $cfg --probes 128 --steps 3 > gpurun_out/r2_ae_prof_$cfg.log 2>&1
  timeout 1800 ncu --set full --import-source on --replay-mode application --clock-control none -k regex:kpm_step_g4 -s 2 -c 1 -f -o gpurun_out/r2_ae_${cfg}_p128 python tools/prof_step.py --config $cfg --probes 128 --steps 3 >> gpurun_out/r2_ae_prof_$cfg.log 2>&1
  echo "rc=$?" >> gpurun_out/r2_ae_prof_$cfg.log
  ncu -i gpurun_out/r2_ae_${cfg}_p128.ncu-rep --page raw --csv > gpurun_out/r2_ae_${cfg}_p128_raw.csv 2>/dev/null
  ncu -i gpurun_out/r2_ae_${cfg}_p128.ncu-rep --page details --csv > gpurun_out/r2_ae_${cfg}_p128_details.csv 2>/dev/null
  ncu -i gpurun_out/r2_ae_${cfg}_p128.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/r2_ae_${cfg}_p128_source.csv.gz
  rm -f gpurun_out/r2_ae_${cfg}_p128.ncu-rep
done
