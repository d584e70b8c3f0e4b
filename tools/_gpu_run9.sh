mkdir -p gpurun_out
timeout 600 python tools/c2_profile.py > gpurun_out/c2_profile.log 2>&1; cat gpurun_out/c2_profile.log | grep '^{'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:kpm_step -c 4 --csv python tools/prof_step.py --config c5 --probes 128 --steps 4 > gpurun_out/c5_launches.csv 2>/dev/null; echo c5ncu_rc=$?
grep -E "dram__bytes|duration|hit_rate" gpurun_out/c5_launches.csv | awk -F, '{print $(NF-3), $NF}'
