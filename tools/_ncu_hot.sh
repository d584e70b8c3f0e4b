M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
KPM_LIB=build/variants/libkpm_base.so ncu --metrics $M --clock-control none -k regex:kpm_step_kernel -s 2 -c 1 --csv python tools/prof_step.py --steps 3 > gpurun_out/ncu_hot_base.csv 2>&1
KPM_HOT_DEGREE=1000 KPM_LIB=build/variants/libkpm_hot2s.so ncu --metrics $M --clock-control none -k regex:kpm_step_kernel -s 2 -c 1 --csv python tools/prof_step.py --steps 3 > gpurun_out/ncu_hot_2s.csv 2>&1
KPM_HOT_DEGREE=300 KPM_LIB=build/variants/libkpm_hot1.so ncu --metrics $M --clock-control none -k regex:kpm_step_kernel -s 2 -c 1 --csv python tools/prof_step.py --steps 3 > gpurun_out/ncu_hot_1.csv 2>&1
grep -h "kpm_step" gpurun_out/ncu_hot_*.csv | awk -F'","' '{print $(NF-2), $NF}'
