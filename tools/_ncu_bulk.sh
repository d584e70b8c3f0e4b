KPM_BULK=1 KPM_HOT_DEGREE=1000 KPM_LIB=build/variants/libkpm_F.so ncu --set full --import-source on --clock-control none -k regex:kpm_step_bulk -s 2 -c 1 -o gpurun_out/prof_c3_bulkF -f python tools/prof_step.py --steps 3 > gpurun_out/ncu_bulkF.log 2>&1
tail -3 gpurun_out/ncu_bulkF.log
