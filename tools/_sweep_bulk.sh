KPM_BULK=2 timeout 900 python tools/_bulk_check.py 2>&1 | grep -v bitwise | tail -3
for v in default s2_8 s2_16m3 s2_24 s2_8m3; do
L=build/variants/libkpm_$v.so; [ $v = default ] && L=paper_1905_09758_b200/libkpm.so
KPM_LIB=$L KPM_BULK=2 python tools/step_timer.py --config c2 --mode 2 --tag c2_ldos_$v
KPM_LIB=$L KPM_BULK=2 python tools/step_timer.py --config c4 --tag c4_$v
KPM_LIB=$L KPM_BULK=2 python tools/step_timer.py --config c3 --probes 64 --tag c3p64_$v
KPM_LIB=$L KPM_BULK=2 python tools/step_timer.py --config c5 --probes 32 --tag c5p32_$v
done
