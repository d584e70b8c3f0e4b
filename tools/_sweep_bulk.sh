python tools/step_timer.py --config c3 --tag default
KPM_LIB=build/variants/libkpm_sh.so python tools/step_timer.py --config c3 --tag streamhints
for d in 64 128 256; do KPM_HOT_DEGREE=$d python tools/step_timer.py --config c3 --tag hot$d; done
KPM_HOT_DEGREE=0 python tools/step_timer.py --config c3 --tag nohints
