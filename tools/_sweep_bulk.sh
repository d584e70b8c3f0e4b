for v in A A2 A3 A4 A5; do
KPM_BULK=1 KPM_HOT_DEGREE=1000 KPM_LIB=build/variants/libkpm_$v.so python tools/step_timer.py --config c3 --tag bulk_${v}_hot1000
done
for d in 200 500 2000 5000; do
KPM_BULK=1 KPM_HOT_DEGREE=$d KPM_LIB=build/variants/libkpm_A.so python tools/step_timer.py --config c3 --tag bulk_A_hot$d
done
