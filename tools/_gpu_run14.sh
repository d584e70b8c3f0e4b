# FMA experiment (gather4 light path): base vs -DKPM_G4_FMA=1, alternating, steady state.
mkdir -p gpurun_out
for rep in 1 2; do
for spec in "c3 128" "c3 64" "c5 32"; do
  set -- $spec
  timeout 300 python tools/step_timer.py --config $1 --probes $2 --steps 10 --warmup 3 --tag base >> gpurun_out/v14_fma.log 2>&1
  KPM_LIB=build/variants/libkpm_fma.so timeout 300 python tools/step_timer.py --config $1 --probes $2 --steps 10 --warmup 3 --tag fma >> gpurun_out/v14_fma.log 2>&1
done
done
grep '^{' gpurun_out/v14_fma.log
