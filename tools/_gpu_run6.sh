mkdir -p gpurun_out
for rep in 1 2; do
for lib in default seg; do
  if [ $lib = default ]; then L=""; else L="KPM_LIB=build/variants/libkpm_$lib.so"; fi
  for spec in "c3 128 0" "c3 32 0" "c2 64 2" "c4 64 0"; do
    set -- $spec
    env $L timeout 300 python tools/step_timer.py --config $1 --probes $2 --mode $3 --steps 10 --warmup 3 --tag $lib >> gpurun_out/v6.log 2>&1
  done
done
done
grep '^{' gpurun_out/v6.log
