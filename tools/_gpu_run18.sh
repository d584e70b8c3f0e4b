# gather4 wave size x CTA size sweep (P=64 layout, C3 P=128 tiles and P=64) + bit-exact light-path test per variant.
mkdir -p gpurun_out
for v in base w20 w24t128 w24t64 w32t64 w16t128 w20t64 base; do
  if [ $v = base ]; then L=paper_1905_09758_b200/libkpm.so; else L=build/variants/libkpm_$v.so; fi
  for spec in "c3 128" "c3 64"; do
    set -- $spec
    KPM_LIB=$L timeout 300 python tools/step_timer.py --config $1 --probes $2 --steps 10 --warmup 3 --tag $v >> gpurun_out/v18_wave.log 2>&1
  done
done
grep '^{' gpurun_out/v18_wave.log
for v in w20 w24t128 w24t64 w32t64 w20t64; do
  KPM_LIB=build/variants/libkpm_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "light_paths or bitexact" > gpurun_out/v18_tests_$v.log 2>&1; echo "$v tests_rc=$?"; tail -1 gpurun_out/v18_tests_$v.log
done
