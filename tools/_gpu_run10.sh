mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "light_paths" > gpurun_out/gpu_tests_hot.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests_hot.log
for spec in "c5 128" "c3 128" "c5 32" "c3 32"; do
  set -- $spec
  for v in "base KPM_G4_HOT=0" "hot64 KPM_G4_HOT=1" "hot32 KPM_G4_HOT=1 KPM_HOT_MB_G4=32" "hot96 KPM_G4_HOT=1 KPM_HOT_MB_G4=96"; do
    set -- $spec $v; cfg=$1; P=$2; tag=$3; shift 3
    env "$@" timeout 300 python tools/step_timer.py --config $cfg --probes $P --steps 6 --warmup 2 --tag $tag >> gpurun_out/v10.log 2>&1
  done
done
grep '^{' gpurun_out/v10.log
for v in "base KPM_G4_HOT=0" "hot64 KPM_G4_HOT=1"; do
  set -- $v; tag=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config c5 --probes 128 --steps 3 2>/dev/null | grep -E "dram__bytes|duration|hit_rate" | sed "s/^/$tag,/"
done
