# L2 hint on every gather4 for the 32-column layout (C5 / C3 P=32), alternating with the default.
mkdir -p gpurun_out
for rep in 1 2; do
for spec in "c5 32" "c3 32"; do
  set -- $spec
  for v in "base KPM_G4_HINT=0" "last KPM_G4_HINT=1" "first KPM_G4_HINT=2"; do
    set -- $spec $v; cfg=$1; P=$2; tag=$3; shift 3
    env "$@" timeout 300 python tools/step_timer.py --config $cfg --probes $P --steps 10 --warmup 3 --tag $tag >> gpurun_out/v22_hint.log 2>&1
  done
done
done
grep '^{' gpurun_out/v22_hint.log
