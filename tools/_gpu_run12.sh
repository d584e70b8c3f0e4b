# Chunk queue order experiment: longest-row-first (default) vs row-id order.
mkdir -p gpurun_out
for spec in "c3 128" "c3 32" "c5 32" "c2 64"; do
  set -- $spec
  for v in "base KPM_CHUNK_ORDER=0" "idorder KPM_CHUNK_ORDER=1" "idorder_c4k KPM_CHUNK_ORDER=1 KPM_CHUNK_COST=4096"; do
    set -- $spec $v; cfg=$1; P=$2; tag=$3; shift 3
    env "$@" timeout 300 python tools/step_timer.py --config $cfg --probes $P --steps 6 --warmup 3 --tag $tag >> gpurun_out/v12_order.log 2>&1
  done
done
grep '^{' gpurun_out/v12_order.log
for v in "base KPM_CHUNK_ORDER=0" "idorder KPM_CHUNK_ORDER=1"; do
  set -- $v; tag=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config c3 --probes 128 --steps 3 2>/dev/null | grep -E "dram__bytes|duration|hit_rate" | sed "s/^/$tag,/"
done
