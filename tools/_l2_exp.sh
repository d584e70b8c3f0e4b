# L2 persistence / eviction-hint experiment on C3 P=128 (step time + ncu DRAM bytes per launch)
mkdir -p gpurun_out
python -c "
import ctypes
lib=ctypes.CDLL('/usr/local/cuda/lib64/libcudart.so')
v=ctypes.c_int(); lib.cudaDeviceGetAttribute(ctypes.byref(v), 108, 0); print('maxPersistingL2', v.value)
v=ctypes.c_int(); lib.cudaDeviceGetAttribute(ctypes.byref(v), 38, 0); print('L2', v.value)
" 
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
run() {
  tag=$1; shift
  env "$@" timeout 300 python tools/step_timer.py --config c3 --steps 10 --warmup 3 --tag $tag >> gpurun_out/l2exp.log 2>&1
  env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:kpm_step -s 4 -c 2 --csv python tools/prof_step.py --steps 4 2>/dev/null | grep -E "dram__bytes|duration|hit_rate" | sed "s/^/$tag,/" >> gpurun_out/l2exp_ncu.csv
}
run A_default
run B_persist_last KPM_PERSIST_MB=-1 KPM_G4_HINT=1
run C_first KPM_G4_HINT=2
run D_persist KPM_PERSIST_MB=-1
run E_bulk KPM_G4=0
run F_bulk_persist KPM_G4=0 KPM_PERSIST_MB=-1
run G_bulk_persist96 KPM_G4=0 KPM_PERSIST_MB=-1 KPM_HOT_MB=96
run H_bulk_persist32 KPM_G4=0 KPM_PERSIST_MB=-1 KPM_HOT_MB=32
grep '^{' gpurun_out/l2exp.log
for spec in "c5_tiles" "c5_bulk KPM_TILE=0" "c5_bulk_persist KPM_TILE=0 KPM_PERSIST_MB=-1" "c5_tiles_persist_last KPM_PERSIST_MB=-1 KPM_G4_HINT=1"; do
  set -- $spec; tag=$1; shift
  env "$@" timeout 300 python tools/step_timer.py --config c5 --probes 128 --steps 6 --warmup 2 --tag $tag >> gpurun_out/l2exp.log 2>&1
done
grep '^{' gpurun_out/l2exp.log | tail -4
cat gpurun_out/l2exp_ncu.csv | awk -F, '{print $1, $(NF-3), $NF}' | head -80
