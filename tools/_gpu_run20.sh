# ncu of the P=32 layout (the per-GPU C5 shard at 8 GPUs) next to the P=128 tiles: C3 P=32, C3 P=128, C5 P=32.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size
for spec in "c3 32" "c3 128" "c5 32"; do
  set -- $spec
  ncu --metrics $M --clock-control none -k regex:kpm_step -s 2 -c 1 --csv python tools/prof_step.py --config $1 --probes $2 --steps 3 2>/dev/null | grep -E "kpm_step" | awk -F'","' '{print "'"$1 $2"'", $(NF-2), $NF}' 
done
ncu --set full --import-source on --clock-control none -k regex:kpm_step -s 2 -c 1 -o gpurun_out/prof_c3_p32 -f python tools/prof_step.py --config c3 --probes 32 --steps 3 > gpurun_out/ncu_p32.log 2>&1; echo full_rc=$?
