# 2-SM kernel sweep on the long-K shape: stages x group_m, DRAM bytes + time via ncu
for st in 4 7; do for gm in 4 8 16; do
  GPCX_TC_KERNEL=2sm GPCX_TC_STAGES2=$st GPCX_TC_GROUPM=$gm timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm2 --csv python tools/prof_target.py --what longk2 2>/dev/null | grep -E "gemm2" | awk -F'","' -v st=$st -v gm=$gm '{print "stages="st" group_m="gm" "$(NF-2)" "$(NF)}'
done; done
