#!/bin/bash
# Per-kernel launch list (warm caches) of one V-cycle at a late Newton iterate of config 4.
#   bash scripts/ncu_vcycle.sh '{"nullspace_dim":4}' tag
mkdir -p gpurun_out
P=${1:-'{}'}
T=${2:+_$2}
CMD="python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 20 --ncu-range --params $P"
$CMD > gpurun_out/vc_plain$T.log 2>&1 && \
ncu --profile-from-start off --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__registers_per_thread,launch__grid_size \
    --csv --log-file gpurun_out/vc_launches$T.csv $CMD > gpurun_out/ncu_vc$T.log 2>&1
echo "exit $?"
