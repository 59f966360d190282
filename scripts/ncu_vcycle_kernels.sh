#!/bin/bash
# Full ncu captures of the V-cycle's main kernels at a late config-4 iterate (one V-cycle inside
# cudaProfilerStart/Stop): fused finest Chebyshev, level-1 coarse Chebyshev, first transfer.
mkdir -p gpurun_out
CMD="python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 3 --ncu-range"
$CMD > gpurun_out/vk_plain.log 2>&1 || exit 1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_cheb3_stream -c 1 \
    -o gpurun_out/prof_chebM $CMD > gpurun_out/ncu_chebM.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_acheb4 -c 1 \
    -o gpurun_out/prof_gcheb $CMD > gpurun_out/ncu_gcheb.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_aspmv -c 2 \
    -o gpurun_out/prof_gspmv $CMD > gpurun_out/ncu_gspmv.log 2>&1
echo "exit $?"
