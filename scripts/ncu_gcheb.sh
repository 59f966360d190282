#!/bin/bash
# Full ncu capture of the level-1 coarse Chebyshev step (first k_gcheb of one V-cycle, config 4).
mkdir -p gpurun_out
CMD="python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 3 --ncu-range"
$CMD > gpurun_out/gc_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_acheb4 -c 2 \
    -o gpurun_out/prof_gcheb $CMD > gpurun_out/ncu_gc.log 2>&1
echo "exit $?"
