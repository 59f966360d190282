#!/bin/bash
mkdir -p gpurun_out
CMD="python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 3 --ncu-range"
$CMD > gpurun_out/c3_plain.log 2>&1 && \
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_cheb3_stream -c 2 \
    -o gpurun_out/prof_cheb3 $CMD > gpurun_out/ncu_c3.log 2>&1
echo "exit $?"
