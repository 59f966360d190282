#!/bin/bash
# Full ncu capture of the SpGEMM hash-path kernels (symbolic + numeric) of one AMG setup (config 4, late iterate).
mkdir -p gpurun_out
CMD="python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 1"
$CMD > gpurun_out/sg_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sgn_|k_sg_hash" --launch-skip 40 -c 14 \
    -o gpurun_out/prof_spgemm2 $CMD > gpurun_out/ncu_sg.log 2>&1
echo "exit $?"
