#!/bin/bash
# Config-5 kernel benchmark (plain), then a full ncu capture of the fused assembly kernel
# (config 4), after a plain run of the same command.
mkdir -p gpurun_out
python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/kernel_bench_cfg5.json 2> gpurun_out/kernel_bench_cfg5.err
CMD="python scripts/kernel_bench.py --config 4 --reps 3"
$CMD > gpurun_out/asm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assemble_had -c 1 \
    -o gpurun_out/prof_asm $CMD > gpurun_out/ncu_asm.log 2>&1
echo "exit $?"
