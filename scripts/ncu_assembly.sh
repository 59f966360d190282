#!/bin/bash
# Assembly variants on config 5 (kernel_bench), then a full ncu capture of the fused assembly
# kernel (config 4), after a plain run of the same command.
mkdir -p gpurun_out
K=${ASM_KERNEL:-k_assemble_had}
python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/asm_cfg5_had.json 2> gpurun_out/asm_cfg5_had.err
SEAICE_ASM_TILE=1 python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/asm_cfg5_had1.json 2> gpurun_out/asm_cfg5_had1.err
SEAICE_ASM_MODAL=1 python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/asm_cfg5_modal.json 2> gpurun_out/asm_cfg5_modal.err
CMD="python scripts/kernel_bench.py --config 4 --reps 3"
$CMD > gpurun_out/asm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
    -o gpurun_out/prof_asm $CMD > gpurun_out/ncu_asm.log 2>&1
echo "exit $?"
