#!/bin/bash
# ncu evidence for the round (run under gpurun): launch list of a short bench and a full
# capture of the top kernels.  Each ncu command follows a plain run of the same command.
set -x
mkdir -p gpurun_out
CMD="python bench.py --warmup 1 --steps 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python scripts/probe_steps.py --config 4 --steps 1"
$CMD2 > gpurun_out/ncu_plain_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_cheb_stencil|k_gcheb|k_gspmv|k_assemble|k_multidot|k_multi_axpy_norm|k_resid_dinv_stencil|k_stencil_spmv" \
    -s 400 -c 10 -o gpurun_out/prof_r01 $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "ncu done"
