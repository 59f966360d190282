#!/bin/bash
# DRAM traffic per launch of the hot kernels at config 4 (for bench.py's roofline "traffic")
# and one full-set capture of the finest Chebyshev kernel.  Each ncu run follows a plain run.
mkdir -p gpurun_out
CMD="python scripts/vcycle_bench.py --config 4 --iterate 6 --reps 20"
$CMD > gpurun_out/ncu_plain_vcb.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_cheb_stencil|k_gcheb|k_stencil_spmv|k_multidot|k_assemble|k_resid_dinv_stencil|k_gspmv|k_multi_axpy_norm|k_gresid|k_delta_energy" \
    -s 300 -c 400 --csv --log-file gpurun_out/traffic.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_cheb_stencil" -s 60 -c 1 \
    -o gpurun_out/prof_cheb0 $CMD > gpurun_out/ncu_full_cheb0.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gcheb" -s 60 -c 1 \
    -o gpurun_out/prof_gcheb $CMD > gpurun_out/ncu_full_gcheb.log 2>&1
echo traffic done
