#!/bin/bash
# ncu evidence for the round (run under gpurun, one GPU).  Every ncu command follows a plain
# run of the same command that exited 0.  Outputs land in gpurun_out/; scripts/summarize_ncu.py
# turns them into the tracked summaries under profiles/.
mkdir -p gpurun_out
# (a) launch list (kernel durations, serialised) of a short bench run
CMD="python bench.py --warmup 1 --steps 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 4000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
# (b) one V-cycle at a late Newton iterate: per-kernel time + DRAM bytes, warm caches
bash scripts/ncu_vcycle.sh
# (c) full-set captures of the hot kernels
bash scripts/ncu_cheb3.sh
bash scripts/ncu_gcheb.sh
bash scripts/ncu_assembly.sh
# (kernel_bench --config 4 ran plain inside ncu_assembly.sh)
ncu --set full --clock-control none -k regex:"k_stencil_spmv|k_multidot|k_multi_axpy_norm" -s 20 -c 3 \
    -o gpurun_out/prof_krylov python scripts/kernel_bench.py --config 4 --reps 3 > gpurun_out/ncu_krylov.log 2>&1
echo "ncu round done"
