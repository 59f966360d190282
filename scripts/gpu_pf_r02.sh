mkdir -p gpurun_out
SEAICE_OWN_PF=0 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_own0.log 2>&1
SEAICE_OWN_PF=1 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_own1.log 2>&1
