mkdir -p gpurun_out
for s in 1 -1; do
SEAICE_SLOT_SHIFT=$s timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_slot$s.log 2>&1
done
SEAICE_CTA_MAXNB=0 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_nocta.log 2>&1
