mkdir -p gpurun_out
for S in 2 3 4 5 6 8; do
SEAICE_CHEB_SEGS=$S timeout 600 python scripts/vcycle_bench.py > gpurun_out/vc_segs$S.log 2>&1
done
