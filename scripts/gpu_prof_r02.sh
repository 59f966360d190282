# setup-phase breakdown + full ncu of the level-1 coarse Chebyshev / residual kernels (b = 4)
mkdir -p gpurun_out
SEAICE_SETUP_TIMING=1 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 5 > gpurun_out/setup_timing.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:"k_acheb4|k_aresid4" --launch-count 4 \
  -o gpurun_out/ncu_acheb4 -f python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 5 --ncu-range > gpurun_out/ncu_acheb4.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_acheb4.log
