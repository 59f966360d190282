mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 20 > gpurun_out/vc4.log 2>&1
SEAICE_SETUP_TIMING=1 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 5 2>&1 | grep -E "tentative|power|aggregate" | tail -12 > gpurun_out/setup2.log
timeout 600 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amgtest.log 2>&1
