mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 20 > gpurun_out/vc7.log 2>&1
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amgtest.log 2>&1
