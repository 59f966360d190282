mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amgtest.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof6.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench6.log 2>&1
