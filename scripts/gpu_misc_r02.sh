mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py tests/test_gpu_parity.py -q -x > gpurun_out/amgtest.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof8.log 2>&1
timeout 900 python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/kernel_bench_cfg5.json 2> gpurun_out/kernel_bench_cfg5.err
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8.log 2>&1
