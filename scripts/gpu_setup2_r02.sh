mkdir -p gpurun_out
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ls1.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --params '{"power_iters":10}' > gpurun_out/bench_pow10.log 2>&1
