mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params '{"krylov_method":1}' > gpurun_out/bench_pcg.log 2>&1
