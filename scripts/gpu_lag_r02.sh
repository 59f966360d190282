mkdir -p gpurun_out
for T in 0 20 40 60 100; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params "{\"amg_lag\":$T}" > gpurun_out/bench_lag$T.log 2>&1
done
