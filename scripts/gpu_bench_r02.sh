mkdir -p gpurun_out
for LAG in 0 20 40 80; do
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --params "{\"amg_lag\":$LAG}" > gpurun_out/bench_lag$LAG.log 2>&1
done
