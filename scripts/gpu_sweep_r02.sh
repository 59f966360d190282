mkdir -p gpurun_out
for P in '{"agg_dist":3}' '{}'; do
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params "$P" >> gpurun_out/bench_dist2.log 2>&1
done
