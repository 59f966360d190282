mkdir -p gpurun_out
i=0
for P in '{"agg_dist0":3}' '{"agg_dist0":3,"amg_lag":20}' '{"agg_dist0":3,"cheb_degree":4,"cheb_fused":1}' '{"amg_lag":10}' '{"amg_lag":30}'; do
i=$((i+1))
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params "$P" > gpurun_out/bench_agg$i.log 2>&1
done
