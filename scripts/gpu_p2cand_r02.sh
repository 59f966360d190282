mkdir -p gpurun_out
i=0
for P in '{}' '{"amg_lag":10}' '{"agg_dist0":3}' '{"amg_lag":10,"agg_dist0":3}'; do
i=$((i+1))
timeout 1500 python scripts/problem2.py --runs 128:192,256:192,512:192,1024:192 --params "$P" > gpurun_out/p2cand$i.jsonl 2> gpurun_out/p2cand$i.err
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params '{"amg_lag":10,"agg_dist0":3}' > gpurun_out/bench_agg6.log 2>&1
