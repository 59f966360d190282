# end-of-round-2 sweeps at config 4 with restart 60: hierarchy lag threshold, finest aggregation distance, PCG
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "hierarchy or galerkin or reuse" > gpurun_out/sg_test.log 2>&1
echo "rc=$?" >> gpurun_out/sg_test.log
i=0
for p in '{}' '{"amg_lag":5}' '{"amg_lag":15}' '{"amg_lag":25}' '{"agg_dist0":3}' '{"krylov_method":1}' '{"cheb_degree":2}' '{"amg_theta":0.08}'; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --params "$p" > gpurun_out/sweep2_$i.log 2>&1
i=$((i+1))
done
