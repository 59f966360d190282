mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -m gpu -q -s -x -k "reuse or lagged or scale or covered" > gpurun_out/reusetest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/reusetest.log
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 --params '{"amg_reuse":1}' > gpurun_out/setup_prof_reuse.log 2>&1
for P in '{}' '{"amg_reuse":1}'; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params "$P" > gpurun_out/bench_reuse_$(echo $P | tr -dc 'a-z0-9').log 2>&1
done
