# final evidence (trimmed: the workload runs of gpu_final_r02.sh are unaffected by the last kernel change)
mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vcycle_bench_cfg4.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s --durations=10 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python scripts/kernel_bench.py --config 5 > gpurun_out/kernel_bench_cfg5.log 2>&1
timeout 2400 bash scripts/ncu_round.sh > gpurun_out/ncu_round.log 2>&1
