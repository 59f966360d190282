# final round-2 evidence with the product defaults: GPU tests, smoke, bench, workload runs, ncu round
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -s --durations=10 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vcycle_bench_cfg4.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_profile_cfg4.log 2>&1
timeout 600 python scripts/kernel_bench.py --config 5 > gpurun_out/kernel_bench_cfg5.log 2>&1
timeout 900 python scripts/problem1.py > gpurun_out/problem1.jsonl 2> gpurun_out/problem1.err
timeout 1500 python scripts/problem2.py --runs 128:192,256:192,512:192,1024:192 > gpurun_out/problem2_4days.jsonl 2> gpurun_out/problem2.err
timeout 900 python scripts/zeta_spread.py --config 3 > gpurun_out/cfg3_zeta.jsonl 2> gpurun_out/cfg3_zeta.err
timeout 2400 bash scripts/ncu_round.sh > gpurun_out/ncu_round.log 2>&1
