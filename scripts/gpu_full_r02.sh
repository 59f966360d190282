# round-2 evidence: GPU tests, bench (N=1, defaults), ncu launch lists and full captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s --durations=20 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 2400 bash scripts/ncu_round.sh > gpurun_out/ncu_round.log 2>&1
