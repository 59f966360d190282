# full GPU test suite (+ optional short bench) — round-2 validation
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -s --durations=15 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
if [ -n "$WITH_BENCH" ]; then
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_PARAMS:+--params "$BENCH_PARAMS"} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
fi
