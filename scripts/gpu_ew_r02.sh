mkdir -p gpurun_out
for e in 0.3 0.03 0.01; do
SEAICE_EW_MAX=$e timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ew$e.log 2>&1
done
