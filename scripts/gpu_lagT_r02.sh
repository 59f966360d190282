mkdir -p gpurun_out
for T in 0 3 5 10; do
timeout 900 python scripts/problem1.py --sizes 1024,2048 --params "{\"amg_lag\":$T}" > gpurun_out/p1_lag$T.jsonl 2> gpurun_out/p1_lag$T.err
done
for T in 3 5; do
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --params "{\"amg_lag\":$T}" > gpurun_out/bench_lagT$T.log 2>&1
done
