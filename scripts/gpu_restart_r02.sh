# FGMRES restart length sweep at config 4 (bench steps 4-6), tail parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "tail" > gpurun_out/tail_test.log 2>&1
echo "rc=$?" >> gpurun_out/tail_test.log
for m in 30 45 60; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --params "{\"restart\":$m}" > gpurun_out/bench_restart$m.log 2>&1
done
timeout 600 python scripts/probe_steps.py --config 4 --steps 5 --newton-log --params '{"restart":60}' > gpurun_out/probe_cfg4_m60.log 2>&1
