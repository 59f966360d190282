mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "eisenstat or lagged or config1 or multistep" > gpurun_out/amgtest_ew.log 2>&1
timeout 2400 python scripts/problem2.py --runs 128:192,256:192,512:192,1024:192 > gpurun_out/problem2_r02b.jsonl 2> gpurun_out/problem2_r02b.err
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench10.log 2>&1
