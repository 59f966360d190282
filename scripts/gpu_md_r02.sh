mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_md.log 2>&1
timeout 600 python -m pytest tests/test_gpu_amg.py tests/test_gpu_parity.py -q -x -k "counts or fgmres or krylov" > gpurun_out/md_test.log 2>&1
echo "rc=$?" >> gpurun_out/md_test.log
