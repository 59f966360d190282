mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -m gpu -q -x -k "lagged or eisenstat or reuse" > gpurun_out/lagfix_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/lagfix_test.log
timeout 900 python scripts/problem1.py > gpurun_out/problem1.jsonl 2> gpurun_out/problem1.err
timeout 900 python scripts/problem2.py --runs 128:192,256:192 > gpurun_out/problem2_small.jsonl 2> gpurun_out/problem2.err
