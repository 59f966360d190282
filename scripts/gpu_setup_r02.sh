mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -m gpu -q -x -k "hierarchy or spgemm or covered or counts" > gpurun_out/sym_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/sym_test.log
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof.log 2>&1
