mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py tests/test_gpu_goldens.py -m gpu -q -s -k "scale or covered or cfg3" > gpurun_out/fixtest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fixtest.log
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof.log 2>&1
echo "rc=$?" >> gpurun_out/setup_prof.log
