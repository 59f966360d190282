mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -s -k "scale or config4 or hierarchy or vcycle" > gpurun_out/amgtest.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof10.log 2>&1
