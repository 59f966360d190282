mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/micro/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.log 2>&1
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 20 > gpurun_out/vc6.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amgtest.log 2>&1
timeout 900 python scripts/zeta_spread.py --config 3 > gpurun_out/zeta3.jsonl 2> gpurun_out/zeta3.err
