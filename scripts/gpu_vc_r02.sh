mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 20 > gpurun_out/vc5.log 2>&1
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 --params '{"krylov_forcing":1}' > gpurun_out/setup_prof.log 2>&1
timeout 600 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amgtest.log 2>&1
