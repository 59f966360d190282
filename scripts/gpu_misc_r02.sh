mkdir -p gpurun_out
timeout 900 python scripts/kernel_bench.py --config 5 --reps 10 > gpurun_out/kernel_bench_cfg5.json 2> gpurun_out/kernel_bench_cfg5.err
timeout 900 python bench.py --cpu-kernels --sample-n 512 > gpurun_out/cpu_kernels.json 2> gpurun_out/cpu_kernels.err
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof7.log 2>&1
