# SpGEMM: pipelined numeric rows + per-lane symbolic inserts: hierarchy parity on every path, setup profile, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "hierarchy or galerkin or reuse or counts" > gpurun_out/sg_test.log 2>&1
echo "rc=$?" >> gpurun_out/sg_test.log
timeout 600 python scripts/setup_profile.py --steps 1 --warmup 3 > gpurun_out/setup_prof3.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_sg.log 2>&1
