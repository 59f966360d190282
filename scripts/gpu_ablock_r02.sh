# coarse row-component kernels: block size / persistent grid sweep (V-cycle at config 4), GPU tests, bench with restart 60
mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_ab256.log 2>&1
for b in 64 128; do
SEAICE_ABLOCK=$b timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_ab$b.log 2>&1
done
SEAICE_AGRID_CAP=1184 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_ab256_cap1184.log 2>&1
SEAICE_ABLOCK=128 SEAICE_AGRID_CAP=2368 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_ab128_cap2368.log 2>&1
SEAICE_ABLOCK=64 SEAICE_AGRID_CAP=4736 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_ab64_cap4736.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_m60.log 2>&1
