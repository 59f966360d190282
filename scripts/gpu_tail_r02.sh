# persistent V-cycle tail: parity tests, V-cycle timing on/off and CTA-count sweep, per-solve log of config 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "tail or vcycle or fused" > gpurun_out/tail_test.log 2>&1
echo "rc=$?" >> gpurun_out/tail_test.log
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 --params '{"vcycle_tail":0}' > gpurun_out/vc_tail0.log 2>&1
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_tail1.log 2>&1
for k in 1 2 8; do
SEAICE_TAIL_CTAS=$k timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_tail1_c$k.log 2>&1
done
SEAICE_TAIL_MB=250 timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_tail1_mb250.log 2>&1
timeout 600 python scripts/probe_steps.py --config 4 --steps 5 --newton-log > gpurun_out/probe_cfg4.log 2>&1
