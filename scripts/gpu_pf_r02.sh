mkdir -p gpurun_out
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_pf2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_amg.py -q -x -k "vcycle or tail or fused or counts" > gpurun_out/pf_test.log 2>&1
echo "rc=$?" >> gpurun_out/pf_test.log
