# streamed finest Chebyshev: parity vs per-step, then V-cycle timing tile vs streamed
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_amg.py -m gpu -q -x -k "fused_chebyshev" > gpurun_out/stream_test.log 2>&1
echo "pytest rc=$?" >> gpurun_out/stream_test.log
timeout 600 python scripts/vcycle_bench.py --params '{"cheb_fused":2}' > gpurun_out/vc_stream.log 2>&1
