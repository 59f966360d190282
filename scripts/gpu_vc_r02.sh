mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_amg.py -x -q > gpurun_out/amgtest.log 2>&1
for P in '{"nullspace_dim":4}' '{"nullspace_dim":4,"krylov_method":1}'; do
  echo "=== $P" >> gpurun_out/vc2.log
  timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --params "$P" >> gpurun_out/vc2.log 2>&1
done
