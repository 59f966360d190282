mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm,clocks.max.mem,temperature.gpu,power.draw,clocks_throttle_reasons.active --format=csv > gpurun_out/chk_smi.log 2>&1
timeout 300 python scripts/vcycle_bench.py --config 4 --iterate 8 --reps 50 > gpurun_out/vc_chk.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,temperature.gpu,power.draw --format=csv >> gpurun_out/chk_smi.log 2>&1
