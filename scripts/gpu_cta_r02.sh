mkdir -p gpurun_out
timeout 600 python scripts/vcycle_bench.py > gpurun_out/vc_cta48.log 2>&1
SEAICE_CTA_MINROW=32 timeout 600 python scripts/vcycle_bench.py > gpurun_out/vc_cta32.log 2>&1
SEAICE_CTA_MINROW=32 SEAICE_CTA_MAXNB=1000 timeout 600 python scripts/vcycle_bench.py > gpurun_out/vc_cta32s.log 2>&1
SEAICE_CTA_MINROW=16 SEAICE_CTA_MAXNB=1000 timeout 600 python scripts/vcycle_bench.py > gpurun_out/vc_cta16s.log 2>&1
