mkdir -p gpurun_out
G='[{"krylov_maxit":2000,"nullspace_dim":4,"amg_theta":0.02},{"krylov_maxit":2000,"nullspace_dim":4,"amg_theta":0.04},{"krylov_maxit":2000,"nullspace_dim":4,"amg_theta":0.08},{"krylov_maxit":2000,"nullspace_dim":4,"amg_theta":0.12},{"krylov_maxit":2000,"nullspace_dim":4,"cheb_lower":0.1},{"krylov_maxit":2000,"nullspace_dim":4,"cheb_lower":0.01},{"krylov_maxit":2000,"nullspace_dim":4,"cheb_degree":2},{"krylov_maxit":2000,"nullspace_dim":4,"cheb_degree":4}]'
timeout 1200 python scripts/amg_sweep.py --config 4 --iterates 3,8,14 --grid "$G" > gpurun_out/sweep4b.log 2>&1
echo "rc=$?" >> gpurun_out/sweep4b.log
