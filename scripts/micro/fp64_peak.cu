// fp64 FMA throughput microbenchmark (B200, sm_100a): many independent FMA chains per thread,
// all SMs, timed with CUDA events.  Reports TFLOP/s (2 flop per DFMA).  Used for the assembly
// kernel's fp64 ridge (verdict r1 item 5).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8, kIters = 4096;

__global__ void k_fma(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int threads = 256;
  for (int blocksPerSm : {4, 8, 16}) {
    const int blocks = sms * blocksPerSm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fma<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_fma<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * kChains * kIters * (double)blocks * threads * reps;
    const double tf = flops / (ms * 1e-3) / 1e12;
    printf("{\"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops_fp64\": %.2f}\n", blocksPerSm, ms / reps, tf);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
