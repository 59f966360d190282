// common.cuh — context, memory, errors, launch helpers and deterministic reductions
// for the B200 sea-ice Newton-Krylov library (sm_100a, fp64 throughout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/seaice.h"

namespace seaice {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SI_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess)                                                                  \
      throw ::seaice::Error(SEAICE_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                              " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

#define SI_CHECK(cond, code, msg)                          \
  do {                                                     \
    if (!(cond)) throw ::seaice::Error((code), (msg));     \
  } while (0)

constexpr int kThreads = 256;
constexpr int kRedBlocks = 1184;  // 148 SMs x 8: fixed grid => fixed summation order

inline int grid_for(long long n, int threads = kThreads) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)g;
}
inline int red_grid(long long n) {
  long long g = (n + kThreads - 1) / kThreads;
  if (g > kRedBlocks) g = kRedBlocks;
  if (g < 1) g = 1;
  return (int)g;
}

// ----------------------------------------------------------------- device memory
struct Allocator {
  seaice_runtime rt{};
  cudaStream_t s = nullptr;
  size_t live_bytes = 0, peak_bytes = 0;
  void* alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    void* p = nullptr;
    if (rt.alloc) {
      p = rt.alloc(bytes, (void*)s, rt.user);
      if (!p) throw Error(SEAICE_ENOMEM, "allocation callback returned NULL for " + std::to_string(bytes) + " B");
    } else {
      cudaError_t e = cudaMallocAsync(&p, bytes, s);
      if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(SEAICE_ENOMEM, "cudaMallocAsync(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
      }
    }
    live_bytes += bytes;
    if (live_bytes > peak_bytes) peak_bytes = live_bytes;
    return p;
  }
  void release(void* p, size_t bytes) {
    if (!p) return;
    if (rt.free)
      rt.free(p, (void*)s, rt.user);
    else
      cudaFreeAsync(p, s);
    live_bytes -= bytes;
  }
};

// Grow-only typed device buffer owned by a context.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  Allocator* A = nullptr;
  void ensure(Allocator& al, size_t n) {
    A = &al;
    if (n <= cap) return;
    if (p) al.release(p, cap * sizeof(T));
    p = (T*)al.alloc(n * sizeof(T));
    cap = n;
  }
  void free_() {
    if (p && A) A->release(p, cap * sizeof(T));
    p = nullptr;
    cap = 0;
  }
  T* get() const { return p; }
};

// ----------------------------------------------------------------- reductions
// Deterministic two-stage reductions: stage 1 writes one partial per block (fixed
// grid, fixed in-block tree), stage 2 sums the partials in one block in fixed order.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum, result valid in thread 0. blockDim.x multiple of 32, <= 1024.
__device__ __forceinline__ double block_sum(double v, double* sh /*[32]*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (wid == 0) v = warp_sum(v);
  return v;
}

}  // namespace seaice
