// Micro-kernels that measure, on the device in use, the pipe peaks the replicate kernel is
// bound by: FP64 DFMA throughput, FP64 exp() throughput and 64x64->128 multiply throughput
// (Philox4x64).  bench.py divides the replicate kernel's counted work by these.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace zks {

__global__ void probe_dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void probe_exp_kernel(double* out, int iters, double step) {
  double acc0 = 0.0, acc1 = 0.0, x = -1e-3 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc0 += exp(x);
      acc1 += exp(x - 0.5);
      x -= step;
    }
  }
  if (acc0 + acc1 == 12345.678) out[0] = acc0;
}

__global__ void probe_mul64_kernel(unsigned long long* out, int iters, unsigned long long m) {
  unsigned long long x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = threadIdx.x * 2654435761ull + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = __umul64hi(x[j], m) ^ (x[j] * m);
  }
  if ((x[0] ^ x[1] ^ x[2] ^ x[3]) == 12345ull) out[0] = x[0];
}

// returns false on a CUDA error
inline bool probe_peaks(cudaStream_t stream, int sms, double* out) {
  double* sink = nullptr;
  if (cudaMalloc(&sink, 64) != cudaSuccess) return false;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 2048;
  const double lanes = double(blocks) * threads;
  double best[3] = {0.0, 0.0, 0.0};
  for (int rep = 0; rep < 3; ++rep) {
    float ms = 0.f;
    cudaEventRecord(e0, stream);
    probe_dfma_kernel<<<blocks, threads, 0, stream>>>(sink, iters, 0.999999, 1e-7);
    cudaEventRecord(e1, stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best[0] = fmax(best[0], 2.0 * 8 * 16 * iters * lanes / (ms * 1e-3));
    cudaEventRecord(e0, stream);
    probe_exp_kernel<<<blocks, threads, 0, stream>>>(sink, iters, 1e-6);
    cudaEventRecord(e1, stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best[1] = fmax(best[1], 8.0 * iters * lanes / (ms * 1e-3));
    cudaEventRecord(e0, stream);
    probe_mul64_kernel<<<blocks, threads, 0, stream>>>(reinterpret_cast<unsigned long long*>(sink), iters,
                                                       0xD2E7470EE14C6C93ull);
    cudaEventRecord(e1, stream);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best[2] = fmax(best[2], 4.0 * 16 * iters * lanes / (ms * 1e-3));
  }
  const bool ok = cudaGetLastError() == cudaSuccess;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  for (int i = 0; i < 3; ++i) out[i] = best[i];
  return ok;
}

}  // namespace zks
