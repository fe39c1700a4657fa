// On-box microbenchmarks for the non-tensor pipes this engine is bound by:
// FP64 DFMA throughput, 64x64->128 multiply throughput (Philox core), and FP64 exp().
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void mul64_kernel(uint64_t* out, int iters, uint64_t m) {
  uint64_t x0 = threadIdx.x + 1, x1 = x0 * 3, x2 = x0 * 5, x3 = x0 * 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = __umul64hi(x0, m) ^ (x0 * m);
      x1 = __umul64hi(x1, m) ^ (x1 * m);
      x2 = __umul64hi(x2, m) ^ (x2 * m);
      x3 = __umul64hi(x3, m) ^ (x3 * m);
    }
  }
  uint64_t s = x0 ^ x1 ^ x2 ^ x3;
  if (s == 12345) out[0] = s;
}

__global__ void exp_kernel(double* out, int iters, double g) {
  double acc = 0.0, x = -1e-3 * threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc += exp(x); x -= g; }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("device %s sms %d\n", p.name, sms);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4096;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(dout, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    mul64_kernel<<<blocks, threads>>>((uint64_t*)dout, iters, 0xD2E7470EE14C6C93ull);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double muls = 4.0 * 16 * (double)iters * blocks * threads;
    printf("mulhilo64: %.1f G/s (%.3f ms)\n", muls / ms / 1e6, ms);
    cudaEventRecord(e0);
    exp_kernel<<<blocks, threads>>>(dout, iters, 1e-6);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double exps = 8.0 * (double)iters * blocks * threads;
    printf("fp64 exp: %.1f G/s (%.3f ms)\n", exps / ms / 1e6, ms);
  }
  return 0;
}
