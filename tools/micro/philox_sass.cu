#include "../../paper_1305_6738_b200/csrc/zks_stream.cuh"
__global__ void k(unsigned long long* out, unsigned long long k0, unsigned long long k1) {
  const zks::Block4 r = zks::philox4x64_10(threadIdx.x + 1ull, k0, k1);
  out[threadIdx.x] = r.w[0] ^ r.w[1] ^ r.w[2] ^ r.w[3];
}
