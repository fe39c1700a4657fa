// Order-statistic selection: the zero-based ranks floor(Decimal(q) * R) of R KS values
// (pkg/src/zipfks/montecarlo.py:119-136, order_quantiles) without sorting.
//
// KS values are non-negative doubles, so their IEEE-754 bit patterns are order-preserving
// uint64 keys.  Radix select, 8 passes of 8-bit digits, all requested ranks at once: every pass
// histograms the digit of the keys that still match each rank's prefix (block-local shared
// histograms merged into global), and the last block to finish picks each rank's digit.
// Traffic per pass is one read of the R keys (8 B each).
#pragma once
#include <cstdint>

namespace zks {

constexpr int kMaxRanks = 16;

struct SelectState {
  unsigned long long prefix[kMaxRanks];
  unsigned long long rank[kMaxRanks];
  unsigned int hist[kMaxRanks][256];
  unsigned int done;
};

struct RankList {
  unsigned long long rank[kMaxRanks];
};

// reset the selection state on the stream (ranks travel as a kernel parameter: no host copy)
__global__ void select_init_kernel(SelectState* st, RankList ranks, int nr) {
  for (int i = threadIdx.x; i < kMaxRanks * 256; i += blockDim.x) st->hist[i >> 8][i & 255] = 0u;
  if (threadIdx.x < kMaxRanks) {
    st->prefix[threadIdx.x] = 0ull;
    st->rank[threadIdx.x] = threadIdx.x < nr ? ranks.rank[threadIdx.x] : 0ull;
  }
  if (threadIdx.x == 0) st->done = 0u;
}

// one 8-bit digit pass; the pass at shift 0 writes the selected values to out[0..nr)
__global__ void __launch_bounds__(256) select_pass_kernel(const unsigned long long* __restrict__ keys, int64_t count,
                                                          int shift, SelectState* st, int nr, double* out) {
  __shared__ unsigned int sh[kMaxRanks][256];
  __shared__ unsigned long long pre[kMaxRanks];
  __shared__ bool last;
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) sh[i >> 8][i & 255] = 0u;
  if (threadIdx.x < nr) pre[threadIdx.x] = st->prefix[threadIdx.x];
  __syncthreads();
  const unsigned long long mask = (shift >= 56) ? 0ull : (~0ull << (shift + 8));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = keys[i];
    const unsigned d = static_cast<unsigned>(key >> shift) & 255u;
    const unsigned long long top = key & mask;
    for (int r = 0; r < nr; ++r)
      if (top == pre[r]) atomicAdd(&sh[r][d], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) {
    const unsigned v = sh[i >> 8][i & 255];
    if (v) atomicAdd(&st->hist[i >> 8][i & 255], v);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&st->done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < nr) {
    const int r = threadIdx.x;
    volatile unsigned int* h = st->hist[r];
    unsigned long long want = st->rank[r], cum = 0;
    unsigned digit = 255;
    for (unsigned d = 0; d < 256; ++d) {
      const unsigned long long c = h[d];
      if (cum + c > want) {
        digit = d;
        break;
      }
      cum += c;
    }
    const unsigned long long key = pre[r] | (static_cast<unsigned long long>(digit) << shift);
    st->prefix[r] = key;
    st->rank[r] = want - cum;
    if (shift == 0) out[r] = __longlong_as_double(static_cast<long long>(key));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) st->hist[i >> 8][i & 255] = 0u;
  if (threadIdx.x == 0) st->done = 0u;
}

}  // namespace zks
