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
  __shared__ int rep[kMaxRanks];  // first rank with the same prefix: ranks sharing one are counted once
  __shared__ bool last;
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) sh[i >> 8][i & 255] = 0u;
  if (threadIdx.x < nr) pre[threadIdx.x] = st->prefix[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nr) {
    int r0 = threadIdx.x;
    for (int q = 0; q < threadIdx.x; ++q)
      if (pre[q] == pre[threadIdx.x]) {
        r0 = q;
        break;
      }
    rep[threadIdx.x] = r0;
  }
  __syncthreads();
  const unsigned long long mask = (shift >= 56) ? 0ull : (~0ull << (shift + 8));
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < count; base += stride) {
    const int64_t i = base + threadIdx.x;  // whole warps iterate together (ballot / match below)
    const bool valid = i < count;
    const unsigned long long key = valid ? keys[i] : 0ull;
    const unsigned d = static_cast<unsigned>(key >> shift) & 255u;
    const unsigned long long top = key & mask;
    for (int r = 0; r < nr; ++r) {
      if (rep[r] != r) continue;
      const bool hit = valid && top == pre[r];
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        // warp-aggregated increment: KS keys crowd a few digits (shared exponent bits)
        const unsigned peers = __match_any_sync(m, d);
        if (lane == __ffs(peers) - 1) atomicAdd(&sh[r][d], static_cast<unsigned>(__popc(peers)));
      }
    }
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
  // stage the merged histograms (coalesced, L2) into shared memory, then one warp per rank
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) sh[i >> 8][i & 255] = __ldcg(&st->hist[i >> 8][i & 255]);
  __syncthreads();
  for (int r = threadIdx.x >> 5; r < nr; r += blockDim.x >> 5) {
    const unsigned* h = sh[rep[r]];
    const unsigned long long want = st->rank[r];
    // lane owns bins [8*lane, 8*lane + 8)
    unsigned long long own = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) own += h[8 * lane + j];
    unsigned long long incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned long long excl = incl - own;
    const unsigned hit = __ballot_sync(0xffffffffu, excl <= want && want < incl);
    const int owner = hit ? __ffs(hit) - 1 : 31;
    if (lane == owner) {
      unsigned long long cum = excl;
      unsigned digit = 8 * lane + 7;
      for (int j = 0; j < 8; ++j) {
        const unsigned long long c = h[8 * lane + j];
        if (cum + c > want) {
          digit = 8 * lane + j;
          break;
        }
        cum += c;
      }
      const unsigned long long key = pre[r] | (static_cast<unsigned long long>(digit) << shift);
      st->prefix[r] = key;
      st->rank[r] = want - cum;
      if (shift == 0) out[r] = __longlong_as_double(static_cast<long long>(key));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) st->hist[i >> 8][i & 255] = 0u;
  if (threadIdx.x == 0) st->done = 0u;
}

}  // namespace zks
