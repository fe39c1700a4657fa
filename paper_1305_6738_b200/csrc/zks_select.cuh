// Order-statistic selection: the zero-based ranks floor(Decimal(q) * R) of R KS values
// (pkg/src/zipfks/montecarlo.py:119-136, order_quantiles) without sorting.
//
// KS values are non-negative doubles, so their IEEE-754 bit patterns are order-preserving
// uint64 keys.  Radix select, 8 passes of 8-bit digits, all requested ranks of up to
// kSelMaxArrays arrays (the cells of a sweep row) at once.  Every pass histograms, array by
// array, the digit of the keys that still match each rank's prefix (per block in shared memory,
// equal runs counted in registers) into the pass's histogram; then one warp per (array, rank)
// picks the digit holding the rank.  After the first two passes the keys matching a rank's
// 16-bit prefix are compacted, so passes 2-7 read only those (a few % of KS values).
//
// The arrays are processed concurrently (ArrayPart: each block works on one array at a time).
// Two drivers of the same steps:
//   * select_kernel: ONE cooperative launch, grid barriers between the steps (one GPU);
//   * select_{init,count,pick,out}_kernel: one launch per step, so that between count and pick
//     the caller can sum the pass histograms of every GPU holding a shard of the arrays (NCCL
//     all-reduce of 4 x 256 counts per cell): a distributed select whose key work stays
//     proportional to the local shard.
#pragma once
#include <cooperative_groups.h>

#include <cstdint>

namespace zks {

constexpr int kMaxRanks = 16;
constexpr int kSelMaxArrays = 24;
#ifndef ZKS_SEL_UNROLL
#define ZKS_SEL_UNROLL 16
#endif
constexpr int kSelUnroll = ZKS_SEL_UNROLL;  // key loads in flight per thread
constexpr int kSelectPasses = 8;
constexpr int kSelSlots = kSelMaxArrays * kMaxRanks;

struct SelectState {
  unsigned int hist[kSelectPasses][kSelSlots][256];  // cooperative driver: used slots zeroed per launch
  unsigned long long pre[kSelSlots], want[kSelSlots];
  int rep[kSelSlots];  // first rank of the same array with the same prefix (counted once)
  unsigned int worst[kSelMaxArrays];  // max status byte per array (optional)
  unsigned long long cand_n[kSelMaxArrays];  // keys matching a rank's 16-bit prefix (after pass 1)
};

// kernel parameters (< 4 KB): the arrays, their lengths, ranks and output pointers
struct SelectBatch {
  const unsigned long long* keys[kSelMaxArrays];
  long long count[kSelMaxArrays];
  double* out[kSelMaxArrays];
  unsigned long long rank[kSelMaxArrays][kMaxRanks];
  const unsigned char* status[kSelMaxArrays];  // optional: replicate status bytes (count[a] of them)
  unsigned char* worst[kSelMaxArrays];         // ... whose maximum lands here
  unsigned long long* cand;  // >= sum(count) keys: the candidates of passes 2..7, array after array
  int narrays, nr;
};

struct SelectShared {
  unsigned int sh[kMaxRanks][256];
  unsigned long long spre[kMaxRanks];
  int srep[kMaxRanks];
};

// Arrays are worked on concurrently: with G >= A blocks, array a takes the blocks b = a (mod A);
// with fewer blocks, block b takes the arrays a = b (mod G).  One block-wide histogram cycle per
// (block, array) instead of every block stepping through every array in turn.
struct ArrayPart {
  int a0, da;      // this block's first array and the step to its next one
  int lb, nb;      // this block's index among its array's blocks, and their number
  __device__ __forceinline__ ArrayPart(int narrays) {
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    if (G >= narrays) {
      a0 = b % narrays;
      da = G;  // one array per block
      lb = b / narrays;
      nb = (G - a0 + narrays - 1) / narrays;
    } else {
      a0 = b;
      da = G;
      lb = 0;
      nb = 1;
    }
  }
  __device__ __forceinline__ int64_t tid() const { return int64_t(lb) * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int64_t stride() const { return int64_t(nb) * blockDim.x; }
};

__device__ __forceinline__ int64_t array_offset(const SelectBatch& B, int a) {
  int64_t off = 0;
  for (int i = 0; i < a; ++i) off += B.count[i];
  return off;
}

// step 0: prefixes, remaining ranks, candidate counts, worst statuses (grid-stride over `tid`)
__device__ __forceinline__ void sel_init(const SelectBatch& B, SelectState* st, int64_t tid, int64_t stride) {
  const int nr = B.nr, slots = B.narrays * nr;
  for (int64_t s = tid; s < slots; s += stride) {
    st->pre[s] = 0ull;
    st->want[s] = B.rank[s / nr][s % nr];
  }
  if (tid < B.narrays) {
    st->worst[tid] = 0u;
    st->cand_n[tid] = 0ull;
  }
}

// worst status per array (montecarlo.py:106-115 failures surface as SimulationError on the host)
__device__ __forceinline__ void sel_worst(const SelectBatch& B, SelectState* st) {
  const ArrayPart P(B.narrays);
  for (int a = P.a0; a < B.narrays; a += P.da) {
    if (!B.status[a]) continue;
    const unsigned char* s8 = B.status[a];
    const int64_t n = B.count[a];
    unsigned w = 0;
    // 16-byte loads from the first aligned byte on, single bytes around them
    const int64_t lead = static_cast<int64_t>((16 - (reinterpret_cast<uintptr_t>(s8) & 15)) & 15);
    const int64_t head = lead < n ? lead : n;
    const int64_t n16 = (n - head) >> 4;
    const uint4* v = reinterpret_cast<const uint4*>(s8 + head);
    for (int64_t i = P.tid(); i < n16; i += P.stride()) {
      const uint4 q = __ldcs(v + i);
      w = __vmaxu4(w, __vmaxu4(__vmaxu4(q.x, q.y), __vmaxu4(q.z, q.w)));  // byte-wise maxima
    }
    w = max(max(w & 0xffu, (w >> 8) & 0xffu), max((w >> 16) & 0xffu, w >> 24));
    for (int64_t i = P.tid(); i < head; i += P.stride()) w = max(w, static_cast<unsigned>(s8[i]));
    for (int64_t i = head + (n16 << 4) + P.tid(); i < n; i += P.stride()) w = max(w, static_cast<unsigned>(s8[i]));
    w = __reduce_max_sync(0xffffffffu, w);
    if ((threadIdx.x & 31) == 0 && w) atomicMax(&st->worst[a], w);
  }
}

// one pass's digit counts of this block's keys into H[slot][256] (slot = array * nr + rank)
__device__ __forceinline__ void sel_count(const SelectBatch& B, SelectState* st, int pass, unsigned* H,
                                          SelectShared& S) {
  const int nr = B.nr;
  const int shift = 56 - 8 * pass;
  const unsigned long long mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
  const ArrayPart P(B.narrays);
  for (int a = P.a0; a < B.narrays; a += P.da) {
    for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) S.sh[i >> 8][i & 255] = 0u;
    if (threadIdx.x < nr) S.spre[threadIdx.x] = __ldcg(&st->pre[a * nr + threadIdx.x]);
    __syncthreads();
    if (threadIdx.x < nr) {
      int r0 = threadIdx.x;
      for (int q = 0; q < threadIdx.x; ++q)
        if (S.spre[q] == S.spre[threadIdx.x]) {
          r0 = q;
          break;
        }
      S.srep[threadIdx.x] = r0;
      if (P.lb == 0) st->rep[a * nr + threadIdx.x] = r0;
    }
    __syncthreads();
    // passes 0-1 read every key; later passes only the keys that matched a 16-bit prefix
    const unsigned long long* keys = pass < 2 ? B.keys[a] : B.cand + array_offset(B, a);
    const int64_t count = pass < 2 ? B.count[a] : static_cast<int64_t>(__ldcg(&st->cand_n[a]));
    // a thread's run of equal (rank, digit) hits is counted in registers and flushed to the
    // block histogram when it changes: the top digits of KS keys repeat (shared exponents)
    int run_r = -1;
    unsigned run_d = 0, run_n = 0;
    const int64_t stride = P.stride();
    for (int64_t i0 = P.tid(); i0 < count; i0 += kSelUnroll * stride) {
      unsigned long long kk[kSelUnroll];  // kSelUnroll loads in flight per thread
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u) {
        const int64_t i = i0 + u * stride;
        kk[u] = i < count ? __ldcg(keys + i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u) {
        if (i0 + u * stride >= count) break;
        const unsigned long long key = kk[u];
        const unsigned d = static_cast<unsigned>(key >> shift) & 255u;
        const unsigned long long top = key & mask;
        int hr = -1;
        for (int r = 0; r < nr; ++r)
          if (S.srep[r] == r && top == S.spre[r]) hr = r;
        if (hr < 0) continue;
        if (hr == run_r && d == run_d) {
          ++run_n;
        } else {
          if (run_n) atomicAdd(&S.sh[run_r][run_d], run_n);
          run_r = hr;
          run_d = d;
          run_n = 1;
        }
      }
    }
    if (run_n) atomicAdd(&S.sh[run_r][run_d], run_n);
    __syncthreads();
    for (int i = threadIdx.x; i < nr * 256; i += blockDim.x) {
      const unsigned v = S.sh[i >> 8][i & 255];
      if (v) atomicAdd(&H[(a * nr + (i >> 8)) * 256 + (i & 255)], v);
    }
    __syncthreads();
  }
}

// the digit holding each rank, from the pass's (summed) histogram: one warp per (array, rank)
__device__ __forceinline__ void sel_pick(const SelectBatch& B, SelectState* st, int pass, const unsigned* H, int gwarp,
                                         int nwarps) {
  const int nr = B.nr, slots = B.narrays * nr, lane = threadIdx.x & 31;
  const int shift = 56 - 8 * pass;
  for (int s = gwarp; s < slots; s += nwarps) {
    const int a = s / nr;
    const unsigned* h = H + (a * nr + __ldcg(&st->rep[s])) * 256;
    const unsigned long long w = __ldcg(&st->want[s]);
    // lane owns bins [8*lane, 8*lane + 8)
    unsigned c[8];
    unsigned long long own = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = __ldcg(h + 8 * lane + j);
      own += c[j];
    }
    unsigned long long incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned long long excl = incl - own;
    const unsigned hit = __ballot_sync(0xffffffffu, excl <= w && w < incl);
    const int owner = hit ? __ffs(hit) - 1 : 31;
    if (lane == owner) {
      unsigned long long cum = excl;
      unsigned digit = 8 * lane + 7;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (cum + c[j] > w) {
          digit = 8 * lane + j;
          break;
        }
        cum += c[j];
      }
      st->pre[s] = __ldcg(&st->pre[s]) | (static_cast<unsigned long long>(digit) << shift);
      st->want[s] = w - cum;
    }
  }
}

// the keys still matching a rank's 16-bit prefix, per array, into B.cand (after pass 1's pick)
__device__ __forceinline__ void sel_compact(const SelectBatch& B, SelectState* st, SelectShared& S) {
  const int nr = B.nr, lane = threadIdx.x & 31;
  const ArrayPart P(B.narrays);
  for (int a = P.a0; a < B.narrays; a += P.da) {
    if (threadIdx.x < nr) S.spre[threadIdx.x] = __ldcg(&st->pre[a * nr + threadIdx.x]);
    __syncthreads();
    const unsigned long long* keys = B.keys[a];
    unsigned long long* cand = B.cand + array_offset(B, a);
    const int64_t n = B.count[a], stride = P.stride();
    for (int64_t base = int64_t(P.lb) * blockDim.x; base < n; base += kSelUnroll * stride) {
      unsigned long long kk[kSelUnroll];
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u) {
        const int64_t i = base + u * stride + threadIdx.x;
        kk[u] = i < n ? __ldcg(keys + i) : ~0ull;
      }
#pragma unroll
      for (int u = 0; u < kSelUnroll; ++u) {
        const int64_t i = base + u * stride + threadIdx.x;  // whole warps iterate together (ballot below)
        const unsigned long long top = kk[u] & (~0ull << 48);
        bool hit = false;
        for (int r = 0; r < nr; ++r) hit |= i < n && top == S.spre[r];
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (m) {
          unsigned long long at = 0;
          if (lane == 0) at = atomicAdd(&st->cand_n[a], static_cast<unsigned long long>(__popc(m)));
          at = __shfl_sync(0xffffffffu, at, 0);
          if (hit) {
            ZKS_CHECK(at + __popc(m & ((1u << lane) - 1u)) < static_cast<unsigned long long>(n));
            cand[at + __popc(m & ((1u << lane) - 1u))] = kk[u];
          }
        }
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void sel_out(const SelectBatch& B, SelectState* st, int64_t tid, int64_t stride) {
  const int nr = B.nr, slots = B.narrays * nr;
  for (int64_t s = tid; s < slots; s += stride)
    B.out[s / nr][s % nr] = __longlong_as_double(static_cast<long long>(__ldcg(&st->pre[s])));
  if (tid < B.narrays && B.worst[tid]) *B.worst[tid] = static_cast<unsigned char>(__ldcg(&st->worst[tid]));
}

__global__ void __launch_bounds__(256) select_kernel(SelectBatch B, SelectState* st) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ SelectShared S;
  static_assert(sizeof(SelectBatch) <= 4096, "kernel parameters");
  const int slots = B.narrays * B.nr;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = tid; i < int64_t(kSelectPasses) * slots * 256; i += stride)
    st->hist[i / (slots * 256)][(i / 256) % slots][i & 255] = 0u;
  sel_init(B, st, tid, stride);
  grid.sync();
  sel_worst(B, st);
  const int gwarp = static_cast<int>(tid >> 5), nwarps = static_cast<int>(stride >> 5);
  for (int pass = 0; pass < kSelectPasses; ++pass) {
    unsigned* H = &st->hist[pass][0][0];
    sel_count(B, st, pass, H, S);
    grid.sync();
    sel_pick(B, st, pass, H, gwarp, nwarps);
    grid.sync();
    if (pass == 1) {
      sel_compact(B, st, S);
      grid.sync();
    }
  }
  sel_out(B, st, tid, stride);
}

// the same steps as separate launches (distributed select; H = the caller's [slots][256]
// histogram of the pass, zeroed before count and summed over GPUs before pick)
__global__ void __launch_bounds__(256) select_init_kernel(SelectBatch B, SelectState* st) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  sel_init(B, st, tid, int64_t(gridDim.x) * blockDim.x);
}
__global__ void __launch_bounds__(256) select_count_kernel(SelectBatch B, SelectState* st, int pass, unsigned* H) {
  __shared__ SelectShared S;
  if (pass == 0) sel_worst(B, st);
  sel_count(B, st, pass, H, S);
}
__global__ void __launch_bounds__(256) select_pick_kernel(SelectBatch B, SelectState* st, int pass, const unsigned* H) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  sel_pick(B, st, pass, H, static_cast<int>(tid >> 5), static_cast<int>((int64_t(gridDim.x) * blockDim.x) >> 5));
}
__global__ void __launch_bounds__(256) select_compact_kernel(SelectBatch B, SelectState* st) {
  __shared__ SelectShared S;
  sel_compact(B, st, S);
}
__global__ void __launch_bounds__(256) select_out_kernel(SelectBatch B, SelectState* st) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  sel_out(B, st, tid, int64_t(gridDim.x) * blockDim.x);
}

}  // namespace zks
