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
__device__ __forceinline__ void sel_worst(const SelectBatch& B, SelectState* st, int64_t tid, int64_t stride) {
  for (int a = 0; a < B.narrays; ++a) {
    if (!B.status[a]) continue;
    unsigned w = 0;
    for (int64_t i = tid; i < B.count[a]; i += stride) w = max(w, static_cast<unsigned>(B.status[a][i]));
    w = __reduce_max_sync(0xffffffffu, w);
    if ((threadIdx.x & 31) == 0 && w) atomicMax(&st->worst[a], w);
  }
}

// one pass's digit counts of this block's keys into H[slot][256] (slot = array * nr + rank)
__device__ __forceinline__ void sel_count(const SelectBatch& B, SelectState* st, int pass, unsigned* H,
                                          SelectShared& S, int64_t tid, int64_t stride) {
  const int nr = B.nr;
  const int shift = 56 - 8 * pass;
  const unsigned long long mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
  int64_t off = 0;
  for (int a = 0; a < B.narrays; ++a) {
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
      if (blockIdx.x == 0) st->rep[a * nr + threadIdx.x] = r0;
    }
    __syncthreads();
    // passes 0-1 read every key; later passes only the keys that matched a 16-bit prefix
    const unsigned long long* keys = pass < 2 ? B.keys[a] : B.cand + off;
    const int64_t count = pass < 2 ? B.count[a] : static_cast<int64_t>(__ldcg(&st->cand_n[a]));
    off += B.count[a];
    // a thread's run of equal (rank, digit) hits is counted in registers and flushed to the
    // block histogram when it changes: the top digits of KS keys repeat (shared exponents)
    int run_r = -1;
    unsigned run_d = 0, run_n = 0;
    for (int64_t i = tid; i < count; i += stride) {
      const unsigned long long key = __ldcg(keys + i);
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
__device__ __forceinline__ void sel_compact(const SelectBatch& B, SelectState* st, SelectShared& S, int64_t stride) {
  const int nr = B.nr, lane = threadIdx.x & 31;
  int64_t off = 0;
  for (int a = 0; a < B.narrays; ++a) {
    if (threadIdx.x < nr) S.spre[threadIdx.x] = __ldcg(&st->pre[a * nr + threadIdx.x]);
    __syncthreads();
    const unsigned long long* keys = B.keys[a];
    unsigned long long* cand = B.cand + off;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < B.count[a]; base += stride) {
      const int64_t i = base + threadIdx.x;  // whole warps iterate together (ballot below)
      const unsigned long long key = i < B.count[a] ? __ldcg(keys + i) : ~0ull;
      const unsigned long long top = key & (~0ull << 48);
      bool hit = false;
      for (int r = 0; r < nr; ++r) hit |= i < B.count[a] && top == S.spre[r];
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (m) {
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&st->cand_n[a], static_cast<unsigned long long>(__popc(m)));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (hit) cand[at + __popc(m & ((1u << lane) - 1u))] = key;
      }
    }
    off += B.count[a];
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
  sel_worst(B, st, tid, stride);
  const int gwarp = static_cast<int>(tid >> 5), nwarps = static_cast<int>(stride >> 5);
  for (int pass = 0; pass < kSelectPasses; ++pass) {
    unsigned* H = &st->hist[pass][0][0];
    sel_count(B, st, pass, H, S, tid, stride);
    grid.sync();
    sel_pick(B, st, pass, H, gwarp, nwarps);
    grid.sync();
    if (pass == 1) {
      sel_compact(B, st, S, stride);
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
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (pass == 0) sel_worst(B, st, tid, stride);
  sel_count(B, st, pass, H, S, tid, stride);
}
__global__ void __launch_bounds__(256) select_pick_kernel(SelectBatch B, SelectState* st, int pass, const unsigned* H) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  sel_pick(B, st, pass, H, static_cast<int>(tid >> 5), static_cast<int>((int64_t(gridDim.x) * blockDim.x) >> 5));
}
__global__ void __launch_bounds__(256) select_compact_kernel(SelectBatch B, SelectState* st) {
  __shared__ SelectShared S;
  sel_compact(B, st, S, int64_t(gridDim.x) * blockDim.x);
}
__global__ void __launch_bounds__(256) select_out_kernel(SelectBatch B, SelectState* st) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  sel_out(B, st, tid, int64_t(gridDim.x) * blockDim.x);
}

}  // namespace zks
