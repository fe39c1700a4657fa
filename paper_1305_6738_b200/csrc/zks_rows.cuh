// Sweep rows: one replicate stream drawn once, counted for every gamma of the row.
//
// build_table seeds every cell with the same base_seed (pkg/src/zipfks/montecarlo.py:276-277),
// so the cells of a row (equal n and repetition, gammas differ) draw replicate index i from the
// identical uniforms u_j = 1 - m_j 2^-53, m_j = x_j >> 11 of Philox word x_j
// (distribution.py:182-187).  A cell's sample is sample() (distribution.py:190-201) of those
// uniforms: value v_j = 1 + #{k : cdf[k] < u_j}, clamped to L.  Since u > h <=> m < M(h), the
// exact 53-bit cut M(h) = #{m : 1 - m 2^-53 > h}, a cell's counts of the values 1..64 follow
// from where its 64 cuts M_k = M(cdf[k]) fall among the row's keys:
//   #{v_j >= k + 2} = P_k = #{m_j < M_k} (cdf non-decreasing => M non-increasing),
//   count(1) = n - P_0,  count(k) = P_{k-2} - P_{k-1} (k = 2..64),
// and the P_63 keys below M_63 are exactly the draws above 64, resolved one by one by the guide
// + cdf search -- or, for a dense finite support (64 < K <= 1024), counted the same way from all
// K - 1 cut positions (count(k) = P_{k-2} - P_{k-1}), with no per-draw search at all.  So per row the kernel draws and buckets n keys once (Philox4x64 + a counting
// sort by the keys' top bits, on chip) and per cell does 64 short bucket scans plus its tail --
// instead of generating or re-reading and classifying all n draws once per gamma.  Entries of
// the cut table from L - 1 on are 0 (the clamp to L: no draw counts above it).
//
// Output per (cell, replicate) is draw_stats_kernel's pre-drawn row (zks_batch.cuh): u16 counts
// of 1..64, the tail values or, for 64 < K <= 1024, u32 counts of 65..vmax, log-sum, min, max,
// tail length -- the input of fit_ks_kernel / retry_kernel.  Single cells in the same n range
// run through here too (ncells = 1), so a cell's results do not depend on whether it was
// computed alone or in a row.
//
// Keys are only bucketed (about two per bucket, buckets in key order), not sorted: a cut's
// position is its bucket's start plus the keys of that bucket below it, and the tail is every
// key below M_63 -- all keys of the buckets under M_63's bucket and those of that bucket below
// it.  The order inside a bucket comes from shared-memory atomics and varies between runs, so
// everything summed over keys is order-free: the log-sum is accumulated in 128-bit fixed point
// (every ln v, v >= 2, is a multiple of 2^-53 below 2^4: ln v 2^53 is an exact integer < 2^57),
// exact and therefore identical for any order; the tail list's order does not matter to the
// fit kernel (it sorts, or histograms, the tail).
#pragma once
#include "zks_batch.cuh"

namespace zks {

constexpr int kRowMaxCells = 32;
constexpr int kRowMaxN = 16384;      // keys (8 B each) + buckets of one row in shared memory
constexpr int kRowStageMaxN = 2048;  // up to here the draw pass parks the keys in shared memory for
                                     // the scatter pass; above it the scatter pass regenerates them
#ifndef ZKS_ROW_MINB
#define ZKS_ROW_MINB 4
#endif

// Exact 53-bit cut of a cdf entry h: the smallest m <= 2^53 with 1 - m 2^-53 <= h (so u > h
// <=> m < M).  1 - m 2^-53 is exact for every m <= 2^53; the estimate from (1 - h) 2^53 is off
// by at most one or two and fixed by the exact test.  h >= 1 (and +inf) gives 0.
__device__ __forceinline__ unsigned long long exact_cut(double h) {
  if (!(h < 1.0)) return 0ull;
  constexpr unsigned long long kTop = 1ull << 53;
  const double d = (1.0 - h) * 0x1p53;
  unsigned long long m = d >= 0x1p53 ? kTop : static_cast<unsigned long long>(ceil(d));
  auto le = [h](unsigned long long mm) { return 1.0 - static_cast<double>(mm) * 0x1p-53 <= h; };
  while (m > 0ull && le(m - 1ull)) --m;
  while (m < kTop && !le(m)) ++m;
  return m;
}

// The cut table of a sampling table: kCutMax entries, so a dense finite support (K <= kDenseMaxK)
// has every cut; from L - 1 on: 0 (the clamp)
constexpr int kCutMax = 1024;
static_assert(kCutMax >= kDenseMaxK, "dense supports take every count from cut positions");
__global__ void cut_kernel(const double* __restrict__ cdf, uint32_t L, unsigned long long* mcut) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < kCutMax) mcut[j] = static_cast<uint32_t>(j) + 1u < L ? exact_cut(cdf[j]) : 0ull;
}

struct RowCell {
  const double* cdf;
  const uint16_t* guide;       // levels 1 and 2 (global memory)
  const uint16_t* guide_fine;  // fine level 2
  const unsigned long long* mcut;
  uint32_t L;
  int guide_levels;
  // this chunk's pre-drawn rows of the cell (row i = replicate first + i)
  uint16_t* head;
  uint16_t* tail;
  uint32_t* m;
  double* ls;
  uint32_t* mn;
  uint32_t* mx;
};

struct RowArgs {
  uint64_t seed, rep, first, count;
  int n;
  int vals_stride;   // u16 slots per tail row (u32 counts when dense)
  int dense_words;   // K - kKsHead for kKsHead < K <= kDenseMaxK, else 0
  int ncells;
  int bucket_bits;   // keys are bucketed by their top bits: 2^bucket_bits buckets
  const double* logs;
  unsigned long long* counters;
  int rng;  // kRngNumpy or kRngPhilox4x32
  // the block's cell schedule: warp w takes cells order[wbeg[w] .. wbeg[w + 1]) (longest
  // processing time first over the host's cost estimates); the last warp, the least loaded, also
  // derives the next row's stream key
  uint8_t order[kRowMaxCells];
  uint8_t wbeg[kWarps + 1];
  RowCell cell[kRowMaxCells];
};

__host__ __device__ constexpr int row_bucket_bits(int n) {
  int b = 0;
  while ((1 << b) < n) ++b;  // ceil(log2 n): about one key per bucket
  // larger rows: 2 (512 < n <= 2048, keys parked) and 4 to 8 keys per bucket, so the 12 B per
  // bucket do not cost a resident block beside the keys' 8-16 n B (measured: n = 700 -7 %,
  // n = 1000 -5 % with 4-warp blocks, n = 2000 -8 %, n = 5000 -43 %)
  if (n > 512) b -= 1;
  if (n > kRowStageMaxN) b -= 2;
  return b < 4 ? 4 : (b > 12 ? 12 : b);  // <= 4096 buckets
}
constexpr int kRowKeyPad = 2;  // sentinel keys (all ones) after the row: pair loads past a bucket's end
// shared memory of one block of `warps` warps: keys + sentinels (+ the parked draw pass), bucket
// starts, ends and counts, and (dense supports, n <= kRowDenseHistMaxN) per-warp histograms of 65..K
constexpr int kRowDenseHistMaxN = 4096;
__host__ __device__ constexpr size_t row_smem_bytes(int n, int dense_words, int warps, int bits) {
  return size_t(round_up(n + kRowKeyPad, 2)) * 8 + (n <= kRowStageMaxN ? size_t(round_up(n, 2)) * 8 : 0) +
         (size_t(1) << bits) * 12 + (n <= kRowDenseHistMaxN ? size_t(warps) * dense_words * 4 : 0);
}


// one cell of the row, by one warp: counts of 1..64 from the cut positions, the tail by search
template <bool kCount>
__device__ __forceinline__ void row_cell(const RowArgs& a, const RowCell& C, uint64_t i,
                                         const unsigned long long* __restrict__ keys, const uint32_t* bstart,
                                         const uint32_t* bend, uint32_t* dense, int lane, unsigned long long& tails) {
  const int n = a.n;
  const int shift = 53 - a.bucket_bits;
  const uint32_t nbk = 1u << a.bucket_bits;
  // P = #{keys < M}: the start of M's bucket plus that bucket's keys below M (about one: the
  // first two are read unconditionally, the sentinels cover the row's end)
  auto pos = [&](unsigned long long M) -> uint32_t {
    const uint32_t bk = static_cast<uint32_t>(M >> shift);
    if (bk >= nbk) return static_cast<uint32_t>(n);
    const uint32_t p = bstart[bk], e = bend[bk];
    const unsigned long long x0 = keys[p], x1 = keys[p + 1];
    uint32_t r = p + (p < e && x0 < M) + (p + 1 < e && x1 < M);
    if (e > p + 2) {
#pragma unroll 1
      for (uint32_t s = p + 2; s < e; ++s) r += keys[s] < M;
    }
    return r;
  };
  const unsigned long long Ma = __ldg(C.mcut + lane), Mb = __ldg(C.mcut + 32 + lane);
  const uint32_t Pa = pos(Ma), Pb = pos(Mb);
  const uint32_t Pa_up = __shfl_up_sync(0xffffffffu, Pa, 1), Pb_up = __shfl_up_sync(0xffffffffu, Pb, 1);
  const uint32_t Pa31 = __shfl_sync(0xffffffffu, Pa, 31);
  const uint32_t c0 = (lane ? Pa_up : static_cast<uint32_t>(n)) - Pa;  // count of value lane + 1
  const uint32_t c1 = (lane ? Pb_up : Pa31) - Pb;                       // count of value lane + 33
  const uint32_t T = __shfl_sync(0xffffffffu, Pb, 31);                  // draws above kKsHead
  unsigned long long shi = 0, slo = 0;  // log-sum, 2^-53 units
  uint32_t vtop = 0, vlow = 0xffffffffu;
  // dense finite support (kKsHead < K <= kDenseMaxK): u32 counts of kKsHead+1..vmax into the
  // row's tail slot (what fit_ks_kernel reads) -- from the K - 65 remaining cut positions, or, when
  // the tail is short against them, from the per-draw searches counted in the warp's histogram
  // (the same counts and, summed exactly, the same log-sum either way)
  const bool by_cuts = a.dense_words && (!dense || T >= static_cast<uint32_t>(a.dense_words) / 4u);
  if (T && by_cuts) {
    // count(k) = P_{k-2} - P_{k-1}, P_{K-1} = 0: no per-draw search
    uint32_t* out = reinterpret_cast<uint32_t*>(C.tail + i * a.vals_stride);
    uint32_t prev = T;  // P_63
    for (int j0 = kKsHead; j0 < a.dense_words + kKsHead; j0 += 32) {
      const int j = j0 + lane;
      const uint32_t P = j < kCutMax ? pos(__ldg(C.mcut + j)) : 0u;
      uint32_t up = __shfl_up_sync(0xffffffffu, P, 1);
      if (lane == 0) up = prev;
      const uint32_t cnt = up - P;  // count of value j + 1
      const int k = j + 1;
      if (k <= static_cast<int>(C.L) && k - kKsHead - 1 < a.dense_words) {
        ZKS_CHECK(2 * (k - kKsHead) <= a.vals_stride);
        out[k - kKsHead - 1] = cnt;
      }
      if (cnt) {
        const unsigned long long lk = log_fixed(a.logs, static_cast<uint32_t>(k));
        add128(shi, slo, __umul64hi(cnt, lk), static_cast<unsigned long long>(cnt) * lk);
        vtop = max(vtop, static_cast<uint32_t>(k));
        vlow = min(vlow, static_cast<uint32_t>(k));
      }
      prev = __shfl_sync(0xffffffffu, P, 31);
      if (prev == 0u) break;  // no draws above this chunk: later counts are never read (k > vmax)
    }
    vtop = warp_max_u32(vtop);
    vlow = warp_min_u32(vlow);
  } else if (T) {
    // the tail list: every key below M_63, i.e. keys[0, E) of the buckets up to M_63's, filtered,
    // each resolved by the guide + cdf search
    const unsigned long long M63 = __shfl_sync(0xffffffffu, Mb, 31);
    const uint32_t bk = static_cast<uint32_t>(M63 >> shift);
    const uint32_t E = bk >= nbk ? static_cast<uint32_t>(n) : bend[bk];
    const bool two = C.guide_levels == 2;
    const unsigned lt = (1u << lane) - 1u;
    uint16_t* tail = C.tail + i * a.vals_stride;
    uint32_t m = 0;
    ZKS_CHECK(E <= static_cast<uint32_t>(n));
    for (uint32_t t0 = 0; t0 < E; t0 += 32) {
      const uint32_t t = t0 + lane;
      const unsigned long long key = t < E ? keys[t] : ~0ull;
      const bool in = key < M63;
      uint32_t v = 0;
      if (in) {
        const double u = 1.0 - static_cast<double>(key) * 0x1p-53;  // exact
        uint32_t lo, hi;
        guide_bracket_fine(u, C.guide, C.guide_fine, two, lo, hi);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (__ldg(C.cdf + mid) >= u)
            hi = mid;
          else
            lo = mid + 1;
        }
        v = min(lo + 1, C.L);
        add128(shi, slo, 0ull, log_fixed(a.logs, v));
        vtop = max(vtop, v);
        vlow = min(vlow, v);
      }
      const unsigned bm = __ballot_sync(0xffffffffu, in);
      if (in) {
        if (a.dense_words) {
          ZKS_CHECK(v > kKsHead && static_cast<int>(v - kKsHead) <= a.dense_words);
          atomicAdd(dense + (v - kKsHead - 1), 1u);
        } else {
          // keys ascend bucket by bucket, so values descend: stored back to front, the list comes
          // out ascending up to the order inside a bucket -- the fit kernel's insertion sort of a
          // short tail is then linear instead of quadratic
          ZKS_CHECK(m + __popc(bm & lt) < T && T <= static_cast<uint32_t>(a.vals_stride));
          tail[T - 1u - (m + __popc(bm & lt))] = static_cast<uint16_t>(v);
        }
      }
      m += __popc(bm);
    }
    vtop = warp_max_u32(vtop);
    vlow = warp_min_u32(vlow);
    if (a.dense_words) {  // the warp's histogram into the row's tail slot, reset
      __syncwarp();
      uint32_t* out = reinterpret_cast<uint32_t*>(tail);
      for (int k = lane; k < static_cast<int>(vtop) - kKsHead; k += 32) {
        out[k] = dense[k];
        dense[k] = 0u;
      }
      __syncwarp();
    }
  }
  {  // the head's share of the log-sum: count x ln k, exact
    const unsigned long long l0 = log_fixed(a.logs, lane + 1), l1 = log_fixed(a.logs, lane + 33);
    add128(shi, slo, __umul64hi(c0, l0), static_cast<unsigned long long>(c0) * l0);
    add128(shi, slo, __umul64hi(c1, l1), static_cast<unsigned long long>(c1) * l1);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, shi, o), olo = __shfl_xor_sync(0xffffffffu, slo, o);
    add128(shi, slo, ohi, olo);
  }
  const double log_sum = fixed_to_double(shi, slo);
  const unsigned h0 = __ballot_sync(0xffffffffu, c0 != 0u), h1 = __ballot_sync(0xffffffffu, c1 != 0u);
  const uint32_t vmin = h0 ? static_cast<uint32_t>(__ffs(h0)) : h1 ? 32u + __ffs(h1) : vlow;
  const uint32_t vmax = T ? vtop : h1 ? 64u - __clz(h1) : 32u - __clz(h0);
  uint16_t* head = C.head + i * kKsHead;
  head[lane] = static_cast<uint16_t>(c0);  // n <= kRowMaxN: u16 counts
  head[lane + 32] = static_cast<uint16_t>(c1);
  if (lane == 0) {
    C.ls[i] = log_sum;
    C.mn[i] = vmin;
    C.mx[i] = vmax;
    C.m[i] = T;
  }
  if (kCount) tails += T;
}

// One block per replicate row (grid-stride over the chunk's rows): draw the n Philox words of
// stream (seed, rep, first + i), bucket their 53-bit keys in shared memory (a count pass, a
// scan, a scatter pass), then the block's warps take the row's cells by the host's schedule.
template <bool kCount>
__global__ void __launch_bounds__(kThreads, ZKS_ROW_MINB) row_draw_kernel(const __grid_constant__ RowArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  const bool parked = n <= kRowStageMaxN;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
  unsigned long long* raw = keys + round_up(n + kRowKeyPad, 2);  // the draw pass's keys in stream order (parked)
  const int nbk = 1 << a.bucket_bits;
  const int shift = 53 - a.bucket_bits;
  uint32_t* bstart = reinterpret_cast<uint32_t*>(raw + (parked ? round_up(n, 2) : 0));
  uint32_t* bend = bstart + nbk;  // running scatter positions = bucket ends
  uint32_t* cnt = bend + nbk;     // bucket sizes of the row being drawn (zeroed by the scan that reads them)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  uint32_t* dense = (a.dense_words && n <= kRowDenseHistMaxN) ? cnt + nbk + warp * a.dense_words : nullptr;
  for (int b = threadIdx.x; b < nbk; b += blockDim.x) cnt[b] = 0u;
  if (dense)
    for (int k = lane; k < a.dense_words; k += 32) dense[k] = 0u;
  __shared__ unsigned long long key_sh[2][2];  // this row's and the next row's stream keys
  __shared__ uint32_t wsum[kWarps];
  if (threadIdx.x < kRowKeyPad) keys[n + threadIdx.x] = ~0ull;
  const int nb = (n + 3) >> 2;
  unsigned long long tails = 0, rows = 0;
  if (warp == warps - 1 && blockIdx.x < a.count) {
    uint64_t k0, k1;
    stream_key(a.seed, a.rep, a.first + blockIdx.x, k0, k1);
    if (lane == 0) {
      key_sh[0][0] = k0;
      key_sh[0][1] = k1;
    }
  }
  __syncthreads();
  int kb = 0;  // key_sh slot of the current row
  for (uint64_t i = blockIdx.x; i < a.count; i += gridDim.x, kb ^= 1) {
    // 1. draw pass: bucket sizes (and the keys parked in stream order); the stream key was
    // derived during the previous row, the counts zeroed by its scan
    const uint64_t k0 = key_sh[kb][0], k1 = key_sh[kb][1];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const Block4 x = rng_block(static_cast<uint64_t>(b) + 1ull, k0, k1, a.rng);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (4 * b + w < n) {
          const unsigned long long m = x.w[w] >> 11;
          atomicAdd(cnt + (m >> shift), 1u);
          if (parked) raw[4 * b + w] = m;
        }
      }
    }
    __syncthreads();
    // 2. exclusive scan of the bucket sizes (each thread a contiguous segment)
    {
      const int seg = (nbk + blockDim.x - 1) / blockDim.x;
      const int b0 = min(nbk, static_cast<int>(threadIdx.x) * seg), b1 = min(nbk, b0 + seg);
      uint32_t s = 0;
      for (int b = b0; b < b1; ++b) s += cnt[b];
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      uint32_t run = incl - s;
      for (int w = 0; w < warp; ++w) run += wsum[w];
      for (int b = b0; b < b1; ++b) {
        const uint32_t c = cnt[b];
        cnt[b] = 0u;  // ready for the next row's draw pass
        bstart[b] = run;
        bend[b] = run;
        run += c;
      }
    }
    __syncthreads();
    // 3. scatter pass (bend[b] ends as the end of bucket b)
    if (parked) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const unsigned long long m = raw[j];
        ZKS_CHECK((m >> shift) < static_cast<unsigned long long>(nbk));
        const uint32_t at = atomicAdd(bend + (m >> shift), 1u);
        ZKS_CHECK(at < static_cast<uint32_t>(n));
        keys[at] = m;
      }
    } else {
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const Block4 x = rng_block(static_cast<uint64_t>(b) + 1ull, k0, k1, a.rng);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const unsigned long long m = x.w[w] >> 11;
          if (4 * b + w < n) {
            const uint32_t at = atomicAdd(bend + (m >> shift), 1u);
            ZKS_CHECK(at < static_cast<uint32_t>(n));
            keys[at] = m;
          }
        }
      }
    }
    __syncthreads();
    // 4. the row's cells by the schedule; the last warp also derives the next row's stream key
    for (int c = a.wbeg[warp]; c < a.wbeg[warp + 1]; ++c)
      row_cell<kCount>(a, a.cell[a.order[c]], i, keys, bstart, bend, dense, lane, tails);
    if (warp == warps - 1 && i + gridDim.x < a.count) {
      uint64_t q0, q1;
      stream_key(a.seed, a.rep, a.first + i + gridDim.x, q0, q1);
      if (lane == 0) {
        key_sh[kb ^ 1][0] = q0;
        key_sh[kb ^ 1][1] = q1;
      }
    }
    ++rows;
    __syncthreads();  // keys and buckets are reused by the next row
  }
  if (kCount && lane == 0) {
    if (threadIdx.x == 0 && rows) {
      atomicAdd(a.counters + 1, rows * static_cast<unsigned long long>(n));  // Philox draws
      atomicAdd(a.counters + kWorkFields, rows * static_cast<unsigned long long>(n));  // keys bucketed
      atomicAdd(a.counters + kWorkFields + 1, rows * static_cast<unsigned long long>(a.ncells));
    }
    if (tails) atomicAdd(a.counters + kWorkFields + 2, tails);
  }
}

}  // namespace zks
