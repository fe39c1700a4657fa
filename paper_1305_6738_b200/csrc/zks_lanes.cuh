// Sweep rows of small samples (n < kLaneDrawMaxN, table-mode MLE): each replicate stream drawn
// once for every gamma of the row, one lane per replicate.
//
// The cells of a sweep row share their uniforms (build_table seeds every cell with the same
// base_seed, pkg/src/zipfks/montecarlo.py:276-277; RandomStream.for_replicate,
// distribution.py:178-187), so a warp takes 32 consecutive replicates, each lane draws its
// replicate's n Philox words ONCE and keeps their top 32 bits t_j = x_j >> 32 (L2-resident
// per-warp rows, [j][lane]), and then runs the lane pipeline of the old per-cell kernel -- fit
// (Newton on the fit tables), KS head walk, short tails lane by lane, long tails and retries
// warp-cooperatively -- for each cell of the row in turn.  Classifying a stored word against a
// cell replaces the Philox block (about 60 integer instructions per word) and the guide + cdf
// search of the per-cell design.
//
// Exactness.  A word's value in a cell is v = 1 + #{k : M_k > m}, m = x >> 11 its 53-bit key,
// M_k = M(cdf[k]) the exact cuts (zks_rows.cuh).  With c_k = M_k >> 21 (32 bits) and t = m >> 21:
// c_k > t implies M_k > m and c_k < t implies M_k <= m, so the head value (<= kKsHead) follows
// from the 64 top-32 cuts unless some c_k == t.  A value above the head comes from the guide +
// cdf search at the top of t's key range, u_hi = 1 - t 2^-32, and is decided when the next lower
// cdf entry lies below the bottom of the range, u_lo = 1 - (t 2^21 + 2^21 - 1) 2^-53.  The
// undecided words (probability ~2^-26 per head word; ~2^-32 / p(v) per tail word) are resolved
// exactly from their Philox block, as the per-cell kernel drew them.  So every (replicate, cell)
// sample is the reference's sample() bit for bit.
//
// The log-sum is accumulated in 64-bit fixed point (ln v 2^53 is an exact integer < 2^57 for
// v <= 65535, and n < 128 terms stay below 2^64): exact, so independent of the classification
// order; fit_target sees it rounded once.
#pragma once
#include "zks_batch.cuh"

namespace zks {

#ifndef ZKS_LANE_MINB
#define ZKS_LANE_MINB 3
#endif
#ifndef ZKS_LANE_GROUP
#define ZKS_LANE_GROUP 4
#endif
constexpr int kLaneGroup = ZKS_LANE_GROUP;  // words classified per step (their loads in flight together)
constexpr int kLaneMaxCells = 32;
// Head cuts are bracketed by a log-scale bucket of the word: the distance x of t to the nearer end
// of the word range (cuts crowd towards both ends -- the tail cuts of a Zipf law near t = 0, the
// first cuts of a flat finite law near 2^32) as a float, its exponent and top 6 mantissa bits.
// Bucket index monotone in t: [0, 2048) for t < 2^31, [2048, 4096) above.
constexpr int kLaneBuckets = 4096;
__device__ __forceinline__ uint32_t lane_bucket(uint32_t t) {
  const bool up = t >> 31;
  const uint32_t x = up ? ~t : t;
  const uint32_t bits = __float_as_uint(__uint2float_rz(x));
  const int q = max(static_cast<int>(bits >> 17) - (126 << 6), 0);  // x = 0 -> 0, x in [1, 2^31) -> [64, 2048)
  return up ? 4095u - static_cast<uint32_t>(q) : static_cast<uint32_t>(q);
}

// Per sampling table (built once, lane_cut_kernel): the head cuts c_k = M_k >> 21 (k < kKsHead,
// non-increasing) and per bucket b the bracket lo | hi << 7: cuts k < lo lie above every word of
// the bucket, cuts in [lo, hi) inside its word range, the rest below it.
struct LaneCut {
  uint32_t cut[kKsHead];
  uint16_t br[kLaneBuckets];
};

__global__ void lane_cut_kernel(const unsigned long long* __restrict__ mcut, LaneCut* out) {
  __shared__ uint32_t c[kKsHead];
  for (int k = threadIdx.x; k < static_cast<int>(kKsHead); k += blockDim.x) {
    // M_k = 2^53 (cdf[k] < 2^-53: every key lies below the cut) clamps to 2^32 - 1, which still
    // reads "above" for every smaller word and undecided (resolved exactly) for the top one
    c[k] = static_cast<uint32_t>(min(mcut[k] >> 21, 0xffffffffull));
    out->cut[k] = c[k];
  }
  __syncthreads();
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < kLaneBuckets; b += gridDim.x * blockDim.x) {
    // the bucket's word range [first, last]: lane_bucket is monotone in t
    auto first_at_least = [](uint32_t bk) {  // smallest t with lane_bucket(t) >= bk (2^32 if none)
      uint64_t lo = 0, hi = 1ull << 32;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (lane_bucket(static_cast<uint32_t>(mid)) >= bk)
          hi = mid;
        else
          lo = mid + 1;
      }
      return lo;
    };
    const uint64_t first = first_at_least(b), next = first_at_least(b + 1);
    uint32_t lo = 0, hi = 0;
    if (first < next) {  // non-empty bucket
      const uint64_t last = next - 1;
      for (int k = 0; k < static_cast<int>(kKsHead); ++k) {
        lo += c[k] > last;
        hi += c[k] >= first;
      }
    }
    out->br[b] = static_cast<uint16_t>(lo | (hi << 7));
  }
}

// C: the parameter block's cell capacity (kLaneMaxCells, or 1 for single cells: a 0.6 KB
// instead of an 18 KB kernel parameter, ~10 us less per launch where launches dominate)
template <int C>
struct LaneArgsT {
  ReplicateArgs cell[C];  // the row's cells (equal n, support, seed, rep, range)
  const LaneCut* cut[C];
  uint32_t* words;  // per resident warp: n x 32 top words, [j][lane]
  int ncells;
  int groups;     // work items = tiles of 32 replicates x cell groups (more items than warps
  int per_group;  // when a launch has few replicates; each group redraws its tile)
};

// ln k 2^53 for k = 0..kKsHead in shared memory (16-byte multiple)
constexpr int kLaneLnBytes = round_up((kKsHead + 1) * 8, 16);

// The value of word j of this lane's stream exactly (the undecided words): its Philox block again.
__device__ __noinline__ uint32_t lane_exact_value(const ReplicateArgs& a, uint64_t idx, int j) {
  uint64_t k0, k1;
  stream_key(a.seed, a.rep, idx, k0, k1);
  const Block4 r = rng_block(static_cast<uint64_t>(j >> 2) + 1ull, k0, k1, a.rng);
  const int w = j & 3;
  const uint64_t x = w == 0 ? r.w[0] : w == 1 ? r.w[1] : w == 2 ? r.w[2] : r.w[3];
  return draw_value(uniform_open_closed(x), a.guide, a.cdf, a.L, a.guide_levels == 2);
}

// lower_bound(cdf, u) + 1 clamped to L, through the fine guide (a bracket of ~one entry in the
// heavy tail)
__device__ __forceinline__ uint32_t lane_search(const ReplicateArgs& a, double u) {
  uint32_t lo, hi;
  guide_bracket_fine(u, a.guide, a.guide_fine, a.guide_levels == 2, lo, hi);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a.cdf + mid) >= u)
      hi = mid;
    else
      lo = mid + 1;
  }
  return min(lo + 1, a.L);
}

// The value of top word t in the cell (a, lc); idx / j locate the word for the exact fallback.
// br = lc->br[lane_bucket(t)], loaded by the caller (several words' loads in flight).
__device__ __forceinline__ uint32_t lane_value(const ReplicateArgs& a, const LaneCut* __restrict__ lc, uint32_t t,
                                               uint32_t br, uint64_t idx, int j) {
  uint32_t lo = br & 0x7fu;
  const uint32_t top = br >> 7;
  // first cut in [lo, top) that is <= t (cuts are non-increasing)
  for (uint32_t hi = top; lo < hi;) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(lc->cut + mid) > t)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < top && __ldg(lc->cut + lo) == t) return lane_exact_value(a, idx, j);
  if (lo < kKsHead) return lo + 1;
  // above the head: the value at the top of t's key range, decided if the range holds no cdf entry
  const double u_hi = 1.0 - static_cast<double>(t) * 0x1p-32;
  const double u_lo = 1.0 - static_cast<double>((static_cast<uint64_t>(t) << 21) | 0x1fffffull) * 0x1p-53;
  const uint32_t v = lane_search(a, u_hi);
  if (__ldg(a.cdf + v - 2) < u_lo) return v;  // v > kKsHead >= 2
  return lane_exact_value(a, idx, j);
}

// After a lane_row_kernel launch: its words (scratch, rewritten by the next launch) are dropped
// from L2 without a write-back -- they would otherwise hold persisting lines through the kernels
// that follow and be written to HBM when evicted
__global__ void lane_release_kernel(uint32_t* words, size_t bytes) {
  const size_t lines = bytes / 128;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < lines; i += size_t(gridDim.x) * blockDim.x)
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<char*>(words) + i * 128) : "memory");
}

template <bool kCount, int C>
__global__ void __launch_bounds__(kThreads, ZKS_LANE_MINB) lane_row_kernel(const __grid_constant__ LaneArgsT<C> la) {
  extern __shared__ __align__(16) unsigned char smem[];
  const ReplicateArgs& b = la.cell[0];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* lnfix = reinterpret_cast<unsigned long long*>(smem);
  const int warp_bytes = batch_warp_bytes(b.hist_words, b.vals_stride, static_cast<int>(b.n));
  unsigned char* mine = smem + kLaneLnBytes + warp * warp_bytes;
  uint32_t* hist = reinterpret_cast<uint32_t*>(mine);
  uint32_t* queue = hist + b.hist_words;
  uint16_t* vals = reinterpret_cast<uint16_t*>(mine + b.hist_words * 4 + 3 * kKsQueue * 4);  // lane tails
  uint16_t* stage = vals + 32 * b.vals_stride;  // one sample of n values (long tails, retries)
  for (int k = threadIdx.x; k <= static_cast<int>(kKsHead); k += blockDim.x) lnfix[k] = log_fixed(b.logs, k);
  clear_hist(hist, b.hist_words, lane);
  __syncthreads();

  const int n = static_cast<int>(b.n);
  const double dn = static_cast<double>(n);
  uint32_t* words = la.words + (static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * static_cast<size_t>(n) * 32;
  const uint64_t tiles = (b.count + 31) / 32;
  const uint64_t items = tiles * static_cast<uint64_t>(la.groups);
  const int nb = (n + 3) >> 2;
  uint8_t* lh = reinterpret_cast<uint8_t*>(hist);  // lane histograms [v][lane], zero between cells
  Work wk{};

  for (;;) {
    unsigned long long bid = 0;
    if (lane == 0) bid = atomicAdd(b.work, 1ull);
    bid = __shfl_sync(0xffffffffu, bid, 0);
    if (bid >= items) break;
    const uint64_t tile = bid / static_cast<unsigned>(la.groups);
    const int grp = static_cast<int>(bid - tile * static_cast<unsigned>(la.groups));
    const uint64_t r0 = tile * 32;
    const uint64_t left = b.count - r0;
    const int nrep = left < 32ull ? static_cast<int>(left) : 32;
    const bool active = lane < nrep;
    const uint64_t idx = b.first + r0 + lane;  // this lane's replicate index

    // 1. the lane's stream, once for every cell of the group: top words in [j][lane] order
    if (active) {
      uint64_t k0, k1;
      stream_key(b.seed, b.rep, idx, k0, k1);
      for (int q = 0; q < nb; ++q) {
        const Block4 r = rng_block(static_cast<uint64_t>(q) + 1ull, k0, k1, b.rng);
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (4 * q + w < n) __stcg(words + (4 * q + w) * 32 + lane, static_cast<uint32_t>(r.w[w] >> 32));
      }
    }
    if (kCount) wk.draws += static_cast<unsigned long long>(nrep) * n;

    const int c_end = min(la.ncells, (grp + 1) * la.per_group);
    for (int c = grp * la.per_group; c < c_end; ++c) {
      // per-cell fields (tables, outputs) through la.cell[c]; everything the row's cells share
      // (support, fit table, n, seed) through cell 0, whose fields are constant-bank operands
      const ReplicateArgs& a = la.cell[c];
      const LaneCut* __restrict__ lc = la.cut[c];
      const int K = b.K;
      const ModelFns M{K, b.logs, b.fit, true};
      uint16_t* mv = vals + lane * b.vals_stride;

      // 2. the sample's statistics in this cell: head counts (lane histogram), tail values,
      // exact log-sum, min / max
      uint32_t vmin = 0xffffffffu, vmax = 0, m = 0;
      unsigned long long lsum = 0;
      if (active) {
        const uint32_t cap = static_cast<uint32_t>(b.vals_stride);
        int j = 0;
        // words stream from L2 (__ldcs: L1 keeps the tables); the next group is in flight while
        // this one is classified
        uint32_t nx[kLaneGroup];
#pragma unroll
        for (int w = 0; w < kLaneGroup; ++w) nx[w] = w < n ? __ldcs(words + w * 32 + lane) : 0u;
        for (; j + kLaneGroup <= n; j += kLaneGroup) {
          uint32_t t[kLaneGroup];
#pragma unroll
          for (int w = 0; w < kLaneGroup; ++w) {
            t[w] = nx[w];
            nx[w] = j + kLaneGroup + w < n ? __ldcs(words + (j + kLaneGroup + w) * 32 + lane) : 0u;
          }
          uint32_t br[kLaneGroup];
#pragma unroll
          for (int w = 0; w < kLaneGroup; ++w) br[w] = __ldg(lc->br + lane_bucket(t[w]));
#pragma unroll
          for (int w = 0; w < kLaneGroup; ++w) {
            const uint32_t v = lane_value(a, lc, t[w], br[w], idx, j + w);
            ZKS_CHECK(v >= 1u && v <= a.L);
            vmin = min(vmin, v);
            vmax = max(vmax, v);
            if (v <= kKsHead) {
              ++lh[v * 32 + lane];
              lsum += lnfix[v];
            } else {
              if (m < cap) mv[m] = static_cast<uint16_t>(v);
              ++m;
              lsum += log_fixed(b.logs, v);
            }
          }
        }
#pragma unroll
        for (int w = 0; w < kLaneGroup - 1; ++w) {  // the last n % kLaneGroup words (already in nx)
          if (j + w >= n) break;
          const uint32_t t = nx[w];
          const uint32_t v = lane_value(a, lc, t, __ldg(lc->br + lane_bucket(t)), idx, j + w);
          ZKS_CHECK(v >= 1u && v <= a.L);
          vmin = min(vmin, v);
          vmax = max(vmax, v);
          if (v <= kKsHead) {
            ++lh[v * 32 + lane];
            lsum += lnfix[v];
          } else {
            if (m < cap) mv[m] = static_cast<uint16_t>(v);
            ++m;
            lsum += log_fixed(b.logs, v);
          }
        }
      }
      __syncwarp();
      if (kCount) wk.attempts += nrep;

      // 3. exponent fits, one replicate per lane
      double g = 0.0, norm = 1.0;
      bool ok = false;
      Work lw{};
      if (active) {
        const double target = fit_target(fixed_to_double(0ull, lsum), vmin, K, dn);
        ok = fit_exponent(M, target, lane, g, lw);
        if (ok) norm = fit_norm(b.fit, g);
        if (!ok) g = target;
        if (kCount && ok) {  // the reference's normaliser and KS terms (min(kmax, 4096), gof.py:49-105)
          lw.norm_terms += ref_norm_terms(b.fit, g);
          lw.ks_terms += min(vmax, static_cast<uint32_t>(kSeam));
        }
      }
      if (kCount) add_lane_work(wk, lw);

      // 4. KS: the head lane by lane, then the tails
      double my_ks = __longlong_as_double(0x7ff8000000000000ll);
      double hS, hD;
      uint32_t hC;
      const bool scored = ks_lane_head(b, ok && active, g, norm, vmax, lh, my_ks, hS, hC, hD);
      clear_hist(hist, kLaneHistWords, lane);
      // short tails lane by lane (insertion sort: quadratic in the tail length), long ones by the warp
      const bool tail = active && ok && !scored;
      const bool short_tail = tail && m <= static_cast<uint32_t>(b.vals_stride);  // all kept by the lane
      uint32_t ends = 0;
      if (short_tail) my_ks = ks_tail_lane(b, g, norm, hS, hC, hD, mv, static_cast<int>(m), ends);
      if (kCount) wk.ks_tails += warp_sum_u32(ends);
      __syncwarp();
      for (unsigned need = __ballot_sync(0xffffffffu, tail && !short_tail); need; need &= need - 1) {
        const int r = __ffs(need) - 1;
        const double gr = __shfl_sync(0xffffffffu, g, r);
        const double nr = __shfl_sync(0xffffffffu, norm, r);
        const uint32_t kmax = __shfl_sync(0xffffffffu, vmax, r);
        // replicate r's sample redrawn exactly by the warp into the staging row (its values <=
        // kKsHead are ignored by the scan); n < kOverCap: the tail fits the register sort
        uint64_t q0, q1;
        stream_key(b.seed, b.rep, b.first + r0 + r, q0, q1);
        draw_sample(a, q0, q1, a.guide, stage, lane);
        __syncwarp();
        const KsOut ko = ks_tail_from_head(b, r, gr, nr, kmax, hS, hC, hD, hist, b.hist_words, 0u, queue, stage,
                                           static_cast<uint32_t>(n), lane, wk);
        __syncwarp();
        if (lane == r) my_ks = ko.D;
      }

      // 5. retries on stream idx + 2^32 (montecarlo.py:106-115), warp-cooperative
      uint8_t status = ok ? 0 : 2;
      for (unsigned fails = __ballot_sync(0xffffffffu, active && !ok); fails; fails &= fails - 1) {
        const int r = __ffs(fails) - 1;
        double ks2, g2;
        const uint8_t s2 = retry_replicate<kCount>(a, M, r0 + r, a.guide, stage, hist, queue, lane, ks2, g2, wk);
        if (lane == r) {
          status = s2;
          my_ks = ks2;
          g = g2;
        }
      }

      if (active) {
        a.ks_out[r0 + lane] = my_ks;
        a.gh_out[r0 + lane] = g;
        a.st_out[r0 + lane] = status;
      }
    }
  }
  if (kCount && lane == 0) {
    const unsigned long long* f = &wk.attempts;
    for (int i = 0; i < kWorkFields; ++i)
      if (f[i]) atomicAdd(b.counters + i, f[i]);
  }
}

}  // namespace zks
