// The fused replicate kernel: stream -> inverse-CDF draws -> histogram + log-sum ->
// Newton/bisection MLE -> fitted normaliser -> KS scan, one warp per replicate.
//
// Restates, per replicate, pkg/src/zipfks/montecarlo.py:89-116 (_attempt / run_replicate)
// with its leaves distribution.py:190-201 (sample), estimate.py:59-146 (log_mean, mle_gamma,
// _bisect) and gof.py:49-105 (ks_statistic, dense and sparse paths).
//
// Layout (per block of kWarps warps):
//   smem  guide[G+2]   uint16  lower_bound(cdf, j/G), j = 0..G, guide[G+1] = L
//         hist[w][H+1] uint32  per-warp counts of values 1..H (H = min(L, 2048))
//   global cdf[L]      fp64    host-built sampling CDF (bit-exact with the reference)
//          logs[65537] fp64    host-built numpy ln k table
//          slab[w][n]  uint16  per-warp list of values > H (only when L > H)
// Draws are never materialised in HBM; per replicate only (ks, gamma_hat, status) is written.
#pragma once
#include <cstdint>

#include "zks_fit.cuh"
#include "zks_ks.cuh"
#include "zks_series.cuh"
#include "zks_stream.cuh"

namespace zks {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kHistMax = 2048;             // histogram bins held in shared memory per warp
constexpr int kGuideLog2 = 12;              // guide table resolution G = 4096
constexpr int kGuide = 1 << kGuideLog2;
constexpr int kGuideLevel = kGuide + 2;     // entries per guide level
// second level: the top 2^-5 of u in 4096 bins of 2^-17 (heavy tails: k ranges per bin stay short)
constexpr double kGuide2Start = 0.96875;    // 1 - 2^-5
constexpr double kGuide2Scale = 131072.0;   // 2^17: level 2 (shared memory), the top 2^-5 in G bins
constexpr int kGuideFineBins = 1 << 16;     // fine level 2 (global memory): the top 2^-5 in 2^16 bins
constexpr int kGuideFineLevel = kGuideFineBins + 2;
constexpr double kGuideFineScale = 2097152.0;  // 2^21
constexpr int kGuideEntries = 2 * kGuideLevel + kGuideFineLevel;  // level 1, level 2, fine level 2
constexpr double kLn2 = 0.69314718055994530942;  // math.log(2.0)

struct ReplicateArgs {
  const double* cdf;
  const uint16_t* guide;      // levels 1 and 2 (2 x kGuideLevel entries; copied to shared memory)
  const uint16_t* guide_fine;  // fine level 2 (kGuideFineLevel entries, read from global memory / L2)
  const double* logs;
  uint32_t L;      // draw-table length: K or 65535
  int32_t K;       // finite support bound, 0 = unbounded
  int32_t H;       // smem histogram bins per warp
  int32_t hist_words;
  double gamma;
  int64_t n;
  uint64_t seed, rep, first, count;
  double* ks_out;
  double* gh_out;
  uint8_t* st_out;
  uint16_t* slab;
  int64_t slab_cap;
  unsigned long long* work;
  unsigned long long* counters;  // optional Work totals (kWorkFields), NULL = off
  FitTable fit;                  // exponent-fit table of this support
  int use_table;                 // 1: table-driven model functions, 0: direct sums
  int batch;                     // replicates per warp batch (lane_row_kernel)
  int vals_stride;               // u16 sample slots per replicate in the batch store
  int guide_levels;              // 1, or 2 for long tables (L > 4096)
  // pre-drawn samples (draw_stats_kernel), row i = replicate index pre_first + i: u16 counts of
  // the values 1..kKsHead at pre_head[i * kKsHead] (128-byte rows), the m = pre_m[i] values
  // above kKsHead at pre_tail[i * vals_stride], log-sum / min / max.  pre_tail is consumed:
  // fit_ks_kernel's page passes compact a long tail in place (ks_scan<..., kCompact>)
  const uint16_t* pre_head;
  uint16_t* pre_tail;
  const uint32_t* pre_m;
  const double* pre_ls;
  const uint32_t* pre_min;
  const uint32_t* pre_max;
  uint64_t pre_first;
  // dense finite supports (kKsHead < K <= kDenseMaxK): the values above kKsHead are kept as u32
  // counts of kKsHead+1..K in the row's tail slot instead of a value list (0 = value lists)
  int dense_words;
  double inv_n;  // 1 / n
  int rng;       // kRngNumpy (bit-exact with the reference) or kRngPhilox4x32 (opt-in fast stream)
  uint32_t tcut[4];     // top 32 bits t of a Philox word: u > cdf_head[j] <=> t < tcut[j] (undecided at equality)
  double cdf_head[4];  // cdf[0..3]; +inf from index L-1 on (every u above it draws L)
};

// guide lookup: [lo, hi] brackets lower_bound(cdf, u)
__device__ __forceinline__ void guide_bracket(double u, const uint16_t* guide, bool two, uint32_t& lo, uint32_t& hi) {
  const bool up = two && u >= kGuide2Start;
  const int j = up ? static_cast<int>((u - kGuide2Start) * kGuide2Scale) : static_cast<int>(u * static_cast<double>(kGuide));
  const uint16_t* g = guide + (up ? kGuideLevel : 0) + j;
  lo = g[0];
  hi = g[1];
}

// the same with the fine level 2 (65536 bins, global memory): a bracket of ~1 entry for heavy
// tails, where the shared level 2 leaves several search steps -- for the queued resolution of
// draw_stats_kernel, whose lanes all search at once
__device__ __forceinline__ void guide_bracket_fine(double u, const uint16_t* guide, const uint16_t* __restrict__ fine,
                                                   bool two, uint32_t& lo, uint32_t& hi) {
  const bool up = two && u >= kGuide2Start;
  const int j = up ? static_cast<int>((u - kGuide2Start) * kGuideFineScale) : static_cast<int>(u * static_cast<double>(kGuide));
  const uint16_t* g = up ? fine + j : guide + j;
  lo = g[0];
  hi = g[1];
}

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// block-cooperative copy of the guide table (levels x kGuideLevel u16, 16-byte aligned) to smem
__device__ __forceinline__ void load_guide(uint16_t* dst, const uint16_t* __restrict__ src, int levels) {
  const int n = levels * kGuideLevel, n16 = n / 8;
  for (int i = threadIdx.x; i < n16; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  for (int i = n16 * 8 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// smallest k (1-based) with cdf[k-1] >= u, clamped to L (distribution.py:200-201)
__device__ __forceinline__ uint32_t draw_value(double u, const uint16_t* __restrict__ guide,
                                               const double* __restrict__ cdf, uint32_t L, bool two) {
  uint32_t lo, hi;
  guide_bracket(u, guide, two, lo, hi);  // exact index arithmetic: u is a multiple of 2^-53
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(cdf + mid) >= u)
      hi = mid;
    else
      lo = mid + 1;
  }
  const uint32_t v = lo + 1;
  return v > L ? L : v;
}

// The four draws of one Philox block, their lower_bound searches interleaved so that up to four
// independent cdf loads are in flight per lane.  Lanes with valid[w] false yield 0.
__device__ __forceinline__ void draw_block_u(const double u[4], const bool valid[4], const uint16_t* __restrict__ guide,
                                             const struct ReplicateArgs& a, uint32_t out[4]);

__device__ __forceinline__ void draw_block(const Block4& r, const bool valid[4], const uint16_t* __restrict__ guide,
                                           const struct ReplicateArgs& a, uint32_t out[4]);

__device__ __forceinline__ void draw_block_u(const double u[4], const bool valid[4], const uint16_t* __restrict__ guide,
                                             const ReplicateArgs& a, uint32_t out[4]) {
  const bool two = a.guide_levels == 2;
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    guide_bracket(u[w], guide, two, lo[w], hi[w]);
    if (!valid[w]) hi[w] = lo[w];
  }
  for (;;) {
    bool act[4];
    uint32_t mid[4];
    double cv[4];
    bool any = false;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      act[w] = lo[w] < hi[w];
      any |= act[w];
      mid[w] = (lo[w] + hi[w]) >> 1;
      cv[w] = act[w] ? __ldg(a.cdf + mid[w]) : 0.0;
    }
    if (!any) break;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (act[w]) {
        if (cv[w] >= u[w])
          hi[w] = mid[w];
        else
          lo[w] = mid[w] + 1;
      }
    }
  }
#pragma unroll
  for (int w = 0; w < 4; ++w) out[w] = valid[w] ? min(lo[w] + 1, a.L) : 0u;
}

__device__ __forceinline__ void draw_block(const Block4& r, const bool valid[4], const uint16_t* __restrict__ guide,
                                           const ReplicateArgs& a, uint32_t out[4]) {
  double u[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) u[w] = uniform_open_closed(r.w[w]);
  draw_block_u(u, valid, guide, a, out);
}

struct SampleStats {
  double log_sum;
  uint32_t vmin, vmax, over;
};


// Draw n values of stream (seed, rep, sidx) into the warp's histogram / overflow slab.
__device__ __forceinline__ SampleStats sample_pass(const ReplicateArgs& a, uint64_t sidx,
                                                   const uint16_t* __restrict__ guide, uint32_t* hist,
                                                   uint16_t* slab, int lane) {
  uint64_t k0, k1;
  stream_key(a.seed, a.rep, sidx, k0, k1);
  const int64_t n = a.n;
  const int64_t nb = (n + 3) >> 2;
  const uint32_t H = static_cast<uint32_t>(a.H);
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t c1 = 0, c2 = 0, c3 = 0, c4 = 0, vmin = 0xffffffffu, vmax = 0, over = 0;
  double ls = 0.0;
  for (int64_t b0 = 0; b0 < nb; b0 += 32) {
    const int64_t b = b0 + lane;
    const Block4 r = rng_block(static_cast<uint64_t>(b) + 1ull, k0, k1, a.rng);
    bool vb[4];
    uint32_t vv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) vb[w] = (4 * b + w) < n;
    draw_block(r, vb, guide, a, vv);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const bool valid = vb[w];
      const uint32_t v = vv[w];
      if (valid) {
        vmin = min(vmin, v);
        vmax = max(vmax, v);
        c1 += (v == 1u);
        c2 += (v == 2u);
        c3 += (v == 3u);
        c4 += (v == 4u);
        if (v > 4u) {
          ls += __ldg(a.logs + v);
          if (v <= H) atomicAdd(hist + v, 1u);
        }
      }
      const bool ov = valid && v > H;
      const unsigned mask = __ballot_sync(0xffffffffu, ov);
      if (ov) slab[over + __popc(mask & lt_mask)] = static_cast<uint16_t>(v);
      over += __popc(mask);
    }
  }
  c1 = warp_sum_u32(c1);
  c2 = warp_sum_u32(c2);
  c3 = warp_sum_u32(c3);
  c4 = warp_sum_u32(c4);
  if (lane == 0) {
    hist[1] = c1;
    hist[2] = c2;
    hist[3] = c3;
    hist[4] = c4;
  }
  __syncwarp();
  SampleStats s;
  const double small = static_cast<double>(c2) * __ldg(a.logs + 2) + static_cast<double>(c3) * __ldg(a.logs + 3) +
                       static_cast<double>(c4) * __ldg(a.logs + 4);
  s.log_sum = warp_sum(ls) + small;
  s.vmin = warp_min_u32(vmin);
  s.vmax = warp_max_u32(vmax);
  s.over = over;
  return s;
}

// The model functions the estimator needs, from the fit table (default) or by direct
// summation exactly as the reference forms them (validation mode).
struct ModelFns {
  int K;
  const double* logs;
  const FitTable& T;  // the kernel parameter's table (read through the constant bank)
  bool table;         // false = direct sums
};

__device__ __forceinline__ bool model_mean_slope(const ModelFns& M, double x, int lane, double& mean, double& slope,
                                                 Work& wk) {
  if (M.table) {
    ++wk.evals;
    wk.eval_terms += ref_moment_terms(M.T, x);
    fit_mean_slope(M.T, x, mean, slope);
    return true;
  }
  Moments m;
  if (!log_moments(x, M.K, M.logs, lane, m, wk)) return false;
  mean = m.s1 / m.s0;
  slope = m.s2 / m.s0 - mean * mean;
  return true;
}

__device__ __forceinline__ double model_mean(const ModelFns& M, double x, int lane, bool& ok, Work& wk) {
  if (M.table) {
    ++wk.evals;
    wk.eval_terms += ref_moment_terms(M.T, x);
    ok = true;
    return fit_mean(M.T, x);
  }
  Moments m;
  ok = log_moments(x, M.K, M.logs, lane, m, wk);
  return m.s1 / m.s0;
}

__device__ __forceinline__ double model_norm(const ModelFns& M, double x, int lane, Work& wk) {
  if (M.table) return fit_norm(M.T, x);
  return normaliser(x, M.K, M.logs, lane, wk);
}

// estimate.py:94-112
__device__ bool bisect_root(const ModelFns& M, double target, int lane, double lo, double hi, double& root,
                            Work& wk) {
  bool ok1, ok2;
  const double f_lo = target - model_mean(M, lo, lane, ok1, wk);
  const double f_hi = target - model_mean(M, hi, lane, ok2, wk);
  if (!ok1 || !ok2) return false;
  if (f_lo == 0.0) {
    root = lo;
    return true;
  }
  if (f_hi == 0.0) {
    root = hi;
    return true;
  }
  if (f_lo * f_hi > 0.0) return false;  // NoRootError
  while (hi - lo > 1e-8) {
    const double mid = 0.5 * (lo + hi);
    bool ok;
    const double f = target - model_mean(M, mid, lane, ok, wk);
    if (f * f_lo <= 0.0)
      hi = mid;
    else
      lo = mid;
  }
  root = 0.5 * (lo + hi);
  return true;
}

// MleSettings (estimate.py:24-50); the Monte Carlo always uses DEFAULT_SETTINGS (montecarlo.py:93)
struct MleParams {
  double x0 = 0.5;
  double tol = 1e-5;
  int max_iter = 200;
  double lo = -20.0, hi = 20.0;  // bracket
};

// estimate.py:86-91 (_search_range) and 115-146 (mle_gamma)
__device__ bool fit_exponent(const ModelFns& M, double target, int lane, double& g, Work& wk,
                             const MleParams& P = MleParams()) {
  double lo = P.lo, hi = P.hi;
  if (M.K == 0) {
    lo = fmax(lo, kMinUnboundedGamma);
    hi = fmin(hi, kMaxUnboundedGamma);
  }
  double x = P.x0;
  if (!(lo < x && x < hi)) x = lo + 0.01;
  for (int it = 0; it < P.max_iter; ++it) {
    double mean, slope;
    if (!model_mean_slope(M, x, lane, mean, slope, wk)) return false;
    const double x_new = x + (mean - target) / slope;
    if (!isfinite(x_new) || x_new < lo || x_new > hi) return bisect_root(M, target, lane, lo, hi, g, wk);
    if (fabs(x_new - x) <= P.tol) {
      g = x_new;
      return true;
    }
    x = x_new;
  }
  return bisect_root(M, target, lane, lo, hi, g, wk);
}

// KS parameters of a replicate launch
__device__ __forceinline__ KsParams ks_params(const ReplicateArgs& a) {
  KsParams p;
  p.n = a.n;
  p.H = static_cast<uint32_t>(a.H);
  p.hist_words = a.hist_words;
  p.logs = a.logs;
  p.exact = false;
  p.inv_n = a.inv_n;
  return p;
}

template <bool kCount>
#ifndef ZKS_REPL_MINB
#define ZKS_REPL_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, ZKS_REPL_MINB) replicate_kernel(ReplicateArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* guide = reinterpret_cast<uint16_t*>(smem);
  const int guide_bytes = round_up(a.guide_levels * kGuideLevel * 2, 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + guide_bytes) + warp * (a.hist_words + 3 * kKsQueue);
  uint32_t* queue = hist + a.hist_words;
  load_guide(guide, a.guide, a.guide_levels);
  clear_hist(hist, a.hist_words, lane);
  __syncthreads();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  uint16_t* slab = a.slab ? a.slab + gw * a.slab_cap : nullptr;
  const int K = a.K;
  const double dn = static_cast<double>(a.n);
  Work wk{};
  const ModelFns M{K, a.logs, a.fit, a.use_table != 0};

  for (;;) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(a.work, 1ull);
    r = __shfl_sync(0xffffffffu, r, 0);
    if (r >= a.count) break;
    const uint64_t idx = a.first + r;
    double ks = __longlong_as_double(0x7ff8000000000000ll), gh = ks;
    uint8_t status = 2;
    for (int attempt = 0; attempt < 2; ++attempt) {
      const uint64_t sidx = idx + (attempt ? (1ull << 32) : 0ull);  // montecarlo.py:29,110
      const SampleStats st = sample_pass(a, sidx, guide, hist, slab, lane);
      ++wk.attempts;
      wk.draws += a.n;
      double target = st.log_sum;
      if (target <= 0.0) target += kLn2;  // estimate.py:71-72
      target /= dn;
      if (K > 0 && st.vmin == static_cast<uint32_t>(K))  // estimate.py:126-129
        target -= (log(static_cast<double>(K)) - log(static_cast<double>(K - 1))) / dn;
      double g = 0.0;
      const bool ok = fit_exponent(M, target, lane, g, wk);
      bool used_pages = false;
      if (ok) {
        const double norm = model_norm(M, g, lane, wk);
        const KsOut ko = ks_scan<uint16_t, false, true>(ks_params(a), g, norm, st.vmax, hist, slab, st.over, queue, lane, wk);
        ks = ko.D;
        used_pages = ko.used_pages;
        gh = g;
        status = static_cast<uint8_t>(attempt);
      } else {
        gh = target;  // diagnostics for the "failed twice" message
      }
      const int top = used_pages ? a.hist_words : round_up(static_cast<int>(min(max(st.vmax, 4u), (uint32_t)a.H)) + 1, 4);
      clear_hist(hist, min(top, a.hist_words), lane);
      if (ok) break;
    }
    if (lane == 0) {
      a.ks_out[r] = ks;
      a.gh_out[r] = gh;
      a.st_out[r] = status;
    }
  }
  if (kCount && lane == 0) {
    const unsigned long long* f = &wk.attempts;
    for (int i = 0; i < kWorkFields; ++i)
      if (f[i]) atomicAdd(a.counters + i, f[i]);
  }
}

// normalization(gamma, support) of one model (distribution.py:71-85), one warp
__global__ void normaliser_kernel(double g, int K, const double* __restrict__ logs, double* out) {
  Work wk{};
  const double v = normaliser(g, K, logs, threadIdx.x & 31, wk);
  if (threadIdx.x == 0) *out = v;
}

// level 1: guide[j] = lower_bound(cdf, j / G), j = 0..G; level 2: lower_bound(cdf,
// 1 - 2^-5 + j 2^-17), j = 0..G; fine level 2: lower_bound(cdf, 1 - 2^-5 + j 2^-21),
// j = 0..kGuideFineBins; each level ends with L
__global__ void guide_kernel(const double* __restrict__ cdf, uint32_t L, uint16_t* guide) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kGuideEntries) return;
  const int level = t < kGuideLevel ? 0 : t < 2 * kGuideLevel ? 1 : 2;
  const int j = t - level * kGuideLevel;
  if (j == (level == 2 ? kGuideFineBins : kGuide) + 1) {
    guide[t] = static_cast<uint16_t>(L);
    return;
  }
  const double u = level == 0 ? static_cast<double>(j) / static_cast<double>(kGuide)
                              : kGuide2Start + static_cast<double>(j) / (level == 1 ? kGuide2Scale : kGuideFineScale);
  uint32_t lo = 0, hi = L;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cdf[mid] >= u)
      hi = mid;
    else
      lo = mid + 1;
  }
  guide[t] = static_cast<uint16_t>(lo);
}

// RandomStream.uniforms (distribution.py:186-187) for one stream, block-parallel
// keyed = 1: (seed, rep) is the Philox key itself (host-derived SeedSequence of another key)
__global__ void uniforms_kernel(uint64_t seed, uint64_t rep, uint64_t idx, int keyed, int64_t count, double* out) {
  uint64_t k0 = seed, k1 = rep;
  if (!keyed) stream_key(seed, rep, idx, k0, k1);
  const int64_t nb = (count + 3) >> 2;
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Block4 r = philox4x64_10(static_cast<uint64_t>(b) + 1ull, k0, k1);
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (4 * b + w < count) out[4 * b + w] = uniform_open_closed(r.w[w]);
  }
}

// sample() given uniforms (the FixedStream seam, test_distribution.py:24-32)
__global__ void draw_kernel(const double* __restrict__ cdf, const uint16_t* __restrict__ guide, uint32_t L,
                            const double* __restrict__ u, int64_t count, int64_t* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = u[i];
    int64_t v;
    if (x > 0.0 && x <= 1.0) {
      v = draw_value(x, guide, cdf, L, true);
    } else {
      // outside (0, 1]: plain lower_bound over the whole table (searchsorted semantics)
      uint32_t lo = 0, hi = L;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cdf[mid] >= x)
          hi = mid;
        else
          lo = mid + 1;
      }
      v = lo + 1 > L ? L : lo + 1;
    }
    out[i] = v;
  }
}

}  // namespace zks
