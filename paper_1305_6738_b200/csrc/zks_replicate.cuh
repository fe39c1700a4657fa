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
#include "zks_series.cuh"
#include "zks_stream.cuh"

namespace zks {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kHistMax = 2048;             // histogram bins held in shared memory per warp
constexpr int kGuideLog2 = 12;              // guide table resolution G = 4096
constexpr int kGuide = 1 << kGuideLog2;
constexpr double kLn2 = 0.69314718055994530942;  // math.log(2.0)
constexpr double kKsMargin = 1e-11;  // early-exit safety margin (>> fp64 rounding of the sums)

struct ReplicateArgs {
  const double* cdf;
  const uint16_t* guide;
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
  int batch;                     // replicates per warp batch (replicate_batch_kernel)
  int vals_stride;               // u16 sample slots per replicate in the batch store
};

__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// smallest k (1-based) with cdf[k-1] >= u, clamped to L (distribution.py:200-201)
__device__ __forceinline__ uint32_t draw_value(double u, const uint16_t* __restrict__ guide,
                                               const double* __restrict__ cdf, uint32_t L) {
  const int j = static_cast<int>(u * static_cast<double>(kGuide));  // exact: G is 2^12
  uint32_t lo = guide[j], hi = guide[j + 1];
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
__device__ __forceinline__ void draw_block(const Block4& r, const bool valid[4], const uint16_t* __restrict__ guide,
                                           const double* __restrict__ cdf, uint32_t L, uint32_t out[4]) {
  double u[4];
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    u[w] = uniform_open_closed(r.w[w]);
    const int j = static_cast<int>(u[w] * static_cast<double>(kGuide));
    lo[w] = valid[w] ? guide[j] : 0u;
    hi[w] = valid[w] ? guide[j + 1] : 0u;
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
      cv[w] = act[w] ? __ldg(cdf + mid[w]) : 0.0;
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
  for (int w = 0; w < 4; ++w) out[w] = valid[w] ? min(lo[w] + 1, L) : 0u;
}

struct SampleStats {
  double log_sum;
  uint32_t vmin, vmax, over;
};

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

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
    const Block4 r = philox4x64_10(static_cast<uint64_t>(b) + 1ull, k0, k1);
    bool vb[4];
    uint32_t vv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) vb[w] = (4 * b + w) < n;
    draw_block(r, vb, guide, a.cdf, a.L, vv);
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

// estimate.py:115-146 with DEFAULT_SETTINGS (x0 = 0.5, tol 1e-5, 200 iterations, [-20, 20])
__device__ bool fit_exponent(const ModelFns& M, double target, int lane, double& g, Work& wk) {
  double lo = -20.0, hi = 20.0;
  if (M.K == 0) {
    lo = kMinUnboundedGamma;
    hi = kMaxUnboundedGamma;
  }
  double x = 0.5;
  if (!(lo < x && x < hi)) x = lo + 0.01;
  for (int it = 0; it < 200; ++it) {
    double mean, slope;
    if (!model_mean_slope(M, x, lane, mean, slope, wk)) return false;
    const double x_new = x + (mean - target) / slope;
    if (!isfinite(x_new) || x_new < lo || x_new > hi) return bisect_root(M, target, lane, lo, hi, g, wk);
    if (fabs(x_new - x) <= 1e-5) {
      g = x_new;
      return true;
    }
    x = x_new;
  }
  return bisect_root(M, target, lane, lo, hi, g, wk);
}

// ---------------------------------------------------------------------------- KS statistic
//
// The reference scans F(k) - E(k) over every k = 1..kmax (gof.py:60-68), or, for an unbounded
// fit with kmax > 4096, only the stretch endpoints v and v-1 of the observed values v, with
// F from the cumulative table below the seam and an Euler-Maclaurin tail above it
// (gof.py:71-105).  Both give the same supremum (E is constant between observations while F
// rises, so each stretch attains its extremes at its ends).  Here:
//   * head, k <= kKsHead: dense, F(k) = S(k) / norm with S the running sum of k^-g, exactly
//     the reference's cumulative form;
//   * k > kKsHead: endpoints only, S(v) = S(kKsHead) + EM(kKsHead+1 .. v) by Euler-Maclaurin
//     through the third-derivative term (the order of series.tail_mass, series.py:141-160),
//     S(v-1) = S(v) - v^-g.  Observed values are gathered tile by tile from the histogram
//     into a per-warp queue and scored 32 at a time, so the exp work scales with the number of
//     distinct values, not with kmax.
// The scan stops once no later k can beat the current maximum:
//   sup_{k' > k} |F(k') - E(k')| <= max(1 - E(k), 1 - F(k)).
constexpr uint32_t kKsHead = 64;
constexpr int kKsQueue = 64;  // per-warp endpoint queue entries

struct KsState {
  double S;       // running sum of k^-g through the last dense k
  double S_head;  // S(min(kmax, kKsHead))
  double Dw;      // warp max of D as of the last flush (warp-uniform)
  uint32_t Cb;    // observations <= last processed k
  double D;       // lane-local running max gap
  bool done;
  uint32_t next_fcheck;  // no F-based exit test before this k
};

struct KsCtx {
  double g, inv, inv_n;
  double fa, a_pow, La;  // f(a) = a^-g, a^(1-g), ln a for a = kKsHead + 1
  const double* logs;
  uint32_t* qk;  // queue: value v
  uint32_t* qc;  // queue: observations < v
  uint32_t* qn;  // queue: observations == v
};

// S(v) - S(kKsHead) = sum_{k=a}^{v} k^-g, a = kKsHead + 1, by Euler-Maclaurin; also returns v^-g
__device__ __forceinline__ double em_block(const KsCtx& c, uint32_t v, double& fv) {
  const double Lv = __ldg(c.logs + v);
  const double b = static_cast<double>(v);
  const double a = static_cast<double>(kKsHead + 1);
  fv = exp(-c.g * Lv);
  const double om = 1.0 - c.g;
  // integral_a^v x^-g dx = a^(1-g) * expm1((1-g) ln(v/a)) / (1-g), continuous through g = 1
  const double integral = (om == 0.0) ? (Lv - c.La) : c.a_pow * expm1(om * (Lv - c.La)) / om;
  const double d1 = -c.g * (fv / b - c.fa / a);  // f'(v) - f'(a)
  const double g3 = c.g * (c.g + 1.0) * (c.g + 2.0);
  const double d3 = -g3 * (fv / (b * b * b) - c.fa / (a * a * a));  // f'''(v) - f'''(a)
  return integral + 0.5 * (c.fa + fv) + d1 / 12.0 - d3 / 720.0;
}

// score queue entries [0, cnt) lane-parallel (cnt <= 32)
__device__ __forceinline__ void ks_flush(KsState& s, const KsCtx& c, int cnt, int lane, Work& wk) {
  if (cnt <= 0) return;
  double Fv = 0.0;
  if (lane < cnt) {
    const uint32_t v = c.qk[lane];
    const uint32_t before = c.qc[lane];
    const uint32_t here = c.qn[lane];
    double fv;
    const double Sv = s.S_head + em_block(c, v, fv);
    Fv = Sv * c.inv;
    const double Fp = (Sv - fv) * c.inv;
    const double E = static_cast<double>(before + here) * c.inv_n;
    const double Eb = static_cast<double>(before) * c.inv_n;
    s.D = fmax(s.D, fmax(fabs(Fv - E), fabs(Fp - Eb)));
  }
  wk.ks_tails += cnt;
}

// exit test: every later gap is bounded by max(1 - E, 1 - F) at the scan position
__device__ __forceinline__ void ks_check(KsState& s, double F_pos, double inv_n) {
  const double Dw = warp_max(s.D);
  const double bound = fmax(1.0 - static_cast<double>(s.Cb) * inv_n, 1.0 - F_pos);
  if (Dw > bound + kKsMargin) s.done = true;
}

// Tiles of 32 consecutive k in [k_first, k_last] with counts[k - base], above the head.
__device__ __forceinline__ void ks_sparse_tiles(KsState& s, const KsCtx& c, int& q, uint32_t k_first,
                                                uint32_t k_last, const uint32_t* counts, uint32_t base, int lane,
                                                Work& wk) {
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t k0 = k_first; k0 <= k_last && !s.done; k0 += 32) {
    ++wk.ks_tiles;
    const uint32_t k = k0 + lane;
    const bool in = k <= k_last;
    const uint32_t cnt = in ? counts[k - base] : 0u;
    const uint32_t C = s.Cb + warp_scan_u32(cnt, lane);
    const unsigned nz = __ballot_sync(0xffffffffu, cnt != 0u);
    if (cnt) {
      const int slot = q + __popc(nz & lt);
      c.qk[slot] = k;
      c.qc[slot] = C - cnt;
      c.qn[slot] = cnt;
    }
    q += __popc(nz);
    s.Cb = __shfl_sync(0xffffffffu, C, 31);
    __syncwarp();
    if (q >= 32) {
      ks_flush(s, c, 32, lane, wk);
      __syncwarp();
      uint32_t a0 = 0, a1 = 0, a2 = 0;
      if (lane < q - 32) {
        a0 = c.qk[32 + lane];
        a1 = c.qc[32 + lane];
        a2 = c.qn[32 + lane];
      }
      __syncwarp();
      if (lane < q - 32) {
        c.qk[lane] = a0;
        c.qc[lane] = a1;
        c.qn[lane] = a2;
      }
      q -= 32;
      __syncwarp();
      s.Dw = warp_max(s.D);
    }
    // exit test, only once the empirical part of the bound allows it (D changes only at flushes)
    const uint32_t k_hi = min(k0 + 31u, k_last);
    // (F checks back off geometrically in k: heavy tails make F approach 1 slowly)
    if (k_hi >= s.next_fcheck && s.Dw > 1.0 - static_cast<double>(s.Cb) * c.inv_n + kKsMargin) {
      ks_flush(s, c, q, lane, wk);
      q = 0;
      __syncwarp();
      s.Dw = warp_max(s.D);
      double fk;
      const double F_pos = (s.S_head + em_block(c, k_hi, fk)) * c.inv;
      ++wk.ks_tails;
      if (s.Dw > fmax(1.0 - static_cast<double>(s.Cb) * c.inv_n, 1.0 - F_pos) + kKsMargin)
        s.done = true;
      else
        s.next_fcheck = 2 * k_hi - kKsHead;
    }
  }
}

// KS of one sample: counts of 1..H in `hist`; values above H are found in over_vals[0..over_n)
// (which may also hold values <= H: they are ignored).  `queue` is 3 * kKsQueue u32 of
// per-warp shared memory.
__device__ double ks_scan(const ReplicateArgs& a, double g, double norm, uint32_t kmax, uint32_t* hist,
                          const uint16_t* over_vals, uint32_t over_n, uint32_t* queue, int lane, bool& used_pages,
                          Work& wk) {
  KsCtx c;
  c.g = g;
  c.inv = 1.0 / norm;
  c.inv_n = 1.0 / static_cast<double>(a.n);
  c.logs = a.logs;
  c.qk = queue;
  c.qc = queue + kKsQueue;
  c.qn = queue + 2 * kKsQueue;
  const uint32_t H = static_cast<uint32_t>(a.H);
  KsState s{0.0, 0.0, 0.0, 0u, 0.0, false, 0u};  // S, S_head, Dw, Cb, D, done, next_fcheck
  used_pages = false;

  // head: dense, exactly the reference's cumulative form
  const uint32_t head_end = min(kmax, kKsHead);
  for (uint32_t k0 = 1; k0 <= head_end && !s.done; k0 += 32) {
    ++wk.ks_tiles;
    const uint32_t k = k0 + lane;
    const bool in = k <= head_end;
    const uint32_t cnt = in ? hist[k] : 0u;
    const uint32_t C = s.Cb + warp_scan_u32(cnt, lane);
    const double term = in ? exp(-g * __ldg(a.logs + k)) : 0.0;
    const double S = s.S + warp_scan(term, lane);
    if (in) s.D = fmax(s.D, fabs(S * c.inv - static_cast<double>(C) * c.inv_n));
    s.S = __shfl_sync(0xffffffffu, S, 31);
    s.Cb = __shfl_sync(0xffffffffu, C, 31);
    wk.ks_terms += min(32u, head_end - k0 + 1);
    ks_check(s, s.S * c.inv, c.inv_n);
  }
  if (s.done || kmax <= kKsHead) return warp_max(s.D);
  s.S_head = s.S;
  s.Dw = warp_max(s.D);
  c.La = __ldg(a.logs + kKsHead + 1);
  c.fa = exp(-g * c.La);
  c.a_pow = static_cast<double>(kKsHead + 1) * c.fa;

  // above the head: endpoints of the observed values
  int q = 0;
  ks_sparse_tiles(s, c, q, kKsHead + 1, min(kmax, H), hist, 0u, lane, wk);
  uint32_t pa = H + 1;
  while (!s.done && pa <= kmax) {
    used_pages = true;
    const uint32_t pb = min(pa + H - 1, kmax);
    // page histogram of the values in [pa, pb]; next occupied value above pb
    for (int i = lane; i < a.hist_words; i += 32) hist[i] = 0u;
    __syncwarp();
    uint32_t next = 0xffffffffu;
    for (uint32_t i = lane; i < over_n; i += 32) {
      const uint32_t v = over_vals[i];
      if (v >= pa && v <= pb)
        atomicAdd(hist + (v - pa), 1u);
      else if (v > pb)
        next = min(next, v);
    }
    next = warp_min_u32(next);
    __syncwarp();
    ks_sparse_tiles(s, c, q, pa, pb, hist, pa, lane, wk);
    pa = pb + 1;
    if (next != 0xffffffffu && next > pa) pa = next;  // no observations in between: no endpoints
  }
  ks_flush(s, c, q, lane, wk);
  return warp_max(s.D);
}

__device__ __forceinline__ void clear_hist(uint32_t* hist, int words, int lane) {
  uint4* h4 = reinterpret_cast<uint4*>(hist);
  for (int i = lane; i < words / 4; i += 32) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
}

template <bool kCount>
__global__ void __launch_bounds__(kThreads, 1) replicate_kernel(ReplicateArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* guide = reinterpret_cast<uint16_t*>(smem);
  const int guide_bytes = round_up((kGuide + 2) * 2, 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + guide_bytes) + warp * (a.hist_words + 3 * kKsQueue);
  uint32_t* queue = hist + a.hist_words;
  for (int i = threadIdx.x; i < kGuide + 2; i += blockDim.x) guide[i] = a.guide[i];
  clear_hist(hist, a.hist_words, lane);
  __syncthreads();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  uint16_t* slab = a.slab ? a.slab + gw * a.slab_cap : nullptr;
  const int K = a.K;
  const double dn = static_cast<double>(a.n);
  Work wk{0, 0, 0, 0, 0, 0, 0, 0};
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
        ks = ks_scan(a, g, norm, st.vmax, hist, slab, st.over, queue, lane, used_pages, wk);
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

// guide[j] = lower_bound(cdf, j / G) for j = 0..G; guide[G + 1] = L
__global__ void guide_kernel(const double* __restrict__ cdf, uint32_t L, uint16_t* guide) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > kGuide + 1) return;
  if (j == kGuide + 1) {
    guide[j] = static_cast<uint16_t>(L);
    return;
  }
  const double u = static_cast<double>(j) / static_cast<double>(kGuide);
  uint32_t lo = 0, hi = L;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cdf[mid] >= u)
      hi = mid;
    else
      lo = mid + 1;
  }
  guide[j] = static_cast<uint16_t>(lo);
}

// RandomStream.uniforms (distribution.py:186-187) for one stream, block-parallel
__global__ void uniforms_kernel(uint64_t seed, uint64_t rep, uint64_t idx, int64_t count, double* out) {
  uint64_t k0, k1;
  stream_key(seed, rep, idx, k0, k1);
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
      v = draw_value(x, guide, cdf, L);
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
