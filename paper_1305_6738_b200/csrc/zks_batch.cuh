// Replicate kernels for small and medium n (table-mode MLE): the shared lane / warp pieces and
// the two-kernel path.
//
// Same per-replicate pipeline as replicate_kernel (montecarlo.py:89-116), re-phased so that no
// phase is serial on a warp:
//   * n < kLaneDrawMaxN (lane_row_kernel, zks_lanes.cuh): a warp takes 32 consecutive replicate
//     indices, one lane each; each lane fits its replicate (Newton/bisection on the fit tables)
//     and walks its KS head k <= kKsHead (ks_lane_walk); short tails are scored lane by lane
//     (ks_tail_lane), long ones and NoRootError retries on stream idx + 2^32 warp-cooperatively;
//   * kLaneDrawMaxN <= n <= kPreMaxN: the draw phase (row_draw_kernel or draw_stats_kernel)
//     keeps only head counts, the tail values, log-sum / min / max; then fit_ks_kernel fits and
//     scores 32 rows per warp the same way, and retry_kernel takes the listed first-attempt
//     failures.
#pragma once
#include <type_traits>

#include "zks_replicate.cuh"

namespace zks {

#ifndef ZKS_DRAW_MINB
#define ZKS_DRAW_MINB 4
#endif
#ifndef ZKS_FIT_MINB
#define ZKS_FIT_MINB 3
#endif
constexpr int kLaneDrawMaxN = 128;  // below this n a lane draws a whole replicate

// warp totals of the lane-parallel fits' work counters into the warp's Work
__device__ __forceinline__ void add_lane_work(Work& wk, const Work& lw) {
  const unsigned long long f[4] = {lw.evals, lw.eval_terms, lw.norm_terms, lw.ks_terms};
  unsigned long long t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    t[i] = f[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t[i] += __shfl_xor_sync(0xffffffffu, t[i], o);
  }
  wk.evals += t[0];
  wk.eval_terms += t[1];
  wk.norm_terms += t[2];
  wk.ks_terms += t[3];
}

struct DrawStats {
  double log_sum;
  uint32_t vmin, vmax;
};

// g += (t < T), as one compare and one predicated add
__device__ __forceinline__ void inc_if_lt(uint32_t& g, uint32_t t, uint32_t T) {
  asm("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}" : "+r"(g) : "r"(t), "r"(T));
}

// f |= 1 if t equals any of T0..T3
__device__ __forceinline__ void flag_if_any_eq(uint32_t& f, uint32_t t, uint32_t T0, uint32_t T1, uint32_t T2,
                                               uint32_t T3) {
  asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\tsetp.eq.or.u32 p, %1, %3, p;\n\t"
      "setp.eq.or.u32 p, %1, %4, p;\n\tsetp.eq.or.u32 p, %1, %5, p;\n\t@p or.b32 %0, %0, 1;\n\t}"
      : "+r"(f)
      : "r"(t), "r"(T0), "r"(T1), "r"(T2), "r"(T3));
}

// Draw the n values of stream key (k0, k1) into v[0..n) (warp-cooperative); warp-reduced stats.
__device__ __forceinline__ DrawStats draw_sample(const ReplicateArgs& a, uint64_t k0, uint64_t k1,
                                                 const uint16_t* __restrict__ guide, uint16_t* v, int lane) {
  const int n = static_cast<int>(a.n);
  const int nb = (n + 3) >> 2;
  double ls = 0.0;
  uint32_t mn = 0xffffffffu, mx = 0;
  for (int b = lane; b < nb; b += 32) {
    const Block4 r = rng_block(static_cast<uint64_t>(b) + 1ull, k0, k1, a.rng);
    bool vb[4];
    uint32_t x[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) vb[w] = 4 * b + w < n;
    draw_block(r, vb, guide, a, x);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (vb[w]) {
        ls += __ldg(a.logs + x[w]);
        mn = min(mn, x[w]);
        mx = max(mx, x[w]);
      }
    }
    *reinterpret_cast<uint2*>(v + 4 * b) = make_uint2(x[0] | (x[1] << 16), x[2] | (x[3] << 16));
  }
  DrawStats s;
  s.log_sum = warp_sum(ls);
  s.vmin = warp_min_u32(mn);
  s.vmax = warp_max_u32(mx);
  return s;
}

__device__ __forceinline__ double fit_target(double log_sum, uint32_t vmin, int K, double dn) {
  double t = log_sum;
  if (t <= 0.0) t += kLn2;  // estimate.py:71-72
  t /= dn;
  if (K > 0 && vmin == static_cast<uint32_t>(K))  // estimate.py:126-129
    t -= (log(static_cast<double>(K)) - log(static_cast<double>(K - 1))) / dn;
  return t;
}

// KS of the stored sample v[0..n): histogram of 1..H, pages above H from v itself.
__device__ __forceinline__ double ks_from_sample(const ReplicateArgs& a, double g, double norm, uint32_t kmax,
                                                 uint32_t* hist, uint32_t* queue, uint16_t* v, int lane, Work& wk) {
  const int n = static_cast<int>(a.n);
  const uint32_t H = static_cast<uint32_t>(a.H);
  // values 1 and 2 (most of the mass for gamma >~ 1.5) are counted in registers: a shared
  // atomic on one bin from 32 lanes would serialise
  uint32_t c1 = 0, c2 = 0;
  for (int i = 4 * lane; i < n; i += 128) {
    const uint2 q = *reinterpret_cast<const uint2*>(v + i);
    const uint32_t x[4] = {q.x & 0xffffu, q.x >> 16, q.y & 0xffffu, q.y >> 16};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (i + w < n) {
        c1 += x[w] == 1u;
        c2 += x[w] == 2u;
        if (x[w] > 2u && x[w] <= H) atomicAdd(hist + x[w], 1u);
      }
    }
  }
  c1 = warp_sum_u32(c1);
  c2 = warp_sum_u32(c2);
  if (lane == 0) {
    hist[1] = c1;
    if (H >= 2) hist[2] = c2;
  }
  __syncwarp();
  const KsOut ko = ks_scan<uint16_t, false, true>(ks_params(a), g, norm, kmax, hist, v, static_cast<uint32_t>(n), queue, lane, wk);
  const int top = ko.used_pages ? a.hist_words : round_up(static_cast<int>(min(kmax, H)) + 1, 4);
  clear_hist(hist, min(top, a.hist_words), lane);
  return ko.D;
}

// Lane-parallel KS head: lane r walks k = 1..min(kmax, kKsHead) of its own replicate with the
// dense form F(k) = S(k)/norm, S the running sum of k^-g in the reference's order, and the
// counts count(k).  Returns true when the replicate is fully scored (kmax <= kKsHead, or the
// exit bound held); otherwise (S, C, D) at k = kKsHead seed the warp-cooperative tail
// (KsParams::from_head).
template <typename CountFn>
__device__ __forceinline__ bool ks_lane_walk(const ReplicateArgs& a, bool on, double g, double norm, uint32_t kmax,
                                             CountFn count, double& ks, double& S_out, uint32_t& C_out,
                                             double& D_out) {
  const uint32_t end = kmax < kKsHead ? kmax : kKsHead;
  const double inv = 1.0 / norm;
  double S = 0.0, D = 0.0;
  uint32_t C = 0;
  bool live = on;
  bool done = false;
  for (uint32_t k = 1; __any_sync(0xffffffffu, live && k <= end); ++k) {
    if (live && k <= end) {
      S += exp_bounded(-g * __ldg(a.logs + k));
      C += count(k);
      const double F = S * inv, E = static_cast<double>(C) * a.inv_n;
      const double gap = fabs(F - E);
      D = gap > D ? gap : D;
      // D > max(1 - E, 1 - F) + margin, without fmax's NaN handling (all finite here)
      if (D > (1.0 - E) + kKsMargin && D > (1.0 - F) + kKsMargin) {
        done = true;
        live = false;
      }
    }
  }
  done = done || kmax <= kKsHead;
  if (on && done) ks = D;
  S_out = S;
  C_out = C;
  D_out = D;
  __syncwarp();
  return on && done;
}

#ifndef ZKS_LANE_TAIL_MAX
#define ZKS_LANE_TAIL_MAX 48
#endif
constexpr uint32_t kLaneTailMax = ZKS_LANE_TAIL_MAX;  // longest tail ks_tail_lane takes (values above kKsHead)
constexpr int kLaneHistWords = (kKsHead + 1) * 32 / 4;  // u8 counts [value 0..64][lane]

// Small samples: the lane walk over lane r's private u8 histogram of its values <= kKsHead
// (value-major, so a warp's lanes touch neighbouring bytes; filled while drawing).
__device__ __forceinline__ bool ks_lane_head(const ReplicateArgs& a, bool on, double g, double norm, uint32_t kmax,
                                             const uint8_t* lh, double& ks, double& S, uint32_t& C, double& D) {
  const int lane = threadIdx.x & 31;
  return ks_lane_walk(a, on, g, norm, kmax, [&](uint32_t k) { return static_cast<uint32_t>(lh[k * 32 + lane]); }, ks,
                      S, C, D);
}

// Tail of replicate r of the warp (kmax > kKsHead) from its lane-walk state: the values above
// kKsHead among over[0..over_n), warp-cooperatively.
__device__ __forceinline__ KsOut ks_tail_from_head(const ReplicateArgs& a, int r, double g, double norm, uint32_t kmax,
                                                   double S, uint32_t C, double D, uint32_t* hist, int hist_words,
                                                   uint32_t page, uint32_t* queue, uint16_t* over,
                                                   uint32_t over_n, int lane, Work& wk) {
  KsParams p = ks_params(a);
  p.H = kKsHead;
  p.hist_words = hist_words;
  p.P = page;
  p.from_head = true;
  p.S0 = __shfl_sync(0xffffffffu, S, r);
  p.C0 = __shfl_sync(0xffffffffu, C, r);
  p.D0 = __shfl_sync(0xffffffffu, D, r);
  return ks_scan<uint16_t, false, true>(p, g, norm, kmax, hist, over, over_n, queue, lane, wk);
}

// Tail of this lane's own replicate (kmax > kKsHead), lane-parallel: its m values above the head
// v[0..m) are sorted by insertion and every distinct value x is scored at k = x - 1 and k = x
// from S(kKsHead) + em_block(x) -- ks_flush's per-endpoint arithmetic, so the statistic is the
// warp path's bit for bit (whose early exit never changes the maximum).  Sorts v in place.
__device__ __forceinline__ double ks_tail_lane(const ReplicateArgs& a, double g, double norm, double S, uint32_t C,
                                               double D, uint16_t* v, int m, uint32_t& endpoints) {
  KsCtx c;
  c.g = g;
  c.inv = 1.0 / norm;
  c.dn = static_cast<double>(a.n);
  c.inv_n = a.inv_n > 0.0 ? a.inv_n : 1.0 / c.dn;
  c.exact = false;
  c.logs = a.logs;
  ks_tail_ctx(c, g);
  for (int i = 1; i < m; ++i) {
    const uint16_t x = v[i];
    int j = i;
    for (; j > 0 && v[j - 1] > x; --j) v[j] = v[j - 1];
    v[j] = x;
  }
  for (int i = 0; i < m;) {
    const uint32_t x = v[i];
    int j = i + 1;
    while (j < m && v[j] == x) ++j;
    double fx;
    const double Sx = S + em_block(c, x, fx);
    D = fmax(D, fabs((Sx - fx) * c.inv - emp(c, C)));
    C += static_cast<uint32_t>(j - i);
    D = fmax(D, fabs(Sx * c.inv - emp(c, C)));
    ++endpoints;
    i = j;
  }
  return D;
}

// One replicate's second attempt on stream idx + 2^32 (montecarlo.py:106-115), warp-cooperative:
// draw into v, fit, score.  Returns the status (1 retried, 2 failed twice).
template <bool kCount>
__device__ __forceinline__ uint8_t retry_replicate(const ReplicateArgs& a, const ModelFns& M, uint64_t rel,
                                                   const uint16_t* guide, uint16_t* v, uint32_t* hist,
                                                   uint32_t* queue, int lane, double& ks, double& g, Work& wk) {
  uint64_t q0, q1;
  stream_key(a.seed, a.rep, a.first + rel + (1ull << 32), q0, q1);
  const DrawStats st = draw_sample(a, q0, q1, guide, v, lane);
  __syncwarp();
  const double t2 = fit_target(st.log_sum, st.vmin, a.K, static_cast<double>(a.n));
  double g2 = 0.0;
  const bool ok2 = fit_exponent(M, t2, lane, g2, wk);  // uniform: same inputs on every lane
  ks = __longlong_as_double(0x7ff8000000000000ll);
  if (ok2) ks = ks_from_sample(a, g2, fit_norm(a.fit, g2), st.vmax, hist, queue, v, lane, wk);
  if (kCount) {
    ++wk.attempts;
    wk.draws += a.n;
  }
  g = ok2 ? g2 : t2;  // failed twice: report the retry sample's mean log (diagnostics)
  return ok2 ? 1 : 2;
}

// per-warp shared memory of lane_row_kernel (zks_lanes.cuh): histogram, queue, 32 lane tail
// buffers of vals_stride values, one staging row of n values (long-tail redraws, retries); 16-byte aligned
__host__ __device__ constexpr int batch_warp_bytes(int hist_words, int vals_stride, int n) {
  return round_up(hist_words * 4 + kKsQueueWords * 4 + 32 * vals_stride * 2 + round_up(n, 4) * 2, 16);
}


constexpr int kHeadRowWords = kKsHead / 2 + 1;        // u16 counts of 1..kKsHead + pad: conflict-free columns
constexpr int kFitHistWords = 32 * kHeadRowWords;      // the head rows, reused as page histogram
constexpr int kFitStageWords = kOverCap / 2;             // one tail of <= kOverCap u16 values
constexpr int kFitWarpWords = kFitHistWords + kKsQueueWords + kFitStageWords;
#ifndef ZKS_FIT_LANE_TAIL_MAX
#define ZKS_FIT_LANE_TAIL_MAX 48
#endif
// longest tail list fit_ks_kernel scores lane by lane (0 = none): the insertion sort's serial
// latency outgrows the warp path's per-replicate cost at about this length
constexpr uint32_t kFitLaneTailMax = ZKS_FIT_LANE_TAIL_MAX;
static_assert(2 * kHeadRowWords >= static_cast<int>(kFitLaneTailMax), "a short tail is sorted in one head row");

// Fit + score of pre-drawn replicates (draw_stats_kernel): a warp takes 32 consecutive rows,
// fits them lane-parallel, walks each head k <= kKsHead lane by lane from the counts, and
// scores the tails that outlive the head warp-cooperatively from the tail lists.  First-attempt
// failures go to retry_list (count at [0], row offsets after) for retry_kernel.
// Rows whose tails outlive the register sort (m > kOverCap: page passes) are not scored by the
// warp that fitted them -- one such tail takes the warp for tens of page passes while its other
// 31 rows wait, and a heavy-tailed launch (gamma ~ 1.25, n ~ 5 x 10^4) then fills a fraction of
// the GPU.  fit_ks_kernel lists them with their head state instead (the retry list's pattern);
// long_tail_kernel scores them one warp per row, with the same function on the same inputs.
struct TailList {
  uint32_t* list;  // [0] = count, then row offsets in the chunk
  double* S;       // head state at k = kKsHead per listed row (ks_lane_walk's S, C, D)
  double* D;
  double* g;       // fitted exponent and normaliser
  double* norm;
  uint32_t* C;
  uint32_t* kmax;
};

template <bool kCount>
__global__ void __launch_bounds__(kThreads, ZKS_FIT_MINB) fit_ks_kernel(ReplicateArgs a, uint32_t* retry_list,
                                                                       TailList tl) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* heads = reinterpret_cast<uint32_t*>(smem) + warp * kFitWarpWords;
  uint32_t* hist = heads;  // page histogram once the lane walks are done
  uint32_t* queue = heads + kFitHistWords;
  uint16_t* stage = reinterpret_cast<uint16_t*>(queue + kKsQueueWords);  // the tail being scored
  const int K = a.K;
  const double dn = static_cast<double>(a.n);
  const uint64_t nbatches = (a.count + 31) / 32;
  Work wk{};
  const ModelFns M{K, a.logs, a.fit, true};

  for (;;) {
    unsigned long long bid = 0;
    if (lane == 0) bid = atomicAdd(a.work, 1ull);
    bid = __shfl_sync(0xffffffffu, bid, 0);
    if (bid >= nbatches) break;
    const uint64_t r0 = bid * 32;
    const uint64_t left = a.count - r0;
    const int nrep = left < 32u ? static_cast<int>(left) : 32;
    const bool active = lane < nrep;
    const uint64_t row = a.first + r0 + lane - a.pre_first;

    // head counts of the 32 rows into shared memory (128-byte rows, 16-byte loads)
    const uint4* src = reinterpret_cast<const uint4*>(a.pre_head + (a.first + r0 - a.pre_first) * kKsHead);
    for (int e = lane; e < nrep * 8; e += 32) {
      const uint4 q = __ldcs(src + e);
      uint32_t* d = heads + (e >> 3) * kHeadRowWords + (e & 7) * 4;
      d[0] = q.x;
      d[1] = q.y;
      d[2] = q.z;
      d[3] = q.w;
    }

    // exponent fits, one replicate per lane
    double g = 0.0, norm = 1.0;
    uint32_t vmax = 0;
    bool ok = false;
    Work lw{};
    uint32_t my_m = 0;
    if (active) {
      my_m = a.pre_m[row];
      vmax = a.pre_max[row];
      const double target = fit_target(a.pre_ls[row], a.pre_min[row], K, dn);
      ok = fit_exponent(M, target, lane, g, lw);
      if (ok) norm = fit_norm(a.fit, g);
      if (!ok) g = target;
      if (kCount && ok) {
        lw.norm_terms += ref_norm_terms(a.fit, g);
        lw.ks_terms += min(vmax, static_cast<uint32_t>(kSeam));
      }
    }
    if (kCount) {
      add_lane_work(wk, lw);
      wk.attempts += nrep;
    }
    __syncwarp();

    // heads lane by lane
    double my_ks = __longlong_as_double(0x7ff8000000000000ll);
    double hS, hD;
    uint32_t hC;
    const uint32_t* hr = heads + lane * kHeadRowWords;
    const bool scored = ks_lane_walk(a, ok && active, g, norm, vmax,
                                     [&](uint32_t k) { return (hr[(k - 1) >> 1] >> (((k - 1) & 1) * 16)) & 0xffffu; },
                                     my_ks, hS, hC, hD);
    // long tails, warp-cooperatively (the head rows are free now: pages reuse them).  The tail
    // values of the next replicate are loaded into registers while the current one is scored,
    // then staged in shared memory (tails of <= kOverCap values; longer ones read from HBM/L2).
    const bool tail = active && ok && !scored;
    // short tail lists lane by lane, sorted in the lane's own head row (free after its walk)
    const bool short_tail = tail && !a.dense_words && my_m <= kFitLaneTailMax;
    uint32_t ends = 0;
    if (short_tail) {
      uint16_t* buf = reinterpret_cast<uint16_t*>(heads + lane * kHeadRowWords);
      const uint16_t* t = a.pre_tail + row * a.vals_stride;
      for (uint32_t i = 0; i < my_m; ++i) buf[i] = t[i];
      my_ks = ks_tail_lane(a, g, norm, hS, hC, hD, buf, static_cast<int>(my_m), ends);
    }
    if (kCount) wk.ks_tails += warp_sum_u32(ends);
    __syncwarp();
    unsigned need = __ballot_sync(0xffffffffu, tail && !short_tail);
    if (!a.dense_words) {  // paged tails to long_tail_kernel, with the lane's head state
      const bool defer = tail && !short_tail && my_m > kOverCap;
      if (defer) {
        const uint32_t at = atomicAdd(tl.list, 1u);
        tl.list[1 + at] = static_cast<uint32_t>(r0 + lane);
        tl.S[at] = hS;
        tl.D[at] = hD;
        tl.g[at] = g;
        tl.norm[at] = norm;
        tl.C[at] = hC;
        tl.kmax[at] = vmax;
      }
      need &= ~__ballot_sync(0xffffffffu, defer);
    }
    if (a.dense_words) {  // dense finite support (K <= kDenseMaxK): the head walk continues
      // lane by lane over the row's counts of kKsHead+1..kmax, the reference's cumulative
      // form (gof.py:60-70) in the head's arithmetic; no endpoint formulas, no warp scans
      const uint32_t* counts = reinterpret_cast<const uint32_t*>(a.pre_tail + row * a.vals_stride);
      const double inv = 1.0 / norm;
      const bool fast_exp = fabs(g) <= 100.0;  // |g ln k| < 708 for k <= 1024
      double S = hS, D = hD;
      uint32_t C = hC;
      bool live = tail;
      for (uint32_t k = kKsHead + 1; __any_sync(0xffffffffu, live && k <= vmax); ++k) {
        if (live && k <= vmax) {
          const double x = -g * __ldg(a.logs + k);
          S += fast_exp ? exp_bounded(x) : exp(x);
          C += counts[k - (kKsHead + 1)];
          const double F = S * inv, E = static_cast<double>(C) * a.inv_n;
          const double gap = fabs(F - E);
          D = gap > D ? gap : D;
          if (D > (1.0 - E) + kKsMargin && D > (1.0 - F) + kKsMargin) live = false;
        }
      }
      if (tail) my_ks = D;
      need = 0;
    }
    uint32_t pv[kOverCap / 32], pm = 0;
    auto issue = [&](int r) {
      pm = __shfl_sync(0xffffffffu, my_m, r);
      const uint16_t* t = a.pre_tail + (a.first + r0 + r - a.pre_first) * a.vals_stride;
#pragma unroll
      for (int j = 0; j < kOverCap / 32; ++j) {
        const uint32_t i = j * 32 + lane;
        pv[j] = (pm <= kOverCap && i < pm) ? t[i] : 0u;
      }
    };
    int r = need ? __ffs(need) - 1 : -1;
    if (r >= 0) issue(r);
    while (r >= 0) {
      __syncwarp();  // the previous scan is done with the stage
      const uint32_t m = pm;
      if (m <= kOverCap) {
#pragma unroll
        for (int j = 0; j < kOverCap / 32; ++j)
          if (j * 32 + lane < m) stage[j * 32 + lane] = static_cast<uint16_t>(pv[j]);
      }
      __syncwarp();
      need &= need - 1;
      const int nx = need ? __ffs(need) - 1 : -1;
      if (nx >= 0) issue(nx);
      const double gr = __shfl_sync(0xffffffffu, g, r);
      const double nr = __shfl_sync(0xffffffffu, norm, r);
      const uint32_t kmax = __shfl_sync(0xffffffffu, vmax, r);
      uint16_t* over =
          m <= kOverCap ? stage : a.pre_tail + (a.first + r0 + r - a.pre_first) * a.vals_stride;
      const KsOut ko =
          ks_tail_from_head(a, r, gr, nr, kmax, hS, hC, hD, hist, kFitHistWords, kFitHistWords, queue, over, m, lane, wk);
      if (lane == r) my_ks = ko.D;
      r = nx;
    }
    __syncwarp();

    if (active) {
      if (!ok) retry_list[1 + atomicAdd(retry_list, 1u)] = static_cast<uint32_t>(r0 + lane);
      a.ks_out[r0 + lane] = my_ks;
      a.gh_out[r0 + lane] = g;
      a.st_out[r0 + lane] = ok ? 0 : 2;
    }
  }
  if (kCount && lane == 0) {
    const unsigned long long* f = &wk.attempts;
    for (int i = 0; i < kWorkFields; ++i)
      if (f[i]) atomicAdd(a.counters + i, f[i]);
  }
}

// The listed long tails (fit_ks_kernel), one warp per row: page passes over the row's tail
// values (compacted in place, ks_scan<..., kCompact>) from the row's head state -- exactly the
// call fit_ks_kernel would have made, with the same page and histogram sizes.
template <bool kCount>
#ifndef ZKS_LONG_MINB
#define ZKS_LONG_MINB 3
#endif
__global__ void __launch_bounds__(kThreads, ZKS_LONG_MINB) long_tail_kernel(ReplicateArgs a, const TailList tl) {
  const uint32_t cnt = *tl.list;
  if (cnt == 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem) + warp * (kFitHistWords + kKsQueueWords);
  uint32_t* queue = hist + kFitHistWords;
  Work wk{};
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t j = blockIdx.x * (blockDim.x >> 5) + warp; j < cnt; j += warps) {
    const uint32_t rel = tl.list[1 + j];
    const uint64_t row = a.first + rel - a.pre_first;
    uint16_t* over = a.pre_tail + row * a.vals_stride;
    const KsOut ko = ks_tail_from_head(a, 0, tl.g[j], tl.norm[j], tl.kmax[j], tl.S[j], tl.C[j], tl.D[j], hist,
                                       kFitHistWords, kFitHistWords, queue, over, a.pre_m[row], lane, wk);
    if (lane == 0) a.ks_out[rel] = ko.D;
    __syncwarp();
  }
  if (kCount && lane == 0) {
    const unsigned long long* f = &wk.attempts;
    for (int i = 0; i < kWorkFields; ++i)
      if (f[i]) atomicAdd(a.counters + i, f[i]);
  }
}

// per-warp shared memory of retry_kernel: histogram, queue, one sample (16-byte aligned)
__host__ __device__ constexpr int retry_warp_bytes(int hist_words, int vals_stride) {
  return round_up(hist_words * 4 + kKsQueueWords * 4 + vals_stride * 2, 16);
}

// Second attempts of the rows fit_ks_kernel listed (montecarlo.py:106-115), one warp each; exits
// at once when the list is empty (the common case).
template <bool kCount>
__global__ void __launch_bounds__(kThreads) retry_kernel(ReplicateArgs a, const uint32_t* retry_list) {
  const uint32_t cnt = *retry_list;
  if (cnt == 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* guide = reinterpret_cast<uint16_t*>(smem);
  const int guide_bytes = round_up(a.guide_levels * kGuideLevel * 2, 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp_bytes = retry_warp_bytes(a.hist_words, a.vals_stride);
  unsigned char* mine = smem + guide_bytes + warp * warp_bytes;
  uint32_t* hist = reinterpret_cast<uint32_t*>(mine);
  uint32_t* queue = hist + a.hist_words;
  uint16_t* vals = reinterpret_cast<uint16_t*>(mine + a.hist_words * 4 + 3 * kKsQueue * 4);
  load_guide(guide, a.guide, a.guide_levels);
  clear_hist(hist, a.hist_words, lane);
  __syncthreads();
  Work wk{};
  const ModelFns M{a.K, a.logs, a.fit, true};
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t j = blockIdx.x * (blockDim.x >> 5) + warp; j < cnt; j += warps) {
    const uint32_t rel = retry_list[1 + j];
    double ks, g;
    const uint8_t s = retry_replicate<kCount>(a, M, rel, guide, vals, hist, queue, lane, ks, g, wk);
    if (lane == 0) {
      a.ks_out[rel] = ks;
      a.gh_out[rel] = g;
      a.st_out[rel] = s;
    }
    __syncwarp();
  }
  if (kCount && lane == 0) {
    const unsigned long long* f = &wk.attempts;
    for (int i = 0; i < kWorkFields; ++i)
      if (f[i]) atomicAdd(a.counters + i, f[i]);
  }
}

// The draw phase on its own, at high occupancy: one warp per replicate of [first, first+count)
// draws its sample and writes what the fit and the KS scan need -- log-sum, min, max, the counts
// of the values 1..kKsHead and the list of values above it -- so fit_ks_kernel never touches the
// n draws again (n above the row kernel's range: kRowMaxN < n <= kPreMaxN, zks_rows.cuh).
//
// Values 1..4 are counted without a search: with h = cdf[0..3] and the exact cuts T_j of the
// 32-bit words (u > h_j <=> t < T_j, t = x >> 32 of the Philox word; h_j = +inf
// from L-1 on clamps to L, distribution.py:200-201), a per-block table indexed by a word's top
// 10 bits holds the count increment of the value every word of that 2^22-wide range takes, or
// 0 when the range holds a cut or lies above h_3.  Those words -- 5 % of them at gamma = 2.5,
// 36 % at 1.5, plus the rare ranges with a cut -- are pushed onto a warp queue and resolved 32 at
// a time by the guide + cdf search with every lane busy, so divergence costs nothing.
constexpr int kDrawQueue = 160;  // entries per warp: < 32 left over + 4 x 32 pushed per step
constexpr int kCutTabBits = 10;  // the cut table: one entry per 2^22-wide range of 32-bit words

// The cut table of a sampling table: entry i covers the words t in [i 2^22, (i+1) 2^22).  With
// the exact cuts T_j (u > cdf[j] <=> t < T_j, t = T_j undecided), a range holding no cut decides
// the value 1 + #{j : T_j > t} of all its words: the entry is the count increment 1 << 8(v-1)
// for v <= 4.  A range above h_3 whose extreme uniforms (u_max = 1 - i 2^-10 and u_min =
// 1 - (i+1) 2^-10 + 2^-53, the bounds of u for a Philox draw whose top 32 bits lie in the range)
// see the same count c of the first 64 cdf entries below them decides the value v = c + 1 <= 64
// of all its words (no cdf entry lies in [u_min, u_max)): the entry is kDirect | v, counted
// straight into the lane's bin.  Any
// other range is 0: queued for the exact search.  head64 = cdf[0..63] (+inf from L-1 on).
constexpr uint32_t kDirect = 0x80000000u;
__device__ __forceinline__ uint32_t count_below(const double* head64, double u) {
  uint32_t lo = 0, hi = 64;  // #{j < 64 : head64[j] < u}
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (head64[mid] < u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ void build_cut_table(uint32_t* tab, const uint32_t tcut[4], const double* head64) {
  for (int i = threadIdx.x; i < (1 << kCutTabBits); i += blockDim.x) {
    const uint32_t lo = static_cast<uint32_t>(i) << (32 - kCutTabBits);
    const uint32_t hi = lo + ((1u << (32 - kCutTabBits)) - 1u);
    int c = 0;
    bool cut = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      c += tcut[j] > hi;
      cut |= tcut[j] >= lo && tcut[j] <= hi;
    }
    uint32_t e = (cut || c == 4) ? 0u : (1u << (8 * c));
    if (!cut && c == 4) {
      const double umax = 1.0 - static_cast<double>(i) * 0x1p-10;
      const double umin = (1.0 - static_cast<double>(i + 1) * 0x1p-10) + 0x1p-53;
      const uint32_t cmin = count_below(head64, umin), cmax = count_below(head64, umax);
      if (cmin == cmax && cmax < 64u) e = kDirect | (cmax + 1u);
    }
    tab[i] = e;
  }
}
constexpr int kPreMaxN = 65535;     // largest n of the two-kernel path (u16 counts; tail rows of 2n B)
constexpr int kDenseMaxK = 1024;       // finite supports kept as dense counts above the head
constexpr int kNarrowBinsMaxN = 3968;  // a lane bins <= n/32 + 1 queued and <= n/32 + 4 direct draws: u8 up to here
// per-warp smem of draw_stats_kernel: bins [v][lane] (u8, or u16 above kNarrowBinsMaxN) + queue
__host__ __device__ constexpr int draw_warp_bytes(bool wide) { return (kKsHead + 1) * 32 * (wide ? 2 : 1) + kDrawQueue * 8; }

struct DrawRowOut {
  double ls;
  uint32_t mn, mx, m;
};

// One replicate row (warp-cooperative).
template <typename BinT>
__device__ __forceinline__ void draw_row(const ReplicateArgs& a, uint64_t idx, const uint16_t* __restrict__ guide,
                                         const uint32_t* __restrict__ ctab, BinT* bins, double* queue,
                                         uint32_t* dense, uint16_t* tail, uint16_t* head, DrawRowOut& o, int lane) {
  const bool two = a.guide_levels == 2;
  const int n = static_cast<int>(a.n);
  const int nb = (n + 3) >> 2;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t k0 = 0, k1 = 0;
  stream_key(a.seed, a.rep, idx, k0, k1);
  double ls = 0.0;
  uint32_t mn = 0xffffffffu, mx = 0, m = 0;
  uint32_t acc = 0;          // this lane's counts of the values 1..4, 8-bit fields (flushed below)
  uint32_t acc02 = 0, acc13 = 0;  // ... accumulated in 16-bit fields
  int qn = 0;                               // queued draws (warp-uniform)
  // one queued draw per lane: value by guide + search, then bin / tail
  auto resolve = [&](double ur, bool ok) {
    uint32_t lo, hi;
    guide_bracket_fine(ur, guide, a.guide_fine, two, lo, hi);
    if (!ok) hi = lo;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(a.cdf + mid) >= ur)
        hi = mid;
      else
        lo = mid + 1;
    }
    const uint32_t v = min(lo + 1, a.L);
    if (ok) {
      mn = min(mn, v);
      mx = max(mx, v);
      ZKS_CHECK(v >= 1u && v <= a.L);
      if (v <= kKsHead) ++bins[v * 32 + lane];
    }
    const bool big = ok && v > kKsHead;
    const unsigned bm = __ballot_sync(0xffffffffu, big);
    if (big) {
      if (dense) {
        ZKS_CHECK(static_cast<int>(v - kKsHead) <= a.dense_words);
        atomicAdd(dense + (v - kKsHead - 1), 1u);
      } else {
        ZKS_CHECK(m + __popc(bm & lt) < static_cast<uint32_t>(a.vals_stride));
        tail[m + __popc(bm & lt)] = static_cast<uint16_t>(v);
      }
      ls += __ldg(a.logs + v);
    }
    m += __popc(bm);
  };
  // one step: lane b's block of 4 draws.  A word's top 10 bits index ctab: the count increment
  // of its value 1..4 (1 << 8(v-1)), or 0 = queue it (value above 4, or a cut inside the bin);
  // kMasked for the last step (words past n count nowhere)
  auto step = [&](int b, auto masked) {
    uint32_t t4[4];
    double w4[4];
    const Block4 r = rng_block(static_cast<uint64_t>(b) + 1ull, k0, k1, a.rng);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      t4[w] = static_cast<uint32_t>(r.w[w] >> 32);
      w4[w] = uniform_open_closed(r.w[w]);
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t e = ctab[t4[w] >> (32 - kCutTabBits)];
      bool big = e == 0u;
      if (decltype(masked)::value && 4 * b + w >= n) {
        e = 0u;
        big = false;
      }
      if (e & kDirect) {  // a value 5..kKsHead decided by its range: the lane's own bin
        ++bins[(e & 0xffu) * 32 + lane];
        e = 0u;
      }
      acc += e;
      const unsigned bm = __ballot_sync(0xffffffffu, big);
      if (big) queue[qn + __popc(bm & lt)] = w4[w];
      qn += __popc(bm);
    }
    __syncwarp();
    while (qn >= 32) {
      qn -= 32;
      const double q = queue[qn + lane];
      __syncwarp();
      resolve(q, true);
    }
  };
  auto flush = [&]() {  // 8-bit fields hold <= 63 steps x 4 words
    acc02 += acc & 0x00ff00ffu;
    acc13 += (acc >> 8) & 0x00ff00ffu;
    acc = 0u;
  };
  const int full = (n >> 2) & ~31;  // blocks in steps whose 4 x 32 words are all in the sample
  int b0 = 0;
  for (int chunk = 0; b0 < full; b0 += 32) {
    step(b0 + lane, std::false_type{});
    if (++chunk == 63) {
      flush();
      chunk = 0;
    }
  }
  for (; b0 < nb; b0 += 32) step(b0 + lane, std::true_type{});
  flush();
  if (qn) {
    const bool ok = lane < qn;
    const double q = ok ? queue[lane] : 0.0;
    __syncwarp();
    resolve(q, ok);
  }
  // counts of 1..4 counted by the cut table (the queued ones are in the bins)
  const uint32_t c02 = warp_sum_u32(acc02), c13 = warp_sum_u32(acc13);  // n < 2^16
  __syncwarp();
  // head[k - 1] = count of value k: lane l sums the 32 lane columns of k = l + 1 and l + 33
  uint32_t hc0 = 0, hc1 = 0;
  const uint32_t* r0 = reinterpret_cast<const uint32_t*>(bins + (lane + 1) * 32);
  const uint32_t* r1 = reinterpret_cast<const uint32_t*>(bins + (lane + 33) * 32);
  constexpr int kWords = 32 * sizeof(BinT) / 4;  // words per bin row
#pragma unroll
  for (int j = 0; j < kWords; ++j) {
    const int jj = (j + lane) & (kWords - 1);  // rotate the word so the warp's loads spread over banks
    const uint32_t w0 = r0[jj], w1 = r1[jj];
    if (sizeof(BinT) == 1) {
      hc0 = __dp4a(w0, 0x01010101u, hc0);  // sum of the word's 4 bytes
      hc1 = __dp4a(w1, 0x01010101u, hc1);
    } else {
      hc0 += (w0 & 0xffffu) + (w0 >> 16);
      hc1 += (w1 & 0xffffu) + (w1 >> 16);
    }
  }
  __syncwarp();
  if (lane < 4) hc0 += ((lane & 1) ? c13 : c02) >> (16 * (lane >> 1)) & 0xffffu;
  for (int i = lane; i < kKsHead * 8 * static_cast<int>(sizeof(BinT)); i += 32)
    reinterpret_cast<uint32_t*>(bins + 32)[i] = 0u;
  if (dense) {  // counts of kKsHead+1..K into the row's tail slot (u32), the warp histogram reset
    __syncwarp();
    uint32_t* out = reinterpret_cast<uint32_t*>(tail);
    for (int i = lane; i < a.dense_words; i += 32) {
      out[i] = dense[i];
      dense[i] = 0u;
    }
    __syncwarp();
  }
  head[lane] = static_cast<uint16_t>(hc0);  // n <= kPreMaxN: u16 counts
  head[lane + 32] = static_cast<uint16_t>(hc1);
  mn = min(mn, hc0 ? lane + 1u : (hc1 ? lane + 33u : 0xffffffffu));
  mx = max(mx, hc1 ? lane + 33u : (hc0 ? lane + 1u : 0u));
  o.mn = warp_min_u32(mn);
  o.mx = warp_max_u32(mx);
  // log-sum: the head from its counts, the tail value by value (estimate.py:59-73 sums ln x_i)
  ls += static_cast<double>(hc0) * __ldg(a.logs + lane + 1) + static_cast<double>(hc1) * __ldg(a.logs + lane + 33);
  o.ls = warp_sum(ls);
  o.m = m;
}

template <bool kCount, bool kWide>
__global__ void __launch_bounds__(kThreads, ZKS_DRAW_MINB) draw_stats_kernel(ReplicateArgs a, uint16_t* head_out,
                                                                 uint16_t* tail_out, uint32_t* m_out, double* ls_out,
                                                                 uint32_t* min_out, uint32_t* max_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint16_t* guide = reinterpret_cast<uint16_t*>(smem);
  const int guide_bytes = round_up(kGuideLevel * 2, 16);  // level 1 only (level 2: the fine one, global)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using BinT = typename std::conditional<kWide, uint16_t, uint8_t>::type;
  uint32_t* ctab = reinterpret_cast<uint32_t*>(smem + guide_bytes);
  unsigned char* wbase = smem + guide_bytes + (4 << kCutTabBits) + warp * (draw_warp_bytes(kWide) + a.dense_words * 4);
  // lane-private counts of the values 5..kKsHead, value-major ([v][lane]): a lane resolves at
  // most one queued draw per pop and there are <= n/32 + 1 pops, plus its direct draws (<= 4 per
  // step of its <= n/128 + 1 steps): u8 up to kNarrowBinsMaxN
  BinT* bins = reinterpret_cast<BinT*>(wbase);
  double* queue = reinterpret_cast<double*>(wbase + (kKsHead + 1) * 32 * sizeof(BinT));
  uint32_t* dense = a.dense_words ? reinterpret_cast<uint32_t*>(wbase + draw_warp_bytes(kWide)) : nullptr;
  for (int i = lane; i < a.dense_words; i += 32) dense[i] = 0u;
  load_guide(guide, a.guide, 1);
  // cdf[0..63] staged in warp 0's queue (not in use yet) for the cut table's direct entries
  double* head64 = reinterpret_cast<double*>(smem + guide_bytes + (4 << kCutTabBits) + (kKsHead + 1) * 32 * sizeof(BinT));
  for (int j = threadIdx.x; j < 64; j += blockDim.x) head64[j] = j + 1 < static_cast<int>(a.L) ? __ldg(a.cdf + j) : __longlong_as_double(0x7ff0000000000000ll);
  __syncthreads();
  build_cut_table(ctab, a.tcut, head64);
  for (int v = 0; v <= static_cast<int>(kKsHead); ++v) bins[v * 32 + lane] = 0;
  __syncthreads();
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (blockDim.x >> 5);
  unsigned long long rows = 0, tails = 0;
  for (uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < a.count; i += warps) {
    const uint64_t idx = a.first + i;
    uint16_t* tail = tail_out + i * a.vals_stride;
    uint16_t* head = head_out + i * kKsHead;
    DrawRowOut o;
    draw_row(a, idx, guide, ctab, bins, queue, dense, tail, head, o, lane);
    if (lane == 0) {
      ls_out[i] = o.ls;
      min_out[i] = o.mn;
      max_out[i] = o.mx;
      m_out[i] = o.m;
    }
    ++rows;
    tails += o.m;
  }
  if (kCount && lane == 0) {
    if (rows) atomicAdd(a.counters + 1, rows * static_cast<unsigned long long>(a.n));  // Philox draws
    if (rows) atomicAdd(a.counters + kWorkFields + 1, rows);
    if (tails) atomicAdd(a.counters + kWorkFields + 2, tails);
  }
}

}  // namespace zks
