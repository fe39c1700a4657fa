// Exponent-fit tables: piecewise polynomial (Chebyshev-fitted, evaluated by split Horner) images of
// the reference's model-moment functions, built once per support on the device.
//
// The reference evaluates, at every Newton / bisection iterate x (estimate.py:76-83, 94-146),
//     mean(x) = s1/s0,  slope(x) = s2/s0 - mean^2,   s_p(x) = sum_k k^-x (ln k)^p
// over 1..K (series.py:68-73) or as the zeta series (series.py:102-123: 256 or 512 direct terms
// plus an Euler-Maclaurin tail, m chosen by a tail-bound rule), and the fitted model's
// normaliser at the root (series.py:126-138).  Each evaluation is 256..32766 exps.  Here the
// three functions mu = s1/s0, m2 = s2/s0 and norm = s0 (zeta_value for K = inf) are tabulated
// over the admissible bracket in intervals of width h with degree-11 polynomials fitted at
// Chebyshev nodes, where every node value is the reference's own formula (same m rule, same
// tails) summed with compensated arithmetic.  Piece boundaries sit on the m-rule switch
// points, so each piece is analytic and the fit error is ~1e-16 relative; slope is formed at
// run time as m2 - mu^2 exactly like the reference, and the Newton control flow is unchanged.
// An evaluation is ~2 x 12 FMAs instead of thousands of exps.
#pragma once
#include <cstdint>

#include "zks_series.cuh"

namespace zks {

constexpr int kFitDeg = 11;
constexpr int kFitCoef = kFitDeg + 1;
constexpr int kFitFuncs = 3;  // mu, m2, norm
constexpr int kFitStride = kFitFuncs * kFitCoef;
constexpr int kFitMaxSeg = 6;

// the reference's m-rule switch points (located by bisection on the oracle, which is
// bit-identical to the reference; tests/test_fit_tables.py re-derives them)
constexpr double kMomSwitchLo = 1.0724527021401063;   // zeta_log_moments and zeta_value: 256 below, 512 above
constexpr double kMomSwitchHi = 2.669354230977903;    // zeta_log_moments: 512 below, 256 above
constexpr double kValSwitchHi = 1.3813464643463403;   // zeta_value:       512 below, 256 above

struct FitSeg {
  double x0;     // left end
  double h;      // interval width
  double inv_h;  // 1 / h
  int n;         // intervals
  int base;      // first interval index
  int m_mom;     // direct terms of the moment series in this segment (unbounded)
  int m_norm;    // direct terms of the zeta_value series (unbounded)
};

struct FitTable {
  const double* coef;  // [intervals][kFitFuncs][kFitCoef], monomial in t in [-1, 1]
  FitSeg seg[kFitMaxSeg];
  int nseg;
  int K;  // 0 = unbounded
  int intervals;
};

__device__ __forceinline__ int fit_locate(const FitTable& T, double x, double& t) {
  int s = 0;
#pragma unroll
  for (int i = 1; i < kFitMaxSeg; ++i)
    if (i < T.nseg && x >= T.seg[i].x0) s = i;
  const FitSeg& g = T.seg[s];
  const double f = (x - g.x0) * g.inv_h;
  int i = static_cast<int>(f);
  i = max(0, min(i, g.n - 1));
  t = 2.0 * (f - static_cast<double>(i)) - 1.0;
  return g.base + i;
}

// Interval layout (kFitStride doubles, 16-byte aligned): (mu_j, m2_j) pairs for j = 0..kFitDeg,
// then norm_0..norm_kFitDeg -- one 16-byte load per Horner step of the Newton pair.

// The degree-11 polynomials are evaluated as two independent Horner halves,
// sum_{j<6} c_j t^j + t^6 sum_{j<6} c_{j+6} t^j: half the dependent fp64 chain of one Horner pass.
constexpr int kFitHalf = kFitCoef / 2;

// mean and slope of ln X at x (estimate.py:76-83)
__device__ __forceinline__ void fit_mean_slope(const FitTable& T, double x, double& mean, double& slope) {
  double t;
  const double2* c = reinterpret_cast<const double2*>(T.coef + static_cast<int64_t>(fit_locate(T, x, t)) * kFitStride);
  const double2 top = __ldg(c + kFitDeg), mid = __ldg(c + kFitHalf - 1);
  double mu_h = top.x, m2_h = top.y, mu_l = mid.x, m2_l = mid.y;
#pragma unroll
  for (int j = kFitHalf - 2; j >= 0; --j) {
    const double2 ch = __ldg(c + kFitHalf + j), cl = __ldg(c + j);
    mu_h = fma(mu_h, t, ch.x);
    m2_h = fma(m2_h, t, ch.y);
    mu_l = fma(mu_l, t, cl.x);
    m2_l = fma(m2_l, t, cl.y);
  }
  const double t3 = t * t * t, t6 = t3 * t3;
  const double mu = fma(mu_h, t6, mu_l), m2 = fma(m2_h, t6, m2_l);
  mean = mu;
  slope = m2 - mu * mu;
}

// one polynomial with coefficients c[j * step], j = 0..kFitDeg
__device__ __forceinline__ double fit_poly(const double* c, int step, double t) {
  double h = __ldg(c + kFitDeg * step), l = __ldg(c + (kFitHalf - 1) * step);
#pragma unroll
  for (int j = kFitHalf - 2; j >= 0; --j) {
    h = fma(h, t, __ldg(c + (kFitHalf + j) * step));
    l = fma(l, t, __ldg(c + j * step));
  }
  const double t3 = t * t * t;
  return fma(h, t3 * t3, l);
}

__device__ __forceinline__ double fit_mean(const FitTable& T, double x) {
  double t;
  const double* c = T.coef + static_cast<int64_t>(fit_locate(T, x, t)) * kFitStride;
  return fit_poly(c, 2, t);
}

__device__ __forceinline__ double fit_norm(const FitTable& T, double x) {
  double t;
  const double* c = T.coef + static_cast<int64_t>(fit_locate(T, x, t)) * kFitStride + 2 * kFitCoef;
  return fit_poly(c, 1, t);
}

// Terms the reference sums for one model-moment evaluation at x (K, or the m rule of the
// segment: series.py:102-123) and for the normaliser (series.py:126-138): the reference
// algorithm's work, counted for the roofline (bench.py) when work counters are on.
__device__ __forceinline__ unsigned ref_moment_terms(const FitTable& T, double x) {
  if (T.K > 0) return static_cast<unsigned>(T.K);
  int s = 0;
  for (int i = 1; i < T.nseg; ++i)
    if (x >= T.seg[i].x0) s = i;
  return static_cast<unsigned>(T.seg[s].m_mom);
}
__device__ __forceinline__ unsigned ref_norm_terms(const FitTable& T, double x) {
  if (T.K > 0) return static_cast<unsigned>(T.K);
  int s = 0;
  for (int i = 1; i < T.nseg; ++i)
    if (x >= T.seg[i].x0) s = i;
  return static_cast<unsigned>(T.seg[s].m_norm);
}

// ---------------------------------------------------------------------------- building

// Neumaier-compensated accumulator
struct CSum {
  double s, c;
  __device__ __forceinline__ void add(double v) {
    const double t = s + v;
    c += (fabs(s) >= fabs(v)) ? (s - t) + v : (v - t) + s;
    s = t;
  }
  __device__ __forceinline__ double value() const { return s + c; }
};

__device__ __forceinline__ void two_sum_reduce(double& s, double& c) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double so = __shfl_xor_sync(0xffffffffu, s, o);
    const double co = __shfl_xor_sync(0xffffffffu, c, o);
    const double t = s + so;
    const double bp = t - s;
    const double err = (s - (t - bp)) + (so - bp);
    s = t;
    c = c + co + err;
  }
}

// compensated warp sums of k^-x (ln k)^p, p = 0..2, over k = lo..hi
__device__ void node_sums(double x, int lo, int hi, const double* __restrict__ logs, int lane, double out[3]) {
  CSum a{0, 0}, b{0, 0}, d{0, 0};
  for (int k = lo + lane; k <= hi; k += 32) {
    const double lk = logs[k];
    const double w = exp(-x * lk);
    a.add(w);
    b.add(w * lk);
    d.add(w * lk * lk);
  }
  double s0 = a.s, c0 = a.c, s1 = b.s, c1 = b.c, s2 = d.s, c2 = d.c;
  two_sum_reduce(s0, c0);
  two_sum_reduce(s1, c1);
  two_sum_reduce(s2, c2);
  out[0] = s0 + c0;
  out[1] = s1 + c1;
  out[2] = s2 + c2;
}

// One warp per interval: node values -> Chebyshev coefficients -> monomial coefficients in t.
__global__ void fit_table_kernel(FitTable T, double* coef, const double* __restrict__ logs) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T.intervals) return;
  int s = 0;
  for (int i = 1; i < T.nseg; ++i)
    if (warp >= T.seg[i].base) s = i;
  const FitSeg g = T.seg[s];
  const double a = g.x0 + static_cast<double>(warp - g.base) * g.h;
  double f[kFitFuncs][kFitCoef];
  for (int k = 0; k < kFitCoef; ++k) {
    const double tk = cos(M_PI * (k + 0.5) / kFitCoef);
    const double x = a + 0.5 * g.h * (1.0 + tk);
    double mom[3], nrm;
    if (T.K > 0) {
      node_sums(x, 1, T.K, logs, lane, mom);
      nrm = mom[0];
    } else {
      double lo[3], hi[3];
      node_sums(x, 1, 256, logs, lane, lo);
      node_sums(x, 257, 512, logs, lane, hi);
      for (int p = 0; p < 3; ++p) {
        double tv, e;
        em_tail(x, g.m_mom + 1, p, tv, e);
        mom[p] = (g.m_mom == 256 ? lo[p] : lo[p] + hi[p]) + tv;
      }
      double tv, e;
      em_tail(x, g.m_norm + 1, 0, tv, e);
      nrm = (g.m_norm == 256 ? lo[0] : lo[0] + hi[0]) + tv;
    }
    f[0][k] = mom[1] / mom[0];
    f[1][k] = mom[2] / mom[0];
    f[2][k] = nrm;
  }
  if (lane >= kFitFuncs) return;
  // Chebyshev coefficients of the interpolant through the nodes
  const double* v = f[lane];
  double cheb[kFitCoef];
  for (int j = 0; j < kFitCoef; ++j) {
    double acc = 0.0;
    for (int k = 0; k < kFitCoef; ++k) acc += v[k] * cos(M_PI * j * (k + 0.5) / kFitCoef);
    cheb[j] = acc * (2.0 / kFitCoef);
  }
  cheb[0] *= 0.5;
  // monomial coefficients: sum_j cheb[j] T_j(t), T_j by the three-term recurrence
  double mono[kFitCoef], tm2[kFitCoef], tm1[kFitCoef], tj[kFitCoef];
  for (int i = 0; i < kFitCoef; ++i) {
    mono[i] = 0.0;
    tm2[i] = 0.0;
    tm1[i] = 0.0;
  }
  tm2[0] = 1.0;  // T_0
  tm1[1] = 1.0;  // T_1
  mono[0] += cheb[0];
  mono[1] += cheb[1];
  for (int j = 2; j < kFitCoef; ++j) {
    for (int i = 0; i < kFitCoef; ++i) tj[i] = (i ? 2.0 * tm1[i - 1] : 0.0) - tm2[i];
    for (int i = 0; i < kFitCoef; ++i) {
      mono[i] += cheb[j] * tj[i];
      tm2[i] = tm1[i];
      tm1[i] = tj[i];
    }
  }
  double* out = coef + static_cast<int64_t>(warp) * kFitStride;
  for (int i = 0; i < kFitCoef; ++i) {
    if (lane < 2)
      out[2 * i + lane] = mono[i];  // mu / m2 pairs
    else
      out[2 * kFitCoef + i] = mono[i];  // norm
  }
}

// diagnostics: evaluate a table at arbitrary points
__global__ void fit_eval_kernel(FitTable T, const double* __restrict__ x, int64_t count, double* mu, double* m2,
                                double* norm) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double mean, slope;
    fit_mean_slope(T, x[i], mean, slope);
    mu[i] = mean;
    m2[i] = slope + mean * mean;
    norm[i] = fit_norm(T, x[i]);
  }
}

// Host-side layout of the table for support K (0 = unbounded).
inline FitTable fit_layout(int K) {
  FitTable T{};
  T.K = K;
  auto add = [&T](double x0, double x1, double h, int m_mom, int m_norm) {
    FitSeg& g = T.seg[T.nseg];
    g.x0 = x0;
    g.n = static_cast<int>((x1 - x0) / h + 0.999999);
    g.h = (x1 - x0) / g.n;
    g.inv_h = 1.0 / g.h;
    g.base = T.nseg ? T.seg[T.nseg - 1].base + T.seg[T.nseg - 1].n : 0;
    g.m_mom = m_mom;
    g.m_norm = m_norm;
    ++T.nseg;
  };
  if (K > 0) {
    add(-20.0, 20.0, 1.0 / 16, 0, 0);
  } else {
    add(kMinUnboundedGamma, kMomSwitchLo, 1.0 / 256, 256, 256);
    add(kMomSwitchLo, 1.25, 1.0 / 256, 512, 512);
    add(1.25, kValSwitchHi, 1.0 / 128, 512, 512);
    add(kValSwitchHi, kMomSwitchHi, 1.0 / 64, 512, 256);
    add(kMomSwitchHi, kMaxUnboundedGamma, 1.0 / 16, 256, 256);
  }
  T.intervals = T.seg[T.nseg - 1].base + T.seg[T.nseg - 1].n;
  return T;
}

}  // namespace zks
