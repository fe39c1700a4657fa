// Fitting and scoring user samples: log_mean, mle_gamma and
// ks_statistic (estimate.py:59-146, gof.py:49-105) for a batch of samples given as one flat
// int64 array plus offsets, one warp per sample; plus the series / solver entry points behind
// the reference's scalar helpers (series.py:68-138, estimate.py:94-112).
#pragma once
#include <cstdint>

#include "zks_replicate.cuh"

namespace zks {

constexpr int kFitExponent = 1;  // ZKS_FIT_EXPONENT
constexpr int kFitKs = 2;        // ZKS_FIT_KS
constexpr int kSamplesHist = 2048;

constexpr uint8_t kStatusNoRoot = 2;
constexpr uint8_t kStatusOutside = 3;
constexpr uint8_t kStatusEmpty = 4;

struct SamplesArgs {
  const int64_t* values;
  const int64_t* offsets;  // nsamples + 1
  int64_t nsamples;
  int K;
  const double* logs;
  FitTable fit;
  int use_table;
  MleParams mle;
  int mode;
  const double* gamma_in;  // exponent to score against when the fit is not requested
  const double* norm_in;   // its normaliser (NULL: computed by direct summation)
  double* log_mean_out;
  double* gamma_out;
  double* ks_out;
  int64_t* argmax_out;
  uint8_t* status_out;
  int hist_words;
  unsigned long long* work;
};

__global__ void __launch_bounds__(kThreads) samples_kernel(SamplesArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem) + warp * (a.hist_words + kKsQueueWords);
  uint32_t* queue = hist + a.hist_words;
  clear_hist(hist, a.hist_words, lane);
  const int K = a.K;
  const ModelFns M{K, a.logs, a.fit, a.use_table != 0};
  Work wk{};
  for (;;) {
    unsigned long long sidx = 0;
    if (lane == 0) sidx = atomicAdd(a.work, 1ull);
    sidx = __shfl_sync(0xffffffffu, sidx, 0);
    if (sidx >= static_cast<unsigned long long>(a.nsamples)) break;
    const int64_t off = a.offsets[sidx];
    const int64_t n = a.offsets[sidx + 1] - off;
    const int64_t* v = a.values + off;
    double lm = 0.0, g = 0.0, ks = __longlong_as_double(0x7ff8000000000000ll);
    int64_t argk = 0;
    uint8_t status = 0;
    if (n <= 0) {
      status = kStatusEmpty;
    } else {
      // log-sum (estimate.py:59-73), range (distribution.py:61-65)
      double ls = 0.0;
      uint64_t vmin = ~0ull, vmax = 0;
      bool bad = false;
      for (int64_t i = lane; i < n; i += 32) {
        const int64_t x = v[i];
        if (x < 1 || x > 0xffffffffll || (K > 0 && x > K)) {
          bad = true;
          continue;
        }
        const uint64_t ux = static_cast<uint64_t>(x);
        ls += ln_of(a.logs, ux);
        vmin = ux < vmin ? ux : vmin;
        vmax = ux > vmax ? ux : vmax;
      }
      bad = __any_sync(0xffffffffu, bad);
      ls = warp_sum(ls);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t t0 = __shfl_xor_sync(0xffffffffu, vmin, o);
        const uint64_t t1 = __shfl_xor_sync(0xffffffffu, vmax, o);
        vmin = t0 < vmin ? t0 : vmin;
        vmax = t1 > vmax ? t1 : vmax;
      }
      const double dn = static_cast<double>(n);
      if (bad) {
        status = kStatusOutside;
      } else {
        lm = (ls <= 0.0 ? ls + kLn2 : ls) / dn;
        bool ok = true;
        if (a.mode & kFitExponent) {
          double target = lm;
          if (K > 0 && vmin == static_cast<uint64_t>(K))
            target -= (log(static_cast<double>(K)) - log(static_cast<double>(K - 1))) / dn;
          ok = fit_exponent(M, target, lane, g, wk, a.mle);
          if (!ok) status = kStatusNoRoot;
        } else if (a.gamma_in) {
          g = a.gamma_in[sidx];
        }
        if (ok && (a.mode & kFitKs)) {
          const double norm = a.norm_in ? a.norm_in[sidx] : normaliser(g, K, a.logs, lane, wk);
          const uint32_t H = static_cast<uint32_t>(a.hist_words - 4);
          uint32_t c1 = 0, c2 = 0;
          for (int64_t i = lane; i < n; i += 32) {
            const uint64_t x = static_cast<uint64_t>(v[i]);
            c1 += x == 1u;
            c2 += x == 2u;
            if (x > 2u && x <= H) atomicAdd(hist + x, 1u);
          }
          c1 = warp_sum_u32(c1);
          c2 = warp_sum_u32(c2);
          if (lane == 0) {
            hist[1] += c1;
            hist[2] += c2;
          }
          __syncwarp();
          KsParams p;
          p.n = n;
          p.H = H;
          p.hist_words = a.hist_words;
          p.logs = a.logs;
          p.exact = true;
          const KsOut r = ks_scan<int64_t, true>(p, g, norm, vmax, hist, v, static_cast<uint32_t>(n), queue, lane, wk);
          ks = r.D;
          argk = r.argk;
          clear_hist(hist, a.hist_words, lane);
        }
      }
    }
    if (lane == 0) {
      a.log_mean_out[sidx] = lm;
      a.gamma_out[sidx] = g;
      a.ks_out[sidx] = ks;
      a.argmax_out[sidx] = argk;
      a.status_out[sidx] = status;
    }
  }
}

// Model moments by the reference formulas (direct sums, m-doubling rule): out[4*i..] =
// (s0, s1, s2, normaliser) at gamma[i].  One warp per exponent.
// tail_mass (series.py:141-160): sum_{k >= start_i} k^-g, Euler-Maclaurin through the third
// derivative, vectorised over start
__global__ void tail_mass_kernel(double g, const double* __restrict__ start, int64_t count, double* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = tail_sum(g, log(start[i]));
}

__global__ void series_kernel(const double* __restrict__ gamma, int64_t count, int K, const double* logs,
                              double* out) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  Work wk{};
  Moments m{0.0, 0.0, 0.0};
  const double g = gamma[w];
  const bool ok = (K > 0 || g > 1.0) ? log_moments(g, K, logs, lane, m, wk) : false;
  const double nrm = (K > 0 || g > 1.0) ? normaliser(g, K, logs, lane, wk) : __longlong_as_double(0x7ff8000000000000ll);
  if (lane == 0) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    out[4 * w + 0] = ok ? m.s0 : nan;
    out[4 * w + 1] = ok ? m.s1 : nan;
    out[4 * w + 2] = ok ? m.s2 : nan;
    out[4 * w + 3] = nrm;
  }
}

// Newton / bisection on given targets (mean log of data): mle_gamma without the sample, and
// _bisect (estimate.py:94-112) when bisect_only.  One warp per target (direct sums: settings
// may reach outside the fit tables).
__global__ void solve_kernel(const double* __restrict__ target, int64_t count, int K, const double* logs,
                             MleParams P, int bisect_only, double* gamma, uint8_t* status) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  Work wk{};
  FitTable none{};
  const ModelFns M{K, logs, none, false};
  double g = 0.0;
  bool ok;
  if (bisect_only) {
    ok = bisect_root(M, target[w], lane, P.lo, P.hi, g, wk);
  } else {
    ok = fit_exponent(M, target[w], lane, g, wk, P);
  }
  if (lane == 0) {
    gamma[w] = ok ? g : __longlong_as_double(0x7ff8000000000000ll);
    status[w] = ok ? 0 : kStatusNoRoot;
  }
}

}  // namespace zks
