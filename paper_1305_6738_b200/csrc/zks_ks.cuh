// KS statistic of one sample, warp-cooperative (gof.py:49-105).
//
// The reference scans F(k) - E(k) over every k = 1..kmax (gof.py:60-68), or, for an unbounded
// fit with kmax > 4096, only the stretch endpoints v and v-1 of the observed values v, with
// F from the cumulative table below the seam and an Euler-Maclaurin tail above it
// (gof.py:71-105).  Both give the same supremum (E is constant between observations while F
// rises, so each stretch attains its extremes at its ends).  Here:
//   * head, k <= kKsHead: dense, F(k) = S(k) / norm with S the running sum of k^-g, the
//     reference's cumulative form;
//   * k > kKsHead: endpoints only, S(v) = S(kKsHead) + EM(kKsHead+1 .. v) by Euler-Maclaurin
//     through the third-derivative term (the order of series.tail_mass, series.py:141-160),
//     S(v-1) = S(v) - v^-g.  Observed values are gathered tile by tile from the histogram
//     into a per-warp queue and scored 32 at a time, so the exp work scales with the number of
//     distinct values, not with kmax.
// The scan stops once no later k can beat the current maximum:
//   sup_{k' > k} |F(k') - E(k')| <= max(1 - E(k), 1 - F(k)).
// kArg also tracks the smallest k attaining the maximum (KsResult.argmax_k); exact mode forms
// E(k) = C(k) / n and the head F(k) as the running sum of (k^-g * (1/norm)), as the reference
// writes them, so trivial samples reproduce the reference's exact values (0, 2/3, ...).
#pragma once
#include <type_traits>
#include <cstdint>

#include "zks_series.cuh"

namespace zks {

constexpr uint32_t kKsHead = 64;
constexpr int kKsQueue = 64;         // per-warp endpoint queue entries
constexpr int kKsQueueWords = 3 * kKsQueue;
constexpr uint32_t kOverCap = 128;     // values above the histogram ordered in registers (<= kKsQueueWords)
constexpr double kKsMargin = 1e-11;  // early-exit safety margin (>> fp64 rounding of the sums)

// warp reductions of 32-bit integers: one REDUX instruction each (sm_80+)
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }

struct KsParams {
  int64_t n;
  uint32_t H;          // histogram bins held in `hist` (values 1..H)
  int hist_words;      // words of `hist` (>= max(H, P) + 1, multiple of 4)
  const double* logs;  // ln k, k = 0..65536
  bool exact;          // reference-exact forms (user-sample API)
  uint32_t P = 0;      // page bins for values above H when they are many (0 = H)
  double inv_n = 0.0;  // 1/n when the caller has it (0 = divide here)
  // continue from a head k = 1..kKsHead already scored lane by lane (ks_lane_head): its running
  // sum S(kKsHead), count C(kKsHead) and max gap; requires H == kKsHead and !kArg
  bool from_head = false;
  double S0 = 0.0, D0 = 0.0;
  uint32_t C0 = 0;
};

struct KsOut {
  double D;
  uint32_t argk;
  bool used_pages;
};

struct KsState {
  double S;       // running sum of k^-g through the last dense k
  double F;       // exact mode: running sum of k^-g / norm
  double S_head;  // S(min(kmax, kKsHead))
  double Dw;      // warp max of D as of the last flush (warp-uniform)
  uint32_t Cb;    // observations <= last processed k
  double D;       // lane-local running max gap
  uint32_t kb;    // lane-local smallest k attaining D (kArg)
  bool done;
  uint64_t next_fcheck;  // no F-based exit test before this k
};

struct KsCtx {
  double g, inv, inv_n, dn;
  double fa, a_pow, La;  // f(a) = a^-g, a^(1-g), ln a for a = kKsHead + 1
  double inv_om, g3, fa1, fa3;  // 1/(1-g), g(g+1)(g+2), f(a)/a, f(a)/a^3
  bool direct;                  // |1-g| large enough for the integral as (v f(v) - a f(a))/(1-g)
  bool exact;
  const double* logs;
  uint32_t* qk;  // queue: value v
  uint32_t* qc;  // queue: observations < v
  uint32_t* qn;  // queue: observations == v
};

__device__ __forceinline__ double ln_of(const double* logs, uint64_t v) {
  return v <= 65536u ? __ldg(logs + v) : log(static_cast<double>(v));
}

__device__ __forceinline__ double emp(const KsCtx& c, uint32_t C) {
  return c.exact ? static_cast<double>(C) / c.dn : static_cast<double>(C) * c.inv_n;
}

template <bool kArg>
__device__ __forceinline__ void take(KsState& s, double gap, uint32_t k) {
  if (kArg) {
    if (gap > s.D) {
      s.D = gap;
      s.kb = k;
    }
  } else {
    s.D = fmax(s.D, gap);
  }
}

// S(v) - S(kKsHead) = sum_{k=a}^{v} k^-g, a = kKsHead + 1, by Euler-Maclaurin; also returns v^-g
__device__ __forceinline__ double em_block(const KsCtx& c, uint64_t v, double& fv) {
  const double Lv = ln_of(c.logs, v);
  const double b = static_cast<double>(v);
  const double ib = 1.0 / b;
  fv = exp_bounded(-c.g * Lv);
  // integral_a^v x^-g dx = (v^(1-g) - a^(1-g)) / (1-g); near g = 1 that difference cancels, so
  // there it is a^(1-g) * expm1((1-g) ln(v/a)) / (1-g), continuous through g = 1
  double integral;
  if (c.direct)
    integral = (b * fv - c.a_pow) * c.inv_om;
  else
    integral = (c.g == 1.0) ? (Lv - c.La) : c.a_pow * expm1((1.0 - c.g) * (Lv - c.La)) * c.inv_om;
  const double d1 = -c.g * (fv * ib - c.fa1);               // f'(v) - f'(a)
  const double d3 = -c.g3 * (fv * (ib * ib * ib) - c.fa3);  // f'''(v) - f'''(a)
  return integral + 0.5 * (c.fa + fv) + d1 * (1.0 / 12.0) - d3 * (1.0 / 720.0);
}

// em_block's constants for the tail above the head at exponent g (c.logs set)
__device__ __forceinline__ void ks_tail_ctx(KsCtx& c, double g) {
  c.La = __ldg(c.logs + kKsHead + 1);
  c.fa = exp_bounded(-g * c.La);
  constexpr double a = static_cast<double>(kKsHead + 1);
  c.a_pow = a * c.fa;
  const double om = 1.0 - g;
  c.direct = fabs(om) >= 0.125;
  c.inv_om = om == 0.0 ? 0.0 : 1.0 / om;
  c.g3 = g * (g + 1.0) * (g + 2.0);
  c.fa1 = c.fa * (1.0 / a);
  c.fa3 = c.fa * (1.0 / (a * a * a));
}

struct FlushTail {
  double F_last;    // fitted cdf at the last scored value
  uint32_t C_last;  // observations <= the last scored value
};

// score queue entries [0, cnt) lane-parallel (cnt <= 32)
template <bool kArg>
__device__ __forceinline__ FlushTail ks_flush(KsState& s, const KsCtx& c, int cnt, int lane, Work& wk) {
  FlushTail ft{0.0, 0u};
  if (cnt <= 0) return ft;
  double Fv = 0.0;
  uint32_t Ca = 0;
  if (lane < cnt) {
    const uint32_t v = c.qk[lane];
    const uint32_t before = c.qc[lane];
    const uint32_t here = c.qn[lane];
    double fv;
    const double Sv = s.S_head + em_block(c, v, fv);
    Fv = Sv * c.inv;
    Ca = before + here;
    const double Fp = (Sv - fv) * c.inv;
    take<kArg>(s, fabs(Fp - emp(c, before)), v - 1);  // k = v - 1 first (smaller k wins ties)
    take<kArg>(s, fabs(Fv - emp(c, Ca)), v);
  }
  wk.ks_tails += cnt;
  ft.F_last = __shfl_sync(0xffffffffu, Fv, cnt - 1);
  ft.C_last = __shfl_sync(0xffffffffu, Ca, cnt - 1);
  return ft;
}

// Tiles of 32 consecutive k in [k_first, k_last] with counts[k - base], above the head.
template <bool kArg>
__device__ __forceinline__ void ks_sparse_tiles(KsState& s, const KsCtx& c, int& q, uint64_t k_first, uint64_t k_last,
                                                const uint32_t* counts, uint64_t base, int lane, Work& wk) {
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t k0 = k_first; k0 <= k_last && !s.done; k0 += 32) {
    ++wk.ks_tiles;
    const uint64_t k = k0 + lane;
    const bool in = k <= k_last;
    const uint32_t cnt = in ? counts[k - base] : 0u;
    const uint32_t C = s.Cb + warp_scan_u32(cnt, lane);
    const unsigned nz = __ballot_sync(0xffffffffu, cnt != 0u);
    if (cnt) {
      const int slot = q + __popc(nz & lt);
      c.qk[slot] = static_cast<uint32_t>(k);
      c.qc[slot] = C - cnt;
      c.qn[slot] = cnt;
    }
    q += __popc(nz);
    s.Cb = __shfl_sync(0xffffffffu, C, 31);
    __syncwarp();
    if (q >= 32) {
      ks_flush<kArg>(s, c, 32, lane, wk);
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
      s.Dw = warp_max_nonneg(s.D);
    }
    // exit test, only once the empirical part of the bound allows it (D changes only at
    // flushes); F-based tests back off geometrically in k (heavy tails approach 1 slowly)
    const uint64_t k_hi = k0 + 31u < k_last ? k0 + 31u : k_last;
    if (k_hi >= s.next_fcheck && s.Dw > 1.0 - emp(c, s.Cb) + kKsMargin) {
      ks_flush<kArg>(s, c, q, lane, wk);
      q = 0;
      __syncwarp();
      s.Dw = warp_max_nonneg(s.D);
      double fk;
      const double F_pos = (s.S_head + em_block(c, k_hi, fk)) * c.inv;
      ++wk.ks_tails;
      if (s.Dw > fmax(1.0 - emp(c, s.Cb), 1.0 - F_pos) + kKsMargin)
        s.done = true;
      else
        s.next_fcheck = 2 * k_hi - kKsHead;
    }
  }
}

// Ascending bitonic sort of 32 * kSl values held as r[slot] (element slot * 32 + lane), fully
// unrolled: shuffles within a slot, register exchanges across slots.
template <int kSl>
__device__ __forceinline__ void bitonic_sort_warp(uint32_t (&r)[kOverCap / 32], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * kSl; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
#pragma unroll
      for (int sl = 0; sl < kSl; ++sl) {
        const int i = sl * 32 + lane;
        const bool up = (i & k) == 0;
        if (jj >= 32) {
          const int ps = sl ^ (jj >> 5);
          if (ps > sl) {
            const uint32_t a0 = r[sl], a1 = r[ps];
            const bool sw = up ? a0 > a1 : a0 < a1;
            r[sl] = sw ? a1 : a0;
            r[ps] = sw ? a0 : a1;
          }
        } else {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, r[sl], jj);
          const bool low = (lane & jj) == 0;
          r[sl] = (low == up) ? min(r[sl], o) : max(r[sl], o);
        }
      }
    }
  }
}

// KS of one sample with counts of 1..H in `hist`; values above H are found in
// over_vals[0..over_n) (which may also hold values <= H: they are ignored).  `queue` is
// kKsQueueWords u32 of per-warp shared memory.  `hist` is left dirty (see used_pages).
// kCompact: over_vals is the caller's scratch (hence non-const); each page pass keeps only the
// values above its page (compacted in place), so later passes read the remaining tail instead of
// all of it, and the caller's list is consumed.
template <typename VT, bool kArg, bool kCompact = false>
__device__ KsOut ks_scan(const KsParams& p, double g, double norm, uint64_t kmax, uint32_t* hist,
                         typename std::conditional<kCompact, VT*, const VT*>::type over_vals, uint32_t over_n,
                         uint32_t* queue, int lane, Work& wk) {
  KsCtx c;
  c.g = g;
  c.inv = 1.0 / norm;
  c.dn = static_cast<double>(p.n);
  c.inv_n = p.inv_n > 0.0 ? p.inv_n : 1.0 / c.dn;
  c.exact = p.exact;
  c.logs = p.logs;
  c.qk = queue;
  c.qc = queue + kKsQueue;
  c.qn = queue + 2 * kKsQueue;
  const uint64_t H = p.H;
  const uint64_t P = p.P ? p.P : p.H;
  KsState s{};
  s.kb = 0xffffffffu;
  KsOut out{0.0, 0u, false};

  // head: dense, the reference's cumulative form
  const uint32_t head_end = static_cast<uint32_t>(kmax < kKsHead ? kmax : kKsHead);
  if (p.from_head) {
    s.S = p.S0;
    s.Cb = p.C0;
    s.D = p.D0;
  }
  for (uint32_t k0 = 1; k0 <= head_end && !s.done && !p.from_head; k0 += 32) {
    ++wk.ks_tiles;
    const uint32_t k = k0 + lane;
    const bool in = k <= head_end;
    const uint32_t cnt = in ? hist[k] : 0u;
    const uint32_t C = s.Cb + warp_scan_u32(cnt, lane);
    const double term = in ? exp_bounded(-g * __ldg(p.logs + k)) : 0.0;
    const double S = s.S + warp_scan(term, lane);
    double F;
    if (c.exact) {
      F = s.F + warp_scan(term * c.inv, lane);
      s.F = __shfl_sync(0xffffffffu, F, 31);
    } else {
      F = S * c.inv;
    }
    if (in) take<kArg>(s, fabs(F - emp(c, C)), k);
    s.S = __shfl_sync(0xffffffffu, S, 31);
    s.Cb = __shfl_sync(0xffffffffu, C, 31);
    wk.ks_terms += min(32u, head_end - k0 + 1);
    const double Dw = warp_max_nonneg(s.D);
    if (Dw > fmax(1.0 - emp(c, s.Cb), 1.0 - s.S * c.inv) + kKsMargin) s.done = true;
  }
  if (!s.done && kmax > kKsHead) {
    s.S_head = s.S;
    s.Dw = p.from_head ? p.D0 : warp_max_nonneg(s.D);  // from_head: D0 is the warp's value
    ks_tail_ctx(c, g);

    // above the head: endpoints of the observed values
    int q = 0;
    ks_sparse_tiles<kArg>(s, c, q, kKsHead + 1, kmax < H ? kmax : H, hist, 0u, lane, wk);
    // Values above `above` (all of over_vals' values above it) in increasing order: with at most
    // kOverCap of them, sorted in registers and scored run by run (no pages).  Returns false
    // (nothing consumed) when there are more.  Used first above H and, on compacting scans,
    // again whenever a page pass leaves few values above its page.
    auto reg_tail = [&](uint64_t above) -> bool {
      if (q) {
        ks_flush<kArg>(s, c, q, lane, wk);  // the emptied queue stages the values
        q = 0;
        __syncwarp();
        s.Dw = warp_max_nonneg(s.D);
      }
      const unsigned lt = (1u << lane) - 1u;
      uint32_t m = 0;
      for (uint32_t i0 = 0; i0 < over_n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint64_t v = i < over_n ? static_cast<uint64_t>(over_vals[i]) : 0ull;
        const bool big = v > above;
        const unsigned b = __ballot_sync(0xffffffffu, big);
        const uint32_t slot = m + __popc(b & lt);
        if (big && slot < kOverCap) queue[slot] = static_cast<uint32_t>(v);
        m += __popc(b);
      }
      __syncwarp();
      if (m > kOverCap) return false;
      {
        constexpr int kSlots = kOverCap / 32;
        const int size = m <= 32u ? 32 : m <= 64u ? 64 : 128;  // sort only the occupied slots
        uint32_t r[kSlots];  // element i = slot * 32 + lane
#pragma unroll
        for (int j = 0; j < kSlots; ++j) {
          const uint32_t idx = j * 32 + lane;
          r[j] = idx < m ? queue[idx] : 0xffffffffu;
        }
        __syncwarp();
        // bitonic sort of the occupied slots across the warp (padding 0xffffffff sorts last)
        if (size == 32)
          bitonic_sort_warp<1>(r, lane);
        else if (size == 64)
          bitonic_sort_warp<2>(r, lane);
        else
          bitonic_sort_warp<4>(r, lane);
        // runs of equal values: each run's last element becomes an endpoint entry
        const unsigned lt = (1u << lane) - 1u;
        int ne = 0;
        uint32_t run_start = 0;  // prefix max of start indices, carried across slots
        for (int sl = 0; sl < kSlots && sl * 32 < size && !s.done; ++sl) {
          const uint32_t v = r[sl];
          const uint32_t i = sl * 32 + lane;
          uint32_t prev = __shfl_up_sync(0xffffffffu, v, 1);
          const uint32_t last_prev = sl ? __shfl_sync(0xffffffffu, r[sl > 0 ? sl - 1 : 0], 31) : 0u;
          if (lane == 0) prev = sl ? last_prev : 0u;
          uint32_t next = __shfl_down_sync(0xffffffffu, v, 1);
          const uint32_t first_next = sl + 1 < kSlots ? __shfl_sync(0xffffffffu, r[sl + 1 < kSlots ? sl + 1 : sl], 0)
                                                      : 0xffffffffu;
          if (lane == 31) next = first_next;
          const bool start = (i == 0) || v != prev;
          uint32_t st_idx = start ? i : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, st_idx, o);
            if (lane >= o) st_idx = max(st_idx, t);
          }
          st_idx = max(st_idx, run_start);
          run_start = __shfl_sync(0xffffffffu, st_idx, 31);
          const bool end = v != 0xffffffffu && v != next;
          const unsigned em = __ballot_sync(0xffffffffu, end);
          if (end) {
            const int slot = ne + __popc(em & lt);
            c.qk[slot] = v;
            c.qc[slot] = s.Cb + st_idx;
            c.qn[slot] = i - st_idx + 1;
          }
          ne += __popc(em);
          __syncwarp();
          if (ne >= 32) {
            const FlushTail fl = ks_flush<kArg>(s, c, 32, lane, wk);
            __syncwarp();
            uint32_t a0 = 0, a1 = 0, a2 = 0;
            if (lane < ne - 32) {
              a0 = c.qk[32 + lane];
              a1 = c.qc[32 + lane];
              a2 = c.qn[32 + lane];
            }
            __syncwarp();
            if (lane < ne - 32) {
              c.qk[lane] = a0;
              c.qc[lane] = a1;
              c.qn[lane] = a2;
            }
            ne -= 32;
            __syncwarp();
            s.Dw = warp_max_nonneg(s.D);
            // observations <= the last scored value, and F there, bound every later gap
            if (s.Dw > fmax(1.0 - emp(c, fl.C_last), 1.0 - fl.F_last) + kKsMargin) s.done = true;
          }
        }
        __syncwarp();
        ks_flush<kArg>(s, c, ne, lane, wk);
        s.Cb += m;
      }
      return true;
    };
    bool paged = !s.done && kmax > H;
    if (paged && reg_tail(H)) paged = false;
    uint64_t pa = H + 1;
    while (paged && !s.done && pa <= kmax) {
      out.used_pages = true;
      const uint64_t pb = pa + P - 1 < kmax ? pa + P - 1 : kmax;
      // page histogram of the values in [pa, pb]; next occupied value above pb
      for (int i = lane; i < p.hist_words; i += 32) hist[i] = 0u;
      __syncwarp();
      uint64_t next = ~0ull;
      if constexpr (kCompact) {
        const unsigned lt = (1u << lane) - 1u;
        VT* keep_out = over_vals;
        uint32_t kept = 0;
        for (uint32_t i0 = 0; i0 < over_n; i0 += 32) {
          const uint32_t i = i0 + lane;
          const uint64_t v = i < over_n ? static_cast<uint64_t>(over_vals[i]) : 0ull;
          if (v >= pa && v <= pb) atomicAdd(hist + (v - pa), 1u);
          const bool keep = v > pb;
          if (keep) next = v < next ? v : next;
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          if (keep) keep_out[kept + __popc(km & lt)] = static_cast<VT>(v);  // slot <= i: read already
          kept += __popc(km);
        }
        over_n = kept;
      } else {
        for (uint32_t i = lane; i < over_n; i += 32) {
          const uint64_t v = static_cast<uint64_t>(over_vals[i]);
          if (v >= pa && v <= pb)
            atomicAdd(hist + (v - pa), 1u);
          else if (v > pb)
            next = v < next ? v : next;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(0xffffffffu, next, o);
        next = t < next ? t : next;
      }
      __syncwarp();
      ks_sparse_tiles<kArg>(s, c, q, pa, pb, hist, pa, lane, wk);
      pa = pb + 1;
      if (next != ~0ull && next > pa) pa = next;  // no observations in between: no endpoints
      // compacted: the values left are exactly those above pb -- once few, one register pass
      // scores them all instead of a page pass per sparse cluster
      if (kCompact && !s.done && over_n <= kOverCap && reg_tail(pb)) break;
    }
    ks_flush<kArg>(s, c, q, lane, wk);
  }
  // warp result: max gap, smallest k among equal maxima
  if (!kArg) {
    out.D = warp_max_nonneg(s.D);
    return out;
  }
  double D = s.D;
  uint32_t kb = s.kb;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double Do = __shfl_xor_sync(0xffffffffu, D, o);
    const uint32_t ko = __shfl_xor_sync(0xffffffffu, kb, o);
    if (Do > D || (Do == D && ko < kb)) {
      D = Do;
      kb = ko;
    }
  }
  out.D = D;
  out.argk = kb;
  return out;
}

__device__ __forceinline__ void clear_hist(uint32_t* hist, int words, int lane) {
  uint4* h4 = reinterpret_cast<uint4*>(hist);
  for (int i = lane; i < words / 4; i += 32) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
}

}  // namespace zks
