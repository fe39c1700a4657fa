// Per-replicate random streams, bit-exact with the reference's numpy streams.
//
// Reference: RandomStream.for_replicate (pkg/src/zipfks/distribution.py:178-187) builds
//   Generator(Philox(SeedSequence([base_seed, repetition, index]))) and draws 1 - random(n).
// The arithmetic is numpy's (SeedSequence hash-mix -> generate_state(2, uint64) as the Philox
// key; Philox4x64-10 with the counter pre-incremented, so draw j is word j%4 of the block at
// counter [1 + j/4, 0, 0, 0]; random() = (x >> 11) * 2^-53).  Restated in oracle/rng.py and
// pinned against numpy by tests/test_oracle_rng.py.
#pragma once
#include <cstdint>

// Bounds checks of the debug build (python -m paper_1305_6738_b200._build --debug-bounds, i.e.
// -DZKS_DEBUG_BOUNDS): a violated index traps the kernel (the launch fails loudly); compiled out
// otherwise.  compute-sanitizer is closed on the GPU pool this engine was built on.
#ifdef ZKS_DEBUG_BOUNDS
#define ZKS_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define ZKS_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace zks {

constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t kPhiloxM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kPhiloxW1 = 0xBB67AE8584CAA73Bull;

struct Block4 {
  uint64_t w[4];
};

// Philox4x64-10 on counter (c0, 0, 0, 0).  20 64x64->128 multiplies per block: this is the
// INT-pipe cost that bounds large-n sampling.
__device__ __forceinline__ Block4 philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1) {
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kPhiloxW0;
      k1 += kPhiloxW1;
    }
    const uint64_t hi0 = __umul64hi(kPhiloxM0, x0), lo0 = kPhiloxM0 * x0;
    const uint64_t hi1 = __umul64hi(kPhiloxM1, x2), lo1 = kPhiloxM1 * x2;
    const uint64_t y0 = hi1 ^ x1 ^ k0;
    const uint64_t y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
  }
  Block4 b;
  b.w[0] = x0;
  b.w[1] = x1;
  b.w[2] = x2;
  b.w[3] = x3;
  return b;
}

// Opt-in fast stream (ZKS_RNG_PHILOX4X32, tier-3 parity only): Philox4x32-10
// (Salmon et al. 2011; the Random123 / curand constants) keyed by the low 64 bits of the same
// SeedSequence-derived key, the other 64 key bits in the counter's upper words.  Block b's four
// 64-bit words are the pairs of the 4x32 blocks at counters 2b and 2b + 1, so every consumer
// still takes x >> 11 as a 53-bit key.  32x32-bit multiplies instead of 64x64: about a quarter
// of the integer-pipe work of Philox4x64-10 per word.
constexpr uint32_t kPhilox32M0 = 0xD2511F53u, kPhilox32M1 = 0xCD9E8D57u;
constexpr uint32_t kPhilox32W0 = 0x9E3779B9u, kPhilox32W1 = 0xBB67AE85u;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kPhilox32W0;
      k1 += kPhilox32W1;
    }
    const uint32_t hi0 = __umulhi(kPhilox32M0, c.x), lo0 = kPhilox32M0 * c.x;
    const uint32_t hi1 = __umulhi(kPhilox32M1, c.z), lo1 = kPhilox32M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

enum : int { kRngNumpy = 0, kRngPhilox4x32 = 1 };

// Block c0 of a stream: numpy's Philox4x64-10 (bit-exact, the default) or the fast stream
__device__ __forceinline__ Block4 rng_block(uint64_t c0, uint64_t k0, uint64_t k1, int rng) {
  if (rng == kRngNumpy) return philox4x64_10(c0, k0, k1);
  const uint32_t ka = static_cast<uint32_t>(k0), kb = static_cast<uint32_t>(k0 >> 32);
  const uint32_t c_hi = static_cast<uint32_t>(c0 >> 31);
  const uint4 p = philox4x32_10(make_uint4(static_cast<uint32_t>(c0 << 1), c_hi, static_cast<uint32_t>(k1),
                                           static_cast<uint32_t>(k1 >> 32)), ka, kb);
  const uint4 q = philox4x32_10(make_uint4(static_cast<uint32_t>(c0 << 1) | 1u, c_hi, static_cast<uint32_t>(k1),
                                           static_cast<uint32_t>(k1 >> 32)), ka, kb);
  Block4 b;
  b.w[0] = (static_cast<uint64_t>(p.x) << 32) | q.x;
  b.w[1] = (static_cast<uint64_t>(p.y) << 32) | q.y;
  b.w[2] = (static_cast<uint64_t>(p.z) << 32) | q.z;
  b.w[3] = (static_cast<uint64_t>(p.w) << 32) | q.w;
  return b;
}

// u = 1 - (x >> 11) * 2^-53, exactly (the 53-bit integer converts exactly; 1 - m*2^-53 is
// representable for every m < 2^53).
__device__ __forceinline__ double uniform_open_closed(uint64_t x) {
  return 1.0 - static_cast<double>(x >> 11) * 0x1.0p-53;
}

// numpy SeedSequence constants (random/bit_generator.pyx)
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

struct HashState {
  uint32_t h;
  __device__ __forceinline__ uint32_t hashmix(uint32_t v) {
    v ^= h;
    h *= kMultA;
    v *= h;
    return v ^ (v >> 16);
  }
};

__device__ __forceinline__ uint32_t seq_mix(uint32_t x, uint32_t y) {
  const uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

// Entropy words of [seed, rep, idx]: each int split into little-endian uint32 words,
// 0 -> one zero word (numpy _coerce_to_uint32_array).  At most 6 words.
struct Entropy {
  uint32_t w[6];
  int n;
  // register-only append (select per slot; no dynamically indexed local memory)
  __device__ __forceinline__ void append(uint32_t v) {
#pragma unroll
    for (int i = 0; i < 6; ++i) w[i] = (i == n) ? v : w[i];
    ++n;
  }
  __device__ __forceinline__ void push(uint64_t v) {
    const uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
    append(lo);
    if (hi) append(hi);
  }
};

// The Philox key numpy derives from SeedSequence([seed, rep, idx]).
__device__ __forceinline__ void stream_key(uint64_t seed, uint64_t rep, uint64_t idx,
                                           uint64_t& k0, uint64_t& k1) {
  Entropy e;
  e.n = 0;
  e.push(seed);
  e.push(rep);
  e.push(idx);
  HashState hs{kInitA};
  uint32_t pool[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pool[i] = hs.hashmix(i < e.n ? e.w[i] : 0u);
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = seq_mix(pool[d], hs.hashmix(pool[s]));
#pragma unroll
  for (int s = 4; s < 6; ++s) {
    if (s < e.n) {
#pragma unroll
      for (int d = 0; d < 4; ++d) pool[d] = seq_mix(pool[d], hs.hashmix(e.w[s]));
    }
  }
  uint32_t hb = kInitB, st[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ hb;
    hb *= kMultB;
    v *= hb;
    st[i] = v ^ (v >> 16);
  }
  k0 = static_cast<uint64_t>(st[0]) | (static_cast<uint64_t>(st[1]) << 32);
  k1 = static_cast<uint64_t>(st[2]) | (static_cast<uint64_t>(st[3]) << 32);
}

}  // namespace zks
