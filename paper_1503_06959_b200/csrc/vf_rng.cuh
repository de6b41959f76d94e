// vf_rng.cuh -- the RANSAC minimal-sample stream of the reference, bit-exact,
// on host and device.
//
// ransac_homography (/root/reference/pkg/src/vidfeat/matching.py:170-174)
// draws `rng.choice(n, 4, replace=False)` once per iteration from
// `rng = np.random.default_rng(seed)`, i.e. numpy's Generator over
// PCG64(SeedSequence(seed)) (numpy 2.3, not vendored in /root/reference).
// Restated here from numpy's published algorithms:
//   * SeedSequence: the seed's 32-bit words are hash-mixed into a 4-word
//     pool; generate_state(4, uint64) draws 8 hashed words from the pool.
//   * PCG64: 128-bit LCG (multiplier 0x2360ED051FC65DA4_4385DF649FCCF645),
//     seeded as setseq(state = s[0]:s[1], inc = (s[2]:s[3]) << 1 | 1), output
//     XSL-RR (rotr64(hi ^ lo, hi >> 58)); 32-bit draws use the low half of a
//     64-bit output first and buffer the high half.
//   * choice(n, 4, replace=False) with n < 2^32: Floyd's sampling over
//     j = n-4 .. n-1 (draw in [0, j] with Lemire's method; a repeat is
//     replaced by j), then a Fisher-Yates pass i = 3, 2, 1 with Lemire draws
//     in [0, i].
// Every iteration therefore consumes D = 7 32-bit words (6 when n == 4: the
// j = 0 draw is free) unless a Lemire draw rejects (probability < n / 2^32
// per draw).  The device generator seeks each (problem, iteration) thread to
// word D * k by LCG jump-ahead and flags rejections; iterations after the
// first rejection are regenerated sequentially (vf_ransac.cu).
// Pinned against numpy itself by tests/test_ransac_host.py.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define VFR_HD __host__ __device__ __forceinline__
#else
#define VFR_HD inline
#endif

namespace vfr {

struct U128 {
  uint64_t hi, lo;
};

VFR_HD U128 mul(U128 a, U128 b)   // low 128 bits of a * b
{
#ifdef __CUDA_ARCH__
  const uint64_t lo = a.lo * b.lo, hi = __umul64hi(a.lo, b.lo);
#else
  const unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  const uint64_t lo = (uint64_t)p, hi = (uint64_t)(p >> 64);
#endif
  return {hi + a.hi * b.lo + a.lo * b.hi, lo};
}

VFR_HD U128 add(U128 a, U128 b)
{
  const uint64_t lo = a.lo + b.lo;
  return {a.hi + b.hi + (lo < a.lo ? 1u : 0u), lo};
}

VFR_HD U128 pcg_mult() { return {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}; }

// SeedSequence(seed).generate_state(4, np.uint64), for 0 <= seed < 2^64
VFR_HD void seed_words(uint64_t seed, uint64_t out[4])
{
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  const uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const int n_ent = (seed >> 32) ? 2 : 1;
  uint32_t hc = INIT_A;
  auto hashmix = [&hc, MULT_A](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [MIX_L, MIX_R](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; i++) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
  for (int a = 0; a < 4; a++)
    for (int b = 0; b < 4; b++)
      if (a != b) pool[b] = mix(pool[b], hashmix(pool[a]));
  uint32_t w[8], hb = INIT_B;
  for (int i = 0; i < 8; i++) {
    uint32_t d = pool[i & 3] ^ hb;
    hb *= MULT_B;
    d *= hb;
    w[i] = d ^ (d >> 16);
  }
  for (int i = 0; i < 4; i++) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

struct Pcg {
  U128 state, inc;
  uint32_t buf;
  bool has;
};

VFR_HD void step(Pcg& g) { g.state = add(mul(g.state, pcg_mult()), g.inc); }

VFR_HD Pcg pcg_seed(uint64_t seed)
{
  uint64_t s[4];
  seed_words(seed, s);
  Pcg g;
  g.inc = {(s[2] << 1) | (s[3] >> 63), (s[3] << 1) | 1u};
  g.state = {0, 0};
  step(g);
  g.state = add(g.state, U128{s[0], s[1]});
  step(g);
  g.has = false;
  g.buf = 0;
  return g;
}

// advance the LCG by `delta` steps in O(log delta) (Brown's jump-ahead)
VFR_HD void advance(Pcg& g, uint64_t delta)
{
  U128 am = {0, 1}, ap = {0, 0}, cm = pcg_mult(), cp = g.inc;
  while (delta) {
    if (delta & 1) {
      am = mul(am, cm);
      ap = add(mul(ap, cm), cp);
    }
    cp = mul(add(cm, U128{0, 1}), cp);
    cm = mul(cm, cm);
    delta >>= 1;
  }
  g.state = add(mul(am, g.state), ap);
}

VFR_HD uint64_t next64(Pcg& g)
{
  step(g);
  const unsigned rot = (unsigned)(g.state.hi >> 58);
  const uint64_t x = g.state.hi ^ g.state.lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

VFR_HD uint32_t next32(Pcg& g)
{
  if (g.has) {
    g.has = false;
    return g.buf;
  }
  const uint64_t v = next64(g);
  g.has = true;
  g.buf = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

// position the 32-bit stream of a freshly seeded generator at word u
VFR_HD void seek32(Pcg& g, uint64_t u)
{
  advance(g, u >> 1);
  if (u & 1) next32(g);
}

// uniform in [0, rng] by Lemire's method on 32-bit words; `rej` set if the
// draw needed more than one word
VFR_HD uint32_t lemire32(Pcg& g, uint32_t rng, bool& rej)
{
  const uint32_t ex = rng + 1u;
  uint64_t m = (uint64_t)next32(g) * ex;
  uint32_t left = (uint32_t)m;
  if (left < ex) {
    const uint32_t th = (0xffffffffu - rng) % ex;
    while (left < th) {
      rej = true;
      m = (uint64_t)next32(g) * ex;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// 32-bit words one rejection-free choice(n, 4, replace=False) consumes
VFR_HD int words_per_choice(int64_t n) { return n == 4 ? 6 : 7; }

// one rng.choice(n, 4, replace=False), n in [4, 2^31); returns true if any
// draw rejected (the iteration used more than words_per_choice words)
VFR_HD bool choice4(Pcg& g, uint32_t n, int32_t out[4])
{
  bool rej = false;
  uint32_t v[4];
  for (int k = 0; k < 4; k++) {
    const uint32_t j = n - 4u + (uint32_t)k;
    uint32_t x = j == 0 ? 0u : lemire32(g, j, rej);
    bool seen = false;
    for (int q = 0; q < k; q++) seen |= v[q] == x;
    v[k] = seen ? j : x;
  }
  for (int i = 3; i >= 1; i--) {
    const uint32_t k = lemire32(g, (uint32_t)i, rej);
    const uint32_t t = v[i];
    v[i] = v[k];
    v[k] = t;
  }
  for (int k = 0; k < 4; k++) out[k] = (int32_t)v[k];
  return rej;
}

}  // namespace vfr
