// numpy 2.x random core, restated for host AND device (bit-exact):
// SeedSequence (bit_generator.pyx: entropy + spawn-key hashing into a 4-word
// pool, generate_state), PCG64 (pcg64.c: 128-bit LCG, XSL-RR output, 32-bit
// halves buffered) and Lemire bounded integers (distributions.c
// random_bounded_uint64 / buffered_bounded_lemire_uint32).  Used by the host
// draw port (draws.cpp) and the device Monte-Carlo draws (mc.cu).
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define B2_HD __host__ __device__ __forceinline__
#else
#define B2_HD inline
#endif

namespace b2 {
namespace rng {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- SeedSequence
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16, POOL = 4;

B2_HD uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= MULT_A;
  value *= hc;
  value ^= value >> XSHIFT;
  return value;
}
B2_HD uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> XSHIFT;
  return r;
}
// _int_to_uint32_array: little-endian 32-bit words of a non-negative int
B2_HD int append_u32(uint32_t* out, int n, uint64_t v) {
  if (v == 0) {
    out[n++] = 0;
    return n;
  }
  while (v) {
    out[n++] = (uint32_t)(v & 0xffffffffu);
    v >>= 32;
  }
  return n;
}

struct SeedSeq {  // entropy: one uint64; spawn key: up to 8 uint64 words (no heap)
  uint32_t pool[POOL];
  B2_HD SeedSeq(uint64_t entropy, const uint64_t* key, int nkey) {
    uint32_t ent[2 + 2 * 8 + POOL];
    int n = append_u32(ent, 0, entropy);
    uint32_t spawn[16];
    int ns = 0;
    for (int i = 0; i < nkey && i < 8; ++i) ns = append_u32(spawn, ns, key[i]);
    if (ns > 0)
      while (n < POOL) ent[n++] = 0u;  // gh-16539 padding when a spawn key is present
    for (int i = 0; i < ns; ++i) ent[n++] = spawn[i];
    uint32_t hc = INIT_A;
    for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
    for (int s = 0; s < POOL; ++s)
      for (int d = 0; d < POOL; ++d)
        if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
    for (int s = POOL; s < n; ++s)
      for (int d = 0; d < POOL; ++d) pool[d] = mixw(pool[d], hashmix(ent[s], hc));
  }
  B2_HD void generate_u64(uint64_t* out, int n) const {  // generate_state(n, uint64), n <= 4
    uint32_t hc = INIT_B;
    uint32_t w[8];
    for (int i = 0; i < 2 * n; ++i) {
      uint32_t v = pool[i % POOL];
      v ^= hc;
      hc *= MULT_B;
      v *= hc;
      v ^= v >> XSHIFT;
      w[i] = v;
    }
    for (int i = 0; i < n; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  }
};

// ---------------------------------------------------------------- PCG64 (XSL-RR 128/64)
struct Pcg64 {
  u128 state, inc;
  int has_u32 = 0;
  uint32_t u32 = 0;
  static constexpr u128 MULT = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  B2_HD explicit Pcg64(uint64_t seed) : Pcg64(SeedSeq(seed, nullptr, 0)) {}  // default_rng(seed)
  B2_HD explicit Pcg64(const SeedSeq& ss) {  // default_rng(SeedSequence(...)): seeding.derive_rng
    uint64_t v[4];
    ss.generate_u64(v, 4);
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    state = 0;
    inc = (initseq << 1) | 1u;
    step();
    state += initstate;
    step();
  }
  B2_HD void step() { state = state * MULT + inc; }
  B2_HD uint64_t next64() {
    step();
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  B2_HD uint32_t next32() {
    if (has_u32) {
      has_u32 = 0;
      return u32;
    }
    const uint64_t n = next64();
    has_u32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)(n & 0xffffffffu);
  }
  // random_bounded_uint64(off=0, rng, mask=0, use_masked=false): Lemire
  B2_HD uint64_t bounded(uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xffffffffull) {
      if (rng == 0xffffffffull) return next32();
      const uint32_t excl = (uint32_t)rng + 1u;
      uint64_t m = (uint64_t)next32() * excl;
      uint32_t left = (uint32_t)m;
      if (left < excl) {
        const uint32_t thr = (uint32_t)((0xffffffffu - (uint32_t)rng) % excl);
        while (left < thr) {
          m = (uint64_t)next32() * excl;
          left = (uint32_t)m;
        }
      }
      return m >> 32;
    }
    if (rng == ~0ull) return next64();
    const uint64_t excl = rng + 1;
    u128 m = (u128)next64() * excl;
    uint64_t left = (uint64_t)m;
    if (left < excl) {
      const uint64_t thr = (~0ull - rng) % excl;
      while (left < thr) {
        m = (u128)next64() * excl;
        left = (uint64_t)m;
      }
    }
    return (uint64_t)(m >> 64);
  }
};

}  // namespace rng
}  // namespace b2
