// Device random streams keyed by (seed, round, particle, step, substep).
//
//  * XoStream    -- the reference's keyed xoshiro256++ (include/asmc/rng.hpp:27-86):
//                   identical 64-bit words, 53-bit uniforms, double Box-Muller with
//                   the cached sine.  Sequential by construction (one lane per particle).
//  * PhiloxKey   -- counter-based Philox4x32-10 with the indexing of
//                   oracle/shadow/asmc/rng.hpp: normal #j lives in block j>>2, so any
//                   lane can draw any coordinate's normal -- 32 lanes share a particle.
//  * PhSeq       -- sequential view of a Philox stream (one lane per particle).
#pragma once

#include <stdint.h>

namespace asmcdev {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

// ---------------------------------------------------------------- xoshiro --
struct XoStream {
  uint64_t s0, s1, s2, s3;
  double cached;
  bool have;

  // rng.hpp:43-55
  __device__ __forceinline__ void init(uint64_t seed, uint64_t round, uint64_t particle,
                                       uint64_t step, uint64_t substep) {
    uint64_t acc = mix64(seed + 0x9E3779B97F4A7C15ULL);
    acc = mix64(acc ^ (round + 0xD1B54A32D192ED03ULL));
    acc = mix64(acc ^ (particle + 0x8CB92BA72F3D8DD7ULL));
    acc = mix64(acc ^ (step + 0xA24BAED4963EE407ULL));
    acc = mix64(acc ^ (substep + 0x9FB21C651E98DF25ULL));
    acc += 0x9E3779B97F4A7C15ULL;
    s0 = mix64(acc);
    acc += 0x9E3779B97F4A7C15ULL;
    s1 = mix64(acc);
    acc += 0x9E3779B97F4A7C15ULL;
    s2 = mix64(acc);
    acc += 0x9E3779B97F4A7C15ULL;
    s3 = mix64(acc);
    if ((s0 | s1 | s2 | s3) == 0) s0 = 1;
    have = false;
    cached = 0.0;
  }
  // rng.hpp:57-68
  __device__ __forceinline__ uint64_t next_u64() {
    const uint64_t result = rotl64(s0 + s3, 23) + s0;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = rotl64(s3, 45);
    return result;
  }
  __device__ __forceinline__ double uniform() {  // rng.hpp:71
    return (double)(next_u64() >> 11) * 0x1.0p-53;
  }
  // rng.hpp:73-86 in double; Real selects the precision the sampler consumes.
  __device__ __forceinline__ double normal() {
    if (have) {
      have = false;
      return cached;
    }
    double u1 = uniform();
    while (u1 == 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586477 * u2;
    double sa, ca;
    sincos(a, &sa, &ca);  // one argument reduction for both (the same bits as sin and cos)
    cached = r * sa;
    have = true;
    return r * ca;
  }
};

// ----------------------------------------------------------------- philox --
// 32x32 -> 64 multiply as one IMAD.WIDE.U32; hi/lo are the register pair halves.
__device__ __forceinline__ void mulwide(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mulwide(0xD2511F53u, c.x, lo0, hi0);
    mulwide(0xCD9E8D57u, c.z, lo1, hi1);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// MUFU (SFU) approximations, ftz: inputs here are never denormal.
__device__ __forceinline__ float mufu_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_sin(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float mufu_cos(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller pair in fp32 from two 32-bit words -- the shadow stream's
// u1 = (a+1) 2^-32, u2 = b 2^-32, r = sqrt(-2 ln u1), angle 2 pi u2
// (oracle/shadow/asmc/rng.hpp) -- on the SFU: 4 MUFU ops + ~20 ALU per pair.
//  * -ln u1: for u1 <= 31/32, -ln2 * lg2(u1) (|log2 u1| >= 0.046, so the SFU's
//    ~2^-22 absolute error is <= 6e-6 relative); for u1 > 31/32 the SFU loses
//    relative accuracy, so t = 1 - u1 = (~a) 2^-32 (exact word arithmetic) and
//    -ln(1 - t) = t (1 + t/2 + t^2/3 + t^3/4 + t^4/5) (truncation < t^5/6 < 2^-27);
//  * the angle as a signed word: (int)b 2^-32 * 2 pi = 2 pi u2 - 2 pi [b >= 2^31]
//    lies in [-pi, pi), the SFU's accurate range (2^-20.5 absolute), with the
//    same sine and cosine.
// Normals agree with the fp64 transform to ~1e-6 absolute (tests/test_gpu_parity.py).
__device__ __forceinline__ void bm_pair_f32(uint32_t a, uint32_t b, float& n_cos, float& n_sin) {
  const float u1 = fmaf(__uint2float_rn(a), 0x1.0p-32f, 0x1.0p-32f);
  const float v_log = -0.693147180559945309f * mufu_lg2(u1);
  const float t = __uint2float_rn(~a) * 0x1.0p-32f;
  float q = fmaf(t, 0.2f, 0.25f);
  q = fmaf(t, q, 0.333333343f);
  q = fmaf(t, q, 0.5f);
  q = fmaf(t, q, 1.0f);
  const float v = t < 0.03125f ? t * q : v_log;  // -ln u1
  const float r = mufu_sqrt(v + v);
  const float ang = __int2float_rn((int)b) * 1.46291807926715968e-09f;  // 2 pi 2^-32
  n_cos = r * mufu_cos(ang);
  n_sin = r * mufu_sin(ang);
}

__device__ __forceinline__ void bm_pair_f64(uint32_t a, uint32_t b, double& n_cos, double& n_sin) {
  const double u1 = ((double)a + 1.0) * 0x1.0p-32;
  const double u2 = (double)b * 0x1.0p-32;
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 6.283185307179586477 * u2;
  double sa, ca;
  sincos(ang, &sa, &ca);
  n_cos = r * ca;
  n_sin = r * sa;
}

template <typename Real>
__device__ __forceinline__ void bm_pair(uint32_t a, uint32_t b, Real& c, Real& s);
template <>
__device__ __forceinline__ void bm_pair<float>(uint32_t a, uint32_t b, float& c, float& s) {
  bm_pair_f32(a, b, c, s);
}
template <>
__device__ __forceinline__ void bm_pair<double>(uint32_t a, uint32_t b, double& c, double& s) {
  bm_pair_f64(a, b, c, s);
}

// the Philox key of (seed, round, substep): the same for every particle and step
__host__ __device__ __forceinline__ void philox_key(uint64_t seed, uint64_t round, uint64_t substep,
                                                    uint32_t& k0, uint32_t& k1) {
  uint64_t acc = mix64(seed + 0x9E3779B97F4A7C15ULL);
  acc = mix64(acc ^ (round + 0xD1B54A32D192ED03ULL));
  acc = mix64(acc ^ (substep + 0x9FB21C651E98DF25ULL));
  k0 = (uint32_t)acc;
  k1 = (uint32_t)(acc >> 32);
}

struct PhiloxKey {
  uint32_t k0, k1, c1, c2, c3;

  __device__ __forceinline__ void init(uint64_t seed, uint64_t round, uint64_t particle,
                                       uint64_t step, uint64_t substep) {
    philox_key(seed, round, substep, k0, k1);
    c1 = (uint32_t)step;
    c2 = (uint32_t)particle;
    c3 = (uint32_t)(particle >> 32) ^ ((uint32_t)(step >> 32) * 0x9E3779B9u);
  }
  __device__ __forceinline__ uint4 block(uint32_t b) const {
    return philox10(make_uint4(b, c1, c2, c3), k0, k1);
  }
  __device__ __forceinline__ uint64_t u64(uint32_t k) const {
    const uint4 w = philox10(make_uint4(0x80000000u | k, c1, c2, c3), k0, k1);
    return ((uint64_t)w.x << 32) | w.y;
  }
  __device__ __forceinline__ double uniform(uint32_t k) const {
    return (double)(u64(k) >> 11) * 0x1.0p-53;
  }
  // the four normals 4b .. 4b+3
  template <typename Real>
  __device__ __forceinline__ void normals4(uint32_t b, Real out[4]) const {
    const uint4 w = block(b);
    bm_pair<Real>(w.x, w.y, out[0], out[1]);
    bm_pair<Real>(w.z, w.w, out[2], out[3]);
  }
  // normals j0 .. j0+3 for an arbitrary (possibly unaligned) j0
  template <typename Real>
  __device__ __forceinline__ void normals4_at(uint64_t j0, Real out[4]) const {
    const uint32_t b = (uint32_t)(j0 >> 2);
    const int off = (int)(j0 & 3);
    Real lo[4];
    normals4<Real>(b, lo);
    if (off == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) out[e] = lo[e];
      return;
    }
    Real hi[4];
    normals4<Real>(b + 1, hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int w = off + e;
      out[e] = w < 4 ? lo[w & 3] : hi[w & 3];
    }
  }
};

// Round keys of one launch-uniform Philox key (k0 + r W0, k1 + r W1, r = 0..9),
// computed on the host: inside a kernel parameter they feed the round LOP3s as
// constant-bank operands, so the hot loops carry no key schedule (no registers,
// no adds).
struct PhiloxRoundKeys {
  uint32_t k0[10], k1[10];
};

inline void philox_round_keys(uint64_t seed, uint64_t round, uint64_t substep, PhiloxRoundKeys& rk) {
  uint32_t k0, k1;
  philox_key(seed, round, substep, k0, k1);
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    rk.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
}

__device__ __forceinline__ uint4 philox10_rk(uint4 c, const PhiloxRoundKeys& rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mulwide(0xD2511F53u, c.x, lo0, hi0);
    mulwide(0xCD9E8D57u, c.z, lo1, hi1);
    c = make_uint4(hi1 ^ c.y ^ rk.k0[r], lo1, hi0 ^ c.w ^ rk.k1[r], lo0);
  }
  return c;
}

// PhiloxKey with the round keys read from a kernel parameter (same stream bits)
struct PhiloxKeyC {
  const PhiloxRoundKeys* rk;
  uint32_t c1, c2, c3;

  __device__ __forceinline__ void init(const PhiloxRoundKeys& keys, uint64_t particle, uint64_t step) {
    rk = &keys;
    c1 = (uint32_t)step;
    c2 = (uint32_t)particle;
    c3 = (uint32_t)(particle >> 32) ^ ((uint32_t)(step >> 32) * 0x9E3779B9u);
  }
  __device__ __forceinline__ uint4 block(uint32_t b) const {
    return philox10_rk(make_uint4(b, c1, c2, c3), *rk);
  }
  __device__ __forceinline__ uint64_t u64(uint32_t k) const {
    const uint4 w = philox10_rk(make_uint4(0x80000000u | k, c1, c2, c3), *rk);
    return ((uint64_t)w.x << 32) | w.y;
  }
  __device__ __forceinline__ double uniform(uint32_t k) const {
    return (double)(u64(k) >> 11) * 0x1.0p-53;
  }
  template <typename Real>
  __device__ __forceinline__ void normals4(uint32_t b, Real out[4]) const {
    const uint4 w = block(b);
    bm_pair<Real>(w.x, w.y, out[0], out[1]);
    bm_pair<Real>(w.z, w.w, out[2], out[3]);
  }
  template <typename Real>
  __device__ __forceinline__ void normals4_at(uint64_t j0, Real out[4]) const {
    const uint32_t b = (uint32_t)(j0 >> 2);
    const int off = (int)(j0 & 3);
    Real lo[4];
    normals4<Real>(b, lo);
    if (off == 0) {
#pragma unroll
      for (int e = 0; e < 4; ++e) out[e] = lo[e];
      return;
    }
    Real hi[4];
    normals4<Real>(b + 1, hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int w = off + e;
      out[e] = w < 4 ? lo[w & 3] : hi[w & 3];
    }
  }
};

// Sequential Philox view: normal()/uniform() calls in stream order, exactly as
// the shadow Stream counts them.
template <typename Real>
struct PhSeq {
  PhiloxKey key;
  uint64_t nn;   // normals drawn
  uint32_t nu;   // u64 draws
  Real cache[4];

  __device__ __forceinline__ void init(uint64_t seed, uint64_t round, uint64_t particle,
                                       uint64_t step, uint64_t substep) {
    key.init(seed, round, particle, step, substep);
    nn = 0;
    nu = 0;
  }
  __device__ __forceinline__ Real normal() {
    const int w = (int)(nn & 3);
    if (w == 0) key.normals4<Real>((uint32_t)(nn >> 2), cache);
    ++nn;
    return w == 0 ? cache[0] : (w == 1 ? cache[1] : (w == 2 ? cache[2] : cache[3]));
  }
  __device__ __forceinline__ double uniform() { return key.uniform(nu++); }
};

// Sequential xoshiro view with the sampler's Real.
template <typename Real>
struct XoSeq {
  XoStream st;
  __device__ __forceinline__ void init(uint64_t seed, uint64_t round, uint64_t particle,
                                       uint64_t step, uint64_t substep) {
    st.init(seed, round, particle, step, substep);
  }
  __device__ __forceinline__ Real normal() { return (Real)st.normal(); }
  __device__ __forceinline__ double uniform() { return st.uniform(); }
};

}  // namespace asmcdev
