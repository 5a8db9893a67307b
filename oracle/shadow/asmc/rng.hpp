#pragma once
// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Philox "shadow" of the reference's keyed RNG header
// (/root/reference/proj/include/asmc/rng.hpp:1-109).  Same names, same Key
// fields, same Stream interface (next_u64 / uniform / normal / categorical),
// but the key addresses a counter-based Philox4x32-10 stream instead of a
// hashed xoshiro256++ state.  Compiling the UNMODIFIED reference sources with
// `-I oracle/shadow` ahead of `-I /root/reference/proj/include` makes
// target.cpp / kernel.cpp / engine.cpp / drivers.cpp draw from this stream,
// which is what the B200 kernels' `rng = philox` mode reproduces in parallel
// (BASELINE.json north_star: "the same Philox streams").
//
// Stream definition (the device implements exactly this indexing):
//   key64 = mix64 chain over (seed, round, substep); Philox key = (lo32, hi32)
//   counter words c1 = lo32(step), c2 = lo32(particle),
//                 c3 = hi32(particle) ^ (hi32(step) * 0x9E3779B9)
//   normal #j   : block b = j >> 2 at counter (b, c1, c2, c3) -> words w0..w3;
//                 pair (w0,w1) gives normals 4b (cos) and 4b+1 (sin),
//                 pair (w2,w3) gives normals 4b+2 (cos) and 4b+3 (sin);
//                 u1 = (w_even + 1) * 2^-32 in (0,1], u2 = w_odd * 2^-32,
//                 r = sqrt(-2 log u1), angle = 2 pi u2   (Box-Muller)
//   next_u64 #k : counter (0x80000000 | k, c1, c2, c3) -> (w0 << 32) | w1
//   uniform     : (next_u64 >> 11) * 2^-53   (as rng.hpp:71)
// Normal and uniform draws use disjoint counter ranges, so the k-th uniform
// and the j-th normal of one stream are addressable independently -- the
// property that lets 32 lanes of a warp draw one particle's proposal.

#include <cmath>
#include <cstdint>
#include <span>

namespace asmc::rng {

struct Key {
  std::uint64_t seed = 0;
  std::uint64_t round = 0;
  std::uint64_t particle = 0;
  std::uint64_t step = 0;
  std::uint64_t substep = 0;
};

inline constexpr std::uint64_t kSubstepInit = 0;
inline constexpr std::uint64_t kSubstepExplore = 1;
inline constexpr std::uint64_t kSubstepResample = 2;
inline constexpr std::uint64_t kSubstepSwap = 3;

namespace detail {

inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline void philox4x32_10(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * c[0];
    const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * c[2];
    const std::uint32_t n0 = static_cast<std::uint32_t>(p1 >> 32) ^ c[1] ^ k0;
    const std::uint32_t n1 = static_cast<std::uint32_t>(p1);
    const std::uint32_t n2 = static_cast<std::uint32_t>(p0 >> 32) ^ c[3] ^ k1;
    const std::uint32_t n3 = static_cast<std::uint32_t>(p0);
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

}  // namespace detail

class Stream {
 public:
  explicit Stream(const Key& k) {
    using detail::mix64;
    std::uint64_t acc = mix64(k.seed + 0x9E3779B97F4A7C15ULL);
    acc = mix64(acc ^ (k.round + 0xD1B54A32D192ED03ULL));
    acc = mix64(acc ^ (k.substep + 0x9FB21C651E98DF25ULL));
    k0_ = static_cast<std::uint32_t>(acc);
    k1_ = static_cast<std::uint32_t>(acc >> 32);
    c1_ = static_cast<std::uint32_t>(k.step);
    c2_ = static_cast<std::uint32_t>(k.particle);
    c3_ = static_cast<std::uint32_t>(k.particle >> 32) ^
          (static_cast<std::uint32_t>(k.step >> 32) * 0x9E3779B9u);
  }

  std::uint64_t next_u64() {
    std::uint32_t c[4] = {0x80000000u | static_cast<std::uint32_t>(n_u64_++), c1_, c2_, c3_};
    detail::philox4x32_10(c, k0_, k1_);
    return (static_cast<std::uint64_t>(c[0]) << 32) | c[1];
  }

  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

  double normal() {
    const std::uint64_t j = n_normal_++;
    const std::uint64_t b = j >> 2;
    if (b != block_) {
      std::uint32_t c[4] = {static_cast<std::uint32_t>(b), c1_, c2_, c3_};
      detail::philox4x32_10(c, k0_, k1_);
      for (int i = 0; i < 4; ++i) words_[i] = c[i];
      block_ = b;
    }
    const unsigned w = static_cast<unsigned>(j & 3);
    const double u1 = (static_cast<double>(words_[w & 2u]) + 1.0) * 0x1.0p-32;
    const double u2 = static_cast<double>(words_[(w & 2u) + 1u]) * 0x1.0p-32;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586477 * u2;
    return (w & 1u) ? r * std::sin(a) : r * std::cos(a);
  }

  std::size_t categorical(std::span<const double> weights) {
    double total = 0.0;
    for (double w : weights) total += w;
    const double u = uniform() * total;
    double c = 0.0;
    for (std::size_t i = 0; i + 1 < weights.size(); ++i) {
      c += weights[i];
      if (u < c) return i;
    }
    return weights.empty() ? 0 : weights.size() - 1;
  }

 private:
  std::uint32_t k0_, k1_, c1_, c2_, c3_;
  std::uint64_t n_u64_ = 0;
  std::uint64_t n_normal_ = 0;
  std::uint64_t block_ = ~std::uint64_t{0};
  std::uint32_t words_[4] = {0, 0, 0, 0};
};

inline Stream stream_for(const Key& k) { return Stream(k); }

}  // namespace asmc::rng
