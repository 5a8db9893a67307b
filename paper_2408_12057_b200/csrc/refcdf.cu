// Systematic resampling with the reference's CDF, bit for bit, computed in parallel.
//
// The reference (proj/src/engine.cpp:61-80) resamples from a SEQUENTIAL fp64 CDF:
//   l1  = logsumexp(log_w)            -- LogAccumulator over particles in order
//                                        (proj/include/asmc/logsum.hpp:18-45, 97-101)
//   cum = e_0, cum += e_j, ...        -- e_j = exp(log_w_j - l1), one rounding per add
//   a_m = first j with !(cum_j < (m + u)/n), clamped to n - 1.
// Both l1 and cum are chains of N dependent fp64 roundings.  This file reproduces those
// chains exactly without running them serially:
//
//  * While a running sum s stays inside one binade [2^k, 2^(k+1)) (grid u_k = 2^(k-52)),
//    fl(s + e) = s + r_k(e) u_k, where r_k(e) = e/u_k rounded to the nearest integer --
//    the rounding of each add no longer depends on s, except at an exact tie (the
//    ties-to-even bit depends on s's parity).  So inside a binade the sequential sum is
//    an INTEGER prefix sum: exact, associative, parallel.
//  * An approximate parallel scan (any order, rigorous error bound 8 j 2^-53 relative)
//    says in which binade the exact sum is during each 256-particle block.  Blocks whose
//    whole range sits strictly inside one binade, with no tie and (for l1) no change of
//    the running max, are "stable": their exact integer totals r_k are summed in parallel.
//  * One CTA walks the runs of stable blocks (one exact integer add per run) and replays
//    the few remaining blocks -- binade crossings (~log2 N of them), ties (~1 per 2^22
//    particles), running-max changes of the LogAccumulator (~ln N) -- element by element
//    with the reference's own fp64 operations.  It re-checks every run's binade on the
//    EXACT value, so the error bound only decides speed, never the bits.
//  * exp is glibc's (libm_exact.cuh: gexp), so e_j are the host's bits.  The one scalar
//    log of l1 is correctly rounded (crlog); glibc's 0.52-ulp log differs from it on ~5e-4
//    of arguments.
// One cooperative launch per resampling event (phases separated by grid.sync()); under
// st->resample_now gating the launch returns at once on steps that do not resample.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "engine_kernels.h"
#include "libm_exact.cuh"

namespace cg = cooperative_groups;

namespace asmcdev {

namespace {

constexpr int kT = 256;           // threads per CTA = particles per block
constexpr int kTile = 4 * kT;     // CTA-0 scans: 1024 blocks per tile
constexpr int kUnstable = -100000;
constexpr int kModeLse = 0, kModeCdf = 1;
constexpr double kNegInfD = -__builtin_huge_val();
constexpr unsigned long long kTwo52 = 1ull << 52, kTwo53 = 1ull << 53;

struct Args {
  const double* lw;
  uint64_t n, nblk;
  SmcState* st;
  int gated;
  RefCdfWork w;
  double* cum;
  uint32_t* anc;
  int want_anc;
};

// binade index of s >= 0: s in [2^k, 2^(k+1)); everything below 2^-1021 shares the
// subnormal grid 2^-1074 and is binade -1022.  Non-finite -> a value no run matches.
__device__ __forceinline__ int binade(double s) {
  if (!(s >= 0x1p-1022)) return -1022;
  const uint64_t b = (uint64_t)__double_as_longlong(s);
  const int ef = (int)((b >> 52) & 0x7ff);
  return ef == 0x7ff ? 0x40000000 : ef - 1023;
}

// s / u_k for s in binade k (the significand with its hidden bit; subnormals without)
__device__ __forceinline__ unsigned long long sum_units(double s) {
  const uint64_t b = (uint64_t)__double_as_longlong(s);
  const uint64_t m = b & (kTwo52 - 1);
  return ((b >> 52) & 0x7ff) ? (m | kTwo52) : m;
}

// units * u_k as a double (units < 2^53; units >= 2^52 unless k == -1022)
__device__ __forceinline__ double units_value(unsigned long long units, int k) {
  if (units >= kTwo52) return __longlong_as_double((long long)((((uint64_t)(k + 1023)) << 52) | (units - kTwo52)));
  return __longlong_as_double((long long)units);  // k == -1022: the subnormal encoding
}

// r_k(e) = e / u_k rounded to nearest; tie: exactly half-way (parity-dependent),
// sat: e >= 2^(k+1)... (cannot stay in the binade)
__device__ __forceinline__ unsigned long long add_units(double e, int k, bool& tie, bool& sat) {
  const uint64_t b = (uint64_t)__double_as_longlong(e);
  if ((b & ~(1ull << 63)) == 0) return 0;
  const int ef = (int)((b >> 52) & 0x7ff);
  uint64_t m = b & (kTwo52 - 1);
  int E = -1022;
  if (ef) {
    E = ef - 1023;
    m |= kTwo52;
  }
  const int sh = k - E;
  if (sh <= 0) {
    sat |= (sh < 0) || (sh == 0 && k > -1022);
    return sh == 0 ? m : 0;
  }
  if (sh > 54) return 0;
  const uint64_t q = m >> sh, rem = m & ((1ull << sh) - 1), half = 1ull << (sh - 1);
  tie |= (rem == half);
  return q + (rem > half ? 1 : 0);
}

// ---- CTA helpers --------------------------------------------------------------
// exclusive prefix max over the CTA's elements (thread order), seeded with `seed`
__device__ __forceinline__ double cta_excl_max(double v, double seed, double* sh) {
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  double inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, inc, o);
    if (ln >= o) inc = fmax(inc, t);
  }
  __syncthreads();
  if (ln == 31) sh[w] = inc;
  __syncthreads();
  double pre = seed;
  for (int i = 0; i < w; ++i) pre = fmax(pre, sh[i]);
  const double up = __shfl_up_sync(0xffffffffu, inc, 1);
  return ln == 0 ? pre : fmax(pre, up);
}

// inclusive prefix sum over the CTA's elements (thread order)
__device__ __forceinline__ unsigned long long cta_incl_u64(unsigned long long v, unsigned long long* sh) {
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (ln >= o) inc += t;
  }
  __syncthreads();
  if (ln == 31) sh[w] = inc;
  __syncthreads();
  unsigned long long pre = 0;
  for (int i = 0; i < w; ++i) pre += sh[i];
  return pre + inc;
}

// The element operation of particle j.  LSE (LogAccumulator::add, logsum.hpp:20-28):
//   log_w == -inf          -> no-op (ADD 0)
//   log_w <= running max   -> s += exp(log_w - max)          (ADD)
//   log_w >  running max   -> s = s * exp(max - log_w) + 1    (RESCALE)
// CDF (engine.cpp:68-75): s += exp(log_w - l1).  warp_ops evaluates them (P2) and caches
// the values (RefCdfWork::opv); classification, replays and materialisation read the cache.
struct Op {
  double v;
  bool rescale;
};

// ---- the grid phases work on one WARP per 256-particle block ------------------
// Lane l holds particles b kT + 8 l .. 8 l + 7, consecutive, so lane-local order is
// particle order and prefix operations are a lane-local pass plus one warp scan.  No CTA
// barrier inside a phase, and each lane has its 8 loads in flight at once (the phases
// are L2-latency bound: the 8 B per particle stay L2-resident across them).
constexpr int kPer = kT / 32;

__device__ __forceinline__ void warp_load(const Args& A, uint64_t b, double (&l)[kPer]) {
  const uint64_t j0 = b * kT + kPer * (threadIdx.x & 31);
#pragma unroll
  for (int e = 0; e < kPer; ++e) l[e] = j0 + e < A.n ? A.lw[j0 + e] : kNegInfD;
}

// block_op for the lane's 8 particles: v[e] and the rescale bits (LSE: the exclusive
// prefix max in particle order, seeded with the blocks before, bmax[b] after P1)
__device__ __forceinline__ unsigned warp_ops(const Args& A, int mode, uint64_t b, const double (&l)[kPer],
                                             double l1, double (&v)[kPer]) {
  const int ln = threadIdx.x & 31;
  const uint64_t j0 = b * kT + kPer * ln;
  if (mode == kModeCdf) {
#pragma unroll
    for (int e = 0; e < kPer; ++e) v[e] = j0 + e < A.n ? gexp(__dsub_rn(l[e], l1)) : 0.0;
    return 0u;
  }
  double inc = l[0];
#pragma unroll
  for (int e = 1; e < kPer; ++e) inc = fmax(inc, l[e]);
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, inc, o);
    if (ln >= o) inc = fmax(inc, t);
  }
  const double up = __shfl_up_sync(0xffffffffu, inc, 1);
  double pm = A.w.bmax[b];
  if (ln > 0) pm = fmax(pm, up);
  unsigned resc = 0u;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    if (l[e] == kNegInfD) {
      v[e] = 0.0;
    } else if (l[e] <= pm) {
      v[e] = gexp(__dsub_rn(l[e], pm));
    } else {
      v[e] = gexp(__dsub_rn(pm, l[e]));
      resc |= 1u << e;
    }
    pm = fmax(pm, l[e]);
  }
  return resc;
}

// the op cache: v with the rescale flag in its sign bit (v >= 0; a rescale by exp(-inf) = 0
// is stored as -0.0)
// (16-byte vector accesses: the cache is 16-byte aligned and a lane's 8 values contiguous)
__device__ __forceinline__ void warp_store_ops(const Args& A, uint64_t b, const double (&v)[kPer], unsigned resc) {
  const uint64_t j0 = b * kT + kPer * (threadIdx.x & 31);
  double c[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) c[e] = ((resc >> e) & 1u) ? -v[e] : v[e];
  if (j0 + kPer <= A.n) {
    double2* dst = reinterpret_cast<double2*>(A.w.opv + j0);
#pragma unroll
    for (int e = 0; e < kPer; e += 2) dst[e / 2] = make_double2(c[e], c[e + 1]);
  } else {
#pragma unroll
    for (int e = 0; e < kPer; ++e)
      if (j0 + e < A.n) A.w.opv[j0 + e] = c[e];
  }
}
__device__ __forceinline__ unsigned warp_cached_ops(const Args& A, uint64_t b, double (&v)[kPer]) {
  const uint64_t j0 = b * kT + kPer * (threadIdx.x & 31);
  double c[kPer];
  if (j0 + kPer <= A.n) {
    const double2* src = reinterpret_cast<const double2*>(A.w.opv + j0);
#pragma unroll
    for (int e = 0; e < kPer; e += 2) {
      const double2 q = src[e / 2];
      c[e] = q.x;
      c[e + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < kPer; ++e) c[e] = j0 + e < A.n ? A.w.opv[j0 + e] : 0.0;
  }
  unsigned resc = 0u;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    if (signbit(c[e])) resc |= 1u << e;
    v[e] = fabs(c[e]);
  }
  return resc;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- phases -------------------------------------------------------------------
// P0: per-block max of log_w (LSE)
__device__ void phase_block_max(const Args& A) {
  const uint64_t nw = (uint64_t)gridDim.x * (kT / 32);
  for (uint64_t b = (uint64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); b < A.nblk; b += nw) {
    double l[kPer];
    warp_load(A, b, l);
    double m = l[0];
#pragma unroll
    for (int e = 1; e < kPer; ++e) m = fmax(m, l[e]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) A.w.bmax[b] = m;
  }
}

// P1 (CTA 0): bmax -> exclusive prefix max over blocks; gmax = max over all
__device__ void phase_scan_max(const Args& A, double* buf, double* sh) {
  double carry = kNegInfD;
  auto load = [&](uint64_t t0, double (&v)[4]) {  // tile t0's entries (next tile prefetched)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t i = t0 + 4 * threadIdx.x + e;
      v[e] = i < A.nblk ? A.w.bmax[i] : kNegInfD;
    }
  };
  double vn[4];
  load(0, vn);
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    double v[4], loc = kNegInfD;
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = vn[e];
    load(t0 + kTile, vn);
    const double pre0 = cta_excl_max(fmax(fmax(v[0], v[1]), fmax(v[2], v[3])), carry, sh);
    loc = pre0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      if (i < m) A.w.bmax[t0 + i] = loc;
      loc = fmax(loc, v[e]);
    }
    // tile max for the next carry: last thread's loc after its elements
    __syncthreads();
    if (threadIdx.x == kT - 1) buf[0] = loc;
    __syncthreads();
    carry = buf[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) A.w.gmax[0] = carry;
}

// affine map s -> a s + b; (l then r) = (ar al, ar bl + br)
struct Aff {
  double a, b;
};
__device__ __forceinline__ Aff aff_then(Aff l, Aff r) {
  return Aff{__dmul_rn(r.a, l.a), __fma_rn(r.a, l.b, r.b)};
}

// P2: per-block composite of the element maps (approximate; any association): the
// lane's 8 maps in order, then an ordered shuffle tree (lane i holds [i, i + 2o))
__device__ void phase_block_affine(const Args& A, int mode, double l1) {
  const int ln = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (kT / 32);
  for (uint64_t b = (uint64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); b < A.nblk; b += nw) {
    double l[kPer], v[kPer];
    warp_load(A, b, l);
    const unsigned resc = warp_ops(A, mode, b, l, l1, v);
    warp_store_ops(A, b, v, resc);
    Aff f = (resc & 1u) ? Aff{v[0], 1.0} : Aff{1.0, v[0]};
#pragma unroll
    for (int e = 1; e < kPer; ++e) f = aff_then(f, ((resc >> e) & 1u) ? Aff{v[e], 1.0} : Aff{1.0, v[e]});
    for (int o = 1; o < 32; o <<= 1) {
      const Aff r{__shfl_down_sync(0xffffffffu, f.a, o), __shfl_down_sync(0xffffffffu, f.b, o)};
      if ((ln & (2 * o - 1)) == 0) f = aff_then(f, r);
    }
    const bool special = __any_sync(0xffffffffu, resc != 0u);
    if (ln == 0) {
      A.w.ba[b] = f.a;
      A.w.bb[b] = f.b;
      A.w.kb[b] = special ? kUnstable : 0;  // refined in P4
    }
  }
}

// P3 (CTA 0): approximate running value at every block start: sstart[b] (b = 0..nblk).
// Tile of 1024 blocks, thread t composes its 4 consecutive maps, warp shuffle scan of
// the composites, warps in order.
__device__ void phase_scan_affine(const Args& A, Aff* wsh) {
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  double carry = 0.0;  // both chains start from s = 0 (logsum.hpp:47-48, engine.cpp:69)
  if (threadIdx.x == 0) A.w.sstart[0] = 0.0;
  auto load = [&](uint64_t t0, Aff (&f)[4]) {  // tile t0's maps (next tile prefetched)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t i = t0 + 4 * threadIdx.x + e;
      f[e] = i < A.nblk ? Aff{A.w.ba[i], A.w.bb[i]} : Aff{1.0, 0.0};
    }
  };
  Aff fn[4];
  load(0, fn);
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    Aff f[4], c{1.0, 0.0};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      f[e] = fn[e];
      c = aff_then(c, f[e]);
    }
    load(t0 + kTile, fn);
    Aff inc = c;  // inclusive over lanes <= ln
    for (int o = 1; o < 32; o <<= 1) {
      const Aff up{__shfl_up_sync(0xffffffffu, inc.a, o), __shfl_up_sync(0xffffffffu, inc.b, o)};
      if (ln >= o) inc = aff_then(up, inc);
    }
    if (ln == 31) wsh[w] = inc;
    __syncthreads();
    Aff pre{1.0, 0.0};
    for (int v = 0; v < w; ++v) pre = aff_then(pre, wsh[v]);
    const Aff lup{__shfl_up_sync(0xffffffffu, inc.a, 1), __shfl_up_sync(0xffffffffu, inc.b, 1)};
    if (ln > 0) pre = aff_then(pre, lup);
    double sv = __fma_rn(pre.a, carry, pre.b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      sv = __fma_rn(f[e].a, sv, f[e].b);
      if (i < m) A.w.sstart[t0 + i + 1] = sv;
    }
    Aff tot{1.0, 0.0};
    for (int v = 0; v < kT / 32; ++v) tot = aff_then(tot, wsh[v]);
    carry = __fma_rn(tot.a, carry, tot.b);
    __syncthreads();
  }
}

// P4: classify each block; stable blocks get their exact integer total at binade k
__device__ void phase_classify(const Args& A, int mode, double l1) {
  const int ln = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (kT / 32);
  for (uint64_t b = (uint64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); b < A.nblk; b += nw) {
    const int pre = A.w.kb[b];
    const uint64_t j0 = b * kT, j1 = min(A.n, j0 + kT);
    const double s0 = A.w.sstart[b], s1 = A.w.sstart[b + 1];
    // |exact - approx| <= 8 j 2^-53 s (nonnegative terms, <= 2 roundings per element in
    // either evaluation) + subnormal slack; a factor 2 of margin on top.
    const double lo = s0 - (s0 * ((double)(16 * j0 + 64) * 0x1p-53) + (double)(j0 + 1) * 0x1p-1072);
    const double hi = s1 + (s1 * ((double)(16 * j1 + 64) * 0x1p-53) + (double)(j1 + 1) * 0x1p-1072);
    const int ka = binade(lo), kbn = binade(hi);
    if (!((pre != kUnstable) && ka == kbn && ka < 2000)) {  // warp-uniform
      if (ln == 0) A.w.kb[b] = kUnstable;
      continue;
    }
    double v[kPer];
    const unsigned resc = warp_cached_ops(A, b, v);  // P2's ops of this chain
    bool tie = false, sat = false;
    unsigned long long r = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) r += add_units(v[e], ka, tie, sat);
    const bool bad = __any_sync(0xffffffffu, tie || sat || resc != 0u);
    const unsigned long long tot = warp_sum_u64(r);
    if (ln == 0) {
      A.w.kb[b] = bad ? kUnstable : ka;
      A.w.tot[b] = tot;
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- the exact walk (CTA 0) ----------------------------------------------------
// Scans of 4 consecutive entries per thread (tile of 1024): exclusive prefix sums.
__device__ __forceinline__ unsigned long long scan4_u64(unsigned long long v[4], unsigned long long ex[4],
                                                        unsigned long long* wsh) {
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long c = v[0] + v[1] + v[2] + v[3];
  unsigned long long inc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (ln >= o) inc += t;
  }
  __syncthreads();
  if (ln == 31) wsh[w] = inc;
  __syncthreads();
  unsigned long long pre = inc - c, tot = 0;
  for (int i = 0; i < kT / 32; ++i) {
    if (i < w) pre += wsh[i];
    tot += wsh[i];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    ex[e] = pre;
    pre += v[e];
  }
  return tot;
}

struct WalkSmem {
  int kb[kTile];
  int hid[kTile];                // run (head) index of each block of the tile
  int heads[kTile + 1];          // first block of each run in the tile (+ m)
  unsigned long long P[kTile + 1];  // exclusive prefix of the stable totals in the tile
  unsigned long long u0[kTile];  // exact start units of each stable run
  unsigned long long wsh[kT / 32];
  double vbuf[kT];
  unsigned char fbuf[kT];
  double s;
  int nh, stop, stop_end, replays, ev_first;
  unsigned long long t_replay;  // profiling: %globaltimer ns spent replaying (thread 0)
};

// Replays block b element by element from the exact value W.s, with the reference's own
// fp64 operations; CDF mode stores cum.  Leaves the new value in W.s.
// Replays block b from the exact value W.s with the reference's own fp64 operations and
// leaves the new value in W.s (CDF mode also stores cum).  Events -- the elements that
// change the binade of the running value, exact ties and the LogAccumulator's rescales --
// are few in a replayed block (typically 1-3), so the block is replayed as segments:
// between two events every add is the integer r_k of the current binade (one CTA prefix
// scan per segment, all elements at once), and each event is applied directly in fp64.
// A block with many events (e.g. log-weights increasing with the index) is replayed by
// one thread, element by element.
__device__ void replay_block(const Args& A, int mode, uint64_t b, WalkSmem& W) {
  const uint64_t jj = b * kT + threadIdx.x;
  const double cached = jj < A.n ? A.w.opv[jj] : 0.0;  // P2's op of this chain
  const Op op{fabs(cached), (bool)signbit(cached)};
  const int i = threadIdx.x;
  const int m = (int)min((uint64_t)kT, A.n - b * kT);
  const double v = i < m ? op.v : 0.0;
  const bool resc = i < m && op.rescale;
  W.vbuf[i] = v;
  W.fbuf[i] = resc ? 1 : 0;
  const int nresc = __syncthreads_count(resc ? 1 : 0);
  if (nresc <= 16) {
    double cum = 0.0;  // this element's value after its op (CDF store)
    int start = 0;
    while (start < m) {  // uniform
      const double s = W.s;
      const int k = binade(s);
      const unsigned long long u0 = sum_units(s);
      bool tie = false, sat = false;
      const unsigned long long r = (i >= start && i < m) ? add_units(v, k, tie, sat) : 0ull;
      const unsigned long long inc = cta_incl_u64(r, W.wsh);
      const bool ev = i >= start && i < m && (resc || tie || sat || u0 + inc >= kTwo53 || k >= 0x40000000);
      // first event at or after `start` (m if none)
      if (i == 0) W.ev_first = m;
      __syncthreads();
      if (ev) atomicMin(&W.ev_first, i);
      __syncthreads();
      const int p = W.ev_first;
      if (i >= start && i < p) cum = units_value(u0 + inc, k);
      __syncthreads();
      if (i == p - 1 && p > start) W.s = cum;  // the value before the event / at the end
      __syncthreads();
      if (p < m) {
        if (i == p) {  // the event, in the reference's fp64 operations
          const double sp = W.s;
          cum = resc ? __dadd_rn(__dmul_rn(sp, v), 1.0) : __dadd_rn(sp, v);
          W.s = cum;
        }
        __syncthreads();
      }
      start = p + 1;
    }
    if (mode == kModeCdf) {
      const uint64_t j = b * kT + i;
      if (j < A.n) A.cum[j] = cum;
    }
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0) {
    double s = W.s;
    for (int i0 = 0; i0 < m; i0 += 8) {  // batches of 8: the loads are off the add chain
      double vv[8];
      unsigned char f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        vv[e] = W.vbuf[i0 + e];
        f[e] = W.fbuf[i0 + e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (i0 + e < m) {
          s = f[e] ? __dadd_rn(__dmul_rn(s, vv[e]), 1.0) : __dadd_rn(s, vv[e]);
          vv[e] = s;
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) W.vbuf[i0 + e] = vv[e];
    }
    W.s = s;
  }
  __syncthreads();
  if (mode == kModeCdf) {
    const uint64_t j = b * kT + threadIdx.x;
    if (j < A.n) A.cum[j] = W.vbuf[threadIdx.x];
  }
  __syncthreads();
}

// P5 (CTA 0): walk the blocks in order with the EXACT running value.  Per tile of 1024
// blocks: runs = maximal spans of stable blocks at one binade (unstable blocks are runs of
// one; a tile start always starts a run).  A stable run is one integer add after checking
// that the exact start lies in the run's binade and the run's total keeps it there; an
// unstable block (or a run failing the check -- not expected) is replayed.  CDF mode
// leaves bstart[b] = exact start units of every stable block for P6.
__device__ double phase_walk(const Args& A, int mode, double l1, double* sh, WalkSmem& W) {
  if (threadIdx.x == 0) {
    W.s = 0.0;
    W.replays = 0;
    W.t_replay = 0;
  }
  // tile t0's classes and stable totals; the next tile's are loaded while this one walks
  auto load = [&](uint64_t t0, int (&k)[4], unsigned long long (&v)[4]) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t i = t0 + 4 * threadIdx.x + e;
      k[e] = i < A.nblk ? A.w.kb[i] : kUnstable;
      v[e] = i < A.nblk ? A.w.tot[i] : 0ull;
    }
  };
  int kn[4];
  unsigned long long vn[4];
  load(0, kn, vn);
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    int k4[4], h4[4];
    unsigned long long v4[4], p4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      k4[e] = kn[e];
      v4[e] = k4[e] != kUnstable ? vn[e] : 0ull;
      if (i < m) W.kb[i] = k4[e];
    }
    load(t0 + kTile, kn, vn);
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      h4[e] = i < m && (i == 0 || k4[e] == kUnstable || W.kb[i - 1] == kUnstable || W.kb[i - 1] != k4[e]);
    }
    const unsigned long long tot = scan4_u64(v4, p4, W.wsh);
    unsigned long long hv[4], hx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) hv[e] = (unsigned long long)h4[e];
    const unsigned long long nh = scan4_u64(hv, hx, W.wsh);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      if (i < m) {
        W.P[i] = p4[e];
        W.hid[i] = (int)(hx[e] + hv[e]) - 1;
        if (h4[e]) W.heads[hx[e]] = i;
      }
    }
    if (threadIdx.x == 0) {
      W.P[m] = tot;
      W.heads[nh] = m;
      W.nh = (int)nh;
      W.stop = 0;
    }
    __syncthreads();
    int h = 0;
    while (h < W.nh) {  // uniform
      if (threadIdx.x == 0) {  // run ahead over the stable runs, stop at the first replay
        double s = W.s;
        int stop = W.nh, stop_end = 0;
        for (; h < W.nh; ++h) {
          const int b0 = W.heads[h], b1 = W.heads[h + 1], k = W.kb[b0];
          if (k != kUnstable) {
            const unsigned long long u0 = sum_units(s), total = W.P[b1] - W.P[b0];
            if (binade(s) == k && u0 + total < kTwo53) {
              W.u0[h] = u0;
              s = units_value(u0 + total, k);
              continue;
            }
          }
          stop = h;
          stop_end = b1;
          break;
        }
        W.s = s;
        W.stop = stop;
        W.stop_end = stop_end;
      }
      __syncthreads();
      h = W.stop;
      if (h >= W.nh) break;
      unsigned long long tr0 = 0;
      if (A.w.prof && threadIdx.x == 0) tr0 = gtimer();
      for (int i = W.heads[h]; i < W.stop_end; ++i) {
        replay_block(A, mode, t0 + i, W);
        if (threadIdx.x == 0) {
          ++W.replays;
          W.kb[i] = kUnstable;
          A.w.kb[t0 + i] = kUnstable;  // P6 skips it: the replay wrote its cum
        }
      }
      if (A.w.prof && threadIdx.x == 0) W.t_replay += gtimer() - tr0;
      ++h;
      __syncthreads();
    }
    if (mode == kModeCdf) {
      for (int i = threadIdx.x; i < m; i += kT) {
        if (W.kb[i] == kUnstable) continue;
        const int hh = W.hid[i];
        A.w.bstart[t0 + i] = W.u0[hh] + (W.P[i] - W.P[W.heads[hh]]);
      }
    }
    __syncthreads();
  }
  return W.s;
}

// P6 (grid, CDF): cum of the stable blocks from their exact start units (the lane's
// inclusive integer prefix plus the warp's exclusive scan of the lane totals)
__device__ void phase_materialize(const Args& A, double l1) {
  const int ln = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (kT / 32);
  for (uint64_t b = (uint64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); b < A.nblk; b += nw) {
    const int k = A.w.kb[b];
    if (k == kUnstable) continue;  // warp-uniform (the walk's replay wrote its cum)
    const unsigned long long u0 = A.w.bstart[b];
    double v[kPer];
    warp_cached_ops(A, b, v);
    bool tie = false, sat = false;
    unsigned long long r[kPer], t = 0;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      t += add_units(v[e], k, tie, sat);
      r[e] = t;
    }
    unsigned long long inc = t;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xffffffffu, inc, o);
      if (ln >= o) inc += x;
    }
    const unsigned long long base = u0 + (inc - t);
    const uint64_t j0 = b * kT + kPer * ln;
#pragma unroll
    for (int e = 0; e < kPer; ++e)
      if (j0 + e < A.n) A.cum[j0 + e] = units_value(base + r[e], k);
  }
}

// P7 (grid): a_m = first j with !(cum_j < pos_m), clamped to n - 1 (engine.cpp:68-76),
// inverted: particle j owns the output slots m with cum_{j-1} < pos_m <= cum_j (the last
// particle also every slot beyond cum_{n-1}), i.e. [M(cum_{j-1}), M(cum_j)) with
// M(c) = first m with pos_m > c.  pos_m = (m + u) / n is evaluated exactly as the
// reference does, M(c) from the estimate c n - u corrected by exact comparisons, so a
// thread reads two neighbouring CDF values (coalesced) and writes its slots: no search.
// pos_m = fl(fl(m + u) / n) > c, decided by a multiply by the rounded reciprocal rn = fl(1/n) unless the
// two are within 2^-50 relative: |x rn - fl(x / n)| <= 3.2 2^-53 (x / n), so outside that
// band the product orders like the quotient; inside it (in practice never) the division
// decides, as the reference computes it
__device__ __forceinline__ bool slot_above(uint64_t m, double u, double dn, double rn, double c) {
  const double x = __dadd_rn((double)m, u);
  const double q = __dmul_rn(x, rn);
  if (q > __dmul_rn(c, 1.0 + 0x1p-50)) return true;
  if (q < __dmul_rn(c, 1.0 - 0x1p-50)) return false;
  return __ddiv_rn(x, dn) > c;
}
__device__ __forceinline__ uint64_t first_slot_above(double c, double u, uint64_t n, double dn, double rn) {
  if (c != c) return n;  // a NaN CDF (NaN log-weights): no walk over all slots
  double est = floor(__fma_rn(c, dn, -u));
  if (!(est >= 0.0)) est = 0.0;  // also NaN
  uint64_t m = est > (double)n ? n : (uint64_t)est;
  while (m > 0 && slot_above(m - 1, u, dn, rn, c)) --m;
  while (m < n && !slot_above(m, u, dn, rn, c)) ++m;
  return m;
}
constexpr uint64_t kSlotRun = 8192;  // longer runs of one ancestor go to the whole grid (P8)
__device__ void phase_ancestors(const Args& A, double u) {
  const double dn = (double)A.n, rn = __drcp_rn(dn);
  const int ln = threadIdx.x & 31;
  // one M(cum) per lane: a warp covers 31 particles, lane l >= 1 owns particle
  // j = j0 + l - 1 and evaluates M(cum_j), its upper end; its lower end M(cum_{j-1}) is
  // lane l - 1's value (lane 0 evaluates M(cum_{j0-1}) only).  Warp-uniform trip count.
  const uint64_t nwarp = (uint64_t)gridDim.x * (kT / 32);
  for (uint64_t j0 = ((uint64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5)) * 31; j0 < A.n; j0 += nwarp * 31) {
    const uint64_t idx = j0 + ln;  // = j + 1: the CDF entry this lane evaluates is idx - 1
    uint64_t mv = 0;
    if (idx >= 1 && idx <= A.n) mv = idx == A.n ? A.n : first_slot_above(A.cum[idx - 1], u, A.n, dn, rn);
    uint64_t lo = __shfl_up_sync(0xffffffffu, mv, 1), hi = mv;
    const bool own = ln >= 1 && idx - 1 < A.n;
    const uint64_t j = idx - 1;
    if (!own) lo = hi = 0;
    if (own && hi - lo > kSlotRun) {  // a heavy ancestor: the rest of its slots go to the grid
      const unsigned int e = atomicAdd(A.w.novf, 1u);
      A.w.ovf[3 * e] = lo + kSlotRun;
      A.w.ovf[3 * e + 1] = hi;
      A.w.ovf[3 * e + 2] = j;
      hi = lo + kSlotRun;
    }
    // short runs (the common case: ~1 slot per particle) by their own lane; the warp
    // writes the longer ones together, 32 slots at a time
    const bool big = hi - lo > 32;
    if (!big)
      for (uint64_t m = lo; m < hi; ++m) A.anc[m] = (uint32_t)j;
    unsigned int bal = __ballot_sync(0xffffffffu, big);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const uint64_t a = __shfl_sync(0xffffffffu, lo, src), e = __shfl_sync(0xffffffffu, hi, src);
      for (uint64_t m = a + ln; m < e; m += 32) A.anc[m] = (uint32_t)(j0 + src - 1);
    }
  }
}

// P8 (grid): the slot runs of heavy ancestors, every CTA striding over each run
__device__ void phase_heavy_slots(const Args& A) {
  const unsigned int ne = *(volatile unsigned int*)A.w.novf;
  for (unsigned int e = 0; e < ne; ++e) {
    const uint64_t lo = A.w.ovf[3 * e], hi = A.w.ovf[3 * e + 1];
    const uint32_t j = (uint32_t)A.w.ovf[3 * e + 2];
    for (uint64_t m = lo + (uint64_t)blockIdx.x * kT + threadIdx.x; m < hi; m += (uint64_t)gridDim.x * kT)
      A.anc[m] = j;
  }
}

__global__ void __launch_bounds__(kT, 4) refcdf_kernel(Args A) {
  if (A.gated && !*(volatile int*)&A.st->resample_now) return;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kT / 32 + 2];
  __shared__ unsigned long long ush[kT / 32 + 2];
  __shared__ union U {
    Aff wa[kT / 32];
    WalkSmem walk;
  } u;
  const bool lead = blockIdx.x == 0;
  // profiling (RefCdfWork::prof != null): CTA 0 stamps %globaltimer at each phase end
#define MARK(i) \
  if (A.w.prof && lead && threadIdx.x == 0) A.w.prof[i] = gtimer();
  MARK(0);
  if (lead && threadIdx.x == 0) *A.w.novf = 0u;

  // ---- l1 = logsumexp(log_w) ----
  phase_block_max(A);
  grid.sync();
  MARK(1);
  if (lead) phase_scan_max(A, sh + 8, sh);
  grid.sync();
  MARK(2);
  phase_block_affine(A, kModeLse, 0.0);
  grid.sync();
  MARK(3);
  if (lead) phase_scan_affine(A, u.wa);
  grid.sync();
  MARK(4);
  phase_classify(A, kModeLse, 0.0);
  grid.sync();
  MARK(5);
  if (lead) {
    const double s = phase_walk(A, kModeLse, 0.0, sh, u.walk);
    if (threadIdx.x == 0 && A.w.prof) {
      A.w.prof[14] = u.walk.replays;
      A.w.prof[12 + 1] = u.walk.t_replay;
    }
    if (threadIdx.x == 0) {
      const double M = A.w.gmax[0];
      // LogAccumulator::log_total (logsum.hpp:40-42)
      const double l1 = M == kNegInfD ? kNegInfD : __dadd_rn(M, crlog(s));
      A.w.l1[0] = l1;
      if (l1 == kNegInfD) A.st->err = ASMC_ERR_DEGENERATE;
    }
  }
  grid.sync();
  MARK(6);
  const double l1 = *(volatile double*)A.w.l1;
  if (l1 == kNegInfD || A.want_anc < 0) return;  // degenerate (engine.cpp:66) / l1 only

  // ---- cum_j, the reference's sequential CDF ----
  phase_block_affine(A, kModeCdf, l1);
  grid.sync();
  MARK(7);
  if (lead) phase_scan_affine(A, u.wa);
  grid.sync();
  MARK(8);
  phase_classify(A, kModeCdf, l1);
  grid.sync();
  MARK(9);
  if (lead) {
    const double s = phase_walk(A, kModeCdf, l1, sh, u.walk);
    if (threadIdx.x == 0 && A.w.prof) A.w.prof[15] = u.walk.replays + (u.walk.t_replay << 20);
    if (threadIdx.x == 0) A.st->total = s;
  }
  grid.sync();
  MARK(10);
  phase_materialize(A, l1);
  if (A.want_anc != 1) return;
  grid.sync();
  MARK(11);
  phase_ancestors(A, A.st->u);
  grid.sync();
  phase_heavy_slots(A);
  if (A.w.prof) {
    grid.sync();
    MARK(12);
  }
#undef MARK
}

__global__ void exact_math_kernel(int which, const double* x, uint64_t n, double* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = which == 0 ? gexp(x[i]) : crlog(x[i]);
}

}  // namespace

cudaError_t launch_exact_math(int which, const double* x, uint64_t n, double* out, cudaStream_t s) {
  const uint64_t blocks = (n + 255) / 256;
  exact_math_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(which, x, n, out);
  return cudaGetLastError();
}

size_t refcdf_work_bytes(uint64_t n) {
  const uint64_t nb = (n + kT - 1) / kT;
  // 6 double/u64 arrays + 1 int array of nb + 2 entries, 3 scalars, 16-byte alignment each
  return (size_t)(nb + 2) * (6 * 8 + 4) + 24 * (nb / 4 + 2) + 18 * 16 + 256 + 8 * (size_t)n + 16;
}

void refcdf_work_carve(void* base, uint64_t n, RefCdfWork* w) {
  const uint64_t nb = (n + kT - 1) / kT;
  char* p = (char*)base;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 15) / 16 * 16;
    return r;
  };
  w->bmax = (double*)take(8 * (nb + 1));
  w->ba = (double*)take(8 * (nb + 1));
  w->bb = (double*)take(8 * (nb + 1));
  w->sstart = (double*)take(8 * (nb + 1));
  w->tot = (unsigned long long*)take(8 * (nb + 1));
  w->bstart = (unsigned long long*)take(8 * (nb + 1));
  w->kb = (int*)take(4 * (nb + 1));
  w->ovf = (unsigned long long*)take(24 * (nb / 4 + 2));
  w->novf = (unsigned int*)take(16);
  w->gmax = (double*)take(16);
  w->l1 = (double*)take(16);
  w->opv = (double*)take(8 * n);
  w->prof = nullptr;
}

cudaError_t launch_refcdf(const double* lw, uint64_t n, SmcState* st, int gated, const RefCdfWork* w,
                          double* cum, uint32_t* anc, int want_anc, int sms, cudaStream_t s) {
  static thread_local int per = 0;
  if (per == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, refcdf_kernel, kT, 0);
    if (e != cudaSuccess) return e;
    if (per < 1) per = 1;
  }
  Args A;
  A.lw = lw;
  A.n = n;
  A.nblk = (n + kT - 1) / kT;
  A.st = st;
  A.gated = gated;
  A.w = *w;
  A.cum = cum;
  A.anc = anc;
  A.want_anc = want_anc;
  uint64_t grid = (uint64_t)sms * (uint64_t)per;
  if (grid > A.nblk) grid = A.nblk > 0 ? A.nblk : 1;
  void* args[] = {&A};
  return cudaLaunchCooperativeKernel((const void*)refcdf_kernel, dim3((unsigned)grid), dim3(kT), args, 0, s);
}

}  // namespace asmcdev
