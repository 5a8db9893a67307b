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
__device__ __forceinline__ double cta_max(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = sh[0];
  for (int i = 1; i < kT / 32; ++i) r = fmax(r, sh[i]);
  return r;
}

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

__device__ __forceinline__ unsigned long long cta_sum_u64(unsigned long long v, unsigned long long* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long r = 0;
  for (int i = 0; i < kT / 32; ++i) r += sh[i];
  return r;
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

// The element operation of particle j = b*kT + threadIdx.x in block b (all threads of
// the CTA call it together).  LSE (LogAccumulator::add, logsum.hpp:20-28):
//   log_w == -inf          -> no-op (ADD 0)
//   log_w <= running max   -> s += exp(log_w - max)          (ADD)
//   log_w >  running max   -> s = s * exp(max - log_w) + 1    (RESCALE)
// CDF (engine.cpp:68-75): s += exp(log_w - l1).
struct Op {
  double v;
  bool rescale;
};
__device__ __forceinline__ Op block_op(const Args& A, int mode, uint64_t b, double l1, double* sh) {
  const uint64_t j = b * kT + threadIdx.x;
  const bool in = j < A.n;
  const double l = in ? A.lw[j] : kNegInfD;
  if (mode == kModeCdf) return Op{in ? gexp(__dsub_rn(l, l1)) : 0.0, false};
  const double pm = cta_excl_max(l, A.w.bmax[b], sh);
  if (l == kNegInfD) return Op{0.0, false};
  if (l <= pm) return Op{gexp(__dsub_rn(l, pm)), false};
  return Op{gexp(__dsub_rn(pm, l)), true};
}

// ---- phases -------------------------------------------------------------------
// P0: per-block max of log_w (LSE)
__device__ void phase_block_max(const Args& A, double* sh) {
  for (uint64_t b = blockIdx.x; b < A.nblk; b += gridDim.x) {
    const uint64_t j = b * kT + threadIdx.x;
    const double m = cta_max(j < A.n ? A.lw[j] : kNegInfD, sh);
    if (threadIdx.x == 0) A.w.bmax[b] = m;
    __syncthreads();
  }
}

// P1 (CTA 0): bmax -> exclusive prefix max over blocks; gmax = max over all
__device__ void phase_scan_max(const Args& A, double* buf, double* sh) {
  double carry = kNegInfD;
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    double v[4], loc = kNegInfD;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * threadIdx.x + e;
      v[e] = i < m ? A.w.bmax[t0 + i] : kNegInfD;
    }
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

// P2: per-block composite of the element maps (approximate; any association)
__device__ void phase_block_affine(const Args& A, int mode, double l1, double* sh, Aff* ash, int* ish) {
  for (uint64_t b = blockIdx.x; b < A.nblk; b += gridDim.x) {
    const Op op = block_op(A, mode, b, l1, sh);
    Aff f = op.rescale ? Aff{op.v, 1.0} : Aff{1.0, op.v};
    const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {  // ordered tree: lane i holds [i, i + 2o) when i % 2o == 0
      const Aff r{__shfl_down_sync(0xffffffffu, f.a, o), __shfl_down_sync(0xffffffffu, f.b, o)};
      if ((ln & (2 * o - 1)) == 0) f = aff_then(f, r);
    }
    const int special = __syncthreads_or(op.rescale ? 1 : 0);
    if (ln == 0) ash[w] = f;
    __syncthreads();
    if (threadIdx.x == 0) {
      Aff t = ash[0];
      for (int i = 1; i < kT / 32; ++i) t = aff_then(t, ash[i]);
      A.w.ba[b] = t.a;
      A.w.bb[b] = t.b;
      A.w.kb[b] = special ? kUnstable : 0;  // refined in P4
    }
    __syncthreads();
  }
  (void)ish;
}

// P3 (CTA 0): approximate running value at every block start: sstart[b] (b = 0..nblk)
__device__ void phase_scan_affine(const Args& A, Aff* tile) {
  double carry = 0.0;  // both chains start from s = 0 (logsum.hpp:47-48, engine.cpp:69)
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    for (int i = threadIdx.x; i < kTile; i += kT)
      tile[i] = i < m ? Aff{A.w.ba[t0 + i], A.w.bb[t0 + i]} : Aff{1.0, 0.0};
    __syncthreads();
    for (int o = 1; o < kTile; o <<= 1) {  // Hillis-Steele inclusive scan
      Aff nv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = threadIdx.x + e * kT;
        nv[e] = i >= o ? aff_then(tile[i - o], tile[i]) : tile[i];
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 4; ++e) tile[threadIdx.x + e * kT] = nv[e];
      __syncthreads();
    }
    for (int i = threadIdx.x; i < m; i += kT) {
      const Aff f = tile[i];
      A.w.sstart[t0 + i + 1] = __fma_rn(f.a, carry, f.b);
    }
    if (t0 == 0 && threadIdx.x == 0) A.w.sstart[0] = 0.0;
    const Aff last = tile[m - 1];
    carry = __fma_rn(last.a, carry, last.b);
    __syncthreads();
  }
}

// P4: classify each block; stable blocks get their exact integer total at binade k
__device__ void phase_classify(const Args& A, int mode, double l1, double* sh, unsigned long long* ush) {
  for (uint64_t b = blockIdx.x; b < A.nblk; b += gridDim.x) {
    const int pre = A.w.kb[b];
    const uint64_t j0 = b * kT, j1 = min(A.n, j0 + kT);
    const double s0 = A.w.sstart[b], s1 = A.w.sstart[b + 1];
    // |exact - approx| <= 8 j 2^-53 s (nonnegative terms, <= 2 roundings per element in
    // either evaluation) + subnormal slack; a factor 2 of margin on top.
    const double lo = s0 - (s0 * ((double)(16 * j0 + 64) * 0x1p-53) + (double)(j0 + 1) * 0x1p-1072);
    const double hi = s1 + (s1 * ((double)(16 * j1 + 64) * 0x1p-53) + (double)(j1 + 1) * 0x1p-1072);
    const int ka = binade(lo), kbn = binade(hi);
    const bool cand = (pre != kUnstable) && ka == kbn && ka < 2000;
    if (!__syncthreads_or(cand ? 1 : 0)) {  // uniform
      if (threadIdx.x == 0) A.w.kb[b] = kUnstable;
      __syncthreads();
      continue;
    }
    const Op op = block_op(A, mode, b, l1, sh);
    bool tie = false, sat = false;
    const unsigned long long r = add_units(op.v, ka, tie, sat);
    const int bad = __syncthreads_or((tie || sat || op.rescale) ? 1 : 0);
    const unsigned long long tot = cta_sum_u64(r, ush);
    if (threadIdx.x == 0) {
      A.w.kb[b] = bad ? kUnstable : ka;
      A.w.tot[b] = tot;
    }
    __syncthreads();
  }
}

// P5 (CTA 0): runs.  A block starts a run when it is unstable, follows an unstable
// block, or changes binade (unstable blocks are runs of one).  hid[b] = its run's index;
// heads[h] = first block of run h (heads[H] = nblk); pw[b] = exclusive prefix of the
// integer totals inside b's run.
__device__ __forceinline__ int run_head(const Args& A, uint64_t b) {
  const int k = A.w.kb[b];
  return (b == 0) || k == kUnstable || A.w.kb[b - 1] == kUnstable || A.w.kb[b - 1] != k;
}

__device__ void phase_runs(const Args& A, int* fbuf, unsigned long long* vbuf, int* sh_i,
                           unsigned long long* sh_u) {
  int hcarry = 0;                 // runs started before this tile
  unsigned long long vcarry = 0;  // inclusive total of the open run at the tile's end
  for (uint64_t t0 = 0; t0 < A.nblk; t0 += kTile) {
    const int m = (int)min((uint64_t)kTile, A.nblk - t0);
    // (a) segmented inclusive scan of (head, total): (fl,vl).(fr,vr) = (fl|fr, fr ? vr : vl+vr)
    for (int i = threadIdx.x; i < kTile; i += kT) {
      const uint64_t b = t0 + i;
      fbuf[i] = i < m ? run_head(A, b) : 1;
      vbuf[i] = (i < m && A.w.kb[b] != kUnstable) ? A.w.tot[b] : 0ull;
    }
    __syncthreads();
    for (int o = 1; o < kTile; o <<= 1) {
      int nf[4];
      unsigned long long nv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = threadIdx.x + e * kT;
        nf[e] = fbuf[i];
        nv[e] = vbuf[i];
        if (i >= o) {
          if (!nf[e]) nv[e] += vbuf[i - o];
          nf[e] |= fbuf[i - o];
        }
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        fbuf[threadIdx.x + e * kT] = nf[e];
        vbuf[threadIdx.x + e * kT] = nv[e];
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < m; i += kT) {
      const uint64_t b = t0 + i;
      const unsigned long long incl = vbuf[i] + (fbuf[i] ? 0ull : vcarry);
      A.w.pw[b] = incl - (A.w.kb[b] != kUnstable ? A.w.tot[b] : 0ull);
      if (i == m - 1) sh_u[0] = incl;
    }
    __syncthreads();
    // (b) run index: inclusive count of heads
    for (int i = threadIdx.x; i < kTile; i += kT) fbuf[i] = i < m ? run_head(A, t0 + i) : 0;
    __syncthreads();
    for (int o = 1; o < kTile; o <<= 1) {
      int nv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = threadIdx.x + e * kT;
        nv[e] = fbuf[i] + (i >= o ? fbuf[i - o] : 0);
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < 4; ++e) fbuf[threadIdx.x + e * kT] = nv[e];
      __syncthreads();
    }
    for (int i = threadIdx.x; i < m; i += kT) {
      const uint64_t b = t0 + i;
      const int h = hcarry + fbuf[i] - 1;
      A.w.hid[b] = h;
      if (run_head(A, b)) A.w.heads[h] = (int)b;
    }
    __syncthreads();
    if (threadIdx.x == 0) sh_i[0] = hcarry + fbuf[m - 1];
    __syncthreads();
    hcarry = sh_i[0];
    vcarry = sh_u[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    A.w.heads[hcarry] = (int)A.nblk;
    A.w.nheads[0] = hcarry;
  }
}

// Replays block b element by element from the exact value s (thread 0's), the
// reference's own operations; CDF mode stores cum.  Returns the new s (thread 0).
__device__ double replay_block(const Args& A, int mode, uint64_t b, double l1, double s, double* sh,
                               double* vbuf, unsigned char* fbuf) {
  const Op op = block_op(A, mode, b, l1, sh);
  vbuf[threadIdx.x] = op.v;
  fbuf[threadIdx.x] = op.rescale ? 1 : 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int m = (int)min((uint64_t)kT, A.n - b * kT);
    for (int i = 0; i < m; ++i) {
      if (fbuf[i]) s = __dadd_rn(__dmul_rn(s, vbuf[i]), 1.0);
      else s = __dadd_rn(s, vbuf[i]);
      vbuf[i] = s;
    }
  }
  __syncthreads();
  if (mode == kModeCdf) {
    const uint64_t j = b * kT + threadIdx.x;
    if (j < A.n) A.cum[j] = vbuf[threadIdx.x];
  }
  __syncthreads();
  return s;
}

// P6 (CTA 0): the exact walk over runs.  Stable run: verify the EXACT start value lies in
// the run's binade and the run's integer total keeps it there -> one integer add; else
// (never expected) replay the run's blocks.  Unstable block: replay.  shead[b] = exact
// value before each stable run's first block.  Returns the final exact value.
__device__ double phase_walk(const Args& A, int mode, double l1, double* sh, double* vbuf,
                             unsigned char* fbuf, int* hb) {
  __shared__ double s_sh;
  __shared__ int flag_sh;
  double s = 0.0;
  const int H = A.w.nheads[0];
  for (int h0 = 0; h0 < H; h0 += kTile) {
    const int hm = min(kTile, H - h0);
    for (int i = threadIdx.x; i <= hm; i += kT) hb[i] = A.w.heads[h0 + i];
    __syncthreads();
    for (int i = 0; i < hm; ++i) {
      const int b = hb[i], bend = hb[i + 1];
      const int k = A.w.kb[b];
      if (threadIdx.x == 0) {
        int ok = 0;
        if (k != kUnstable) {
          const unsigned long long u0 = sum_units(s);
          const unsigned long long total = A.w.pw[bend - 1] + A.w.tot[bend - 1];
          if (binade(s) == k && (k == -1022 || u0 >= kTwo52) && u0 + total < kTwo53) {
            A.w.shead[b] = s;
            s = units_value(u0 + total, k);
            ok = 1;
          }
        }
        flag_sh = ok;
        s_sh = s;
      }
      __syncthreads();
      if (!flag_sh) {
        for (int bb = b; bb < bend; ++bb) {
          s = replay_block(A, mode, (uint64_t)bb, l1, s_sh, sh, vbuf, fbuf);
          if (threadIdx.x == 0) {
            A.w.kb[bb] = kUnstable;  // cum (CDF) written by the replay
            s_sh = s;
          }
          __syncthreads();
        }
      }
      s = s_sh;
      __syncthreads();
    }
  }
  return s;
}

// P7 (grid, CDF): cum of the stable blocks from their run's exact start value
__device__ void phase_materialize(const Args& A, double l1, double* sh, unsigned long long* ush) {
  for (uint64_t b = blockIdx.x; b < A.nblk; b += gridDim.x) {
    const int k = A.w.kb[b];
    if (k == kUnstable) continue;  // uniform per CTA
    const int hb = A.w.heads[A.w.hid[b]];
    const unsigned long long u0 = sum_units(A.w.shead[hb]) + A.w.pw[b];
    const Op op = block_op(A, kModeCdf, b, l1, sh);
    bool tie = false, sat = false;
    const unsigned long long r = add_units(op.v, k, tie, sat);
    const unsigned long long inc = cta_incl_u64(r, ush);
    const uint64_t j = b * kT + threadIdx.x;
    if (j < A.n) A.cum[j] = units_value(u0 + inc, k);
    __syncthreads();
  }
}

// P8 (grid): a_m = first j with !(cum_j < pos_m), clamped (engine.cpp:68-76)
__device__ void phase_ancestors(const Args& A, double u) {
  const double dn = (double)A.n;
  for (uint64_t m = (uint64_t)blockIdx.x * kT + threadIdx.x; m < A.n; m += (uint64_t)gridDim.x * kT) {
    const double pos = __ddiv_rn(__dadd_rn((double)m, u), dn);
    uint64_t lo = 0, hi = A.n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (A.cum[mid] < pos) lo = mid + 1;
      else hi = mid;
    }
    A.anc[m] = (uint32_t)(lo < A.n ? lo : A.n - 1);
  }
}

__global__ void __launch_bounds__(kT) refcdf_kernel(Args A) {
  if (A.gated && !*(volatile int*)&A.st->resample_now) return;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kT / 32 + 2];
  __shared__ unsigned long long ush[kT / 32 + 2];
  __shared__ __align__(16) unsigned char big[kTile * sizeof(Aff)];
  __shared__ double vbuf[kT];
  __shared__ unsigned char fbuf[kT];
  __shared__ int sh_i[2];
  Aff* atile = reinterpret_cast<Aff*>(big);
  int* ibuf = reinterpret_cast<int*>(big);
  unsigned long long* ubuf = reinterpret_cast<unsigned long long*>(big + kTile * sizeof(int));
  // big holds kTile Aff (16 KB) = kTile ints (4 KB) + kTile + 1 u64 (8 KB) as well
  const bool lead = blockIdx.x == 0;

  // ---- l1 = logsumexp(log_w) ----
  phase_block_max(A, sh);
  grid.sync();
  if (lead) phase_scan_max(A, sh + 8, sh);
  grid.sync();
  phase_block_affine(A, kModeLse, 0.0, sh, atile, ibuf);
  grid.sync();
  if (lead) phase_scan_affine(A, atile);
  grid.sync();
  phase_classify(A, kModeLse, 0.0, sh, ush);
  grid.sync();
  if (lead) phase_runs(A, ibuf, ubuf, sh_i, ush + 8);
  grid.sync();
  if (lead) {
    const double s = phase_walk(A, kModeLse, 0.0, sh, vbuf, fbuf, ibuf);
    if (threadIdx.x == 0) {
      const double M = A.w.gmax[0];
      // LogAccumulator::log_total (logsum.hpp:40-42)
      const double l1 = M == kNegInfD ? kNegInfD : __dadd_rn(M, crlog(s));
      A.w.l1[0] = l1;
      if (l1 == kNegInfD) A.st->err = ASMC_ERR_DEGENERATE;
    }
  }
  grid.sync();
  const double l1 = *(volatile double*)A.w.l1;
  if (l1 == kNegInfD || A.want_anc < 0) return;  // degenerate (engine.cpp:66) / l1 only

  // ---- cum_j, the reference's sequential CDF ----
  phase_block_affine(A, kModeCdf, l1, sh, atile, ibuf);
  grid.sync();
  if (lead) phase_scan_affine(A, atile);
  grid.sync();
  phase_classify(A, kModeCdf, l1, sh, ush);
  grid.sync();
  if (lead) phase_runs(A, ibuf, ubuf, sh_i, ush + 8);
  grid.sync();
  if (lead) {
    const double s = phase_walk(A, kModeCdf, l1, sh, vbuf, fbuf, ibuf);
    if (threadIdx.x == 0) A.st->total = s;
  }
  grid.sync();
  phase_materialize(A, l1, sh, ush);
  if (A.want_anc != 1) return;
  grid.sync();
  phase_ancestors(A, A.st->u);
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
  // 7 double/u64 arrays + 3 int arrays of nb + 2 entries, 3 scalars, 16-byte alignment each
  return (size_t)(nb + 2) * (7 * 8 + 3 * 4) + 16 * 16 + 256;
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
  w->pw = (unsigned long long*)take(8 * (nb + 1));
  w->shead = (double*)take(8 * (nb + 1));
  w->kb = (int*)take(4 * (nb + 1));
  w->hid = (int*)take(4 * (nb + 1));
  w->heads = (int*)take(4 * (nb + 2));
  w->gmax = (double*)take(16);
  w->l1 = (double*)take(16);
  w->nheads = (int*)take(16);
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
