// Fused particle pass, many-lanes-per-particle variant (fp32, Philox streams).
//
// G lanes (4 or 32) share one particle whose coordinates live in SHARED memory
// as float4 quads (quad q of the particle sits at xq[q]; lane l owns quads
// l, l+G, ...: consecutive lanes hit consecutive 16-byte words, so every
// LDS.128/STS.128 is conflict-free).  Keeping x out of registers lets the quad
// loop stay a real loop (small code, no I-cache thrash), keeps the register
// count low (high occupancy), and lifts the dimension limit to the shared
// memory budget instead of a compile-time register array.
//
// Reductions are per warp: after each (particle, step) a warp folds its groups'
// (log w, lg) pairs with a fixed xor tree and lane 0 adds the result to the
// warp's running accumulator for that step (shared memory).  Warps never wait
// on each other inside the pass; the block partial is formed once at the end
// by folding the 8 warp accumulators in warp order -- a fixed, GPU-count
// independent tree.
#pragma once

#include "pass_kernel.cuh"

namespace asmcdev {

constexpr int kWarps = kBlock / 32;
constexpr int kNoChecks = 99;  // SmemOps::delta_pass: no early-rejection checks

// dynamic shared memory: [groups][words][nquads] float4 (x, and vterm(x) for targets
// that cache it), then [kWarps][T+1][nacc] LogAcc
__host__ __device__ inline size_t smem_pass_bytes(int G, uint64_t d, int T, int nacc, int words = 1) {
  const size_t nq = (size_t)((d + 3) / 4);
  return (size_t)(kBlock / G) * nq * 16 * words + (size_t)kWarps * (T + 1) * nacc * sizeof(LogAcc);
}

template <class Tgt>
struct CacheWords {
  static constexpr int value = Tgt::kCacheV ? 2 : 1;
};

// RWMH on uncached targets keeps two rows per particle: the MH pass writes the
// proposal x + s z into the spare row and an accepted proposal just flips rows
// (no regeneration of its normals).  Same footprint as a cached target's x + vterm.
template <class Tgt, bool kHmc>
struct RowWords {
  static constexpr bool kDual = !kHmc;
  static constexpr int value = CacheWords<Tgt>::value * (kDual ? 2 : 1);
};

// kMove: 0 = RWMH (also idealized), 1 = HMC, 2 = elliptical slice -- separate
// instantiations, so each hot loop keeps its own registers and code layout
constexpr int kMoveRwmh = 0, kMoveHmc = 1, kMoveSlice = 2;

template <class Tgt, int G, int kMove = kMoveRwmh>
struct SmemOps {
  static constexpr bool kHmc = kMove == kMoveHmc;
  static constexpr bool kCache = Tgt::kCacheV;
  static constexpr bool kDual = RowWords<Tgt, kHmc>::kDual;

  // normals 4q .. 4q+3 of the draw set based at `base`
  __device__ static void quad(const PhiloxKeyC& k, uint64_t base, int q, float z[4]) {
    const uint64_t j0 = base + 4 * (uint64_t)q;
    if ((base & 3) == 0) k.template normals4<float>((uint32_t)(j0 >> 2), z);
    else k.template normals4_at<float>(j0, z);
  }

  __device__ static float4 vquad(const typename Tgt::F32& kf, float4 x) {
    return make_float4(Tgt::vpart(kf, x.x), Tgt::vpart(kf, x.y), Tgt::vpart(kf, x.z),
                       Tgt::vpart(kf, x.w));
  }

  // vq[q] = vterm(x) for the cached-potential targets (after a load or a redraw); returns
  // this lane's sum of the vterms (== vsum for these targets, same order); targets with
  // per-proposal checks also get the lane's sum of x^2 (their bound from sums, move())
  __device__ static float refresh_v(const TgtParams& T, int lane, int d, float4* xq) {
    float x2;
    return refresh_vx(T, lane, d, xq, x2);
  }
  __device__ static float refresh_vx(const TgtParams& T, int lane, int d, float4* xq, float& x2) {
    float s = 0.f;
    x2 = 0.f;
    if constexpr (kCache) {
      const int nq = (d + 3) >> 2;
      const typename Tgt::F32 kf = Tgt::f32(T, 0.0);
      for (int q = lane; q < nq; q += G) {
        const float4 x = xq[q];
        const float4 v = vquad(kf, x);
        xq[nq + q] = v;
        const float vv[4] = {v.x, v.y, v.z, v.w}, xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (4 * q + e < d) {
            s += vv[e];
            if constexpr (Tgt::kPerProposalCheck) x2 = fmaf(xv[e], xv[e], x2);
          }
      }
    }
    return s;
  }

  // x ~ eta for this lane's quads; returns the lane's vpart sum (vsum of the new x, same
  // order), so no separate pass over the row
  __device__ static float init(const TgtParams& T, int lane, int d, float4* xq, const PhiloxKeyC& k,
                               uint32_t& drawn) {
    const int nq = (d + 3) >> 2;
    const typename Tgt::F32 kf = Tgt::f32(T, 0.0);
    float s = 0.f;
    if ((d & 3) == 0) {  // every quad full: no per-coordinate tail checks
      for (int q = lane; q < nq; q += G) {
        ++drawn;
        float z[4];
        k.template normals4<float>((uint32_t)q, z);
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = Tgt::ref_draw32(T, z[e]);
        xq[q] = make_float4(v[0], v[1], v[2], v[3]);
        if constexpr (!kCache) {
#pragma unroll
          for (int e = 0; e < 4; ++e) s += Tgt::vpart(kf, v[e]);
        }
      }
    } else {
      for (int q = lane; q < nq; q += G) {
        ++drawn;
        float z[4];
        quad(k, 0, q, z);
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (4 * q + e < d) ? Tgt::ref_draw32(T, z[e]) : 0.f;
        xq[q] = make_float4(v[0], v[1], v[2], v[3]);
        if constexpr (!kCache) {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (4 * q + e < d) s += Tgt::vpart(kf, v[e]);
        }
      }
    }
    if constexpr (kCache) s = refresh_v(T, lane, d, xq);
    return s;
  }

  // this lane's sum of vpart(x) over its coordinates (quads lane, lane+G, ...; the
  // order delta_pass accumulates the proposal's sum in).  vpart does not depend on
  // beta for any target, so the pass carries the sum across steps and the weight is
  // one group reduction: V(x) = v_from(sum over lanes).
  __device__ static float vsum(const TgtParams& T, int lane, int d, const float4* xq) {
    const typename Tgt::F32 kf = Tgt::f32(T, 0.0);
    const int nq = (d + 3) >> 2;
    float s = 0.f;
    for (int q = lane; q < nq; q += G) {
      float xv[4];
      if constexpr (kCache) {
        const float4 v = xq[nq + q];
        xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
      } else {
        const float4 x = xq[q];
        xv[0] = Tgt::vpart(kf, x.x); xv[1] = Tgt::vpart(kf, x.y);
        xv[2] = Tgt::vpart(kf, x.z); xv[3] = Tgt::vpart(kf, x.w);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < d) s += xv[e];
    }
    return s;
  }

  __device__ static double weight(const TgtParams& T, double b0, double b1, float vs) {
    return (b1 - b0) * Tgt::v_from(T, group_sum<G>((double)vs));
  }

  // kernel.cpp:26-63 on this particle; vs (the lane's vpart sum) follows x
  // x2: this lane's sum of x^2 when known (Tgt::kPerProposalCheck targets after a load),
  // else NaN -- the early-rejection bound is then summed from the row (bound_total)
  __device__ static void move(const TgtParams& T, const KernelCfg& kc, int lane, int d,
                              double beta, float4*& xq, float4*& xalt, const PhiloxKeyC& k, uint32_t& drawn,
                              float& vs, float& x2) {
    const int nq = (d + 3) >> 2;
    const float x2_unknown = __int_as_float(0x7fffffff);
    if (kc.kind == ASMC_KERNEL_IDEALIZED) {
      const double mu = Tgt::exact_mu(T, beta);
      for (int q = lane; q < nq; q += G) {
        float z[4];
        quad(k, 0, q, z);
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (4 * q + e < d) ? (float)Tgt::exact_draw(T, mu, (double)z[e]) : 0.f;
        xq[q] = make_float4(v[0], v[1], v[2], v[3]);
      }
      __syncwarp();
      refresh_v(T, lane, d, xq);
      __syncwarp();
      vs = vsum(T, lane, d, xq);
      x2 = x2_unknown;
      return;
    }
    if constexpr (kMove == kMoveSlice) {
      if (kc.kind == ASMC_KERNEL_SLICE) slice(T, kc, lane, d, beta, xq, xalt, k, drawn, vs);
      x2 = x2_unknown;
      return;
    } else {
    if (kc.kind != (kHmc ? ASMC_KERNEL_HMC : ASMC_KERNEL_RWMH)) return;
    const typename Tgt::F32 kf = Tgt::f32(T, beta);
    const int nprop = kc.sweeps * kc.n_steps;
    double lu_pre = 0.0;  // lane l holds log u of proposal (q0 + l)
    const int gbase = (int)(threadIdx.x & 31) & ~(G - 1);
    if constexpr (kHmc) {
      // oracle/restate.c:hmc_cycle_move, coordinate-separable: each lane integrates
      // its coordinates' trajectories, the energy difference is reduced over the
      // group, and an accepted trajectory is re-integrated from regenerated momenta.
      const bool aligned = (d & 3) == 0;
      for (int p = 0; p < nprop; ++p) {
        const float eps = (float)kc.steps[p % kc.n_steps];
        const uint64_t base = (uint64_t)p * (uint64_t)d;
        if ((p % G) == 0) {
          const int pp = p + lane;
          lu_pre = pp < nprop ? log(k.uniform((uint32_t)pp)) : 0.0;
        }
        const float dl = aligned ? hmc_pass<true, false>(kf, k, lane, d, nq, base, eps, kc.leapfrog, xq)
                                 : hmc_pass<false, false>(kf, k, lane, d, nq, base, eps, kc.leapfrog, xq);
        const double delta = group_sum<G>((double)dl);
        const double log_u = __shfl_sync(0xffffffffu, lu_pre, gbase + (p % G));
        if (log_u < delta) {
          if (aligned) hmc_pass<true, true>(kf, k, lane, d, nq, base, eps, kc.leapfrog, xq);
          else hmc_pass<false, true>(kf, k, lane, d, nq, base, eps, kc.leapfrog, xq);
        }
      }
      __syncwarp();
      vs = vsum(T, lane, d, xq);
      x2 = x2_unknown;
      return;
    }
    // d % 4 == 0: every proposal's draw set starts on a Philox block, so the
    // hot loops use the one-block path with no tail checks (one copy of the
    // generator per loop: the loop body stays inside the L0 I-cache).
    const bool aligned = (d & 3) == 0;
    // early rejection: this lane's sum of max_h dlg(x_i, h) over its coordinates
    // (targets with kBoundFromV derive it from vs inside delta_pass)
    constexpr bool kBnd = Tgt::kEarly && !Tgt::kBoundFromV;
    float bnd = 0.f;
    bool bnd_ok = false;  // bnd holds the current row's bound (computed before a checking proposal)
    double u_pre = 1.0;  // lane l holds u of proposal (q0 + l)
    int si = 0;  // p % n_steps
    for (int p = 0; p < nprop; ++p) {
      const float s = (float)kc.steps[si];
      si = si + 1 == kc.n_steps ? 0 : si + 1;
      bool chk = Tgt::kEarly;  // does this proposal run early-rejection checks?
      if constexpr (Tgt::kPerProposalCheck) chk = !kc.no_early && Tgt::early_worth(kf, s, d, 4 * G);
      if (kBnd && chk && !bnd_ok) {
        if constexpr (Tgt::kPerProposalCheck) {
          // the bound from the lane's sums when they are known: no pass over the row
          bnd = x2 == x2 ? Tgt::bound_of_sums(kf, lane_coords(lane, d, nq), vs, x2) : bound_total(kf, lane, d, nq, xq);
        } else {
          bnd = bound_total(kf, lane, d, nq, xq);
        }
        bnd_ok = true;
      }
      const uint64_t base = (uint64_t)p * (uint64_t)d;
      if ((p % G) == 0) {  // lane l draws the uniform of proposal p + l
        const int pp = p + lane;
        u_pre = pp < nprop ? k.uniform((uint32_t)pp) : 1.0;
      }
      const double u = __shfl_sync(0xffffffffu, u_pre, gbase + (p % G));
      // log u on the SFU (|error| <= 1e-6 (1 + |log u|)); the fp64 log only when the
      // decision is that close (accept_decision): decisions equal log(u) < delta exactly
      const float log_u = sfu_lg2((float)u) * 0.693147180559945309f;
      bool rejected = false;
      float vs_new = 0.f;
      // checks after every quad-iteration up to the 7th (the test hook turns them off)
      // the first quad-iteration whose check can plausibly reject (checks are warp-uniform
      // and exact whichever ones run -- skipping one only draws more normals): for the
      // scale family the partial sum after c coordinates is ~ -tau s^2 c / 2 and the bound
      // of the rest tau X (1 - c / d) / 2 (X = sum x^2, from lane 0's carried sum): a check
      // is useless before c ~ X / (s^2 + X / d), 2 quad-iterations of slack
      // (G = 32 only: with several particles per warp the check -- a warp vote -- must
      // start at the same iteration for every group)
      int mfirst = kc.no_early ? kNoChecks : 0;
      if constexpr (Tgt::kBoundFromV && G == 32) {
        if (!kc.no_early) {
          const float X = __shfl_sync(0xffffffffu, vs, gbase) * (float)G;
          const float need = X / (4.f * (float)G * fmaf(s, s, X / (float)d));
          mfirst = max(0, (int)ceilf(need) - 2);
        }
      }
      float x2_new = 0.f;
#define ASMC_DELTA(A, C) \
  delta_pass<A, C>(kf, k, lane, d, nq, base, s, xq, xalt, log_u, bnd, vs, mfirst, rejected, vs_new, x2_new, drawn)
      float dl;
      if constexpr (Tgt::kPerProposalCheck) {
        if (chk) dl = aligned ? ASMC_DELTA(true, true) : ASMC_DELTA(false, true);
        else dl = aligned ? ASMC_DELTA(true, false) : ASMC_DELTA(false, false);
      } else {
        dl = aligned ? ASMC_DELTA(true, Tgt::kEarly) : ASMC_DELTA(false, Tgt::kEarly);
      }
#undef ASMC_DELTA
      if (rejected) continue;  // certainly rejected: the remaining normals are never drawn
      const double delta = group_sum<G>((double)dl);
      if (accept_decision(u, log_u, delta)) {  // kernel.cpp:35: accept iff log u < delta
        if constexpr (kDual) {  // the proposal is already in the spare row
          // only this particle's lanes take the branch (G < 32: other groups may reject)
          __syncwarp(G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gbase));
          float4* t = xq;
          xq = xalt;
          xalt = t;
          vs = vs_new;
          x2 = Tgt::kPerProposalCheck ? x2_new : x2_unknown;
          bnd_ok = false;
        } else {  // regenerate the proposal's normals
          const float nb = aligned ? accept_pass<true>(kf, k, lane, nq, base, s, xq)
                                   : accept_pass<false>(kf, k, lane, nq, base, s, xq);
          drawn += (uint32_t)((nq - lane + G - 1) / G);
          bnd = nb;
          bnd_ok = kBnd;
          vs = vsum(T, lane, d, xq);
          x2 = x2_unknown;
        }
      }
    }
  }  // kMove != kMoveSlice
  }

  // Elliptical slice w.r.t. eta (oracle/restate.c:slice_move; the one-lane fp32 form in
  // pass_kernel.cuh), G lanes per particle.  Sweep s draws nu ~ eta from normals
  // s d .. s d + d - 1 of the (particle, step) stream, then uniforms u (log y), theta and
  // one per bracket shrink, in that order -- the one-lane pass's stream order.  Each
  // candidate regenerates nu from the counter-based stream, writes x' (and its cached
  // vterm) to the spare row, and an accepted candidate flips the rows.  The shrink loop
  // runs warp-uniformly (G < 32 holds several particles per warp): a group that has
  // accepted idles until every group of the warp is done.
  __device__ static void slice(const TgtParams& T, const KernelCfg& kc, int lane, int d, double beta,
                               float4*& xq, float4*& xalt, const PhiloxKeyC& k, uint32_t& drawn, float& vs) {
    const int nq = (d + 3) >> 2;
    const typename Tgt::F32 kb = Tgt::f32(T, beta), k0 = Tgt::f32(T, 0.0);
    const float mu = (float)Tgt::ref_draw(T, 0.0);
    constexpr double kTwoPiS = 6.283185307179586476925286766559;
    uint32_t ku = 0;  // uniforms drawn from this (particle, step) stream
    for (int sw = 0; sw < kc.sweeps; ++sw) {
      const uint64_t base = (uint64_t)sw * (uint64_t)d;
      const double log_u = log(k.uniform(ku++));
      double theta = k.uniform(ku++) * kTwoPiS;
      double lo = theta - kTwoPiS, hi = theta;
      bool done = false;
      for (int it = 0; it < ASMC_SLICE_MAX_SHRINK; ++it) {
        if (__all_sync(0xffffffffu, done)) break;
        const float c = (float)cos(theta), sn = (float)sin(theta);
        float dl = 0.f;  // beta (V(x') - V(x)) as a difference of log-density differences
        for (int q = lane; q < nq; q += G) {
          if (done) break;
          ++drawn;
          float z[4];
          quad(k, base, q, z);
          const float4 x4 = xq[q];
          const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
          float xp[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (4 * q + e < d) {
              const float nu = (float)Tgt::ref_draw(T, (double)z[e]);
              xp[e] = mu + (xv[e] - mu) * c + (nu - mu) * sn;
              const float h = xp[e] - xv[e];
              dl += Tgt::dlg(kb, xv[e], h) - Tgt::dlg(k0, xv[e], h);
            } else {
              xp[e] = 0.f;
            }
          }
          const float4 xn = make_float4(xp[0], xp[1], xp[2], xp[3]);
          xalt[q] = xn;
          if constexpr (kCache) xalt[nq + q] = vquad(k0, xn);
        }
        const double delta = group_sum<G>((double)dl);
        const bool accept = !done && delta > log_u;
        __syncwarp();
        if (accept) {  // the candidate is the spare row: flip
          float4* t = xq;
          xq = xalt;
          xalt = t;
        }
        if (!done && !accept) {
          if (theta < 0.0) lo = theta;
          else hi = theta;
          theta = lo + (hi - lo) * k.uniform(ku++);
        }
        done = done || accept;
        __syncwarp();
      }
    }
    __syncwarp();
    vs = vsum(T, lane, d, xq);
  }

  // number of coordinates in this lane's quads (lane, lane + G, ...; the last quad may be partial)
  __device__ static int lane_coords(int lane, int d, int nq) {
    if (lane >= nq) return 0;
    const int mine = (nq - 1 - lane) / G + 1;
    return 4 * mine - (((nq - 1) % G == lane) ? 4 * nq - d : 0);
  }

  // sum of the early-rejection bound over this lane's coordinates (same order as delta_pass)
  __device__ static float bound_total(const typename Tgt::F32& kf, int lane, int d, int nq, const float4* xq) {
    float b = 0.f;
#pragma unroll 1
    for (int q = lane; q < nq; q += G) {
      const float4 x = xq[q];
      const float xv[4] = {x.x, x.y, x.z, x.w};
      float vv[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (kCache) {
        const float4 v = xq[nq + q];
        vv[0] = v.x; vv[1] = v.y; vv[2] = v.z; vv[3] = v.w;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < d) b += Tgt::dmax(kf, xv[e], vv[e]);
    }
    return b;
  }

  // one coordinate's leapfrog trajectory from (x, p); returns x', sets p'
  __device__ static float trajectory(const typename Tgt::F32& kf, float x, float p, float eps, int L,
                                     float& pend) {
    const float he = 0.5f * eps;
    float g = Tgt::grad32(kf, x);
    for (int l = 0; l < L; ++l) {
      p = fmaf(he, g, p);
      x = fmaf(eps, p, x);
      g = Tgt::grad32(kf, x);
      p = fmaf(he, g, p);
    }
    pend = p;
    return x;
  }

  // HMC over this lane's quads: kWrite = false -> energy difference
  // H(x,p0) - H(x',p'); kWrite = true -> store the accepted x' (and vterm)
  template <bool kAligned, bool kWrite>
  __device__ static float hmc_pass(const typename Tgt::F32& kf, const PhiloxKeyC& k, int lane, int d,
                                   int nq, uint64_t base, float eps, int L, float4* xq) {
    float dl = 0.f;
#pragma unroll 1
    for (int q = lane; q < nq; q += G) {
      float z[4];
      if (kAligned) k.template normals4<float>((uint32_t)(base >> 2) + (uint32_t)q, z);
      else k.template normals4_at<float>(base + 4 * (uint64_t)q, z);
      const float4 x4 = xq[q];
      float xv[4] = {x4.x, x4.y, x4.z, x4.w};
      float vv[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (kCache && !kWrite) {
        const float4 v = xq[nq + q];
        vv[0] = v.x; vv[1] = v.y; vv[2] = v.z; vv[3] = v.w;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!kAligned && 4 * q + e >= d) continue;
        float pend;
        const float xx = trajectory(kf, xv[e], z[e], eps, L, pend);
        if (kWrite) {
          xv[e] = xx;
        } else {
          float dlg;
          if constexpr (kCache) dlg = Tgt::dlg_cached(kf, xv[e], vv[e], xx);
          else dlg = Tgt::dlg(kf, xv[e], xx - xv[e]);
          dl += dlg + 0.5f * (z[e] - pend) * (z[e] + pend);
        }
      }
      if (kWrite) {
        const float4 xn = make_float4(xv[0], xv[1], xv[2], xv[3]);
        xq[q] = xn;
        if constexpr (kCache) xq[nq + q] = vquad(kf, xn);
      }
    }
    return dl;
  }

  // log u < delta, with log u from the SFU unless the two are within its error bound
  __device__ static bool accept_decision(double u, float log_u_sfu, double delta) {
    const double tol = 1e-5 * (1.0 + fabs((double)log_u_sfu));
    if (delta > (double)log_u_sfu + tol) return true;
    if (delta < (double)log_u_sfu - tol) return false;
    return log(u) < delta;
  }

  // is the proposal certainly rejected?  v = this lane's partial MH sum + the bound of its
  // unprocessed coordinates + a margin dominating the fp32 rounding of both sums
  // (1e-4 (|dl| + rem) per lane, plus 1e-2 against log u).
  //  G == 32 (one particle per warp): each lane's v rounded UP to a multiple of 2^-8
  //    (clamped below at -4096, which only raises it; values above 65536 become 2^17,
  //    which keeps the total positive), summed exactly by one REDUX: an upper bound of
  //    the real sum, warp-uniform, no shuffle chain.
  //  G < 32: an fp32 group butterfly and a warp vote (the exit must be warp-uniform).
  __device__ static bool certainly_rejected(float dl, float rem, float lu) {
    const float v = dl + rem + 1e-4f * (fabsf(dl) + rem);
    if constexpr (G == 32) {
      float c = fmaxf(v * 256.f, -0x1.0p20f);
      c = c > 0x1.0p24f ? 0x1.0p25f : c;
      const int S = __reduce_add_sync(0xffffffffu, __float2int_ru(c));
      return S < __float2int_ru((lu - 1e-2f) * 256.f);
    } else {
      const float sum = group_sumf<G>(v);
      return __all_sync(0xffffffffu, sum < lu - 1e-2f);
    }
  }

  // sum over this lane's quads of f_beta(x + s z) - f_beta(x), writing x + s z to the
  // spare row and its vpart sum to vs_new.  Early rejection (exact): after quad-iteration
  // m (m < 7 in Tgt::kCheckMask, m >= mfirst; kNoChecks = none) the warp checks
  //   partial + sum over unprocessed coordinates of max_h dlg  <  log u
  // (certainly_rejected); then the proposal is rejected whatever the remaining normals
  // are, so they are not drawn.  Accepted proposals see the identical sum.
  static constexpr int kLastCheck = 31 - __builtin_clz(Tgt::kCheckMask | 1u);  // last checked quad-iteration

  template <bool kAligned, bool kCheck>
  __device__ static float delta_pass(const typename Tgt::F32& kf, const PhiloxKeyC& k, int lane, int d, int nq,
                                     uint64_t base, float s, const float4* xq, float4* xalt, float log_u,
                                     float bnd, float vs, int mfirst, bool& rejected, float& vs_new,
                                     float& x2_new, uint32_t& drawn) {
    float dl = 0.f, bp = 0.f, vn = 0.f, x2n = 0.f;
    float sA = 0.f, sB = 0.f;  // Tgt::kQuadMH: sum z x, sum z^2 (dl = Tgt::dl_from(s, A, B))
    const float lu = log_u;
    const int mmax = (nq + G - 1) / G;
    int q = lane;
    // unrolled: the quad-iterations' Philox chains interleave (A/B on one box, config 2
    // (G = 32): 1x 2.75e8, 2x 2.84e8, 4x 2.87e8, 8x 2.47e8 p-steps/s -- the fully unrolled
    // loop leaves the instruction cache; config 3 (G = 4, mixture): 2x 8.92e8, 4x 8.78e8,
    // 8x 8.81e8), same registers
#pragma unroll (G == 4 ? 2 : 4)
    for (int m = 0; m < mmax; ++m, q += G) {
      if (q < nq) {
        ++drawn;
        float z[4];
        if (kAligned) k.template normals4<float>((uint32_t)(base >> 2) + (uint32_t)q, z);
        else k.template normals4_at<float>(base + 4 * (uint64_t)q, z);
        const float4 x = xq[q];
        const float xv[4] = {x.x, x.y, x.z, x.w};
        float xp[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) xp[e] = fmaf(s, z[e], xv[e]);
        if constexpr (kCache) {
          const float4 v = xq[nq + q];
          const float vv[4] = {v.x, v.y, v.z, v.w};
          float vp[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) vp[e] = Tgt::vterm(kf, xp[e]);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (kAligned || 4 * q + e < d) {
              dl += Tgt::dlg_vv(kf, xv[e], vv[e], xp[e], vp[e]);  // == dlg_cached
              if constexpr (Tgt::kPerProposalCheck) x2n = fmaf(xp[e], xp[e], x2n);
              if (kCheck && (kLastCheck >= 6 || m <= kLastCheck)) bp += Tgt::dmax(kf, xv[e], vv[e]);
              vn += vp[e];
            }
          if constexpr (kDual) xalt[nq + q] = make_float4(vp[0], vp[1], vp[2], vp[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (kAligned || 4 * q + e < d) {
              if constexpr (Tgt::kQuadMH) {
                sA = fmaf(z[e], xv[e], sA);
                sB = fmaf(z[e], z[e], sB);
              } else {
                dl += Tgt::dlg(kf, xv[e], s * z[e]);
              }
              if (kCheck && (kLastCheck >= 6 || m <= kLastCheck))
                bp += Tgt::kBoundFromV ? Tgt::vpart(kf, xv[e]) : Tgt::dmax(kf, xv[e], 0.f);
              vn += Tgt::vpart(kf, xp[e]);
            }
        }
        if constexpr (kDual) xalt[q] = make_float4(xp[0], xp[1], xp[2], xp[3]);
      }
      if constexpr (kCheck) {
        // warp-uniform: every lane runs mmax iterations
        if (((Tgt::kCheckMask >> m) & 1u) && m + 1 < mmax && m >= mfirst) {
          const float rem = Tgt::kBoundFromV ? Tgt::bound_of_v(kf, vs - bp) : bnd - bp;
          if constexpr (Tgt::kQuadMH) dl = Tgt::dl_from(kf, s, sA, sB);
          if (certainly_rejected(dl, rem, lu)) {
            rejected = true;
            return dl;
          }
        }
      }
    }
    vs_new = vn;
    x2_new = x2n;
    if constexpr (Tgt::kQuadMH) dl = Tgt::dl_from(kf, s, sA, sB);
    return dl;
  }

  template <bool kAligned>
  __device__ static float accept_pass(const typename Tgt::F32& kf, const PhiloxKeyC& k, int lane,
                                      int nq, uint64_t base, float s, float4* xq) {
    float b = 0.f;  // the new x's early-rejection bound (same order as bound_total)
#pragma unroll 1
    for (int q = lane; q < nq; q += G) {
      float z[4];
      if (kAligned) k.template normals4<float>((uint32_t)(base >> 2) + (uint32_t)q, z);
      else k.template normals4_at<float>(base + 4 * (uint64_t)q, z);
      float4 x = xq[q];
      x.x = fmaf(s, z[0], x.x);
      x.y = fmaf(s, z[1], x.y);
      x.z = fmaf(s, z[2], x.z);
      x.w = fmaf(s, z[3], x.w);
      xq[q] = x;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (kCache) {
        v = vquad(kf, x);
        xq[nq + q] = v;
      }
      if (Tgt::kEarly) {
        b += Tgt::dmax(kf, x.x, v.x);
        b += Tgt::dmax(kf, x.y, v.y);
        b += Tgt::dmax(kf, x.z, v.z);
        b += Tgt::dmax(kf, x.w, v.w);
      }
    }
    return b;
  }

};

// per-warp fold of this warp's groups for one (particle iteration, step), added
// into the warp's running accumulators acc[a] (lane 0 holds the result)
template <int G>
__device__ __forceinline__ void warp_fold(double lw_pre, double lg, double lw_post, bool active,
                                          int nacc, LogAcc* acc) {
  const int ln = threadIdx.x & 31;
  if (G == 32) {
    // one particle per warp: lane a owns accumulator a (no tree, no serial chain)
    // (lanes 0-4 share one signed add: lacc_add(l) == sacc_add(l, 1), one exp for all)
    if (ln < nacc && active) {
      LogAcc v = acc[ln];
      if (ln == kAccTop2) {
        top2_add(v, lw_post);
      } else {
        double l = ln == kAccG0 ? lw_pre : (ln == kAccG1 ? lw_pre + lg : lw_pre + 2.0 * lg);
        double sign = 1.0;
        if (ln == kAccSq) l = 2.0 * lw_post;
        if (ln == kAccElbo) {
          l = lg != 0.0 ? lw_pre + log_abs_sfu(lg) : -__builtin_huge_val();
          sign = lg > 0.0 ? 1.0 : -1.0;
        }
        sacc_add(v, l, sign);
      }
      acc[ln] = v;
    }
    return;
  }
  // G < 32: the warp holds 32/G particles.  Lane l of every group evaluates accumulator
  // a = a0 + l for its particle, the groups' values are combined by a max butterfly and
  // one exp per lane followed by a sum butterfly (every lane ends with the same bits),
  // and group 0's lane l merges the resulting (max, signed sum) into the warp's running
  // accumulator: 2 fp64 exps per accumulator row instead of one per tree level.
  const int l = ln % G;
  const int nlog = nacc > kAccTop2 ? kAccTop2 : nacc;  // log-sum accumulators (top-2 below)
  for (int a0 = 0; a0 < nlog; a0 += G) {
    const int a = a0 + l;
    double val = -__builtin_huge_val(), sign = 1.0;
    if (active && a < nlog) {
      val = a == kAccG0 ? lw_pre : (a == kAccG1 ? lw_pre + lg : lw_pre + 2.0 * lg);
      if (a == kAccSq) val = 2.0 * lw_post;
      if (a == kAccElbo) {
        val = lg != 0.0 ? lw_pre + log_abs_sfu(lg) : -__builtin_huge_val();
        sign = lg > 0.0 ? 1.0 : -1.0;
      }
    }
    double mx = val;
#pragma unroll
    for (int m = G; m < 32; m <<= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    double e = val == -__builtin_huge_val() ? 0.0 : sign * exp(val - mx);
#pragma unroll
    for (int m = G; m < 32; m <<= 1) e += __shfl_xor_sync(0xffffffffu, e, m);
    if (ln < G && a < nlog && mx != -__builtin_huge_val()) lacc_combine(acc[a], LogAcc{mx, e});
  }
  if (nacc > kAccTop2) {  // top-2 of the post-update log-weights (exact, order-free)
    LogAcc v{active ? lw_post : -__builtin_huge_val(), -__builtin_huge_val()};
#pragma unroll
    for (int m = G; m < 32; m <<= 1) top2_merge(v, shfl_xor_acc(v, m));
    if (ln == 0) top2_merge(acc[kAccTop2], v);
  }
}

// SMC step mode with several particles per warp (G < 32): each lane keeps ONE running
// accumulator in registers across the CTA's particle rounds -- lane l of a group owns
// accumulator l (g0, g1, g2, elbo), lane 0 also the sq and top-2 rows -- one exp per
// (particle, step) and no shuffles; the groups of a warp are combined once at the end
// (warp_regfold_finish).  Same sums as warp_fold, another fixed association.
struct RegFold {
  LogAcc acc, sq, top;
};
template <int G>
__device__ __forceinline__ void warp_regfold_add(double lw_pre, double lg, double lw_post, bool active,
                                                 RegFold& f) {
  const int l = (threadIdx.x & 31) % G;
  if (!active) return;
  // one signed add for every lane (sacc_add(l, 1) == lacc_add(l) bit for bit): a single
  // exp per warp instead of one per branch
  const double la = log_abs_sfu(lg);
  double val = l == kAccG0 ? lw_pre : (l == kAccG1 ? lw_pre + lg : lw_pre + 2.0 * lg), sg = 1.0;
  if (l == kAccElbo) {
    val = lg != 0.0 ? lw_pre + la : -__builtin_huge_val();
    sg = lg > 0.0 ? 1.0 : -1.0;
  }
  sacc_add(f.acc, val, sg);
  if (l == 0) {
    lacc_add(f.sq, 2.0 * lw_post);
    top2_add(f.top, lw_post);
  }
}
template <int G>
__device__ __forceinline__ void warp_regfold_finish(RegFold& f, int nacc, LogAcc* acc) {
  const int ln = threadIdx.x & 31, l = ln % G;
#pragma unroll
  for (int m = G; m < 32; m <<= 1) {
    lacc_combine(f.acc, shfl_xor_acc(f.acc, m));
    lacc_combine(f.sq, shfl_xor_acc(f.sq, m));
    top2_merge(f.top, shfl_xor_acc(f.top, m));
  }
  if (ln < G && l < 4) acc[l] = f.acc;
  if (ln == 0 && nacc > kAccSq) {
    acc[kAccSq] = f.sq;
    acc[kAccTop2] = f.top;
  }
}

template <class Tgt, int G, int kMove = kMoveRwmh>
// RWMH passes: <= 85 registers (3 CTAs/SM; the dual-row footprint allows no more at d = 1000)
// G = 4 RWMH on cached-potential targets: 4 rows per particle, so shared memory holds
// 2 CTAs/SM anyway and the registers may grow to 128 (the row prefetch below)
__global__ void __launch_bounds__(kBlock, kMove == kMoveHmc ? 4 : ((G == 4 && Tgt::kCacheV) ? 2 : 3))
    pass_smem_kernel(const __grid_constant__ PassArgs A) {
  constexpr int NG = kBlock / G;
  const int tid = threadIdx.x, g = tid / G, lane = tid % G, warp = tid >> 5;
  const int d = (int)A.tg.dim;
  const int nq = (d + 3) >> 2;
  const uint64_t blk = blockIdx.x;
  const int nacc = mode_nacc(A.mode);
  const bool loads = mode_loads(A.mode);
  if (block_err_set(A.err)) return;

  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool kHmc = kMove == kMoveHmc;
  constexpr int kWords = RowWords<Tgt, kHmc>::value;
  float4* xq = reinterpret_cast<float4*>(smem) + (size_t)g * nq * kWords;
  float4* xalt = xq + (size_t)nq * CacheWords<Tgt>::value;  // spare row (kDual only)
  LogAcc* wacc = reinterpret_cast<LogAcc*>(smem + (size_t)NG * nq * 16 * kWords);
  const int rows = A.t_end - A.t_begin + 1;
  LogAcc* myacc = wacc + (size_t)warp * rows * nacc;  // [row][a] of this warp
  if ((tid & 31) == 0)
    for (int i = 0; i < rows * nacc; ++i)
      myacc[i] = (i % nacc == kAccTop2) ? LogAcc{-__builtin_huge_val(), -__builtin_huge_val()}
                                         : lacc_empty();
  using Ops = SmemOps<Tgt, G, kMove>;
  // G < 32 SMC step: per-lane register accumulators (one step per launch)
  const bool regfold = G < 32 && A.mode == kModeSmcStep && rows == 1;
  RegFold rf{lacc_empty(), lacc_empty(), LogAcc{-__builtin_huge_val(), -__builtin_huge_val()}};
  uint32_t drawn = 0;  // quads of normals this lane generated (profiling)

  // SMC step, G = 4: the next round's particle row is loaded into registers while this
  // round's particle is processed, so its HBM latency is hidden behind the MH passes
  constexpr bool kPre = G == 4 && Tgt::kCacheV && !kHmc;
  constexpr int kPQ = kPre ? 8 : 1;  // quads per lane held (d <= 128)
  float4 pre[kPQ];
  const bool use_pre = kPre && loads && (d & 3) == 0 && nq <= G * kPQ;
  const bool pend = pass_pending(A);  // deferred gather: rows through anc, out to the other buffer
  auto load_pre = [&](uint64_t loc) {
    const bool act = loc < A.n_local;
    const uint64_t row = act ? (pend ? (uint64_t)A.anc[loc] : loc) : 0;
    const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(A.xbuf[*A.xcur]) +
                                                        row * (uint64_t)d);
#pragma unroll
    for (int i = 0; i < kPQ; ++i) {
      const int q = lane + G * i;
      if (q < nq) pre[i] = act ? src[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (use_pre) load_pre(blk * kBlock + (uint64_t)g);
  for (int r = 0; r < G; ++r) {
    const uint64_t local = blk * kBlock + (uint64_t)r * NG + g;
    const bool active = local < A.n_local;
    if (loads && !pend && tid == 0 && r + 1 < G) {
      // the next round's NG particle rows are one contiguous span of the state buffer:
      // one bulk L2 prefetch now, so their loads a particle-iteration later hit L2
      const uint64_t nl = blk * kBlock + (uint64_t)(r + 1) * NG;
      if (nl < A.n_local) {
        const uint64_t cnt = A.n_local - nl < (uint64_t)NG ? A.n_local - nl : (uint64_t)NG;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(
            reinterpret_cast<const float*>(A.xbuf[*A.xcur]) + nl * (uint64_t)d);
        const uintptr_t a1 = a0 + cnt * (uint64_t)d * sizeof(float);
        const uintptr_t lo = a0 & ~(uintptr_t)15, hi = (a1 + 15) & ~(uintptr_t)15;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
      }
    }
    const uint64_t pid = A.mode == kModeTraj ? (active ? A.pids[local] : 0) : A.p_begin + local;
    double lw = 0.0;
    float vs = 0.f;  // this lane's sum of vpart(x) (SmemOps::vsum)
    float x2 = __int_as_float(0x7fffffff);  // this lane's sum of x^2 if known (SmemOps::move)
    if (loads && use_pre) {
#pragma unroll
      for (int i = 0; i < kPQ; ++i) {
        const int q = lane + G * i;
        if (q < nq) xq[q] = pre[i];
      }
      if (r + 1 < G) load_pre(blk * kBlock + (uint64_t)(r + 1) * NG + g);
      lw = (active && !pend) ? A.lw[local] : 0.0;
      __syncwarp();
      vs = Ops::refresh_vx(A.tg, lane, d, xq, x2);  // the prefetch path is cached-target only
    } else if (loads) {
      const uint64_t row = (pend && active) ? (uint64_t)A.anc[local] : local;
      const float4* src = reinterpret_cast<const float4*>(
          reinterpret_cast<const float*>(A.xbuf[*A.xcur]) + row * (uint64_t)d);
      const bool vec = (d & 3) == 0;
      for (int q = lane; q < nq; q += G) {
        if (!active) {
          xq[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else if (vec) {
          xq[q] = src[q];
        } else {
          const float* s = reinterpret_cast<const float*>(src);
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = 4 * q + e < d ? s[4 * q + e] : 0.f;
          xq[q] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
      lw = (active && !pend) ? A.lw[local] : 0.0;
      __syncwarp();
      if constexpr (Tgt::kCacheV) vs = Ops::refresh_vx(A.tg, lane, d, xq, x2);
      else vs = Ops::vsum(A.tg, lane, d, xq);
    } else {
      PhiloxKeyC k;
      k.init(A.rk[0], pid, 0);
      vs = Ops::init(A.tg, lane, d, xq, k, drawn);
    }
    __syncwarp();
    if (A.mode == kModeSmcInit) {
      if (active) {
        float* dst = reinterpret_cast<float*>(A.xbuf[*A.xcur]) + local * (uint64_t)d;
        for (int q = lane; q < nq; q += G) {
          const float4 x = xq[q];
          const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (4 * q + e < d) dst[4 * q + e] = xv[e];
        }
        if (lane == 0) A.lw[local] = 0.0;
      }
      __syncwarp();
      continue;
    }
    if (A.mode == kModeTraj && active) {
      double* rx = A.rec_x + (local * (uint64_t)(A.T + 1)) * d;
      for (int i = lane; i < d; i += G) rx[i] = (double)reinterpret_cast<const float*>(xq)[i];
      if (lane == 0) A.rec_lw[local * (uint64_t)(A.T + 1)] = 0.0;
    }
    for (int t = A.t_begin; t <= A.t_end; ++t) {
      const double b0 = A.betas[t - 1], b1 = A.betas[t];
      const double lg = Ops::weight(A.tg, b0, b1, vs);
      PhiloxKeyC k;
      k.init(A.rk[1], pid, (uint64_t)t);
      __syncwarp();
      Ops::move(A.tg, A.kc, lane, d, b1, xq, xalt, k, drawn, vs, x2);
      __syncwarp();
      const double pre = lw;
      lw += lg;
      if (A.mode == kModeTraj) {
        if (active) {
          double* rx = A.rec_x + (local * (uint64_t)(A.T + 1) + t) * d;
          for (int i = lane; i < d; i += G) rx[i] = (double)reinterpret_cast<const float*>(xq)[i];
          if (lane == 0) A.rec_lw[local * (uint64_t)(A.T + 1) + t] = lw;
        }
        continue;
      }
      if (G < 32 && regfold) warp_regfold_add<G>(pre, lg, lw, active, rf);
      else warp_fold<G>(pre, lg, lw, active, nacc, myacc + (size_t)(t - A.t_begin) * nacc);
    }
    if (mode_stores(A.mode) && active) {
      float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(A.xbuf[*A.xcur ^ (pend ? 1 : 0)]) +
                                              local * (uint64_t)d);
      if ((d & 3) == 0) {
        for (int q = lane; q < nq; q += G) dst[q] = xq[q];
      } else {
        float* df = reinterpret_cast<float*>(dst);
        for (int i = lane; i < d; i += G) df[i] = reinterpret_cast<const float*>(xq)[i];
      }
      if (lane == 0) A.lw[local] = lw;
    }
    __syncwarp();
  }
  if (A.drawn) {  // profiling: normals generated by this warp (one atomic per warp)
    unsigned long long c = drawn;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((tid & 31) == 0) atomicAdd(A.drawn, 4ull * c);
  }
  if (A.mode == kModeTraj || A.mode == kModeSmcInit) return;
  if (G < 32 && regfold) warp_regfold_finish<G>(rf, nacc, myacc);
  __syncthreads();
  // block partial = warps folded in order (fixed tree)
  for (int i = tid; i < rows * nacc; i += blockDim.x) {
    const int row = i / nacc, a = i % nacc;
    LogAcc acc = wacc[(size_t)row * nacc + a];
    for (int w = 1; w < kWarps; ++w) acc_merge(a, acc, wacc[((size_t)w * rows + row) * nacc + a]);
    A.part[((size_t)(A.t_begin + row - A.row_base) * kNAcc + a) * A.part_stride + blk] = acc;
  }
}

}  // namespace asmcdev
