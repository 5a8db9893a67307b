// Non-reversible parallel tempering (NRPT, src/pt.cpp:21-128) on the device:
// one CTA per run (replica r = seed0 + r), thread n = the chain at level n, the whole
// iteration loop in one launch.  Per iteration: level 0 takes a fresh reference
// draw (key (seed, round, 0, step, init)), levels n >= 1 one kernel application at
// beta_n (key (seed, round, n, step, explore)) -- the same one-lane move code as the
// SMC pass, so fp64 runs the reference's operation order --, V recorded
// (post-exploration, pre-swap), then the DEO swap phase: pairs (lo, lo+1) with
// lo = it mod 2, 4, ..., accepted iff log_alpha >= 0 or log u < log_alpha with u from
// key (seed, round, lo+1, step, swap).  Chains are exchanged through a per-run global
// scratch row (L1/L2-resident), so the level count is bounded by the CTA size only.
// Replicas fill the GPU: a 64-level run is two warps, 1000 replicas ~ 7 CTAs / SM.
#include <cuda_runtime.h>

#include "pass_kernel.cuh"
#include "pt.h"

#ifndef ASMC_PT_TGT
#error "compile pt_inst.cu with -DASMC_PT_TGT=0|1|2"
#endif

namespace asmcdev {

template <class Tgt, int RNG, typename Real, int KMAX>
__global__ void __launch_bounds__(kPtMaxLevels + 1) pt_kernel(PtArgs A) {
  const int n = threadIdx.x, L = A.levels, d = (int)A.tg.dim;
  const bool active = n <= L;
  const uint64_t seed = A.seed0 + blockIdx.x;
  Real* scratch = reinterpret_cast<Real*>(A.scratch) + (size_t)blockIdx.x * (L + 1) * d;
  double* trace = A.trace + (size_t)blockIdx.x * A.iterations * (L + 1);
  uint8_t* acc = A.accepted + (size_t)blockIdx.x * A.iterations * (L + 1);
  __shared__ double s_v[kPtMaxLevels + 1];
  __shared__ int s_swap[kPtMaxLevels + 1];
  using SeqD = typename std::conditional<RNG == ASMC_RNG_XOSHIRO, XoSeq<double>, PhSeq<double>>::type;
  using Ex = Exact<Tgt, SeqD, KMAX>;
  using Fs = Fast<Tgt, RNG, 1, KMAX>;
  Real x[KMAX], prop[KMAX];
  double V = 0.0;
  auto potential = [&]() {
    double v = 0.0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
    for (int k = 0; k < KMAX; ++k)
      if (k < d) v += Tgt::v64(A.tg, (double)x[k]);
    return v;
  };
  auto reference_draw = [&](uint64_t step) {  // pt.cpp:33-36, 50-55
    if constexpr (sizeof(Real) == 8) {
      SeqD st;
      st.init(seed, A.round, (uint64_t)n, step, 0);
      Ex::init(A.tg, d, reinterpret_cast<double*>(x), st);
    } else {
      typename Fs::Src src;
      src.init(seed, A.round, (uint64_t)n, step, 0);
      Fs::init(A.tg, 0, d, reinterpret_cast<float*>(x), src);
    }
  };
  if (active) {
    reference_draw(0);
    V = potential();
  }
  for (int it = 0; it < A.iterations; ++it) {
    const uint64_t step = (uint64_t)it + 1;
    if (active) {
      if (n == 0) {
        reference_draw(step);
      } else {  // pt.cpp:56-61: propagate at beta_n
        if constexpr (sizeof(Real) == 8) {
          SeqD st;
          st.init(seed, A.round, (uint64_t)n, step, 1);
          Ex::move(A.tg, A.kc, d, A.betas[n], reinterpret_cast<double*>(x), reinterpret_cast<double*>(prop), st);
        } else {
          typename Fs::Src src;
          src.init(seed, A.round, (uint64_t)n, step, 1);
          Fs::move(A.tg, A.kc, 0, d, A.betas[n], reinterpret_cast<float*>(x), src);
        }
      }
      V = potential();
      trace[(size_t)it * (L + 1) + n] = V;
      s_v[n] = V;
      s_swap[n] = 0;
#pragma unroll(KMAX <= 64 ? KMAX : 1)
      for (int k = 0; k < KMAX; ++k)
        if (k < d) scratch[(size_t)n * d + k] = x[k];
    }
    __syncthreads();
    // pt.cpp:66-81: DEO pairs; thread lo decides its pair
    const int first = it & 1;
    if (active && n >= first && ((n - first) & 1) == 0 && n + 1 <= L) {
      const int hi = n + 1;
      const double delta_beta = A.betas[hi] - A.betas[n];
      const double log_alpha = delta_beta * (s_v[n] - s_v[hi]);
      double u;
      if constexpr (RNG == ASMC_RNG_XOSHIRO) {
        XoStream xs;
        xs.init(seed, A.round, (uint64_t)hi, step, 3);
        u = xs.uniform();
      } else {
        PhiloxKey pk;
        pk.init(seed, A.round, (uint64_t)hi, step, 3);
        u = pk.uniform(0);
      }
      if (log_alpha >= 0.0 || log(u) < log_alpha) {
        s_swap[n] = 1;
        acc[(size_t)it * (L + 1) + n] = 1;
      }
    }
    __syncthreads();
    if (active) {
      const int partner = (n >= 1 && s_swap[n - 1]) ? n - 1 : (s_swap[n] ? n + 1 : -1);
      if (partner >= 0) {
#pragma unroll(KMAX <= 64 ? KMAX : 1)
        for (int k = 0; k < KMAX; ++k)
          if (k < d) x[k] = scratch[(size_t)partner * d + k];
        V = s_v[partner];
      }
    }
    __syncthreads();
  }
}

template <class Tgt>
static cudaError_t go_pt(const PtArgs& A, bool fp64, int rng, cudaStream_t s) {
  const unsigned threads = (unsigned)((A.levels + 1 + 31) / 32 * 32);
  const bool small = A.tg.dim <= 16;
#define PT_LAUNCH(RNG_, REAL_, KM_) pt_kernel<Tgt, RNG_, REAL_, KM_><<<A.replicas, threads, 0, s>>>(A)
  if (fp64) {
    if (rng == ASMC_RNG_XOSHIRO) {
      if (small) PT_LAUNCH(ASMC_RNG_XOSHIRO, double, 16);
      else PT_LAUNCH(ASMC_RNG_XOSHIRO, double, 1024);
    } else {
      if (small) PT_LAUNCH(ASMC_RNG_PHILOX, double, 16);
      else PT_LAUNCH(ASMC_RNG_PHILOX, double, 1024);
    }
  } else {
    if (rng == ASMC_RNG_XOSHIRO) {
      if (small) PT_LAUNCH(ASMC_RNG_XOSHIRO, float, 16);
      else PT_LAUNCH(ASMC_RNG_XOSHIRO, float, 1024);
    } else {
      if (small) PT_LAUNCH(ASMC_RNG_PHILOX, float, 16);
      else PT_LAUNCH(ASMC_RNG_PHILOX, float, 1024);
    }
  }
#undef PT_LAUNCH
  return cudaGetLastError();
}

#if ASMC_PT_TGT == 0
cudaError_t launch_pt_t0(const PtArgs& A, bool fp64, int rng, cudaStream_t s) { return go_pt<TgtGaussShift>(A, fp64, rng, s); }
#elif ASMC_PT_TGT == 1
cudaError_t launch_pt_t1(const PtArgs& A, bool fp64, int rng, cudaStream_t s) { return go_pt<TgtMixture>(A, fp64, rng, s); }
#else
cudaError_t launch_pt_t2(const PtArgs& A, bool fp64, int rng, cudaStream_t s) { return go_pt<TgtScale>(A, fp64, rng, s); }
#endif

}  // namespace asmcdev
