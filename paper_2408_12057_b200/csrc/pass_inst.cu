// One (precision, target) slice of the particle-pass instantiations; the
// Makefile compiles this file six times (-DASMC_PREC=64|32 -DASMC_TGT=0|1|2)
// so the heavy template instantiations build in parallel.  The fp64 slices
// are compiled with -fmad=false (reference operation order, no contraction).
#include "dispatch.h"
#include "pass_smem.cuh"

#ifndef ASMC_PREC
#error "ASMC_PREC must be 64 or 32"
#endif
#ifndef ASMC_TGT
#error "ASMC_TGT must be a target kind"
#endif

namespace asmcdev {

#if ASMC_TGT == ASMC_TARGET_GAUSSIAN_SHIFT
using Tgt = TgtGaussShift;
#elif ASMC_TGT == ASMC_TARGET_MIXTURE
using Tgt = TgtMixture;
#elif ASMC_TGT == ASMC_TARGET_SCALE_GAUSSIAN
using Tgt = TgtScale;
#endif

template <int RNG, typename Real, int G, int K>
static cudaError_t go(const PassArgs& A, uint64_t blocks, cudaStream_t s) {
  pass_kernel<Tgt, RNG, Real, G, K><<<(unsigned)blocks, kBlock, 0, s>>>(A);
  return cudaGetLastError();
}

#if ASMC_PREC == 32
template <int G, int kMove>
static cudaError_t go_smem_k(const PassArgs& A, uint64_t blocks, cudaStream_t s) {
  const int nacc = mode_nacc(A.mode);
  const int rows = A.t_end - A.t_begin + 1 > 0 ? A.t_end - A.t_begin + 1 : 1;
  const size_t bytes = smem_pass_bytes(G, A.tg.dim, rows - 1, nacc, RowWords<Tgt, kMove == kMoveHmc>::value);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(pass_smem_kernel<Tgt, G, kMove>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  PassArgs Ak = A;
  philox_round_keys(A.seed, A.round, 0, Ak.rk[0]);
  philox_round_keys(A.seed, A.round, 1, Ak.rk[1]);
  pass_smem_kernel<Tgt, G, kMove><<<(unsigned)blocks, kBlock, bytes, s>>>(Ak);
  return cudaGetLastError();
}
// HMC gets its own instantiation so the RWMH pass keeps its lean register allocation
template <int G>
static cudaError_t go_smem(const PassArgs& A, uint64_t blocks, cudaStream_t s) {
  if (A.kc.kind == ASMC_KERNEL_HMC) return go_smem_k<G, kMoveHmc>(A, blocks, s);
  if (A.kc.kind == ASMC_KERNEL_SLICE) return go_smem_k<G, kMoveSlice>(A, blocks, s);
  return go_smem_k<G, kMoveRwmh>(A, blocks, s);
}
#endif

#define CAT_(a, b, c) a##b##_##c
#define CAT(a, b, c) CAT_(a, b, c)

cudaError_t CAT(launch_pass_fp, ASMC_PREC, ASMC_TGT)(int rng, Layout L, const PassArgs& A,
                                                     uint64_t blocks, cudaStream_t s) {
#if ASMC_PREC == 64
  if (L.lanes != 1) return cudaErrorInvalidValue;
  if (rng == ASMC_RNG_XOSHIRO) {
    if (L.kmax == 16) return go<ASMC_RNG_XOSHIRO, double, 1, 16>(A, blocks, s);
    if (L.kmax == 1024) return go<ASMC_RNG_XOSHIRO, double, 1, 1024>(A, blocks, s);
  } else {
    if (L.kmax == 16) return go<ASMC_RNG_PHILOX, double, 1, 16>(A, blocks, s);
    if (L.kmax == 1024) return go<ASMC_RNG_PHILOX, double, 1, 1024>(A, blocks, s);
  }
#else
  if (rng == ASMC_RNG_XOSHIRO) {
    if (L.lanes != 1) return cudaErrorInvalidValue;
    if (L.kmax == 16) return go<ASMC_RNG_XOSHIRO, float, 1, 16>(A, blocks, s);
    if (L.kmax == 1024) return go<ASMC_RNG_XOSHIRO, float, 1, 1024>(A, blocks, s);
    return cudaErrorInvalidValue;
  }
  if (L.lanes == 1 && L.kmax == 16) return go<ASMC_RNG_PHILOX, float, 1, 16>(A, blocks, s);
  if (L.lanes == 1 && L.kmax == 1024) return go<ASMC_RNG_PHILOX, float, 1, 1024>(A, blocks, s);
  if (L.lanes == 4) return go_smem<4>(A, blocks, s);
  if (L.lanes == 32) return go_smem<32>(A, blocks, s);
#endif
  return cudaErrorInvalidValue;
}

}  // namespace asmcdev
