// Shared device definitions for the B200 SAIS/SSMC kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "asmc_b200.h"

namespace asmcdev {

constexpr int kBlock = 256;  // particles per reduction block (include/asmc/logsum.hpp:15)
constexpr int kNAcc = 6;     // per-step accumulators: g0, g1, g2, elbo, sq(2 log w), top-2 max
constexpr int kAccG0 = 0, kAccG1 = 1, kAccG2 = 2, kAccElbo = 3, kAccSq = 4, kAccTop2 = 5;
constexpr int kChunkBlocks = ASMC_FOLD_CHUNK / kBlock;  // 1024 blocks per fold chunk

struct LogAcc {
  double max;
  double sum;
};

__host__ __device__ __forceinline__ LogAcc lacc_empty() { return LogAcc{-__builtin_huge_val(), 0.0}; }

// LogAccumulator::add (include/asmc/logsum.hpp:20-28).  One exp whichever branch
// is taken (the branches differ only in the argument and the update), so lanes that
// disagree on the branch still share a single exp: the same bits as the reference's
// two-branch form.
__device__ __forceinline__ void lacc_add(LogAcc& a, double l) {
  if (l == -__builtin_huge_val()) return;
  const bool below = l <= a.max;
  const double e = exp(below ? l - a.max : a.max - l);
  if (below) {
    a.sum += e;
  } else {
    a.sum = a.sum * e + 1.0;
    a.max = l;
  }
}

// SignedLogAccumulator::add (logsum.hpp:55-63); sign = 1 gives lacc_add's bits
__device__ __forceinline__ void sacc_add(LogAcc& a, double log_abs, double sign) {
  if (log_abs == -__builtin_huge_val() || sign == 0.0) return;
  const bool below = log_abs <= a.max;
  const double e = exp(below ? log_abs - a.max : a.max - log_abs);
  if (below) {
    a.sum += sign * e;
  } else {
    a.sum = a.sum * e + sign;
    a.max = log_abs;
  }
}

// LogAccumulator::combine / SignedLogAccumulator::combine (logsum.hpp:30-38, 65-73).
// Both branches give the same bits for combine(a,b) and combine(b,a), so the
// xor-butterfly trees below leave every lane with the identical value.
__device__ __forceinline__ void lacc_combine(LogAcc& a, const LogAcc& o) {
  if (o.max == -__builtin_huge_val()) return;
  const bool below = o.max <= a.max;
  const double e = exp(below ? o.max - a.max : a.max - o.max);
  if (below) {
    a.sum += o.sum * e;
  } else {
    a.sum = a.sum * e + o.sum;
    a.max = o.max;
  }
}

// log|x| for the fp32 passes' ELBO accumulator (x = lg != 0, computed from fp32 potentials):
// the binary exponent exactly, the log2 of the [1, 2) significand on the SFU (absolute error
// < 2^-21), ~10 instructions instead of a full fp64 log -- the fp32 lg already carries ~1e-7
// relative error.  Subnormal x take the fp64 log.
__device__ __forceinline__ double log_abs_sfu(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x) & ~(1ull << 63);
  const int e = (int)(b >> 52) - 1023;
  if (e == -1023) return log(__longlong_as_double((long long)b));
  const float m = (float)__longlong_as_double((long long)((b & ((1ull << 52) - 1)) | (1023ull << 52)));
  float l2;
  asm("lg2.approx.f32 %0, %1;" : "=f"(l2) : "f"(m));
  return ((double)e + (double)l2) * 0.69314718055994530942;
}

// top-2 maxima as (max=m1, sum=m2); exact and order-free (engine_detail.hpp:130-154)
__device__ __forceinline__ void top2_add(LogAcc& a, double v) {
  if (v > a.max) {
    a.sum = a.max;
    a.max = v;
  } else if (v > a.sum) {
    a.sum = v;
  }
}
__device__ __forceinline__ void top2_merge(LogAcc& a, const LogAcc& b) {
  if (b.max > a.max) {
    a.sum = fmax(a.max, b.sum);
    a.max = b.max;
  } else {
    a.sum = fmax(a.sum, b.max);
  }
}

__device__ __forceinline__ void acc_merge(int a, LogAcc& x, const LogAcc& y) {
  if (a == kAccTop2) top2_merge(x, y);
  else lacc_combine(x, y);
}

__device__ __forceinline__ LogAcc shfl_xor_acc(const LogAcc& v, int m, unsigned mask = 0xffffffffu) {
  return LogAcc{__shfl_xor_sync(mask, v.max, m), __shfl_xor_sync(mask, v.sum, m)};
}

// Block-uniform read of the error word at kernel entry: thread 0 reads it and the CTA
// agrees.  A per-thread read could split a block when another CTA of the same launch
// raises the error meanwhile (e.g. a zero density in ExactT::weight), leaving the
// threads that stayed waiting at a barrier the others never reach.
__device__ __forceinline__ bool block_err_set(const int* err) {
  if (!err) return false;
  return __syncthreads_or(threadIdx.x == 0 ? *(volatile const int*)err : 0) != 0;
}

// Error word: the first failing particle records its code (ASMC_ERR_*).
__device__ __forceinline__ void raise_error(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

}  // namespace asmcdev
