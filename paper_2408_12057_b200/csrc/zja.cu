// ZJA online schedule selection on the device (src/schedule.cpp:201-264).
//
// zja_next_beta picks the largest beta' in (beta, 1] whose one-step discrepancy
//   D(beta') = lse(lw + 2 lg) - 2 lse(lw + lg) + lse(lw),   lg = log gamma_beta'(x) - log gamma_beta(x),
// stays <= delta*, by bisection to 1e-10 plus a 16-point monotonicity scan: ~50
// probes per annealing step, each a log-sum-exp over all particles.  With log eta(x)
// and V(x) cached per particle (zja_eval_kernel, once per step) a probe reads 24 B
// per particle and never touches the particle state.
//
//  * exact (reference mode): one thread, sequential LogAccumulators in particle
//    order -- the reference's own accumulation order, so the probe values agree with
//    it to libm ulps and the bisection takes the same branches.
//  * cooperative (throughput mode): the whole search in ONE persistent cooperative
//    launch; per probe every CTA folds its strided particles (thread: sequential;
//    warp: xor butterfly; warps in order), writes its partial, one grid.sync(), then
//    every CTA folds the CTA partials in order and takes the same branch.  No host
//    round trip per probe; the per-particle arrays stay L2-resident across probes.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "zja.h"

namespace asmcdev {
namespace cg = cooperative_groups;

template <class Tgt, typename Real>
__global__ void zja_eval_kernel(TgtParams T, const void* const* xbuf, const int* xcur, uint64_t n,
                                double* lr, double* V, const int* err) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n || (err && *err)) return;
  const int d = (int)T.dim;
  const Real* x = reinterpret_cast<const Real*>(xbuf[*xcur]) + p * (uint64_t)d;
  double L = 0.0, v = 0.0;  // target.cpp:34-39: two ordered sums
  for (int k = 0; k < d; ++k) L += Tgt::lr64(T, (double)x[k]);
  for (int k = 0; k < d; ++k) v += Tgt::v64(T, (double)x[k]);
  lr[p] = L;
  V[p] = v;
}

// log_incremental_weight (kernel.cpp:65-73) from cached log eta and V
__device__ __forceinline__ double zja_lg(double lr, double V, double b2, double beta) {
  const double g2 = b2 == 0.0 ? lr : lr + b2 * V;
  const double g1 = beta == 0.0 ? lr : lr + beta * V;
  return g2 - g1;
}

__device__ __forceinline__ double lacc_log_total(const LogAcc& a) {
  return a.max == -__builtin_huge_val() ? -__builtin_huge_val() : a.max + log(a.sum);
}

// The search itself, shared by both modes: `dhat(b2)` and `lse_lw()` are the probes.
template <class Probe>
__device__ void zja_search(const ZjaArgs& A, Probe& P, double* out_beta, int* out_warn) {
  const double beta = A.betas[A.t - 1];
  const double delta = A.delta, tol = A.tol;
  *out_warn = 0;
  if (P.dhat(1.0) <= delta) {
    *out_beta = 1.0;
    return;
  }
  auto bisect = [&](double lo, double hi) {
    while (hi - lo > tol) {
      const double mid = 0.5 * (lo + hi);
      if (P.dhat(mid) <= delta) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  const double root = bisect(beta, 1.0);
  constexpr int kGridPoints = 16;  // schedule.cpp:254-261
  for (int i = 1; i < kGridPoints; ++i) {
    const double probe = beta + (root - beta) * (double)i / kGridPoints;
    if (P.dhat(probe) > delta * (1.0 + 1e-12)) {
      *out_beta = bisect(beta, probe);
      *out_warn = 1;
      return;
    }
  }
  *out_beta = root;
}

struct SeqProbe {
  const ZjaArgs& A;
  double beta, log_m0;
  __device__ double dhat(double b2) const {  // schedule.cpp:201-215
    LogAcc m1 = lacc_empty(), m2 = lacc_empty();
    for (uint64_t p = 0; p < A.n; ++p) {
      const double lg = zja_lg(A.lr[p], A.V[p], b2, beta);
      lacc_add(m1, A.lw[p] + lg);
      lacc_add(m2, A.lw[p] + 2.0 * lg);
    }
    const double raw = lacc_log_total(m2) - 2.0 * lacc_log_total(m1) + log_m0;
    return raw > 0.0 ? raw : 0.0;
  }
};

__global__ void zja_exact_kernel(ZjaArgs A) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || *A.err) return;
  LogAcc m0 = lacc_empty();  // logsumexp (logsum.hpp:97-101)
  for (uint64_t p = 0; p < A.n; ++p) lacc_add(m0, A.lw[p]);
  const double log_m0 = lacc_log_total(m0);
  if (log_m0 == -__builtin_huge_val()) {
    *A.err = ASMC_ERR_DEGENERATE;
    return;
  }
  SeqProbe P{A, A.betas[A.t - 1], log_m0};
  int warn = 0;
  double nb;
  zja_search(A, P, &nb, &warn);
  A.betas[A.t] = nb;
  if (warn) *A.warn = 1;
}

constexpr int kZjaThreads = 256;

struct GridProbe {
  const ZjaArgs& A;
  double beta, log_m0;
  int parity;
  double* s_w;    // [2 accumulators][8 warps] scratch
  double* s_out;  // unused (kept for the launch layout)

  // CTA-wide log-sum-exp of (max, sum) pairs in max-then-sum form: the CTA max by warp
  // shuffles (fmax, exact), then every thread rescales its sum with ONE exp and the sums
  // are added by a fixed tree (xor butterfly, warps in order).  Every thread receives the
  // totals; the same inputs give the same bits in every CTA.
  __device__ void cta_fold2(LogAcc& a, LogAcc& b) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NW = kZjaThreads / 32;
    double ma = a.max, mb = b.max;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      ma = fmax(ma, __shfl_xor_sync(0xffffffffu, ma, m));
      mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, m));
    }
    if (lane == 0) {
      s_w[w] = ma;
      s_w[NW + w] = mb;
    }
    __syncthreads();
    ma = s_w[0];
    mb = s_w[NW];
#pragma unroll
    for (int i = 1; i < NW; ++i) {
      ma = fmax(ma, s_w[i]);
      mb = fmax(mb, s_w[NW + i]);
    }
    __syncthreads();
    double sa = (a.max == -__builtin_huge_val()) ? 0.0 : a.sum * exp(a.max - ma);
    double sb = (b.max == -__builtin_huge_val()) ? 0.0 : b.sum * exp(b.max - mb);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, m);
      sb += __shfl_xor_sync(0xffffffffu, sb, m);
    }
    if (lane == 0) {
      s_w[w] = sa;
      s_w[NW + w] = sb;
    }
    __syncthreads();
    double ta = 0.0, tb = 0.0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      ta += s_w[i];
      tb += s_w[NW + i];
    }
    __syncthreads();
    a = LogAcc{ma, ta};
    b = LogAcc{mb, tb};
  }

  // fold (a, b) over the grid in a fixed order; every thread receives the totals
  __device__ void fold2(LogAcc a, LogAcc b, LogAcc& ta, LogAcc& tb) {
    cta_fold2(a, b);
    LogAcc* buf = A.part + (size_t)parity * 2 * gridDim.x;
    parity ^= 1;
    if (threadIdx.x == 0) {
      buf[blockIdx.x] = a;
      buf[gridDim.x + blockIdx.x] = b;
    }
    cg::this_grid().sync();
    // CTA partials: thread i folds partials i, i + 256, ... in order, then the CTA tree
    LogAcc x = lacc_empty(), y = lacc_empty();
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      lacc_combine(x, buf[i]);
      lacc_combine(y, buf[gridDim.x + i]);
    }
    cta_fold2(x, y);
    ta = x;
    tb = y;
  }

  // per thread: the max of its particles' terms first, then one exp per particle with
  // no dependence between them (the running-max form chains the exps)
  __device__ double dhat(double b2) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t p0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double m1 = -__builtin_huge_val(), m2 = -__builtin_huge_val();
    for (uint64_t p = p0; p < A.n; p += stride) {
      const double lg = (b2 - beta) * A.V[p];  // difference form of zja_lg
      m1 = fmax(m1, A.lw[p] + lg);
      m2 = fmax(m2, A.lw[p] + 2.0 * lg);
    }
    double s1 = 0.0, s2 = 0.0;
    if (m1 != -__builtin_huge_val()) {
      for (uint64_t p = p0; p < A.n; p += stride) {
        const double lg = (b2 - beta) * A.V[p];
        s1 += exp(A.lw[p] + lg - m1);
        s2 += exp(A.lw[p] + 2.0 * lg - m2);
      }
    }
    LogAcc t1, t2;
    fold2(LogAcc{m1, s1}, LogAcc{m2, s2}, t1, t2);
    const double raw = lacc_log_total(t2) - 2.0 * lacc_log_total(t1) + log_m0;
    return raw > 0.0 ? raw : 0.0;
  }
};

__global__ void __launch_bounds__(kZjaThreads) zja_coop_kernel(ZjaArgs A) {
  __shared__ double s_w[2 * (kZjaThreads / 32)];
  __shared__ double s_out[2];
  const int err0 = *(volatile int*)A.err;  // uniform across the grid (read before any write)
  if (err0) return;
  GridProbe P{A, A.betas[A.t - 1], 0.0, 0, s_w, s_out};
  LogAcc m0 = lacc_empty();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < A.n; p += stride) lacc_add(m0, A.lw[p]);
  LogAcc t0, unused;
  P.fold2(m0, lacc_empty(), t0, unused);
  P.log_m0 = lacc_log_total(t0);
  if (P.log_m0 == -__builtin_huge_val()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *A.err = ASMC_ERR_DEGENERATE;
    return;
  }
  double nb;
  int warn;
  zja_search(A, P, &nb, &warn);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    A.betas[A.t] = nb;
    if (warn) *A.warn = 1;
  }
}

cudaError_t launch_zja_eval(const TgtParams& T, bool fp64_state, const void* const* xbuf, const int* xcur,
                            uint64_t n, double* lr, double* V, const int* err, cudaStream_t s) {
  const unsigned g = (unsigned)((n + 127) / 128);
#define ZJA_EVAL(TG)                                                                            \
  (fp64_state ? (zja_eval_kernel<TG, double><<<g, 128, 0, s>>>(T, xbuf, xcur, n, lr, V, err), 0) \
              : (zja_eval_kernel<TG, float><<<g, 128, 0, s>>>(T, xbuf, xcur, n, lr, V, err), 0))
  switch (T.kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT: ZJA_EVAL(TgtGaussShift); break;
    case ASMC_TARGET_MIXTURE: ZJA_EVAL(TgtMixture); break;
    case ASMC_TARGET_SCALE_GAUSSIAN: ZJA_EVAL(TgtScale); break;
    default: return cudaErrorInvalidValue;
  }
#undef ZJA_EVAL
  return cudaGetLastError();
}

// Sharded probes (multi-GPU ZJA): per 256-particle block the pair (m1, m2) of
// dhat(b2) -- or, with b2 < 0, the log-sum-exp of the log-weights in m1 -- as a fixed
// tree (thread = particle, warp xor butterfly, warps in order), written to
// part[a * stride + blk] (a = 0: m1, a = 1: m2); the caller folds blocks into chunks.
__device__ __forceinline__ void zja_probe_body(const double* lw, const double* V, uint64_t n, double beta,
                                               double b2, LogAcc* part, uint64_t stride) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  LogAcc m1 = lacc_empty(), m2 = lacc_empty();
  if (p < n) {
    if (b2 < 0.0) {
      lacc_add(m1, lw[p]);
    } else {
      const double lg = (b2 - beta) * V[p];
      lacc_add(m1, lw[p] + lg);
      lacc_add(m2, lw[p] + 2.0 * lg);
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    lacc_combine(m1, shfl_xor_acc(m1, m));
    lacc_combine(m2, shfl_xor_acc(m2, m));
  }
  __shared__ LogAcc w[2][8];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  if (lane == 0) {
    w[0][wi] = m1;
    w[1][wi] = m2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    LogAcc a = lacc_empty();
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) lacc_combine(a, w[threadIdx.x][i]);
    part[(size_t)threadIdx.x * stride + blockIdx.x] = a;
  }
}

__global__ void zja_probe_blocks_kernel(const double* lw, const double* V, uint64_t n, double beta, double b2,
                                        LogAcc* part, uint64_t stride) {
  zja_probe_body(lw, V, n, beta, b2, part, stride);
}

cudaError_t launch_zja_probe_blocks(const double* lw, const double* V, uint64_t n, double beta, double b2,
                                    LogAcc* part, uint64_t stride, cudaStream_t s) {
  zja_probe_blocks_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lw, V, n, beta, b2, part, stride);
  return cudaGetLastError();
}

// ---- device-resident multi-GPU search: zja_search above as a resumable state machine
// whose probe point lives in HBM.  Every rank holds an identical ZjaSearch and advances
// it from the same all-gathered chunk partials, so the ranks stay in lock step with no
// host round trip per probe: probe (reads S->b2) -> all-gather -> step (folds in chunk
// order, takes the branch, writes the next S->b2).  Once done, further probes are no-ops.
enum : int { kZsM0 = 0, kZsTest1 = 1, kZsBisect = 2, kZsScan = 3, kZsFallback = 4, kZsDone = kZjaSearchDone };
constexpr int kZjaGridPoints = 16;  // schedule.cpp:254-261

__global__ void zja_search_init_kernel(ZjaSearch* S, const double* betas, int t, double delta, double tol) {
  ZjaSearch z{};
  z.beta = betas[t - 1];
  z.delta = delta;
  z.tol = tol;
  z.b2 = -1.0;
  z.chosen = z.beta;
  z.phase = kZsM0;
  *S = z;
}

__global__ void zja_probe_dev_kernel(const double* lw, const double* V, uint64_t n, const ZjaSearch* S,
                                     LogAcc* part, uint64_t stride) {
  const int phase = S->phase;  // block-uniform
  if (phase == kZsDone) return;
  zja_probe_body(lw, V, n, S->beta, phase == kZsM0 ? -1.0 : S->b2, part, stride);
}

// chunk-major (m1, m2) pairs: the exchange layout (all-gathered = chunk order over ranks)
__global__ void zja_interleave_kernel(const LogAcc* zchunk, uint64_t nch, const ZjaSearch* S, LogAcc* out) {
  if (S->phase == kZsDone) return;
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += (uint64_t)gridDim.x * blockDim.x) {
    out[2 * c] = zchunk[c];
    out[2 * c + 1] = zchunk[nch + c];
  }
}

__device__ __forceinline__ bool zs_bisect_next(ZjaSearch& z) {
  if (z.hi - z.lo > z.tol) {
    z.b2 = 0.5 * (z.lo + z.hi);
    return true;
  }
  return false;
}

__device__ __forceinline__ void zs_scan_point(ZjaSearch& z) {
  z.b2 = z.beta + (z.root - z.beta) * (double)z.scan_i / kZjaGridPoints;
}

__device__ __forceinline__ void zs_start_scan(ZjaSearch& z) {
  z.root = z.lo;
  z.phase = kZsScan;
  z.scan_i = 1;
  zs_scan_point(z);
}

__device__ __forceinline__ void zs_finish(ZjaSearch& z, double v) {
  z.chosen = v;
  z.phase = kZsDone;
}

__global__ void zja_search_step_kernel(ZjaSearch* S, const LogAcc* all, uint64_t nch, double* betas, int t,
                                       int* warn, int* err) {
  ZjaSearch z = *S;
  if (z.phase == kZsDone) return;
  LogAcc a = lacc_empty(), b = lacc_empty();
  for (uint64_t c = 0; c < nch; ++c) {  // chunk order: the same bits on every rank
    lacc_combine(a, all[2 * c]);
    lacc_combine(b, all[2 * c + 1]);
  }
  ++z.probes;
  if (z.phase == kZsM0) {  // logsumexp of the log-weights (drivers.cpp's log_m0)
    z.log_m0 = lacc_log_total(a);
    if (z.log_m0 == -__builtin_huge_val()) {
      *err = ASMC_ERR_DEGENERATE;
      z.phase = kZsDone;
    } else {
      z.phase = kZsTest1;
      z.b2 = 1.0;
    }
    *S = z;
    return;
  }
  const double raw = lacc_log_total(b) - 2.0 * lacc_log_total(a) + z.log_m0;  // schedule.cpp:201-215
  const double d = raw > 0.0 ? raw : 0.0;
  const double x = z.b2;  // the point just probed
  switch (z.phase) {
    case kZsTest1:
      if (d <= z.delta) {
        zs_finish(z, 1.0);
        break;
      }
      z.lo = z.beta;
      z.hi = 1.0;
      z.phase = kZsBisect;
      if (!zs_bisect_next(z)) zs_start_scan(z);
      break;
    case kZsBisect:
      if (d <= z.delta) z.lo = x;
      else z.hi = x;
      if (!zs_bisect_next(z)) zs_start_scan(z);
      break;
    case kZsScan:
      if (d > z.delta * (1.0 + 1e-12)) {  // non-monotone: bisect (beta, probe]
        z.warn = 1;
        z.lo = z.beta;
        z.hi = x;
        z.phase = kZsFallback;
        if (!zs_bisect_next(z)) zs_finish(z, z.lo);
      } else if (++z.scan_i < kZjaGridPoints) {
        zs_scan_point(z);
      } else {
        zs_finish(z, z.root);
      }
      break;
    case kZsFallback:
      if (d <= z.delta) z.lo = x;
      else z.hi = x;
      if (!zs_bisect_next(z)) zs_finish(z, z.lo);
      break;
    default:
      break;
  }
  if (z.phase == kZsDone) {
    betas[t] = z.chosen;
    if (z.warn && warn) *warn = 1;
  }
  *S = z;
}

cudaError_t launch_zja_search_init(ZjaSearch* S, const double* betas, int t, double delta, double tol,
                                   cudaStream_t s) {
  zja_search_init_kernel<<<1, 1, 0, s>>>(S, betas, t, delta, tol);
  return cudaGetLastError();
}

cudaError_t launch_zja_probe_dev(const double* lw, const double* V, uint64_t n, const ZjaSearch* S, LogAcc* part,
                                 uint64_t stride, cudaStream_t s) {
  zja_probe_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lw, V, n, S, part, stride);
  return cudaGetLastError();
}

cudaError_t launch_zja_interleave(const LogAcc* zchunk, uint64_t nch, const ZjaSearch* S, LogAcc* out,
                                  cudaStream_t s) {
  zja_interleave_kernel<<<(unsigned)((nch + 127) / 128), 128, 0, s>>>(zchunk, nch, S, out);
  return cudaGetLastError();
}

cudaError_t launch_zja_search_step(ZjaSearch* S, const LogAcc* all, uint64_t nch, double* betas, int t, int* warn,
                                   int* err, cudaStream_t s) {
  zja_search_step_kernel<<<1, 1, 0, s>>>(S, all, nch, betas, t, warn, err);
  return cudaGetLastError();
}

int zja_grid_blocks(int device) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, zja_coop_kernel, kZjaThreads, 0);
  if (per > 2) per = 2;  // 2 CTAs / SM saturate the L2 reads; fewer partials to fold
  return sms * (per > 0 ? per : 1);
}

cudaError_t launch_zja_next_beta(const ZjaArgs& A, int grid_blocks, cudaStream_t s) {
  if (A.exact) {
    zja_exact_kernel<<<1, 32, 0, s>>>(A);
    return cudaGetLastError();
  }
  ZjaArgs a = A;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((const void*)zja_coop_kernel, dim3(grid_blocks), dim3(kZjaThreads), args, 0,
                                     s);
}

}  // namespace asmcdev
