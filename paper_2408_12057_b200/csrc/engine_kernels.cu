// Reduction, estimator, resampling and schedule kernels.  Compiled with
// -fmad=false: the scalar fp64 code here (Fritsch-Carlson inversion, barrier
// sums, estimator bookkeeping) is the reference's IEEE operation sequence, so
// generate_schedule is bit-exact with the host oracle for given knots.
#include <cuda_runtime.h>

#include "engine_kernels.h"

namespace asmcdev {

constexpr double kNegInf = -__builtin_huge_val();
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------------ folds --
// Exact order (reference): acc = ((e . b0) . b1) . ... over all blocks
// (engine_detail.hpp:143-154, drivers.cpp:137-145).  One CTA per (row, acc).  As in the
// pass's exact fold, each combine needs only the running max before it (an exclusive
// prefix max of the partials' maxima, carried across tiles): the CTA scans it, computes
// every partial's exp in parallel (same argument -> same bits), and thread 0 replays the
// chain of adds in block order.  The top-2 row (no exps) is folded directly.
__global__ void __launch_bounds__(256) fold_exact_kernel(const LogAcc* part, uint64_t stride, uint64_t nblk,
                                                         int row0, int nacc, LogAcc* out) {
  constexpr int kTile = 1024, kPer = kTile / 256;
  const int row = row0 + blockIdx.x / nacc, a = blockIdx.x % nacc;
  const LogAcc* src = part + ((size_t)row * kNAcc + a) * stride;
  __shared__ LogAcc tile[kTile];
  __shared__ double e_s[kTile];
  __shared__ unsigned char f_s[kTile];  // 0 = skipped (empty partial), 1 = below, 2 = new max
  __shared__ double wmax[8];
  const int tid = threadIdx.x, ln = tid & 31, w = tid >> 5;
  LogAcc acc = (a == kAccTop2) ? LogAcc{kNegInf, kNegInf} : lacc_empty();
  double carried = kNegInf;  // running max after the previous tiles (all threads)
  for (uint64_t b0 = 0; b0 < nblk; b0 += kTile) {
    const int m = (int)umin64((uint64_t)kTile, (uint64_t)(nblk - b0));
    for (int i = tid; i < m; i += blockDim.x) tile[i] = src[b0 + i];
    __syncthreads();
    if (a == kAccTop2) {
      if (tid == 0)
        for (int i = 0; i < m; ++i) top2_merge(acc, tile[i]);
      __syncthreads();
      continue;
    }
    // thread t owns elements kPer t .. kPer t + kPer - 1 (in order)
    double loc = kNegInf;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int i = kPer * tid + e;
      if (i < m) loc = fmax(loc, tile[i].max);
    }
    double inc = loc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, inc, off);
      if (ln >= off) inc = fmax(inc, o);
    }
    if (ln == 31) wmax[w] = inc;
    __syncthreads();
    double pre = carried;
    for (int v = 0; v < w; ++v) pre = fmax(pre, wmax[v]);
    const double up = __shfl_up_sync(0xffffffffu, inc, 1);
    double run = ln == 0 ? pre : fmax(pre, up);  // running max before this thread's first element
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
      const int i = kPer * tid + e;
      if (i >= m) break;
      const double om = tile[i].max;
      if (om == kNegInf) {  // lacc_combine returns early
        f_s[i] = 0;
        continue;
      }
      const bool below = om <= run;
      e_s[i] = exp(below ? om - run : run - om);
      f_s[i] = below ? 1 : 2;
      run = fmax(run, om);
    }
    double tot = carried;
    for (int v = 0; v < 8; ++v) tot = fmax(tot, wmax[v]);
    __syncthreads();
    if (tid == 0) {
      for (int i = 0; i < m; ++i) {
        const unsigned char f = f_s[i];
        if (f == 0) continue;
        if (f == 1) {
          acc.sum += tile[i].sum * e_s[i];
        } else {
          acc.sum = acc.sum * e_s[i] + tile[i].sum;
          acc.max = tile[i].max;
        }
      }
    }
    carried = tot;
    __syncthreads();
  }
  if (tid == 0) out[(size_t)row * kNAcc + a] = acc;
}

// Fixed tree within a fold chunk of kChunkBlocks blocks: thread i folds blocks
// 4i..4i+3 in order, xor-butterfly across the warp, warps 0..7 in order.
__global__ void fold_chunk_kernel(const LogAcc* part, uint64_t stride, uint64_t nblk, int row0,
                                  int nacc, uint64_t nchunks, LogAcc* chunk_out) {
  const uint64_t c = blockIdx.x % nchunks;
  const int ra = (int)(blockIdx.x / nchunks);
  const int row = row0 + ra / nacc, a = ra % nacc;
  const LogAcc* src = part + ((size_t)row * kNAcc + a) * stride;
  const LogAcc empty = (a == kAccTop2) ? LogAcc{kNegInf, kNegInf} : lacc_empty();
  LogAcc acc = empty;
  const uint64_t b0 = c * kChunkBlocks + 4 * threadIdx.x;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (b0 + e < nblk) acc_merge(a, acc, src[b0 + e]);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc_merge(a, acc, shfl_xor_acc(acc, m));
  __shared__ LogAcc w[8];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    LogAcc t = empty;
    for (int i = 0; i < 8; ++i) acc_merge(a, t, w[i]);
    chunk_out[((size_t)row * kNAcc + a) * nchunks + c] = t;
  }
}

// Sequential over chunks (the exchange unit between GPUs).
__global__ void fold_chunks_final_kernel(const LogAcc* chunk, uint64_t nchunks, int row0,
                                         int nrows, int nacc, LogAcc* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows * nacc) return;
  const int row = row0 + i / nacc, a = i % nacc;
  const LogAcc* src = chunk + ((size_t)row * kNAcc + a) * nchunks;
  LogAcc acc = (a == kAccTop2) ? LogAcc{kNegInf, kNegInf} : lacc_empty();
  for (uint64_t c = 0; c < nchunks; ++c) acc_merge(a, acc, src[c]);
  out[(size_t)row * kNAcc + a] = acc;
}

__device__ __forceinline__ double lacc_total(const LogAcc& a) {
  return a.max == kNegInf ? kNegInf : a.max + log(a.sum);
}
__device__ __forceinline__ double sacc_value_scaled(const LogAcc& a, double log_scale) {
  if (a.max == kNegInf) return 0.0;
  return a.sum * exp(a.max - log_scale);
}
__device__ __forceinline__ double dhat_raw(double g0, double g1, double g2) {
  const double raw = g2 - 2.0 * g1 + g0;
  return raw > 0.0 ? raw : 0.0;  // schedule.cpp:27-31
}

// --------------------------------------------------------- SAIS report --
// drivers.cpp:148-176 + barrier_estimate (schedule.cpp:41-56).
__device__ void sais_report_body(const LogAcc* tot, int T, uint64_t n, RoundDev* rd) {
  const double log_n = log((double)n);
  rd->log_g0[0] = rd->log_g1[0] = rd->log_g2[0] = kNegInf;
  for (int t = 1; t <= T; ++t) {
    const LogAcc* r = tot + (size_t)t * kNAcc;
    rd->log_g0[t] = lacc_total(r[kAccG0]);
    rd->log_g1[t] = lacc_total(r[kAccG1]);
    rd->log_g2[t] = lacc_total(r[kAccG2]);
    if (rd->log_g1[t] == kNegInf && rd->state->err == 0) {
      rd->state->err = ASMC_ERR_DEGENERATE;
      rd->state->err_step = t;
    }
  }
  double elbo = 0.0, den_log = log_n;
  for (int t = 1; t <= T; ++t) {
    elbo += sacc_value_scaled(tot[(size_t)t * kNAcc + kAccElbo], den_log);
    den_log = rd->log_g1[t];
  }
  const double log_z = rd->log_g1[T] - log_n;
  for (int t = 0; t <= T; ++t) {
    rd->cum_log_z[t] = 0.0;
    rd->resampled[t] = 0;
  }
  rd->cum_log_z[T] = log_z;
  rd->scalars[0] = log_z;
  rd->scalars[1] = elbo;
  rd->lambda[0] = 0.0;
  for (int t = 1; t <= T; ++t)
    rd->lambda[t] = rd->lambda[t - 1] + sqrt(dhat_raw(rd->log_g0[t], rd->log_g1[t], rd->log_g2[t]));
}
__global__ void sais_report_kernel(const LogAcc* tot, int T, uint64_t n, RoundDev* rd) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  sais_report_body(tot, T, n, rd);
}
// batched seeds: CTA s reports seed s (tot rows s (T + 1) .. s (T + 1) + T, rd[s])
__global__ void sais_report_batch_kernel(const LogAcc* tot, int T, uint64_t n, RoundDev* rd) {
  if (threadIdx.x != 0) return;
  sais_report_body(tot + (size_t)blockIdx.x * (T + 1) * kNAcc, T, n, rd + blockIdx.x);
}

// ---------------------------------------------------------- SSMC decide --
__device__ uint64_t smc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// engine.cpp:132-182 for step t: statistics, ESS, degeneracy, ELBO, the
// resampling decision and the estimator update.  Draws the resampling
// uniform from key (seed, round, 0, t, resample) when ancestors are selected.
// T < 0: open-ended schedule (run_zja, drivers.cpp:300-336): step t is the last
// iff zja_betas[t] == 1.
__global__ void smc_decide_kernel(const LogAcc* tot, int t, int T_in, uint64_t n, int policy,
                                  double rho, uint64_t seed, uint64_t round, int rng,
                                  RoundDev* rd, const double* zja_betas) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  SmcState* st = rd->state;
  if (st->err) return;
  const int T = T_in >= 0 ? T_in : (zja_betas[t] == 1.0 ? t : 0x7fffffff);
  const double log_n = log((double)n);
  if (T_in < 0) rd->resampled[t] = 0;
  if (t == 1) {
    for (int i = 0; i <= (T_in >= 0 ? T : 0); ++i) {
      rd->log_g0[i] = rd->log_g1[i] = rd->log_g2[i] = kNegInf;
      rd->ess[i] = (double)n;
      rd->cum_log_z[i] = 0.0;
      rd->resampled[i] = 0;
    }
    st->log_z = 0.0;
    st->elbo = 0.0;
    st->acc_dhat = 0.0;
    st->den_log = log_n;
    st->n_resample = 0;
  }
  const LogAcc* r = tot;  // row of this step
  const double g0 = lacc_total(r[kAccG0]), g1 = lacc_total(r[kAccG1]), g2 = lacc_total(r[kAccG2]);
  rd->log_g0[t] = g0;
  rd->log_g1[t] = g1;
  rd->log_g2[t] = g2;
  st->resample_now = 0;
  if (g1 == kNegInf) {
    st->err = ASMC_ERR_DEGENERATE;
    st->err_step = t;
    return;
  }
  double ess_t = exp(2.0 * g1 - lacc_total(r[kAccSq]));
  ess_t = fmin((double)n, fmax(1.0, ess_t));
  rd->ess[t] = ess_t;
  // engine_detail.hpp:159-168
  const double m1 = r[kAccTop2].max, m2 = r[kAccTop2].sum;
  if (n > 1 && ess_t < 1.0 + 1e-9) {
    const double gap = (m2 == kNegInf) ? __builtin_huge_val() : m1 - m2;
    if (gap > 700.0) {
      st->err = ASMC_ERR_DEGENERATE + 100;  // "weights degenerate" message variant
      st->err_step = t;
      st->err_val = m1;
      return;
    }
  }
  st->elbo += sacc_value_scaled(r[kAccElbo], st->den_log);
  st->acc_dhat += dhat_raw(g0, g1, g2);
  bool fire = false;  // engine.cpp:82-95
  switch (policy) {
    case ASMC_POLICY_NEVER: fire = (t == T); break;
    case ASMC_POLICY_ALWAYS: fire = true; break;
    case ASMC_POLICY_ADAPTIVE_ESS: fire = ess_t < rho * (double)n; break;
    case ASMC_POLICY_STABILIZED: fire = st->acc_dhat > -log(rho); break;
  }
  const bool select = fire && policy != ASMC_POLICY_NEVER;
  if (t == T || fire) {
    st->log_z += g1 - log_n;
    if (select) {
      double u;
      if (rng == ASMC_RNG_XOSHIRO) {
        XoStream xs;
        xs.init(seed, round, 0, (uint64_t)t, 2);
        u = xs.uniform();
      } else {
        PhiloxKey pk;
        pk.init(seed, round, 0, (uint64_t)t, 2);
        u = pk.uniform(0);
      }
      st->u = u;
      st->max_lw = m1;
      st->resample_now = 1;
      rd->resampled[t] = 1;
    }
    st->den_log = log_n;
    st->acc_dhat = 0.0;
    rd->resample_times[st->n_resample++] = t;
  } else {
    st->den_log = g1;
  }
  rd->cum_log_z[t] = st->log_z;
  if (t == T) {
    rd->scalars[0] = st->log_z;
    rd->scalars[1] = st->elbo;
    rd->lambda[0] = 0.0;
    for (int i = 1; i <= T; ++i)
      rd->lambda[i] =
          rd->lambda[i - 1] + sqrt(dhat_raw(rd->log_g0[i], rd->log_g1[i], rd->log_g2[i]));
  }
}

// ------------------------------------------------------- resampling --
// Ancestors: refcdf.cu (the reference's sequential CDF, bit for bit).
// x_new[m] = x[a_m] (row copy, 16-byte vectors when the row allows), lw <- 0
// gated on `flag` (st->resample_now)
__global__ void gather_kernel(const uint32_t* anc, uint64_t n, uint64_t row_bytes,
                              void* const* xbuf, int* xcur, double* lw, const int* flag) {
  if (!*flag) return;
  const int cur = *xcur;
  const char* src = (const char*)xbuf[cur];
  char* dst = (char*)xbuf[cur ^ 1];
  const uint64_t vec = row_bytes / 16;
  if (row_bytes % 16 == 0) {
    const uint64_t total = n * vec;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t m = i / vec, v = i % vec;
      const uint4* s = (const uint4*)(src + (uint64_t)anc[m] * row_bytes) + v;
      ((uint4*)(dst + m * row_bytes))[v] = *s;
    }
  } else {
    const uint64_t w4 = row_bytes / 4, total = n * w4;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t m = i / w4, v = i % w4;
      ((uint32_t*)(dst + m * row_bytes))[v] = ((const uint32_t*)(src + (uint64_t)anc[m] * row_bytes))[v];
    }
  }
  for (uint64_t m = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n;
       m += (uint64_t)gridDim.x * blockDim.x)
    lw[m] = 0.0;
}

__global__ void flip_kernel(int* xcur, SmcState* st) {
  if (st->resample_now) *xcur ^= 1;
  st->resample_now = 0;
}

__global__ void defer_gather_kernel(SmcState* st) {
  if (st->resample_now) st->gather_pending = 1;
  st->resample_now = 0;
}

__global__ void settle_kernel(int* xcur, SmcState* st) {
  if (st->gather_pending) *xcur ^= 1;
  st->gather_pending = 0;
}

// ------------------------------------------------------------ schedule --
__device__ int upper_idx(const double* x, int n, double q) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = lo + (hi - lo) / 2;
    if (q < x[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo - 1;
}

// MonotoneCubic ctor (schedule.cpp:58-90); returns an ASMC_ERR code.
__device__ int mono_init(const double* x, const double* y, int n, double* m, double* h, double* d) {
  if (n < 2) return ASMC_ERR_INVALID_ARGUMENT;
  for (int i = 1; i < n; ++i)
    if (!(x[i] > x[i - 1])) return ASMC_ERR_INVALID_ARGUMENT;
  for (int i = 0; i + 1 < n; ++i) {
    h[i] = x[i + 1] - x[i];
    d[i] = (y[i + 1] - y[i]) / h[i];
  }
  m[0] = d[0];
  m[n - 1] = d[n - 2];
  for (int i = 1; i + 1 < n; ++i) {
    if (d[i - 1] == 0.0 || d[i] == 0.0 || (d[i - 1] > 0.0) != (d[i] > 0.0)) {
      m[i] = 0.0;
    } else {
      const double w1 = 2.0 * h[i] + h[i - 1];
      const double w2 = h[i] + 2.0 * h[i - 1];
      m[i] = (w1 + w2) / (w1 / d[i - 1] + w2 / d[i]);
    }
  }
  return 0;
}

// MonotoneCubic::eval (schedule.cpp:92-106)
__device__ double mono_eval(const double* x, const double* y, const double* m, int n, double q) {
  if (q <= x[0]) return y[0] + m[0] * (q - x[0]);
  if (q >= x[n - 1]) return y[n - 1] + m[n - 1] * (q - x[n - 1]);
  const int i = upper_idx(x, n, q);
  const double h = x[i + 1] - x[i];
  const double s = (q - x[i]) / h;
  const double s2 = s * s;
  const double s3 = s2 * s;
  const double h00 = 2.0 * s3 - 3.0 * s2 + 1.0;
  const double h10 = s3 - 2.0 * s2 + s;
  const double h01 = -2.0 * s3 + 3.0 * s2;
  const double h11 = s3 - s2;
  return h00 * y[i] + h10 * h * m[i] + h01 * y[i + 1] + h11 * h * m[i + 1];
}

// MonotoneCubic::derivative (schedule.cpp:108-117)
__device__ double mono_deriv(const double* x, const double* y, const double* m, int n, double q) {
  if (q <= x[0]) return m[0];
  if (q >= x[n - 1]) return m[n - 1];
  const int i = upper_idx(x, n, q);
  const double h = x[i + 1] - x[i];
  const double s = (q - x[i]) / h;
  const double s2 = s * s;
  const double g00 = (6.0 * s2 - 6.0 * s) / h;
  const double g10 = 3.0 * s2 - 4.0 * s + 1.0;
  const double g01 = (-6.0 * s2 + 6.0 * s) / h;
  const double g11 = 3.0 * s2 - 2.0 * s;
  return g00 * y[i] + g10 * m[i] + g01 * y[i + 1] + g11 * m[i + 1];
}

// schedule.cpp:121-141
__device__ int validate_barrier(const double* lambda, const double* beta, int n) {
  if (n < 2) return ASMC_ERR_INVALID_ARGUMENT;
  if (lambda[0] != 0.0) return ASMC_ERR_INVALID_ARGUMENT;
  if (beta[0] != 0.0 || beta[n - 1] != 1.0) return ASMC_ERR_INVALID_ARGUMENT;
  for (int i = 1; i < n; ++i) {
    if (lambda[i] < lambda[i - 1]) return ASMC_ERR_INVALID_ARGUMENT;
    if (!(beta[i] > beta[i - 1])) return ASMC_ERR_INVALID_ARGUMENT;
  }
  return 0;
}

// generate_schedule (schedule.cpp:144-187), one thread.  scratch: 5 * knots doubles.
__device__ void generate_schedule_body(const double* lambda, const double* beta, int knots,
                                       int t_new, double* out, double* scratch, int* err) {
  if (*err) return;
  int rc = validate_barrier(lambda, beta, knots);
  if (!rc && t_new < 1) rc = ASMC_ERR_INVALID_ARGUMENT;
  if (rc) {
    *err = rc;
    return;
  }
  const double total = lambda[knots - 1];
  double* xs = scratch;
  double* ys = scratch + knots;
  double* m = scratch + 2 * knots;
  double* h = scratch + 3 * knots;
  double* d = scratch + 4 * knots;
  int cnt = 0;
  bool uniform = total == 0.0;
  if (!uniform) {
    for (int i = 0; i < knots; ++i) {
      if (cnt > 0 && lambda[i] == xs[cnt - 1]) {
        ys[cnt - 1] = beta[i];
      } else {
        xs[cnt] = lambda[i];
        ys[cnt] = beta[i];
        ++cnt;
      }
    }
    if (cnt < 2) uniform = true;
  }
  if (uniform) {  // Schedule::uniform, engine.cpp:16-27
    for (int t = 0; t <= t_new; ++t) out[t] = (double)t / (double)t_new;
    out[0] = 0.0;
    out[t_new] = 1.0;
    return;
  }
  rc = mono_init(xs, ys, cnt, m, h, d);
  if (rc) {
    *err = rc;
    return;
  }
  out[0] = 0.0;
  out[t_new] = 1.0;
  for (int t = 1; t < t_new; ++t) {
    const double q = total * (double)t / (double)t_new;
    double b = mono_eval(xs, ys, m, cnt, q);
    b = fmin(1.0, fmax(0.0, b));
    out[t] = b;
  }
  for (int t = 1; t < t_new; ++t)
    if (out[t] <= out[t - 1]) out[t] = nextafter(out[t - 1], 1.0);
  for (int t = t_new - 1; t >= 1; --t)
    if (out[t] >= out[t + 1]) out[t] = nextafter(out[t + 1], 0.0);
  for (int t = 1; t <= t_new; ++t)
    if (!(out[t] > out[t - 1])) {
      *err = ASMC_ERR_INVALID_ARGUMENT;
      return;
    }
}

__global__ void generate_schedule_kernel(const double* lambda, const double* beta, int knots,
                                         int t_new, double* out, double* scratch, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  generate_schedule_body(lambda, beta, knots, t_new, out, scratch, err);
}
// batched seeds: CTA s regenerates seed s's grid (knots = T + 1 -> t_new + 1 betas), its
// own error word err[s]
__global__ void generate_schedule_batch_kernel(const double* lambda, uint64_t lam_stride, const double* beta,
                                               int knots, int t_new, double* out, double* scratch,
                                               int* err) {
  if (threadIdx.x != 0) return;
  const uint64_t s = blockIdx.x;
  generate_schedule_body(lambda + s * lam_stride, beta + s * knots, knots, t_new, out + s * (uint64_t)(t_new + 1),
                         scratch + s * 5 * (uint64_t)knots, err + s);
}

// local_barrier (schedule.cpp:189-197)
__global__ void local_barrier_kernel(const double* lambda, const double* beta, int knots,
                                     double* out, double* scratch, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int rc = validate_barrier(lambda, beta, knots);
  if (!rc) rc = mono_init(beta, lambda, knots, scratch, scratch + knots, scratch + 2 * knots);
  if (rc) {
    *err = rc;
    return;
  }
  for (int i = 0; i < knots; ++i) out[i] = mono_deriv(beta, lambda, scratch, knots, beta[i]);
}

// barrier_estimate (schedule.cpp:41-56)
__global__ void barrier_kernel(const double* g0, const double* g1, const double* g2, int T,
                               double* lambda, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  lambda[0] = 0.0;
  for (int t = 1; t <= T; ++t) {
    if (g0[t] == kNegInf) {
      *err = ASMC_ERR_INVALID_ARGUMENT;
      return;
    }
    lambda[t] = lambda[t - 1] + sqrt(dhat_raw(g0[t], g1[t], g2[t]));
  }
}

// ------------------------------------------------------------ rng hooks --
__global__ void rng_kernel(int rng, int what, int precision, uint64_t k0, uint64_t k1,
                           uint64_t k2, uint64_t k3, uint64_t k4, uint64_t count, void* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (rng == ASMC_RNG_XOSHIRO) {
    XoStream s;
    s.init(k0, k1, k2, k3, k4);
    for (uint64_t i = 0; i < count; ++i) {
      if (what == 0) ((uint64_t*)out)[i] = s.next_u64();
      else if (what == 1) ((double*)out)[i] = s.uniform();
      else ((double*)out)[i] = precision == ASMC_PREC_FP32 ? (double)(float)s.normal() : s.normal();
    }
  } else {
    PhiloxKey pk;
    pk.init(k0, k1, k2, k3, k4);
    for (uint64_t i = 0; i < count; ++i) {
      if (what == 0) ((uint64_t*)out)[i] = pk.u64((uint32_t)i);
      else if (what == 1) ((double*)out)[i] = pk.uniform((uint32_t)i);
      else {
        const uint32_t b = (uint32_t)(i >> 2);
        if (precision == ASMC_PREC_FP32) {
          float q[4];
          pk.normals4<float>(b, q);
          ((double*)out)[i] = (double)q[i & 3];
        } else {
          double q[4];
          pk.normals4<double>(b, q);
          ((double*)out)[i] = q[i & 3];
        }
      }
    }
  }
}

// ESS helper (engine.cpp:46-59): sequential LogAccumulators over the weights
__global__ void ess_kernel(const double* lw, uint64_t n, double* out, int* err) {
  __shared__ double tile[2048];
  LogAcc l1 = lacc_empty(), l2 = lacc_empty();
  for (uint64_t b0 = 0; b0 < n; b0 += 2048) {
    const int m = (int)umin64((uint64_t)(2048), (uint64_t)(n - b0));
    for (int i = threadIdx.x; i < m; i += blockDim.x) tile[i] = lw[b0 + i];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < m; ++i) {
        lacc_add(l1, tile[i]);
        lacc_add(l2, 2.0 * tile[i]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (lacc_total(l1) == kNegInf) {
      *err = ASMC_ERR_DEGENERATE;
      return;
    }
    const double e = exp(2.0 * lacc_total(l1) - lacc_total(l2));
    *out = fmin((double)n, fmax(1.0, e));
  }
}

// max of log-weights (exact; order-free)

// ============================================================ launchers ===
#define LAUNCH_OK() cudaGetLastError()

cudaError_t launch_fold(bool exact, const LogAcc* part, uint64_t stride, uint64_t nblk, int row0,
                        int nrows, int nacc, LogAcc* chunk_scratch, LogAcc* out, cudaStream_t s) {
  if (exact) {
    fold_exact_kernel<<<nrows * nacc, 256, 0, s>>>(part, stride, nblk, row0, nacc, out);
    return LAUNCH_OK();
  }
  const uint64_t nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  fold_chunk_kernel<<<(unsigned)(nrows * nacc * nchunks), 256, 0, s>>>(part, stride, nblk, row0,
                                                                         nacc, nchunks, chunk_scratch);
  cudaError_t e = LAUNCH_OK();
  if (e != cudaSuccess) return e;
  fold_chunks_final_kernel<<<(nrows * nacc + 127) / 128, 128, 0, s>>>(chunk_scratch, nchunks, row0,
                                                                       nrows, nacc, out);
  return LAUNCH_OK();
}

cudaError_t launch_fold_chunks(const LogAcc* part, uint64_t stride, uint64_t nblk, int row0,
                               int nrows, int nacc, uint64_t nchunks, LogAcc* chunk_out,
                               cudaStream_t s) {
  fold_chunk_kernel<<<(unsigned)(nrows * nacc * nchunks), 256, 0, s>>>(part, stride, nblk, row0,
                                                                         nacc, nchunks, chunk_out);
  return LAUNCH_OK();
}

cudaError_t launch_fold_chunks_final(const LogAcc* chunk, uint64_t nchunks, int row0, int nrows,
                                     int nacc, LogAcc* out, cudaStream_t s) {
  fold_chunks_final_kernel<<<(nrows * nacc + 127) / 128, 128, 0, s>>>(chunk, nchunks, row0, nrows,
                                                                       nacc, out);
  return LAUNCH_OK();
}

cudaError_t launch_sais_report(const LogAcc* tot, int T, uint64_t n, RoundDev* rd, cudaStream_t s) {
  sais_report_kernel<<<1, 1, 0, s>>>(tot, T, n, rd);
  return LAUNCH_OK();
}

cudaError_t launch_smc_decide(const LogAcc* tot_row, int t, int T, uint64_t n, int policy,
                              double rho, uint64_t seed, uint64_t round, int rng, RoundDev* rd,
                              cudaStream_t s, const double* zja_betas) {
  smc_decide_kernel<<<1, 1, 0, s>>>(tot_row, t, T, n, policy, rho, seed, round, rng, rd, zja_betas);
  return LAUNCH_OK();
}

cudaError_t launch_gather(const uint32_t* anc, uint64_t n, uint64_t row_bytes, void* const* xbuf,
                          int* xcur, double* lw, SmcState* st, int sms, cudaStream_t s) {
  gather_kernel<<<sms * 8, 256, 0, s>>>(anc, n, row_bytes, xbuf, xcur, lw, &st->resample_now);
  cudaError_t e = LAUNCH_OK();
  if (e != cudaSuccess) return e;
  flip_kernel<<<1, 1, 0, s>>>(xcur, st);
  return LAUNCH_OK();
}

cudaError_t launch_defer_gather(SmcState* st, cudaStream_t s) {
  defer_gather_kernel<<<1, 1, 0, s>>>(st);
  return LAUNCH_OK();
}

cudaError_t launch_settle(int* xcur, SmcState* st, cudaStream_t s) {
  settle_kernel<<<1, 1, 0, s>>>(xcur, st);
  return LAUNCH_OK();
}


cudaError_t launch_generate_schedule(const double* lambda, const double* beta, int knots, int t_new,
                                     double* out, double* scratch, int* err, cudaStream_t s) {
  generate_schedule_kernel<<<1, 1, 0, s>>>(lambda, beta, knots, t_new, out, scratch, err);
  return LAUNCH_OK();
}

cudaError_t launch_sais_report_batch(const LogAcc* tot, int T, uint64_t n, RoundDev* rd, int nseeds,
                                     cudaStream_t s) {
  sais_report_batch_kernel<<<nseeds, 1, 0, s>>>(tot, T, n, rd);
  return LAUNCH_OK();
}

cudaError_t launch_generate_schedule_batch(const double* lambda, uint64_t lam_stride, const double* beta, int knots,
                                           int t_new, double* out, double* scratch, int* err, int nseeds,
                                           cudaStream_t s) {
  generate_schedule_batch_kernel<<<nseeds, 1, 0, s>>>(lambda, lam_stride, beta, knots, t_new, out, scratch, err);
  return LAUNCH_OK();
}

cudaError_t launch_local_barrier(const double* lambda, const double* beta, int knots, double* out,
                                 double* scratch, int* err, cudaStream_t s) {
  local_barrier_kernel<<<1, 1, 0, s>>>(lambda, beta, knots, out, scratch, err);
  return LAUNCH_OK();
}

cudaError_t launch_barrier(const double* g0, const double* g1, const double* g2, int T,
                           double* lambda, int* err, cudaStream_t s) {
  barrier_kernel<<<1, 1, 0, s>>>(g0, g1, g2, T, lambda, err);
  return LAUNCH_OK();
}

cudaError_t launch_rng(int rng, int what, int precision, const uint64_t key[5], uint64_t count,
                       void* out, cudaStream_t s) {
  rng_kernel<<<1, 1, 0, s>>>(rng, what, precision, key[0], key[1], key[2], key[3], key[4], count, out);
  return LAUNCH_OK();
}

cudaError_t launch_ess(const double* lw, uint64_t n, double* out, int* err, cudaStream_t s) {
  ess_kernel<<<1, 1024, 0, s>>>(lw, n, out, err);
  return LAUNCH_OK();
}

// ------------------------------------------------------ sharded SSMC --
// Exchange layout of the per-step fold partials: chunk-major [c][kNAcc], so the
// rank-ordered concatenation of every shard's chunks is the global chunk order.
__global__ void chunk_major_kernel(const LogAcc* in, uint64_t nch, LogAcc* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch * kNAcc) return;
  const uint64_t c = i / kNAcc;
  const int a = (int)(i % kNAcc);
  out[i] = in[(size_t)a * nch + c];
}

// Same merge sequence as fold_chunks_final_kernel (chunks 0..C-1 from empty):
// the all-gathered partials fold to the single-GPU totals bit for bit.
__global__ void fold_chunk_major_kernel(const LogAcc* in, uint64_t nch, LogAcc* tot) {
  const int a = threadIdx.x;
  if (a >= kNAcc) return;
  LogAcc acc = (a == kAccTop2) ? LogAcc{kNegInf, kNegInf} : lacc_empty();
  for (uint64_t c = 0; c < nch; ++c) acc_merge(a, acc, in[c * kNAcc + a]);
  tot[a] = acc;
}

// Output slot m lands in shard r iff its ancestor does: a_m is non-decreasing in m, so
// shard r's slots are [first m with a_m >= p_r, first m with a_m >= p_{r+1}).
__global__ void slot_bounds_kernel(const uint32_t* anc, uint64_t n, const uint64_t* shard_p, int world,
                                   const SmcState* st, uint64_t* slot_begin) {
  const int r = threadIdx.x;
  if (r > world || !st->resample_now) return;
  const uint64_t p = shard_p[r];
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((uint64_t)anc[mid] < p) lo = mid + 1;
    else hi = mid;
  }
  slot_begin[r] = r == world ? n : lo;
}

// rows of global ancestors anc[0..count) (this shard starts at particle p0), slot order
__global__ void pack_rows_kernel(const uint32_t* anc, uint64_t count, uint64_t p0, uint64_t row_bytes,
                                 const char* src, char* dst) {
  if (row_bytes % 16 == 0) {
    const uint64_t vec = row_bytes / 16, total = count * vec;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t m = i / vec, v = i % vec;
      ((uint4*)(dst + m * row_bytes))[v] = ((const uint4*)(src + ((uint64_t)anc[m] - p0) * row_bytes))[v];
    }
  } else {
    const uint64_t w4 = row_bytes / 4, total = count * w4;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t m = i / w4, v = i % w4;
      ((uint32_t*)(dst + m * row_bytes))[v] = ((const uint32_t*)(src + ((uint64_t)anc[m] - p0) * row_bytes))[v];
    }
  }
}

// SAIS chunk partials between the fold layout chunk[(t * kNAcc + a) * nch + c] and the
// exchange layout x[(c * (T + 1) + t) * 4 + a] (include/asmc_b200.h, asmc_sais_partials),
// on the device (multi-GPU SAIS keeps its partials out of host memory)
__global__ void chunks_to_exchange_kernel(const LogAcc* chunk, uint64_t nch, int T, LogAcc* x) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch * (uint64_t)(T + 1) * 4) return;
  const int a = (int)(i % 4), t = (int)((i / 4) % (T + 1));
  const uint64_t c = i / (4 * (uint64_t)(T + 1));
  x[i] = t == 0 ? LogAcc{kNegInf, 0.0} : chunk[((size_t)t * kNAcc + a) * nch + c];
}
__global__ void exchange_to_chunks_kernel(const LogAcc* x, uint64_t nch, int T, LogAcc* chunk) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch * (uint64_t)(T + 1) * kNAcc) return;
  const uint64_t c = i % nch;
  const int a = (int)((i / nch) % kNAcc), t = (int)(i / (nch * kNAcc));
  chunk[i] = (t == 0 || a >= 4) ? LogAcc{kNegInf, 0.0} : x[(c * (uint64_t)(T + 1) + t) * 4 + a];
}
cudaError_t launch_chunks_to_exchange(const LogAcc* chunk, uint64_t nch, int T, LogAcc* x, cudaStream_t s) {
  const uint64_t n = nch * (uint64_t)(T + 1) * 4;
  chunks_to_exchange_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(chunk, nch, T, x);
  return LAUNCH_OK();
}
cudaError_t launch_exchange_to_chunks(const LogAcc* x, uint64_t nch, int T, LogAcc* chunk, cudaStream_t s) {
  const uint64_t n = nch * (uint64_t)(T + 1) * kNAcc;
  exchange_to_chunks_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, nch, T, chunk);
  return LAUNCH_OK();
}

cudaError_t launch_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* out, cudaStream_t s) {
  const uint64_t n = nch * kNAcc;
  chunk_major_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(in, nch, out);
  return LAUNCH_OK();
}

cudaError_t launch_fold_chunk_major(const LogAcc* in, uint64_t nch, LogAcc* tot, cudaStream_t s) {
  fold_chunk_major_kernel<<<1, 32, 0, s>>>(in, nch, tot);
  return LAUNCH_OK();
}

cudaError_t launch_slot_bounds(const uint32_t* anc, uint64_t n, const uint64_t* shard_p, int world,
                               const SmcState* st, uint64_t* slot_begin, cudaStream_t s) {
  slot_bounds_kernel<<<1, 1024, 0, s>>>(anc, n, shard_p, world, st, slot_begin);
  return LAUNCH_OK();
}

cudaError_t launch_pack_rows(const uint32_t* anc, uint64_t count, uint64_t p0, uint64_t row_bytes, const void* x,
                             void* dst, int sms, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  pack_rows_kernel<<<sms * 8, 256, 0, s>>>(anc, count, p0, row_bytes, (const char*)x, (char*)dst);
  return LAUNCH_OK();
}

}  // namespace asmcdev
