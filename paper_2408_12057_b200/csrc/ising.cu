// Config 5: relaxed Ising model on an L x L torus, one CTA
// per particle, the lattice in registers + shared memory, RWMH or HMC moves.
//
// Relaxation (Hubbard-Stratonovich, written in the y = A^{-1} x parametrisation so
// both the log density and its gradient are 5-point stencils):
//   A = delta I + K (Adj + 4 I)           (positive definite; c = delta + 4K on the diagonal)
//   u = A y
//   log p~(y) = sum_i [ -y_i u_i / 2 + log 2cosh(u_i) ]        (marginal of the spins)
//   eta = N(0, sigma^2 I),  V = log p~ - log eta
//   grad log gamma_beta = beta A (tanh(u) - y) - (1 - beta) y / sigma^2
// and Z(1) = (2 pi)^{n/2} |A|^{-1/2} e^{c n / 2} Z_Ising(K) in closed form (Kaufman).
//
// Lattice -> threads: coordinate i = a L + b.  Thread t owns column block
// b in [b0, b0 + R) of row a = t mod L (R = L / 4, b0 = (t / L) R, 4L threads), so its
// coordinates are contiguous (4-aligned Philox normal blocks) and its b-neighbours are
// in registers.  Shared memory holds the lattice transposed, S[b L + a], so the
// a-neighbour loads of a warp (consecutive a) are conflict-free.  Per gradient:
// write y, sync, u = c y + K nb(y), v = tanh(u) - y, write v, sync, g = c v + K nb(v).
// RNG (Philox shadow stream, as every fp32 path): init = normals j of stream
// (p, 0, init); move trajectory q (sweep-major over step sizes) = normals q n + j of
// stream (p, t, explore) and uniform q.  Energies: fp32 per-thread partials over R
// sites, fp64 fixed-tree block sums; MH in difference form.
#include <cuda_runtime.h>

#include "ising.h"

namespace asmcdev {

__device__ __forceinline__ float log2cosh_f(float u) {
  const float a = fabsf(u);
  return a + __logf(1.0f + __expf(-2.0f * a));
}

// tanh u = 1 - 2 / (e^{2u} + 1) on the SFU (ex2 + rcp); saturates correctly without a
// clamp: e^{2u} -> inf gives 1, e^{2u} -> 0 gives -1.
__device__ __forceinline__ float sfu_ex2(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float sfu_rcp(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float tanh_f(float u) {
  return fmaf(-2.0f, sfu_rcp(sfu_ex2(2.8853900817779268f * u) + 1.0f), 1.0f);  // 2 log2(e) u
}
// tanh u - y in one FFMA after the SFU pair
__device__ __forceinline__ float tanh_minus(float u, float y) {
  return fmaf(-2.0f, sfu_rcp(sfu_ex2(2.8853900817779268f * u) + 1.0f), 1.0f - y);
}

template <int L>
struct IsCta {
  static constexpr int NT = 4 * L, R = L / 4, N = L * L, NW = NT / 32;
  float* Sy;
  float* Sv;
  float* S0;
  double* red;
  int a, b0;
  float K, c;

  __device__ __forceinline__ float nb(const float* S, const float (&v)[R], int r) const {
    const int b = b0 + r;
    const float up = S[b * L + ((a + L - 1) & (L - 1))];
    const float dn = S[b * L + ((a + 1) & (L - 1))];
    const float lf = r > 0 ? v[r > 0 ? r - 1 : 0] : S[((b0 + L - 1) & (L - 1)) * L + a];
    const float rt = r < R - 1 ? v[r < R - 1 ? r + 1 : 0] : S[((b0 + R) & (L - 1)) * L + a];
    return (up + dn) + (lf + rt);
  }

  __device__ __forceinline__ void put(float* S, const float (&v)[R]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) S[(b0 + r) * L + a] = v[r];
  }

  __device__ __forceinline__ void get(const float* S, float (&v)[R]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = S[(b0 + r) * L + a];
  }

  // partial sums over the owned sites: e = sum(-y u / 2 + log 2cosh u), yy = sum y^2
  __device__ __forceinline__ void energy(const float (&y)[R], float& e, float& yy) const {
    put(Sy, y);
    __syncthreads();
    e = 0.f;
    yy = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float u = c * y[r] + K * nb(Sy, y, r);
      e += -0.5f * y[r] * u + log2cosh_f(u);
      yy += y[r] * y[r];
    }
  }

  // gradient of log gamma_beta at y, applied as p += kick * grad; energy partials at y
  // only when kEnergy (the trajectory's end point)
  template <bool kEnergy>
  __device__ __forceinline__ void grad_kick(const float (&y)[R], float (&p)[R], float beta, float inv_s2,
                                            float kick, float& e, float& yy) const {
    float v[R];
    put(Sy, y);
    __syncthreads();
    if (kEnergy) {
      e = 0.f;
      yy = 0.f;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float u = c * y[r] + K * nb(Sy, y, r);
      if (kEnergy) {
        e += -0.5f * y[r] * u + log2cosh_f(u);
        yy += y[r] * y[r];
      }
      v[r] = tanh_f(u) - y[r];
    }
    put(Sv, v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float g = c * v[r] + K * nb(Sv, v, r);
      p[r] += kick * (beta * g - (1.0f - beta) * inv_s2 * y[r]);
    }
  }

  // fixed-tree block sums (xor butterfly, warps in order); every thread gets the totals
  template <int M>
  __device__ __forceinline__ void block_sum(double (&v)[M]) const {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < M; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], m);
      if (lane == 0) red[w * M + k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double s = 0.0;
      for (int i = 0; i < NW; ++i) s += red[i * M + k];
      v[k] = s;
    }
    __syncthreads();
  }
};

template <int R>
__device__ __forceinline__ void normals_run(const PhiloxKey& k, uint64_t j0, float (&out)[R]) {
  if constexpr (R % 4 == 0) {
#pragma unroll
    for (int i = 0; i < R / 4; ++i) {
      float q[4];
      k.normals4<float>((uint32_t)(j0 >> 2) + i, q);
#pragma unroll
      for (int e = 0; e < 4; ++e) out[4 * i + e] = q[e];
    }
  } else {
    float q[4];
    k.normals4_at<float>(j0, q);
#pragma unroll
    for (int e = 0; e < R; ++e) out[e] = q[e];
  }
}

template <int L>
__global__ void __launch_bounds__(4 * L, L == 64 ? 3 : 4) is_move_kernel(const IsArgs A, int mode, const double* betas, int t) {
  using Cta = IsCta<L>;
  constexpr int R = Cta::R, N = Cta::N;
  extern __shared__ float is_smem[];
  if (block_err_set(A.err)) return;
  Cta C;
  C.Sy = is_smem;
  C.Sv = is_smem + N;
  C.S0 = is_smem + 2 * N;
  C.red = reinterpret_cast<double*>(is_smem + 3 * N);
  C.a = threadIdx.x % L;
  C.b0 = (threadIdx.x / L) * R;
  C.K = A.K;
  C.c = A.c;
  const uint64_t local = blockIdx.x;
  const uint64_t pid = A.p_begin + local;
  const int j0 = C.a * L + C.b0;  // first owned coordinate
  float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
  float y[R];
  if (mode == 0) {  // sample_reference: y = sigma z
    PhiloxKey ki;
    ki.init(A.seed, A.round, pid, 0, 0);
    normals_run<R>(ki, (uint64_t)j0, y);
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] *= A.sigma;
  } else if constexpr (R % 4 == 0) {  // 16-byte loads: 4x fewer LSU wavefronts than scalars
#pragma unroll
    for (int r = 0; r < R; r += 4) {
      const float4 q = *reinterpret_cast<const float4*>(row + j0 + r);
      y[r] = q.x;
      y[r + 1] = q.y;
      y[r + 2] = q.z;
      y[r + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) y[r] = row[j0 + r];
  }
  float e_p, yy_p;
  C.energy(y, e_p, yy_p);
  double cur[2] = {(double)e_p, (double)yy_p};
  C.template block_sum<2>(cur);
  double ecur = cur[0], yycur = cur[1];

  if (mode == 1 && A.kc.kind != ASMC_KERNEL_IDENTITY) {
    const double beta = betas[t];
    const float bf = (float)beta;
    PhiloxKey kx;
    kx.init(A.seed, A.round, pid, (uint64_t)t, 1);
    const bool hmc = A.kc.kind == ASMC_KERNEL_HMC;
    uint32_t q = 0;
    for (int sw = 0; sw < A.kc.sweeps; ++sw) {
      for (int si = 0; si < A.kc.n_steps; ++si, ++q) {
        const float eps = (float)A.kc.steps[si];
        C.put(C.S0, y);  // own slots only: no barrier needed to read them back
        float z[R];
        normals_run<R>(kx, (uint64_t)q * N + j0, z);
        double dlg;
        double s4[4];
        if (!hmc) {  // kernel.cpp:31-40: x' = x + s xi, accept iff log u < lg(x') - lg(x)
#pragma unroll
          for (int r = 0; r < R; ++r) y[r] += eps * z[r];
          float e1, yy1;
          C.energy(y, e1, yy1);
          double s2[2] = {(double)e1, (double)yy1};
          C.template block_sum<2>(s2);
          s4[0] = s2[0];
          s4[1] = s2[1];
          dlg = beta * (s4[0] - ecur) - (1.0 - beta) * 0.5 * (double)A.inv_s2 * (s4[1] - yycur);
        } else {  // leapfrog, unit mass, kick-drift-kick with the inner kicks merged
          float k0 = 0.f;
#pragma unroll
          for (int r = 0; r < R; ++r) k0 += z[r] * z[r];
          float e1 = 0.f, yy1 = 0.f;
          C.template grad_kick<false>(y, z, bf, A.inv_s2, 0.5f * eps, e1, yy1);
          for (int l = 0; l + 1 < A.kc.leapfrog; ++l) {
#pragma unroll
            for (int r = 0; r < R; ++r) y[r] += eps * z[r];
            C.template grad_kick<false>(y, z, bf, A.inv_s2, eps, e1, yy1);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) y[r] += eps * z[r];
          C.template grad_kick<true>(y, z, bf, A.inv_s2, 0.5f * eps, e1, yy1);
          float k1 = 0.f;
#pragma unroll
          for (int r = 0; r < R; ++r) k1 += z[r] * z[r];
          double s[4] = {(double)e1, (double)yy1, (double)k0, (double)k1};
          C.template block_sum<4>(s);
          s4[0] = s[0];
          s4[1] = s[1];
          dlg = beta * (s4[0] - ecur) - (1.0 - beta) * 0.5 * (double)A.inv_s2 * (s4[1] - yycur) +
                0.5 * (s[2] - s[3]);
        }
        const double log_u = log(kx.uniform(q));
        if (log_u < dlg) {
          ecur = s4[0];
          yycur = s4[1];
        } else {
          C.get(C.S0, y);
        }
      }
    }
  }
  if constexpr (R % 4 == 0) {
#pragma unroll
    for (int r = 0; r < R; r += 4) *reinterpret_cast<float4*>(row + j0 + r) = make_float4(y[r], y[r + 1], y[r + 2], y[r + 3]);
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) row[j0 + r] = y[r];
  }
  if (threadIdx.x == 0)
    *reinterpret_cast<double*>(row + N) = ecur + 0.5 * (double)A.inv_s2 * yycur + A.vconst;
}

// ---------------------------------------------------------------------------
// 4 x 4 register tiles (L = 32, 64): thread t owns sites a in [4 ta, 4 ta + 4),
// b in [4 tb, 4 tb + 4) (ta = t / TPR, tb = t % TPR, TPR = L / 4 tiles per tile row,
// L^2 / 16 threads).  A stencil needs only the tile's halo: the left / right columns
// come from the neighbouring tiles of the same tile row by warp shuffles (a tile row
// is TPR <= 16 consecutive lanes, the torus wrap stays inside it); the up / down rows
// from the neighbouring tile rows through shared memory, where each tile publishes
// its top and bottom rows as one 16-byte store each.  Per stencil and 16 sites:
// 2 STS.128 + 2 LDS.128 + 8 SHFL and one barrier (edge buffers alternate, so the next
// stencil's stores never race this one's loads) -- the row layout above needs ~100
// shared-memory accesses for the same 16 sites.  Coordinates, Philox normals
// (row i of the tile = one 4-aligned normal block) and the HBM row layout are the
// row kernel's; only the fp32 summation order of the per-thread partials differs.
template <int L>
struct IsTile {
  static constexpr int TPR = L / 4, NT = L * L / 16, N = L * L, NW = NT / 32, TA = L / 4;
  float4* E;  // edge buffers [2][2 (top, bottom)][TA][TPR]
  float4* Y0;  // [NT][4]: the pre-proposal tile (own slots)
  double* red;
  int ta, tb, buf;
  float K, c;

  // nb[i][k] = sum of the four torus neighbours of site (4ta+i, 4tb+k) of field f
  __device__ __forceinline__ void neighbours(const float (&f)[4][4], float (&nb)[4][4]) {
    float4* Eb = E + (size_t)buf * 2 * TA * TPR;
    Eb[ta * TPR + tb] = make_float4(f[0][0], f[0][1], f[0][2], f[0][3]);            // top row
    Eb[(TA + ta) * TPR + tb] = make_float4(f[3][0], f[3][1], f[3][2], f[3][3]);     // bottom row
    float lf[4], rt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      lf[i] = __shfl_sync(0xffffffffu, f[i][3], (tb + TPR - 1) & (TPR - 1), TPR);
      rt[i] = __shfl_sync(0xffffffffu, f[i][0], (tb + 1) & (TPR - 1), TPR);
    }
    __syncthreads();
    const float4 up = Eb[(TA + ((ta + TA - 1) & (TA - 1))) * TPR + tb];  // bottom row of the tile above
    const float4 dn = Eb[((ta + 1) & (TA - 1)) * TPR + tb];               // top row of the tile below
    buf ^= 1;
    const float upv[4] = {up.x, up.y, up.z, up.w}, dnv[4] = {dn.x, dn.y, dn.z, dn.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float u = i > 0 ? f[i > 0 ? i - 1 : 0][k] : upv[k];
        const float d = i < 3 ? f[i < 3 ? i + 1 : 0][k] : dnv[k];
        const float l = k > 0 ? f[i][k > 0 ? k - 1 : 0] : lf[i];
        const float r = k < 3 ? f[i][k < 3 ? k + 1 : 0] : rt[i];
        nb[i][k] = (u + d) + (l + r);
      }
  }

  __device__ __forceinline__ void energy(const float (&y)[4][4], float& e, float& yy) {
    float nb[4][4];
    neighbours(y, nb);
    e = 0.f;
    yy = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float u = c * y[i][k] + K * nb[i][k];
        e += -0.5f * y[i][k] * u + log2cosh_f(u);
        yy += y[i][k] * y[i][k];
      }
  }

  // p += kick (beta A (tanh(Ay) - y) - (1 - beta) y / s^2), with the constants folded:
  // p = kbc v + kbK nb(v) - ky y + p  (three FFMAs per site)
  template <bool kEnergy>
  __device__ __forceinline__ void grad_kick(const float (&y)[4][4], float (&p)[4][4], float beta, float inv_s2,
                                            float kick, float& e, float& yy) {
    float nb[4][4], v[4][4];
    neighbours(y, nb);
    if (kEnergy) {
      e = 0.f;
      yy = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float u = fmaf(K, nb[i][k], c * y[i][k]);
        if (kEnergy) {
          e += -0.5f * y[i][k] * u + log2cosh_f(u);
          yy += y[i][k] * y[i][k];
        }
        v[i][k] = tanh_minus(u, y[i][k]);
      }
    neighbours(v, nb);
    const float kb = kick * beta, kbc = kb * c, kbK = kb * K, ky = kick * (1.0f - beta) * inv_s2;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) p[i][k] = fmaf(kbc, v[i][k], fmaf(kbK, nb[i][k], fmaf(-ky, y[i][k], p[i][k])));
  }

  template <int M>
  __device__ __forceinline__ void block_sum(double (&v)[M]) const {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < M; ++k) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], m);
      if (lane == 0) red[w * M + k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double s = 0.0;
      for (int i = 0; i < NW; ++i) s += red[i * M + k];
      v[k] = s;
    }
    __syncthreads();
  }

  __device__ __forceinline__ void save(const float (&y)[4][4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) Y0[threadIdx.x * 4 + i] = make_float4(y[i][0], y[i][1], y[i][2], y[i][3]);
  }
  __device__ __forceinline__ void restore(float (&y)[4][4]) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 q = Y0[threadIdx.x * 4 + i];
      y[i][0] = q.x; y[i][1] = q.y; y[i][2] = q.z; y[i][3] = q.w;
    }
  }
};

// normals j0 .. j0+3 (j0 4-aligned) of a Philox stream into one tile row
__device__ __forceinline__ void normals_row(const PhiloxKey& k, uint64_t j0, float (&out)[4]) {
  k.normals4<float>((uint32_t)(j0 >> 2), out);
}

template <int L>
__global__ void __launch_bounds__(L * L / 16, L == 64 ? 3 : 8) is_tile_kernel(const IsArgs A, int mode,
                                                                              const double* betas, int t) {
  using Cta = IsTile<L>;
  constexpr int N = Cta::N;
  extern __shared__ float4 is_tsmem[];
  if (block_err_set(A.err)) return;
  Cta C;
  C.E = is_tsmem;
  C.Y0 = is_tsmem + 4 * Cta::TA * Cta::TPR;
  C.red = reinterpret_cast<double*>(C.Y0 + 4 * Cta::NT);
  C.ta = threadIdx.x / Cta::TPR;
  C.tb = threadIdx.x % Cta::TPR;
  C.buf = 0;
  C.K = A.K;
  C.c = A.c;
  const uint64_t local = blockIdx.x;
  const uint64_t pid = A.p_begin + local;
  const int j0 = 4 * C.ta * L + 4 * C.tb;  // first owned coordinate; row i starts at j0 + i L
  float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
  float y[4][4];
  if (mode == 0) {  // sample_reference: y = sigma z
    PhiloxKey ki;
    ki.init(A.seed, A.round, pid, 0, 0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      normals_row(ki, (uint64_t)(j0 + i * L), y[i]);
#pragma unroll
      for (int k = 0; k < 4; ++k) y[i][k] *= A.sigma;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 q = *reinterpret_cast<const float4*>(row + j0 + i * L);
      y[i][0] = q.x; y[i][1] = q.y; y[i][2] = q.z; y[i][3] = q.w;
    }
  }
  float e_p, yy_p;
  C.energy(y, e_p, yy_p);
  double cur[2] = {(double)e_p, (double)yy_p};
  C.template block_sum<2>(cur);
  double ecur = cur[0], yycur = cur[1];

  if (mode == 1 && A.kc.kind != ASMC_KERNEL_IDENTITY) {
    const double beta = betas[t];
    const float bf = (float)beta;
    PhiloxKey kx;
    kx.init(A.seed, A.round, pid, (uint64_t)t, 1);
    const bool hmc = A.kc.kind == ASMC_KERNEL_HMC;
    uint32_t q = 0;
    for (int sw = 0; sw < A.kc.sweeps; ++sw) {
      for (int si = 0; si < A.kc.n_steps; ++si, ++q) {
        const float eps = (float)A.kc.steps[si];
        C.save(y);  // own slots only: no barrier needed to read them back
        float z[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) normals_row(kx, (uint64_t)q * N + j0 + i * L, z[i]);
        double dlg;
        double s4[4];
        if (!hmc) {  // kernel.cpp:31-40: x' = x + s xi, accept iff log u < lg(x') - lg(x)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) y[i][k] += eps * z[i][k];
          float e1, yy1;
          C.energy(y, e1, yy1);
          double s2[2] = {(double)e1, (double)yy1};
          C.template block_sum<2>(s2);
          s4[0] = s2[0];
          s4[1] = s2[1];
          dlg = beta * (s4[0] - ecur) - (1.0 - beta) * 0.5 * (double)A.inv_s2 * (s4[1] - yycur);
        } else {  // leapfrog, unit mass, kick-drift-kick with the inner kicks merged
          float k0 = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) k0 += z[i][k] * z[i][k];
          float e1 = 0.f, yy1 = 0.f;
          C.template grad_kick<false>(y, z, bf, A.inv_s2, 0.5f * eps, e1, yy1);
          for (int l = 0; l + 1 < A.kc.leapfrog; ++l) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int k = 0; k < 4; ++k) y[i][k] += eps * z[i][k];
            C.template grad_kick<false>(y, z, bf, A.inv_s2, eps, e1, yy1);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) y[i][k] += eps * z[i][k];
          C.template grad_kick<true>(y, z, bf, A.inv_s2, 0.5f * eps, e1, yy1);
          float k1 = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) k1 += z[i][k] * z[i][k];
          double s[4] = {(double)e1, (double)yy1, (double)k0, (double)k1};
          C.template block_sum<4>(s);
          s4[0] = s[0];
          s4[1] = s[1];
          dlg = beta * (s4[0] - ecur) - (1.0 - beta) * 0.5 * (double)A.inv_s2 * (s4[1] - yycur) +
                0.5 * (s[2] - s[3]);
        }
        const double log_u = log(kx.uniform(q));
        if (log_u < dlg) {
          ecur = s4[0];
          yycur = s4[1];
        } else {
          C.restore(y);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<float4*>(row + j0 + i * L) = make_float4(y[i][0], y[i][1], y[i][2], y[i][3]);
  if (threadIdx.x == 0)
    *reinterpret_cast<double*>(row + N) = ecur + 0.5 * (double)A.inv_s2 * yycur + A.vconst;
}

bool ising_side_supported(int L) { return L == 8 || L == 16 || L == 32 || L == 64; }

static bool ising_tiled(int L) { return L >= 32; }

size_t ising_smem_bytes(int L) {
  if (ising_tiled(L)) {  // edge buffers + Y0 tiles + block-sum scratch
    const size_t TA = L / 4, TPR = L / 4, NT = (size_t)L * L / 16;
    return (4 * TA * TPR + 4 * NT) * 16 + (NT / 32 + 1) * 4 * sizeof(double);
  }
  return 3 * (size_t)L * L * sizeof(float) + (size_t)(4 * L / 32 + 1) * 4 * sizeof(double);
}

template <int L>
static cudaError_t go_is(const IsArgs& A, int mode, const double* betas, int t, cudaStream_t s) {
  const size_t bytes = ising_smem_bytes(L);
  if constexpr (L >= 32) {
    cudaError_t e = cudaFuncSetAttribute(is_tile_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    is_tile_kernel<L><<<(unsigned)A.n_local, L * L / 16, bytes, s>>>(A, mode, betas, t);
  } else {
    cudaError_t e = cudaFuncSetAttribute(is_move_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    is_move_kernel<L><<<(unsigned)A.n_local, 4 * L, bytes, s>>>(A, mode, betas, t);
  }
  return cudaGetLastError();
}

cudaError_t launch_is_move(const IsArgs& A, int mode, const double* betas, int t, cudaStream_t s) {
  if (A.n_local == 0) return cudaSuccess;
  switch (A.L) {
    case 8: return go_is<8>(A, mode, betas, t, s);
    case 16: return go_is<16>(A, mode, betas, t, s);
    case 32: return go_is<32>(A, mode, betas, t, s);
    case 64: return go_is<64>(A, mode, betas, t, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace asmcdev
