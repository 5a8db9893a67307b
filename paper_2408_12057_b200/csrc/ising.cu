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

__device__ __forceinline__ float tanh_f(float u) {
  const float e = __expf(2.0f * fminf(fmaxf(u, -15.0f), 15.0f));
  return 1.0f - __fdividef(2.0f, e + 1.0f);
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
  if (A.err && *(volatile int*)A.err) return;
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

bool ising_side_supported(int L) { return L == 8 || L == 16 || L == 32 || L == 64; }

size_t ising_smem_bytes(int L) { return 3 * (size_t)L * L * sizeof(float) + (size_t)(4 * L / 32 + 1) * 4 * sizeof(double); }

template <int L>
static cudaError_t go_is(const IsArgs& A, int mode, const double* betas, int t, cudaStream_t s) {
  const size_t bytes = ising_smem_bytes(L);
  cudaError_t e = cudaFuncSetAttribute(is_move_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  is_move_kernel<L><<<(unsigned)A.n_local, 4 * L, bytes, s>>>(A, mode, betas, t);
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
