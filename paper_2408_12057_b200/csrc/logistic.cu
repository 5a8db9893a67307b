// Config 4 on tcgen05: the Bayesian-logistic-regression likelihood of many
// particles as one tensor-core contraction per RWMH proposal.
//
// For a CTA's 128 particles, l = Theta' X^T (128 particles x n data rows, K = d)
// is computed tile by tile on the 5th-gen tensor cores and immediately folded
// into V(theta') = sum_j y_j l_j - softplus(l_j) -- the 128 x n matrix never
// leaves TMEM, HBM sees only X (re-read from L2) and the particle rows.
//
//   A (M = 128 particles x K = d)  : theta' = theta + s z, built by all threads,
//                                    split bf16 hi + lo, K-major SWIZZLE_128B smem,
//                                    resident for the whole proposal;
//   B (N = 128 data rows x K = d)  : X split bf16 hi + lo, K-major SWIZZLE_128B,
//                                    streamed by TMA through a 2-stage mbarrier ring
//                                    (one 64-wide K chunk of hi and lo per stage);
//   D (128 x 128 fp32)             : TMEM, double-buffered (2 x 128 columns) so the
//                                    epilogue of tile i overlaps the MMAs of tile i+1;
//   precision                      : l = A_hi B_hi + A_hi B_lo + A_lo B_hi (3 MMAs per
//                                    K step, fp32 accumulate; ~2^-17 relative products),
//                                    softplus in fp32 (MUFU), V accumulated in fp64.
//   epilogue                       : V = theta' . w - sum_j softplus(l_j) with w = X^T y
//                                    (fp64, once per call): the linear term never touches
//                                    the logits; sum_j log1p(e^-|l_j|) = log2 of a running
//                                    product of (1 + e^-|l_j|) in [1, 2] over 32 logits
//                                    (<= 2^32): one SFU ex2 per logit, one lg2 per 32.
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// elected thread), warp 2 = TMEM allocator, warps 4..7 = epilogue (TMEM lanes
// 0..127 = the CTA's particles), everyone builds A and writes accepted rows.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "logistic.h"
#include "pass_kernel.cuh"

namespace asmcdev {

constexpr int LG_M = 128, LG_N = 128, LG_KC = 64, LG_STAGES = 3, LG_THREADS = 256;
constexpr int LG_CHUNK_BYTES = LG_M * LG_KC * 2;  // 16 KB: one 128-row x 64-col bf16 tile
constexpr int LG_STAGE_BYTES = 2 * LG_CHUNK_BYTES;  // hi + lo
// 2-SM pair (cta_group::2): M = 256 particles (128 per SM), N = 256 data rows (each SM
// stages 128 of them), D = 128 x 256 fp32 per SM in TMEM
constexpr int LG_PN = 2 * LG_N;  // data rows per pair tile
constexpr uint32_t LG_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LG_PN >> 3) << 17) |
                              ((uint32_t)((2 * LG_M) >> 4) << 24);  // bf16 x bf16 -> f32, K-major, 256x256

size_t logistic_smem_bytes(int d) {
  const int kch = d / LG_KC;
  // the dynamic window is 1024-aligned (__align__ below, no static shared memory), so no
  // slack: A (hi + lo) + 3 stages = 224 KB at d = 256 leaves room only for the scalars
  return 2 * (size_t)kch * LG_CHUNK_BYTES + (size_t)LG_STAGES * LG_STAGE_BYTES +
         (2 * LG_STAGES + 4) * sizeof(uint64_t) + 16 /*tmem slot*/ + LG_M * sizeof(double) +
         LG_M * sizeof(float) + LG_M * sizeof(int);
}

// ---------------------------------------------------------------- PTX --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;" ::"r"(bytes), "r"(smem_u32(bar)));
}
// 2-SM TMA: the box lands in this CTA's shared memory, the byte count is signalled on the
// pair leader's barrier (bar_cluster = leader_addr(...))
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
// K-major SWIZZLE_128B UMMA smem descriptor: rows 128 B apart, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t umma_desc(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(LG_IDESC), "r"(accumulate));
}
// arrive on the barrier at this offset in BOTH CTAs of the pair when the MMAs retire
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3));
}
// the peer-0 (leader) address of a shared-memory object in the cluster window
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// ------------------------------------------------------------- kernels --
// X (n x d fp32) -> zero-padded split bf16 [n_pad x d] hi and lo
__global__ void lg_split_kernel(const float* X, uint64_t n, int d, uint64_t n_pad, __nv_bfloat16* hi,
                                __nv_bfloat16* lo) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pad * (uint64_t)d) return;
  const float x = i < n * (uint64_t)d ? X[i] : 0.0f;
  const __nv_bfloat16 h = __float2bfloat16_rn(x);
  hi[i] = h;
  lo[i] = __float2bfloat16_rn(x - __bfloat162float(h));
}

// theta_0 ~ N(0, sigma_p^2 I) from the init stream (seed, round, p, 0, 0), V = 0
__global__ void lg_init_kernel(LgArgs A) {
  const uint64_t local = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= A.n_local) return;
  PhiloxKey k;
  k.init(A.seed, A.round, A.p_begin + local, 0, 0);
  float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
  for (int b = 0; b < A.d / 4; ++b) {
    float z[4];
    k.normals4<float>((uint32_t)b, z);
    for (int e = 0; e < 4; ++e) row[4 * b + e] = (float)(A.sigma_p * (double)z[e]);
  }
  *reinterpret_cast<double*>(row + A.d) = 0.0;
}

// weight + per-step block partials (engine_detail.hpp:122-140 per particle):
// lg = (beta_t - beta_{t-1}) V(theta), partials of (lw, lg, lw + lg), lw += lg
__global__ void __launch_bounds__(kBlock) lg_weight_kernel(LgArgs A, const double* betas, int t,
                                                          LogAcc* part, uint64_t stride) {
  __shared__ double s_lw[kBlock], s_lg[kBlock], s_post[kBlock];
  __shared__ int s_act[kBlock];
  __shared__ LogAcc s_dst[kNAcc];
  if (block_err_set(A.err)) return;
  const double b0 = betas[t - 1], b1 = betas[t];
  const uint64_t local = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
  const bool active = local < A.n_local;
  double lw = 0.0, lg = 0.0;
  if (active) {
    const float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
    const double V = *reinterpret_cast<const double*>(row + A.d);
    lg = (b1 - b0) * V;
    lw = A.lw[local];
    A.lw[local] = lw + lg;
  }
  s_lw[threadIdx.x] = lw;
  s_lg[threadIdx.x] = lg;
  s_post[threadIdx.x] = lw + lg;
  s_act[threadIdx.x] = active ? 1 : 0;
  __syncthreads();
  block_reduce<false, kBlock>(s_lw, s_lg, s_post, s_act, kNAcc, s_dst, true);
  __syncthreads();
  if (threadIdx.x < kNAcc) part[(size_t)threadIdx.x * stride + blockIdx.x] = s_dst[threadIdx.x];
}

// One likelihood evaluation per particle of the CTA: mode 0 sets V(theta); mode 1
// evaluates the RWMH proposal theta' = theta + s z (normals q d .. q d + d - 1 of
// stream (p, t, explore)) and accepts it iff log u_q < dlog eta + beta (V' - V).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(LG_THREADS, 1)
    lg_eval_kernel(const __grid_constant__ CUtensorMap tmap_hi, const __grid_constant__ CUtensorMap tmap_lo,
                   const __grid_constant__ LgArgs A, int mode, const double* betas, float step, int q) {
  const double beta = mode == 1 ? betas[A.t] : 0.0;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw;  // SWIZZLE_128B tiles need 1024-byte alignment (checked below)
  const int kch = A.d / LG_KC;
  unsigned char* a_hi = smem;
  unsigned char* a_lo = a_hi + (size_t)kch * LG_CHUNK_BYTES;
  unsigned char* stages = a_lo + (size_t)kch * LG_CHUNK_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + LG_STAGES * LG_STAGE_BYTES);
  uint64_t* empty = full + LG_STAGES;
  uint64_t* tfull = empty + LG_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // first halves (threads 0..127) of theta' . w and of the prior difference; the second
  // halves stay in the registers of threads 128..255, which are the epilogue threads
  double* lin0 = reinterpret_cast<double*>(tmem_slot + 4);  // [LG_M]
  float* prior0 = reinterpret_cast<float*>(lin0 + LG_M);    // [LG_M]
  int* accept = reinterpret_cast<int*>(prior0 + LG_M);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t crank = cluster_rank();  // 0 = pair leader (issues the MMAs)
  const uint64_t p0 = (uint64_t)blockIdx.x * LG_M;  // pair (blockIdx.x / 2) holds 256 particles
  const int d = A.d;
  // per-thread read, cluster-safe: nothing in this launch raises the word before this
  // point except the alignment check below, which every CTA takes alike
  if (A.err && *(volatile int*)A.err) return;
  if (smem_u32(smem_raw) & 1023u) {  // uniform across the CTA: fail loudly, never mis-swizzle
    if (tid == 0) raise_error(A.err, ASMC_ERR_CUDA);
    return;
  }
  float pd_own = 0.0f;   // this thread's half of theta'^2 - theta^2
  double ld_own = 0.0;   // this thread's half of theta' . w

  if (tid == 0) {
    for (int s = 0; s < LG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);  // the epilogue warps of both CTAs (leader's copy is used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }

  // ---- A = theta' of the CTA's particles: thread (r, half) owns d/2 coordinates
  {
    const int r = tid & (LG_M - 1), half = tid >> 7;
    const uint64_t local = p0 + r;
    const bool active = local < A.n_local;
    const float* row = A.state[*A.xcur] + (active ? local : 0) * (uint64_t)A.row;
    PhiloxKey k;
    k.init(A.seed, A.round, A.p_begin + local, (uint64_t)A.t, 1);
    const uint64_t base = (uint64_t)q * (uint64_t)d;
    float pd = 0.0f;
    double ld = 0.0;  // this half of theta' . w
    const int i0 = half * (d / 2), i1 = i0 + d / 2;
    for (int i = i0; i < i1; i += 8) {
      float th[8];
      const float4 u = reinterpret_cast<const float4*>(row + i)[0];
      const float4 w = reinterpret_cast<const float4*>(row + i)[1];
      th[0] = u.x; th[1] = u.y; th[2] = u.z; th[3] = u.w;
      th[4] = w.x; th[5] = w.y; th[6] = w.z; th[7] = w.w;
      if (!active) {
#pragma unroll
        for (int e = 0; e < 8; ++e) th[e] = 0.0f;
      } else if (mode == 1) {
        float z[8];
        k.normals4<float>((uint32_t)((base + i) >> 2), z);
        k.normals4<float>((uint32_t)((base + i) >> 2) + 1, z + 4);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float h = step * z[e];
          pd += h * (2.0f * th[e] + h);  // theta'^2 - theta^2
          th[e] += h;
        }
      }
      float hv[8], lv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) ld = fma((double)th[e], A.w[i + e], ld);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        hv[e] = __bfloat162float(__float2bfloat16_rn(th[e]));
        lv[e] = th[e] - hv[e];
      }
      const uint4 H = make_uint4(pack_bf16(hv[0], hv[1]), pack_bf16(hv[2], hv[3]), pack_bf16(hv[4], hv[5]),
                                 pack_bf16(hv[6], hv[7]));
      const uint4 L = make_uint4(pack_bf16(lv[0], lv[1]), pack_bf16(lv[2], lv[3]), pack_bf16(lv[4], lv[5]),
                                 pack_bf16(lv[6], lv[7]));
      const int c = i / LG_KC, unit = (i % LG_KC) / 8;
      const size_t off = (size_t)c * LG_CHUNK_BYTES + (size_t)r * 128 + (size_t)((unit ^ (r & 7)) * 16);
      *reinterpret_cast<uint4*>(a_hi + off) = H;
      *reinterpret_cast<uint4*>(a_lo + off) = L;
    }
    if (half == 0) {
      prior0[r] = pd;
      lin0[r] = ld;
    }
    pd_own = pd;
    ld_own = ld;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' A halves, barriers and TMEM are ready before any MMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntiles = (int)((A.n + LG_PN - 1) / LG_PN);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int tile = 0; tile < ntiles; ++tile) {
        for (int c = 0; c < kch; ++c) {
          const int it = tile * kch + c, s = it % LG_STAGES;
          const uint32_t ph = (uint32_t)(it / LG_STAGES) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);  // both CTAs' stage s retired (multicast commit)
          unsigned char* st = stages + (size_t)s * LG_STAGE_BYTES;
          // this CTA stages data rows [tile * 256 + 128 crank, +128); both halves count on
          // the leader's full[s], which expects the pair's bytes
          if (crank == 0) mbar_expect_tx(&full[s], 2 * LG_STAGE_BYTES);
          const int row0 = tile * LG_PN + (int)crank * LG_N;
          const uint32_t fb = leader_addr(&full[s]);
          tma_load_2d(st, &tmap_hi, c * LG_KC, row0, fb);
          tma_load_2d(st + LG_CHUNK_BYTES, &tmap_lo, c * LG_KC, row0, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && crank == 0) {  // ---- MMA issuer (pair leader only)
      for (int tile = 0; tile < ntiles; ++tile) {
        const int b = tile & 1;
        mbar_wait(&tempty[b], (((uint32_t)tile >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dt = tmem + (uint32_t)(b * LG_PN);
        for (int c = 0; c < kch; ++c) {
          const int it = tile * kch + c, s = it % LG_STAGES;
          mbar_wait(&full[s], (uint32_t)(it / LG_STAGES) & 1u);
          tc_fence_after();
          const unsigned char* st = stages + (size_t)s * LG_STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < LG_KC / 16; ++kk) {
            const uint64_t ah = umma_desc(a_hi + (size_t)c * LG_CHUNK_BYTES + kk * 32);
            const uint64_t al = umma_desc(a_lo + (size_t)c * LG_CHUNK_BYTES + kk * 32);
            const uint64_t bh = umma_desc(st + kk * 32);
            const uint64_t bl = umma_desc(st + LG_CHUNK_BYTES + kk * 32);
            umma_bf16(dt, ah, bh, (c | kk) != 0 ? 1u : 0u);
            umma_bf16(dt, ah, bl, 1u);
            umma_bf16(dt, al, bh, 1u);
          }
          umma_commit(&empty[s]);  // frees stage s in both CTAs when these MMAs retire
        }
        umma_commit(&tfull[b]);  // both CTAs' accumulator halves ready for their epilogues
      }
    }
  } else if (warp >= 4) {  // ---- epilogue: thread = particle row of D
    const int w = warp - 4, r = w * 32 + lane;
    const uint32_t tempty_leader[2] = {leader_addr(&tempty[0]), leader_addr(&tempty[1])};
    double V = 0.0;
    for (int tile = 0; tile < ntiles; ++tile) {
      const int b = tile & 1;
      mbar_wait(&tfull[b], ((uint32_t)tile >> 1) & 1u);
      tc_fence_after();
      const uint64_t row_base = (uint64_t)tile * LG_PN;  // D column c = data row row_base + c
      const int valid_tile = A.n > row_base + LG_PN ? LG_PN : (int)(A.n - row_base);
      float smax = 0.0f, slog2 = 0.0f;  // sum max(l, 0), sum log2(1 + e^-|l|)
#pragma unroll 1
      for (int cc = 0; cc < LG_PN / 32; ++cc) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + (uint32_t)(b * LG_PN + cc * 32), v);
        float prod = 1.0f;
        if (valid_tile == LG_PN) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float e;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(v[j]) * -1.4426950408889634f));
            prod *= 1.0f + e;
            smax += fmaxf(v[j], 0.0f);
          }
        } else {  // the last, partial tile: padded rows (l = 0) contribute nothing
          const int valid = valid_tile - cc * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float e;
            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fabsf(v[j]) * -1.4426950408889634f));
            prod *= j < valid ? 1.0f + e : 1.0f;
            smax += j < valid ? fmaxf(v[j], 0.0f) : 0.0f;
          }
        }
        float g;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(prod));
        slog2 += g;
      }
      const float acc = -fmaf(slog2, 0.69314718055994531f, smax);  // - sum softplus
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty_leader[b]);  // the leader waits for all 8 warps
      V += (double)acc;
    }
    V += lin0[r] + ld_own;  // thread 128 + r built the second half of particle r
    // ---- MH decision (kernel.cpp:35 in difference form) / V store
    const uint64_t local = p0 + r;
    int acc_flag = 0;
    if (local < A.n_local) {
      float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
      double* vrow = reinterpret_cast<double*>(row + d);
      if (mode == 0) {
        *vrow = V;
      } else {
        const double dprior = -0.5 * ((double)prior0[r] + (double)pd_own) /
                              (A.sigma_p * A.sigma_p);
        const double delta = dprior + beta * (V - *vrow);
        PhiloxKey k;
        k.init(A.seed, A.round, A.p_begin + local, (uint64_t)A.t, 1);
        const double log_u = log(k.uniform((uint32_t)q));
        if (log_u < delta) {
          acc_flag = 1;
          *vrow = V;
        }
      }
    }
    accept[r] = acc_flag;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // ---- write accepted proposals (same arithmetic as the A build, in fp32)
  if (mode == 1) {
    const int r = tid & (LG_M - 1), half = tid >> 7;
    const uint64_t local = p0 + r;
    if (local < A.n_local && accept[r]) {
      float* row = A.state[*A.xcur] + local * (uint64_t)A.row;
      PhiloxKey k;
      k.init(A.seed, A.round, A.p_begin + local, (uint64_t)A.t, 1);
      const uint64_t base = (uint64_t)q * (uint64_t)d;
      for (int i = half * (d / 2); i < (half + 1) * (d / 2); i += 4) {
        float z[4];
        k.normals4<float>((uint32_t)((base + i) >> 2), z);
        float4 x = reinterpret_cast<float4*>(row + i)[0];
        x.x += step * z[0];
        x.y += step * z[1];
        x.z += step * z[2];
        x.w += step * z[3];
        reinterpret_cast<float4*>(row + i)[0] = x;
      }
    }
  }
  // the leader's MMAs read this CTA's shared memory and both CTAs' TMEM is one
  // allocation: neither CTA leaves before the other is done
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------ launchers --
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t make_x_maps(const void* hi, const void* lo, uint64_t n_pad, int d, CUtensorMap* mhi,
                        CUtensorMap* mlo) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n_pad};
  const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  const cuuint32_t box[2] = {LG_KC, LG_N};
  const cuuint32_t elem[2] = {1, 1};
  for (int i = 0; i < 2; ++i) {
    CUresult r = encode(i == 0 ? mhi : mlo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void*>(i == 0 ? hi : lo), dims, strides, box, elem,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

cudaError_t launch_lg_split(const float* X, uint64_t n, int d, uint64_t n_pad, void* hi, void* lo,
                            cudaStream_t s) {
  const uint64_t tot = n_pad * (uint64_t)d;
  lg_split_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(X, n, d, n_pad, (__nv_bfloat16*)hi,
                                                                (__nv_bfloat16*)lo);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) lg_xty_kernel(const float* X, const float* y, uint64_t n, int d,
                                                     double* w) {
  __shared__ double red[256];
  const int k = blockIdx.x;
  double s = 0.0;
  for (uint64_t j = threadIdx.x; j < n; j += 256) s = fma((double)y[j], (double)X[j * (uint64_t)d + k], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) w[k] = red[0];
}

cudaError_t launch_lg_xty(const float* X, const float* y, uint64_t n, int d, double* w, cudaStream_t s) {
  lg_xty_kernel<<<d, 256, 0, s>>>(X, y, n, d, w);
  return cudaGetLastError();
}

cudaError_t launch_lg_init(const LgArgs& A, cudaStream_t s) {
  lg_init_kernel<<<(unsigned)((A.n_local + 255) / 256), 256, 0, s>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_lg_weight(const LgArgs& A, const double* betas, int t, LogAcc* part, uint64_t stride,
                             cudaStream_t s) {
  lg_weight_kernel<<<(unsigned)((A.n_local + kBlock - 1) / kBlock), kBlock, 0, s>>>(A, betas, t, part, stride);
  return cudaGetLastError();
}

cudaError_t launch_lg_eval(const CUtensorMap& mhi, const CUtensorMap& mlo, const LgArgs& A, int mode,
                           const double* betas, float step, int q, cudaStream_t s) {
  const size_t bytes = logistic_smem_bytes(A.d);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(lg_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const unsigned pairs = (unsigned)((A.n_local + 2 * LG_M - 1) / (2 * LG_M));
  lg_eval_kernel<<<2 * pairs, LG_THREADS, bytes, s>>>(mhi, mlo, A, mode, betas,
                                                                                       step, q);
  return cudaGetLastError();
}

}  // namespace asmcdev
