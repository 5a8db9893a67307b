// C-ABI entry points (include/asmc_b200.h) and the host-side orchestration of
// the device pipelines.  Host code here only validates, sizes buffers and
// enqueues kernels; every sampler computation runs on the GPU.  There is no
// CPU fallback: without a device every sampler entry returns ASMC_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "asmc_b200.h"
#include "dispatch.h"
#include "engine_kernels.h"
#include "ising.h"
#include "logistic.h"
#include "pt.h"
#include "zja.h"

using namespace asmcdev;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ASMC_ERR_CUDA, "CUDA error %s at %s:%d", cudaGetErrorString(e_),       \
                  __FILE__, __LINE__);                                                   \
  } while (0)
#define TRY(expr)          \
  do {                     \
    int rc_ = (expr);      \
    if (rc_) return rc_;   \
  } while (0)
#define LCH(expr)          \
  do {                     \
    ++g_launches;          \
    CU(expr);              \
  } while (0)

struct DevCtx {
  cudaStream_t stream = nullptr;
  int sms = 148;
  char* pinned = nullptr;  // page-locked staging for the per-call result copies (grown on demand)
  size_t pinned_cap = 0;
  std::vector<cudaEvent_t> events;  // reusable timing events (asmc_run_rounds)
};

// page-locked staging of at least `bytes` (kept for the context's lifetime)
int pinned_staging(DevCtx* C, size_t bytes, char** out) {
  if (C->pinned_cap < bytes) {
    if (C->pinned) cudaFreeHost(C->pinned);
    C->pinned = nullptr;
    C->pinned_cap = 0;
    const size_t cap = bytes < 65536 ? 65536 : bytes * 2;
    CU(cudaHostAlloc(reinterpret_cast<void**>(&C->pinned), cap, cudaHostAllocPortable));
    C->pinned_cap = cap;
  }
  *out = C->pinned;
  return 0;
}

int get_ctx(int device, DevCtx** out, uint64_t user_stream = 0) {
  static thread_local std::map<int, DevCtx> ctxs;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(ASMC_ERR_CUDA, "no CUDA device available (the sampler has no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(ASMC_ERR_CUDA, "invalid CUDA device %d", device);
  CU(cudaSetDevice(device));
  auto it = ctxs.find(device);
  if (it == ctxs.end()) {
    DevCtx c;
    CU(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    CU(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, device));
    // keep freed stream-ordered allocations reserved: every round re-allocates
    // its partial buffers, which must not go back to the OS at each sync
    cudaMemPool_t pool;
    CU(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = ~0ull;
    CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    it = ctxs.emplace(device, c).first;
  }
  // the caller's stream: a per-device view with its own (persistent) staging and events
  static thread_local std::map<int, DevCtx> users;
  if (user_stream) {
    DevCtx& user = users[device];
    user.stream = reinterpret_cast<cudaStream_t>(user_stream);
    user.sms = it->second.sms;
    *out = &user;
    return 0;
  }
  *out = &it->second;
  return 0;
}

// Stream-ordered device buffer (cudaMallocAsync pool).
template <class T>
struct DBuf {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  bool own = true;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p && own) cudaFreeAsync(p, s);
  }
  void borrow(T* q) {  // a view into a caller-owned arena (not freed here)
    p = q;
    own = false;
  }
  int alloc(size_t n, cudaStream_t st) {
    s = st;
    if (n == 0) n = 1;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st));
    return 0;
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Systematic resampling with the reference's sequential CDF (refcdf.cu): one cooperative
// launch, returns at once on steps whose decision did not fire.  work: refcdf_work_bytes(n).
cudaError_t launch_resample_ref(DevCtx* C, const double* lw, uint64_t n, SmcState* st, void* work,
                                double* cum, uint32_t* anc, int gated = 1) {
  RefCdfWork w;
  refcdf_work_carve(work, n, &w);
  return launch_refcdf(lw, n, st, gated, &w, cum, anc, 1, C->sms, C->stream);
}
uint64_t refcdf_work_doubles(uint64_t n) { return (refcdf_work_bytes(n) + 7) / 8; }

// ---------------------------------------------------------------- checks --
// Schedule::validate (src/engine.cpp:29-39)
int check_schedule(const double* b, int T) {
  if (!b || T < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "schedule needs at least one step");
  if (b[0] != 0.0) return fail(ASMC_ERR_INVALID_ARGUMENT, "schedule must start at beta = 0");
  if (b[T] != 1.0) return fail(ASMC_ERR_INVALID_ARGUMENT, "schedule must end at beta = 1");
  for (int t = 1; t <= T; ++t)
    if (!(b[t] > b[t - 1]))
      return fail(ASMC_ERR_INVALID_ARGUMENT, "schedule must be strictly increasing at index %d", t);
  return 0;
}

// validate_kernel (src/kernel.cpp:12-22)
int check_kernel(const asmc_kernel_desc* k) {
  if (!k) return fail(ASMC_ERR_INVALID_ARGUMENT, "null kernel descriptor");
  if (k->kind == ASMC_KERNEL_RWMH) {
    if (k->n_step_sizes < 1)
      return fail(ASMC_ERR_INVALID_ARGUMENT, "rwmh_cycle requires at least one step size");
    if (k->n_step_sizes > ASMC_MAX_STEP_SIZES)
      return fail(ASMC_ERR_CAPABILITY, "at most %d rwmh step sizes are supported on the device",
                  ASMC_MAX_STEP_SIZES);
    for (int i = 0; i < k->n_step_sizes; ++i)
      if (!(k->step_sizes[i] > 0.0))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "rwmh step sizes must be positive");
    if (k->sweeps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "rwmh sweeps must be at least 1");
  } else if (k->kind == ASMC_KERNEL_HMC) {  // new kernel; same checks as oracle/restate.c
    if (k->n_step_sizes < 1 || k->n_step_sizes > ASMC_MAX_STEP_SIZES)
      return fail(ASMC_ERR_INVALID_ARGUMENT, "hmc requires 1..16 step sizes");
    for (int i = 0; i < k->n_step_sizes; ++i)
      if (!(k->step_sizes[i] > 0.0))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "hmc step sizes must be positive");
    if (k->sweeps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "hmc sweeps must be at least 1");
    if (k->leapfrog < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "hmc leapfrog steps must be at least 1");
  } else if (k->kind == ASMC_KERNEL_SLICE) {  // new kernel; same checks as oracle/restate.c
    if (k->sweeps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "slice sweeps must be at least 1");
  } else if (k->kind != ASMC_KERNEL_IDEALIZED && k->kind != ASMC_KERNEL_IDENTITY) {
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown kernel kind");
  }
  return 0;
}

// constructor checks (src/target.cpp:57-63, 115-131; scale plugin)
int check_target(const asmc_target_desc* t) {
  if (!t) return fail(ASMC_ERR_INVALID_ARGUMENT, "null target descriptor");
  const double* p = t->p;
  switch (t->kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT:
      if (!(p[2] > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "sigma must be positive");
      break;
    case ASMC_TARGET_MIXTURE:
      if (!(p[0] > 0.0 && p[3] > 0.0 && p[5] > 0.0))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "mixture sigmas must be positive");
      if (!(p[1] > 0.0 && p[1] < 1.0))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "mixture weight must lie strictly in (0, 1)");
      break;
    case ASMC_TARGET_SCALE_GAUSSIAN:
      if (!(p[0] > 0.0 && p[1] > 0.0))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "scale sigmas must be positive");
      break;
    case ASMC_TARGET_LOGISTIC:
      if (!(p[0] > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "prior sigma must be positive");
      if (!(p[1] >= 1.0) || !t->data ||
          t->data_bytes < (uint64_t)p[1] * (t->dim + 1) * sizeof(float))
        return fail(ASMC_ERR_INVALID_ARGUMENT, "logistic target needs X (n x dim) and y (n) data");
      break;
    case ASMC_TARGET_ISING: {
      const int L = (int)p[0];
      if (!((double)L == p[0] && L >= 3) || t->dim != (uint64_t)L * (uint64_t)L)
        return fail(ASMC_ERR_INVALID_ARGUMENT, "ising target needs an integer side L >= 3 and dim = L * L");
      if (!(p[1] >= 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "ising coupling must be non-negative");
      if (!(p[2] > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "ising relaxation delta must be positive");
      if (!(p[3] > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "reference sigma must be positive");
      break;
    }
    default:
      return fail(ASMC_ERR_CAPABILITY, "target kind %d has no device implementation", t->kind);
  }
  if (t->dim == 0) return fail(ASMC_ERR_INVALID_ARGUMENT, "dim must be at least 1");
  if (t->dim > 16384)
    return fail(ASMC_ERR_CAPABILITY, "dim %llu exceeds the device kernels' limit of 16384",
                (unsigned long long)t->dim);
  return 0;
}

// shared-memory words per particle quad of the RWMH pass for the target being launched
// (pass_smem.cuh RowWords: two rows, x + cached vterm for the mixture); set by check_pair
thread_local int g_row_words = 2;

int check_pair(const asmc_target_desc* t, const asmc_kernel_desc* k) {
  TRY(check_target(t));
  g_row_words = (t->kind == ASMC_TARGET_MIXTURE ? 2 : 1) * (k && k->kind == ASMC_KERNEL_HMC ? 1 : 2);
  TRY(check_kernel(k));
  if (k->kind == ASMC_KERNEL_IDEALIZED &&
      (t->kind == ASMC_TARGET_MIXTURE || t->kind == ASMC_TARGET_ISING || t->kind == ASMC_TARGET_LOGISTIC))
    return fail(ASMC_ERR_CAPABILITY, "idealized_exact kernel requires an exact sampler");
  return 0;
}

// entry points built on the fused particle pass only (not the step-outer engines
// of the data-backed / lattice targets)
int check_pass_target(const asmc_target_desc* t, const char* what) {
  if (t->kind == ASMC_TARGET_LOGISTIC || t->kind == ASMC_TARGET_ISING)
    return fail(ASMC_ERR_CAPABILITY, "%s does not support the %s target yet", what,
                t->kind == ASMC_TARGET_LOGISTIC ? "logistic" : "ising");
  return 0;
}

// host-side constants with glibc, so the fp64 path sees the reference's bits
TgtParams make_params(const asmc_target_desc* t) {
  TgtParams P;
  std::memset(&P, 0, sizeof P);
  P.kind = t->kind;
  P.dim = t->dim;
  for (int i = 0; i < 8; ++i) P.p[i] = t->p[i];
  const double* p = t->p;
  switch (t->kind) {
    case ASMC_TARGET_GAUSSIAN_SHIFT:
      P.c[0] = std::log(p[2]);
      P.c[1] = (p[1] - p[0]) / (p[2] * p[2]);
      P.c[2] = 0.5 * (p[0] + p[1]);
      P.c[3] = 1.0 / (p[2] * p[2]);
      break;
    case ASMC_TARGET_MIXTURE:
      P.c[0] = std::log(p[0]);
      P.c[1] = std::log(p[1]);
      P.c[2] = std::log1p(-p[1]);
      P.c[3] = std::log(p[3]);
      P.c[4] = std::log(p[5]);
      {  // TgtMixture::F32 (targets.cuh): log-normal constants folded, base-2 vterm terms
        const double l1 = P.c[1] - P.c[3] + P.c[0], l2 = P.c[2] - P.c[4] + P.c[0];
        const double lm = (l1 > l2 ? l1 : l2) + std::log1p(std::exp(-std::fabs(l1 - l2)));
        const double log2e = 1.4426950408889634, h = std::sqrt(0.5 * log2e);
        const double c1 = h / p[3], c2 = h / p[5];
        const double v[16] = {1.0 / p[0], l1, p[2], 1.0 / p[3], l2, p[4], 1.0 / p[5], lm,
                              c1, -p[2] * c1, c2, -p[4] * c2, l1 * log2e, l2 * log2e,
                              0.5 * log2e / (p[0] * p[0]), 0.5 / (p[0] * p[0])};
        for (int i = 0; i < 16; ++i) P.f[i] = static_cast<float>(v[i]);
      }
      break;
    case ASMC_TARGET_SCALE_GAUSSIAN:
      P.c[0] = std::log(p[0]);
      P.c[1] = std::log(p[1]);
      P.c[2] = 1.0 / (p[0] * p[0]);
      P.c[3] = 1.0 / (p[1] * p[1]);
      P.c[4] = 0.5 * (P.c[2] - P.c[3]);
      P.c[5] = P.c[1] - P.c[0];
      break;
  }
  return P;
}

KernelCfg make_kcfg(const asmc_kernel_desc* k) {
  KernelCfg c;
  std::memset(&c, 0, sizeof c);
  c.kind = k->kind;
  c.n_steps = k->n_step_sizes;
  c.sweeps = k->sweeps;
  c.leapfrog = k->leapfrog;
  // test hook: exact early rejection off, so tests can show it never changes a decision
  const char* ne = std::getenv("ASMC_NO_EARLY_REJECT");
  c.no_early = ne && ne[0] == '1';
  for (int i = 0; i < k->n_step_sizes && i < ASMC_MAX_STEP_SIZES; ++i) c.steps[i] = k->step_sizes[i];
  if (c.kind == ASMC_KERNEL_SLICE) c.n_steps = 1;
  if (c.kind != ASMC_KERNEL_RWMH && c.kind != ASMC_KERNEL_HMC && c.kind != ASMC_KERNEL_SLICE) {
    c.n_steps = 1;
    c.sweeps = 1;
  }
  return c;
}

asmc_exec default_exec() {
  asmc_exec e;
  e.rng = ASMC_RNG_XOSHIRO;
  e.precision = ASMC_PREC_FP64;
  e.device = 0;
  e.lanes = 0;
  e.stream = 0;
  return e;
}

int check_smem(Layout L, uint64_t d, int rows, int nacc);

int choose_layout_impl(const asmc_exec& ex, int kind, uint64_t d, Layout* L);

// rows / nacc: per-launch step rows and accumulators, for the shared-memory budget
int choose_layout(const asmc_exec& ex, int kind, uint64_t d, Layout* L, int rows = 1, int nacc = kNAcc) {
  TRY(choose_layout_impl(ex, kind, d, L));
  return check_smem(*L, d, rows, nacc);
}

int choose_layout_impl(const asmc_exec& ex, int kind, uint64_t d, Layout* L) {
  if (ex.rng != ASMC_RNG_XOSHIRO && ex.rng != ASMC_RNG_PHILOX)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown rng %d", ex.rng);
  if (ex.precision != ASMC_PREC_FP64 && ex.precision != ASMC_PREC_FP32)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown precision %d", ex.precision);
  const bool seq_only = ex.precision == ASMC_PREC_FP64 || ex.rng == ASMC_RNG_XOSHIRO;
  if (seq_only) {
    if (ex.lanes > 1)
      return fail(ASMC_ERR_CAPABILITY, "lanes > 1 needs rng = philox and precision = fp32");
    if (d > 1024)
      return fail(ASMC_ERR_CAPABILITY,
                  "dim %llu > 1024 needs rng = philox, precision = fp32 (shared-memory pass)",
                  (unsigned long long)d);
    *L = Layout{1, d <= 16 ? 16 : 1024};
    return 0;
  }
  int lanes = ex.lanes;
  if (lanes == 0) lanes = d <= 16 ? 1 : (d <= 128 ? 4 : 32);
  if (lanes == 1 && d <= 1024) *L = Layout{1, d <= 16 ? 16 : 1024};
  else if (lanes == 4 || lanes == 32) *L = Layout{lanes, 0};  // shared-memory particle store
  else return fail(ASMC_ERR_CAPABILITY, "lanes %d not available for dim %llu", lanes, (unsigned long long)d);
  return 0;
}

// shared-memory budget of the many-lanes pass (x quads + per-warp step accumulators)
int check_smem(Layout L, uint64_t d, int rows, int nacc) {
  if (L.lanes == 1) return 0;
  const size_t bytes = smem_pass_bytes(L.lanes, d, rows - 1, nacc, g_row_words);
  if (bytes > 227 * 1024)
    return fail(ASMC_ERR_CAPABILITY,
                "pass needs %zu B of shared memory (dim %llu, %d steps); limit 227 KB", bytes,
                (unsigned long long)d, rows);
  return 0;
}

// Long-T SAIS (drivers.cpp:86-146 has no T cap): the shared-memory pass keeps per-warp
// step accumulators for the steps of ONE launch, so a round whose T would lower the
// pass's occupancy (or overflow 227 KB) runs in t-tiles of this many steps, the particle
// rows parked in HBM between tiles (8d + 8 bytes per particle per tile).
int sais_tile_rows(Layout L, uint64_t d, int T) {
  if (L.lanes == 1 || T < 2) return T;  // one-lane pass: partials in global memory, no cap
  if (const char* e = std::getenv("ASMC_SAIS_TILE")) {  // test hook: force the tile length
    const int f = std::atoi(e);
    if (f >= 1) return f < T ? f : T;
  }
  auto occ = [&](int rows) {
    const size_t b = smem_pass_bytes(L.lanes, d, rows - 1, 4, g_row_words) + 1024;
    const int o = (int)((228 * 1024) / b);
    return o < 3 ? o : 3;  // the pass's register budget allows 3 CTAs/SM
  };
  const int o1 = occ(1);
  if (occ(T) >= o1) return T;
  int lo = 1, hi = T;  // largest rows with the same occupancy as one step
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (occ(mid) >= o1) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Live per-launch timing of the particle pass (bench.py roofline): events on
// the launching stream around each pass, plus its algorithmic normal draws.
struct ProfRec {
  cudaEvent_t a, b;
  double normals;                        // algorithmic units of the launch
  unsigned long long* drawn = nullptr;   // device counter: normals actually generated (smem pass)
};
thread_local bool g_prof = false;
thread_local std::vector<ProfRec> g_prof_recs;

double pass_normals(const PassArgs& A, uint64_t nparticles) {
  const double d = (double)A.tg.dim;
  double per_step = 0.0;
  if (A.kc.kind == ASMC_KERNEL_RWMH || A.kc.kind == ASMC_KERNEL_HMC)
    per_step = (double)A.kc.sweeps * A.kc.n_steps * d;
  else if (A.kc.kind == ASMC_KERNEL_IDEALIZED) per_step = d;
  const double steps = A.mode == kModeSmcInit ? 0.0 : (double)(A.t_end - A.t_begin + 1);
  const double init = (A.mode == kModeSmcStep) ? 0.0 : d;
  return (double)nparticles * (init + steps * per_step);
}

cudaError_t launch_pass(const asmc_exec& ex, Layout L, const PassArgs& A, uint64_t blocks,
                        cudaStream_t s) {
  if (blocks == 0) return cudaSuccess;
  ProfRec rec{};
  PassArgs Ap = A;
  if (g_prof) {
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    if (cudaMallocAsync(reinterpret_cast<void**>(&rec.drawn), sizeof(unsigned long long), s) == cudaSuccess) {
      cudaMemsetAsync(rec.drawn, 0, sizeof(unsigned long long), s);
      Ap.drawn = rec.drawn;
    }
    cudaEventRecord(rec.a, s);
  }
  const cudaError_t e = ex.precision == ASMC_PREC_FP64
                            ? launch_pass_fp64(A.tg.kind, ex.rng, L, Ap, blocks, s)
                            : launch_pass_fp32(A.tg.kind, ex.rng, L, Ap, blocks, s);
  if (g_prof) {
    cudaEventRecord(rec.b, s);
    rec.normals = pass_normals(A, A.n_local);
    g_prof_recs.push_back(rec);
  }
  return e;
}

PassArgs base_args(const asmc_target_desc* t, const asmc_kernel_desc* k) {
  PassArgs A;
  std::memset(&A, 0, sizeof A);
  A.tg = make_params(t);
  A.kc = make_kcfg(k);
  return A;
}

uint64_t nblocks(uint64_t n) { return (n + kBlock - 1) / kBlock; }

// Map the device error word / state to the reference's exception texts.
int device_error(int code, int step, double val) {
  switch (code) {
    case 0: return 0;
    case ASMC_ERR_DEGENERATE:
      return fail(ASMC_ERR_DEGENERATE, "all log-weights are -inf at step %d", step);
    case ASMC_ERR_DEGENERATE + 100:
      return fail(ASMC_ERR_DEGENERATE, "weights degenerate at step %d (max log-weight %f)", step, val);
    case ASMC_ERR_EVALUATION:
      return fail(ASMC_ERR_EVALUATION, "incremental weight undefined: gamma_beta(x) = 0");
    default:
      return fail(code, "device error %d", code);
  }
}

// Device buffers of one round's outputs.
struct RoundBufs {
  DBuf<double> g0, g1, g2, ess, cz, lam, scal;
  DBuf<uint8_t> rs;
  DBuf<int32_t> rt;
  DBuf<SmcState> st;
  DBuf<RoundDev> rd;
  RoundDev host{};
  int alloc(int T, cudaStream_t s) {
    TRY(g0.alloc(T + 1, s));
    TRY(g1.alloc(T + 1, s));
    TRY(g2.alloc(T + 1, s));
    TRY(ess.alloc(T + 1, s));
    TRY(cz.alloc(T + 1, s));
    TRY(lam.alloc(T + 1, s));
    TRY(scal.alloc(2, s));
    TRY(rs.alloc(T + 1, s));
    TRY(rt.alloc(T + 1, s));
    TRY(st.alloc(1, s));
    TRY(rd.alloc(1, s));
    CU(cudaMemsetAsync(st.p, 0, sizeof(SmcState), s));
    host = RoundDev{g0.p, g1.p, g2.p, ess.p, cz.p, rs.p, rt.p, lam.p, scal.p, st.p};
    CU(cudaMemcpyAsync(rd.p, &host, sizeof host, cudaMemcpyHostToDevice, s));
    return 0;
  }
  // the same buffers as views into one arena (asmc_run_rounds: one allocation and one
  // zero-fill for all rounds; the caller uploads `host` to rd)
  static size_t a256(size_t b) { return (b + 255) / 256 * 256; }
  static size_t carve_bytes(int T) {
    const size_t d8 = sizeof(double) * (T + 1);
    return 6 * a256(d8) + a256(2 * sizeof(double)) + a256(T + 1) + a256(sizeof(int32_t) * (T + 1)) +
           a256(sizeof(SmcState)) + a256(sizeof(RoundDev));
  }
  void carve(int T, char*& cur) {
    const size_t d8 = sizeof(double) * (T + 1);
    auto take = [&](size_t b) {
      char* r = cur;
      cur += a256(b);
      return r;
    };
    g0.borrow(reinterpret_cast<double*>(take(d8)));
    g1.borrow(reinterpret_cast<double*>(take(d8)));
    g2.borrow(reinterpret_cast<double*>(take(d8)));
    ess.borrow(reinterpret_cast<double*>(take(d8)));
    cz.borrow(reinterpret_cast<double*>(take(d8)));
    lam.borrow(reinterpret_cast<double*>(take(d8)));
    scal.borrow(reinterpret_cast<double*>(take(2 * sizeof(double))));
    rs.borrow(reinterpret_cast<uint8_t*>(take(T + 1)));
    rt.borrow(reinterpret_cast<int32_t*>(take(sizeof(int32_t) * (T + 1))));
    st.borrow(reinterpret_cast<SmcState*>(take(sizeof(SmcState))));
    rd.borrow(reinterpret_cast<RoundDev*>(take(sizeof(RoundDev))));
    host = RoundDev{g0.p, g1.p, g2.p, ess.p, cz.p, rs.p, rt.p, lam.p, scal.p, st.p};
  }
};

// ---------------------------------------------------------------- SAIS --
// One SAIS round over particles [0, n): fused pass + fold + report.
struct SaisWork {
  DBuf<LogAcc> part, chunk, tot;
  DBuf<char> xs;  // long-T tiles: particle rows between tiles
  DBuf<void*> xbuf;
  DBuf<int> xcur;
  DBuf<double> lw;
};

// The SAIS pass over steps 1..T for particles [p_begin, p_begin + n_local): one launch,
// or t-tiles (sais_tile_rows) with the particle rows in HBM between them.  Either way
// the same per-(block, step) partials, bit for bit (tests/test_gpu_long_t.py).
int launch_sais_pass(DevCtx* C, const asmc_exec& ex, Layout L, PassArgs A, uint64_t nblk, int T,
                     DBuf<char>& xs, DBuf<void*>& xbuf, DBuf<int>& xcur, DBuf<double>& lw) {
  const int tile = sais_tile_rows(L, A.tg.dim, T);
  A.T = T;
  A.row_base = 0;
  if (tile >= T) {
    A.t_begin = 1;
    A.t_end = T;
    A.mode = kModeSais;
    LCH(launch_pass(ex, L, A, nblk, C->stream));
    return 0;
  }
  const size_t real = ex.precision == ASMC_PREC_FP64 ? sizeof(double) : sizeof(float);
  TRY(xs.alloc(A.n_local * A.tg.dim * real, C->stream));
  TRY(xbuf.alloc(2, C->stream));
  TRY(xcur.alloc(1, C->stream));
  TRY(lw.alloc(A.n_local, C->stream));
  void* ptrs[2] = {xs.p, xs.p};
  CU(cudaMemcpyAsync(xbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(xcur.p, 0, sizeof(int), C->stream));
  A.xbuf = xbuf.p;
  A.xcur = xcur.p;
  A.lw = lw.p;
  for (int t0 = 1; t0 <= T; t0 += tile) {
    A.t_begin = t0;
    A.t_end = t0 + tile - 1 < T ? t0 + tile - 1 : T;
    A.mode = t0 == 1 ? kModeSaisFirst : kModeSaisNext;
    LCH(launch_pass(ex, L, A, nblk, C->stream));
  }
  return 0;
}

int enqueue_sais_round(DevCtx* C, const asmc_exec& ex, Layout L, const PassArgs& base,
                       const double* d_betas, int T, uint64_t n, uint64_t seed, uint64_t round,
                       RoundDev* d_rd, int* d_err, SaisWork& W) {
  const uint64_t nblk = nblocks(n);
  const uint64_t nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  TRY(W.part.alloc((size_t)(T + 1) * kNAcc * nblk, C->stream));
  TRY(W.chunk.alloc((size_t)(T + 1) * kNAcc * nchunks, C->stream));
  TRY(W.tot.alloc((size_t)(T + 1) * kNAcc, C->stream));
  PassArgs A = base;
  A.betas = d_betas;
  A.n = n;
  A.p_begin = 0;
  A.n_local = n;
  A.seed = seed;
  A.round = round;
  A.part = W.part.p;
  A.part_stride = nblk;
  A.err = d_err;
  TRY(launch_sais_pass(C, ex, L, A, nblk, T, W.xs, W.xbuf, W.xcur, W.lw));
  LCH(launch_fold(ex.precision == ASMC_PREC_FP64, W.part.p, nblk, nblk, 1, T, 4, W.chunk.p, W.tot.p,
                  C->stream));
  LCH(launch_sais_report(W.tot.p, T, n, d_rd, C->stream));
  return 0;
}

// ---------------------------------------------------------------- SSMC --
struct SmcWork {
  DBuf<char> xa, xb;
  DBuf<void*> xbuf;
  DBuf<int> xcur;
  DBuf<double> lw, cum, btot;
  DBuf<uint32_t> anc;
  DBuf<LogAcc> part, chunk, tot;
};

int enqueue_smc_round(DevCtx* C, const asmc_exec& ex, Layout L, const PassArgs& base,
                      const double* d_betas, int T, uint64_t n, int policy, double rho,
                      uint64_t seed, uint64_t round, RoundDev* d_rd, SmcState* d_st, SmcWork& W) {
  const uint64_t d = base.tg.dim;
  const size_t real = ex.precision == ASMC_PREC_FP64 ? sizeof(double) : sizeof(float);
  const uint64_t nblk = nblocks(n);
  const uint64_t nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  TRY(W.xa.alloc(n * d * real, C->stream));
  TRY(W.xb.alloc(n * d * real, C->stream));
  TRY(W.xbuf.alloc(2, C->stream));
  TRY(W.xcur.alloc(1, C->stream));
  TRY(W.lw.alloc(n, C->stream));
  TRY(W.cum.alloc(n, C->stream));
  TRY(W.btot.alloc(refcdf_work_doubles(n), C->stream));  // refcdf scratch
  TRY(W.anc.alloc(n, C->stream));
  TRY(W.part.alloc((size_t)kNAcc * nblk, C->stream));
  TRY(W.chunk.alloc((size_t)kNAcc * nchunks, C->stream));
  TRY(W.tot.alloc(kNAcc, C->stream));
  void* ptrs[2] = {W.xa.p, W.xb.p};
  CU(cudaMemcpyAsync(W.xbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(W.xcur.p, 0, sizeof(int), C->stream));

  PassArgs A = base;
  A.betas = d_betas;
  A.T = T;
  A.n = n;
  A.p_begin = 0;
  A.n_local = n;
  A.seed = seed;
  A.round = round;
  A.xbuf = W.xbuf.p;
  A.xcur = W.xcur.p;
  A.lw = W.lw.p;
  A.part = W.part.p;
  A.part_stride = nblk;
  A.err = &d_st->err;
  A.mode = kModeSmcInit;  // engine_detail.hpp:91-100
  LCH(launch_pass(ex, L, A, nblk, C->stream));
  const bool exact = ex.precision == ASMC_PREC_FP64;
  // engine.cpp:161-173's gather x_new[m] = x[a_m], lw <- 0 is deferred into the next step
  // pass: it reads row a_m and starts from log w = 0 (PassArgs::anc / pend), so a
  // resampling event moves no rows of its own (2 n d B of HBM traffic saved per event)
  A.anc = W.anc.p;
  A.pend = &d_st->gather_pending;
  for (int t = 1; t <= T; ++t) {
    A.mode = kModeSmcStep;
    A.t_begin = A.t_end = t;
    A.row_base = t;
    LCH(launch_pass(ex, L, A, nblk, C->stream));
    if (t > 1) LCH(launch_settle(W.xcur.p, d_st, C->stream));
    LCH(launch_fold(exact, W.part.p, nblk, nblk, 0, 1, kNAcc, W.chunk.p, W.tot.p, C->stream));
    LCH(launch_smc_decide(W.tot.p, t, T, n, policy, rho, seed, round, ex.rng, d_rd, C->stream));
    LCH(launch_resample_ref(C, W.lw.p, n, d_st, W.btot.p, W.cum.p, W.anc.p));
    LCH(launch_defer_gather(d_st, C->stream));
    g_launches += 1;
  }
  // a final-step event leaves its gather pending: no caller reads a round's final
  // particles (the reports come from the accumulators), so the copy is never made
  return 0;
}

// ------------------------------------------------- config 4: logistic --
// Data-backed target: X and y uploaded once per call, X split into bf16 hi/lo
// rows padded to the 128-row MMA tile, TMA descriptors over both halves.
struct LgData {
  DBuf<float> raw;  // X (n x d) then y (n), fp32 as given
  DBuf<uint16_t> hi, lo;
  DBuf<double> w;  // X^T y
  CUtensorMap mhi, mlo;
  uint64_t n = 0, n_pad = 0;
  int d = 0;
};

int lg_check(const asmc_target_desc* t, const asmc_kernel_desc* k, const asmc_exec& ex) {
  if (ex.rng != ASMC_RNG_PHILOX || ex.precision != ASMC_PREC_FP32)
    return fail(ASMC_ERR_CAPABILITY,
                "the logistic-regression target runs on the tensor-core path: rng = philox, precision = fp32");
  if (t->dim % 64 != 0 || t->dim > 256)
    return fail(ASMC_ERR_CAPABILITY, "logistic target needs dim a multiple of 64, at most 256");
  if (k->kind != ASMC_KERNEL_RWMH && k->kind != ASMC_KERNEL_IDENTITY)
    return fail(ASMC_ERR_CAPABILITY, "logistic target supports the rwmh_cycle and identity kernels");
  return 0;
}

int lg_upload(DevCtx* C, const asmc_target_desc* t, LgData& D) {
  D.d = (int)t->dim;
  D.n = (uint64_t)t->p[1];
  D.n_pad = (D.n + 127) / 128 * 128;
  TRY(D.raw.alloc(D.n * (D.d + 1), C->stream));
  CU(cudaMemcpyAsync(D.raw.p, t->data, D.n * (D.d + 1) * sizeof(float), cudaMemcpyHostToDevice, C->stream));
  TRY(D.hi.alloc(D.n_pad * D.d, C->stream));
  TRY(D.lo.alloc(D.n_pad * D.d, C->stream));
  LCH(launch_lg_split(D.raw.p, D.n, D.d, D.n_pad, D.hi.p, D.lo.p, C->stream));
  TRY(D.w.alloc(D.d, C->stream));
  LCH(launch_lg_xty(D.raw.p, D.raw.p + D.n * (uint64_t)D.d, D.n, D.d, D.w.p, C->stream));
  CU(make_x_maps(D.hi.p, D.lo.p, D.n_pad, D.d, &D.mhi, &D.mlo));
  return 0;
}

struct LgWork {
  DBuf<float> sa, sb;
  DBuf<float*> sbuf;
  DBuf<int> xcur;
  DBuf<double> lw, cum, btot;
  DBuf<uint32_t> anc;
  DBuf<LogAcc> part, chunk, tot;
};

// one likelihood evaluation launch, timed like the particle pass when profiling
int lg_eval(DevCtx* C, const LgData& D, const LgArgs& A, int mode, const double* betas, float step, int q) {
  ProfRec rec{};
  if (g_prof) {
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, C->stream);
  }
  LCH(launch_lg_eval(D.mhi, D.mlo, A, mode, betas, step, q, C->stream));
  if (g_prof) {
    cudaEventRecord(rec.b, C->stream);
    rec.normals = 2.0 * (double)D.n * D.d * (double)A.n_local;  // algorithmic flops of X theta'
    g_prof_recs.push_back(rec);
  }
  return 0;
}

// one lattice-move launch, timed like the particle pass when profiling
int is_move(DevCtx* C, const IsArgs& A, int mode, const double* betas, int t) {
  ProfRec rec{};
  if (g_prof) {
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, C->stream);
  }
  LCH(launch_is_move(A, mode, betas, t, C->stream));
  if (g_prof) {
    cudaEventRecord(rec.b, C->stream);
    // algorithmic unit: site-gradient evaluations (HMC: leapfrog + 1 per trajectory; RWMH: 1 energy)
    const double traj = mode == 1 && A.kc.kind != ASMC_KERNEL_IDENTITY ? (double)A.kc.sweeps * A.kc.n_steps : 0.0;
    const double per = A.kc.kind == ASMC_KERNEL_HMC ? (double)(A.kc.leapfrog + 1) : 1.0;
    rec.normals = (double)A.L * A.L * (double)A.n_local * (1.0 + traj * per);
    g_prof_recs.push_back(rec);
  }
  return 0;
}

// run_smc (engine.cpp:97-188) for the logistic target: step-outer because the
// likelihood of all particles is one GEMM per proposal (SAIS = policy never).
// chunk_out != nullptr: SAIS partial mode for particles [p_begin, p_begin + n) of a
// sharded round (asmc_sais_partials): per step the chunk partials of g0 g1 g2 elbo are
// written to chunk_out[(t * kNAcc + a) * nch + c]; no decision / resampling.
int enqueue_lg_round(DevCtx* C, const LgData& D, const asmc_target_desc* t, const asmc_kernel_desc* k,
                     const double* d_betas, int T, uint64_t n, int policy, double rho, uint64_t seed,
                     uint64_t round, RoundDev* d_rd, SmcState* d_st, LgWork& W, uint64_t p_begin = 0,
                     LogAcc* chunk_out = nullptr, int* d_err = nullptr) {
  const int d = D.d, row = d + 4;
  const uint64_t nblk = nblocks(n), nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  TRY(W.sa.alloc(n * row, C->stream));
  TRY(W.sb.alloc(n * row, C->stream));
  TRY(W.sbuf.alloc(2, C->stream));
  TRY(W.xcur.alloc(1, C->stream));
  TRY(W.lw.alloc(n, C->stream));
  TRY(W.cum.alloc(n, C->stream));
  TRY(W.btot.alloc(refcdf_work_doubles(n), C->stream));  // refcdf scratch
  TRY(W.anc.alloc(n, C->stream));
  TRY(W.part.alloc((size_t)kNAcc * nblk, C->stream));
  TRY(W.chunk.alloc((size_t)kNAcc * nchunks, C->stream));
  TRY(W.tot.alloc(kNAcc, C->stream));
  float* ptrs[2] = {W.sa.p, W.sb.p};
  CU(cudaMemcpyAsync(W.sbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(W.xcur.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(W.lw.p, 0, n * sizeof(double), C->stream));
  LgArgs A;
  std::memset(&A, 0, sizeof A);
  A.state = W.sbuf.p;
  A.xcur = W.xcur.p;
  A.lw = W.lw.p;
  A.y = D.raw.p + D.n * (uint64_t)d;
  A.w = D.w.p;
  A.n = D.n;
  A.n_local = n;
  A.d = d;
  A.row = row;
  A.seed = seed;
  A.round = round;
  A.sigma_p = t->p[0];
  A.err = chunk_out ? d_err : &d_st->err;
  A.p_begin = p_begin;
  LCH(launch_lg_init(A, C->stream));        // engine_detail.hpp:91-100
  TRY(lg_eval(C, D, A, 0, d_betas, 0.f, 0));  // V(theta_0)
  const int nprop = k->kind == ASMC_KERNEL_RWMH ? k->sweeps * k->n_step_sizes : 0;
  for (int s = 1; s <= T; ++s) {
    A.t = s;
    LCH(launch_lg_weight(A, d_betas, s, W.part.p, nblk, C->stream));
    if (chunk_out) {
      LCH(launch_fold_chunks(W.part.p, nblk, nblk, 0, 1, 4, nchunks, chunk_out + (size_t)s * kNAcc * nchunks,
                             C->stream));
      for (int q = 0; q < nprop; ++q)
        TRY(lg_eval(C, D, A, 1, d_betas, (float)k->step_sizes[q % k->n_step_sizes], q));
      continue;
    }
    LCH(launch_fold(false, W.part.p, nblk, nblk, 0, 1, kNAcc, W.chunk.p, W.tot.p, C->stream));
    LCH(launch_smc_decide(W.tot.p, s, T, n, policy, rho, seed, round, ASMC_RNG_PHILOX, d_rd, C->stream));
    for (int q = 0; q < nprop; ++q)  // kernel.cpp:31-40 at beta_t
      TRY(lg_eval(C, D, A, 1, d_betas, (float)k->step_sizes[q % k->n_step_sizes], q));
    LCH(launch_resample_ref(C, W.lw.p, n, d_st, W.btot.p, W.cum.p, W.anc.p));
    LCH(launch_gather(W.anc.p, n, (uint64_t)row * sizeof(float), reinterpret_cast<void* const*>(W.sbuf.p),
                      W.xcur.p, W.lw.p, d_st, C->sms, C->stream));
    g_launches += 1;
  }
  return 0;
}

int copy_round(DevCtx* C, RoundBufs& R, int T, bool smc, asmc_report* out, SmcState* st);

// ------------------------------------------------------ config 5: Ising --
int is_check(const asmc_target_desc* t, const asmc_kernel_desc* k, const asmc_exec& ex) {
  if (ex.rng != ASMC_RNG_PHILOX || ex.precision != ASMC_PREC_FP32)
    return fail(ASMC_ERR_CAPABILITY, "the ising target runs on the fp32 lattice path: rng = philox, precision = fp32");
  if (!ising_side_supported((int)t->p[0]))
    return fail(ASMC_ERR_CAPABILITY, "ising device kernels support L in {8, 16, 32, 64}");
  if (k->kind != ASMC_KERNEL_RWMH && k->kind != ASMC_KERNEL_HMC && k->kind != ASMC_KERNEL_IDENTITY)
    return fail(ASMC_ERR_CAPABILITY, "ising target supports the rwmh_cycle, hmc and identity kernels");
  return 0;
}

IsArgs is_args(const asmc_target_desc* t, const asmc_kernel_desc* k) {
  IsArgs A;
  std::memset(&A, 0, sizeof A);
  const int L = (int)t->p[0];
  const double n = (double)L * L;
  A.L = L;
  A.row = L * L + 4;
  A.K = (float)t->p[1];
  A.c = (float)(t->p[2] + 4.0 * t->p[1]);
  A.inv_s2 = (float)(1.0 / (t->p[3] * t->p[3]));
  A.sigma = (float)t->p[3];
  A.vconst = n * (std::log(t->p[3]) + 0.91893853320467274178);
  A.kc = make_kcfg(k);
  return A;
}

// run_smc (engine.cpp:97-188) for the lattice target, step-outer: per step the weight
// kernel (lg = dbeta V(y), V cached in the state row), fold, decide, one move launch
// (the whole RWMH / HMC cycle at beta_t per particle), resample + gather.
int enqueue_is_round(DevCtx* C, const asmc_target_desc* t, const asmc_kernel_desc* k, const double* d_betas,
                     int T, uint64_t n, int policy, double rho, uint64_t seed, uint64_t round, RoundDev* d_rd,
                     SmcState* d_st, LgWork& W, uint64_t p_begin = 0, LogAcc* chunk_out = nullptr,
                     int* d_err = nullptr) {
  IsArgs I = is_args(t, k);
  const int row = I.row;
  const uint64_t nblk = nblocks(n), nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  TRY(W.sa.alloc(n * row, C->stream));
  TRY(W.sb.alloc(n * row, C->stream));
  TRY(W.sbuf.alloc(2, C->stream));
  TRY(W.xcur.alloc(1, C->stream));
  TRY(W.lw.alloc(n, C->stream));
  TRY(W.cum.alloc(n, C->stream));
  TRY(W.btot.alloc(refcdf_work_doubles(n), C->stream));  // refcdf scratch
  TRY(W.anc.alloc(n, C->stream));
  TRY(W.part.alloc((size_t)kNAcc * nblk, C->stream));
  TRY(W.chunk.alloc((size_t)kNAcc * nchunks, C->stream));
  TRY(W.tot.alloc(kNAcc, C->stream));
  float* ptrs[2] = {W.sa.p, W.sb.p};
  CU(cudaMemcpyAsync(W.sbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(W.xcur.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(W.lw.p, 0, n * sizeof(double), C->stream));
  I.state = W.sbuf.p;
  I.xcur = W.xcur.p;
  I.n_local = n;
  I.p_begin = p_begin;
  I.seed = seed;
  I.round = round;
  I.err = chunk_out ? d_err : &d_st->err;
  LgArgs A;  // the weight kernel and gather see the same state-row layout
  std::memset(&A, 0, sizeof A);
  A.state = W.sbuf.p;
  A.xcur = W.xcur.p;
  A.lw = W.lw.p;
  A.n_local = n;
  A.d = I.L * I.L;
  A.row = row;
  A.err = I.err;
  TRY(is_move(C, I, 0, d_betas, 0));  // engine_detail.hpp:91-100 (+ V(y_0))
  for (int s = 1; s <= T; ++s) {
    LCH(launch_lg_weight(A, d_betas, s, W.part.p, nblk, C->stream));
    if (chunk_out) {  // SAIS partial mode (see enqueue_lg_round)
      LCH(launch_fold_chunks(W.part.p, nblk, nblk, 0, 1, 4, nchunks, chunk_out + (size_t)s * kNAcc * nchunks,
                             C->stream));
      TRY(is_move(C, I, 1, d_betas, s));
      continue;
    }
    LCH(launch_fold(false, W.part.p, nblk, nblk, 0, 1, kNAcc, W.chunk.p, W.tot.p, C->stream));
    LCH(launch_smc_decide(W.tot.p, s, T, n, policy, rho, seed, round, ASMC_RNG_PHILOX, d_rd, C->stream));
    TRY(is_move(C, I, 1, d_betas, s));  // kernel.cpp:26-63 at beta_t
    LCH(launch_resample_ref(C, W.lw.p, n, d_st, W.btot.p, W.cum.p, W.anc.p));
    LCH(launch_gather(W.anc.p, n, (uint64_t)row * sizeof(float), reinterpret_cast<void* const*>(W.sbuf.p),
                      W.xcur.p, W.lw.p, d_st, C->sms, C->stream));
    g_launches += 1;
  }
  return 0;
}

int run_is_single(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas, int T,
                  uint64_t n, int policy, double rho, uint64_t seed, uint64_t round, const asmc_exec& ex,
                  asmc_report* out, bool smc) {
  TRY(is_check(target, kernel, ex));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const double t0 = now_s();
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  LgWork W;
  TRY(enqueue_is_round(C, target, kernel, d_betas.p, T, n, policy, rho, seed, round, R.rd.p, R.st.p, W));
  SmcState st;
  TRY(copy_round(C, R, T, smc, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  out->wall_seconds = now_s() - t0;
  return 0;
}


// asmc_run_smc / asmc_run_sais_single body for the logistic target
int run_lg_single(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas, int T,
                  uint64_t n, int policy, double rho, uint64_t seed, uint64_t round, const asmc_exec& ex,
                  asmc_report* out, bool smc) {
  TRY(lg_check(target, kernel, ex));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const double t0 = now_s();
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  LgData D;
  TRY(lg_upload(C, target, D));
  LgWork W;
  TRY(enqueue_lg_round(C, D, target, kernel, d_betas.p, T, n, policy, rho, seed, round, R.rd.p, R.st.p, W));
  SmcState st;
  TRY(copy_round(C, R, T, smc, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  out->wall_seconds = now_s() - t0;
  return 0;
}

// asmc_sais_partials for the step-outer engines (logistic: tcgen05 likelihood; Ising:
// lattice moves): the engine runs its particle range in SAIS partial mode and the
// per-step chunk partials are returned in the fused pass's layout.
int stepouter_partials(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas, int T,
                       uint64_t p_begin, uint64_t p_end, uint64_t seed, uint64_t round, const asmc_exec& ex,
                       asmc_logacc* partials) {
  const bool lg = target->kind == ASMC_TARGET_LOGISTIC;
  TRY(lg ? lg_check(target, kernel, ex) : is_check(target, kernel, ex));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const uint64_t nloc = p_end - p_begin;
  const uint64_t nch = asmc_fold_chunks(p_begin, p_end);
  if (nch == 0) return 0;
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  DBuf<LogAcc> chunk;
  DBuf<int> err;
  TRY(chunk.alloc((size_t)(T + 1) * kNAcc * nch, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  LgWork W;
  if (lg) {
    LgData D;
    TRY(lg_upload(C, target, D));
    TRY(enqueue_lg_round(C, D, target, kernel, d_betas.p, T, nloc, ASMC_POLICY_NEVER, 0.5, seed, round, nullptr,
                         nullptr, W, p_begin, chunk.p, err.p));
    CU(cudaStreamSynchronize(C->stream));  // D (the uploaded data) is released at scope exit
  } else {
    TRY(enqueue_is_round(C, target, kernel, d_betas.p, T, nloc, ASMC_POLICY_NEVER, 0.5, seed, round, nullptr,
                         nullptr, W, p_begin, chunk.p, err.p));
  }
  std::vector<LogAcc> h((size_t)(T + 1) * kNAcc * nch);
  CU(cudaMemcpyAsync(h.data(), chunk.p, h.size() * sizeof(LogAcc), cudaMemcpyDeviceToHost, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  TRY(device_error(herr, 0, 0.0));
  for (uint64_t c = 0; c < nch; ++c)
    for (int t = 0; t <= T; ++t)
      for (int a = 0; a < 4; ++a) {
        const LogAcc v = t == 0 ? LogAcc{-HUGE_VAL, 0.0} : h[((size_t)t * kNAcc + a) * nch + c];
        partials[(c * (T + 1) + t) * 4 + a] = asmc_logacc{v.max, v.sum};
      }
  return 0;
}

int copy_round(DevCtx* C, RoundBufs& R, int T, bool smc, asmc_report* out, SmcState* st) {
  // one page-locked staging area, one synchronisation (see asmc_run_rounds)
  cudaStream_t s = C->stream;
  const size_t d8 = sizeof(double) * (T + 1);
  const size_t o_g0 = 0, o_g1 = d8, o_g2 = 2 * d8, o_es = 3 * d8, o_cz = 4 * d8, o_scal = 5 * d8,
               o_st = o_scal + 16, o_rt = o_st + (sizeof(SmcState) + 15) / 16 * 16,
               o_rs = o_rt + (sizeof(int32_t) * (T + 1) + 15) / 16 * 16, bytes = o_rs + T + 1;
  char* H;
  TRY(pinned_staging(C, bytes, &H));
  auto get = [&](const void* src, size_t off, size_t n, bool want) -> int {
    if (!want) return 0;
    CU(cudaMemcpyAsync(H + off, src, n, cudaMemcpyDeviceToHost, s));
    return 0;
  };
  TRY(get(R.g0.p, o_g0, d8, out->log_g0 != nullptr));
  TRY(get(R.g1.p, o_g1, d8, out->log_g1 != nullptr));
  TRY(get(R.g2.p, o_g2, d8, out->log_g2 != nullptr));
  TRY(get(R.ess.p, o_es, d8, smc && out->ess_trace != nullptr));
  TRY(get(R.cz.p, o_cz, d8, out->cum_log_z != nullptr));
  TRY(get(R.rs.p, o_rs, T + 1, out->resampled != nullptr));
  TRY(get(R.scal.p, o_scal, 2 * sizeof(double), true));
  TRY(get(R.st.p, o_st, sizeof(SmcState), true));
  TRY(get(R.rt.p, o_rt, sizeof(int32_t) * (T + 1), smc));
  CU(cudaStreamSynchronize(s));
  if (out->log_g0) std::memcpy(out->log_g0, H + o_g0, d8);
  if (out->log_g1) std::memcpy(out->log_g1, H + o_g1, d8);
  if (out->log_g2) std::memcpy(out->log_g2, H + o_g2, d8);
  if (smc && out->ess_trace) std::memcpy(out->ess_trace, H + o_es, d8);
  if (out->cum_log_z) std::memcpy(out->cum_log_z, H + o_cz, d8);
  if (out->resampled) std::memcpy(out->resampled, H + o_rs, T + 1);
  double scal[2];
  std::memcpy(scal, H + o_scal, sizeof scal);
  std::memcpy(st, H + o_st, sizeof(SmcState));
  out->log_z_hat = scal[0];
  out->elbo_hat = scal[1];
  if (smc) {
    out->n_resample_times = st->n_resample;
    if (out->resample_times)
      std::memcpy(out->resample_times, H + o_rt, sizeof(int32_t) * (size_t)st->n_resample);
  } else {
    out->n_resample_times = 1;
    if (out->resample_times) out->resample_times[0] = T;
  }
  return 0;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* asmc_last_error(void) { return g_err.c_str(); }
int asmc_version(void) { return 1; }
int asmc_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}
uint64_t asmc_launch_count(int reset) {
  const uint64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

int asmc_run_sais_single(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                         const double* betas, int32_t T, uint64_t n, uint64_t seed,
                         uint64_t round, const asmc_exec* exec, asmc_report* out) {
  TRY(check_schedule(betas, T));
  if (n < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  TRY(check_pair(target, kernel));
  if (!out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null report");
  const asmc_exec ex = exec ? *exec : default_exec();
  if (target->kind == ASMC_TARGET_LOGISTIC)  // SAIS == run_smc(never) (drivers.hpp:80-86)
    return run_lg_single(target, kernel, betas, T, n, ASMC_POLICY_NEVER, 0.5, seed, round, ex, out, false);
  if (target->kind == ASMC_TARGET_ISING)
    return run_is_single(target, kernel, betas, T, n, ASMC_POLICY_NEVER, 0.5, seed, round, ex, out, false);
  Layout L;
  TRY(choose_layout(ex, kernel->kind, target->dim, &L, 1, 4));  // long T runs in t-tiles
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const double t0 = now_s();
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  SaisWork W;
  const PassArgs base = base_args(target, kernel);
  TRY(enqueue_sais_round(C, ex, L, base, d_betas.p, T, n, seed, round, R.rd.p, &R.st.p->err, W));
  SmcState st;
  TRY(copy_round(C, R, T, false, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  out->wall_seconds = now_s() - t0;
  return 0;
}

int asmc_run_smc(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                 const double* betas, int32_t T, uint64_t n, int32_t policy, double rho,
                 uint64_t seed, uint64_t round, const asmc_exec* exec, asmc_report* out) {
  TRY(check_schedule(betas, T));
  if (n < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "rho must lie in [0, 1]");
  if (policy < ASMC_POLICY_NEVER || policy > ASMC_POLICY_STABILIZED)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown resampling policy");
  TRY(check_pair(target, kernel));
  if (!out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null report");
  if (n > 0xffffffffull) return fail(ASMC_ERR_CAPABILITY, "ancestor indices are 32-bit");
  const asmc_exec ex = exec ? *exec : default_exec();
  if (target->kind == ASMC_TARGET_LOGISTIC)
    return run_lg_single(target, kernel, betas, T, n, policy, rho, seed, round, ex, out, true);
  if (target->kind == ASMC_TARGET_ISING)
    return run_is_single(target, kernel, betas, T, n, policy, rho, seed, round, ex, out, true);
  Layout L;
  TRY(choose_layout(ex, kernel->kind, target->dim, &L));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const double t0 = now_s();
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  SmcWork W;
  const PassArgs base = base_args(target, kernel);
  TRY(enqueue_smc_round(C, ex, L, base, d_betas.p, T, n, policy, rho, seed, round, R.rd.p, R.st.p, W));
  SmcState st;
  TRY(copy_round(C, R, T, true, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  out->wall_seconds = now_s() - t0;
  return 0;
}

int asmc_budget(uint64_t n, int32_t steps, uint64_t dim, uint64_t cap, int32_t mode,
                uint64_t* n_out, int32_t* t_out) {
  // drivers.cpp:33-49 (integer/double plumbing of the round loop)
  if (n < 1 || steps < 1)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "budget needs n_particles and steps >= 1");
  const double root2 = std::sqrt(2.0);
  const uint64_t gn = (uint64_t)std::ceil(root2 * (double)n);
  const int gt = (int)std::ceil(root2 * (double)steps);
  if (mode == ASMC_MODE_SSMC) {
    const double bytes = (double)gn * (double)dim * 8.0;
    if (bytes > (double)cap) {
      *n_out = n;
      *t_out = 2 * steps;
      return 0;
    }
  }
  *n_out = gn;
  *t_out = gt;
  return 0;
}

int asmc_run_rounds(const asmc_target_desc* target, const asmc_kernel_desc* kernel, int32_t mode,
                    uint64_t n1, int32_t rounds, int32_t policy, double rho, uint64_t seed,
                    uint64_t memory_cap, const asmc_exec* exec, asmc_rounds_out* out) {
  // DriverOptions::validate (drivers.cpp:16-21)
  if (n1 < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (rounds < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "rounds must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "rho must lie in [0, 1]");
  if (mode != ASMC_MODE_SAIS && mode != ASMC_MODE_SSMC)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown driver mode");
  TRY(check_pair(target, kernel));
  if (!out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null output");
  const asmc_exec ex = exec ? *exec : default_exec();
  Layout L;
  const bool lg = target->kind == ASMC_TARGET_LOGISTIC;
  const bool is = target->kind == ASMC_TARGET_ISING;
  if (lg) {
    TRY(lg_check(target, kernel, ex));
    L = Layout{1, 0};
  } else if (is) {
    TRY(is_check(target, kernel, ex));
    L = Layout{1, 0};
  } else {
    TRY(choose_layout_impl(ex, kernel->kind, target->dim, &L));
  }
  // The (N_k, T_k) plan depends on the budget rule only, so the whole round
  // loop is enqueued up front; only the betas are data-dependent (device).
  std::vector<uint64_t> ns(rounds);
  std::vector<int> ts(rounds);
  ns[0] = n1;
  ts[0] = 1;
  for (int k = 1; k < rounds; ++k) TRY(asmc_budget(ns[k - 1], ts[k - 1], target->dim, memory_cap, mode, &ns[k], &ts[k]));
  int tmax = 0;
  for (int k = 0; k < rounds; ++k) tmax = ts[k] > tmax ? ts[k] : tmax;
  TRY(check_smem(L, target->dim, 1, mode == ASMC_MODE_SAIS ? 4 : kNAcc));  // SAIS: long T in t-tiles
  if (tmax > out->max_steps) return fail(ASMC_ERR_INVALID_ARGUMENT, "max_steps too small (%d needed)", tmax);
  if (mode == ASMC_MODE_SSMC)
    for (int k = 0; k < rounds; ++k)
      if (ns[k] > 0xffffffffull) return fail(ASMC_ERR_CAPABILITY, "ancestor indices are 32-bit");
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  LgData lgd;
  if (lg) TRY(lg_upload(C, target, lgd));
  const int stride = out->max_steps + 1;
  // every round's outputs, schedules and scratch in one arena (one allocation, one
  // zero-fill), the uploads from the page-locked staging, the timing events reused: a
  // small run (config 1) is otherwise dominated by ~50 tiny allocations and copies
  std::vector<RoundBufs> R(rounds);
  std::vector<DBuf<double>> betas(rounds);
  DBuf<double> sched_scratch;
  DBuf<int> gerr;  // pass-kernel evaluation errors and schedule-generation failures
  size_t arena_bytes = 256 + RoundBufs::a256(sizeof(double) * 5 * (tmax + 1));
  for (int k = 0; k < rounds; ++k)
    arena_bytes += RoundBufs::carve_bytes(ts[k]) + RoundBufs::a256(sizeof(double) * (ts[k] + 1));
  DBuf<char> arena;
  TRY(arena.alloc(arena_bytes, C->stream));
  CU(cudaMemsetAsync(arena.p, 0, arena_bytes, C->stream));  // SmcState, gerr = 0
  {
    char* cur = arena.p;
    gerr.borrow(reinterpret_cast<int*>(cur));
    cur += 256;
    sched_scratch.borrow(reinterpret_cast<double*>(cur));
    cur += RoundBufs::a256(sizeof(double) * 5 * (tmax + 1));
    for (int k = 0; k < rounds; ++k) {
      R[k].carve(ts[k], cur);
      betas[k].borrow(reinterpret_cast<double*>(cur));
      cur += RoundBufs::a256(sizeof(double) * (ts[k] + 1));
    }
  }
  // the results come back as ONE copy of the arena into the page-locked staging (after
  // the rounds, see below); the uploads use the staging's head before that
  const size_t up_bytes = 16 + sizeof(RoundDev) * rounds;
  char* H;
  TRY(pinned_staging(C, arena_bytes > up_bytes ? arena_bytes : up_bytes, &H));
  {
    const double b01[2] = {0.0, 1.0};
    std::memcpy(H, b01, sizeof b01);
    for (int k = 0; k < rounds; ++k) std::memcpy(H + 16 + sizeof(RoundDev) * k, &R[k].host, sizeof(RoundDev));
    CU(cudaMemcpyAsync(betas[0].p, H, sizeof b01, cudaMemcpyHostToDevice, C->stream));
    for (int k = 0; k < rounds; ++k)
      CU(cudaMemcpyAsync(R[k].rd.p, H + 16 + sizeof(RoundDev) * k, sizeof(RoundDev), cudaMemcpyHostToDevice,
                         C->stream));
  }
  const PassArgs base = base_args(target, kernel);
  while ((int)C->events.size() < rounds + 1) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    C->events.push_back(e);
  }
  const std::vector<cudaEvent_t> ev(C->events.begin(), C->events.begin() + rounds + 1);
  CU(cudaEventRecord(ev[0], C->stream));
  for (int k = 0; k < rounds; ++k) {
    if (lg) {  // config 4: step-outer tensor-core engine (SAIS = policy never)
      LgWork w;
      TRY(enqueue_lg_round(C, lgd, target, kernel, betas[k].p, ts[k], ns[k],
                           mode == ASMC_MODE_SAIS ? ASMC_POLICY_NEVER : policy, rho, seed,
                           (uint64_t)(k + 1), R[k].rd.p, R[k].st.p, w));
    } else if (is) {  // config 5: step-outer lattice engine (SAIS = policy never)
      LgWork w;
      TRY(enqueue_is_round(C, target, kernel, betas[k].p, ts[k], ns[k],
                           mode == ASMC_MODE_SAIS ? ASMC_POLICY_NEVER : policy, rho, seed, (uint64_t)(k + 1),
                           R[k].rd.p, R[k].st.p, w));
    } else if (mode == ASMC_MODE_SAIS) {
      SaisWork w;  // stream-ordered: freed after this round's kernels retire
      TRY(enqueue_sais_round(C, ex, L, base, betas[k].p, ts[k], ns[k], seed, (uint64_t)(k + 1),
                             R[k].rd.p, gerr.p, w));
    } else {
      SmcWork w;
      TRY(enqueue_smc_round(C, ex, L, base, betas[k].p, ts[k], ns[k], policy, rho, seed,
                            (uint64_t)(k + 1), R[k].rd.p, R[k].st.p, w));
    }
    if (k + 1 < rounds) {
      LCH(launch_generate_schedule(R[k].lam.p, betas[k].p, ts[k] + 1, ts[k + 1], betas[k + 1].p,
                                   sched_scratch.p, gerr.p, C->stream));
    }
    CU(cudaEventRecord(ev[k + 1], C->stream));
  }
  // every result of every round (the whole arena) in one copy to the page-locked staging,
  // enqueued behind the rounds: one synchronisation for the call
  CU(cudaMemcpyAsync(H, arena.p, arena_bytes, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  auto host_of = [&](const void* dp) { return H + (static_cast<const char*>(dp) - arena.p); };
  int herr = 0;
  std::memcpy(&herr, host_of(gerr.p), sizeof(int));
  int rc = 0;
  for (int k = 0; k < rounds && !rc; ++k) {
    const int T = ts[k];
    const double* g0 = reinterpret_cast<const double*>(host_of(R[k].g0.p));
    const double* g1 = reinterpret_cast<const double*>(host_of(R[k].g1.p));
    const double* g2 = reinterpret_cast<const double*>(host_of(R[k].g2.p));
    const double* es = reinterpret_cast<const double*>(host_of(R[k].ess.p));
    const double* cz = reinterpret_cast<const double*>(host_of(R[k].cz.p));
    const double* lam = reinterpret_cast<const double*>(host_of(R[k].lam.p));
    const double* b = reinterpret_cast<const double*>(host_of(betas[k].p));
    const double* scal = reinterpret_cast<const double*>(host_of(R[k].scal.p));
    const uint8_t* rs = reinterpret_cast<const uint8_t*>(host_of(R[k].rs.p));
    SmcState st;
    std::memcpy(&st, host_of(R[k].st.p), sizeof st);
    TRY(device_error(st.err, st.err_step, st.err_val));
    if (herr == ASMC_ERR_EVALUATION) return device_error(herr, 0, 0.0);
    if (herr) return fail(herr, "schedule generation after round %d failed validation", k + 1);
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
    const size_t r0 = (size_t)k * stride;
    if (out->n_particles) out->n_particles[k] = ns[k];
    if (out->steps) out->steps[k] = T;
    for (int t = 0; t <= T; ++t) {
      if (out->betas) out->betas[r0 + t] = b[t];
      if (out->log_g0) out->log_g0[r0 + t] = g0[t];
      if (out->log_g1) out->log_g1[r0 + t] = g1[t];
      if (out->log_g2) out->log_g2[r0 + t] = g2[t];
      if (out->ess_trace && mode == ASMC_MODE_SSMC) out->ess_trace[r0 + t] = es[t];
      if (out->cum_log_z) out->cum_log_z[r0 + t] = cz[t];
      if (out->resampled) out->resampled[r0 + t] = rs[t];
      if (out->lambda) out->lambda[r0 + t] = lam[t];
    }
    if (out->log_z_hat) out->log_z_hat[k] = scal[0];
    if (out->elbo_hat) out->elbo_hat[k] = scal[1];
    if (out->wall_seconds) out->wall_seconds[k] = ms * 1e-3;
    if (out->kernel_applications) out->kernel_applications[k] = ns[k] * (uint64_t)T;
  }
  return rc;
}

// Batched seeds: run_sais (drivers.cpp:186-232) for many
// seeds with the seed as an extra launch dimension -- one pass launch, one fold, one
// report and one schedule launch per round for ALL seeds (the one-lane pass: CTA
// s * nblk + b is block b of seed s).  Each seed's numbers are those of its own
// asmc_run_rounds(SAIS) call, bit for bit (same kernels, same per-seed trees).
int asmc_run_sais_seeds(const asmc_target_desc* target, const asmc_kernel_desc* kernel, uint64_t n1,
                        int32_t rounds, const uint64_t* seeds, int32_t nseeds, const asmc_exec* exec,
                        asmc_seeds_out* out) {
  if (n1 < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (rounds < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "rounds must be at least 1");
  if (nseeds < 1 || !seeds) return fail(ASMC_ERR_INVALID_ARGUMENT, "need at least one seed");
  TRY(check_pair(target, kernel));
  TRY(check_pass_target(target, "asmc_run_sais_seeds"));
  if (!out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null output");
  const asmc_exec ex = exec ? *exec : default_exec();
  const uint64_t d = target->dim;
  if (ex.lanes > 1) return fail(ASMC_ERR_CAPABILITY, "batched seeds run the one-lane pass (lanes = 1)");
  if (d > 1024) return fail(ASMC_ERR_CAPABILITY, "batched seeds support dim <= 1024");
  const Layout L{1, d <= 16 ? 16 : 1024};
  const int S = nseeds;
  std::vector<uint64_t> ns(rounds);
  std::vector<int> ts(rounds);
  ns[0] = n1;
  ts[0] = 1;
  for (int k = 1; k < rounds; ++k)
    TRY(asmc_budget(ns[k - 1], ts[k - 1], d, 4096ull << 20, ASMC_MODE_SAIS, &ns[k], &ts[k]));
  int tmax = 0;
  for (int k = 0; k < rounds; ++k) tmax = ts[k] > tmax ? ts[k] : tmax;
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  cudaStream_t st = C->stream;
  DBuf<uint64_t> d_seeds;
  TRY(d_seeds.alloc(S, st));
  CU(cudaMemcpyAsync(d_seeds.p, seeds, sizeof(uint64_t) * S, cudaMemcpyHostToDevice, st));
  std::vector<DBuf<double>> betas(rounds);
  for (int k = 0; k < rounds; ++k) TRY(betas[k].alloc((size_t)S * (ts[k] + 1), st));
  {
    std::vector<double> b01(2 * (size_t)S);
    for (int s = 0; s < S; ++s) {
      b01[2 * s] = 0.0;
      b01[2 * s + 1] = 1.0;
    }
    CU(cudaMemcpyAsync(betas[0].p, b01.data(), sizeof(double) * b01.size(), cudaMemcpyHostToDevice, st));
  }
  // per-seed round outputs: arrays of S (T + 1) (or S) entries, S RoundDev views
  struct Out {
    DBuf<double> g0, g1, g2, ess, cz, lam, scal;
    DBuf<uint8_t> rs;
    DBuf<int32_t> rt;
    DBuf<SmcState> stt;
    DBuf<RoundDev> rd;
  };
  std::vector<Out> O(rounds);
  DBuf<int> gerr, serr;
  TRY(gerr.alloc(1, st));
  TRY(serr.alloc(S, st));
  CU(cudaMemsetAsync(gerr.p, 0, sizeof(int), st));
  CU(cudaMemsetAsync(serr.p, 0, sizeof(int) * S, st));
  DBuf<double> sched_scratch;
  TRY(sched_scratch.alloc((size_t)S * 5 * (tmax + 1), st));
  const bool exact = ex.precision == ASMC_PREC_FP64;
  const PassArgs base = base_args(target, kernel);
  std::vector<cudaEvent_t> ev(rounds + 1);
  for (auto& e : ev) CU(cudaEventCreate(&e));
  CU(cudaEventRecord(ev[0], st));
  for (int k = 0; k < rounds; ++k) {
    const int T = ts[k];
    const uint64_t n = ns[k], nblk = nblocks(n), rows = (uint64_t)S * (T + 1);
    const uint64_t nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
    Out& o = O[k];
    const size_t R1 = (size_t)S * (T + 1);
    TRY(o.g0.alloc(R1, st));
    TRY(o.g1.alloc(R1, st));
    TRY(o.g2.alloc(R1, st));
    TRY(o.ess.alloc(R1, st));
    TRY(o.cz.alloc(R1, st));
    TRY(o.lam.alloc(R1, st));
    TRY(o.scal.alloc(2 * (size_t)S, st));
    TRY(o.rs.alloc(R1, st));
    TRY(o.rt.alloc(R1, st));
    TRY(o.stt.alloc(S, st));
    TRY(o.rd.alloc(S, st));
    CU(cudaMemsetAsync(o.stt.p, 0, sizeof(SmcState) * S, st));
    std::vector<RoundDev> hv(S);
    for (int s = 0; s < S; ++s) {
      const size_t r0 = (size_t)s * (T + 1);
      hv[s] = RoundDev{o.g0.p + r0, o.g1.p + r0, o.g2.p + r0, o.ess.p + r0, o.cz.p + r0, o.rs.p + r0,
                       o.rt.p + r0, o.lam.p + r0, o.scal.p + 2 * (size_t)s, o.stt.p + s};
    }
    CU(cudaMemcpyAsync(o.rd.p, hv.data(), sizeof(RoundDev) * S, cudaMemcpyHostToDevice, st));
    DBuf<LogAcc> part, chunk, tot;  // stream-ordered frees after this round's kernels
    TRY(part.alloc(rows * kNAcc * nblk, st));
    TRY(chunk.alloc(rows * kNAcc * nchunks, st));
    TRY(tot.alloc(rows * kNAcc, st));
    CU(cudaMemsetAsync(part.p, 0, sizeof(LogAcc) * rows * kNAcc * nblk, st));  // row 0 of each seed: unused
    PassArgs A = base;
    A.betas = betas[k].p;
    A.T = T;
    A.t_begin = 1;
    A.t_end = T;
    A.mode = kModeSais;
    A.row_base = 0;
    A.n = n;
    A.p_begin = 0;
    A.n_local = n;
    A.seed = 0;
    A.round = (uint64_t)(k + 1);
    A.part = part.p;
    A.part_stride = nblk;
    A.err = gerr.p;
    A.seeds = d_seeds.p;
    A.blocks_per_seed = nblk;
    A.betas_stride = (uint64_t)T + 1;
    A.part_seed_stride = (uint64_t)(T + 1) * kNAcc * nblk;
    LCH(launch_pass(ex, L, A, (uint64_t)S * nblk, st));
    LCH(launch_fold(exact, part.p, nblk, nblk, 0, (int)rows, 4, chunk.p, tot.p, st));
    LCH(launch_sais_report_batch(tot.p, T, n, o.rd.p, S, st));
    if (k + 1 < rounds)
      LCH(launch_generate_schedule_batch(o.lam.p, (uint64_t)T + 1, betas[k].p, T + 1, ts[k + 1], betas[k + 1].p,
                                         sched_scratch.p, serr.p, S, st));
    CU(cudaEventRecord(ev[k + 1], st));
  }
  CU(cudaStreamSynchronize(st));
  int herr = 0;
  CU(cudaMemcpy(&herr, gerr.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr) return device_error(herr, 0, 0.0);
  std::vector<int> se(S);
  CU(cudaMemcpy(se.data(), serr.p, sizeof(int) * S, cudaMemcpyDeviceToHost));
  for (int s = 0; s < S; ++s)
    if (se[s]) return fail(se[s], "schedule generation for seed %llu failed validation", (unsigned long long)seeds[s]);
  for (int k = 0; k < rounds; ++k) {
    const int T = ts[k];
    std::vector<SmcState> sts(S);
    std::vector<double> scal(2 * (size_t)S), lam((size_t)S * (T + 1));
    CU(cudaMemcpy(sts.data(), O[k].stt.p, sizeof(SmcState) * S, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(scal.data(), O[k].scal.p, sizeof(double) * 2 * S, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(lam.data(), O[k].lam.p, sizeof(double) * S * (T + 1), cudaMemcpyDeviceToHost));
    for (int s = 0; s < S; ++s) TRY(device_error(sts[s].err, sts[s].err_step, sts[s].err_val));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
    if (out->n_particles) out->n_particles[k] = ns[k];
    if (out->steps) out->steps[k] = T;
    if (out->wall_seconds) out->wall_seconds[k] = ms * 1e-3;
    for (int s = 0; s < S; ++s) {
      const size_t i = (size_t)s * rounds + k;
      if (out->log_z_hat) out->log_z_hat[i] = scal[2 * s];
      if (out->elbo_hat) out->elbo_hat[i] = scal[2 * s + 1];
      if (out->lambda_total) out->lambda_total[i] = lam[(size_t)s * (T + 1) + T];
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return 0;
}

uint64_t asmc_fold_chunks(uint64_t p_begin, uint64_t p_end) {
  if (p_end <= p_begin) return 0;
  return (p_end - p_begin + ASMC_FOLD_CHUNK - 1) / ASMC_FOLD_CHUNK;
}

static int sais_partials_impl(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                              const double* betas, int32_t T, uint64_t n, uint64_t p_begin, uint64_t p_end,
                              uint64_t seed, uint64_t round, const asmc_exec* exec, asmc_logacc* partials,
                              bool device_out) {
  TRY(check_schedule(betas, T));
  TRY(check_pair(target, kernel));
  if (p_begin % ASMC_FOLD_CHUNK != 0)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "p_begin must be a multiple of ASMC_FOLD_CHUNK");
  if (p_end > n || p_end < p_begin) return fail(ASMC_ERR_INVALID_ARGUMENT, "bad particle range");
  const asmc_exec ex = exec ? *exec : default_exec();
  if (ex.precision == ASMC_PREC_FP64)
    return fail(ASMC_ERR_CAPABILITY, "sharded partials use the fp32 tree fold; fp64 reference order is single-GPU");
  if (target->kind == ASMC_TARGET_LOGISTIC || target->kind == ASMC_TARGET_ISING) {
    if (!device_out) return stepouter_partials(target, kernel, betas, T, p_begin, p_end, seed, round, ex, partials);
    // step-outer engines produce host partials; stage them into the caller's device buffer
    const uint64_t nch = asmc_fold_chunks(p_begin, p_end);
    std::vector<asmc_logacc> h(nch * (uint64_t)(T + 1) * 4);
    TRY(stepouter_partials(target, kernel, betas, T, p_begin, p_end, seed, round, ex, h.data()));
    DevCtx* C;
    TRY(get_ctx(ex.device, &C, ex.stream));
    CU(cudaMemcpyAsync(partials, h.data(), h.size() * sizeof(asmc_logacc), cudaMemcpyHostToDevice, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    return 0;
  }
  Layout L;
  TRY(choose_layout(ex, kernel->kind, target->dim, &L, 1, 4));  // long T runs in t-tiles
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const uint64_t nloc = p_end - p_begin, nblk = nblocks(nloc);
  const uint64_t nch = asmc_fold_chunks(p_begin, p_end);
  if (nch == 0) return 0;
  DBuf<double> d_betas;
  TRY(d_betas.alloc(T + 1, C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  DBuf<LogAcc> part, chunk;
  DBuf<int> err;
  TRY(part.alloc((size_t)(T + 1) * kNAcc * nblk, C->stream));
  TRY(chunk.alloc((size_t)(T + 1) * kNAcc * nch, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  PassArgs A = base_args(target, kernel);
  A.betas = d_betas.p;
  A.n = n;
  A.p_begin = p_begin;
  A.n_local = nloc;
  A.seed = seed;
  A.round = round;
  A.part = part.p;
  A.part_stride = nblk;
  A.err = err.p;
  DBuf<char> xs;
  DBuf<void*> xbuf;
  DBuf<int> xcur;
  DBuf<double> lwb;
  TRY(launch_sais_pass(C, ex, L, A, nblk, T, xs, xbuf, xcur, lwb));
  LCH(launch_fold_chunks(part.p, nblk, nblk, 1, T, 4, nch, chunk.p, C->stream));
  if (device_out) {  // partials stay on the device: the caller all-gathers them there
    LCH(launch_chunks_to_exchange(chunk.p, nch, T, reinterpret_cast<LogAcc*>(partials), C->stream));
    int herr = 0;
    CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    return device_error(herr, 0, 0.0);
  }
  std::vector<LogAcc> h((size_t)(T + 1) * kNAcc * nch);
  CU(cudaMemcpyAsync(h.data(), chunk.p, h.size() * sizeof(LogAcc), cudaMemcpyDeviceToHost, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  TRY(device_error(herr, 0, 0.0));
  for (uint64_t c = 0; c < nch; ++c)
    for (int t = 0; t <= T; ++t)
      for (int a = 0; a < 4; ++a) {
        const LogAcc v = t == 0 ? LogAcc{-HUGE_VAL, 0.0} : h[((size_t)t * kNAcc + a) * nch + c];
        partials[(c * (T + 1) + t) * 4 + a] = asmc_logacc{v.max, v.sum};
      }
  return 0;
}

int asmc_sais_partials(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                       const double* betas, int32_t T, uint64_t n, uint64_t p_begin, uint64_t p_end,
                       uint64_t seed, uint64_t round, const asmc_exec* exec, asmc_logacc* partials) {
  return sais_partials_impl(target, kernel, betas, T, n, p_begin, p_end, seed, round, exec, partials, false);
}

int asmc_sais_partials_dev(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                           const double* betas, int32_t T, uint64_t n, uint64_t p_begin, uint64_t p_end,
                           uint64_t seed, uint64_t round, const asmc_exec* exec, asmc_logacc* partials_dev) {
  if (!partials_dev) return fail(ASMC_ERR_INVALID_ARGUMENT, "null partials buffer");
  return sais_partials_impl(target, kernel, betas, T, n, p_begin, p_end, seed, round, exec, partials_dev, true);
}

// the device fold of all-gathered partials (device buffer, exchange layout): the same
// fold_chunks_final order as asmc_fold_partials, no host copy of the partials
int asmc_fold_partials_dev(const asmc_logacc* partials_dev, uint64_t chunks, int32_t T, uint64_t n,
                           const asmc_exec* exec, asmc_report* out) {
  if (T < 1 || chunks == 0 || !partials_dev) return fail(ASMC_ERR_INVALID_ARGUMENT, "nothing to fold");
  const asmc_exec ex = exec ? *exec : default_exec();
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  DBuf<LogAcc> chunk, tot;
  TRY(chunk.alloc((size_t)(T + 1) * kNAcc * chunks, C->stream));
  TRY(tot.alloc((size_t)(T + 1) * kNAcc, C->stream));
  LCH(launch_exchange_to_chunks(reinterpret_cast<const LogAcc*>(partials_dev), chunks, T, chunk.p, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  LCH(launch_fold_chunks_final(chunk.p, chunks, 1, T, 4, tot.p, C->stream));
  LCH(launch_sais_report(tot.p, T, n, R.rd.p, C->stream));
  SmcState st;
  TRY(copy_round(C, R, T, false, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  return 0;
}

int asmc_fold_partials(const asmc_logacc* partials, uint64_t chunks, int32_t T, uint64_t n,
                       asmc_report* out) {
  if (T < 1 || chunks == 0) return fail(ASMC_ERR_INVALID_ARGUMENT, "nothing to fold");
  int dev = 0;
  CU(cudaGetDevice(&dev));
  DevCtx* C;
  TRY(get_ctx(dev, &C));
  std::vector<LogAcc> h((size_t)(T + 1) * kNAcc * chunks, LogAcc{-HUGE_VAL, 0.0});
  for (uint64_t c = 0; c < chunks; ++c)
    for (int t = 1; t <= T; ++t)
      for (int a = 0; a < 4; ++a) {
        const asmc_logacc v = partials[(c * (T + 1) + t) * 4 + a];
        h[((size_t)t * kNAcc + a) * chunks + c] = LogAcc{v.max, v.sum};
      }
  DBuf<LogAcc> chunk, tot;
  TRY(chunk.alloc(h.size(), C->stream));
  TRY(tot.alloc((size_t)(T + 1) * kNAcc, C->stream));
  CU(cudaMemcpyAsync(chunk.p, h.data(), h.size() * sizeof(LogAcc), cudaMemcpyHostToDevice, C->stream));
  RoundBufs R;
  TRY(R.alloc(T, C->stream));
  LCH(launch_fold_chunks_final(chunk.p, chunks, 1, T, 4, tot.p, C->stream));
  LCH(launch_sais_report(tot.p, T, n, R.rd.p, C->stream));
  SmcState st;
  TRY(copy_round(C, R, T, false, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = n * (uint64_t)T;
  return 0;
}

int asmc_trajectories(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                      const double* betas, int32_t T, uint64_t seed, uint64_t round,
                      const uint64_t* particles, uint64_t count, const asmc_exec* exec,
                      double* x_out, double* log_w_out) {
  TRY(check_schedule(betas, T));
  TRY(check_pair(target, kernel));
  TRY(check_pass_target(target, "asmc_trajectories"));
  const asmc_exec ex = exec ? *exec : default_exec();
  Layout L;
  TRY(choose_layout(ex, kernel->kind, target->dim, &L, T, 4));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const uint64_t d = target->dim;
  DBuf<double> d_betas, rx, rl;
  DBuf<uint64_t> pids;
  DBuf<int> err;
  TRY(d_betas.alloc(T + 1, C->stream));
  TRY(rx.alloc(count * (T + 1) * d, C->stream));
  TRY(rl.alloc(count * (T + 1), C->stream));
  TRY(pids.alloc(count, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(pids.p, particles, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, C->stream));
  PassArgs A = base_args(target, kernel);
  A.betas = d_betas.p;
  A.T = T;
  A.t_begin = 1;
  A.t_end = T;
  A.mode = kModeTraj;
  A.n_local = count;
  A.seed = seed;
  A.round = round;
  A.pids = pids.p;
  A.rec_x = rx.p;
  A.rec_lw = rl.p;
  A.err = err.p;
  LCH(launch_pass(ex, L, A, nblocks(count), C->stream));
  CU(cudaMemcpyAsync(x_out, rx.p, sizeof(double) * count * (T + 1) * d, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(log_w_out, rl.p, sizeof(double) * count * (T + 1), cudaMemcpyDeviceToHost, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  return device_error(herr, 0, 0.0);
}

static int rng_common(int32_t rng, int what, int32_t prec, const uint64_t key[5], uint64_t count,
                      void* out) {
  if (rng != ASMC_RNG_XOSHIRO && rng != ASMC_RNG_PHILOX)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown rng %d", rng);
  DevCtx* C;
  TRY(get_ctx(0, &C));
  DBuf<uint64_t> buf;
  TRY(buf.alloc(count, C->stream));
  LCH(launch_rng(rng, what, prec, key, count, buf.p, C->stream));
  CU(cudaMemcpyAsync(out, buf.p, 8 * count, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  return 0;
}
int asmc_rng_u64(int32_t rng, const uint64_t key[5], uint64_t count, uint64_t* out) {
  return rng_common(rng, 0, ASMC_PREC_FP64, key, count, out);
}
int asmc_rng_uniform(int32_t rng, const uint64_t key[5], uint64_t count, double* out) {
  return rng_common(rng, 1, ASMC_PREC_FP64, key, count, out);
}
int asmc_rng_normal(int32_t rng, int32_t precision, const uint64_t key[5], uint64_t count,
                    double* out) {
  return rng_common(rng, 2, precision, key, count, out);
}

// engine.cpp:61-80 on the device (refcdf.cu): the reference's sequential CDF bit for bit
// (cum_out, optional: the n CDF values; l1_out, optional: logsumexp(log_w)).
static int resample_common(const double* log_w, uint64_t n, double u, int32_t device, uint32_t* ancestors,
                           double* cum_out, double* l1_out, int what) {
  if (n == 0) return fail(ASMC_ERR_INVALID_ARGUMENT, "cannot resample an empty system");
  if (n > 0xffffffffull) return fail(ASMC_ERR_CAPABILITY, "ancestor indices are 32-bit");
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> lw, cum, work;
  DBuf<uint32_t> anc;
  DBuf<SmcState> st;
  TRY(lw.alloc(n, C->stream));
  TRY(cum.alloc(n, C->stream));
  TRY(work.alloc(refcdf_work_doubles(n), C->stream));
  TRY(anc.alloc(n, C->stream));
  TRY(st.alloc(1, C->stream));
  SmcState h;
  std::memset(&h, 0, sizeof h);
  h.resample_now = 1;
  h.u = u;
  CU(cudaMemcpyAsync(st.p, &h, sizeof h, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(lw.p, log_w, sizeof(double) * n, cudaMemcpyHostToDevice, C->stream));
  RefCdfWork w;
  refcdf_work_carve(work.p, n, &w);
  DBuf<unsigned long long> prof;  // ASMC_REFCDF_PROF=1: per-phase %globaltimer stamps to stderr
  const bool profile = std::getenv("ASMC_REFCDF_PROF") != nullptr;
  if (profile) {
    TRY(prof.alloc(16, C->stream));
    CU(cudaMemsetAsync(prof.p, 0, 16 * sizeof(unsigned long long), C->stream));
    w.prof = prof.p;
  }
  LCH(launch_refcdf(lw.p, n, st.p, 0, &w, cum.p, anc.p, what, C->sms, C->stream));
  if (profile) {
    unsigned long long ts[16];
    CU(cudaMemcpyAsync(ts, prof.p, sizeof ts, cudaMemcpyDeviceToHost, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    std::fprintf(stderr, "refcdf n=%llu phases(us):", (unsigned long long)n);
    for (int i = 1; i < 13; ++i)
      if (ts[i] > ts[0]) std::fprintf(stderr, " %d:%.1f", i, (ts[i] - ts[0]) * 1e-3);
    std::fprintf(stderr, " replays lse=%llu (%.1f us) cdf=%llu (%.1f us)\n", ts[14], ts[13] * 1e-3,
                 ts[15] & 0xfffff, (ts[15] >> 20) * 1e-3);
  }
  if (ancestors && what == 1)
    CU(cudaMemcpyAsync(ancestors, anc.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, C->stream));
  if (cum_out && what >= 0)
    CU(cudaMemcpyAsync(cum_out, cum.p, sizeof(double) * n, cudaMemcpyDeviceToHost, C->stream));
  double l1 = 0.0;
  CU(cudaMemcpyAsync(&l1, w.l1, sizeof(double), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&h, st.p, sizeof h, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (l1_out) *l1_out = l1;
  if (h.err) return fail(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  return 0;
}

int asmc_systematic_resample(const double* log_w, uint64_t n, double u, int32_t device,
                             uint32_t* ancestors) {
  return resample_common(log_w, n, u, device, ancestors, nullptr, nullptr, 1);
}

int asmc_resample_cdf(const double* log_w, uint64_t n, int32_t device, double* cum_out, double* l1_out) {
  return resample_common(log_w, n, 0.0, device, nullptr, cum_out, l1_out, 0);
}

int asmc_logsumexp(const double* log_w, uint64_t n, int32_t device, double* out) {
  if (n == 0) {  // logsum.hpp:40-42 on an empty accumulator
    if (out) *out = -__builtin_huge_val();
    return 0;
  }
  const int rc = resample_common(log_w, n, 0.0, device, nullptr, nullptr, out, -1);
  if (rc == ASMC_ERR_DEGENERATE) {  // an all -inf input is a value here, not an error
    if (out) *out = -__builtin_huge_val();
    return 0;
  }
  return rc;
}

int asmc_exact_math(int32_t which, const double* x, uint64_t n, int32_t device, double* out) {
  if (which != 0 && which != 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "which must be 0 (exp) or 1 (log)");
  if (n == 0) return 0;
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> a, b;
  TRY(a.alloc(n, C->stream));
  TRY(b.alloc(n, C->stream));
  CU(cudaMemcpyAsync(a.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, C->stream));
  LCH(launch_exact_math(which, a.p, n, b.p, C->stream));
  CU(cudaMemcpyAsync(out, b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  return 0;
}

int asmc_ess(const double* log_w, uint64_t n, int32_t device, double* out) {
  if (n == 0) return fail(ASMC_ERR_INVALID_ARGUMENT, "ess of empty weight vector");
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> lw, r;
  DBuf<int> err;
  TRY(lw.alloc(n, C->stream));
  TRY(r.alloc(1, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(lw.p, log_w, sizeof(double) * n, cudaMemcpyHostToDevice, C->stream));
  LCH(launch_ess(lw.p, n, r.p, err.p, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(out, r.p, sizeof(double), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (herr) return fail(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  return 0;
}

// schedule.cpp:121-141 messages, checked on the host before the device inversion
static int check_barrier(const double* lambda, const double* beta, int n) {
  if (n < 2) return fail(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate needs at least two matched knots");
  if (lambda[0] != 0.0) return fail(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate must start at Lambda = 0");
  if (beta[0] != 0.0 || beta[n - 1] != 1.0)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "barrier estimate must span beta in [0, 1]");
  for (int i = 1; i < n; ++i) {
    if (lambda[i] < lambda[i - 1]) return fail(ASMC_ERR_INVALID_ARGUMENT, "barrier knots must be nondecreasing");
    if (!(beta[i] > beta[i - 1]))
      return fail(ASMC_ERR_INVALID_ARGUMENT, "barrier beta knots must be strictly increasing");
  }
  return 0;
}

int asmc_barrier_estimate(const double* g0, const double* g1, const double* g2,
                          const double* betas, int32_t T, int32_t device, double* lambda) {
  TRY(check_schedule(betas, T));
  for (int t = 1; t <= T; ++t)
    if (g0[t] == -HUGE_VAL)
      return fail(ASMC_ERR_INVALID_ARGUMENT, "no increment statistics recorded for step %d", t);
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> a, b, c, l;
  DBuf<int> err;
  TRY(a.alloc(T + 1, C->stream));
  TRY(b.alloc(T + 1, C->stream));
  TRY(c.alloc(T + 1, C->stream));
  TRY(l.alloc(T + 1, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(a.p, g0, 8 * (T + 1), cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(b.p, g1, 8 * (T + 1), cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(c.p, g2, 8 * (T + 1), cudaMemcpyHostToDevice, C->stream));
  LCH(launch_barrier(a.p, b.p, c.p, T, l.p, err.p, C->stream));
  CU(cudaMemcpyAsync(lambda, l.p, 8 * (T + 1), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  return 0;
}

int asmc_generate_schedule(const double* lambda, const double* beta, int32_t knots, int32_t t_new,
                           int32_t device, double* out) {
  TRY(check_barrier(lambda, beta, knots));
  if (t_new < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "schedule needs at least one step");
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> l, b, o, s;
  DBuf<int> err;
  TRY(l.alloc(knots, C->stream));
  TRY(b.alloc(knots, C->stream));
  TRY(o.alloc(t_new + 1, C->stream));
  TRY(s.alloc(5 * (size_t)knots, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(l.p, lambda, 8 * knots, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(b.p, beta, 8 * knots, cudaMemcpyHostToDevice, C->stream));
  LCH(launch_generate_schedule(l.p, b.p, knots, t_new, o.p, s.p, err.p, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(out, o.p, 8 * (t_new + 1), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (herr) return fail(herr, "generated schedule is not strictly increasing");
  return 0;
}

int asmc_local_barrier(const double* lambda, const double* beta, int32_t knots, int32_t device,
                       double* out) {
  TRY(check_barrier(lambda, beta, knots));
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<double> l, b, o, s;
  DBuf<int> err;
  TRY(l.alloc(knots, C->stream));
  TRY(b.alloc(knots, C->stream));
  TRY(o.alloc(knots, C->stream));
  TRY(s.alloc(3 * (size_t)knots, C->stream));
  TRY(err.alloc(1, C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(l.p, lambda, 8 * knots, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(b.p, beta, 8 * knots, cudaMemcpyHostToDevice, C->stream));
  LCH(launch_local_barrier(l.p, b.p, knots, o.p, s.p, err.p, C->stream));
  int herr = 0;
  CU(cudaMemcpyAsync(out, o.p, 8 * knots, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (herr) return fail(herr, "interpolant abscissae must be strictly increasing");
  return 0;
}

int asmc_profile_enable(int on) {
  g_prof = on != 0;
  return 0;
}

int asmc_profile_collect_drawn(double* ms, double* normals, double* drawn, int max_launches, int* n_launches) {
  int i = 0;
  for (auto& r : g_prof_recs) {
    CU(cudaEventSynchronize(r.b));
    if (i < max_launches) {
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, r.a, r.b));
      if (ms) ms[i] = t;
      if (normals) normals[i] = r.normals;
      if (drawn) {
        unsigned long long c = 0;
        if (r.drawn) CU(cudaMemcpy(&c, r.drawn, sizeof c, cudaMemcpyDeviceToHost));
        drawn[i] = r.drawn ? (double)c : r.normals;
      }
    }
    if (r.drawn) cudaFree(r.drawn);
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
    ++i;
  }
  if (n_launches) *n_launches = i;
  g_prof_recs.clear();
  return 0;
}

int asmc_profile_collect(double* ms, double* normals, int max_launches, int* n_launches) {
  return asmc_profile_collect_drawn(ms, normals, nullptr, max_launches, n_launches);
}

int asmc_peak_normals(int32_t device, int32_t blocks, uint64_t quads_per_thread, double* seconds) {
  DevCtx* C;
  TRY(get_ctx(device, &C));
  DBuf<float> sink;
  TRY(sink.alloc(1, C->stream));
  cudaEvent_t a, b;
  CU(cudaEventCreate(&a));
  CU(cudaEventCreate(&b));
  LCH(launch_peak_normals(blocks, quads_per_thread / 8 + 1, sink.p, C->stream));  // warm-up
  CU(cudaEventRecord(a, C->stream));
  LCH(launch_peak_normals(blocks, quads_per_thread, sink.p, C->stream));
  CU(cudaEventRecord(b, C->stream));
  CU(cudaEventSynchronize(b));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, a, b));
  *seconds = ms * 1e-3;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return 0;
}

}  // extern "C"

// ===================================================================== ZJA
extern "C" {

int asmc_zja_next_beta(const asmc_target_desc* target, double beta, const double* positions, uint64_t n,
                       const double* log_weights, double delta_star, double tol, const asmc_exec* exec,
                       double* beta_next, int32_t* warning) {
  // schedule.cpp:219-231
  if (!(beta >= 0.0 && beta < 1.0)) return fail(ASMC_ERR_DOMAIN, "zja_next_beta requires beta in [0, 1)");
  if (!(delta_star > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "delta_star must be positive");
  if (!(tol > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "tol must be positive");
  if (n == 0 || !positions || !log_weights)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "particle arrays inconsistent with n_particles");
  TRY(check_target(target));
  TRY(check_pass_target(target, "asmc_zja_next_beta"));
  if (!beta_next) return fail(ASMC_ERR_INVALID_ARGUMENT, "null output");
  const asmc_exec ex = exec ? *exec : default_exec();
  const bool exact = ex.precision == ASMC_PREC_FP64;
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const uint64_t d = target->dim;
  DBuf<char> x;
  DBuf<void*> xbuf;
  DBuf<int> xcur, warn, err;
  DBuf<double> lw, lr, V, betas;
  DBuf<LogAcc> part;
  const int grid = zja_grid_blocks(ex.device);
  TRY(x.alloc(n * d * sizeof(double), C->stream));
  TRY(xbuf.alloc(2, C->stream));
  TRY(xcur.alloc(1, C->stream));
  TRY(warn.alloc(1, C->stream));
  TRY(err.alloc(1, C->stream));
  TRY(lw.alloc(n, C->stream));
  TRY(lr.alloc(n, C->stream));
  TRY(V.alloc(n, C->stream));
  TRY(betas.alloc(2, C->stream));
  TRY(part.alloc((size_t)4 * grid, C->stream));
  std::vector<float> xf;
  if (exact) {
    CU(cudaMemcpyAsync(x.p, positions, n * d * sizeof(double), cudaMemcpyHostToDevice, C->stream));
  } else {
    xf.assign(positions, positions + n * d);
    CU(cudaMemcpyAsync(x.p, xf.data(), n * d * sizeof(float), cudaMemcpyHostToDevice, C->stream));
  }
  void* ptrs[2] = {x.p, x.p};
  CU(cudaMemcpyAsync(xbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(xcur.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(warn.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(err.p, 0, sizeof(int), C->stream));
  CU(cudaMemcpyAsync(lw.p, log_weights, n * sizeof(double), cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemcpyAsync(betas.p, &beta, sizeof(double), cudaMemcpyHostToDevice, C->stream));
  LCH(launch_zja_eval(make_params(target), exact, xbuf.p, xcur.p, n, lr.p, V.p, err.p, C->stream));
  ZjaArgs A{lw.p, lr.p, V.p, n, betas.p, 1, exact ? 1 : 0, delta_star, tol, warn.p, err.p, part.p};
  LCH(launch_zja_next_beta(A, grid, C->stream));
  double nb[2];
  int h[2];
  CU(cudaMemcpyAsync(nb, betas.p, sizeof nb, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&h[0], warn.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(&h[1], err.p, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (h[1]) return fail(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  *beta_next = nb[1];
  if (warning) *warning = h[0];
  return 0;
}

int asmc_run_zja(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const asmc_zja_opts* o,
                 const asmc_exec* exec, asmc_zja_out* out) {
  if (!o || !out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null options or output");
  // ZjaOptions::validate (drivers.cpp:23-31)
  if (o->n_particles < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (o->target_steps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "target_steps must be at least 1");
  if (o->max_steps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "max_steps must be at least 1");
  if (!(o->delta_star >= 0.0) || !std::isfinite(o->delta_star))
    return fail(ASMC_ERR_INVALID_ARGUMENT, "delta_star must be finite and >= 0");
  TRY(check_pair(target, kernel));
  TRY(check_pass_target(target, "asmc_run_zja"));
  const asmc_exec ex = exec ? *exec : default_exec();
  const bool exact = ex.precision == ASMC_PREC_FP64;
  const uint64_t n = o->n_particles, d = target->dim;
  if (out->capacity < 2) return fail(ASMC_ERR_INVALID_ARGUMENT, "output capacity must be at least 2");
  Layout L;
  TRY(choose_layout(ex, kernel->kind, d, &L));
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const PassArgs base = base_args(target, kernel);
  double delta = o->delta_star;
  uint64_t main_round = 1;
  out->pilot_ran = 0;
  out->warning = 0;
  if (delta <= 0.0) {  // drivers.cpp:244-265: uniform-K pilot, policy never, round 1
    const int K = o->target_steps;
    std::vector<double> pb(K + 1);
    for (int t = 0; t <= K; ++t) pb[t] = (double)t / (double)K;
    pb[0] = 0.0;
    pb[K] = 1.0;
    DBuf<double> d_pb;
    TRY(d_pb.alloc(K + 1, C->stream));
    CU(cudaMemcpyAsync(d_pb.p, pb.data(), sizeof(double) * (K + 1), cudaMemcpyHostToDevice, C->stream));
    RoundBufs R;
    TRY(R.alloc(K, C->stream));
    SmcWork W;  // run_smc(policy never): the report carries the ESS trace, as the reference's pilot
    TRY(enqueue_smc_round(C, ex, L, base, d_pb.p, K, n, ASMC_POLICY_NEVER, 0.5, o->seed, 1, R.rd.p, R.st.p, W));
    SmcState st;
    TRY(copy_round(C, R, K, true, &out->pilot, &st));
    TRY(device_error(st.err, st.err_step, st.err_val));
    out->pilot.kernel_applications = n * (uint64_t)K;
    std::vector<double> lam(K + 1);
    CU(cudaMemcpy(lam.data(), R.lam.p, sizeof(double) * (K + 1), cudaMemcpyDeviceToHost));
    if (out->pilot_lambda) std::memcpy(out->pilot_lambda, lam.data(), sizeof(double) * (K + 1));
    const double step_lam = lam[K] / (double)K;
    delta = std::max(1e-12, step_lam * step_lam);
    out->pilot_ran = 1;
    main_round = 2;
  }
  out->delta_star = delta;
  const double t0 = now_s();
  const int cap = o->max_steps;
  const size_t real = exact ? sizeof(double) : sizeof(float);
  const uint64_t nblk = nblocks(n), nchunks = (nblk + kChunkBlocks - 1) / kChunkBlocks;
  const int grid = zja_grid_blocks(ex.device);
  DBuf<char> x;
  DBuf<void*> xbuf;
  DBuf<int> xcur, warn;
  DBuf<double> lw, lr, V, betas;
  DBuf<LogAcc> part, chunk, tot, zpart;
  RoundBufs R;
  TRY(x.alloc(n * d * real, C->stream));
  TRY(xbuf.alloc(2, C->stream));
  TRY(xcur.alloc(1, C->stream));
  TRY(warn.alloc(1, C->stream));
  TRY(lw.alloc(n, C->stream));
  TRY(lr.alloc(n, C->stream));
  TRY(V.alloc(n, C->stream));
  TRY(betas.alloc(cap + 1, C->stream));
  TRY(part.alloc((size_t)kNAcc * nblk, C->stream));
  TRY(chunk.alloc((size_t)kNAcc * nchunks, C->stream));
  TRY(tot.alloc(kNAcc, C->stream));
  TRY(zpart.alloc((size_t)4 * grid, C->stream));
  TRY(R.alloc(cap, C->stream));
  void* ptrs[2] = {x.p, x.p};  // no resampling in ZJA: one live buffer
  CU(cudaMemcpyAsync(xbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(xcur.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(warn.p, 0, sizeof(int), C->stream));
  CU(cudaMemsetAsync(betas.p, 0, sizeof(double), C->stream));
  PassArgs A = base;
  A.betas = betas.p;
  A.T = cap;
  A.n = n;
  A.p_begin = 0;
  A.n_local = n;
  A.seed = o->seed;
  A.round = main_round;
  A.xbuf = xbuf.p;
  A.xcur = xcur.p;
  A.lw = lw.p;
  A.part = part.p;
  A.part_stride = nblk;
  A.err = &R.st.p->err;
  A.mode = kModeSmcInit;  // detail::init_particles at the main round
  LCH(launch_pass(ex, L, A, nblk, C->stream));
  const TgtParams tp = make_params(target);
  int t = 0;
  double bt = 0.0;
  while (bt < 1.0) {
    ++t;
    if (t > cap)
      return fail(ASMC_ERR_EVALUATION, "online adaptation failed to reach beta = 1 within %d steps", cap);
    LCH(launch_zja_eval(tp, exact, xbuf.p, xcur.p, n, lr.p, V.p, &R.st.p->err, C->stream));
    ZjaArgs Z{lw.p, lr.p, V.p, n, betas.p, t, exact ? 1 : 0, delta, 1e-10, warn.p, &R.st.p->err, zpart.p};
    LCH(launch_zja_next_beta(Z, grid, C->stream));
    A.mode = kModeSmcStep;
    A.t_begin = A.t_end = t;
    A.row_base = t;
    LCH(launch_pass(ex, L, A, nblk, C->stream));
    LCH(launch_fold(exact, part.p, nblk, nblk, 0, 1, kNAcc, chunk.p, tot.p, C->stream));
    LCH(launch_smc_decide(tot.p, t, -1, n, ASMC_POLICY_NEVER, 0.5, o->seed, main_round, ex.rng, R.rd.p, C->stream,
                          betas.p));
    SmcState st;
    CU(cudaMemcpyAsync(&bt, betas.p + t, sizeof(double), cudaMemcpyDeviceToHost, C->stream));
    CU(cudaMemcpyAsync(&st, R.st.p, sizeof st, cudaMemcpyDeviceToHost, C->stream));
    CU(cudaStreamSynchronize(C->stream));
    TRY(device_error(st.err, st.err_step, st.err_val));
  }
  if (t + 1 > out->capacity) return fail(ASMC_ERR_INVALID_ARGUMENT, "output capacity too small (%d needed)", t + 1);
  SmcState st;
  TRY(copy_round(C, R, t, true, &out->main, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->main.kernel_applications = n * (uint64_t)t;
  out->main.wall_seconds = now_s() - t0;
  out->steps = t;
  if (out->betas) CU(cudaMemcpy(out->betas, betas.p, sizeof(double) * (t + 1), cudaMemcpyDeviceToHost));
  if (out->lambda) CU(cudaMemcpy(out->lambda, R.lam.p, sizeof(double) * (t + 1), cudaMemcpyDeviceToHost));
  int hw = 0;
  CU(cudaMemcpy(&hw, warn.p, sizeof(int), cudaMemcpyDeviceToHost));
  out->warning = hw;
  return 0;
}

}  // extern "C"

// ==================================================================== NRPT
namespace {
// LogAccumulator (logsum.hpp:18-49), host copy for the stepping-stone estimator
struct HostLogAcc {
  double max = -HUGE_VAL, sum = 0.0;
  void add(double l) {
    if (l == -HUGE_VAL) return;
    if (l <= max) {
      sum += std::exp(l - max);
    } else {
      sum = sum * std::exp(max - l) + 1.0;
      max = l;
    }
  }
  double log_total() const { return max == -HUGE_VAL ? -HUGE_VAL : max + std::log(sum); }
};
}  // namespace

extern "C" int asmc_run_pt(const asmc_target_desc* target, const asmc_kernel_desc* kernel, const double* betas,
                           int32_t levels, const asmc_pt_opts* o, const asmc_exec* exec, asmc_pt_out* out) {
  if (!o || !out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null options or output");
  TRY(check_schedule(betas, levels));
  // PtOptions::validate (pt.cpp:14-19)
  if (o->iterations < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "iterations must be at least 1");
  if (o->burn_in >= o->iterations)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "burn_in must leave at least one recorded iteration");
  if (o->replicas < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "replicas must be at least 1");
  TRY(check_pair(target, kernel));
  TRY(check_pass_target(target, "asmc_run_pt"));
  if (levels > kPtMaxLevels) return fail(ASMC_ERR_CAPABILITY, "at most %d levels per run on the device", kPtMaxLevels);
  if (target->dim > 1024) return fail(ASMC_ERR_CAPABILITY, "asmc_run_pt supports dim <= 1024");
  const asmc_exec ex = exec ? *exec : default_exec();
  if (ex.rng != ASMC_RNG_XOSHIRO && ex.rng != ASMC_RNG_PHILOX) return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown rng");
  const bool fp64 = ex.precision == ASMC_PREC_FP64;
  DevCtx* C;
  TRY(get_ctx(ex.device, &C, ex.stream));
  const double t0 = now_s();
  const int L = levels, I = o->iterations, R = o->replicas;
  const int burn = o->burn_in < 0 ? I / 10 : o->burn_in;
  const size_t rows = (size_t)R * I * (L + 1);
  DBuf<double> d_betas, trace;
  DBuf<uint8_t> acc;
  DBuf<char> scratch;
  TRY(d_betas.alloc(L + 1, C->stream));
  TRY(trace.alloc(rows, C->stream));
  TRY(acc.alloc(rows, C->stream));
  TRY(scratch.alloc((size_t)R * (L + 1) * target->dim * (fp64 ? 8 : 4), C->stream));
  CU(cudaMemcpyAsync(d_betas.p, betas, sizeof(double) * (L + 1), cudaMemcpyHostToDevice, C->stream));
  CU(cudaMemsetAsync(acc.p, 0, rows, C->stream));
  PtArgs A;
  std::memset(&A, 0, sizeof A);
  A.tg = make_params(target);
  A.kc = make_kcfg(kernel);
  A.betas = d_betas.p;
  A.levels = L;
  A.iterations = I;
  A.seed0 = o->seed;
  A.round = o->round;
  A.replicas = R;
  A.scratch = scratch.p;
  A.trace = trace.p;
  A.accepted = acc.p;
  LCH(launch_pt(A, fp64, ex.rng, C->stream));
  std::vector<double> tr(rows);
  std::vector<uint8_t> ac(rows);
  CU(cudaMemcpyAsync(tr.data(), trace.p, rows * sizeof(double), cudaMemcpyDeviceToHost, C->stream));
  CU(cudaMemcpyAsync(ac.data(), acc.p, rows, cudaMemcpyDeviceToHost, C->stream));
  CU(cudaStreamSynchronize(C->stream));
  if (out->trace) std::memcpy(out->trace, tr.data(), rows * sizeof(double));
  if (out->swap_accepted) std::memcpy(out->swap_accepted, ac.data(), rows);
  const double log_used = std::log((double)(I - burn));
  for (int r = 0; r < R; ++r) {
    const double* t = tr.data() + (size_t)r * I * (L + 1);
    double log_z = 0.0;  // stepping_stone (pt.cpp:130-152)
    for (int n = 1; n <= L; ++n) {
      const double delta_beta = betas[n] - betas[n - 1];
      HostLogAcc a;
      for (int it = burn; it < I; ++it) a.add(delta_beta * t[(size_t)it * (L + 1) + n - 1]);
      log_z += a.log_total() - log_used;
    }
    if (out->log_z_hat) out->log_z_hat[r] = log_z;
    for (int lo = 0; lo <= L; ++lo) {  // run_pt's attempt / accept counters (pt.cpp:110-121)
      uint64_t att = 0, accn = 0;
      for (int it = 0; it < I; ++it)
        if (lo + 1 <= L && (lo & 1) == (it & 1)) {
          ++att;
          accn += ac[((size_t)r * I + it) * (L + 1) + lo];
        }
      if (out->swap_attempts) out->swap_attempts[(size_t)r * (L + 1) + lo] = att;
      if (out->swap_accepts) out->swap_accepts[(size_t)r * (L + 1) + lo] = accn;
    }
  }
  out->kernel_applications = (uint64_t)L * (uint64_t)I;
  out->wall_seconds = now_s() - t0;
  out->burn_in = burn;
  return 0;
}

// ============================================================ sharded SSMC
// One particle shard of a multi-GPU run_smc (include/asmc_b200.h).  The state,
// log-weights and block CDF stay on this GPU; what crosses GPUs is the chunk
// partials (ASMC_SHARD_NACC x 16 B per 262144 particles per step), the block CDF
// totals (8 B per 256 particles per resampling event) and the resampled rows.
struct asmc_smc_shard {
  DevCtx C;
  asmc_exec ex;
  Layout L;
  PassArgs A;
  int T = 0, policy = 0, t_done = 0, me = -1, resampling = 0;
  double rho = 0.5;
  uint64_t n = 0, p_begin = 0, n_local = 0, seed = 0, round = 0;
  uint64_t nblk = 0, nch = 0, row_bytes = 0, anc_cap = 0;
  DBuf<double> betas, lw, cum;
  DBuf<char> x;
  DBuf<void*> xbuf;
  DBuf<int> xcur;
  DBuf<uint32_t> anc;
  DBuf<LogAcc> part, chunk, tot;
  DBuf<uint64_t> rank_blk, slot_dev;
  DBuf<double> cum_all, work;  // resampling: global CDF + refcdf scratch (allocated on first event)
  RoundBufs R;
  std::vector<uint64_t> slots;
  // multi-GPU ZJA mode: open-ended schedule (betas[t] set per step), potential cache, probes
  int zja = 0, zt = 0;
  DBuf<double> lr, V;
  DBuf<LogAcc> zpart, zchunk;
  DBuf<ZjaSearch> zs;  // device-resident search state (asmc_zja_shard_search_*)
};

extern "C" {

int asmc_smc_shard_create(const asmc_target_desc* target, const asmc_kernel_desc* kernel,
                          const double* betas, int32_t T, uint64_t n, uint64_t p_begin, uint64_t p_end,
                          int32_t policy, double rho, uint64_t seed, uint64_t round,
                          const asmc_exec* exec, asmc_smc_shard** out) {
  if (!out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null shard handle");
  *out = nullptr;
  TRY(check_schedule(betas, T));
  if (n < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "n_particles must be at least 1");
  if (!(rho >= 0.0 && rho <= 1.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "rho must lie in [0, 1]");
  if (policy < ASMC_POLICY_NEVER || policy > ASMC_POLICY_STABILIZED)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "unknown resampling policy");
  TRY(check_pair(target, kernel));
  if (n > 0xffffffffull) return fail(ASMC_ERR_CAPABILITY, "ancestor indices are 32-bit");
  if (p_begin % ASMC_FOLD_CHUNK != 0)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "p_begin must be a multiple of ASMC_FOLD_CHUNK");
  if (p_end > n || p_end <= p_begin) return fail(ASMC_ERR_INVALID_ARGUMENT, "bad particle range");
  if (p_end != n && p_end % ASMC_FOLD_CHUNK != 0)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "p_end must be n_particles or a multiple of ASMC_FOLD_CHUNK");
  const asmc_exec ex = exec ? *exec : default_exec();
  if (ex.precision == ASMC_PREC_FP64 || ex.rng != ASMC_RNG_PHILOX)
    return fail(ASMC_ERR_CAPABILITY,
                "sharded SSMC uses the fp32 tree fold (rng = philox, precision = fp32); the fp64 reference order is single-GPU");
  TRY(check_pass_target(target, "sharded SSMC"));
  auto* h = new asmc_smc_shard;
  auto drop = [&](int rc) { delete h; return rc; };
  int rc = choose_layout(ex, kernel->kind, target->dim, &h->L);
  if (rc) return drop(rc);
  DevCtx* C;
  if ((rc = get_ctx(ex.device, &C, ex.stream))) return drop(rc);
  h->C = *C;
  h->C.pinned = nullptr;  // the shard's own staging (the context's stays the context's)
  h->C.pinned_cap = 0;
  h->ex = ex;
  h->T = T;
  h->policy = policy;
  h->rho = rho;
  h->n = n;
  h->p_begin = p_begin;
  h->n_local = p_end - p_begin;
  h->seed = seed;
  h->round = round;
  h->nblk = nblocks(h->n_local);
  h->nch = asmc_fold_chunks(p_begin, p_end);
  h->row_bytes = target->dim * sizeof(float);
  cudaStream_t s = h->C.stream;
  const uint64_t nl = h->n_local;
  rc = [&]() -> int {
    TRY(h->betas.alloc(T + 1, s));
    CU(cudaMemcpyAsync(h->betas.p, betas, sizeof(double) * (T + 1), cudaMemcpyHostToDevice, s));
    TRY(h->x.alloc(nl * h->row_bytes, s));
    TRY(h->xbuf.alloc(2, s));
    TRY(h->xcur.alloc(1, s));
    TRY(h->lw.alloc(nl, s));
    TRY(h->part.alloc((size_t)kNAcc * h->nblk, s));
    TRY(h->chunk.alloc((size_t)kNAcc * h->nch, s));
    TRY(h->tot.alloc(kNAcc, s));
    TRY(h->R.alloc(T, s));
    void* ptrs[2] = {h->x.p, h->x.p};  // in-place state: resampled rows arrive via accept
    CU(cudaMemcpyAsync(h->xbuf.p, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, s));
    CU(cudaMemsetAsync(h->xcur.p, 0, sizeof(int), s));
    PassArgs& A = h->A;
    A = base_args(target, kernel);
    A.betas = h->betas.p;
    A.T = T;
    A.n = n;
    A.p_begin = p_begin;
    A.n_local = nl;
    A.seed = seed;
    A.round = round;
    A.xbuf = h->xbuf.p;
    A.xcur = h->xcur.p;
    A.lw = h->lw.p;
    A.part = h->part.p;
    A.part_stride = h->nblk;
    A.err = &h->R.st.p->err;
    A.mode = kModeSmcInit;  // engine_detail.hpp:91-100, global particle ids
    LCH(launch_pass(h->ex, h->L, A, h->nblk, s));
    return 0;
  }();
  if (rc) return drop(rc);
  *out = h;
  return 0;
}

void asmc_smc_shard_destroy(asmc_smc_shard* h) {
  if (!h) return;
  cudaStreamSynchronize(h->C.stream);
  if (h->C.pinned) cudaFreeHost(h->C.pinned);
  delete h;
}

uint64_t asmc_smc_shard_chunks(const asmc_smc_shard* h) { return h ? h->nch : 0; }
uint64_t asmc_smc_shard_exchange_len(const asmc_smc_shard* h) { return h ? h->n_local : 0; }
uint64_t asmc_smc_shard_row_bytes(const asmc_smc_shard* h) { return h ? h->row_bytes : 0; }

int asmc_smc_shard_step(asmc_smc_shard* h, int32_t t, asmc_logacc* partials_dev) {
  if (!h || !partials_dev) return fail(ASMC_ERR_INVALID_ARGUMENT, "null shard or partials");
  if (t != h->t_done + 1 || t > h->T || h->resampling)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "shard step %d out of order (last completed %d)", t, h->t_done);
  cudaStream_t s = h->C.stream;
  PassArgs A = h->A;
  A.mode = kModeSmcStep;
  A.t_begin = A.t_end = t;
  A.row_base = t;
  LCH(launch_pass(h->ex, h->L, A, h->nblk, s));
  LCH(launch_fold_chunks(h->part.p, h->nblk, h->nblk, 0, 1, kNAcc, h->nch, h->chunk.p, s));
  LCH(launch_chunk_major(h->chunk.p, h->nch, reinterpret_cast<LogAcc*>(partials_dev), s));
  return 0;
}

int asmc_smc_shard_decide(asmc_smc_shard* h, int32_t t, const asmc_logacc* all_dev, uint64_t all_chunks,
                          double* lw_out_dev, int32_t* resample) {
  if (!h || !all_dev || !lw_out_dev || !resample) return fail(ASMC_ERR_INVALID_ARGUMENT, "null argument");
  if (t != h->t_done + 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "decide for step %d out of order", t);
  if (all_chunks != asmc_fold_chunks(0, h->n))
    return fail(ASMC_ERR_INVALID_ARGUMENT, "expected %llu chunk partials, got %llu",
                (unsigned long long)asmc_fold_chunks(0, h->n), (unsigned long long)all_chunks);
  cudaStream_t s = h->C.stream;
  LCH(launch_fold_chunk_major(reinterpret_cast<const LogAcc*>(all_dev), all_chunks, h->tot.p, s));
  LCH(launch_smc_decide(h->tot.p, t, h->zja ? -1 : h->T, h->n, h->policy, h->rho, h->seed, h->round, h->ex.rng,
                        h->R.rd.p, s, h->zja ? h->betas.p : nullptr));
  SmcState st;
  CU(cudaMemcpyAsync(&st, h->R.st.p, sizeof st, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  TRY(device_error(st.err, st.err_step, st.err_val));
  if (st.resample_now)  // this shard's log-weights, for the caller's all-gather
    CU(cudaMemcpyAsync(lw_out_dev, h->lw.p, h->n_local * sizeof(double), cudaMemcpyDeviceToDevice, s));
  h->t_done = t;
  h->resampling = st.resample_now;
  *resample = st.resample_now;
  return 0;
}

int asmc_smc_shard_plan(asmc_smc_shard* h, const double* all_lw_dev, uint64_t all_len, int32_t world,
                        const uint64_t* shard_p_begin, uint64_t* slot_begin) {
  if (!h || !all_lw_dev || !shard_p_begin || !slot_begin)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "null argument");
  if (!h->resampling) return fail(ASMC_ERR_INVALID_ARGUMENT, "plan without a resampling decision");
  if (world < 1 || world > 1023) return fail(ASMC_ERR_INVALID_ARGUMENT, "world size must be in [1, 1023]");
  if (all_len != h->n)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "expected %llu log-weights, got %llu", (unsigned long long)h->n,
                (unsigned long long)all_len);
  if (shard_p_begin[0] != 0 || shard_p_begin[world] != h->n)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "shard boundaries must span [0, n_particles)");
  h->me = -1;
  for (int r = 0; r < world; ++r) {
    if (shard_p_begin[r] > shard_p_begin[r + 1] || shard_p_begin[r] % ASMC_FOLD_CHUNK)
      return fail(ASMC_ERR_INVALID_ARGUMENT, "shard boundaries must be ordered multiples of ASMC_FOLD_CHUNK");
    if (shard_p_begin[r] == h->p_begin && shard_p_begin[r + 1] == h->p_begin + h->n_local) h->me = r;
  }
  if (h->me < 0) return fail(ASMC_ERR_INVALID_ARGUMENT, "this shard's range is not among the shard boundaries");
  cudaStream_t s = h->C.stream;
  if (!h->rank_blk.p || (int)h->slots.size() != world + 1) {
    h->rank_blk.~DBuf();
    new (&h->rank_blk) DBuf<uint64_t>();
    h->slot_dev.~DBuf();
    new (&h->slot_dev) DBuf<uint64_t>();
    TRY(h->rank_blk.alloc(world + 1, s));
    TRY(h->slot_dev.alloc(world + 1, s));
    h->slots.assign(world + 1, 0);
  }
  if (!h->cum_all.p) {  // the global CDF and ancestors, identical on every rank
    TRY(h->cum_all.alloc(h->n, s));
    TRY(h->work.alloc(refcdf_work_doubles(h->n), s));
    TRY(h->anc.alloc(h->n, s));
    h->anc_cap = h->n;
  }
  CU(cudaMemcpyAsync(h->rank_blk.p, shard_p_begin, sizeof(uint64_t) * (world + 1), cudaMemcpyHostToDevice, s));
  RefCdfWork w;
  refcdf_work_carve(h->work.p, h->n, &w);
  LCH(launch_refcdf(all_lw_dev, h->n, h->R.st.p, 1, &w, h->cum_all.p, h->anc.p, 1, h->C.sms, s));
  LCH(launch_slot_bounds(h->anc.p, h->n, h->rank_blk.p, world, h->R.st.p, h->slot_dev.p, s));
  CU(cudaMemcpyAsync(h->slots.data(), h->slot_dev.p, sizeof(uint64_t) * (world + 1), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  std::memcpy(slot_begin, h->slots.data(), sizeof(uint64_t) * (world + 1));
  return 0;
}

int asmc_smc_shard_pack(asmc_smc_shard* h, void* rows_dev) {
  if (!h || h->me < 0 || !h->resampling) return fail(ASMC_ERR_INVALID_ARGUMENT, "pack before plan");
  const uint64_t lo = h->slots[h->me], count = h->slots[h->me + 1] - lo;
  if (count && !rows_dev) return fail(ASMC_ERR_INVALID_ARGUMENT, "null row buffer");
  LCH(launch_pack_rows(h->anc.p + lo, count, h->p_begin, h->row_bytes, h->x.p, rows_dev, h->C.sms, h->C.stream));
  return 0;
}

int asmc_smc_shard_accept(asmc_smc_shard* h, const void* rows_dev) {
  if (!h || !rows_dev || !h->resampling) return fail(ASMC_ERR_INVALID_ARGUMENT, "accept without a resampling step");
  cudaStream_t s = h->C.stream;
  CU(cudaMemcpyAsync(h->x.p, rows_dev, h->n_local * h->row_bytes, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemsetAsync(h->lw.p, 0, h->n_local * sizeof(double), s));  // engine.cpp:170-172
  CU(cudaMemsetAsync(&h->R.st.p->resample_now, 0, sizeof(int), s));
  h->resampling = 0;
  h->me = -1;
  return 0;
}

int asmc_smc_shard_report(asmc_smc_shard* h, asmc_report* out) {
  if (!h || !out) return fail(ASMC_ERR_INVALID_ARGUMENT, "null argument");
  const int T = h->zja ? h->t_done : h->T;
  if (T < 1 || h->t_done != T || h->resampling)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "report before step %d completed", h->T);
  SmcState st;
  TRY(copy_round(&h->C, h->R, T, true, out, &st));
  TRY(device_error(st.err, st.err_step, st.err_val));
  out->kernel_applications = h->n * (uint64_t)T;
  return 0;
}

int asmc_smc_shard_state(asmc_smc_shard* h, void* rows_host, double* lw_host) {
  if (!h) return fail(ASMC_ERR_INVALID_ARGUMENT, "null shard");
  cudaStream_t s = h->C.stream;
  if (rows_host)
    CU(cudaMemcpyAsync(rows_host, h->x.p, h->n_local * h->row_bytes, cudaMemcpyDeviceToHost, s));
  if (lw_host) CU(cudaMemcpyAsync(lw_host, h->lw.p, h->n_local * sizeof(double), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return 0;
}

}  // extern "C"

// ====================================================== multi-GPU ZJA shards
extern "C" {

int asmc_zja_shard_create(const asmc_target_desc* target, const asmc_kernel_desc* kernel, uint64_t n,
                          uint64_t p_begin, uint64_t p_end, uint64_t seed, uint64_t round, int32_t max_steps,
                          const asmc_exec* exec, asmc_smc_shard** out) {
  if (max_steps < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "max_steps must be at least 1");
  TRY(check_pass_target(target, "asmc_zja_shard_create"));
  std::vector<double> b(max_steps + 1);  // placeholder schedule; betas[t] are chosen per step
  for (int t = 0; t <= max_steps; ++t) b[t] = (double)t / (double)max_steps;
  b[0] = 0.0;
  b[max_steps] = 1.0;
  TRY(asmc_smc_shard_create(target, kernel, b.data(), max_steps, n, p_begin, p_end, ASMC_POLICY_NEVER, 0.5, seed,
                            round, exec, out));
  asmc_smc_shard* h = *out;
  h->zja = 1;
  cudaStream_t s = h->C.stream;
  const int rc = [&]() -> int {
    TRY(h->lr.alloc(h->n_local, s));
    TRY(h->V.alloc(h->n_local, s));
    TRY(h->zpart.alloc(2 * h->nblk, s));
    TRY(h->zchunk.alloc((size_t)kNAcc * h->nch, s));
    TRY(h->zs.alloc(1, s));
    return 0;
  }();
  if (rc) {
    asmc_smc_shard_destroy(h);
    *out = nullptr;
  }
  return rc;
}

// log eta / V at the shard's current particles (once per ZJA step, before the probes)
int asmc_zja_shard_eval(asmc_smc_shard* h) {
  if (!h || !h->zja) return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard");
  LCH(launch_zja_eval(h->A.tg, false, h->xbuf.p, h->xcur.p, h->n_local, h->lr.p, h->V.p, &h->R.st.p->err,
                      h->C.stream));
  return 0;
}

// chunk partials of one probe: out[c * 2 + 0] = m1, [c * 2 + 1] = m2 of dhat(b2) over this
// shard's chunks (b2 < 0: out[c * 2] = lse of the log-weights); host buffer, synchronous
int asmc_zja_shard_probe(asmc_smc_shard* h, double beta, double b2, asmc_logacc* out) {
  if (!h || !h->zja || !out) return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard or null output");
  cudaStream_t s = h->C.stream;
  LCH(launch_zja_probe_blocks(h->lw.p, h->V.p, h->n_local, beta, b2, h->zpart.p, h->nblk, s));
  LCH(launch_fold_chunks(h->zpart.p, h->nblk, h->nblk, 0, 1, 2, h->nch, h->zchunk.p, s));
  std::vector<LogAcc> c(2 * h->nch);
  CU(cudaMemcpyAsync(c.data(), h->zchunk.p, c.size() * sizeof(LogAcc), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  for (uint64_t i = 0; i < h->nch; ++i) {
    out[2 * i] = asmc_logacc{c[i].max, c[i].sum};
    out[2 * i + 1] = asmc_logacc{c[h->nch + i].max, c[h->nch + i].sum};
  }
  return 0;
}

// Device-resident search (no host round trip per probe): begin(t) arms the state machine
// at beta_{t-1}; each probe_dev writes this shard's (chunks, 2) partials at the search's
// current point to device memory; the caller all-gathers them (chunk order over ranks)
// and search_step folds them and advances the search -- identically on every rank --,
// writing betas[t] once it is done.  poll() is the only synchronising call.
int asmc_zja_shard_search_begin(asmc_smc_shard* h, int32_t t, double delta_star) {
  if (!h || !h->zja) return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard");
  if (!(delta_star > 0.0)) return fail(ASMC_ERR_INVALID_ARGUMENT, "delta_star must be positive");
  if (t < 1 || t > h->T) return fail(ASMC_ERR_EVALUATION, "online adaptation failed to reach beta = 1 within %d steps", h->T);
  h->zt = t;
  LCH(launch_zja_search_init(h->zs.p, h->betas.p, t, delta_star, 1e-10, h->C.stream));
  return 0;
}

int asmc_zja_shard_probe_dev(asmc_smc_shard* h, asmc_logacc* partials_dev) {
  if (!h || !h->zja || !partials_dev || h->zt < 1)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard with an open search, or null output");
  cudaStream_t s = h->C.stream;
  LCH(launch_zja_probe_dev(h->lw.p, h->V.p, h->n_local, h->zs.p, h->zpart.p, h->nblk, s));
  LCH(launch_fold_chunks(h->zpart.p, h->nblk, h->nblk, 0, 1, 2, h->nch, h->zchunk.p, s));
  LCH(launch_zja_interleave(h->zchunk.p, h->nch, h->zs.p, reinterpret_cast<LogAcc*>(partials_dev), s));
  return 0;
}

int asmc_zja_shard_search_step(asmc_smc_shard* h, const asmc_logacc* all_partials_dev, uint64_t all_chunks) {
  if (!h || !h->zja || !all_partials_dev || h->zt < 1)
    return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard with an open search, or null partials");
  LCH(launch_zja_search_step(h->zs.p, reinterpret_cast<const LogAcc*>(all_partials_dev), all_chunks, h->betas.p,
                             h->zt, nullptr, &h->R.st.p->err, h->C.stream));
  return 0;
}

int asmc_zja_shard_search_poll(asmc_smc_shard* h, int32_t* done, double* beta, int32_t* warn, int32_t* probes) {
  if (!h || !h->zja || h->zt < 1) return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard with an open search");
  ZjaSearch z;
  int err = 0;
  cudaStream_t s = h->C.stream;
  CU(cudaMemcpyAsync(&z, h->zs.p, sizeof z, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&err, &h->R.st.p->err, sizeof err, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (err == ASMC_ERR_DEGENERATE) return fail(ASMC_ERR_DEGENERATE, "all log-weights are -inf");
  TRY(device_error(err, h->zt, 0.0));
  if (done) *done = z.phase == kZjaSearchDone;
  if (beta) *beta = z.chosen;
  if (warn) *warn = z.warn;
  if (probes) *probes = z.probes;
  return 0;
}

int asmc_zja_shard_set_beta(asmc_smc_shard* h, int32_t t, double beta) {
  if (!h || !h->zja) return fail(ASMC_ERR_INVALID_ARGUMENT, "not a ZJA shard");
  if (t < 1 || t > h->T) return fail(ASMC_ERR_EVALUATION, "online adaptation failed to reach beta = 1 within %d steps", h->T);
  CU(cudaMemcpyAsync(h->betas.p + t, &beta, sizeof(double), cudaMemcpyHostToDevice, h->C.stream));
  CU(cudaStreamSynchronize(h->C.stream));  // &beta is a host stack value
  return 0;
}

}  // extern "C"
