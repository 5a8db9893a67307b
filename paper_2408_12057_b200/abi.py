"""ctypes layouts of include/asmc_b200.h (types and constants only; loads nothing).

Shared by the product binding (capi.py) and by the test-only oracle loader
(oracle/__init__.py), so both sides are fed byte-identical descriptors.
"""
import ctypes as C

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_DOMAIN = 2
ERR_CAPABILITY = 3
ERR_DEGENERATE = 4
ERR_EVALUATION = 5
ERR_CUDA = 6
ERR_INTERNAL = 7

TARGET_GAUSSIAN_SHIFT = 0
TARGET_MIXTURE = 1
TARGET_SCALE_GAUSSIAN = 2
TARGET_LOGISTIC = 3
TARGET_ISING = 4

KERNEL_IDEALIZED = 0
KERNEL_RWMH = 1
KERNEL_IDENTITY = 2
KERNEL_HMC = 3
KERNEL_SLICE = 4  # elliptical slice w.r.t. the Gaussian reference
SLICE_MAX_SHRINK = 100
MAX_STEP_SIZES = 16

POLICY_NEVER = 0
POLICY_ALWAYS = 1
POLICY_ADAPTIVE_ESS = 2
POLICY_STABILIZED = 3

MODE_SSMC = 0
MODE_SAIS = 1

RNG_XOSHIRO = 0
RNG_PHILOX = 1
PREC_FP64 = 0
PREC_FP32 = 1

FOLD_CHUNK = 262144
BLOCK = 256  # kReductionBlock, include/asmc/logsum.hpp:15
SHARD_NACC = 6  # ASMC_SHARD_NACC: g0 g1 g2 elbo sq top2 per chunk partial


class TargetDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("dim", C.c_uint64),
                ("p", C.c_double * 8), ("data", C.c_void_p), ("data_bytes", C.c_uint64)]


class KernelDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_step_sizes", C.c_int32), ("sweeps", C.c_int32),
                ("leapfrog", C.c_int32), ("step_sizes", C.c_double * MAX_STEP_SIZES)]


class Exec(C.Structure):
    _fields_ = [("rng", C.c_int32), ("precision", C.c_int32), ("device", C.c_int32),
                ("lanes", C.c_int32), ("stream", C.c_uint64)]


class LogAcc(C.Structure):
    _fields_ = [("max", C.c_double), ("sum", C.c_double)]


class Report(C.Structure):
    _fields_ = [("log_g0", C.POINTER(C.c_double)), ("log_g1", C.POINTER(C.c_double)),
                ("log_g2", C.POINTER(C.c_double)), ("ess_trace", C.POINTER(C.c_double)),
                ("cum_log_z", C.POINTER(C.c_double)), ("resampled", C.POINTER(C.c_uint8)),
                ("resample_times", C.POINTER(C.c_int32)), ("n_resample_times", C.c_int32),
                ("reserved", C.c_int32), ("log_z_hat", C.c_double), ("elbo_hat", C.c_double),
                ("wall_seconds", C.c_double), ("kernel_applications", C.c_uint64)]


class RoundsOut(C.Structure):
    _fields_ = [("max_steps", C.c_int32), ("reserved", C.c_int32),
                ("n_particles", C.POINTER(C.c_uint64)), ("steps", C.POINTER(C.c_int32)),
                ("betas", C.POINTER(C.c_double)), ("log_g0", C.POINTER(C.c_double)),
                ("log_g1", C.POINTER(C.c_double)), ("log_g2", C.POINTER(C.c_double)),
                ("ess_trace", C.POINTER(C.c_double)), ("cum_log_z", C.POINTER(C.c_double)),
                ("resampled", C.POINTER(C.c_uint8)), ("lambda_", C.POINTER(C.c_double)),
                ("log_z_hat", C.POINTER(C.c_double)), ("elbo_hat", C.POINTER(C.c_double)),
                ("wall_seconds", C.POINTER(C.c_double)),
                ("kernel_applications", C.POINTER(C.c_uint64))]


class SeedsOut(C.Structure):  # asmc_seeds_out
    _fields_ = [("n_particles", C.POINTER(C.c_uint64)), ("steps", C.POINTER(C.c_int32)),
                ("wall_seconds", C.POINTER(C.c_double)), ("log_z_hat", C.POINTER(C.c_double)),
                ("elbo_hat", C.POINTER(C.c_double)), ("lambda_total", C.POINTER(C.c_double))]


class ZjaOpts(C.Structure):
    _fields_ = [("n_particles", C.c_uint64), ("target_steps", C.c_int32), ("max_steps", C.c_int32),
                ("delta_star", C.c_double), ("seed", C.c_uint64)]


class ZjaOut(C.Structure):
    _fields_ = [("capacity", C.c_int32), ("steps", C.c_int32), ("pilot_ran", C.c_int32),
                ("warning", C.c_int32), ("delta_star", C.c_double), ("betas", C.POINTER(C.c_double)),
                ("lambda_", C.POINTER(C.c_double)), ("main", Report),
                ("pilot_lambda", C.POINTER(C.c_double)), ("pilot", Report)]


class PtOpts(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("burn_in", C.c_int32), ("seed", C.c_uint64), ("round", C.c_uint64),
                ("replicas", C.c_int32), ("reserved", C.c_int32)]


class PtOut(C.Structure):
    _fields_ = [("log_z_hat", C.POINTER(C.c_double)), ("trace", C.POINTER(C.c_double)),
                ("swap_accepted", C.POINTER(C.c_uint8)), ("swap_attempts", C.POINTER(C.c_uint64)),
                ("swap_accepts", C.POINTER(C.c_uint64)), ("kernel_applications", C.c_uint64),
                ("wall_seconds", C.c_double), ("burn_in", C.c_int32), ("reserved", C.c_int32)]


def pt_buffers(levels, iterations, burn_in=-1, seed=0, round=1, replicas=1):
    """(PtOpts, PtOut, numpy buffers) for asmc_run_pt / ora_run_pt."""
    import numpy as np
    o = PtOpts()
    o.iterations, o.burn_in, o.seed, o.round, o.replicas = iterations, burn_in, seed, round, replicas
    L1 = levels + 1
    b = dict(log_z_hat=np.zeros(replicas), trace=np.zeros((replicas, iterations, L1)),
             swap_accepted=np.zeros((replicas, iterations, L1), np.uint8),
             swap_attempts=np.zeros((replicas, L1), np.uint64), swap_accepts=np.zeros((replicas, L1), np.uint64))
    out = PtOut()
    out.log_z_hat = b["log_z_hat"].ctypes.data_as(C.POINTER(C.c_double))
    out.trace = b["trace"].ctypes.data_as(C.POINTER(C.c_double))
    out.swap_accepted = b["swap_accepted"].ctypes.data_as(C.POINTER(C.c_uint8))
    out.swap_attempts = b["swap_attempts"].ctypes.data_as(C.POINTER(C.c_uint64))
    out.swap_accepts = b["swap_accepts"].ctypes.data_as(C.POINTER(C.c_uint64))
    return o, out, b


def pt_finish(out, b):
    d = dict(b)
    d.update(kernel_applications=out.kernel_applications, wall_seconds=out.wall_seconds, burn_in=out.burn_in)
    return d


def zja_opts(n, target_steps=32, delta_star=0.0, seed=0, max_steps=100000):
    o = ZjaOpts()
    o.n_particles, o.target_steps, o.max_steps, o.delta_star, o.seed = n, target_steps, max_steps, delta_star, seed
    return o


def _report_bufs(T):
    import numpy as np
    bufs = dict(log_g0=np.full(T + 1, -np.inf), log_g1=np.full(T + 1, -np.inf),
                log_g2=np.full(T + 1, -np.inf), ess_trace=np.zeros(T + 1), cum_log_z=np.zeros(T + 1),
                resampled=np.zeros(T + 1, np.uint8), resample_times=np.zeros(T + 1, np.int32))
    rep = Report()
    for k in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
        setattr(rep, k, bufs[k].ctypes.data_as(C.POINTER(C.c_double)))
    rep.resampled = bufs["resampled"].ctypes.data_as(C.POINTER(C.c_uint8))
    rep.resample_times = bufs["resample_times"].ctypes.data_as(C.POINTER(C.c_int32))
    return rep, bufs


def zja_buffers(opts):
    """ZjaOut with numpy-backed arrays (main: max_steps + 1 entries, pilot: K + 1)."""
    import numpy as np
    out = ZjaOut()
    cap = opts.max_steps + 1
    out.capacity = cap
    keep = {}
    out.main, keep["main"] = _report_bufs(cap - 1)
    out.pilot, keep["pilot"] = _report_bufs(opts.target_steps)
    keep["betas"], keep["lambda_"], keep["pilot_lambda"] = np.zeros(cap), np.zeros(cap), np.zeros(opts.target_steps + 1)
    for k in ("betas", "lambda_", "pilot_lambda"):
        setattr(out, k, keep[k].ctypes.data_as(C.POINTER(C.c_double)))
    return out, keep


def zja_finish(out, keep):
    """ZjaOutcome as a dict: 'rounds' = [pilot?, main], each a run report + betas/lambda."""
    T = out.steps
    def rep(r, b, n):
        d = {k: v[: n + 1].copy() for k, v in b.items() if k != "resample_times"}
        d["resample_times"] = [int(v) for v in b["resample_times"][: r.n_resample_times]]
        d.update(log_z_hat=r.log_z_hat, elbo_hat=r.elbo_hat, kernel_applications=r.kernel_applications,
                 wall_seconds=r.wall_seconds)
        return d
    main = rep(out.main, keep["main"], T)
    main.update(round=2 if out.pilot_ran else 1, betas=keep["betas"][: T + 1].copy(),
                lambda_=keep["lambda_"][: T + 1].copy())
    rounds = [main]
    if out.pilot_ran:
        K = len(keep["pilot_lambda"]) - 1
        pilot = rep(out.pilot, keep["pilot"], K)
        pilot.update(round=1, lambda_=keep["pilot_lambda"].copy())
        rounds.insert(0, pilot)
    return {"rounds": rounds, "delta_star": out.delta_star, "warning": bool(out.warning), "steps": T}


def target(kind, dim, *params):
    t = TargetDesc()
    t.kind = kind
    t.dim = dim
    for i, v in enumerate(params):
        t.p[i] = float(v)
    return t


def gaussian_shift(mu0, mu1, sigma, dim=1):
    return target(TARGET_GAUSSIAN_SHIFT, dim, mu0, mu1, sigma)


def mixture(ref_sigma, weight, mu1, sigma1, mu2, sigma2, dim=1):
    return target(TARGET_MIXTURE, dim, ref_sigma, weight, mu1, sigma1, mu2, sigma2)


def scale_gaussian(sigma0, sigma1, dim=1):
    return target(TARGET_SCALE_GAUSSIAN, dim, sigma0, sigma1)


def ising(L, K, delta=1.0, sigma=1.0):
    """Config 5: relaxed Ising on an L x L torus (ASMC_TARGET_ISING), coupling K = beta J."""
    return target(TARGET_ISING, L * L, L, K, delta, sigma)


def _bf16_round(a):
    """round-to-nearest-even float32 -> bfloat16, returned as float32"""
    import numpy as np
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def logistic_data(n=100000, d=256, seed=0, split_exact=False):
    """Config-4 synthetic data: X ~ N(0, 1/d) in fp32, theta* ~ N(0, I),
    y ~ Bernoulli(sigmoid(X theta*)).  Deterministic in `seed` (numpy PCG64).
    split_exact=True rounds X to values exactly representable as a bf16 hi + bf16 lo pair
    (the device's split operand is then exact: a test hook isolating the other error
    sources); the default is general fp32 X, where the split drops x - hi - lo
    (|.| <= 2^-17 |x|) -- the precision scheme's stated error."""
    import numpy as np
    g = np.random.default_rng(seed)
    X = (g.standard_normal((n, d)) / np.sqrt(d)).astype(np.float32)
    if split_exact:
        hi = _bf16_round(X)
        lo = _bf16_round(X - hi)
        X = (hi + lo).astype(np.float32)
    theta = g.standard_normal(d)
    p = 1.0 / (1.0 + np.exp(-(X.astype(np.float64) @ theta)))
    y = (g.uniform(size=n) < p).astype(np.float32)
    return X, y


def logistic(X, y, sigma_p=1.0):
    """Descriptor of the logistic-regression posterior; keeps the packed data alive."""
    import numpy as np
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    n, d = X.shape
    buf = np.concatenate([X.ravel(), y])
    t = target(TARGET_LOGISTIC, d, sigma_p, float(n))
    t.data = buf.ctypes.data
    t.data_bytes = buf.nbytes
    t._keep = buf
    return t


def kernel(kind=KERNEL_IDEALIZED, step_sizes=(0.1, 1.0, 10.0), sweeps=1, leapfrog=10):
    k = KernelDesc()
    k.kind = kind
    k.n_step_sizes = len(step_sizes)
    k.sweeps = sweeps
    k.leapfrog = leapfrog
    for i, s in enumerate(step_sizes):
        k.step_sizes[i] = float(s)
    return k


def execopts(rng=RNG_XOSHIRO, precision=PREC_FP64, device=0, lanes=0, stream=0):
    e = Exec()
    e.rng, e.precision, e.device, e.lanes, e.stream = rng, precision, device, lanes, stream
    return e
