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


def logistic_data(n=100000, d=256, seed=0):
    """Config-4 synthetic data: X ~ N(0, 1/d) rounded to values exactly representable as a
    bf16 hi + bf16 lo pair (so the device's split-bf16 operand is exact), theta* ~ N(0, I),
    y ~ Bernoulli(sigmoid(X theta*)).  Deterministic in `seed` (numpy PCG64)."""
    import numpy as np
    g = np.random.default_rng(seed)
    x = (g.standard_normal((n, d)) / np.sqrt(d)).astype(np.float32)
    hi = _bf16_round(x)
    lo = _bf16_round(x - hi)
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
