"""ORACLE -- test infrastructure only, never the product.

Loads the CPU checkers built by oracle/Makefile into oracle/_ref/:

* ``ref``          -- libasmc_ref.so: the UNMODIFIED reference sources
                      (/root/reference/proj/src/*.cpp) behind a C harness
                      (oracle/ref_harness.cpp), keyed-xoshiro streams.
* ``ref_philox``   -- libasmc_ref_philox.so: the same reference sources compiled
                      against the Philox shadow header oracle/shadow/asmc/rng.hpp.
* ``ref_release``  -- libasmc_ref_release.so: the unmodified reference at its own
                      Release flags (-O3 -DNDEBUG), the CPU baseline bench.py times.
* ``restate``      -- liborarestate.so: oracle/restate.c, the plain-C
                      restatement of the path (both stream families), pinned
                      bit-for-bit against the two above by tests/test_oracle.py.

Only tests/, bench.py (cpu_baseline leg and ``--impl reference``) and
__graft_entry__.smoke() may import this package, and only as the checker.
"""
import ctypes as C
import math
import os

import numpy as np

from paper_2408_12057_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_P = C.POINTER
_D = _P(C.c_double)


def _arr(a, ctype):
    return a.ctypes.data_as(_P(ctype))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class Oracle:
    """ctypes view over one oracle library (same C signatures for all three)."""

    def __init__(self, path, rng=None):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        self.path = path
        self.rng = rng
        L = self.lib
        L.ora_last_error.restype = C.c_char_p

    # -- plumbing -------------------------------------------------------
    def _call(self, name, *args):
        if self.rng is not None:
            self.lib.ora_set_rng(C.c_int(self.rng))
        rc = getattr(self.lib, name)(*args)
        if rc != 0:
            raise OracleError(rc, self.lib.ora_last_error().decode())

    @staticmethod
    def _report(T):
        bufs = dict(
            log_g0=np.full(T + 1, -np.inf), log_g1=np.full(T + 1, -np.inf),
            log_g2=np.full(T + 1, -np.inf), ess_trace=np.zeros(T + 1),
            cum_log_z=np.zeros(T + 1), resampled=np.zeros(T + 1, np.uint8),
            resample_times=np.zeros(T + 1, np.int32))
        rep = abi.Report()
        for k in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
            setattr(rep, k, _arr(bufs[k], C.c_double))
        rep.resampled = _arr(bufs["resampled"], C.c_uint8)
        rep.resample_times = _arr(bufs["resample_times"], C.c_int32)
        return rep, bufs

    @staticmethod
    def _finish(rep, bufs):
        out = dict(bufs)
        out["resample_times"] = [int(v) for v in bufs["resample_times"][: rep.n_resample_times]]
        out.update(log_z_hat=rep.log_z_hat, elbo_hat=rep.elbo_hat,
                   kernel_applications=rep.kernel_applications, wall_seconds=rep.wall_seconds)
        return out

    # -- samplers -------------------------------------------------------
    def run_smc(self, target, kernel, betas, n, policy=abi.POLICY_ADAPTIVE_ESS, rho=0.5,
                seed=0, round=0, workers=1):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        T = len(betas) - 1
        rep, bufs = self._report(T)
        self._call("ora_run_smc", C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                   C.c_int32(T), C.c_uint64(n), C.c_int32(policy), C.c_double(rho),
                   C.c_uint64(seed), C.c_uint64(round), C.c_int32(workers), C.byref(rep))
        return self._finish(rep, bufs)

    def run_pt(self, target, kernel, betas, iterations=1024, burn_in=-1, seed=0, round=1, replicas=1):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        L = len(betas) - 1
        o, out, b = abi.pt_buffers(L, iterations, burn_in, seed, round, replicas)
        self._call("ora_run_pt", C.byref(target), C.byref(kernel), _arr(betas, C.c_double), C.c_int32(L),
                   C.byref(o), C.byref(out))
        return abi.pt_finish(out, b)

    def run_zja(self, target, kernel, n, target_steps=32, delta_star=0.0, seed=0, max_steps=100000, workers=1):
        o = abi.zja_opts(n, target_steps, delta_star, seed, max_steps)
        out, keep = abi.zja_buffers(o)
        self._call("ora_run_zja", C.byref(target), C.byref(kernel), C.byref(o), C.c_int32(workers), C.byref(out))
        return abi.zja_finish(out, keep)

    def zja_next_beta(self, target, beta, positions, log_weights, delta_star, tol=1e-10):
        x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1)
        lw = np.ascontiguousarray(log_weights, dtype=np.float64)
        nb, w = C.c_double(0.0), C.c_int32(0)
        self._call("ora_zja_next_beta", C.byref(target), C.c_double(beta), _arr(x, C.c_double),
                   C.c_uint64(len(lw)), _arr(lw, C.c_double), C.c_double(delta_star), C.c_double(tol),
                   C.byref(nb), C.byref(w))
        return nb.value, bool(w.value)

    def run_sais_single(self, target, kernel, betas, n, seed=0, round=0, workers=1, chunk=0):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        T = len(betas) - 1
        rep, bufs = self._report(T)
        self._call("ora_run_sais_single", C.byref(target), C.byref(kernel),
                   _arr(betas, C.c_double), C.c_int32(T), C.c_uint64(n), C.c_uint64(seed),
                   C.c_uint64(round), C.c_int32(workers), C.c_uint64(chunk), C.byref(rep))
        return self._finish(rep, bufs)

    def run_rounds(self, target, kernel, mode, n, rounds, policy=abi.POLICY_ADAPTIVE_ESS,
                   rho=0.5, seed=0, memory_cap=4096 << 20, workers=1, max_steps=None):
        if max_steps is None:
            t, ms = 1, 1
            for _ in range(rounds):
                ms = max(ms, t)
                t = max(math.ceil(math.sqrt(2.0) * t), 2 * t)
            max_steps = ms
        R, S = rounds, max_steps + 1
        bufs = dict(n_particles=np.zeros(R, np.uint64), steps=np.zeros(R, np.int32),
                    betas=np.zeros((R, S)), log_g0=np.zeros((R, S)), log_g1=np.zeros((R, S)),
                    log_g2=np.zeros((R, S)), ess_trace=np.zeros((R, S)),
                    cum_log_z=np.zeros((R, S)), resampled=np.zeros((R, S), np.uint8),
                    lambda_=np.zeros((R, S)), log_z_hat=np.zeros(R), elbo_hat=np.zeros(R),
                    wall_seconds=np.zeros(R), kernel_applications=np.zeros(R, np.uint64))
        out = abi.RoundsOut()
        out.max_steps = max_steps
        types = dict(n_particles=C.c_uint64, steps=C.c_int32, resampled=C.c_uint8,
                     kernel_applications=C.c_uint64)
        for k, v in bufs.items():
            setattr(out, k, _arr(v, types.get(k, C.c_double)))
        self._call("ora_run_rounds", C.byref(target), C.byref(kernel), C.c_int32(mode),
                   C.c_uint64(n), C.c_int32(rounds), C.c_int32(policy), C.c_double(rho),
                   C.c_uint64(seed), C.c_uint64(memory_cap), C.c_int32(workers), C.byref(out))
        return bufs

    def trajectory(self, target, kernel, betas, seed, round, particle):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        T = len(betas) - 1
        x = np.zeros((T + 1, target.dim))
        lw = np.zeros(T + 1)
        lg = np.zeros(T + 1)
        self._call("ora_trajectory", C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                   C.c_int32(T), C.c_uint64(seed), C.c_uint64(round), C.c_uint64(particle),
                   _arr(x, C.c_double), _arr(lw, C.c_double), _arr(lg, C.c_double))
        return x, lw, lg

    # -- rng ------------------------------------------------------------
    def _key(self, key):
        return (C.c_uint64 * 5)(*[int(k) for k in key])

    def rng_u64(self, key, count):
        out = np.zeros(count, np.uint64)
        self._call("ora_rng_u64", self._key(key), C.c_uint64(count), _arr(out, C.c_uint64))
        return out

    def rng_uniform(self, key, count):
        out = np.zeros(count)
        self._call("ora_rng_uniform", self._key(key), C.c_uint64(count), _arr(out, C.c_double))
        return out

    def rng_normal(self, key, count):
        out = np.zeros(count)
        self._call("ora_rng_normal", self._key(key), C.c_uint64(count), _arr(out, C.c_double))
        return out

    # -- engine helpers -------------------------------------------------
    def systematic_resample(self, log_w, key):
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        out = np.zeros(len(lw), np.uint32)
        self._call("ora_systematic_resample", _arr(lw, C.c_double), C.c_uint64(len(lw)),
                   self._key(key), _arr(out, C.c_uint32))
        return out

    def systematic_resample_u(self, log_w, u):
        """engine.cpp:61-80 with the uniform given (restatement only)."""
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        out = np.zeros(len(lw), np.uint32)
        self._call("ora_systematic_resample_u", _arr(lw, C.c_double), C.c_uint64(len(lw)),
                   C.c_double(u), _arr(out, C.c_uint32))
        return out

    def resample_cdf(self, log_w):
        """(cum, l1): the sequential CDF engine.cpp:64-75 walks (restatement only)."""
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        cum = np.zeros(len(lw))
        l1 = C.c_double()
        self._call("ora_resample_cdf", _arr(lw, C.c_double), C.c_uint64(len(lw)), _arr(cum, C.c_double),
                   C.byref(l1))
        return cum, l1.value

    def cdf_given_l1(self, log_w, l1):
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        cum = np.zeros(len(lw))
        self._call("ora_cdf_given_l1", _arr(lw, C.c_double), C.c_uint64(len(lw)), C.c_double(l1),
                   _arr(cum, C.c_double))
        return cum

    def libm(self, which, x):
        """The host libm's exp (which=0) / log (which=1), element-wise."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(len(x))
        self._call("ora_libm", C.c_int(which), _arr(x, C.c_double), C.c_uint64(len(x)), _arr(out, C.c_double))
        return out

    def ess(self, log_w):
        lw = np.ascontiguousarray(log_w, dtype=np.float64)
        out = C.c_double()
        self._call("ora_ess", _arr(lw, C.c_double), C.c_uint64(len(lw)), C.byref(out))
        return out.value

    # -- schedule -------------------------------------------------------
    def barrier_estimate(self, g0, g1, g2, betas):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        g = [np.ascontiguousarray(v, dtype=np.float64) for v in (g0, g1, g2)]
        T = len(betas) - 1
        lam = np.zeros(T + 1)
        self._call("ora_barrier_estimate", *[_arr(v, C.c_double) for v in g],
                   _arr(betas, C.c_double), C.c_int32(T), _arr(lam, C.c_double))
        return lam

    def generate_schedule(self, lam, beta, t_new):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        beta = np.ascontiguousarray(beta, dtype=np.float64)
        out = np.zeros(t_new + 1)
        self._call("ora_generate_schedule", _arr(lam, C.c_double), _arr(beta, C.c_double),
                   C.c_int32(len(lam)), C.c_int32(t_new), _arr(out, C.c_double))
        return out

    def local_barrier(self, lam, beta):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        beta = np.ascontiguousarray(beta, dtype=np.float64)
        out = np.zeros(len(lam))
        self._call("ora_local_barrier", _arr(lam, C.c_double), _arr(beta, C.c_double),
                   C.c_int32(len(lam)), _arr(out, C.c_double))
        return out

    def budget(self, n, steps, dim, cap, mode):
        nn, tt = C.c_uint64(), C.c_int32()
        self._call("ora_budget", C.c_uint64(n), C.c_int32(steps), C.c_uint64(dim),
                   C.c_uint64(cap), C.c_int32(mode), C.byref(nn), C.byref(tt))
        return nn.value, tt.value

    def hardware_threads(self):
        return self.lib.ora_hardware_threads()


_cache = {}


def load(which="restate", rng=abi.RNG_XOSHIRO):
    """which: 'ref' (unmodified reference; rng picks xoshiro or the Philox shadow
    build), 'ref_release' (the same sources at the reference's Release -O3, for timing)
    or 'restate' (oracle/restate.c, rng selects the stream family)."""
    key = (which, rng)
    if key not in _cache:
        if which == "ref":
            name = "libasmc_ref.so" if rng == abi.RNG_XOSHIRO else "libasmc_ref_philox.so"
            _cache[key] = Oracle(os.path.join(REF_DIR, name))
        elif which == "ref_release":  # the timed CPU baseline: reference Release flags (-O3)
            _cache[key] = Oracle(os.path.join(REF_DIR, "libasmc_ref_release.so"))
        elif which == "restate":
            _cache[key] = Oracle(os.path.join(REF_DIR, "liborarestate.so"), rng=rng)
        else:
            raise ValueError(which)
    return _cache[key]


def available(which="ref", rng=abi.RNG_XOSHIRO):
    name = {("ref", 0): "libasmc_ref.so", ("ref", 1): "libasmc_ref_philox.so",
            ("ref_release", 0): "libasmc_ref_release.so"}.get((which, rng), "liborarestate.so")
    return os.path.exists(os.path.join(REF_DIR, name))
