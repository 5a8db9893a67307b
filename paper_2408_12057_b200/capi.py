"""ctypes binding of the C-ABI in include/asmc_b200.h (libasmc_b200.so).

This is the reference-facing drop-in boundary seen from Python: plain host
arrays in, host arrays out, one call per sampler invocation.  Loading fails
loudly when the native library is missing -- there is no CPU fallback.
"""
import ctypes as C
import math
import os

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ASMC_B200_LIB", os.path.join(HERE, "libasmc_b200.so"))

_P = C.POINTER


def _arr(a, ctype):
    return a.ctypes.data_as(_P(ctype))


class AsmcError(RuntimeError):
    """Raised for a non-zero C-ABI return code; ``code`` is the ASMC_ERR_* value."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.msg = msg


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libasmc_b200.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.asmc_last_error.restype = C.c_char_p
        L.asmc_launch_count.restype = C.c_uint64
        L.asmc_launch_count.argtypes = [C.c_int]
        L.asmc_fold_chunks.restype = C.c_uint64
        L.asmc_fold_chunks.argtypes = [C.c_uint64, C.c_uint64]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise AsmcError(rc, lib().asmc_last_error().decode())


def device_count():
    return lib().asmc_device_count()


def launch_count(reset=False):
    return lib().asmc_launch_count(1 if reset else 0)


def _report(T):
    bufs = dict(log_g0=np.full(T + 1, -np.inf), log_g1=np.full(T + 1, -np.inf),
                log_g2=np.full(T + 1, -np.inf), ess_trace=np.zeros(T + 1),
                cum_log_z=np.zeros(T + 1), resampled=np.zeros(T + 1, np.uint8),
                resample_times=np.zeros(T + 1, np.int32))
    rep = abi.Report()
    for k in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
        setattr(rep, k, _arr(bufs[k], C.c_double))
    rep.resampled = _arr(bufs["resampled"], C.c_uint8)
    rep.resample_times = _arr(bufs["resample_times"], C.c_int32)
    return rep, bufs


def _finish(rep, bufs, smc):
    out = dict(bufs)
    if not smc:
        out["ess_trace"] = np.zeros(0)
    out["resample_times"] = [int(v) for v in bufs["resample_times"][: rep.n_resample_times]]
    out.update(log_z_hat=rep.log_z_hat, elbo_hat=rep.elbo_hat,
               kernel_applications=rep.kernel_applications, wall_seconds=rep.wall_seconds)
    return out


def run_smc(target, kernel, betas, n, policy=abi.POLICY_ADAPTIVE_ESS, rho=0.5, seed=0, round=0,
            exec_=None):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    T = len(betas) - 1
    rep, bufs = _report(T)
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_smc(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                              C.c_int32(T), C.c_uint64(n), C.c_int32(policy), C.c_double(rho),
                              C.c_uint64(seed), C.c_uint64(round), C.byref(ex), C.byref(rep)))
    return _finish(rep, bufs, True)


def run_sais_single(target, kernel, betas, n, seed=0, round=0, exec_=None):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    T = len(betas) - 1
    rep, bufs = _report(T)
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_sais_single(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                                      C.c_int32(T), C.c_uint64(n), C.c_uint64(seed),
                                      C.c_uint64(round), C.byref(ex), C.byref(rep)))
    return _finish(rep, bufs, False)


def plan_steps(rounds, n1, dim, memory_cap, mode):
    ns, ts = [n1], [1]
    for _ in range(1, rounds):
        nn, tt = budget(ns[-1], ts[-1], dim, memory_cap, mode)
        ns.append(nn)
        ts.append(tt)
    return ns, ts


def run_rounds(target, kernel, mode, n, rounds, policy=abi.POLICY_ADAPTIVE_ESS, rho=0.5, seed=0,
               memory_cap=4096 << 20, exec_=None):
    _, ts = plan_steps(rounds, n, target.dim, memory_cap, mode)
    max_steps = max(ts)
    R, S = rounds, max_steps + 1
    bufs = dict(n_particles=np.zeros(R, np.uint64), steps=np.zeros(R, np.int32),
                betas=np.zeros((R, S)), log_g0=np.zeros((R, S)), log_g1=np.zeros((R, S)),
                log_g2=np.zeros((R, S)), ess_trace=np.zeros((R, S)), cum_log_z=np.zeros((R, S)),
                resampled=np.zeros((R, S), np.uint8), lambda_=np.zeros((R, S)),
                log_z_hat=np.zeros(R), elbo_hat=np.zeros(R), wall_seconds=np.zeros(R),
                kernel_applications=np.zeros(R, np.uint64))
    out = abi.RoundsOut()
    out.max_steps = max_steps
    types = dict(n_particles=C.c_uint64, steps=C.c_int32, resampled=C.c_uint8,
                 kernel_applications=C.c_uint64)
    for k, v in bufs.items():
        setattr(out, k, _arr(v, types.get(k, C.c_double)))
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_rounds(C.byref(target), C.byref(kernel), C.c_int32(mode), C.c_uint64(n),
                                 C.c_int32(rounds), C.c_int32(policy), C.c_double(rho),
                                 C.c_uint64(seed), C.c_uint64(memory_cap), C.byref(ex),
                                 C.byref(out)))
    return bufs


def run_sais_seeds(target, kernel, n, rounds, seeds, exec_=None):
    """run_sais for many seeds in one batched launch per kernel (asmc_run_sais_seeds).
    Returns dict: per round n_particles, steps, wall_seconds; per (seed, round) arrays
    log_z_hat, elbo_hat, lambda_total of shape (nseeds, rounds)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    S = len(seeds)
    bufs = dict(n_particles=np.zeros(rounds, np.uint64), steps=np.zeros(rounds, np.int32),
                wall_seconds=np.zeros(rounds), log_z_hat=np.zeros((S, rounds)), elbo_hat=np.zeros((S, rounds)),
                lambda_total=np.zeros((S, rounds)))
    out = abi.SeedsOut()
    types = dict(n_particles=C.c_uint64, steps=C.c_int32)
    for k, v in bufs.items():
        setattr(out, k, _arr(v, types.get(k, C.c_double)))
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_sais_seeds(C.byref(target), C.byref(kernel), C.c_uint64(n), C.c_int32(rounds),
                                     _arr(seeds, C.c_uint64), C.c_int32(S), C.byref(ex), C.byref(out)))
    return bufs


def fold_chunks(p_begin, p_end):
    return lib().asmc_fold_chunks(C.c_uint64(p_begin), C.c_uint64(p_end))


def sais_partials(target, kernel, betas, n, p_begin, p_end, seed=0, round=0, exec_=None):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    T = len(betas) - 1
    nch = fold_chunks(p_begin, p_end)
    out = np.zeros((max(nch, 1), T + 1, 4, 2))
    ex = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    _check(lib().asmc_sais_partials(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                                    C.c_int32(T), C.c_uint64(n), C.c_uint64(p_begin),
                                    C.c_uint64(p_end), C.c_uint64(seed), C.c_uint64(round),
                                    C.byref(ex), _arr(out, C.c_double)))
    return out[:nch]


def sais_partials_dev(target, kernel, betas, n, p_begin, p_end, out_ptr, seed=0, round=0, exec_=None):
    """asmc_sais_partials_dev: this rank's chunk partials written to a DEVICE buffer
    (out_ptr, e.g. a float64 tensor of shape (chunks, T+1, 4, 2)) on exec_.stream."""
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    T = len(betas) - 1
    ex = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    _check(lib().asmc_sais_partials_dev(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                                        C.c_int32(T), C.c_uint64(n), C.c_uint64(p_begin), C.c_uint64(p_end),
                                        C.c_uint64(seed), C.c_uint64(round), C.byref(ex), C.c_void_p(out_ptr)))


def fold_partials_dev(partials_ptr, chunks, T, n, exec_=None):
    """asmc_fold_partials_dev: fold all-gathered DEVICE partials on the GPU."""
    rep, bufs = _report(T)
    ex = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    _check(lib().asmc_fold_partials_dev(C.c_void_p(partials_ptr), C.c_uint64(chunks), C.c_int32(T),
                                        C.c_uint64(n), C.byref(ex), C.byref(rep)))
    return _finish(rep, bufs, False)


def fold_partials(partials, n):
    partials = np.ascontiguousarray(partials, dtype=np.float64)
    chunks, T1 = partials.shape[0], partials.shape[1]
    T = T1 - 1
    rep, bufs = _report(T)
    _check(lib().asmc_fold_partials(_arr(partials, C.c_double), C.c_uint64(chunks), C.c_int32(T),
                                    C.c_uint64(n), C.byref(rep)))
    return _finish(rep, bufs, False)


def trajectories(target, kernel, betas, seed, round, particles, exec_=None):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    T = len(betas) - 1
    pids = np.ascontiguousarray(particles, dtype=np.uint64)
    x = np.zeros((len(pids), T + 1, target.dim))
    lw = np.zeros((len(pids), T + 1))
    ex = exec_ or abi.execopts()
    _check(lib().asmc_trajectories(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                                   C.c_int32(T), C.c_uint64(seed), C.c_uint64(round),
                                   _arr(pids, C.c_uint64), C.c_uint64(len(pids)), C.byref(ex),
                                   _arr(x, C.c_double), _arr(lw, C.c_double)))
    return x, lw


def _key(key):
    return (C.c_uint64 * 5)(*[int(k) for k in key])


def rng_u64(rng, key, count):
    out = np.zeros(count, np.uint64)
    _check(lib().asmc_rng_u64(C.c_int32(rng), _key(key), C.c_uint64(count), _arr(out, C.c_uint64)))
    return out


def rng_uniform(rng, key, count):
    out = np.zeros(count)
    _check(lib().asmc_rng_uniform(C.c_int32(rng), _key(key), C.c_uint64(count),
                                  _arr(out, C.c_double)))
    return out


def rng_normal(rng, key, count, precision=abi.PREC_FP64):
    out = np.zeros(count)
    _check(lib().asmc_rng_normal(C.c_int32(rng), C.c_int32(precision), _key(key),
                                 C.c_uint64(count), _arr(out, C.c_double)))
    return out


def systematic_resample(log_w, u, device=0):
    lw = np.ascontiguousarray(log_w, dtype=np.float64)
    out = np.zeros(len(lw), np.uint32)
    _check(lib().asmc_systematic_resample(_arr(lw, C.c_double), C.c_uint64(len(lw)),
                                          C.c_double(u), C.c_int32(device), _arr(out, C.c_uint32)))
    return out


def resample_cdf(log_w, device=0):
    """(cum, l1): the sequential CDF engine.cpp:64-75 walks, built on the device."""
    lw = np.ascontiguousarray(log_w, dtype=np.float64)
    cum = np.zeros(len(lw))
    l1 = C.c_double()
    _check(lib().asmc_resample_cdf(_arr(lw, C.c_double), C.c_uint64(len(lw)), C.c_int32(device),
                                   _arr(cum, C.c_double), C.byref(l1)))
    return cum, l1.value


def logsumexp(log_w, device=0):
    """asmc::logsumexp (logsum.hpp:97-101) on the device."""
    lw = np.ascontiguousarray(log_w, dtype=np.float64)
    out = C.c_double()
    _check(lib().asmc_logsumexp(_arr(lw, C.c_double), C.c_uint64(len(lw)), C.c_int32(device), C.byref(out)))
    return out.value


def exact_math(which, x, device=0):
    """The device's glibc-exact exp (which=0) / correctly rounded log (which=1)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(len(x))
    _check(lib().asmc_exact_math(C.c_int32(which), _arr(x, C.c_double), C.c_uint64(len(x)), C.c_int32(device),
                                 _arr(out, C.c_double)))
    return out


def ess(log_w, device=0):
    lw = np.ascontiguousarray(log_w, dtype=np.float64)
    out = C.c_double()
    _check(lib().asmc_ess(_arr(lw, C.c_double), C.c_uint64(len(lw)), C.c_int32(device),
                          C.byref(out)))
    return out.value


def barrier_estimate(g0, g1, g2, betas, device=0):
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    g = [np.ascontiguousarray(v, dtype=np.float64) for v in (g0, g1, g2)]
    T = len(betas) - 1
    lam = np.zeros(T + 1)
    _check(lib().asmc_barrier_estimate(*[_arr(v, C.c_double) for v in g], _arr(betas, C.c_double),
                                       C.c_int32(T), C.c_int32(device), _arr(lam, C.c_double)))
    return lam


def generate_schedule(lam, beta, t_new, device=0):
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    out = np.zeros(t_new + 1)
    _check(lib().asmc_generate_schedule(_arr(lam, C.c_double), _arr(beta, C.c_double),
                                        C.c_int32(len(lam)), C.c_int32(t_new), C.c_int32(device),
                                        _arr(out, C.c_double)))
    return out


def local_barrier(lam, beta, device=0):
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    out = np.zeros(len(lam))
    _check(lib().asmc_local_barrier(_arr(lam, C.c_double), _arr(beta, C.c_double),
                                    C.c_int32(len(lam)), C.c_int32(device), _arr(out, C.c_double)))
    return out


def budget(n, steps, dim, cap, mode):
    nn, tt = C.c_uint64(), C.c_int32()
    _check(lib().asmc_budget(C.c_uint64(n), C.c_int32(steps), C.c_uint64(dim), C.c_uint64(cap),
                             C.c_int32(mode), C.byref(nn), C.byref(tt)))
    return nn.value, tt.value


def profile_enable(on=True):
    _check(lib().asmc_profile_enable(C.c_int(1 if on else 0)))


def profile_collect(max_launches=65536, drawn=False):
    """(ms, algorithmic units) per profiled launch; with drawn=True also the normals
    each launch actually generated (early-rejected RWMH proposals draw fewer)."""
    ms = np.zeros(max_launches)
    nrm = np.zeros(max_launches)
    drw = np.zeros(max_launches)
    cnt = C.c_int()
    _check(lib().asmc_profile_collect_drawn(_arr(ms, C.c_double), _arr(nrm, C.c_double), _arr(drw, C.c_double),
                                            C.c_int(max_launches), C.byref(cnt)))
    k = min(cnt.value, max_launches)
    return (ms[:k], nrm[:k], drw[:k]) if drawn else (ms[:k], nrm[:k])


def peak_normals(device, blocks, quads_per_thread):
    s = C.c_double()
    _check(lib().asmc_peak_normals(C.c_int32(device), C.c_int32(blocks),
                                   C.c_uint64(quads_per_thread), C.byref(s)))
    return s.value


def run_pt(target, kernel, betas, iterations=1024, burn_in=-1, seed=0, round=1, replicas=1, exec_=None):
    """asmc::run_pt (pt.cpp:84-128) for `replicas` seeds at once; returns per-replica arrays."""
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    L = len(betas) - 1
    o, out, b = abi.pt_buffers(L, iterations, burn_in, seed, round, replicas)
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_pt(C.byref(target), C.byref(kernel), _arr(betas, C.c_double), C.c_int32(L), C.byref(o),
                             C.byref(ex), C.byref(out)))
    return abi.pt_finish(out, b)


def run_zja(target, kernel, n, target_steps=32, delta_star=0.0, seed=0, max_steps=100000, exec_=None):
    """asmc::run_zja (drivers.cpp:234-341) on the device; returns abi.zja_finish's dict."""
    o = abi.zja_opts(n, target_steps, delta_star, seed, max_steps)
    out, keep = abi.zja_buffers(o)
    ex = exec_ or abi.execopts()
    _check(lib().asmc_run_zja(C.byref(target), C.byref(kernel), C.byref(o), C.byref(ex), C.byref(out)))
    return abi.zja_finish(out, keep)


def zja_next_beta(target, beta, positions, log_weights, delta_star, tol=1e-10, exec_=None):
    """asmc::zja_next_beta (schedule.cpp:219-264); positions n x dim.  Returns (beta_next, warning)."""
    x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1)
    lw = np.ascontiguousarray(log_weights, dtype=np.float64)
    nb, w = C.c_double(0.0), C.c_int32(0)
    ex = exec_ or abi.execopts()
    _check(lib().asmc_zja_next_beta(C.byref(target), C.c_double(beta), _arr(x, C.c_double), C.c_uint64(len(lw)),
                                    _arr(lw, C.c_double), C.c_double(delta_star), C.c_double(tol), C.byref(ex),
                                    C.byref(nb), C.byref(w)))
    return nb.value, bool(w.value)


class SmcShard:
    """One GPU's particle shard of a multi-GPU run_smc (asmc_smc_shard_* in
    include/asmc_b200.h).  Buffers passed to the methods are DEVICE addresses
    (ints, e.g. ``tensor.data_ptr()``) on ``exec_.device``; the caller owns them
    and the collectives between the calls (paper_2408_12057_b200/distributed.py)."""

    def __init__(self, target, kernel, betas, n, p_begin, p_end, policy=abi.POLICY_ADAPTIVE_ESS,
                 rho=0.5, seed=0, round=0, exec_=None):
        L = lib()
        self._lib = L
        for f in ("asmc_smc_shard_chunks", "asmc_smc_shard_exchange_len", "asmc_smc_shard_row_bytes"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.asmc_smc_shard_destroy.argtypes = [C.c_void_p]
        L.asmc_smc_shard_destroy.restype = None
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        self.T = len(betas) - 1
        self.n, self.p_begin, self.p_end = n, p_begin, p_end
        self.exec_ = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
        self._target = target  # keeps a data-backed target's buffer alive
        h = C.c_void_p()
        _check(L.asmc_smc_shard_create(C.byref(target), C.byref(kernel), _arr(betas, C.c_double),
                                       C.c_int32(self.T), C.c_uint64(n), C.c_uint64(p_begin),
                                       C.c_uint64(p_end), C.c_int32(policy), C.c_double(rho),
                                       C.c_uint64(seed), C.c_uint64(round), C.byref(self.exec_),
                                       C.byref(h)))
        self._h = h
        self.chunks = L.asmc_smc_shard_chunks(h)
        self.exchange_len = L.asmc_smc_shard_exchange_len(h)
        self.row_bytes = L.asmc_smc_shard_row_bytes(h)

    def step(self, t, partials_ptr):
        _check(self._lib.asmc_smc_shard_step(self._h, C.c_int32(t), C.c_void_p(partials_ptr)))

    def decide(self, t, all_partials_ptr, all_chunks, lw_out_ptr):
        """Fold + decision; on a resampling step copies this shard's log-weights
        (exchange_len doubles) to lw_out_ptr for the caller's all-gather."""
        flag = C.c_int32(0)
        _check(self._lib.asmc_smc_shard_decide(self._h, C.c_int32(t), C.c_void_p(all_partials_ptr),
                                                C.c_uint64(all_chunks), C.c_void_p(lw_out_ptr),
                                                C.byref(flag)))
        return bool(flag.value)

    def plan(self, all_lw_ptr, n_all, shard_p_begin):
        """Global reference CDF over the all-gathered log-weights -> slot_begin."""
        b = np.ascontiguousarray(shard_p_begin, dtype=np.uint64)
        out = np.zeros(len(b), np.uint64)
        _check(self._lib.asmc_smc_shard_plan(self._h, C.c_void_p(all_lw_ptr),
                                              C.c_uint64(n_all), C.c_int32(len(b) - 1),
                                              _arr(b, C.c_uint64), _arr(out, C.c_uint64)))
        return [int(v) for v in out]

    def pack(self, rows_ptr):
        _check(self._lib.asmc_smc_shard_pack(self._h, C.c_void_p(rows_ptr)))

    def accept(self, rows_ptr):
        _check(self._lib.asmc_smc_shard_accept(self._h, C.c_void_p(rows_ptr)))

    def report(self):
        rep, bufs = _report(self.T)
        _check(self._lib.asmc_smc_shard_report(self._h, C.byref(rep)))
        return _finish(rep, bufs, True)

    def state(self):
        nl = self.p_end - self.p_begin
        rows = np.zeros(nl * self.row_bytes, np.uint8)
        lw = np.zeros(nl)
        _check(self._lib.asmc_smc_shard_state(self._h, _arr(rows, C.c_uint8), _arr(lw, C.c_double)))
        return rows.view(np.float32).reshape(nl, -1), lw

    def close(self):
        if getattr(self, "_h", None):
            self._lib.asmc_smc_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class ZjaShard(SmcShard):
    """One GPU's particle shard of a multi-GPU run_zja (asmc_zja_shard_* + the SMC
    shard step/decide); see distributed.run_zja_multi."""

    def __init__(self, target, kernel, n, p_begin, p_end, seed=0, round=1, max_steps=100000, exec_=None):
        L = lib()
        self._lib = L
        for f in ("asmc_smc_shard_chunks", "asmc_smc_shard_exchange_len", "asmc_smc_shard_row_bytes"):
            getattr(L, f).restype = C.c_uint64
            getattr(L, f).argtypes = [C.c_void_p]
        L.asmc_smc_shard_destroy.argtypes = [C.c_void_p]
        L.asmc_smc_shard_destroy.restype = None
        self.T = max_steps
        self.n, self.p_begin, self.p_end = n, p_begin, p_end
        self.exec_ = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
        self._target = target
        h = C.c_void_p()
        _check(L.asmc_zja_shard_create(C.byref(target), C.byref(kernel), C.c_uint64(n), C.c_uint64(p_begin),
                                       C.c_uint64(p_end), C.c_uint64(seed), C.c_uint64(round),
                                       C.c_int32(max_steps), C.byref(self.exec_), C.byref(h)))
        self._h = h
        self.chunks = L.asmc_smc_shard_chunks(h)
        self.exchange_len = L.asmc_smc_shard_exchange_len(h)
        self.row_bytes = L.asmc_smc_shard_row_bytes(h)

    def eval(self):
        _check(self._lib.asmc_zja_shard_eval(self._h))

    def probe(self, beta, b2):
        """(chunks, 2, 2) array: per chunk (m1, m2) as (max, sum)."""
        out = np.zeros((self.chunks, 2, 2))
        _check(self._lib.asmc_zja_shard_probe(self._h, C.c_double(beta), C.c_double(b2), _arr(out, C.c_double)))
        return out

    def set_beta(self, t, beta):
        _check(self._lib.asmc_zja_shard_set_beta(self._h, C.c_int32(t), C.c_double(beta)))

    # device-resident search: no host round trip per probe (asmc_zja_shard_search_*)
    def search_begin(self, t, delta_star):
        _check(self._lib.asmc_zja_shard_search_begin(self._h, C.c_int32(t), C.c_double(delta_star)))

    def probe_dev(self, out_ptr):
        """this shard's (chunks, 2) partials at the search's current point -> device out_ptr"""
        _check(self._lib.asmc_zja_shard_probe_dev(self._h, C.c_void_p(out_ptr)))

    def search_step(self, all_ptr, all_chunks):
        _check(self._lib.asmc_zja_shard_search_step(self._h, C.c_void_p(all_ptr), C.c_uint64(all_chunks)))

    def search_poll(self):
        """(done, chosen beta, warning, probes taken); synchronises the shard's stream"""
        done, warn, probes, beta = C.c_int32(), C.c_int32(), C.c_int32(), C.c_double()
        _check(self._lib.asmc_zja_shard_search_poll(self._h, C.byref(done), C.byref(beta), C.byref(warn),
                                                    C.byref(probes)))
        return bool(done.value), beta.value, bool(warn.value), probes.value

    def report(self, T=None):
        rep, bufs = _report(self.T if T is None else T)
        _check(self._lib.asmc_smc_shard_report(self._h, C.byref(rep)))
        return _finish(rep, bufs, True)


EXPORTED = [
    "asmc_last_error", "asmc_version", "asmc_device_count", "asmc_launch_count", "asmc_run_smc",
    "asmc_run_sais_single", "asmc_run_rounds", "asmc_run_sais_seeds", "asmc_fold_chunks", "asmc_sais_partials",
    "asmc_fold_partials", "asmc_sais_partials_dev", "asmc_fold_partials_dev", "asmc_rng_u64", "asmc_rng_uniform", "asmc_rng_normal",
    "asmc_trajectories", "asmc_systematic_resample", "asmc_resample_cdf", "asmc_logsumexp",
    "asmc_exact_math", "asmc_ess", "asmc_barrier_estimate",
    "asmc_generate_schedule", "asmc_local_barrier", "asmc_budget", "asmc_profile_enable",
    "asmc_profile_collect", "asmc_peak_normals", "asmc_smc_shard_create", "asmc_smc_shard_destroy",
    "asmc_smc_shard_chunks", "asmc_smc_shard_exchange_len", "asmc_smc_shard_row_bytes",
    "asmc_smc_shard_step", "asmc_smc_shard_decide", "asmc_smc_shard_plan", "asmc_smc_shard_pack",
    "asmc_smc_shard_accept", "asmc_smc_shard_report", "asmc_smc_shard_state", "asmc_run_zja",
    "asmc_zja_next_beta", "asmc_run_pt", "asmc_profile_collect_drawn", "asmc_zja_shard_create",
    "asmc_zja_shard_eval", "asmc_zja_shard_probe", "asmc_zja_shard_set_beta", "asmc_zja_shard_search_begin",
    "asmc_zja_shard_probe_dev", "asmc_zja_shard_search_step", "asmc_zja_shard_search_poll",
]
