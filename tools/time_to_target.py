"""Time to a target relative variance of Z-hat (BASELINE metric, second half).

Config 1 family (SAIS, d = 10 Gaussian shift, exact log Z = 0, RWMH {0.1,1,10},
N_1 = 2^14, doubling rounds).  For R seeds, rel-var_k = Var(Z_k)/E[Z_k]^2 of the
round-k estimate; k* = first round with rel-var_k <= target.  Time to target =
mean over seeds of the cumulative round times up to k*:
  * B200: CUDA-event round times from asmc_run_rounds (reference arithmetic:
    keyed xoshiro + fp64, so the estimates -- and hence k* -- are the
    reference's own; the Philox/fp32 mode is reported beside it);
  * CPU: the unmodified reference (oracle/_ref) run_sais for k* rounds with
    workers = all host cores, on a few seeds (its time does not depend on the seed).
As in the paper process start and JIT are excluded.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_12057_b200 import abi  # noqa: E402


def rel_var(log_z):
    z = np.exp(np.asarray(log_z) - 0.0)
    return float(np.var(z, ddof=1) / np.mean(z) ** 2)


def gpu_runs(seeds, rounds, n1, rng, prec, device=0, streams=16):
    """All seeds' round loops, `streams` at a time: each host thread drives its own
    CUDA stream (the library keeps a per-thread context), so independent replicas
    overlap on the device; per-seed round times are that seed's CUDA events."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2408_12057_b200 import capi
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
    k = abi.kernel(abi.KERNEL_RWMH)
    ex = abi.execopts(rng, prec, device=device)

    def one(s):
        r = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, rounds, seed=int(s), exec_=ex)
        return r["log_z_hat"].copy(), r["wall_seconds"].copy()

    with ThreadPoolExecutor(max_workers=streams) as pool:
        res = list(pool.map(one, seeds))
    return np.array([a for a, _ in res]), np.array([b for _, b in res])


def cpu_time(rounds, n1, workers, seeds):
    import oracle
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
    k = abi.kernel(abi.KERNEL_RWMH)
    ts = []
    for s in seeds:
        t0 = time.perf_counter()
        ref.run_rounds(tg, k, abi.MODE_SAIS, n1, rounds, seed=int(s), workers=workers)
        ts.append(time.perf_counter() - t0)
    return float(np.mean(ts))


def measure(n_seeds=1000, target=0.05, rounds=6, n1=1 << 14, cpu_seeds=3, timing_seeds=20):
    out = {"config": "config1: SAIS d=10 Gaussian shift (log Z = 0), RWMH {0.1,1,10}, N1=2^14, doubling rounds",
           "target_rel_var": target, "seeds": n_seeds}
    # estimator statistics over all seeds: concurrent streams (replicas overlap on the
    # device); the time-to-target itself: CUDA-event round times of uncontended runs
    t0 = time.perf_counter()
    lz, _ = gpu_runs(range(1, n_seeds + 1), rounds, n1, abi.RNG_XOSHIRO, abi.PREC_FP64, streams=16)
    out["all_seeds_wall_seconds"] = time.perf_counter() - t0
    _, wall = gpu_runs(range(1, timing_seeds + 1), rounds, n1, abi.RNG_XOSHIRO, abi.PREC_FP64, streams=1)
    rv = [rel_var(lz[:, k]) for k in range(rounds)]
    out["rel_var_by_round"] = rv
    hit = [k for k in range(rounds) if rv[k] <= target]
    if not hit:
        out["reached"] = False
        return out
    ks = hit[0]
    out.update(reached=True, rounds_needed=ks + 1,
               b200_seconds=float(np.mean(np.sum(wall[:, : ks + 1], axis=1))))
    lz32, _ = gpu_runs(range(1, n_seeds + 1), rounds, n1, abi.RNG_PHILOX, abi.PREC_FP32, streams=16)
    _, wall32 = gpu_runs(range(1, timing_seeds + 1), rounds, n1, abi.RNG_PHILOX, abi.PREC_FP32, streams=1)
    rv32 = [rel_var(lz32[:, k]) for k in range(rounds)]
    hit32 = [k for k in range(rounds) if rv32[k] <= target]
    out["philox_fp32"] = {"rel_var_by_round": rv32,
                          "rounds_needed": hit32[0] + 1 if hit32 else None,
                          "b200_seconds": float(np.mean(np.sum(wall32[:, : hit32[0] + 1], axis=1)))
                          if hit32 else None}
    workers = os.cpu_count() or 1
    out["cpu_seconds"] = cpu_time(ks + 1, n1, workers, range(1, cpu_seeds + 1))
    out["cpu_seconds_1core"] = cpu_time(ks + 1, n1, 1, range(1, 2))
    out["cpu_cores"] = workers
    out["cpu_kind"] = "reference (oracle/_ref, unmodified run_sais)"
    out["speedup_vs_cpu_all_cores"] = out["cpu_seconds"] / out["b200_seconds"]
    return out


if __name__ == "__main__":
    import json
    print(json.dumps(measure(), indent=1))
