"""Throughput of the other BASELINE configs on one B200 (bench.py covers config 2).

  config 1: SAIS d=10 Gaussian shift, RWMH, N1=2^14, 4 rounds (a parity config:
            the whole run is ~4e5 p-steps, so it is latency-bound)
  config 3: SSMC, adaptive-ESS (rho 0.5) systematic resampling, d=100 bimodal
            MixtureTarget(2, .5, -1, .5, 1, .5), RWMH, N1=2^22, 6 rounds with the
            reference's default 4 GiB memory cap (SSMC budget: N fixed, T doubles)
Device time = the per-round CUDA-event times asmc_run_rounds reports.  The CPU
rate is the unmodified reference (oracle/_ref) on a bounded sample with all
host cores.  Prints one JSON document.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_12057_b200 import abi, capi  # noqa: E402

CONFIGS = {
    "config1": dict(target=abi.gaussian_shift(0.0, 1.0, 1.0, 10), mode=abi.MODE_SAIS, n1=1 << 14,
                    rounds=4, policy=abi.POLICY_NEVER, cpu_n1=1 << 14),
    "config3": dict(target=abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100), mode=abi.MODE_SSMC,
                    n1=1 << 22, rounds=6, policy=abi.POLICY_ADAPTIVE_ESS, cpu_n1=1 << 11),
}


def run_gpu(c, rng, prec, reps=2):
    k = abi.kernel(abi.KERNEL_RWMH)
    ex = abi.execopts(rng, prec)
    capi.run_rounds(c["target"], k, c["mode"], min(c["n1"], 4096), c["rounds"], policy=c["policy"],
                    seed=1, exec_=ex)  # warm-up
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = capi.run_rounds(c["target"], k, c["mode"], c["n1"], c["rounds"], policy=c["policy"],
                            seed=1, exec_=ex)
        wall = time.perf_counter() - t0
        dev = float(np.sum(r["wall_seconds"]))
        ps = int(np.sum(r["kernel_applications"]))
        rec = {"psteps": ps, "device_s": dev, "wall_s": wall, "psteps_per_s": ps / dev,
               "n": [int(v) for v in r["n_particles"]], "T": [int(v) for v in r["steps"]],
               "log_z_hat": [float(v) for v in r["log_z_hat"]]}
        if best is None or rec["device_s"] < best["device_s"]:
            best = rec
    return best


def run_cpu(c):
    import oracle
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    workers = os.cpu_count() or 1
    t0 = time.perf_counter()
    r = ref.run_rounds(c["target"], abi.kernel(abi.KERNEL_RWMH), c["mode"], c["cpu_n1"], c["rounds"],
                       policy=c["policy"], seed=1, workers=workers, max_steps=64)
    dt = time.perf_counter() - t0
    ps = int(np.sum(r["kernel_applications"]))
    return {"psteps": ps, "wall_s": dt, "psteps_per_s": ps / dt, "cores": workers, "n1": c["cpu_n1"]}


def main():
    out = {}
    for name, c in CONFIGS.items():
        out[name] = {"b200_reference_mode": run_gpu(c, abi.RNG_XOSHIRO, abi.PREC_FP64),
                     "b200_philox_fp32": run_gpu(c, abi.RNG_PHILOX, abi.PREC_FP32)}
        try:
            out[name]["cpu_reference"] = run_cpu(c)
        except Exception as exc:
            out[name]["cpu_reference"] = {"unavailable": str(exc)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
