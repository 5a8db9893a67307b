"""Config 5 (relaxed Ising on an L x L torus, HMC) checks and timing.

  --check : device vs the oracle at L = 8 -- identity kernel (V parity) and RWMH
            against the unmodified reference engine + Ising plugin, HMC against the
            restatement; log Z-hat against Kaufman's exact value
  default : throughput at L = 64 (4096 sites) for N particles and T steps:
            particle-steps/s, and site-gradient evaluations per second of the
            move kernel (CUDA events)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi, exact  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--check", action="store_true")
ap.add_argument("--L", type=int, default=64)
ap.add_argument("--K", type=float, default=exact.K_CRITICAL)
ap.add_argument("--N", type=int, default=1 << 16)
ap.add_argument("--T", type=int, default=4)
ap.add_argument("--eps", type=float, default=0.25)
ap.add_argument("--leapfrog", type=int, default=10)
ap.add_argument("--exact-T", type=int, default=0, help="also run T steps and compare log Z-hat with exact")
a = ap.parse_args()
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
ex = abi.execopts(PH, F32)

if a.check:
    import oracle
    out = {}
    L, K = 8, exact.K_CRITICAL
    tg = abi.ising(L, K, 1.0, 1.0)
    betas = np.linspace(0, 1, 9)
    ref = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    rst = oracle.load("restate", PH)
    for kname, k, o in (("identity", abi.kernel(abi.KERNEL_IDENTITY), ref),
                        ("rwmh", abi.kernel(abi.KERNEL_RWMH, (0.1, 0.3), 1), ref),
                        ("hmc", abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=6), rst)):
        r0 = o.run_sais_single(tg, k, betas, 512, seed=2, round=1)
        r1 = capi.run_sais_single(tg, k, betas, 512, seed=2, round=1, exec_=ex)
        out[kname] = {"oracle_log_g1": [float(v) for v in r0["log_g1"][1:]],
                      "dev_log_g1": [float(v) for v in r1["log_g1"][1:]],
                      "oracle_log_z": r0["log_z_hat"], "dev_log_z": r1["log_z_hat"],
                      "max_rel_dlog_g": float(max(np.max(np.abs(r0[g][1:] - r1[g][1:]) / np.abs(r0[g][1:]).clip(1))
                                                  for g in ("log_g0", "log_g1", "log_g2")))}
    k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=8)
    for L in (8, 16):
        tg = abi.ising(L, K, 1.0, 1.0)
        T = 64 if L == 8 else 256
        r = capi.run_sais_single(tg, k, np.linspace(0, 1, T + 1), 1 << 14, seed=3, round=1, exec_=ex)
        out[f"log_z_L{L}"] = {"T": T, "N": 1 << 14, "dev": r["log_z_hat"],
                              "exact": exact.ising_relaxed_log_z(L, K, 1.0)}
    print(json.dumps(out, indent=1))
    sys.exit(0)

tg = abi.ising(a.L, a.K, 1.0, 1.0)
k = abi.kernel(abi.KERNEL_HMC, (a.eps,), 1, leapfrog=a.leapfrog)
betas = np.linspace(0, 1, a.T + 1)
capi.run_sais_single(tg, k, betas, 256, seed=1, round=1, exec_=ex)  # warm-up
capi.profile_enable(True)
t0 = time.perf_counter()
r = capi.run_sais_single(tg, k, betas, a.N, seed=1, round=1, exec_=ex)
wall = time.perf_counter() - t0
ms, sites = capi.profile_collect()
capi.profile_enable(False)
res = {"L": a.L, "K": a.K, "N": a.N, "T": a.T, "eps": a.eps, "leapfrog": a.leapfrog,
       "move_launches": len(ms), "move_ms": [float(v) for v in ms],
       "site_grads_per_s": float(np.sum(sites) / (np.sum(ms) * 1e-3)),
       "wall_s": wall, "psteps_per_s": a.N * a.T / wall, "log_z_hat": r["log_z_hat"],
       "exact_log_z": exact.ising_relaxed_log_z(a.L, a.K, 1.0)}
if a.exact_T:
    betas = np.linspace(0, 1, a.exact_T + 1)
    t0 = time.perf_counter()
    r = capi.run_sais_single(tg, k, betas, a.N, seed=2, round=1, exec_=ex)
    res["exact_run"] = {"T": a.exact_T, "wall_s": time.perf_counter() - t0, "log_z_hat": r["log_z_hat"]}
print(json.dumps(res, indent=1))
