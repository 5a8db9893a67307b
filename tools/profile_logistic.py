"""Config 4 (Bayesian logistic regression, likelihood on tcgen05) checks and timing.

  --check : identity-kernel and RWMH parity against the oracle (the unmodified reference
            engine with the logistic plugin, Philox shadow streams) at a small size
  default : throughput at the config-4 shape (n = 1e5, d = 256) for N particles: the
            likelihood evaluations' CUDA-event time and TFLOP/s (split-bf16 counts 3 MMAs
            per product; algorithmic flops = 2 n d per particle-proposal)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--check", action="store_true")
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--d", type=int, default=256)
ap.add_argument("--N", type=int, default=1 << 17)
ap.add_argument("--T", type=int, default=1)
a = ap.parse_args()
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
ex = abi.execopts(PH, F32)

if a.check:
    import oracle
    ref = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    X, y = abi.logistic_data(3000, 64, 0)
    tg = abi.logistic(X, y, 1.0)
    betas = np.linspace(0, 1, 5)
    out = {}
    for kname, k in (("identity", abi.kernel(abi.KERNEL_IDENTITY)),
                     ("rwmh", abi.kernel(abi.KERNEL_RWMH, (0.01, 0.03, 0.1), 1))):
        r0 = ref.run_sais_single(tg, k, betas, 384, seed=2, round=1)
        r1 = capi.run_sais_single(tg, k, betas, 384, seed=2, round=1, exec_=ex)
        out[kname] = {"ref_log_g1": [float(v) for v in r0["log_g1"][1:]],
                      "dev_log_g1": [float(v) for v in r1["log_g1"][1:]],
                      "ref_log_z": r0["log_z_hat"], "dev_log_z": r1["log_z_hat"],
                      "max_abs_dlog_g": float(max(np.max(np.abs(r0[g][1:] - r1[g][1:]))
                                                  for g in ("log_g0", "log_g1", "log_g2")))}
    print(json.dumps(out, indent=1))
    sys.exit(0)

X, y = abi.logistic_data(a.n, a.d, 0)
tg = abi.logistic(X, y, 1.0)
k = abi.kernel(abi.KERNEL_RWMH, (0.002, 0.005, 0.01), 1)
betas = np.linspace(0, 1, a.T + 1)
capi.run_sais_single(tg, k, betas, 1024, seed=1, round=1, exec_=ex)  # warm-up
capi.profile_enable(True)
t0 = time.perf_counter()
r = capi.run_sais_single(tg, k, betas, a.N, seed=1, round=1, exec_=ex)
wall = time.perf_counter() - t0
ms, flops = capi.profile_collect()
capi.profile_enable(False)
alg = float(np.sum(flops))
print(json.dumps({"n": a.n, "d": a.d, "N": a.N, "T": a.T, "evals": len(ms), "eval_ms": [float(v) for v in ms],
                  "algorithmic_tflops": alg / (np.sum(ms) * 1e-3) / 1e12,
                  "tensor_tflops_issued_split3": 3 * alg / (np.sum(ms) * 1e-3) / 1e12,
                  "wall_s": wall, "psteps_per_s": a.N * a.T / wall, "log_z_hat": r["log_z_hat"]}, indent=1))
