"""ZJA (online adaptation, paper Sec. on the GPU comparison) vs SAIS rounds on one B200.

For a target and particle count: device time of run_zja (pilot + adaptive run, K
target steps) and of the SAIS round loop reaching a comparable final resolution,
with the ZJA per-step cost split into the next-beta search (probes) and the step
pass (asmc profiling events cover only the pass launches).  CPU reference for both
on a bounded sample.  Output JSON -> profiles/.
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
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--K", type=int, default=32)
ap.add_argument("--dim", type=int, default=10)
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--cpu-n", type=int, default=4096)
a = ap.parse_args()
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
ex = abi.execopts(PH, F32)
tg = abi.gaussian_shift(0.0, 1.0, 1.0, a.dim)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
capi.run_zja(tg, k, 4096, target_steps=4, seed=9, exec_=ex)  # warm-up
capi.run_rounds(tg, k, abi.MODE_SAIS, 4096, 2, seed=9, exec_=ex)
capi.profile_enable(True)
t0 = time.perf_counter()
z = capi.run_zja(tg, k, a.n, target_steps=a.K, seed=1, exec_=ex)
zwall = time.perf_counter() - t0
ms, _ = capi.profile_collect()
capi.profile_enable(False)
main = z["rounds"][-1]
psteps_zja = sum(r["kernel_applications"] for r in z["rounds"])
t0 = time.perf_counter()
s = capi.run_rounds(tg, k, abi.MODE_SAIS, a.n // 8, a.rounds, seed=1, exec_=ex)
swall = time.perf_counter() - t0
res = {"target": f"gaussian_shift d={a.dim} z=1", "kernel": "rwmh [0.1,1,10]", "mode": "philox/fp32",
       "zja": {"n": a.n, "K": a.K, "delta_star": z["delta_star"], "steps": z["steps"], "wall_s": zwall,
               "pass_ms_total": float(np.sum(ms)), "psteps": int(psteps_zja),
               "search_and_overhead_s": zwall - float(np.sum(ms)) * 1e-3,
               "log_z_hat": main["log_z_hat"], "final_lambda": float(main["lambda_"][-1])},
       "sais_rounds": {"n1": a.n // 8, "rounds": a.rounds, "steps": [int(v) for v in s["steps"]],
                       "n": [int(v) for v in s["n_particles"]], "wall_s": swall,
                       "device_s": float(np.sum(s["wall_seconds"])),
                       "psteps": int(np.sum(s["kernel_applications"])),
                       "log_z_hat": [float(v) for v in s["log_z_hat"]]}}
try:
    import oracle
    o = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    t0 = time.perf_counter()
    zc = o.run_zja(tg, k, a.cpu_n, target_steps=a.K, seed=1, workers=os.cpu_count() or 1)
    res["cpu_reference_zja"] = {"n": a.cpu_n, "wall_s": time.perf_counter() - t0, "steps": zc["steps"],
                                "psteps": int(sum(r["kernel_applications"] for r in zc["rounds"])),
                                "cores": os.cpu_count()}
except Exception as e:  # noqa: BLE001
    res["cpu_reference_zja"] = {"unavailable": str(e)}
print(json.dumps(res, indent=1))
