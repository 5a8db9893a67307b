"""Per-step-size pass time of the config-2 RWMH pass (early-rejection check):
one SAIS round, T steps, a single step size per run; CUDA-event time of the pass."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
tg = abi.scale_gaussian(1.0, 2.0, 1000)
betas = np.linspace(0, 1, 6)
N = 1 << 20
out = {}
for s in (0.1, 1.0, 10.0):
    k = abi.kernel(abi.KERNEL_RWMH, (s,), 1)
    capi.run_sais_single(tg, k, betas, 4096, seed=1, round=1, exec_=ex)
    capi.profile_enable(True)
    capi.run_sais_single(tg, k, betas, N, seed=1, round=1, exec_=ex)
    ms, nrm = capi.profile_collect()
    capi.profile_enable(False)
    out[str(s)] = {"pass_ms": float(np.sum(ms)), "normals_alg": float(np.sum(nrm))}
k = abi.kernel(abi.KERNEL_IDENTITY)
capi.profile_enable(True)
capi.run_sais_single(tg, k, betas, N, seed=1, round=1, exec_=ex)
ms, nrm = capi.profile_collect()
capi.profile_enable(False)
out["identity"] = {"pass_ms": float(np.sum(ms))}
print(json.dumps(out, indent=1))
