"""Config 3's SMC-step passes with the drawn-normal counter: pass time, algorithmic and
drawn normals (early rejection A/B on the mixture); run under ASMC_B200_LIB=... builds."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
capi.run_rounds(tg, k, abi.MODE_SSMC, n1, 6, policy=abi.POLICY_ADAPTIVE_ESS, seed=1, exec_=ex)
capi.profile_enable(True)
r = capi.run_rounds(tg, k, abi.MODE_SSMC, n1, 6, policy=abi.POLICY_ADAPTIVE_ESS, seed=1, exec_=ex)
ms, nrm, drw = capi.profile_collect(drawn=True)
capi.profile_enable(False)
print("launches", len(ms), "pass_ms", float(np.sum(ms)), "alg", float(np.sum(nrm)), "drawn", float(np.sum(drw)),
      "drawn/alg", float(np.sum(drw) / np.sum(nrm)))
q = np.argsort(-ms)[:5]
print("slowest launches ms", [round(float(ms[i]), 3) for i in q], "drawn/alg", [round(float(drw[i] / nrm[i]), 3) for i in q])
