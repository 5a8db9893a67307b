"""Config 3 exactly as bench.py runs it (SSMC adaptive ESS, d=100 mixture, N1=2^22, 6 rounds):
one warm-up, one timed run; used for the ncu launch list of the SSMC step loop."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

n1 = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
for _ in range(2):
    r = capi.run_rounds(tg, k, abi.MODE_SSMC, n1, 6, policy=abi.POLICY_ADAPTIVE_ESS, seed=1, exec_=ex)
ps = float(np.sum(r["kernel_applications"]))
print("psteps", ps, "wall", float(np.sum(r["wall_seconds"])), "psteps/s(wall)", ps / float(np.sum(r["wall_seconds"])),
      "events", int(np.sum(r["resampled"])), "log_z_hat", [float(v) for v in r["log_z_hat"]])
