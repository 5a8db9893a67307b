"""Config 1 (SAIS, d=10 Gaussian shift, N1=2^14, 4 doubling rounds) in both arithmetic
modes, as time_to_target runs it: one warm-up and one timed call each (for launch lists)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
for name, ex in (("reference", abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64)),
                 ("philox_fp32", abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32))):
    for _ in range(2):
        t0 = time.perf_counter()
        r = capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 14, 4, seed=1, exec_=ex)
        wall = time.perf_counter() - t0
    print(name, "wall_s", wall, "round wall_s", [float(v) for v in r["wall_seconds"]],
          "log_z_hat", [float(v) for v in r["log_z_hat"]])
