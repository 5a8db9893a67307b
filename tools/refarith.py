"""Config 2 shape in reference arithmetic (fp64 / keyed xoshiro, one lane per particle):
p-steps/s over a 4-round run at N1 = 2^16 (bench.py's reference_arithmetic), 3 reps."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi  # noqa: E402

tg = abi.scale_gaussian(1.0, 2.0, 1000)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
ex = abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64)
capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 10, 2, seed=1, exec_=ex)
for _ in range(3):
    r = capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 16, 4, seed=1, exec_=ex)
    print("p-steps/s", float(np.sum(r["kernel_applications"])) / float(np.sum(r["wall_seconds"])),
          "log_z_hat", [float(v) for v in r["log_z_hat"]])
