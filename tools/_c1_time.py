import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2408_12057_b200 import abi, capi
tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
for name, ex in (("fp64", abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64, lanes=1)), ("fp32", abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32))):
    for _ in range(5):
        capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 14, 4, seed=1, exec_=ex)
    ts = []
    dev = []
    for i in range(50):
        t0 = time.perf_counter()
        r = capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 14, 4, seed=1 + i, exec_=ex)
        ts.append(time.perf_counter() - t0)
        dev.append(float(np.sum(r["wall_seconds"])))
    print(name, "e2e median ms", 1e3 * np.median(ts), "device ms", 1e3 * np.median(dev))
