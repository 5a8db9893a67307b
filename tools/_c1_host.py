import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2408_12057_b200 import abi, capi
L = capi.lib()
orig = L.asmc_run_rounds
acc = []
class W:
    def __init__(self, f): self.f = f; self.argtypes = f.argtypes; self.restype = f.restype
    def __call__(self, *a):
        t0 = time.perf_counter(); r = self.f(*a); acc.append(time.perf_counter() - t0); return r
L.asmc_run_rounds = W(orig)
tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
ex = abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64, lanes=1)
for _ in range(5): capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 14, 4, seed=1, exec_=ex)
acc.clear(); ts=[]; dev=[]
for i in range(50):
    t0 = time.perf_counter(); r = capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 14, 4, seed=1+i, exec_=ex); ts.append(time.perf_counter()-t0)
    dev.append(float(np.sum(r["wall_seconds"])))
print("e2e", 1e3*np.median(ts), "C call", 1e3*np.median(acc), "device", 1e3*np.median(dev))
