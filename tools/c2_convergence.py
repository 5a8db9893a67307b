import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2408_12057_b200 import abi, capi
tg = abi.scale_gaussian(1.0, 2.0, 1000)
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
for name, k, n1, R in [("hmc0.5", abi.kernel(abi.KERNEL_HMC, (0.5,), 1, 10), 1 << 10, 13),
                       ("hmc0.3", abi.kernel(abi.KERNEL_HMC, (0.3,), 1, 5), 1 << 10, 13),
                       ("ideal", abi.kernel(abi.KERNEL_IDEALIZED), 1 << 10, 13),
                       ("rwmh", abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1), 1 << 10, 19)]:
    t0 = time.perf_counter()
    try:
        r = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, R, seed=1, exec_=abi.execopts(PH, F32))
        print(name, f"{time.perf_counter()-t0:.1f}s", [int(v) for v in r["steps"]], [round(float(v), 3) for v in r["log_z_hat"]], flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True)
