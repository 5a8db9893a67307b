import json, time, numpy as np, sys
sys.path.insert(0, "/root/repo")
from paper_2408_12057_b200 import abi, capi, exact
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
tg = abi.ising(64, exact.K_CRITICAL, 1.0, 1.0)
k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=10)
for n1, rounds in ((1 << 13, 10), (1 << 12, 12)):
    t0 = time.perf_counter()
    r = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, rounds, seed=1, exec_=ex)
    dt = time.perf_counter() - t0
    print(json.dumps({"n1": n1, "rounds": rounds, "wall_s": dt, "N": [int(v) for v in r["n_particles"]],
                      "T": [int(v) for v in r["steps"]],
                      "Lambda": [float(r["lambda_"][i][r["steps"][i]]) for i in range(rounds)],
                      "log_z_hat": [float(v) for v in r["log_z_hat"]],
                      "psteps": int(np.sum(r["kernel_applications"])),
                      "exact": exact.ising_relaxed_log_z(64, exact.K_CRITICAL, 1.0)}))
