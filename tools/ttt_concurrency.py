import sys, time, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import time_to_target as T
from paper_2408_12057_b200 import abi
res = {}
for streams in (1, 16):
    t0 = time.perf_counter()
    lz, wall = T.gpu_runs(range(1, 1001), 6, 1 << 14, abi.RNG_XOSHIRO, abi.PREC_FP64, streams=streams)
    res[streams] = {"wall_all_seeds_s": time.perf_counter() - t0, "mean_round_sum_s": float(wall.sum(1).mean()),
                    "rv_last": T.rel_var(lz[:, 5])}
print(json.dumps(res, indent=1))
