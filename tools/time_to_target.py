"""Time to a target relative variance of Z-hat, wall clock on both sides (BASELINE
metric, second half; SURVEY 8d "Time-to-target", 8f-1/8f-2).

Definitions (the paper's GPU experiment, and the reference's
replicate loop, experiment.cpp:96-140):
  * an effort level = one sampler run for one seed: SAIS = the doubling round loop
    run to round k (run_sais, drivers.cpp:186-232; the schedule of round k needs rounds
    1..k); ZJA = run_zja (drivers.cpp:234-341) with delta* = (Lambda / T)^2, the paper's
    matching of ZJA's conditional-ESS threshold to T steps;
  * rel-var of a level = Var(Z-hat) / E[Z-hat]^2 over R seeds (exact log Z = 0, so
    Z-hat = exp(log Z-hat));
  * time of a level = WALL-CLOCK seconds of one seed's run (time.perf_counter around the
    public call, host buffers in and out), median over a few seeds; the B200 batched
    figure (asmc_run_sais_seeds: all R seeds in one launch per kernel) is reported
    beside it as wall seconds per seed;
  * time to target = the time of the cheapest level whose rel-var <= target.
CPU: the unmodified reference (oracle/_ref/libasmc_ref_release.so, -O3) on the box's
host cores (workers = nproc), wall clock of the same level for a few seeds.
Process start and JIT are excluded, as in the paper.

  python tools/time_to_target.py [--configs 1,2,3] [--zja] [--seeds 1000]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_12057_b200 import abi  # noqa: E402

XO, PH, F64, F32 = abi.RNG_XOSHIRO, abi.RNG_PHILOX, abi.PREC_FP64, abi.PREC_FP32
RWMH = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)


def rel_var(log_z, c=0.0):
    lz = np.asarray(log_z, float) - c
    m = np.max(lz)
    z = np.exp(lz - m)  # rel-var is scale invariant
    return float(np.var(z, ddof=1) / np.mean(z) ** 2)


def wall(fn, reps):
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        fn(i)
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def cpu_ref():
    import oracle
    return oracle.load("ref_release") if oracle.available("ref_release") else oracle.load("ref", XO)


IDEAL = abi.kernel(abi.KERNEL_IDEALIZED)

CONFIGS = {
    # target, mode, n1, max rounds, exec, seeds batched on the device?, target rel-var, kernel
    "1": dict(name="config1: SAIS d=10 Gaussian shift (log Z = 0), RWMH {0.1,1,10}, N1=2^14",
            target=lambda: abi.gaussian_shift(0.0, 1.0, 1.0, 10), mode=abi.MODE_SAIS, n1=1 << 14, rounds=6,
            ex=lambda: abi.execopts(XO, F64, lanes=1), batched=True, rv=0.05, kernel=RWMH),
    # config 2's RWMH {0.1, 1, 10} cannot follow the annealed scale in d = 1000 within
    # reachable T (log Z-hat ~ -250, seed-dominated: DESIGN.md 3.10); the same target with
    # the reference's idealized kernel gives the schedule-limited time to target
    "2": dict(name="config2: SAIS d=1000 scale-mismatch Gaussian (log Z = 0), RWMH {0.1,1,10}, N1=2^14",
              target=lambda: abi.scale_gaussian(1.0, 2.0, 1000), mode=abi.MODE_SAIS, n1=1 << 14, rounds=8,
              ex=lambda: abi.execopts(PH, F32), batched=False, rv=0.05, kernel=RWMH),
    "2i": dict(name="config2 target, idealized kernel (exact pi_beta draws), N1=2^12",
               target=lambda: abi.scale_gaussian(1.0, 2.0, 1000), mode=abi.MODE_SAIS, n1=1 << 12, rounds=14,
               ex=lambda: abi.execopts(PH, F32), batched=False, rv=0.05, kernel=IDEAL),
    # the same target with HMC (eps 0.3, 5 leapfrog steps): the reference has no HMC, so
    # the CPU side is the oracle's plain-C port (one core), marked kind "port"
    "2h": dict(name="config2 target, HMC eps=0.3 x 5 leapfrog, N1=2^12",
               target=lambda: abi.scale_gaussian(1.0, 2.0, 1000), mode=abi.MODE_SAIS, n1=1 << 12, rounds=15,
               ex=lambda: abi.execopts(PH, F32), batched=False, rv=0.05,
               kernel=abi.kernel(abi.KERNEL_HMC, (0.3,), 1, 5), cpu="port"),
    "3": dict(name="config3: SSMC adaptive-ESS d=100 mixture (log Z = 0), RWMH {0.1,1,10}, N1=2^16",
              target=lambda: abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100), mode=abi.MODE_SSMC, n1=1 << 16,
              rounds=15, ex=lambda: abi.execopts(PH, F32), batched=False, rv=0.05, kernel=RWMH),
}


def sais_levels(cfg, seeds, timing_reps=5):
    """rel-var and per-seed wall time of every round-loop level on the B200."""
    from paper_2408_12057_b200 import capi
    tg, ex, R, K = cfg["target"](), cfg["ex"](), cfg["rounds"], cfg["kernel"]
    out = {"seeds": len(seeds)}
    t0 = time.perf_counter()
    if cfg["batched"]:
        b = capi.run_sais_seeds(tg, K, cfg["n1"], R, seeds, exec_=ex)
        lz = b["log_z_hat"]
        out["batched_wall_s"] = time.perf_counter() - t0
        out["batched_device_s_by_round"] = [float(v) for v in b["wall_seconds"]]
    else:
        lz = np.array([capi.run_rounds(tg, K, cfg["mode"], cfg["n1"], R, seed=int(s), exec_=ex)["log_z_hat"]
                       for s in seeds])
        out["sequential_wall_s"] = time.perf_counter() - t0
    out["rel_var_by_round"] = [rel_var(lz[:, k]) for k in range(R)]
    out["log_z_mean_by_round"] = [float(np.mean(lz[:, k])) for k in range(R)]
    capi.run_rounds(tg, K, cfg["mode"], cfg["n1"], 1, seed=99, exec_=ex)  # warm-up
    out["b200_wall_s_by_round"] = [
        wall(lambda i, k=k: capi.run_rounds(tg, K, cfg["mode"], cfg["n1"], k + 1, seed=int(seeds[i]), exec_=ex),
             timing_reps) for k in range(R)]
    if cfg["batched"]:
        out["b200_batched_wall_s_per_seed_by_round"] = []
        for k in range(R):
            t0 = time.perf_counter()
            capi.run_sais_seeds(tg, K, cfg["n1"], k + 1, seeds, exec_=ex)
            out["b200_batched_wall_s_per_seed_by_round"].append((time.perf_counter() - t0) / len(seeds))
    return out


def first_hit(rv, target):
    for k, v in enumerate(rv):
        if v <= target:
            return k
    return None


def measure_config(c, n_seeds, cpu_reps=3):
    cfg = CONFIGS[c]
    seeds = np.arange(1, n_seeds + 1, dtype=np.uint64)
    res = {"config": cfg["name"], "target_rel_var": cfg["rv"]}
    res.update(sais_levels(cfg, seeds))
    k = first_hit(res["rel_var_by_round"], cfg["rv"])
    res["reached"] = k is not None
    if k is None:
        return res
    workers = os.cpu_count() or 1
    port = cfg.get("cpu") == "port"
    if port:
        import oracle
        ref, workers = oracle.load("restate", PH), 1
    else:
        ref = cpu_ref()
    tg = cfg["target"]()
    # p-steps of the level; a level the CPU cannot run in ~20 s is timed on a scaled-down N1
    # (same rounds, same T plan) and scaled by the p-step ratio (reported as extrapolated):
    # the sample size comes from the CPU rate of a small probe run
    from paper_2408_12057_b200 import capi
    plan_n, plan_t = capi.plan_steps(k + 1, cfg["n1"], tg.dim, 4096 << 20, cfg["mode"])
    ps_full = sum(a * b for a, b in zip(plan_n, plan_t))
    # probe: a few rounds (round 1 alone is overhead-dominated and understates the rate,
    # which would shrink the sample and inflate the extrapolated CPU time)
    n1p, rp = max(64, cfg["n1"] // 64), min(k + 1, 3)
    pn, pt = capi.plan_steps(rp, n1p, tg.dim, 4096 << 20, cfg["mode"])
    t_probe = wall(lambda i: ref.run_rounds(tg, cfg["kernel"], cfg["mode"], n1p, rp, seed=int(seeds[0]),
                                            workers=workers), 1)
    rate = sum(a * b for a, b in zip(pn, pt)) / max(t_probe, 1e-6)
    n1c, rc, reps = cfg["n1"], k + 1, cpu_reps

    def ps_of(n1_, r_):
        a, b = capi.plan_steps(r_, n1_, tg.dim, 4096 << 20, cfg["mode"])
        return sum(x * y for x, y in zip(a, b))

    if ps_full / rate > 20.0:  # scale N1 down, then drop the last rounds if still too long
        n1c, reps = max(256, int(cfg["n1"] * 20.0 * rate / ps_full)), 1
        while rc > 1 and ps_of(n1c, rc) / rate > 30.0:
            rc -= 1
    ps_cpu = ps_of(n1c, rc)
    cpu = wall(lambda i: ref.run_rounds(tg, cfg["kernel"], cfg["mode"], n1c, rc, seed=int(seeds[i]),
                                        workers=workers), reps) * ps_full / ps_cpu
    res["time_to_target"] = {
        "rounds_needed": k + 1, "b200_wall_s": res["b200_wall_s_by_round"][k], "cpu_wall_s": cpu,
        "cpu_cores": workers,
        "cpu_kind": "port (oracle/restate.c, one core: the reference has no HMC)" if port else
                    "reference (unmodified run_sais/run_ssmc, -O3)",
        "cpu_extrapolated": n1c != cfg["n1"] or rc != k + 1, "cpu_sample_n1": n1c, "cpu_sample_rounds": rc,
        "cpu_sample_psteps": ps_cpu, "psteps_full": ps_full,
        "speedup_wall": cpu / res["b200_wall_s_by_round"][k]}
    if cfg["batched"]:
        res["time_to_target"]["b200_batched_wall_s_per_seed"] = res["b200_batched_wall_s_per_seed_by_round"][k]
    return res


def zja_vs_sais(n_seeds_sais=1000, n_seeds_zja=200, target=0.05, Ts=(2, 4, 8, 16, 32), timing_reps=5):
    """The paper's GPU experiment on the config-1 family: 2^14
    particles, SAIS effort = rounds, ZJA effort = T via delta* = (Lambda / T)^2."""
    from paper_2408_12057_b200 import capi
    cfg = CONFIGS["1"]
    tg, n = cfg["target"](), 1 << 14
    ex = abi.execopts(PH, F32, lanes=1)  # both samplers in the throughput mode
    out = {"config": "config1 family (d=10 Gaussian shift), 2^14 particles, philox/fp32", "target_rel_var": target}
    seeds = np.arange(1, n_seeds_sais + 1, dtype=np.uint64)
    b = capi.run_sais_seeds(tg, RWMH, n, 6, seeds, exec_=ex)
    lam = float(np.mean(b["lambda_total"][:, -1]))
    out["lambda_hat"] = lam
    rv_s = [rel_var(b["log_z_hat"][:, k]) for k in range(6)]
    capi.run_rounds(tg, RWMH, abi.MODE_SAIS, n, 1, seed=99, exec_=ex)
    t_s = [wall(lambda i, k=k: capi.run_rounds(tg, RWMH, abi.MODE_SAIS, n, k + 1, seed=int(seeds[i]), exec_=ex),
                timing_reps) for k in range(6)]
    out["sais"] = {"rel_var_by_round": rv_s, "wall_s_by_round": t_s}
    zs = {"T": list(Ts), "delta_star": [], "rel_var": [], "wall_s": [], "steps_mean": []}
    capi.run_zja(tg, RWMH, n, delta_star=(lam / 4) ** 2, seed=99, exec_=ex)
    for T in Ts:
        ds = (lam / T) ** 2
        lz, steps = [], []
        for s in range(1, n_seeds_zja + 1):
            z = capi.run_zja(tg, RWMH, n, delta_star=ds, seed=s, exec_=ex)
            lz.append(z["rounds"][-1]["log_z_hat"])
            steps.append(z["steps"])
        zs["delta_star"].append(ds)
        zs["rel_var"].append(rel_var(lz))
        zs["steps_mean"].append(float(np.mean(steps)))
        zs["wall_s"].append(wall(lambda i, ds=ds: capi.run_zja(tg, RWMH, n, delta_star=ds, seed=int(i + 1), exec_=ex),
                                 timing_reps))
    out["zja"] = zs
    ks, kz = first_hit(rv_s, target), first_hit(zs["rel_var"], target)
    out["sais_time_to_target_s"] = t_s[ks] if ks is not None else None
    out["zja_time_to_target_s"] = zs["wall_s"][kz] if kz is not None else None
    if ks is not None and kz is not None:
        out["zja_over_sais"] = out["zja_time_to_target_s"] / out["sais_time_to_target_s"]
        # the same two effort levels on the host CPU (reference Philox build: same streams)
        import oracle
        ref = oracle.load("ref", PH) if oracle.available("ref", PH) else None
        if ref is not None:
            workers = os.cpu_count() or 1
            cs = wall(lambda i: ref.run_rounds(tg, RWMH, abi.MODE_SAIS, n, ks + 1, seed=i + 1, workers=workers), 3)
            cz = wall(lambda i: ref.run_zja(tg, RWMH, n, delta_star=zs["delta_star"][kz], seed=i + 1,
                                            workers=workers), 3)
            out["cpu"] = {"cores": workers, "sais_wall_s": cs, "zja_wall_s": cz, "zja_over_sais": cz / cs,
                          "kind": "reference Philox build (oracle/_ref/libasmc_ref_philox.so, -O2)"}
    return out


def measure(n_seeds=1000):
    """bench.py's time_to_target field: config 1 (batched seeds, wall clock both sides)."""
    return measure_config("1", n_seeds)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,2i,2h,3")
    ap.add_argument("--seeds", type=int, default=1000)
    ap.add_argument("--seeds-slow", type=int, default=32, help="seeds for the configs run one seed at a time")
    ap.add_argument("--zja", action="store_true")
    a = ap.parse_args()
    res = {}
    for c in [v for v in a.configs.split(",") if v]:
        res[f"config{c}"] = measure_config(c, a.seeds if CONFIGS[c]["batched"] else a.seeds_slow)
        print(json.dumps({f"config{c}": res[f"config{c}"]}), flush=True)
    if a.zja:
        res["zja_vs_sais"] = zja_vs_sais()
        print(json.dumps({"zja_vs_sais": res["zja_vs_sais"]}), flush=True)


if __name__ == "__main__":
    main()
