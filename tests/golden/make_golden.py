"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref/libasmc_ref*.so).

Run in the build container (where /root/reference exists and `make -C oracle ref`
has built the reference):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py) and the device
(tests/test_gpu_parity.py) on boxes where the reference sources are absent.
Values are stored as float.hex() strings so every bit survives JSON.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2408_12057_b200 import abi  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def target_spec(name):
    return {"gauss10": ("gaussian_shift", (0.0, 1.0, 1.0), 10),
            "gauss1": ("gaussian_shift", (0.0, 1.0, 1.0), 1),
            "mix5": ("mixture", (2.0, 0.5, -1.0, 0.5, 1.0, 0.5), 5),
            "scale7": ("scale_gaussian", (1.0, 2.0), 7)}[name]


def make_target(name):
    kind, p, d = target_spec(name)
    return getattr(abi, kind)(*p, dim=d)


KERNELS = {"rwmh": abi.kernel(abi.KERNEL_RWMH), "ideal": abi.kernel(abi.KERNEL_IDEALIZED),
           "ident": abi.kernel(abi.KERNEL_IDENTITY)}


def main():
    out = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (unmodified reference)"}
    for rng, tag in ((abi.RNG_XOSHIRO, "xoshiro"), (abi.RNG_PHILOX, "philox")):
        ref = oracle.load("ref", rng)
        g = out.setdefault(tag, {})
        keys = [(42, 3, 17, 5, 1), (0, 0, 0, 0, 0), (7, 1, 123456789, 4, 2), (2024, 0, 0, 0, 0)]
        g["rng"] = [{"key": list(k), "u64": [str(int(v)) for v in ref.rng_u64(k, 64)],
                     "uniform": hexs(ref.rng_uniform(k, 16)), "normal": hexs(ref.rng_normal(k, 33))}
                    for k in keys]
        runs = []
        for tname in ("gauss10", "mix5", "scale7"):
            for kname in ("rwmh", "ideal", "ident"):
                if tname == "mix5" and kname == "ideal":
                    continue
                tg, k = make_target(tname), KERNELS[kname]
                betas = [0.0, 0.1, 0.35, 0.7, 1.0]
                sais = ref.run_sais_single(tg, k, betas, 700, seed=5, round=1)
                rec = {"target": tname, "kernel": kname, "betas": hexs(betas), "n": 700, "seed": 5,
                       "round": 1, "sais": {kk: hexs(sais[kk]) for kk in ("log_g0", "log_g1", "log_g2")},
                       "sais_log_z": float(sais["log_z_hat"]).hex(),
                       "sais_elbo": float(sais["elbo_hat"]).hex()}
                for pol in (abi.POLICY_NEVER, abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS,
                            abi.POLICY_STABILIZED):
                    smc = ref.run_smc(tg, k, betas, 300, policy=pol, rho=0.6, seed=9, round=2)
                    rec[f"smc_{pol}"] = {kk: hexs(smc[kk]) for kk in
                                          ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z")}
                    rec[f"smc_{pol}"]["resample_times"] = smc["resample_times"]
                    rec[f"smc_{pol}"]["log_z"] = float(smc["log_z_hat"]).hex()
                    rec[f"smc_{pol}"]["elbo"] = float(smc["elbo_hat"]).hex()
                x, lw, _ = ref.trajectory(tg, k, betas, 5, 1, 123)
                rec["traj_p123"] = {"x": hexs(x), "lw": hexs(lw)}
                runs.append(rec)
        g["runs"] = runs
        rounds = []
        for mode in (abi.MODE_SAIS, abi.MODE_SSMC):
            r = ref.run_rounds(make_target("gauss1"), KERNELS["rwmh"], mode, 64, 4, seed=11,
                               max_steps=5)
            rounds.append({"mode": mode, "n": [int(v) for v in r["n_particles"]],
                           "steps": [int(v) for v in r["steps"]], "betas": hexs(r["betas"]),
                           "lambda": hexs(r["lambda_"]), "log_z": hexs(r["log_z_hat"])})
        g["rounds"] = rounds
    ref = oracle.load("ref")
    rng = np.random.default_rng(3)
    res = []
    for n in (1, 2, 3, 255, 256, 257, 5000):
        lw = rng.normal(0, 2, n)
        key = (3, 0, 0, 1, abi.POLICY_ALWAYS)
        res.append({"log_w": hexs(lw), "key": list(key),
                    "ancestors": [int(a) for a in ref.systematic_resample(lw, key)]})
    out["systematic"] = res
    sched = []
    cases = [([0.0, 0.7, 1.4, 2.1], [0.0, 0.1, 0.55, 1.0], 3),
             ([0.0, 1.0, 1.5], [0.0, 0.3, 1.0], 1),
             ([0.0, 0.5, 0.5, 1.0], [0.0, 0.3, 0.6, 1.0], 2),
             ([0.0, 0.0, 0.0], [0.0, 0.4, 1.0], 4),
             ([0.0, 1.0, 1.0, 1.0001, 3.0], [0.0, 0.2, 0.21, 0.8, 1.0], 33)]
    knots = 128
    cases.append(([(t / knots) ** 2 for t in range(knots + 1)], [t / knots for t in range(knots + 1)], 16))
    for lam, beta, tn in cases:
        sched.append({"lambda": hexs(lam), "beta": hexs(beta), "t_new": tn,
                      "out": hexs(ref.generate_schedule(lam, beta, tn)),
                      "local": hexs(ref.local_barrier(lam, beta))})
    out["schedule"] = sched
    out["budget"] = [{"args": list(a), "out": list(ref.budget(*a))} for a in
                     [(16, 8, 1, 1 << 40, 0), (16, 8, 1, 1 << 40, 1), (64, 1, 1, 1 << 40, 0),
                      (16, 8, 4, 23 * 4 * 8 - 1, 0), (16, 8, 4, 23 * 4 * 8 - 1, 1),
                      (1 << 24, 1, 1000, 4096 << 20, 1)]]
    path = os.path.join(OUT, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
