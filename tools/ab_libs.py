"""A/B timing of several builds of libasmc_b200.so on one box (same GPU, interleaved runs).

  python tools/ab_libs.py base=ab/libasmc_base.so new=paper_2408_12057_b200/libasmc_b200.so \
      [--reps 2] [--what bench|config3|logistic|ising]

Each build is loaded through ASMC_B200_LIB (capi.py) in a fresh process; runs alternate
between builds so clock or thermal drift hits all of them alike.  Prints one line per run
(build, metric value, and the estimate so bit-identity can be checked by eye).  Used for
every kept/rejected micro-optimisation recorded in DESIGN.md.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CMDS = {
    "bench": [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-ttt",
              "--no-configs"],
    "config3": [sys.executable, "tools/profile_config3.py"],
    "logistic": [sys.executable, "tools/profile_logistic.py", "--N", "1048576", "--T", "1"],
    "ising": [sys.executable, "tools/profile_ising.py", "--N", "262144", "--T", "2"],
}


def parse(what, out):
    if what == "bench":
        d = json.loads(out.strip().splitlines()[-1])
        return d["value"], d["last_log_z_hat"][-1]
    if what == "config3":
        f = out.split()
        return float(f[f.index("psteps/s(wall)") + 1]), out.split("log_z_hat")[1].strip()[:40]
    d = json.loads(out[out.index("{"):])
    key = {"logistic": "algorithmic_tflops", "ising": "site_grads_per_s"}[what]
    return d[key], d.get("log_z_hat")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("builds", nargs="+", help="name=path/to/libasmc_b200.so")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--what", default="bench", choices=sorted(CMDS))
    a = ap.parse_args()
    builds = [b.split("=", 1) for b in a.builds]
    for _ in range(a.reps):
        for name, path in builds:
            env = dict(os.environ, ASMC_B200_LIB=os.path.abspath(path))
            r = subprocess.run(CMDS[a.what], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
            if r.returncode != 0:
                print(name, "FAILED", r.stderr[-300:], flush=True)
                continue
            value, est = parse(a.what, r.stdout)
            print(f"{name:12s} {value:.6g}  estimate {est}", flush=True)


if __name__ == "__main__":
    main()
