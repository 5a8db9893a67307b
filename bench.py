#!/usr/bin/env python
"""Benchmark: SAIS throughput on BASELINE.json config 2 (particle-steps/s).

Workload (BASELINE.json configs[1]): SAIS round loop (run_sais, 4 doubling
rounds) on the d = 1000 scale-mismatch Gaussian N(0, I) -> N(0, 2^2 I), RWMH
cycle {0.1, 1, 10} x 1 sweep, N_1 = 2^24 particles per GPU (weak scaling),
Philox4x32-10 streams, fp32 positions / fp64 weights and accumulators.
One bench "step" = one full run_sais call (4 rounds, 4.0e8 particle-steps per
GPU): every round's fused particle pass, folds, barrier estimate and schedule
regeneration.  Synthetic: the only inputs are the target/kernel parameters.

  python bench.py [--gpus N --steps K --warmup W]          our B200 path
  python bench.py --impl reference [...]                    the reference CPU path
  torchrun --nproc-per-node N bench.py --gpus N             one rank per GPU

Prints one JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2408_12057_b200 import abi  # noqa: E402

D = 1000
SIGMA0, SIGMA1 = 1.0, 2.0
STEPS = (0.1, 1.0, 10.0)
ROUNDS = 4
N1_PER_GPU = 1 << 24
SEED = 1
METRIC = "particle-steps/sec"


def workload(n1, dim=D, rounds=ROUNDS):
    return {"workload": f"config2: SAIS d={dim} scale-mismatch Gaussian N(0,{SIGMA0}^2 I)->N(0,{SIGMA1}^2 I), "
                        f"RWMH {list(STEPS)}x1, {rounds} doubling rounds (run_sais)",
            "n_particles_round1": n1, "dim": dim, "rounds": rounds,
            "kernel": "rwmh_cycle", "step_sizes": list(STEPS), "sweeps": 1}


def plan(n1, rounds, dim):
    ns, ts = [n1], [1]
    for _ in range(1, rounds):
        ns.append(int(math.ceil(math.sqrt(2.0) * ns[-1])))
        ts.append(int(math.ceil(math.sqrt(2.0) * ts[-1])))
    return ns, ts


def psteps(n1, rounds, dim):
    ns, ts = plan(n1, rounds, dim)
    return sum(n * t for n, t in zip(ns, ts))


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                try:
                    rows.append((float(f[1]), float(f[2]), f[5:9]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        active = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": rows[0][1],
                "reasons": active, "samples": len(rows)}


# -------------------------------------------------------- reference (CPU) --
def host_cpu():
    """nproc and the lscpu model of the box's host."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "model": model}


def cpu_reference_run(n1, dim, rounds, workers):
    """The unmodified reference run_sais (oracle/_ref/libasmc_ref_release.so: the
    reference's sources at its own Release flags, -O3 -DNDEBUG) on the host cores."""
    import oracle
    ref = oracle.load("ref_release")
    tg = abi.scale_gaussian(SIGMA0, SIGMA1, dim)
    k = abi.kernel(abi.KERNEL_RWMH, STEPS, 1)
    t0 = time.perf_counter()
    out = ref.run_rounds(tg, k, abi.MODE_SAIS, n1, rounds, seed=SEED, workers=workers)
    dt = time.perf_counter() - t0
    ka = int(np.sum(out["kernel_applications"]))
    return ka, dt


def cpu_sample(budget_s, dim, rounds, workers, window=None, tries=4):
    """Size N_1 (a multiple of 256) so one 4-round run takes budget_s of wall time: start
    from a 4096-particle run and rescale from each real sample (p-steps are linear in N_1)
    until the sample lands inside `window`.  Returns (n1, kernel_applications, seconds,
    inside_window)."""
    if window is None:  # 10-30 s of CPU work (wider only for a budget outside it)
        window = (min(10.0, 0.8 * budget_s), max(30.0, 1.5 * budget_s))
    n1 = 4096
    ka, dt = cpu_reference_run(n1, dim, rounds, workers)
    for _ in range(tries):
        if window[0] <= dt <= window[1]:
            break
        n1 = max(256, int(n1 * budget_s / max(dt, 1e-3)) // 256 * 256)
        ka, dt = cpu_reference_run(n1, dim, rounds, workers)
    return n1, ka, dt, window[0] <= dt <= window[1]


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    workers = os.cpu_count() or 1
    n1, _, _, _ = cpu_sample(args.cpu_budget, args.dim, ROUNDS, workers)
    for _ in range(args.warmup):
        cpu_reference_run(n1 // 4 or 1, args.dim, ROUNDS, workers)
    tot_ka, tot_dt, dts = 0, 0.0, []
    for _ in range(args.steps):
        ka, dt = cpu_reference_run(n1, args.dim, ROUNDS, workers)
        tot_ka += ka
        tot_dt += dt
        dts.append(round(dt, 2))
    value = tot_ka / tot_dt
    sample = (f"unmodified reference run_sais (Release -O3) with N_1={n1} (same d={args.dim}, {ROUNDS} rounds, "
              f"RWMH {list(STEPS)}), workers={workers}; per-step seconds {dts}")
    line = {"metric": METRIC, "value": value, "unit": "particle-steps/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload(n1, args.dim), note="reference CPU path, bounded sample of the workload"),
            "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": workers,
                             "kind": "reference", "sample": sample, "host": host_cpu(),
                             "build": "oracle/_ref/libasmc_ref_release.so (-O3 -DNDEBUG -std=gnu++20)"},
            "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    mapped = repo_objects_mapped()
    if mapped:  # the reference arm must run none of this repo's native code
        raise RuntimeError(f"reference arm mapped the repo's own libraries: {mapped}")
    print(json.dumps(line), flush=True)
    return 0


def repo_objects_mapped():
    """Shared objects of this package mapped into the process (Linux /proc/self/maps)."""
    pkg = os.path.join(ROOT, "paper_2408_12057_b200")
    try:
        maps = open("/proc/self/maps").read().splitlines()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps if ln.split() and ln.split()[-1].startswith(pkg)})


# ------------------------------------------------------------- our path --
def load_profile_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_pass_traffic.json")
    if os.path.exists(path):
        try:
            return json.load(open(path))
        except ValueError:
            return None
    return None


def load_profile_issue():
    """Issue-slot utilisation of the bench's own pass launch from its ncu capture
    (profiles/r1_bench_pass_ncu_full.json): the pass is ALU/SFU-issue bound, so this
    is its hardware roofline fraction beside the generator-peak one."""
    path = os.path.join(ROOT, "profiles", "r2_bench_pass_ncu_full.json")
    try:
        d = json.load(open(path))[0]
        pk = json.load(open(os.path.join(ROOT, "profiles", "r2_peak_ncu_full.json")))[0]
    except (OSError, ValueError, IndexError, KeyError):
        return None
    def pct(key):
        v = d.get(key)
        return None if v is None else round(float(str(v).split()[0]) / 100.0, 4)
    return {"issue_active": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "alu_pipe": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "xu_pipe": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "peak_kernel_issue_active": round(float(pk["smsp__issue_active.avg.pct_of_peak_sustained_active"].split()[0])
                                              / 100.0, 4),
            "note": "the generator microbenchmark itself issues on 66 % of cycles (math-pipe throttle: Philox's "
                    "IMAD.WIDE on the heavy FMA pipe), so the pass's issue share already exceeds its peak's",
            "source": "profiles/r2_bench_pass_ncu_full.json, r2_peak_ncu_full.json (ncu --set full of bench.py's "
                      "round-1 pass launch and of its generator-peak launch)"}


def other_cpu_baselines():
    """The reference's CPU path beside configs 3-5, on bounded samples of each workload
    (same targets, kernels and rounds, smaller N): config 3 and 4 through the unmodified
    reference engine (oracle/_ref, all host cores), config 5's HMC through the oracle port
    (the reference has no HMC; one core)."""
    import oracle
    from paper_2408_12057_b200 import exact
    workers = os.cpu_count() or 1
    out = {}
    ref = oracle.load("ref_release") if oracle.available("ref_release") else None
    if ref is not None:
        tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)
        t0 = time.perf_counter()
        r = ref.run_rounds(tg, abi.kernel(abi.KERNEL_RWMH, STEPS, 1), abi.MODE_SSMC, 4096, 6,
                           policy=abi.POLICY_ADAPTIVE_ESS, seed=SEED, workers=workers)
        dt = time.perf_counter() - t0
        ka = float(np.sum(r["kernel_applications"]))
        out["config3"] = {"value": ka / dt, "unit": "particle-steps/s", "cores": workers, "kind": "reference",
                          "sample": f"run_ssmc N1=4096, 6 rounds, {dt:.1f}s"}
        X, y = abi.logistic_data(100000, 256, 0)
        tg = abi.logistic(X, y, 1.0)
        refp = oracle.load("ref", abi.RNG_PHILOX)
        t0 = time.perf_counter()
        refp.run_sais_single(tg, abi.kernel(abi.KERNEL_RWMH, (0.002, 0.005, 0.01), 1), [0.0, 1.0], 32, seed=SEED,
                             round=1, workers=workers)
        dt = time.perf_counter() - t0
        out["config4"] = {"value": 32 / dt, "unit": "particle-steps/s", "cores": workers, "kind": "reference",
                          "sample": f"run_sais_single with the logistic plugin, N=32, T=1, {dt:.1f}s"}
    rs = oracle.load("restate", abi.RNG_PHILOX)
    tg = abi.ising(64, exact.K_CRITICAL, 1.0, 1.0)
    t0 = time.perf_counter()
    rs.run_sais_single(tg, abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=10), [0.0, 0.5, 1.0], 16, seed=SEED,
                       round=1)
    dt = time.perf_counter() - t0
    out["config5"] = {"value": 32 / dt, "unit": "particle-steps/s", "cores": 1, "kind": "port",
                      "sample": f"oracle restatement (HMC: no reference kernel), N=16, T=2, {dt:.1f}s"}
    return out


def reference_arithmetic(stream, n1=1 << 16):
    """Config 2 in the device's reference mode (keyed xoshiro streams, fp64, one lane per
    particle, the reference's operation order): the cost of the reference's own
    arithmetic on the B200, beside the fp32/Philox headline (bounded N1)."""
    import torch
    from paper_2408_12057_b200 import capi
    tg = abi.scale_gaussian(SIGMA0, SIGMA1, D)
    k = abi.kernel(abi.KERNEL_RWMH, STEPS, 1)
    ex64 = abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64, stream=stream.cuda_stream)
    capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 10, 2, seed=SEED, exec_=ex64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    r = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, ROUNDS, seed=SEED, exec_=ex64)
    e1.record(stream)
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3
    ps = float(np.sum(r["kernel_applications"]))
    return {"workload": f"config2 shape (d={D}, 4 rounds) with N1={n1}", "rng": "keyed xoshiro256++",
            "precision": "fp64, reference operation order", "value": ps / dt, "unit": "particle-steps/s",
            "device_s": dt, "psteps": ps}


ISSUE_PEAK = 148 * 4 * 32 * 1.965e9  # thread-instructions/s at the max SM clock


def other_configs(stream, ex, peak_normals, peaks):
    """BASELINE.json configs 3-5 on this GPU (single-GPU shapes), device time by CUDA
    events on the library's stream; inputs resident, one warm-up each.  Each carries the
    roofline of its dominant kernel and an e2e wall-clock figure through the
    public call (host buffers in and out)."""
    import torch
    from paper_2408_12057_b200 import capi, exact
    out = {}

    def timed(fn, prof=False):
        fn()  # warm-up (JIT-free, but first-touch of pools / data upload)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if prof:
            capi.profile_enable(True)
        t0 = time.perf_counter()
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        pr = None
        if prof:
            pr = capi.profile_collect(drawn=True)  # (ms, algorithmic units, drawn normals) per launch
            capi.profile_enable(False)
        return r, e0.elapsed_time(e1) * 1e-3, wall, pr

    # config 3: SSMC, adaptive ESS, d=100 bimodal mixture, N=2^22, 6 rounds
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)
    k = abi.kernel(abi.KERNEL_RWMH, STEPS, 1)
    r, dt, wall, (pms, pnorm, pdrawn) = timed(lambda: capi.run_rounds(tg, k, abi.MODE_SSMC, 1 << 22, 6,
                                                                     policy=abi.POLICY_ADAPTIVE_ESS, seed=SEED,
                                                                     exec_=ex), prof=True)
    ps = float(np.sum(r["kernel_applications"]))
    pass_s = float(np.sum(pms)) * 1e-3
    ach = float(np.sum(pnorm)) / pass_s
    out["config3"] = {"workload": "SSMC adaptive-ESS (rho 0.5) d=100 mixture, N1=2^22, 6 rounds, RWMH [0.1,1,10]",
                      "psteps": ps, "device_s": dt, "value": ps / dt, "unit": "particle-steps/s",
                      "e2e": {"value": ps / wall, "unit": "particle-steps/s", "wall_s": wall,
                              "path": "C-ABI asmc_run_rounds (run_ssmc), host outputs"},
                      "roofline": {"bound": "issue", "kernel": "pass_smem_kernel<TgtMixture, 4> (SMC step mode)",
                                   "achieved": ach / 1e9, "peak": peak_normals / 1e9, "unit": "Gnormal/s",
                                   "frac": ach / peak_normals, "pass_share_of_device_time": pass_s / dt,
                                   "algorithmic_units": "normals = N*d per init + N*S*d per step (the RWMH "
                                                        "algorithm's draws)",
                                   "drawn": {"fraction_of_algorithmic": float(np.sum(pdrawn)) / float(np.sum(pnorm)),
                                             "frac": float(np.sum(pdrawn)) / pass_s / peak_normals,
                                             "note": "normals generated: the s = 10 proposals are early-rejected "
                                                     "after their first quad-iteration (TgtMixture::early_worth)"},
                                   "hbm": {"bytes_per_pstep": 8 * 100 + 16,
                                           "achieved_gbs": ps * (8 * 100 + 16) / pass_s / 1e9,
                                           "peak": peaks.get("hbm_gbs"),
                                           "frac": ps * (8 * 100 + 16) / pass_s / 1e9 / peaks.get("hbm_gbs", 6543.1),
                                           "note": "step mode loads and stores each fp32 row (8d) and log-w (16 B)"}},
                      "resampling_events": int(np.sum(r["resampled"])),
                      "last_log_z_hat": float(r["log_z_hat"][-1]), "exact_log_z": 0.0}
    # config 4: SAIS Bayesian logistic regression, X 1e5 x 256, N=2^20 (tensor cores)
    X, y = abi.logistic_data(100000, 256, 0)
    tg = abi.logistic(X, y, 1.0)
    k = abi.kernel(abi.KERNEL_RWMH, (0.002, 0.005, 0.01), 1)
    betas = np.linspace(0.0, 1.0, 5)
    r, dt, wall, (ms, flops, _) = timed(lambda: capi.run_sais_single(tg, k, betas, 1 << 20, seed=SEED, round=1,
                                                                   exec_=ex), prof=True)
    ev_ms, ev_flops = float(np.sum(ms)), float(np.sum(flops))
    alg_tf = ev_flops / (ev_ms * 1e-3) / 1e12
    sus = peaks.get("bf16_tflops_sustained", 1398.3)
    out["config4"] = {"workload": "SAIS logistic regression n=1e5 d=256 (general fp32 X), N=2^20, T=4, RWMH x3 "
                                  "(split-bf16 tcgen05)",
                      "psteps": float((1 << 20) * 4), "device_s": dt, "value": (1 << 20) * 4 / dt,
                      "unit": "particle-steps/s",
                      "e2e": {"value": (1 << 20) * 4 / wall, "unit": "particle-steps/s", "wall_s": wall,
                              "path": "C-ABI asmc_run_sais_single, host X/y in, host report out"},
                      "roofline": {"bound": "tensor", "kernel": "lg_eval_kernel (tcgen05.mma cta_group::2)",
                                   "achieved": alg_tf, "peak": sus, "unit": "TFLOP/s", "frac": alg_tf / sus,
                                   "issued_tflops": 3 * alg_tf, "issued_frac": 3 * alg_tf / sus,
                                   "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside "
                                                  "a long step)",
                                   "algorithmic_units": "2 n d flop per particle-proposal (X theta'); the 3-MMA "
                                                        "split-bf16 scheme issues 3x",
                                   "likelihood_share_of_device_time": ev_ms * 1e-3 / dt}}
    # config 5: SAIS relaxed Ising 64x64 at K_c, HMC, schedule adaptation over 12 doubling
    # rounds ending at N = 2^18 (N1 = 5793: the budget rule's sqrt(2) growth)
    tg = abi.ising(64, exact.K_CRITICAL, 1.0, 1.0)
    k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=10)
    r, dt, wall, _ = timed(lambda: capi.run_rounds(tg, k, abi.MODE_SAIS, 5793, 12, seed=SEED, exec_=ex))
    ps = float(np.sum(r["kernel_applications"]))
    steps = [int(v) for v in r["steps"]]
    sg = ps * 11 * 4096 / dt
    out["config5"] = {"workload": "SAIS relaxed Ising 64x64 K=K_c, HMC eps 0.25 x 10 leapfrog, 12 adaptive rounds, "
                                  "N 5793 -> 2^18, T 1 -> 104",
                      "psteps": ps, "device_s": dt, "value": ps / dt, "unit": "particle-steps/s",
                      "site_gradients_per_s": sg,
                      "e2e": {"value": ps / wall, "unit": "particle-steps/s", "wall_s": wall,
                              "path": "C-ABI asmc_run_rounds (run_sais), host outputs"},
                      "roofline": {"bound": "issue", "kernel": "is_tile_kernel<64> (HMC leapfrog, 4x4 tiles)",
                                   "achieved": sg / 1e12, "peak": ISSUE_PEAK / 20 / 1e12,
                                   "unit": "Tsite-gradient/s", "frac": sg / (ISSUE_PEAK / 20),
                                   "peak_source": "derived: 148 SMs x 4 schedulers x 32 lanes x 1.965 GHz over "
                                                  "the 20 thread-instructions of one site-gradient (leapfrog loop "
                                                  "SASS, DESIGN.md 3.7); achieved over the whole device time"},
                      "n_final": int(r["n_particles"][-1]), "T": steps,
                      "lambda_hat": [float(r["lambda_"][i][steps[i]]) for i in range(len(steps))],
                      "log_z_hat": [float(v) for v in r["log_z_hat"]],
                      "exact_log_z": exact.ising_relaxed_log_z(64, exact.K_CRITICAL, 1.0)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n1", type=int, default=N1_PER_GPU, help="round-1 particles per GPU")
    ap.add_argument("--dim", type=int, default=D)
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds per CPU sample (10-30 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-target measurement")
    ap.add_argument("--ttt-seeds", type=int, default=1000)
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 3-5 measurements")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional multi-rank check on one GPU (CPU collectives; not for timing)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU chunk-partial round loop even at one rank")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    from paper_2408_12057_b200 import capi, distributed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo" and "ASMC_BENCH_DEVICE" in os.environ:  # functional check on one GPU
        local = int(os.environ["ASMC_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the NCCL INIT lines show the ranks and transports
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    # a non-default stream, current for torch and passed to the library: the library
    # enqueues on it (asmc_exec.stream), so the CUDA events below bracket its kernels
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, device=local, stream=stream.cuda_stream)
    tg = abi.scale_gaussian(SIGMA0, SIGMA1, args.dim)
    kern = abi.kernel(abi.KERNEL_RWMH, STEPS, 1)
    n1 = args.n1 * world
    total_psteps = psteps(n1, ROUNDS, args.dim)

    def one_step():
        if world == 1 and not args.sharded:
            return capi.run_rounds(tg, kern, abi.MODE_SAIS, n1, ROUNDS, seed=SEED, exec_=ex)
        return distributed.run_sais(tg, kern, n1, ROUNDS, SEED, ex, rank, world,
                                    device="cpu" if args.dist_backend == "gloo" else None)

    # generator peak (same Philox + fp32 Box-Muller code path, registers only)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak_blocks = sms * 8
    quads = 1 << 14
    peak_s = capi.peak_normals(local, peak_blocks, quads)
    peak_normals = peak_blocks * 256 * quads * 4 / peak_s

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    dev_ms, wall_s = 0.0, 0.0
    prof_ms, prof_normals, prof_drawn = [], [], []
    last = None
    capi.launch_count(reset=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between timed iterations (outside the events)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            capi.profile_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            last = one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            wall_s += time.perf_counter() - t0
            dev_ms += e0.elapsed_time(e1)
            ms, nrm, drw = capi.profile_collect(drawn=True)
            capi.profile_enable(False)
            prof_ms += list(ms)
            prof_normals += list(nrm)
            prof_drawn += list(drw)
    launches = capi.launch_count(reset=True)
    if world > 1:
        t = torch.tensor([dev_ms, wall_s], device="cuda" if args.dist_backend == "nccl" else "cpu",
                         dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms, wall_s = float(t[0]), float(t[1])
    clocks = clk.summary()

    value = total_psteps * args.steps / (dev_ms * 1e-3)
    e2e = total_psteps * args.steps / wall_s
    # roofline of the dominant kernel (the fused particle pass)
    pass_ms = float(np.sum(prof_ms)) if prof_ms else float("nan")
    pass_normals = float(np.sum(prof_normals)) if prof_normals else float("nan")
    pass_drawn = float(np.sum(prof_drawn)) if prof_drawn else float("nan")
    achieved = pass_normals / (pass_ms * 1e-3)
    drawn_rate = pass_drawn / (pass_ms * 1e-3)
    # step-outer HBM bytes the pass would move if state lived in HBM (8d + 16 B / p-step)
    hbm_alg = (8 * args.dim + 16) * total_psteps / world * args.steps / (pass_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic = load_profile_traffic()
    h2d, d2h = distributed.io_bytes(plan(n1, ROUNDS, args.dim)[1])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            workers = os.cpu_count() or 1
            nc, ka, dt, inside = cpu_sample(args.cpu_budget, args.dim, ROUNDS, workers)
            cpu = {"value": ka / dt, "unit": "particle-steps/s", "cores": workers,
                   "kind": "reference", "host": host_cpu(), "sample_seconds": dt,
                   "sample_in_window": inside,
                   "build": "oracle/_ref/libasmc_ref_release.so (-O3 -DNDEBUG -std=gnu++20)",
                   "sample": f"unmodified reference run_sais (Release -O3) N_1={nc}, d={args.dim}, "
                             f"{ROUNDS} rounds, workers={workers}, {dt:.1f}s"}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "particle-steps/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": dict(workload(n1, args.dim), rng="philox4x32-10", precision="fp32 x / fp64 log-w",
                           lanes_per_particle=32, l2="flushed between steps (512 MB write)",
                           parallelism=f"dp{world} (particle shards, per-round chunk-partial allgather)"),
            "e2e": {"value": e2e, "unit": "particle-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "C-ABI asmc_run_rounds (run_sais) with host outputs, per step"},
            "roofline": {
                "bound": "issue", "kernel": "pass_smem_kernel<TgtScale, 32> (fused init+weight+RWMH pass)",
                "achieved": achieved / 1e9, "peak": peak_normals / 1e9, "unit": "Gnormal/s",
                "frac": achieved / peak_normals,
                "issue_frac": (load_profile_issue() or {}).get("issue_active"),
                "peak_source": "asmc_peak_normals: the pass's own generator (PhiloxKeyC, parameter-bank round keys, "
                               "normals4<float> SFU Box-Muller, 4x unrolled), registers only, measured live",
                "algorithmic_units": "normals = N*(d + T*S*d) per pass launch (the RWMH algorithm's draws)",
                "drawn": {"achieved": drawn_rate / 1e9, "frac": drawn_rate / peak_normals,
                          "fraction_of_algorithmic": pass_drawn / pass_normals,
                          "note": "normals actually generated (device counter): exact early rejection skips "
                                  "the draws of proposals whose partial MH sum plus an upper bound on the "
                                  "remaining terms is already below log u; frac here is generator-issue "
                                  "efficiency, 'frac' above is the effective rate in algorithmic units"},
                # dram__bytes_read.sum + dram__bytes_write.sum per pass launch (ncu --set full of
                # the bench's own launch); the particles never touch HBM in SAIS
                "traffic": (traffic["dram_read_bytes_per_launch"] + traffic["dram_write_bytes_per_launch"])
                if traffic else None,
                "traffic_detail": traffic,
                "ncu_issue": load_profile_issue(),
                "hbm": {"achieved_gbs_if_step_outer": hbm_alg, "peak": hbm_peak,
                        "frac": hbm_alg / hbm_peak,
                        "note": "SAIS keeps particles in registers; this is the 8d+16 B/p-step a step-outer design would move"},
            },
            "gpu_launches": int(launches),
            "clocks": clocks,
            "round_plan": {"n": plan(n1, ROUNDS, args.dim)[0], "T": plan(n1, ROUNDS, args.dim)[1]},
            "last_log_z_hat": [float(v) for v in np.asarray(last["log_z_hat"]).ravel()],
            "exact_log_z": 0.0,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if world == 1 and not args.no_configs:
            try:
                line["other_configs"] = other_configs(stream, ex, peak_normals, peaks)
                line["reference_arithmetic"] = reference_arithmetic(stream)
                if not args.no_cpu_baseline:
                    for key, v in other_cpu_baselines().items():
                        line["other_configs"][key]["cpu_baseline"] = v
            except Exception as exc:  # reported, never required
                line["other_configs"] = dict(line.get("other_configs", {}), unavailable=str(exc))
        if world == 1 and not args.no_ttt:
            try:
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                import time_to_target
                line["time_to_target"] = time_to_target.measure(n_seeds=args.ttt_seeds)
                # the paper's GPU claim: SAIS vs ZJA at equal relative variance
                line["time_to_target"]["zja_vs_sais"] = time_to_target.zja_vs_sais()
            except Exception as exc:  # reported, never required
                line["time_to_target"] = {"unavailable": str(exc)}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
