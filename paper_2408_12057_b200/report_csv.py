"""Experiment CSV outputs from device reports.

Restates the reference's writer (src/experiment.cpp:23-76, headers
include/asmc/experiment.hpp:10-16): summary.csv, trace.csv, schedule.csv and
barrier.csv, every double printed with "%.17g", wall_clock_seconds pinned to 0
unless `timing`.  Fed from the B200 round reports (capi.run_rounds,
distributed.run_sais, capi.run_zja), so a B200 run produces the same files a
reference run does; tests/test_report_csv.py pins the bytes against the
reference's own run_experiment on the same reports.  Host-side formatting only.
"""
import math
import os

import numpy as np

SUMMARY = "round,N,T,log_Z_hat,elbo_hat,Lambda_hat,kernel_applications,wall_clock_seconds"
TRACE = "round,t,beta,log_g0,log_g1,log_g2,ess,resampled,cum_log_Z"
SCHEDULE = "round,t,beta"
BARRIER = "round,t,beta,D_hat,Lambda_hat,lambda_hat"
PT_TRACE = "iteration,level,beta,V,swap_accepted"


def fmt(v):
    """printf("%.17g") as experiment.cpp:25-29 (inf / nan spelled as glibc does)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def discrepancy_hat(g0, g1, g2):
    raw = g2 - 2.0 * g1 + g0  # schedule.cpp:27-31
    return raw if raw > 0.0 else 0.0


def rounds_from_run_rounds(res, ssmc):
    """capi.run_rounds / oracle run_rounds arrays -> per-round dicts (RoundResult)."""
    out = []
    for k in range(len(res["steps"])):
        T = int(res["steps"][k])
        sl = slice(0, T + 1)
        out.append(dict(round=k + 1, n=int(res["n_particles"][k]), steps=T,
                        betas=res["betas"][k][sl], log_g0=res["log_g0"][k][sl], log_g1=res["log_g1"][k][sl],
                        log_g2=res["log_g2"][k][sl], ess=res["ess_trace"][k][sl] if ssmc else None,
                        resampled=res["resampled"][k][sl], cum_log_z=res["cum_log_z"][k][sl],
                        lambda_=res["lambda_"][k][sl], log_z_hat=float(res["log_z_hat"][k]),
                        elbo_hat=float(res["elbo_hat"][k]),
                        kernel_applications=int(res["kernel_applications"][k]),
                        wall_seconds=float(res["wall_seconds"][k])))
    return out


def rounds_from_zja(res, n):
    """capi.run_zja / oracle run_zja dict -> per-round dicts (pilot first)."""
    out = []
    for r in res["rounds"]:
        T = len(r["lambda_"]) - 1
        betas = r["betas"] if "betas" in r else np.array([t / T for t in range(T)] + [1.0])
        out.append(dict(round=r["round"], n=n, steps=T, betas=betas, log_g0=r["log_g0"], log_g1=r["log_g1"],
                        log_g2=r["log_g2"], ess=r["ess_trace"], resampled=r["resampled"], cum_log_z=r["cum_log_z"],
                        lambda_=r["lambda_"], log_z_hat=r["log_z_hat"], elbo_hat=r["elbo_hat"],
                        kernel_applications=int(r["kernel_applications"]), wall_seconds=r["wall_seconds"]))
    return out


def write_experiment(out_dir, replicates, local_barrier, timing=False):
    """run_particle_driver's outputs (experiment.cpp:83-141): `replicates` is a list
    (one entry per replicate) of round-dict lists; detail files from replicate 0.
    `local_barrier(lambda, beta)` is schedule.cpp:189-197 (device or oracle)."""
    os.makedirs(out_dir, exist_ok=True)
    files = {name: open(os.path.join(out_dir, name), "w", newline="\n")
             for name in ("summary.csv", "trace.csv", "schedule.csv", "barrier.csv")}
    try:
        files["summary.csv"].write(SUMMARY + "\n")
        files["trace.csv"].write(TRACE + "\n")
        files["schedule.csv"].write(SCHEDULE + "\n")
        files["barrier.csv"].write(BARRIER + "\n")
        for i, rounds in enumerate(replicates):
            for r in rounds:
                files["summary.csv"].write(
                    f"{r['round']},{r['n']},{r['steps']},{fmt(r['log_z_hat'])},{fmt(r['elbo_hat'])},"
                    f"{fmt(r['lambda_'][-1])},{r['kernel_applications']},"
                    f"{fmt(r['wall_seconds'] if timing else 0.0)}\n")
            if i:
                continue
            for r in rounds:
                loc = local_barrier(np.asarray(r["lambda_"], dtype=np.float64),
                                    np.asarray(r["betas"], dtype=np.float64))
                for t in range(r["steps"] + 1):
                    b = fmt(r["betas"][t])
                    ess = fmt(r["ess"][t]) if r["ess"] is not None else "nan"
                    files["trace.csv"].write(
                        f"{r['round']},{t},{b},{fmt(r['log_g0'][t])},{fmt(r['log_g1'][t])},"
                        f"{fmt(r['log_g2'][t])},{ess},{int(r['resampled'][t])},{fmt(r['cum_log_z'][t])}\n")
                    files["schedule.csv"].write(f"{r['round']},{t},{b}\n")
                    dh = 0.0 if t == 0 else discrepancy_hat(r["log_g0"][t], r["log_g1"][t], r["log_g2"][t])
                    files["barrier.csv"].write(
                        f"{r['round']},{t},{b},{fmt(dh)},{fmt(r['lambda_'][t])},{fmt(loc[t])}\n")
    finally:
        for f in files.values():
            f.close()


def write_pt_experiment(out_dir, betas, reports, timing=False):
    """run_pt_driver's outputs (experiment.cpp:143-186) from capi.run_pt / oracle
    run_pt (all replicas of one call): summary.csv rows per replica, schedule.csv and
    pt_trace.csv from replicate 0, trace.csv and barrier.csv header-only."""
    os.makedirs(out_dir, exist_ok=True)
    nan = float("nan")
    L = len(betas) - 1
    with open(os.path.join(out_dir, "summary.csv"), "w", newline="\n") as f:
        f.write(SUMMARY + "\n")
        for r in range(len(reports["log_z_hat"])):
            f.write(f"1,{L},{reports['trace'].shape[1]},{fmt(reports['log_z_hat'][r])},{fmt(nan)},{fmt(nan)},"
                    f"{reports['kernel_applications']},{fmt(reports['wall_seconds'] if timing else 0.0)}\n")
    for name, hdr in (("trace.csv", TRACE), ("barrier.csv", BARRIER)):
        with open(os.path.join(out_dir, name), "w", newline="\n") as f:
            f.write(hdr + "\n")
    with open(os.path.join(out_dir, "schedule.csv"), "w", newline="\n") as f:
        f.write(SCHEDULE + "\n")
        for t in range(L + 1):
            f.write(f"1,{t},{fmt(betas[t])}\n")
    with open(os.path.join(out_dir, "pt_trace.csv"), "w", newline="\n") as f:
        f.write(PT_TRACE + "\n")
        tr, acc = reports["trace"][0], reports["swap_accepted"][0]
        for it in range(tr.shape[0]):
            for n in range(L + 1):
                f.write(f"{it},{n},{fmt(betas[n])},{fmt(tr[it, n])},{int(acc[it, n])}\n")
