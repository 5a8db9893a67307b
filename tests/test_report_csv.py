"""Experiment CSV parity: paper_2408_12057_b200/report_csv.py
writes the reference's summary/trace/schedule/barrier files (experiment.cpp:23-141).

* CPU: the writer fed with the reference's own reports (oracle/_ref run_rounds,
  run_zja) reproduces the bytes of the reference's run_experiment on the same
  config -- the format is pinned.
* GPU: device reports (fp64 reference mode) give the same files up to libm ulps;
  SAIS sharded over 1 or 3 virtual GPUs gives byte-identical files (the analogue of
  acceptance criterion 10, acceptance.cpp:408-457)."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, report_csv

XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
FILES = ("summary.csv", "trace.csv", "schedule.csv", "barrier.csv")

CONFIGS = {
    "sais": ("driver = sais\ntarget = gaussian_shift\ndim = 10\nkernel = rwmh\nn = 1024\nrounds = 3\n"
             "seed = 1\nworkers = 1\nreplicates = 2\n",
             dict(tg=abi.gaussian_shift(0.0, 1.0, 1.0, 10), mode=abi.MODE_SAIS, n=1024, rounds=3, seed=1, reps=2)),
    "ssmc": ("driver = ssmc\ntarget = mixture\ndim = 3\nkernel = rwmh\nn = 512\nrounds = 3\nseed = 7\n"
             "workers = 1\n",
             dict(tg=abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 3), mode=abi.MODE_SSMC, n=512, rounds=3, seed=7,
                  reps=1)),
}
ZJA = "driver = ais_zja\ntarget = gaussian_shift\ndim = 1\nkernel = idealized\nn = 1024\nzja_steps = 8\nseed = 22\n"


def _reference_csvs(text, tmp_path):
    """The reference's run_experiment, in a fresh interpreter: the reference library's
    std::filesystem / iostream code must be loaded before numpy's bundled runtimes."""
    if not oracle.available("ref", XO):
        pytest.skip("reference not built here")
    d = str(tmp_path / "ref")
    code = ("import ctypes, sys; lib = ctypes.CDLL(sys.argv[1]); "
            "sys.exit(lib.ora_run_experiment(sys.argv[2].encode(), sys.argv[3].encode()))")
    r = subprocess.run([sys.executable, "-c", code, oracle.load("ref", XO).path, text, d],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return {f: open(os.path.join(d, f)).read() for f in FILES}


def _read(d):
    return {f: open(os.path.join(d, f)).read() for f in FILES}


@pytest.mark.parametrize("name", ["sais", "ssmc"])
def test_writer_reproduces_reference_bytes(name, tmp_path):
    text, c = CONFIGS[name]
    ref_files = _reference_csvs(text, tmp_path)
    o = oracle.load("ref", XO)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    reps = [report_csv.rounds_from_run_rounds(
        o.run_rounds(c["tg"], k, c["mode"], c["n"], c["rounds"], seed=c["seed"] + i), c["mode"] == abi.MODE_SSMC)
        for i in range(c["reps"])]
    report_csv.write_experiment(str(tmp_path / "ours"), reps, o.local_barrier)
    assert _read(str(tmp_path / "ours")) == ref_files


def test_writer_reproduces_reference_bytes_zja(tmp_path):
    ref_files = _reference_csvs(ZJA, tmp_path)
    o = oracle.load("ref", XO)
    r = o.run_zja(abi.gaussian_shift(0.0, 1.0, 1.0, 1), abi.kernel(abi.KERNEL_IDEALIZED), 1024, target_steps=8,
                  seed=22)
    report_csv.write_experiment(str(tmp_path / "ours"), [report_csv.rounds_from_zja(r, 1024)], o.local_barrier)
    assert _read(str(tmp_path / "ours")) == ref_files


def _numeric(files):
    out = {}
    for f, txt in files.items():
        rows = list(csv.reader(txt.splitlines()))
        out[f] = (rows[0], np.array([[float(v) for v in r] for r in rows[1:]]))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sais", "ssmc"])
def test_device_reports_give_reference_csvs(name, tmp_path):
    from paper_2408_12057_b200 import capi
    text, c = CONFIGS[name]
    ref_files = _numeric(_reference_csvs(text, tmp_path))
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    reps = [report_csv.rounds_from_run_rounds(
        capi.run_rounds(c["tg"], k, c["mode"], c["n"], c["rounds"], seed=c["seed"] + i,
                        exec_=abi.execopts(XO, abi.PREC_FP64)), c["mode"] == abi.MODE_SSMC)
        for i in range(c["reps"])]
    report_csv.write_experiment(str(tmp_path / "dev"), reps, capi.local_barrier)
    ours = _numeric(_read(str(tmp_path / "dev")))
    for f in FILES:
        assert ours[f][0] == ref_files[f][0] and ours[f][1].shape == ref_files[f][1].shape, f
        a, b = ours[f][1], ref_files[f][1]
        same = (a == b) | (np.isnan(a) & np.isnan(b))
        close = np.abs(a - b) <= 1e-11 * np.maximum(1.0, np.abs(b))
        assert np.all(same | close), f


@pytest.mark.gpu
def test_sharded_csvs_byte_identical(tmp_path):
    from paper_2408_12057_b200 import capi, distributed
    tg = abi.scale_gaussian(1.0, 2.0, 50)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.5, 1.0), 1)
    ex = abi.execopts(PH, abi.PREC_FP32)
    n1 = 3 * abi.FOLD_CHUNK + 1000
    # world 3 via virtual shards: partials of each rank's chunk range, folded in chunk order
    def run_virtual(world):
        import numpy as np
        betas, n, T = np.array([0.0, 1.0]), n1, 1
        res = {key: [] for key in ("n_particles", "steps", "betas", "log_g0", "log_g1", "log_g2", "lambda_",
                                   "log_z_hat", "elbo_hat", "kernel_applications", "cum_log_z", "resampled",
                                   "wall_seconds")}
        for r in range(1, 4):
            ranges = distributed.chunk_partition(n, world)
            allp = np.concatenate([capi.sais_partials(tg, k, betas, n, p0, p1, seed=5, round=r, exec_=ex)
                                   for p0, p1 in ranges if p1 > p0])
            rep = capi.fold_partials(allp, n)
            lam = capi.barrier_estimate(rep["log_g0"], rep["log_g1"], rep["log_g2"], betas)
            for key, v in (("n_particles", n), ("steps", T), ("betas", betas.copy()), ("log_g0", rep["log_g0"]),
                           ("log_g1", rep["log_g1"]), ("log_g2", rep["log_g2"]), ("lambda_", lam),
                           ("log_z_hat", rep["log_z_hat"]), ("elbo_hat", rep["elbo_hat"]),
                           ("kernel_applications", n * T), ("cum_log_z", rep["cum_log_z"]),
                           ("resampled", rep["resampled"]), ("wall_seconds", 0.0)):
                res[key].append(v)
            if r < 3:
                n2, T2 = capi.budget(n, T, tg.dim, 4096 << 20, abi.MODE_SAIS)
                betas = capi.generate_schedule(lam, betas, T2)
                n, T = n2, T2
        return res
    dirs = []
    for world in (1, 3):
        res = run_virtual(world)
        rounds = [dict(round=i + 1, n=int(res["n_particles"][i]), steps=int(res["steps"][i]), betas=res["betas"][i],
                       log_g0=res["log_g0"][i], log_g1=res["log_g1"][i], log_g2=res["log_g2"][i], ess=None,
                       resampled=res["resampled"][i], cum_log_z=res["cum_log_z"][i], lambda_=res["lambda_"][i],
                       log_z_hat=res["log_z_hat"][i], elbo_hat=res["elbo_hat"][i],
                       kernel_applications=res["kernel_applications"][i], wall_seconds=0.0) for i in range(3)]
        d = str(tmp_path / f"w{world}")
        report_csv.write_experiment(d, [rounds], capi.local_barrier)
        dirs.append(_read(d))
    assert dirs[0] == dirs[1]
    assert dirs[0]["summary.csv"].count("\n") == 4


PT_TEXT = ("driver = pt\ntarget = gaussian_shift\ndim = 2\nkernel = rwmh\nlevels = 6\niterations = 200\n"
           "seed = 3\nreplicates = 3\nworkers = 1\n")


def test_pt_writer_reproduces_reference_bytes(tmp_path):
    ref_files = _reference_csvs(PT_TEXT, tmp_path)
    o = oracle.load("ref", XO)
    betas = np.array([t / 6 for t in range(6)] + [1.0])
    r = o.run_pt(abi.gaussian_shift(0.0, 1.0, 1.0, 2), abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1), betas,
                 iterations=200, seed=3, replicas=3)
    report_csv.write_pt_experiment(str(tmp_path / "ours"), betas, r)
    ours = _read(str(tmp_path / "ours"))
    ours["pt_trace.csv"] = open(str(tmp_path / "ours" / "pt_trace.csv")).read()
    ref_files["pt_trace.csv"] = open(str(tmp_path / "ref" / "pt_trace.csv")).read()
    assert ours == ref_files
