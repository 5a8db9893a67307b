"""Exact early rejection never changes a decision (GPU).

The shared-memory RWMH pass stops drawing a proposal's normals once the partial MH
sum plus an upper bound on the remaining coordinates' terms (plus a rounding margin)
is below log u, with the warp sum formed by one fixed-point REDUX (G = 32) or an fp32
butterfly (G < 32), on a per-step-size check schedule.  Rejection is then certain, so
every output must be bit-identical to the run that evaluates every proposal in full
(env ASMC_NO_EARLY_REJECT=1, read by the library at each call) -- while drawing
fewer normals.
"""
import numpy as np
import pytest

from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu

RWMH = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


def _both(monkeypatch, fn):
    capi.profile_enable(True)
    a = fn()
    _, _, drawn_a = capi.profile_collect(drawn=True)
    monkeypatch.setenv("ASMC_NO_EARLY_REJECT", "1")
    b = fn()
    _, _, drawn_b = capi.profile_collect(drawn=True)
    monkeypatch.delenv("ASMC_NO_EARLY_REJECT")
    capi.profile_enable(False)
    return a, b, float(np.sum(drawn_a)), float(np.sum(drawn_b))


def _same(a, b, keys):
    for k in keys:
        x, y = np.asarray(a[k], float), np.asarray(b[k], float)
        assert np.array_equal(x, y, equal_nan=True), (k, x, y)


CASES = [("config2_scale1000", abi.scale_gaussian(1.0, 2.0, 1000), 32),
         ("scale300", abi.scale_gaussian(1.0, 2.0, 300), 32),
         ("scale302_ragged", abi.scale_gaussian(1.0, 2.0, 302), 32),
         ("gauss1000", abi.gaussian_shift(0.0, 1.0, 1.0, 1000), 32),
         ("gauss100_g4", abi.gaussian_shift(0.0, 0.3, 1.0, 100), 4),
         ("scale100_g4", abi.scale_gaussian(1.0, 2.0, 100), 4)]


@pytest.mark.parametrize("name,tg,lanes", CASES)
def test_sais_bit_identical_without_early_rejection(monkeypatch, name, tg, lanes):
    ex = abi.execopts(PH, F32, lanes=lanes)
    betas = np.linspace(0.0, 1.0, 4)
    a, b, da, db = _both(monkeypatch, lambda: capi.run_sais_single(tg, RWMH, betas, 4096, seed=5, round=2,
                                                                     exec_=ex))
    _same(a, b, ["log_g0", "log_g1", "log_g2", "log_z_hat", "elbo_hat"])
    assert da < db, (name, da, db)  # early rejection did skip draws


@pytest.mark.parametrize("name,tg,lanes", CASES[:2] + CASES[4:5])
def test_smc_step_mode_bit_identical_without_early_rejection(monkeypatch, name, tg, lanes):
    ex = abi.execopts(PH, F32, lanes=lanes)
    betas = np.linspace(0.0, 1.0, 7)
    a, b, da, db = _both(monkeypatch, lambda: capi.run_smc(tg, RWMH, betas, 4096, policy=abi.POLICY_ADAPTIVE_ESS,
                                                             seed=3, round=1, exec_=ex))
    _same(a, b, ["log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z", "log_z_hat", "elbo_hat"])
    assert list(a["resample_times"]) == list(b["resample_times"])
    assert da < db


def test_trajectories_bit_identical_without_early_rejection(monkeypatch):
    tg = abi.scale_gaussian(1.0, 2.0, 1000)
    ex = abi.execopts(PH, F32, lanes=32)
    pids = np.arange(0, 4096, 37)
    betas = np.linspace(0.0, 1.0, 5)
    a, b, _, _ = _both(monkeypatch, lambda: capi.trajectories(tg, RWMH, betas, 9, 1, pids, ex))
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("steps", [(1e-4, 1e2, 1e4), (3.0, 30.0, 300.0)])
def test_extreme_step_sizes_bit_identical(monkeypatch, steps):
    """Per-lane partial sums far outside the fixed-point window (clamped at -4096 below,
    saturated above 65536) and near zero: decisions still equal the full evaluation's."""
    tg = abi.scale_gaussian(1.0, 2.0, 1000)
    k = abi.kernel(abi.KERNEL_RWMH, steps, 2)
    ex = abi.execopts(PH, F32, lanes=32)
    betas = np.linspace(0.0, 1.0, 4)
    a, b, da, db = _both(monkeypatch, lambda: capi.run_sais_single(tg, k, betas, 2048, seed=11, round=1,
                                                                     exec_=ex))
    _same(a, b, ["log_g0", "log_g1", "log_g2", "log_z_hat", "elbo_hat"])
    assert da < db

