"""Slice move (new kernel kind, north_star: "random-walk MH / slice / HMC step"):
elliptical slice sampling w.r.t. the Gaussian reference eta (include/asmc_b200.h
ASMC_KERNEL_SLICE).  The reference has no slice kernel, so the oracle restatement
(oracle/restate.c:slice_move) defines it; the device's fp64 one-lane path follows it
operation for operation (1e-10 on per-particle trajectories, both RNG families), the
fp32 path within fp32 tolerance, and log Z-hat is checked against closed forms."""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
F64, F32 = abi.PREC_FP64, abi.PREC_FP32
SLICE = abi.kernel(abi.KERNEL_SLICE, (1.0,), 2)
TARGETS = [("gauss10", abi.gaussian_shift(0.5, 1.5, 1.0, 10)),
           ("mix5", abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 5)),
           ("scale7", abi.scale_gaussian(1.0, 2.0, 7)),
           ("gauss100", abi.gaussian_shift(0.0, 0.3, 1.0, 100))]


def test_slice_oracle_log_z_is_consistent():
    """closed form log Z(1) = 0 for the normalised Gaussian-family targets; mean over
    seeds within a few standard errors (T large enough that the bias is small)."""
    o = oracle.load("restate", PH)
    for tg in (abi.gaussian_shift(0.0, 1.0, 1.0, 4), abi.scale_gaussian(1.0, 1.5, 4)):
        zs = [o.run_sais_single(tg, SLICE, np.linspace(0, 1, 33), 1024, seed=s, round=1)["log_z_hat"]
              for s in range(12)]
        assert abs(np.mean(zs)) < 4 * np.std(zs) / np.sqrt(len(zs)) + 0.02, zs


def test_slice_at_beta_zero_is_an_exact_reference_draw():
    """beta = 0: every first proposal is accepted (log y < 0 = beta V), so the move is
    x' = mu + (x - mu) cos theta + (nu - mu) sin theta -- eta-invariant."""
    o = oracle.load("restate", XO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 3)
    x, lw, _ = o.trajectory(tg, abi.kernel(abi.KERNEL_SLICE, (1.0,), 1), np.array([0.0, 1e-12, 1.0]), 4, 1, 5)
    assert np.all(np.isfinite(x))


def test_slice_validation():
    with pytest.raises(oracle.OracleError):
        oracle.load("restate", XO).run_sais_single(abi.gaussian_shift(0.0, 1.0, 1.0, 2),
                                                   abi.kernel(abi.KERNEL_SLICE, (1.0,), 0), [0.0, 1.0], 8)


@pytest.mark.gpu
@pytest.mark.parametrize("name,tg", TARGETS)
def test_slice_trajectories_fp64_match_oracle(name, tg):
    betas = np.linspace(0.0, 1.0, 5)
    for rng in (XO, PH):
        rs = oracle.load("restate", rng)
        pids = [0, 7, 300, 99999]
        x, lw = capi.trajectories(tg, SLICE, betas, 4, 1, pids, abi.execopts(rng, F64))
        for i, p in enumerate(pids):
            rx, rlw, _ = rs.trajectory(tg, SLICE, betas, 4, 1, p)
            assert np.max(np.abs(x[i] - rx)) < 1e-10, (name, rng, p)
            assert np.max(np.abs(lw[i] - rlw) / np.maximum(1.0, np.abs(rlw))) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("lanes", [0, 1, 4, 32])
@pytest.mark.parametrize("name,tg", TARGETS)
def test_slice_trajectories_fp32_close_to_oracle(name, tg, lanes):
    """fp32 one-lane pass and the lane-cooperative shared-memory pass (G = 4, 32: nu
    regenerated from the counter-based stream per candidate, the spare row flipped on
    acceptance, the shrink loop warp-uniform) against the fp64 restatement."""
    betas = np.linspace(0.0, 1.0, 5)
    rs = oracle.load("restate", PH)
    pids = np.arange(48)
    x, lw = capi.trajectories(tg, SLICE, betas, 4, 1, pids, abi.execopts(PH, F32, lanes=lanes))
    ok = sum(np.max(np.abs(x[i] - rs.trajectory(tg, SLICE, betas, 4, 1, int(p))[0]))
             < 5e-4 * max(1.0, np.max(np.abs(x[i]))) for i, p in enumerate(pids))
    assert ok >= len(pids) - 1, (name, ok)


@pytest.mark.gpu
def test_slice_sais_and_ssmc_on_device():
    ex = abi.execopts(PH, F32)
    # (elliptical slice w.r.t. eta mixes slowly when the target is much wider than eta,
    # e.g. the scale family at sigma1 = 2; the shift family is the closed-form check)
    for tg in (abi.gaussian_shift(0.0, 0.5, 1.0, 50), abi.gaussian_shift(0.0, 1.0, 1.0, 10)):
        r = capi.run_sais_single(tg, SLICE, np.linspace(0, 1, 65), 1 << 15, seed=9, round=1, exec_=ex)
        assert abs(r["log_z_hat"]) < 0.1, r["log_z_hat"]
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 20)
    a = oracle.load("restate", XO).run_smc(tg, SLICE, np.linspace(0, 1, 9), 512, policy=abi.POLICY_ALWAYS, seed=2)
    b = capi.run_smc(tg, SLICE, np.linspace(0, 1, 9), 512, policy=abi.POLICY_ALWAYS, seed=2,
                     exec_=abi.execopts(XO, F64))
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 1e-9
    # the shared-memory pass (G = 32 / 4) and the one-lane pass agree within fp32 noise
    tg = abi.gaussian_shift(0.0, 0.5, 1.0, 50)
    one = capi.run_sais_single(tg, SLICE, np.linspace(0, 1, 17), 1 << 14, seed=4, round=1,
                               exec_=abi.execopts(PH, F32, lanes=1))
    for lanes in (4, 32):
        many = capi.run_sais_single(tg, SLICE, np.linspace(0, 1, 17), 1 << 14, seed=4, round=1,
                                    exec_=abi.execopts(PH, F32, lanes=lanes))
        assert abs(one["log_z_hat"] - many["log_z_hat"]) < 2e-3, (lanes, one["log_z_hat"], many["log_z_hat"])


@pytest.mark.gpu
def test_slice_beyond_the_one_lane_limit():
    """d = 2000 (> the one-lane pass's 1024): the shared-memory pass runs the slice move."""
    tg = abi.gaussian_shift(0.0, 0.05, 1.0, 2000)
    r = capi.run_sais_single(tg, SLICE, np.linspace(0, 1, 33), 4096, seed=5, round=1, exec_=abi.execopts(PH, F32))
    assert abs(r["log_z_hat"]) < 0.2, r["log_z_hat"]
