"""Non-reversible parallel tempering: asmc_run_pt against the
unmodified reference run_pt (oracle/_ref, both RNG families), with the reference's
own test_pt.cpp:37-129 cases restated on the device.  fp64 (reference mode) runs
the reference's operation order, so traces, swap decisions and log Z-hat agree to
libm ulps; replicas (seeds seed .. seed + R - 1) run in one launch."""
import math

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
F64, F32 = abi.PREC_FP64, abi.PREC_FP32
IDEAL = abi.kernel(abi.KERNEL_IDEALIZED)


def _ref(rng):
    if not oracle.available("ref", rng):
        pytest.skip("reference not built here")
    return oracle.load("ref", rng)


def test_reference_pt_known_answers_via_oracle():
    o = _ref(XO)
    r = o.run_pt(abi.gaussian_shift(0.0, 0.0, 1.0, 1), IDEAL, np.linspace(0, 1, 5), iterations=64, seed=5)
    assert r["log_z_hat"][0] == 0.0 and r["burn_in"] == 6 and r["kernel_applications"] == 4 * 64
    assert list(r["swap_attempts"][0]) == [32, 32, 32, 32, 0]
    assert np.array_equal(r["swap_accepts"][0], r["swap_attempts"][0])


@pytest.mark.gpu
@pytest.mark.parametrize("rng", [XO, PH])
def test_device_pt_fp64_matches_reference(rng):
    o = _ref(rng)
    for tg, k in ((abi.gaussian_shift(0.0, 2.0, 1.0, 3), abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)),
                  (abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 4), abi.kernel(abi.KERNEL_RWMH, (0.3, 1.0), 2)),
                  (abi.scale_gaussian(1.0, 2.0, 20), abi.kernel(abi.KERNEL_IDEALIZED))):
        betas = np.linspace(0, 1, 7)
        a = o.run_pt(tg, k, betas, iterations=300, seed=11, replicas=3)
        b = capi.run_pt(tg, k, betas, iterations=300, seed=11, replicas=3, exec_=abi.execopts(rng, F64))
        assert np.max(np.abs(a["trace"] - b["trace"]) / np.maximum(1.0, np.abs(a["trace"]))) < 1e-11
        assert np.array_equal(a["swap_accepted"], b["swap_accepted"])
        assert np.array_equal(a["swap_accepts"], b["swap_accepts"])
        assert np.array_equal(a["swap_attempts"], b["swap_attempts"])
        assert np.max(np.abs(a["log_z_hat"] - b["log_z_hat"])) < 1e-11


@pytest.mark.gpu
def test_device_pt_reference_cases():
    ex = abi.execopts(XO, F64)
    # flat target: every swap accepted, exact (test_pt.cpp:37-59)
    r = capi.run_pt(abi.gaussian_shift(0.0, 0.0, 1.0, 1), IDEAL, np.linspace(0, 1, 5), iterations=64, seed=5,
                    exec_=ex)
    assert r["log_z_hat"][0] == 0.0 and r["burn_in"] == 6 and np.all(r["trace"] == 0.0)
    assert list(r["swap_attempts"][0]) == [32, 32, 32, 32, 0]
    assert np.array_equal(r["swap_accepts"][0], r["swap_attempts"][0])
    # two-level swap rate = 2 Phi(-z / sqrt 2) (test_pt.cpp:83-100)
    r = capi.run_pt(abi.gaussian_shift(0.0, 1.0, 1.0, 1), IDEAL, [0.0, 1.0], iterations=20000, burn_in=0, seed=31,
                    exec_=ex)
    rate = r["swap_accepts"][0][0] / r["swap_attempts"][0][0]
    closed = 2.0 * 0.5 * math.erfc(1.0 / math.sqrt(2.0) / math.sqrt(2.0))
    assert r["swap_attempts"][0][0] == 10000 and abs(rate - closed) < 4 * 0.5 / math.sqrt(10000)
    # unbiased Z = 1 over 300 seeds, all replicas in ONE launch (test_pt.cpp:118-129)
    r = capi.run_pt(abi.gaussian_shift(0.0, 1.0, 1.0, 1), IDEAL, [0.0, 1.0], iterations=64, burn_in=0, seed=800,
                    replicas=300, exec_=ex)
    zs = np.exp(r["log_z_hat"])
    assert abs(zs.mean() - 1.0) <= 3.0 * zs.std() / math.sqrt(len(zs))


@pytest.mark.gpu
def test_device_pt_fp32_close_to_reference():
    tg, k = abi.gaussian_shift(0.0, 2.0, 1.0, 3), abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    betas = np.linspace(0, 1, 7)
    a = _ref(PH).run_pt(tg, k, betas, iterations=200, seed=4, replicas=8)
    b = capi.run_pt(tg, k, betas, iterations=200, seed=4, replicas=8, exec_=abi.execopts(PH, F32))
    same = np.mean(a["swap_accepted"] == b["swap_accepted"])
    assert same > 0.99
    assert np.max(np.abs(a["log_z_hat"] - b["log_z_hat"])) < 0.05


@pytest.mark.gpu
def test_drop_in_run_pt():
    import paper_2408_12057_b200 as asmc
    t = asmc.GaussianShiftTarget(0.0, 2.0, 1.0, 3)
    k = asmc.Kernel()
    o = asmc.PtOptions()
    o.iterations, o.seed = 200, 11
    rep = asmc.run_pt(t, k, asmc.Schedule.uniform(6), o)
    ref = _ref(XO).run_pt(abi.gaussian_shift(0.0, 2.0, 1.0, 3), IDEAL, np.linspace(0, 1, 7), iterations=200, seed=11)
    assert abs(rep.log_z_hat - ref["log_z_hat"][0]) < 1e-11 and rep.burn_in == 20
    assert abs(asmc.stepping_stone(rep.trace, rep.schedule, rep.burn_in) - rep.log_z_hat) < 1e-13
    reps = asmc.run_pt_replicas(t, k, asmc.Schedule.uniform(6), o, 4)
    assert len(reps) == 4 and reps[0].log_z_hat == rep.log_z_hat
