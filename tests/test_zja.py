"""ZJA online schedule adaptation: asmc_run_zja /
asmc_zja_next_beta against the unmodified reference (run_zja, zja_next_beta via
oracle/_ref) and the restatement (oracle/restate.c), plus the reference's own
known-answer tests (test_drivers.cpp:244-295, test_schedule.cpp:244-278) restated.

Device contract: precision fp64 (reference mode) runs the search as the reference's
sequential accumulation, so schedules and estimates agree to libm ulps (1e-12);
fp32 (throughput mode) folds each probe over a fixed cooperative-grid tree from fp32
particle states, so its betas agree to ~1e-6 and estimates to Monte-Carlo-free 1e-5.
"""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
F64, F32 = abi.PREC_FP64, abi.PREC_FP32


def _ref(rng):
    return oracle.load("ref", rng) if oracle.available("ref", rng) else oracle.load("restate", rng)


@pytest.mark.parametrize("rng", [XO, PH])
def test_restatement_matches_reference_run_zja(rng):
    if not oracle.available("ref", rng):
        pytest.skip("reference not built here")
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 1)
    k = abi.kernel(abi.KERNEL_IDEALIZED)
    for kw in (dict(n=256, delta_star=0.04, seed=21), dict(n=1024, target_steps=8, seed=22)):
        a = oracle.load("ref", rng).run_zja(tg, k, **kw)
        b = oracle.load("restate", rng).run_zja(tg, k, **kw)
        assert a["delta_star"] == b["delta_star"] and a["steps"] == b["steps"]
        for ra, rb in zip(a["rounds"], b["rounds"]):
            for key in ("log_g0", "log_g1", "log_g2", "cum_log_z", "lambda_"):
                assert np.array_equal(ra[key], rb[key]), key
            assert ra["log_z_hat"] == rb["log_z_hat"] and ra["elbo_hat"] == rb["elbo_hat"]
        assert np.array_equal(a["rounds"][-1]["betas"], b["rounds"][-1]["betas"])


def test_reference_known_answers_on_the_oracle():
    """test_drivers.cpp:244-295 restated on the restatement (xoshiro streams)."""
    o = oracle.load("restate", XO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 1)
    k = abi.kernel(abi.KERNEL_IDEALIZED)
    r = o.run_zja(tg, k, 256, delta_star=0.04, seed=21)
    assert len(r["rounds"]) == 1 and r["rounds"][0]["round"] == 1 and r["delta_star"] == 0.04
    m = r["rounds"][0]
    assert m["betas"][-1] == 1.0 and 3 <= r["steps"] <= 9 and m["kernel_applications"] == 256 * r["steps"]
    r = o.run_zja(tg, k, 1024, target_steps=8, seed=22)
    assert len(r["rounds"]) == 2 and r["delta_star"] > 0 and 5 <= r["steps"] <= 12 and not r["warning"]
    flat = abi.gaussian_shift(0.0, 0.0, 1.0, 1)
    r = o.run_zja(flat, k, 64, delta_star=1e-6, seed=23)
    assert list(r["rounds"][0]["betas"]) == [0.0, 1.0] and r["rounds"][0]["log_z_hat"] == 0.0


def _exact_beta_samples(n, beta, rng):
    """x_p ~ pi_beta from key (5, 1, p, 0, init), as test_schedule.cpp:249-255 draws them."""
    o = oracle.load("restate", rng)
    return np.array([0.0 + beta * 1.0 + o.rng_normal([5, 1, p, 0, 0], 1)[0] for p in range(n)])


def test_zja_next_beta_known_answers_on_the_oracle():
    """test_schedule.cpp:244-278 restated."""
    o = _ref(XO)
    n, z, beta = 1 << 14, 1.0, 0.3
    tg = abi.gaussian_shift(0.0, z, 1.0, 1)
    xs = _exact_beta_samples(n, beta, XO)
    lw = np.zeros(n)
    assert o.zja_next_beta(tg, beta, xs, lw, 1.2 * z * z) == (1.0, False)
    b, w = o.zja_next_beta(tg, beta, xs, lw, 0.01 * z * z)
    assert abs(b - (beta + 0.1)) < 0.01 and not w
    flat = abi.gaussian_shift(0.0, 0.0, 1.0, 1)
    assert o.zja_next_beta(flat, 0.0, xs, lw, 1e-8) == (1.0, False)


@pytest.mark.gpu
def test_device_zja_next_beta_matches_reference():
    n, beta = 1 << 12, 0.3
    xs = _exact_beta_samples(n, beta, XO)
    lw = np.random.default_rng(0).normal(0, 0.3, n)
    for tg in (abi.gaussian_shift(0.0, 1.0, 1.0, 1), abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 1)):
        for delta in (0.003, 0.01, 0.05, 10.0):
            a = _ref(XO).zja_next_beta(tg, beta, xs, lw, delta)
            b = capi.zja_next_beta(tg, beta, xs, lw, delta, exec_=abi.execopts(XO, F64))
            c = capi.zja_next_beta(tg, beta, xs, lw, delta, exec_=abi.execopts(PH, F32))
            assert abs(a[0] - b[0]) < 1e-12 and a[1] == b[1]
            assert abs(a[0] - c[0]) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1 << 19, (1 << 20) + 12345])
def test_cooperative_search_at_scale_matches_exact_mode(n):
    """The cooperative (fp32 / Philox) probe search holds several particles per thread
    only when N > grid x 256 (~1.5e5 threads): at N >= 2^19 its max-then-sum probe
    reductions are compared with the exact mode's reference-order search on the same
    particles (same betas to fp32-potential accuracy, same warning flags)."""
    g = np.random.default_rng(n)
    beta = 0.3
    xs = beta + g.standard_normal(n)
    lw = g.normal(0, 0.5, n)
    for tg in (abi.gaussian_shift(0.0, 1.0, 1.0, 1), abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 1)):
        for delta in (1e-4, 0.003, 0.05):
            a = capi.zja_next_beta(tg, beta, xs, lw, delta, exec_=abi.execopts(XO, F64))
            b = capi.zja_next_beta(tg, beta, xs, lw, delta, exec_=abi.execopts(PH, F32))
            assert abs(a[0] - b[0]) < 1e-6 * max(1.0, a[0]), (n, delta, a, b)
            assert a[1] == b[1]


@pytest.mark.gpu
@pytest.mark.parametrize("rng,prec", [(XO, F64), (PH, F32)])
def test_device_run_zja_matches_reference(rng, prec):
    tg = abi.gaussian_shift(0.0, 2.0, 1.0, 4)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.5, 1.0), 1)
    for kw in (dict(n=2048, delta_star=0.05, seed=3), dict(n=1024, target_steps=8, seed=4)):
        a = _ref(rng).run_zja(tg, k, **kw)
        b = capi.run_zja(tg, k, exec_=abi.execopts(rng, prec), **kw)
        assert a["steps"] == b["steps"] and len(a["rounds"]) == len(b["rounds"])
        tol = 1e-12 if prec == F64 else 1e-5
        assert abs(a["delta_star"] - b["delta_star"]) <= tol * a["delta_star"]
        assert np.max(np.abs(a["rounds"][-1]["betas"] - b["rounds"][-1]["betas"])) < (1e-12 if prec == F64 else 1e-4)
        for ra, rb in zip(a["rounds"], b["rounds"]):
            assert abs(ra["log_z_hat"] - rb["log_z_hat"]) < (1e-10 if prec == F64 else 2e-3)
            assert ra["resample_times"] == rb["resample_times"]
        assert b["rounds"][-1]["kernel_applications"] == kw["n"] * b["steps"]


@pytest.mark.gpu
def test_device_run_zja_known_answers_and_errors():
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 1)
    k = abi.kernel(abi.KERNEL_IDEALIZED)
    ex = abi.execopts(PH, F32)
    r = capi.run_zja(tg, k, 1 << 16, delta_star=0.04, seed=21, exec_=ex)
    assert r["rounds"][0]["betas"][-1] == 1.0 and 3 <= r["steps"] <= 9
    flat = abi.gaussian_shift(0.0, 0.0, 1.0, 1)
    r = capi.run_zja(flat, k, 64, delta_star=1e-6, seed=23, exec_=ex)
    assert list(r["rounds"][0]["betas"]) == [0.0, 1.0] and r["rounds"][0]["log_z_hat"] == 0.0
    with pytest.raises(capi.AsmcError) as e:
        capi.run_zja(tg, k, 64, delta_star=1e-9, max_steps=3, exec_=ex)
    assert e.value.code == abi.ERR_EVALUATION and "within 3 steps" in e.value.msg
    with pytest.raises(capi.AsmcError) as e:
        capi.run_zja(tg, k, 64, delta_star=-1.0, exec_=ex)
    assert e.value.code == abi.ERR_INVALID_ARGUMENT


@pytest.mark.gpu
def test_drop_in_run_zja_matches_reference():
    """The reference-shaped API (asmc.run_zja / ZjaOptions / ZjaOutcome) on the device."""
    import paper_2408_12057_b200 as asmc
    t = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 1)
    o = asmc.ZjaOptions()
    o.n_particles, o.target_steps, o.seed = 1024, 8, 22
    out = asmc.run_zja(t, asmc.Kernel(), o)
    ref = _ref(XO).run_zja(abi.gaussian_shift(0.0, 1.0, 1.0, 1), abi.kernel(abi.KERNEL_IDEALIZED), 1024,
                           target_steps=8, seed=22)
    assert len(out.rounds) == 2 and [r.round for r in out.rounds] == [1, 2]
    assert abs(out.delta_star - ref["delta_star"]) < 1e-12 * ref["delta_star"]
    m = out.rounds[1].report
    assert np.max(np.abs(np.array(m.schedule.betas) - ref["rounds"][1]["betas"])) < 1e-12
    assert abs(m.log_z_hat - ref["rounds"][1]["log_z_hat"]) < 1e-10
    assert m.kernel_applications == 1024 * (len(m.schedule.betas) - 1)
    r = asmc.zja_next_beta(t, 0.0, [0.1 * i for i in range(64)], 64, [0.0] * 64, 0.01)
    assert 0.0 < r.beta_next <= 1.0
