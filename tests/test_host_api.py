"""The drop-in Python API (the _core pybind module over the host C++ mirror) on CPU:
the reference's per-point target and scalar-helper tests (proj/tests/test_model.cpp,
test_engine.cpp triggers, test_drivers.cpp budget/profile, test_smoke.py theory),
exception classes, and that sampling without a GPU fails loudly (no CPU fallback)."""
import math

import numpy as np
import pytest

import paper_2408_12057_b200 as asmc


def quad_log_z(t, beta, lo, hi, intervals):  # test_model.cpp:16-28 (Simpson)
    h = (hi - lo) / intervals
    s = 0.0
    for i in range(intervals + 1):
        w = 1.0 if i in (0, intervals) else (4.0 if i % 2 else 2.0)
        s += w * math.exp(t.log_gamma(beta, [lo + i * h]))
    return math.log(s * h / 3.0)


def test_log_density_endpoints_and_affinity():  # test_model.cpp:30-52
    t = asmc.GaussianShiftTarget(0.0, 2.0, 1.0, 1)
    assert t.log_gamma(0.0, [0.7]) == t.log_reference([0.7])
    assert abs(t.log_gamma(1.0, [0.7]) - (t.log_reference([0.7]) + t.potential([0.7]))) < 1e-15
    direct = 0.5 * (-0.5 - math.log(math.sqrt(2 * math.pi))) + 0.5 * (-0.5 - math.log(math.sqrt(2 * math.pi)))
    assert abs(t.log_gamma(0.5, [1.0]) - direct) < 1e-14
    t3 = asmc.GaussianShiftTarget(-1.0, 3.0, 0.7, 3)
    x = [0.2, -0.4, 1.1]
    mid = t3.log_gamma(0.5, x)
    assert abs(2 * mid - (t3.log_gamma(0.15, x) + t3.log_gamma(0.85, x))) < 1e-12


def test_dimension_and_beta_range_enforced():  # test_model.cpp:54-63
    t = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 2)
    with pytest.raises(ValueError):
        t.log_gamma(0.5, [0.0])
    with pytest.raises(ValueError):
        t.log_gamma(-0.1, [0.0, 0.0])
    with pytest.raises(ValueError):
        asmc.GaussianShiftTarget(0.0, 1.0, 0.0, 1)
    with pytest.raises(ValueError):
        asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 0)


def test_analytic_log_z_closed_form_and_quadrature():  # test_model.cpp:65-92
    z2 = asmc.GaussianShiftTarget(0.0, 2.0, 1.0, 1)
    assert z2.analytic_log_z(0.0) == 0.0 and z2.analytic_log_z(1.0) == 0.0
    assert abs(z2.analytic_log_z(0.5) + 0.5) < 1e-15
    for z in (0.5, 1.0, 2.0, 4.0):
        t = asmc.GaussianShiftTarget(0.0, z, 1.0, 1)
        for beta in (0.1, 0.35, 0.5, 0.8):
            assert abs(t.analytic_log_z(beta) - quad_log_z(t, beta, -10.0, z + 10.0, 4000)) < 1e-6
    one, seven = asmc.GaussianShiftTarget(0.0, 1.5, 0.9, 1), asmc.GaussianShiftTarget(0.0, 1.5, 0.9, 7)
    for beta in (0.2, 0.5, 0.9):
        assert seven.analytic_log_z(beta) == 7.0 * one.analytic_log_z(beta)


def test_delta_and_discrepancy():  # test_model.cpp:94-107
    t = asmc.GaussianShiftTarget(0.0, 2.0, 1.0, 3)
    assert abs(t.analytic_delta(0.1) - 12.0) < 1e-14
    z2 = asmc.GaussianShiftTarget(0.0, 2.0, 1.0, 1)
    assert z2.analytic_discrepancy(0.3, 0.3) == 0.0
    assert abs(z2.analytic_discrepancy(0.25, 0.5) - 0.25) < 1e-12
    with pytest.raises(ValueError):
        z2.analytic_discrepancy(0.0, 0.6)


def test_scale_gaussian_closed_forms():
    """Config-2 plugin: log Z(beta) matches quadrature; D = A(2b'-b) + A(b) - 2A(b')."""
    t = asmc.ScaleGaussianTarget(1.0, 2.0, 1)
    assert abs(t.analytic_log_z(0.0)) < 1e-15 and abs(t.analytic_log_z(1.0)) < 1e-15
    for beta in (0.2, 0.5, 0.9):
        assert abs(t.analytic_log_z(beta) - quad_log_z(t, beta, -30.0, 30.0, 6000)) < 1e-7
    t1000 = asmc.ScaleGaussianTarget(1.0, 2.0, 1000)
    lam = math.sqrt(1000 / 2) * abs(math.log(0.25))  # Lambda = sqrt(d/2) |log(tau1/tau0)|
    assert 30.9 < lam < 31.1


def test_mixture_normalized_and_capabilities():  # test_model.cpp:122-149
    m = asmc.MixtureTarget(2.0, 0.3, -1.0, 0.5, 1.5, 0.8, 1)
    assert abs(quad_log_z(m, 1.0, -14.0, 14.0, 6000)) < 1e-6
    assert abs(quad_log_z(m, 0.0, -14.0, 14.0, 6000)) < 1e-6
    with pytest.raises(asmc.CapabilityError):
        m.analytic_log_z(0.5)


def test_resampling_triggers():  # test_engine.cpp:128-151
    P = asmc.ResamplePolicy
    n = 100
    assert not any(asmc.decide_resample(P.never, t, 8, 1.0, n, 100.0, 0.5) for t in range(1, 8))
    assert asmc.decide_resample(P.never, 8, 8, n, n, 0.0, 0.5)
    assert asmc.decide_resample(P.always, 3, 8, n, n, 0.0, 0.5)
    assert not asmc.decide_resample(P.adaptive_ess, 3, 8, n, n, 0.0, 0.5)
    assert asmc.decide_resample(P.adaptive_ess, 3, 8, 49.9, n, 0.0, 0.5)
    assert not asmc.decide_resample(P.adaptive_ess, 3, 8, 50.0, n, 0.0, 0.5)
    d = 0.35
    rho = math.exp(-3 * d)
    assert [asmc.decide_resample(P.stabilized, k, 8, n, n, k * d, rho) for k in range(1, 5)] == \
        [False, False, False, True]


def test_budget_schedule_profile():  # test_drivers.cpp:43-68, 122-136; engine.cpp:16-27
    b = asmc.budget(16, 8, 1, 1 << 40, asmc.DriverMode.ssmc)
    assert (b.n_particles, b.steps) == (23, 12)
    b = asmc.budget(16, 8, 4, 23 * 4 * 8 - 1, asmc.DriverMode.ssmc)
    assert (b.n_particles, b.steps) == (16, 16)
    s = asmc.Schedule.uniform(4)
    assert s.betas == [0.0, 0.25, 0.5, 0.75, 1.0] and s.steps() == 4
    with pytest.raises(ValueError):
        asmc.Schedule.uniform(0)
    small, large = asmc.sais_memory_profile(16, 2, 64), asmc.sais_memory_profile(16, 2, 1 << 14)
    assert small.moment_accumulators == large.moment_accumulators == 3 * 17
    assert large.signed_accumulators == 17 and large.wave_block_slots == (1 << 14) // 256
    assert asmc.sais_memory_profile(16, 4, 0).wave_block_slots == 4


def test_theory_helpers():  # proj/tests/python/test_smoke.py:34-41
    rv = asmc.theory.rel_variance(1.0, 1.0, 1.0)
    assert abs(rv - (math.e - 1.0)) < 1e-12
    solved = asmc.theory.solve_r_eff(4.0, 256.0, asmc.theory.rel_variance(4.0, 8.0, 256.0))
    assert abs(solved - 8.0) < 1e-5
    b = asmc.theory.stabilized_r_eff_bounds(2.0, 1.0, 8.0, math.exp(-1.0))
    assert abs(b.lower - 1.0) < 1e-12 and abs(b.upper - 1.5) < 1e-12
    pb = asmc.theory.particle_bounds(2.0, 1.0, 1.0, 4.0, 0.1)  # acceptance criterion 11
    assert abs(pb.n_min - 17.18281828459045) <= 1e-9 and abs(pb.n_max - 18.02831378543967) <= 1e-9
    R = asmc.theory.Regime
    grid = [(0.0, 0.0, R.coarse), (1.0, 0.5, R.coarse), (1.9, 0.0, R.coarse), (2.0, 0.0, R.stable),
            (1.0, 1.0, R.stable), (0.0, 2.0, R.stable), (3.0, 1.5, R.stable), (0.0, 2.5, R.dense),
            (1.0, 3.0, R.dense)]
    assert all(asmc.theory.classify_regime(a, t) == w for a, t, w in grid)


def test_validation_errors_before_the_device():
    t = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 1)
    bad = asmc.Schedule()
    bad.betas = [0.0, 0.5]
    with pytest.raises(ValueError, match="end at beta = 1"):
        asmc.run_smc(t, asmc.Kernel(), bad, asmc.RunOptions())
    k = asmc.Kernel()
    k.kind = asmc.KernelKind.rwmh_cycle
    k.step_sizes = []
    with pytest.raises(ValueError):
        asmc.run_smc(t, k, asmc.Schedule.uniform(2), asmc.RunOptions())


@pytest.mark.skipif(asmc.device_count() > 0, reason="checks the no-GPU behaviour")
def test_sampling_without_gpu_fails_loudly():
    t = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 1)
    with pytest.raises(asmc.DeviceError, match="no CPU fallback"):
        asmc.run_smc(t, asmc.Kernel(), asmc.Schedule.uniform(2), asmc.RunOptions())
    with pytest.raises(asmc.DeviceError):
        asmc.run_sais(t, asmc.Kernel(), asmc.DriverOptions())
