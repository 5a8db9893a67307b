"""Edge cases the reference's own tests exercise, on the device: degenerate weights
(test_engine.cpp:286-311), ESS of an all -inf vector (test_engine.cpp:71-83), a single
particle, a single step, ragged particle counts, and schedules too long for the
shared-memory accumulators (a clean capability error, never a wrong answer).  The
reference (oracle/_ref) gives the expected outcome and message on the same inputs."""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu
XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
F64, F32 = abi.PREC_FP64, abi.PREC_FP32


def _ref():
    return oracle.load("ref", XO) if oracle.available("ref", XO) else oracle.load("restate", XO)


def test_degenerate_weights_abort_like_the_reference():
    spread = abi.gaussian_shift(0.0, 1e6, 1.0, 1)
    ident = abi.kernel(abi.KERNEL_IDENTITY)
    with pytest.raises(oracle.OracleError) as r:
        _ref().run_smc(spread, ident, [0.0, 1.0], 2, policy=abi.POLICY_NEVER, seed=1)
    for ex in (abi.execopts(XO, F64), abi.execopts(PH, F32)):
        with pytest.raises(capi.AsmcError) as e:
            capi.run_smc(spread, ident, [0.0, 1.0], 2, policy=abi.POLICY_NEVER, seed=1, exec_=ex)
        assert e.value.code == abi.ERR_DEGENERATE == r.value.code
        assert "degenerate" in e.value.msg


def test_ess_edge_cases():
    with pytest.raises(capi.AsmcError) as e:
        capi.ess(np.array([-np.inf, -np.inf]))
    assert e.value.code == abi.ERR_DEGENERATE
    assert abs(capi.ess(np.array([0.0, -np.inf, -np.inf, -np.inf])) - 1.0) < 1e-12
    assert abs(capi.ess(np.full(8, -1.3)) - 8.0) < 1e-12 * 8


@pytest.mark.parametrize("policy", [abi.POLICY_NEVER, abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS])
def test_single_particle_and_single_step(policy):
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 3)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    ex = abi.execopts(XO, F64)
    for n, betas in ((1, np.linspace(0, 1, 6)), (300, [0.0, 1.0]), (257, np.linspace(0, 1, 4))):
        a = _ref().run_smc(tg, k, betas, n, policy=policy, seed=4, round=2)
        b = capi.run_smc(tg, k, betas, n, policy=policy, seed=4, round=2, exec_=ex)
        assert a["resample_times"] == b["resample_times"]
        assert abs(a["log_z_hat"] - b["log_z_hat"]) < 1e-10 * max(1.0, abs(a["log_z_hat"]))
    a = _ref().run_sais_single(tg, k, [0.0, 1.0], 1, seed=2, round=1)
    b = capi.run_sais_single(tg, k, [0.0, 1.0], 1, seed=2, round=1, exec_=ex)
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 1e-10


def test_long_schedule_runs_in_t_tiles():
    """T far beyond one launch's shared-memory accumulators (2000 steps at d = 1000) runs
    in t-tiles instead of being refused (the reference has no T cap, drivers.cpp:59-146);
    the values against the reference: tests/test_gpu_long_t.py."""
    tg = abi.scale_gaussian(1.0, 2.0, 1000)
    k = abi.kernel(abi.KERNEL_RWMH, (0.05,), 1)
    betas = np.linspace(0, 1, 2001)
    r = capi.run_sais_single(tg, k, betas, 512, seed=1, round=1, exec_=abi.execopts(PH, F32))
    assert np.all(np.isfinite(r["log_g1"][1:])) and np.isfinite(r["log_z_hat"])


def test_ragged_counts_fp32_paths():
    """particle counts that are not multiples of the 256-block or the 262144 fold chunk"""
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 30)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    for n in (1, 255, 257, 262145):
        r = capi.run_smc(tg, k, np.linspace(0, 1, 5), n, policy=abi.POLICY_ALWAYS, seed=3,
                         exec_=abi.execopts(PH, F32))
        assert np.all(np.isfinite(r["log_g1"][1:])) and r["resample_times"] == [1, 2, 3, 4]
