"""GPU tests through the drop-in Python API and the multi-GPU partial path.

* proj/tests/python/test_smoke.py, restated against `paper_2408_12057_b200 as asmc`;
* closed-form log Z: estimates within Monte-Carlo error of the exact value;
* unbiasedness of Z-hat over seeds (test_engine.cpp:166-185 analogue) on the
  fp32 Philox path;
* GPU-count invariance: chunk partials of any particle split fold to the same
  bits as the single-launch pass (the virtual-shard mode of SURVEY 4);
* SSMC fp64 Philox vs the oracle's restatement (the reference's resampling rule).
"""
import math

import numpy as np
import pytest

import oracle
import paper_2408_12057_b200 as asmc
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu

PH, F32, F64 = abi.RNG_PHILOX, abi.PREC_FP32, abi.PREC_FP64


# ---- proj/tests/python/test_smoke.py --------------------------------------
def test_flat_target_is_exact():
    target = asmc.GaussianShiftTarget(0.0, 0.0, 1.0, 1)
    opts = asmc.RunOptions()
    opts.n_particles = 64
    opts.policy = asmc.ResamplePolicy.never
    opts.seed = 3
    report = asmc.run_smc(target, asmc.Kernel(), asmc.Schedule.uniform(4), opts)
    assert report.log_z_hat == 0.0
    assert report.elbo_hat == 0.0
    assert report.resample_times == [4]


def test_streaming_matches_in_memory():
    target = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 1)
    schedule = asmc.Schedule.uniform(6)
    opts = asmc.RunOptions()
    opts.n_particles = 128
    opts.policy = asmc.ResamplePolicy.never
    opts.seed = 11
    a = asmc.run_smc(target, asmc.Kernel(), schedule, opts)
    b = asmc.run_sais_single(target, asmc.Kernel(), schedule, opts)
    assert a.log_z_hat == b.log_z_hat
    assert a.stats.log_g1 == b.stats.log_g1


def test_schedule_generation_round_trip():
    est = asmc.BarrierEstimate()
    est.beta = [0.0, 0.25, 0.5, 1.0]
    est.lambda_knots = [0.0, 1.0, 2.0, 3.0]
    out = asmc.generate_schedule(est, 3)
    assert max(abs(b - e) for b, e in zip(out.betas, est.beta)) < 1e-12


def test_round_driver():
    target = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 1)
    opts = asmc.DriverOptions()
    opts.n_particles = 32
    opts.rounds = 2
    opts.seed = 5
    rounds = asmc.run_ssmc(target, asmc.Kernel(), opts)
    assert [r.round for r in rounds] == [1, 2]
    assert rounds[1].report.n_particles == 46
    assert rounds[1].report.schedule.steps() == 2
    assert math.isfinite(rounds[1].barrier.total())


# ---- the drop-in API reproduces the reference bit-for-bit-ish --------------
def test_api_run_sais_matches_reference_library():
    ref = oracle.load("ref", abi.RNG_XOSHIRO) if oracle.available("ref") else oracle.load("restate")
    target = asmc.GaussianShiftTarget(0.0, 1.0, 1.0, 10)
    k = asmc.Kernel()
    k.kind = asmc.KernelKind.rwmh_cycle
    opts = asmc.DriverOptions()
    opts.n_particles = 2000
    opts.rounds = 4
    opts.seed = 7
    rounds = asmc.run_sais(target, k, opts)
    want = ref.run_rounds(abi.gaussian_shift(0.0, 1.0, 1.0, 10), abi.kernel(abi.KERNEL_RWMH),
                          abi.MODE_SAIS, 2000, 4, seed=7, max_steps=5)
    for i, r in enumerate(rounds):
        assert r.report.n_particles == int(want["n_particles"][i])
        assert abs(r.report.log_z_hat - want["log_z_hat"][i]) < 1e-9
        T = r.report.schedule.steps()
        assert np.max(np.abs(np.array(r.report.schedule.betas) - want["betas"][i][: T + 1])) < 1e-9


# ---- closed-form log Z (north_star: within Monte-Carlo error) --------------
def test_config1_sais_log_z_within_mc_error():
    """Config 1: SAIS, d=10 Gaussian shift (exact log Z(1) = 0), RWMH, N1=2^14, 4 rounds."""
    for rng, prec in ((abi.RNG_XOSHIRO, F64), (PH, F32)):
        r = capi.run_rounds(abi.gaussian_shift(0.0, 1.0, 1.0, 10), abi.kernel(abi.KERNEL_RWMH),
                            abi.MODE_SAIS, 1 << 14, 4, seed=1, exec_=abi.execopts(rng, prec))
        assert list(r["n_particles"]) == [16384, 23171, 32769, 46343]
        assert list(r["steps"]) == [1, 2, 3, 5]
        assert abs(r["log_z_hat"][-1]) < 0.2, r["log_z_hat"]


def test_scale_gaussian_log_z_and_barrier():
    """Config-2 family at d=64 with enough steps: log Z-hat ~ 0, Lambda-hat ~ sqrt(d/2) log 4."""
    d = 64
    tg = abi.scale_gaussian(1.0, 2.0, d)
    betas = np.linspace(0.0, 1.0, 257)
    r = capi.run_sais_single(tg, abi.kernel(abi.KERNEL_IDEALIZED), betas, 1 << 16, seed=2, round=1,
                             exec_=abi.execopts(PH, F32))
    assert abs(r["log_z_hat"]) < 0.05
    lam = capi.barrier_estimate(r["log_g0"], r["log_g1"], r["log_g2"], betas)
    assert abs(lam[-1] - math.sqrt(d / 2) * math.log(4.0)) < 0.05 * lam[-1]


def test_fp32_unbiased_over_seeds():
    """mean of Z-hat over seeds is 1 within 3 standard errors (test_engine.cpp:166-185)."""
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 1)
    betas = np.linspace(0, 1, 17)
    for policy in (abi.POLICY_NEVER, abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS):
        z = np.array([math.exp(capi.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, 256, policy=policy,
                                            seed=1000 + s, exec_=abi.execopts(PH, F32))["log_z_hat"])
                      for s in range(600)])
        assert abs(z.mean() - 1.0) <= 3.0 * z.std(ddof=1) / math.sqrt(len(z)), policy


# ---- GPU-count invariance (virtual shards) ---------------------------------
def test_chunk_partials_are_shard_invariant():
    tg = abi.scale_gaussian(1.0, 2.0, 100)
    k = abi.kernel(abi.KERNEL_RWMH)
    betas = np.array([0.0, 0.3, 0.7, 1.0])
    n = 2 * abi.FOLD_CHUNK + 12345
    ex = abi.execopts(PH, F32)
    whole = capi.sais_partials(tg, k, betas, n, 0, n, seed=4, round=2, exec_=ex)
    cut = abi.FOLD_CHUNK
    split = np.concatenate([capi.sais_partials(tg, k, betas, n, 0, cut, seed=4, round=2, exec_=ex),
                            capi.sais_partials(tg, k, betas, n, cut, n, seed=4, round=2, exec_=ex)])
    assert whole.shape == split.shape and np.array_equal(whole.view(np.uint64), split.view(np.uint64))
    a = capi.fold_partials(split, n)
    b = capi.run_sais_single(tg, k, betas, n, seed=4, round=2, exec_=ex)
    for key in ("log_g0", "log_g1", "log_g2"):
        assert np.array_equal(a[key], b[key]), key
    assert a["log_z_hat"] == b["log_z_hat"]


# ---- SSMC on the device ----------------------------------------------------
@pytest.mark.parametrize("policy", [abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS])
def test_ssmc_fp64_philox_matches_restatement(policy):
    rs = oracle.load("restate", PH)
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 3)
    betas = np.linspace(0, 1, 11)
    a = rs.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, 3000, policy=policy, seed=8, round=1)
    b = capi.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, 3000, policy=policy, seed=8, round=1,
                     exec_=abi.execopts(PH, F64))
    assert a["resample_times"] == b["resample_times"]
    for key in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
        x, y = a[key][1:], b[key][1:]  # slot 0 is -inf / N by definition
        assert np.max(np.abs(x - y) / np.maximum(1, np.abs(x))) < 1e-10, key


@pytest.mark.parametrize("lanes", [1, 4, 32])
def test_ssmc_fp32_lanes_close_to_reference(lanes):
    ref = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 12)
    betas = np.linspace(0, 1, 9)
    a = ref.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, 4000, policy=abi.POLICY_ADAPTIVE_ESS,
                    seed=5, round=1)
    b = capi.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, 4000, policy=abi.POLICY_ADAPTIVE_ESS,
                     seed=5, round=1, exec_=abi.execopts(PH, F32, lanes=lanes))
    assert a["resample_times"] == b["resample_times"]
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 0.02


def test_sharded_round_loop_matches_device_round_loop():
    """distributed.run_sais (chunk partials + fold + device schedule, the multi-GPU
    path) at one rank reproduces asmc_run_rounds bit for bit."""
    from paper_2408_12057_b200 import distributed
    tg = abi.scale_gaussian(1.0, 2.0, 200)
    k = abi.kernel(abi.KERNEL_RWMH)
    ex = abi.execopts(PH, F32)
    n1 = abi.FOLD_CHUNK + 999
    a = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, 3, seed=6, exec_=ex)
    b = distributed.run_sais(tg, k, n1, 3, 6, ex, 0, 1)
    for r in range(3):
        T = int(a["steps"][r])
        assert b["steps"][r] == T and b["n_particles"][r] == int(a["n_particles"][r])
        assert np.array_equal(np.asarray(b["betas"][r]), a["betas"][r][: T + 1])
        assert np.array_equal(np.asarray(b["log_g1"][r]), a["log_g1"][r][: T + 1])
        assert b["log_z_hat"][r] == a["log_z_hat"][r]


@pytest.mark.parametrize("width", ["mix100", "scale300"])
def test_smc_step_mode_wide_targets_close_to_reference(width):
    """SMC step mode (state loaded from / stored to HBM every step, dual rows, early
    rejection for the scale family) at widths with several quad-iterations per lane."""
    ref = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100) if width == "mix100" else abi.scale_gaussian(1.0, 2.0, 300)
    k = abi.kernel(abi.KERNEL_RWMH, (0.05, 0.2, 1.0), 1)
    betas = np.linspace(0, 1, 9)
    a = ref.run_smc(tg, k, betas, 2000, policy=abi.POLICY_NEVER, seed=5, round=1)
    b = capi.run_smc(tg, k, betas, 2000, policy=abi.POLICY_NEVER, seed=5, round=1, exec_=abi.execopts(PH, F32))
    assert np.max(np.abs(a["log_g1"][1:] - b["log_g1"][1:]) / np.abs(a["log_g1"][1:]).clip(1)) < 1e-3
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 0.05 * max(1.0, abs(a["log_z_hat"]))
