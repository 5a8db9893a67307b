"""The oracle (oracle/restate.c) pinned to the reference.

1. Bit-exact against tests/golden/reference_golden.json, produced from the
   UNMODIFIED reference (oracle/_ref) by tests/golden/make_golden.py.
2. Bit-exact against the live reference library when it is built here.
3. The reference's own known-answer tests for this path, restated
   (proj/tests/test_engine.cpp, test_schedule.cpp, test_drivers.cpp, test_rng.cpp).
CPU only.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "reference_golden.json")))

TARGETS = {"gauss10": abi.gaussian_shift(0.0, 1.0, 1.0, 10),
           "gauss1": abi.gaussian_shift(0.0, 1.0, 1.0, 1),
           "mix5": abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 5),
           "scale7": abi.scale_gaussian(1.0, 2.0, 7)}
KERNELS = {"rwmh": abi.kernel(abi.KERNEL_RWMH), "ideal": abi.kernel(abi.KERNEL_IDEALIZED),
           "ident": abi.kernel(abi.KERNEL_IDENTITY)}
RNGS = {"xoshiro": abi.RNG_XOSHIRO, "philox": abi.RNG_PHILOX}


def unhex(a):
    return np.array([float.fromhex(v) for v in a])


def same_bits(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and bool(np.all(a.view(np.uint64) == b.view(np.uint64)))


# ------------------------------------------------------------- golden pins --
@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_restatement_rng_matches_golden(tag):
    rs = oracle.load("restate", RNGS[tag])
    for rec in GOLD[tag]["rng"]:
        k = rec["key"]
        assert [str(int(v)) for v in rs.rng_u64(k, 64)] == rec["u64"]
        assert same_bits(rs.rng_uniform(k, 16), unhex(rec["uniform"]))
        assert same_bits(rs.rng_normal(k, 33), unhex(rec["normal"]))


@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_restatement_runs_match_golden(tag):
    rs = oracle.load("restate", RNGS[tag])
    for rec in GOLD[tag]["runs"]:
        tg, k = TARGETS[rec["target"]], KERNELS[rec["kernel"]]
        betas = unhex(rec["betas"])
        s = rs.run_sais_single(tg, k, betas, rec["n"], seed=rec["seed"], round=rec["round"])
        for key in ("log_g0", "log_g1", "log_g2"):
            assert same_bits(s[key], unhex(rec["sais"][key])), (tag, rec["target"], rec["kernel"], key)
        assert s["log_z_hat"] == float.fromhex(rec["sais_log_z"])
        assert s["elbo_hat"] == float.fromhex(rec["sais_elbo"])
        for pol in range(4):
            g = rec[f"smc_{pol}"]
            m = rs.run_smc(tg, k, betas, 300, policy=pol, rho=0.6, seed=9, round=2)
            for key in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
                assert same_bits(m[key], unhex(g[key])), (tag, rec["target"], pol, key)
            assert m["resample_times"] == g["resample_times"]
            assert m["log_z_hat"] == float.fromhex(g["log_z"])
            assert m["elbo_hat"] == float.fromhex(g["elbo"])
        x, lw, _ = rs.trajectory(tg, k, betas, 5, 1, 123)
        assert same_bits(x, unhex(rec["traj_p123"]["x"]).reshape(x.shape))
        assert same_bits(lw, unhex(rec["traj_p123"]["lw"]))


@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_restatement_round_loop_matches_golden(tag):
    rs = oracle.load("restate", RNGS[tag])
    for rec in GOLD[tag]["rounds"]:
        r = rs.run_rounds(TARGETS["gauss1"], KERNELS["rwmh"], rec["mode"], 64, 4, seed=11, max_steps=5)
        assert [int(v) for v in r["n_particles"]] == rec["n"]
        assert [int(v) for v in r["steps"]] == rec["steps"]
        assert same_bits(r["betas"].ravel(), unhex(rec["betas"]))
        assert same_bits(r["lambda_"].ravel(), unhex(rec["lambda"]))
        assert same_bits(r["log_z_hat"], unhex(rec["log_z"]))


def test_restatement_schedule_and_budget_match_golden():
    rs = oracle.load("restate")
    for rec in GOLD["schedule"]:
        lam, beta = unhex(rec["lambda"]), unhex(rec["beta"])
        assert same_bits(rs.generate_schedule(lam, beta, rec["t_new"]), unhex(rec["out"]))
        assert same_bits(rs.local_barrier(lam, beta), unhex(rec["local"]))
    for rec in GOLD["budget"]:
        assert list(rs.budget(*rec["args"])) == rec["out"]


def test_restatement_systematic_matches_golden():
    rs = oracle.load("restate")
    for rec in GOLD["systematic"]:
        a = rs.systematic_resample(unhex(rec["log_w"]), rec["key"])
        assert [int(v) for v in a] == rec["ancestors"]


# ------------------------------------------------------- live reference ----
@pytest.mark.skipif(not oracle.available("ref"), reason="reference not built here")
@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_restatement_bit_exact_vs_live_reference(tag):
    ref, rs = oracle.load("ref", RNGS[tag]), oracle.load("restate", RNGS[tag])
    g = np.random.default_rng(7)
    for _ in range(6):
        tname = ["gauss10", "mix5", "scale7"][int(g.integers(3))]
        kname = ["rwmh", "ident"][int(g.integers(2))]
        tg, k = TARGETS[tname], abi.kernel(abi.KERNEL_RWMH, tuple(g.uniform(0.05, 3.0, 2)), 2) \
            if kname == "rwmh" else KERNELS[kname]
        T = int(g.integers(1, 9))
        betas = np.concatenate([[0.0], np.sort(g.uniform(0, 1, T - 1)), [1.0]])
        n, seed, pol = int(g.integers(1, 900)), int(g.integers(1 << 40)), int(g.integers(4))
        a = ref.run_smc(tg, k, betas, n, policy=pol, rho=0.7, seed=seed, round=3)
        b = rs.run_smc(tg, k, betas, n, policy=pol, rho=0.7, seed=seed, round=3)
        for key in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
            assert same_bits(a[key], b[key]), (tname, key)
        lw = g.normal(0, 5, n)
        key = (seed, 1, 0, 3, 2)
        assert (ref.systematic_resample(lw, key) == rs.systematic_resample(lw, key)).all()


# ------------------------------- reference known-answer tests, restated ----
def test_ess_closed_forms():  # test_engine.cpp:71-83
    rs = oracle.load("restate")
    assert abs(rs.ess(np.full(8, -1.3)) - 8.0) < 1e-12 * 8
    assert abs(rs.ess([0.0, -np.inf, -np.inf, -np.inf]) - 1.0) < 1e-12
    assert abs(rs.ess([math.log(2.0), 0.0, 0.0]) - 16.0 / 6.0) < 1e-12 * 3
    with pytest.raises(oracle.OracleError) as e:
        rs.ess([-np.inf, -np.inf])
    assert e.value.code == abi.ERR_DEGENERATE


def test_systematic_stratified():  # test_engine.cpp:85-96
    rs = oracle.load("restate")
    key = (3, 0, 0, 1, 2)
    assert list(rs.systematic_resample([math.log(0.5)] * 2, key)) == [0, 1]
    assert all(a == 1 for a in rs.systematic_resample([-np.inf, 0.0, -np.inf], key))


def test_systematic_multiplicity_within_one():  # test_engine.cpp:98-126
    rs = oracle.load("restate")
    n = 100
    lw = np.log(np.arange(1, n + 1, dtype=float))
    expect = n * np.arange(1, n + 1) / np.sum(np.arange(1, n + 1))
    for s in range(300):
        a = rs.systematic_resample(lw, (s, 0, 0, 1, 2))
        mult = np.bincount(a, minlength=n)
        assert np.all(np.abs(mult - expect) < 1.0)
    for u in np.linspace(0, 1, 37, endpoint=False):
        mult = np.bincount(rs.systematic_resample_u(lw, u), minlength=n)
        assert np.all(np.abs(mult - expect) < 1.0)


def test_resample_given_u_and_cdf_match_keyed_reference():
    """ora_systematic_resample_u / ora_resample_cdf (the hooks the GPU parity tests
    compare the device with) are engine.cpp:61-80 itself: same ancestors as the keyed
    call, and the search rule over the exposed CDF gives them again."""
    rs = oracle.load("restate")
    g = np.random.default_rng(0)
    for n in (1, 7, 256, 1000, 65537):
        for trial in range(3):
            lw = g.normal(0, 3, n)
            lw[g.integers(0, n, n // 10)] = -np.inf
            if np.all(lw == -np.inf):
                lw[0] = 0.0
            key = (trial, 0, 0, 1, 2)
            u = rs.rng_uniform(key, 1)[0]
            a = rs.systematic_resample(lw, key)
            assert (a == rs.systematic_resample_u(lw, u)).all()
            cum, l1 = rs.resample_cdf(lw)
            pos = (np.arange(n) + u) / n
            b = np.minimum(np.searchsorted(cum, pos, side="left"), n - 1)
            assert (a == b).all()
            assert np.all(np.diff(cum) >= 0)


def test_libm_hook_is_the_host_libm():
    rs = oracle.load("restate")
    xs = -np.random.default_rng(1).uniform(0, 745, 3000)
    assert np.array_equal(rs.libm(0, xs), np.array([math.exp(x) for x in xs]))
    ys = np.random.default_rng(2).uniform(1, 1e6, 3000)
    assert np.array_equal(rs.libm(1, ys), np.array([math.log(y) for y in ys]))


def test_barrier_sums():  # test_schedule.cpp:66-79
    rs = oracle.load("restate")
    d1, d2 = 0.09, 0.25
    g0 = [-np.inf, 0.0, 0.0]
    g1 = [-np.inf, 0.0, 0.0]
    g2 = [-np.inf, d1, d2]
    lam = rs.barrier_estimate(g0, g1, g2, [0.0, 0.4, 1.0])
    assert lam[0] == 0.0 and abs(lam[1] - 0.3) < 1e-12 and abs(lam[2] - 0.8) < 1e-12


def test_generate_schedule_cases():  # test_schedule.cpp:96-162
    rs = oracle.load("restate")
    out = rs.generate_schedule([0.0, 0.7, 1.4, 2.1], [0.0, 0.1, 0.55, 1.0], 3)
    assert np.max(np.abs(out - [0.0, 0.1, 0.55, 1.0])) < 1e-12
    assert list(rs.generate_schedule([0.0, 1.0, 1.5], [0.0, 0.3, 1.0], 1)) == [0.0, 1.0]
    knots = 128
    beta = np.arange(knots + 1) / knots
    out = rs.generate_schedule(beta ** 2, beta, 16)
    assert np.max(np.abs(out - np.sqrt(np.arange(17) / 16))) < 0.01
    out = rs.generate_schedule([0.0, 0.5, 0.5, 1.0], [0.0, 0.3, 0.6, 1.0], 2)
    assert abs(out[1] - 0.6) < 1e-12
    out = rs.generate_schedule([0.0, 0.0, 0.0], [0.0, 0.4, 1.0], 4)
    assert np.max(np.abs(out - np.arange(5) / 4)) < 1e-12
    for tn in (1, 2, 5, 9, 33):
        out = rs.generate_schedule([0.0, 1.0, 1.0, 1.0001, 3.0], [0.0, 0.2, 0.21, 0.8, 1.0], tn)
        assert np.all(np.diff(out) > 0) and out[0] == 0.0 and out[-1] == 1.0
    with pytest.raises(oracle.OracleError):
        rs.generate_schedule([0.1, 1.0], [0.0, 1.0], 3)


def test_local_barrier_slope():  # test_schedule.cpp:164-171
    rs = oracle.load("restate")
    lam = rs.local_barrier([0.0, 0.5, 1.0, 2.0], [0.0, 0.25, 0.5, 1.0])
    assert np.max(np.abs(lam - 2.0)) < 1e-10


def test_budget_growth():  # test_drivers.cpp:43-68
    rs = oracle.load("restate")
    big = 1 << 40
    assert rs.budget(16, 8, 1, big, abi.MODE_SSMC) == (23, 12)
    assert rs.budget(16, 8, 1, big, abi.MODE_SAIS) == (23, 12)
    assert rs.budget(64, 1, 1, big, abi.MODE_SSMC) == (91, 2)
    assert rs.budget(16, 8, 4, 23 * 4 * 8 - 1, abi.MODE_SSMC) == (16, 16)
    assert rs.budget(16, 8, 4, 23 * 4 * 8 - 1, abi.MODE_SAIS) == (23, 12)


def test_round_loop_growth():  # test_drivers.cpp:138-158
    rs = oracle.load("restate")
    r = rs.run_rounds(TARGETS["gauss1"], KERNELS["ideal"], abi.MODE_SSMC, 16, 4, seed=11, max_steps=8)
    assert list(r["n_particles"]) == [16, 23, 33, 47]
    assert list(r["steps"]) == [1, 2, 3, 5]
    assert list(r["kernel_applications"]) == [16, 46, 99, 235]
    capped = rs.run_rounds(TARGETS["gauss1"], KERNELS["ideal"], abi.MODE_SSMC, 16, 4, seed=11,
                           memory_cap=16 * 8, max_steps=8)
    assert list(capped["n_particles"]) == [16] * 4 and list(capped["steps"]) == [1, 2, 4, 8]


@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_sais_bit_identical_to_smc_never(tag):  # test_drivers.cpp:70-99, acceptance crit. 7
    rs = oracle.load("restate", RNGS[tag])
    betas = np.linspace(0, 1, 9)
    for n in (64, 1 << 12):
        a = rs.run_smc(TARGETS["gauss1"], KERNELS["ideal"], betas, n, policy=abi.POLICY_NEVER, seed=42, round=1)
        b = rs.run_sais_single(TARGETS["gauss1"], KERNELS["ideal"], betas, n, seed=42, round=1)
        assert a["log_z_hat"] == b["log_z_hat"] and a["elbo_hat"] == b["elbo_hat"]
        for k in ("log_g0", "log_g1", "log_g2", "cum_log_z"):
            assert same_bits(a[k], b[k])


def test_zero_shift_exact_under_every_policy():  # test_engine.cpp "zero shift"
    rs = oracle.load("restate")
    flat = abi.gaussian_shift(0.0, 0.0, 1.0, 1)
    for pol in range(4):
        r = rs.run_smc(flat, KERNELS["ideal"], np.linspace(0, 1, 6), 32, policy=pol, seed=9)
        assert r["log_z_hat"] == 0.0 and r["elbo_hat"] == 0.0 and r["resample_times"][-1] == 5


def test_degenerate_weights_abort():  # test_engine.cpp:286-311 (SpreadTarget analogue)
    rs = oracle.load("restate")
    spread = abi.gaussian_shift(0.0, 1e6, 1.0, 1)
    with pytest.raises(oracle.OracleError) as e:
        rs.run_smc(spread, KERNELS["ident"], [0.0, 1.0], 2, policy=abi.POLICY_NEVER, seed=1)
    assert e.value.code == abi.ERR_DEGENERATE and "degenerate" in e.value.msg


# ------------------------- new kernel (no reference code): HMC in the oracle --
@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
@pytest.mark.parametrize("tname", ["gauss10", "mix5", "scale7"])
def test_hmc_oracle_log_z_unbiased_enough(tag, tname):
    """HMC leaves pi_beta invariant, so SAIS with HMC moves estimates log Z(1) = 0
    for these normalized families within Monte-Carlo error."""
    rs = oracle.load("restate", RNGS[tag])
    k = abi.kernel(abi.KERNEL_HMC, (0.05, 0.2), 1, leapfrog=8)
    r = rs.run_sais_single(TARGETS[tname], k, np.linspace(0, 1, 33), 1 << 13, seed=3, round=1)
    assert abs(r["log_z_hat"]) < 0.1, r["log_z_hat"]


def test_hmc_oracle_converges_to_pi_beta():
    """A long HMC chain at beta = 1 started from eta = N(0, 1) reaches pi_1 = N(2, 0.7^2)
    (stationarity of the new kernel; test_kernel.cpp:119-146 analogue)."""
    rs = oracle.load("restate")
    tg = abi.gaussian_shift(0.0, 2.0, 0.7, 1)
    k = abi.kernel(abi.KERNEL_HMC, (0.3,), 40, leapfrog=5)
    xs = np.array([rs.trajectory(tg, k, [0.0, 1.0], 13, 0, p)[0][1, 0] for p in range(3000)])
    se = 0.7 / math.sqrt(len(xs))
    assert abs(xs.mean() - 2.0) < 5 * se
    assert abs(xs.var() - 0.49) < 0.05


# ------------------------------------- streams (test_rng.cpp, both families) --
@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_stream_identity_and_sensitivity(tag):  # test_rng.cpp:15-34
    rs = oracle.load("restate", RNGS[tag])
    k = (42, 3, 17, 5, 1)
    assert (rs.rng_u64(k, 1000) == rs.rng_u64(k, 1000)).all()
    first = rs.rng_u64((7, 1, 2, 3, 0), 1)[0]
    for v in [(8, 1, 2, 3, 0), (7, 2, 2, 3, 0), (7, 1, 3, 3, 0), (7, 1, 2, 4, 0), (7, 1, 2, 3, 1)]:
        assert rs.rng_u64(v, 1)[0] != first


@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_stream_uniform_ks_and_normal_moments(tag):  # test_rng.cpp:52-84
    rs = oracle.load("restate", RNGS[tag])
    u = np.sort(rs.rng_uniform((2024, 0, 0, 0, 0), 100000))
    i = np.arange(len(u))
    d = max(np.max(np.abs(u - i / len(u))), np.max(np.abs(u - (i + 1) / len(u))))
    assert d < 1.63 / math.sqrt(len(u))
    x = rs.rng_normal((99, 0, 0, 0, 0), 200000)
    assert abs(x.mean()) < 0.01 and abs(np.mean(x ** 2) - 1) < 0.02
    assert abs(np.mean(x ** 3)) < 0.05 and abs(np.mean(x ** 4) - 3) < 0.1


@pytest.mark.parametrize("tag", ["xoshiro", "philox"])
def test_stream_first_outputs_rarely_collide(tag):  # test_rng.cpp:36-50 (10^5 keys)
    rs = oracle.load("restate", RNGS[tag])
    firsts = [int(rs.rng_u64((1, 1, p, t, 1), 1)[0]) for p in range(1000) for t in range(100)]
    assert len(set(firsts)) == len(firsts)
