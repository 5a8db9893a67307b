"""GPU parity: the B200 kernels (through the C-ABI) against the CPU oracle.

Oracles: oracle/_ref/libasmc_ref.so (the unmodified reference, keyed xoshiro),
oracle/_ref/libasmc_ref_philox.so (reference sources + Philox shadow header)
and oracle/_ref/liborarestate.so (plain-C restatement, pinned to both).

Tolerances (stated per BASELINE.json north_star):
  * integer / index work (RNG words, ancestors, schedule grids): bit-exact;
  * rng=xoshiro, precision=fp64 (reference arithmetic on device): 1e-12
    relative (libm last-ulp differences between CUDA and glibc only);
  * precision=fp32: per-particle x within 2e-4 absolute * scale for particles
    whose MH decisions all match; log Z / increment statistics within the
    tolerances written in each test.
"""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu

XO, PH = abi.RNG_XOSHIRO, abi.RNG_PHILOX
F64, F32 = abi.PREC_FP64, abi.PREC_FP32

RWMH = abi.kernel(abi.KERNEL_RWMH)
IDEAL = abi.kernel(abi.KERNEL_IDEALIZED)
IDENT = abi.kernel(abi.KERNEL_IDENTITY)


def targets():
    return [("gauss10", abi.gaussian_shift(0.0, 1.0, 1.0, 10)),
            ("mix5", abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 5)),
            ("scale7", abi.scale_gaussian(1.0, 2.0, 7)),
            ("gauss100", abi.gaussian_shift(0.0, 0.3, 1.0, 100)),
            # wide mixtures: several quad-iterations per lane (G = 4: d = 100; G = 32: d = 300),
            # the multi-segment MH sums of the shared-memory pass without early rejection
            ("mix100", abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)),
            ("mix300", abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 300)),
            ("scale300", abi.scale_gaussian(1.0, 2.0, 300))]


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):
        d = np.where(both_inf, 0.0, np.abs(a - b) / np.maximum(1.0, np.abs(b)))
    return float(np.max(d)) if d.size else 0.0


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU parity tests must run on the B200 box")


@pytest.mark.parametrize("rng", [XO, PH])
def test_rng_words_bit_exact(rng):
    ref = oracle.load("ref", rng)
    for key in [(42, 3, 17, 5, 1), (0, 0, 0, 0, 0), (7, 1, 123456789, 4, 2)]:
        assert (capi.rng_u64(rng, key, 257) == ref.rng_u64(key, 257)).all()
        assert (capi.rng_uniform(rng, key, 101) == ref.rng_uniform(key, 101)).all()


@pytest.mark.parametrize("rng", [XO, PH])
def test_rng_normals(rng):
    ref = oracle.load("ref", rng)
    key = (9, 2, 77, 3, 1)
    want = ref.rng_normal(key, 4000)
    got64 = capi.rng_normal(rng, key, 4000, F64)
    assert np.max(np.abs(got64 - want)) < 1e-13
    got32 = capi.rng_normal(rng, key, 4000, F32)
    assert np.max(np.abs(got32 - want) / np.maximum(1.0, np.abs(want))) < 3e-6


@pytest.mark.parametrize("name,tg", targets())
@pytest.mark.parametrize("kern", ["rwmh", "ideal", "ident"])
def test_trajectories_fp64_xoshiro(name, tg, kern):
    k = dict(rwmh=RWMH, ideal=IDEAL, ident=IDENT)[kern]
    if kern == "ideal" and tg.kind == abi.TARGET_MIXTURE:
        pytest.skip("mixture has no exact sampler")
    betas = np.linspace(0.0, 1.0, 6)
    ref = oracle.load("ref", XO)
    pids = [0, 1, 255, 256, 1000, 123457]
    x, lw = capi.trajectories(tg, k, betas, 5, 1, pids, abi.execopts(XO, F64))
    for i, p in enumerate(pids):
        rx, rlw, _ = ref.trajectory(tg, k, betas, 5, 1, p)
        assert np.max(np.abs(x[i] - rx)) < 1e-12, (name, kern, p)
        assert rel(lw[i], rlw) < 1e-12


@pytest.mark.parametrize("name,tg", targets())
def test_trajectories_fp32_philox(name, tg):
    betas = np.linspace(0.0, 1.0, 5)
    ref = oracle.load("ref", PH)
    pids = np.arange(64)
    for lanes in (1, 4, 32):
        if lanes == 1 and tg.dim > 16 or lanes == 4 and tg.dim > 128:
            continue
        x, lw = capi.trajectories(tg, RWMH, betas, 3, 2, pids, abi.execopts(PH, F32, lanes=lanes))
        ok = 0
        for i, p in enumerate(pids):
            rx, rlw, _ = ref.trajectory(tg, RWMH, betas, 3, 2, int(p))
            if np.max(np.abs(x[i] - rx)) < 2e-4 * max(1.0, np.max(np.abs(rx))):
                ok += 1
                assert abs(lw[i][-1] - rlw[-1]) < 1e-3 * max(1.0, abs(rlw[-1])), (name, lanes, p)
        # an MH decision flip diverges one trajectory; allow at most 1 of 64
        assert ok >= len(pids) - 1, (name, lanes, ok)


@pytest.mark.parametrize("name,tg", targets())
def test_sais_single_fp64_matches_reference(name, tg):
    betas = np.array([0.0, 0.1, 0.3, 0.6, 1.0])
    ref = oracle.load("ref", XO)
    for n in (1, 255, 700, 5000):
        a = ref.run_sais_single(tg, RWMH, betas, n, seed=7, round=1)
        b = capi.run_sais_single(tg, RWMH, betas, n, seed=7, round=1, exec_=abi.execopts(XO, F64))
        for k in ("log_g0", "log_g1", "log_g2", "cum_log_z"):
            assert rel(b[k], a[k]) < 1e-12, (name, n, k)
        assert rel(b["log_z_hat"], a["log_z_hat"]) < 1e-12
        assert rel(b["elbo_hat"], a["elbo_hat"]) < 1e-10
        assert b["resample_times"] == a["resample_times"]
        assert b["kernel_applications"] == a["kernel_applications"]


@pytest.mark.parametrize("policy", [abi.POLICY_NEVER, abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS,
                                    abi.POLICY_STABILIZED])
def test_run_smc_fp64_matches_reference(policy):
    ref = oracle.load("ref", XO)
    betas = np.linspace(0, 1, 9)
    for name, tg in targets()[:3]:
        a = ref.run_smc(tg, RWMH, betas, 777, policy=policy, rho=0.6, seed=11, round=2)
        b = capi.run_smc(tg, RWMH, betas, 777, policy=policy, rho=0.6, seed=11, round=2,
                         exec_=abi.execopts(XO, F64))
        assert b["resample_times"] == a["resample_times"], name
        for k in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
            assert rel(b[k], a[k]) < 1e-10, (name, k, b[k], a[k])
        assert (b["resampled"] == a["resampled"]).all()


def test_systematic_resample_bit_exact():
    """engine.cpp:61-80 for given log-weights and u: the device's ancestors equal the
    reference rule's (restatement, pinned to the reference in test_oracle.py)."""
    rs = oracle.load("restate")
    g = np.random.default_rng(0)
    for n in (1, 2, 255, 256, 257, 10000, 1 << 20):
        lw = g.normal(0, 3, n)
        for u in (0.0, 0.3, 0.999):
            dev = capi.systematic_resample(lw, u)
            assert (dev == rs.systematic_resample_u(lw, u)).all(), (n, u)


def test_schedule_bit_exact():
    ref = oracle.load("ref", XO)
    g = np.random.default_rng(1)
    cases = [([0.0, 0.7, 1.4, 2.1], [0.0, 0.1, 0.55, 1.0], 3),
             ([0.0, 0.5, 0.5, 1.0], [0.0, 0.3, 0.6, 1.0], 2),
             ([0.0, 1.0, 1.0, 1.0001, 3.0], [0.0, 0.2, 0.21, 0.8, 1.0], 33),
             ([0.0, 0.0, 0.0], [0.0, 0.4, 1.0], 4)]
    for _ in range(20):
        T = int(g.integers(2, 60))
        lam = np.concatenate([[0.0], np.cumsum(g.exponential(1.0, T))])
        beta = np.concatenate([[0.0], np.sort(g.uniform(0, 1, T - 1)), [1.0]])
        cases.append((lam, beta, int(g.integers(1, 100))))
    for lam, beta, tn in cases:
        a = ref.generate_schedule(lam, beta, tn)
        b = capi.generate_schedule(lam, beta, tn)
        assert (a == b).all()
        assert (ref.local_barrier(lam, beta) == capi.local_barrier(lam, beta)).all()


@pytest.mark.parametrize("mode", [abi.MODE_SAIS, abi.MODE_SSMC])
def test_rounds_fp64_match_reference(mode):
    ref = oracle.load("ref", XO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 3)
    b = capi.run_rounds(tg, RWMH, mode, 300, 5, seed=3, exec_=abi.execopts(XO, F64))
    a = ref.run_rounds(tg, RWMH, mode, 300, 5, seed=3, max_steps=b["betas"].shape[1] - 1)
    assert (a["n_particles"] == b["n_particles"]).all()
    assert (a["steps"] == b["steps"]).all()
    assert rel(b["log_z_hat"], a["log_z_hat"]) < 1e-9
    assert rel(b["betas"], a["betas"]) < 1e-9


def test_sais_fp32_philox_close_to_reference():
    ref = oracle.load("ref", PH)
    tg = abi.scale_gaussian(1.0, 2.0, 100)
    betas = np.linspace(0, 1, 6)
    a = ref.run_sais_single(tg, RWMH, betas, 4096, seed=1, round=1)
    b = capi.run_sais_single(tg, RWMH, betas, 4096, seed=1, round=1, exec_=abi.execopts(PH, F32))
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 2e-3 * max(1, abs(a["log_z_hat"]))


# ---- HMC (new kernel; the oracle restatement defines it: oracle/restate.c) --------------
HMC = abi.kernel(abi.KERNEL_HMC, (0.05, 0.2), 1, leapfrog=6)


@pytest.mark.parametrize("name,tg", targets())
def test_hmc_trajectories_fp64_match_oracle(name, tg):
    betas = np.linspace(0.0, 1.0, 5)
    for rng in (XO, PH):
        rs = oracle.load("restate", rng)
        pids = [0, 7, 300, 99999]
        x, lw = capi.trajectories(tg, HMC, betas, 4, 1, pids, abi.execopts(rng, F64))
        for i, p in enumerate(pids):
            rx, rlw, _ = rs.trajectory(tg, HMC, betas, 4, 1, p)
            assert np.max(np.abs(x[i] - rx)) < 1e-11, (name, rng, p)
            assert rel(lw[i], rlw) < 1e-11


@pytest.mark.parametrize("name,tg", targets())
def test_hmc_trajectories_fp32_close_to_oracle(name, tg):
    betas = np.linspace(0.0, 1.0, 5)
    rs = oracle.load("restate", PH)
    pids = np.arange(48)
    for lanes in (1, 4, 32):
        if lanes == 1 and tg.dim > 16:
            continue
        x, lw = capi.trajectories(tg, HMC, betas, 4, 1, pids, abi.execopts(PH, F32, lanes=lanes))
        ok = 0
        for i, p in enumerate(pids):
            rx, rlw, _ = rs.trajectory(tg, HMC, betas, 4, 1, int(p))
            if np.max(np.abs(x[i] - rx)) < 5e-4 * max(1.0, np.max(np.abs(rx))):
                ok += 1
        assert ok >= len(pids) - 1, (name, lanes, ok)


def test_hmc_sais_log_z_on_device():
    for tg in (abi.scale_gaussian(1.0, 2.0, 100), abi.gaussian_shift(0.0, 0.5, 1.0, 100)):
        r = capi.run_sais_single(tg, abi.kernel(abi.KERNEL_HMC, (0.05, 0.15), 1, leapfrog=10),
                                 np.linspace(0, 1, 65), 1 << 15, seed=9, round=1,
                                 exec_=abi.execopts(PH, F32))
        assert abs(r["log_z_hat"]) < 0.1, r["log_z_hat"]
