"""GPU: systematic resampling with the reference's sequential CDF (csrc/refcdf.cu).

The reference (proj/src/engine.cpp:61-80) walks a CDF built by N dependent fp64 adds
of std::exp terms after a sequential LogAccumulator (logsum.hpp:97-101).  The device
builds the same CDF in parallel (binade-segmented integer scan + exact replay of the
few blocks that change binade, tie or rescale).  Bars:
  * exp: the device's gexp equals the host libm bit for bit;
  * CDF for a given l1: every cum_j bit-equal to the sequential chain;
  * l1: equal to the reference's, except where glibc's 0.52-ulp log misrounds sum
    (then 1 ulp; the device's log is correctly rounded) -- counted, never > 1 ulp;
  * ancestors for given log-weights and u: equal to the unmodified reference's
    systematic_resample (oracle/_ref/libasmc_ref.so), 0 mismatches, up to N = 2^22.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU parity tests must run on the B200 box")


def ulps(a, b):
    ia = np.asarray([a], np.float64).view(np.int64)[0]
    ib = np.asarray([b], np.float64).view(np.int64)[0]
    return abs(int(ia) - int(ib))


def weight_sets(g):
    """Log-weight families that stress every path of the exact scan."""
    yield "normal1", g.normal(0, 1, 100_000)
    yield "normal3", g.normal(0, 3, 300_001)
    yield "normal30", g.normal(0, 30, 65_537)   # few dominant particles: many crossings early
    lw = g.normal(0, 2, 50_000)
    lw[g.integers(0, len(lw), 5000)] = -np.inf  # -inf entries: no-ops in both chains
    yield "with_neginf", lw
    yield "increasing", np.linspace(-50, 50, 70_000)  # running max changes at every particle
    yield "decreasing", np.linspace(50, -50, 70_000)
    yield "constant", np.zeros(123_457)            # ties everywhere (equal terms)
    yield "tiny_head", np.concatenate([np.full(1000, -740.0), g.normal(0, 1, 20_000)])  # subnormal start
    yield "huge_spread", np.concatenate([g.normal(-700, 5, 30_000), [0.0], g.normal(-20, 5, 30_000)])
    for n in (1, 2, 3, 255, 256, 257, 511, 1025):
        yield f"n{n}", g.normal(0, 3, n)
    yield "laplace", g.laplace(0, 4, 200_000)
    lw = np.full(300_000, -800.0)
    lw[123_457] = 0.0  # one particle carries all the mass: every slot is its (heavy-run path)
    yield "one_heavy", lw
    lw = g.normal(0, 1, 250_000)
    lw[[17, 99_999, 200_003]] = 40.0  # three heavy ancestors
    yield "three_heavy", lw


def test_gexp_bit_exact_vs_host_libm():
    rs = oracle.load("restate")
    g = np.random.default_rng(11)
    x = np.concatenate([-745.2 * g.random(1 << 20), -40 * g.random(1 << 20), -g.random(1 << 18),
                        1420 * g.random(1 << 18) - 720.0,
                        [0.0, -0.0, -np.inf, np.inf, 709.9, -1e9, float.fromhex("0x1p-54")]])
    dev = capi.exact_math(0, x)
    ref = rs.libm(0, x)
    bad = np.flatnonzero(dev.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, (bad.size, x[bad[:5]], dev[bad[:5]], ref[bad[:5]])


def test_crlog_device_vs_glibc():
    rs = oracle.load("restate")
    y = 1.0 + np.random.default_rng(12).random(1 << 20) * 4194303.0
    dev = capi.exact_math(1, y)
    ref = rs.libm(1, y)
    d = np.abs(dev.view(np.int64) - ref.view(np.int64))
    assert d.max() <= 1
    assert np.mean(d > 0) < 2e-3  # glibc's log misrounds ~5e-4 of arguments


def test_cdf_and_l1_bit_exact():
    rs = oracle.load("restate")
    g = np.random.default_rng(5)
    l1_off = 0
    for name, lw in weight_sets(g):
        cum, l1 = capi.resample_cdf(lw)
        ref_cum, ref_l1 = rs.resample_cdf(lw)
        assert ulps(l1, ref_l1) <= 1, (name, l1, ref_l1)
        l1_off += l1 != ref_l1
        want = rs.cdf_given_l1(lw, l1)  # the reference chain of adds for the device's l1
        bad = np.flatnonzero(cum.view(np.uint64) != want.view(np.uint64))
        assert bad.size == 0, (name, bad.size, bad[:5], cum[bad[:3]], want[bad[:3]])
        if l1 == ref_l1:
            assert np.array_equal(cum.view(np.uint64), ref_cum.view(np.uint64)), name
    assert l1_off <= 2, l1_off


def test_logsumexp_matches_reference_logsumexp():
    rs = oracle.load("restate")
    g = np.random.default_rng(6)
    for name, lw in weight_sets(g):
        _, ref_l1 = rs.resample_cdf(lw)
        assert ulps(capi.logsumexp(lw), ref_l1) <= 1, name
    assert capi.logsumexp([-np.inf, -np.inf]) == -np.inf
    assert capi.logsumexp([]) == -np.inf


@pytest.mark.skipif(not oracle.available("ref", abi.RNG_XOSHIRO), reason="reference not built")
@pytest.mark.parametrize("sigma", [1.0, 3.0, 10.0])
def test_ancestors_zero_mismatch_vs_reference_at_2_22(sigma):
    """The done-bar: N = 2^22 ancestors from the unmodified reference's
    systematic_resample on the same log-weights and key (same u), 0 mismatches."""
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    n = 1 << 22
    lw = np.random.default_rng(int(sigma * 10)).normal(0, sigma, n)
    key = (9, 2, 0, 5, 2)
    u = ref.rng_uniform(key, 1)[0]
    a = ref.systematic_resample(lw, key)
    b = capi.systematic_resample(lw, u)
    assert int(np.sum(a != b)) == 0


@pytest.mark.skipif(not oracle.available("ref", abi.RNG_XOSHIRO), reason="reference not built")
def test_ancestors_vs_reference_every_family():
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    g = np.random.default_rng(8)
    for i, (name, lw) in enumerate(weight_sets(g)):
        key = (i, 1, 0, 3, 2)
        u = ref.rng_uniform(key, 1)[0]
        assert (ref.systematic_resample(lw, key) == capi.systematic_resample(lw, u)).all(), name


def test_degenerate_all_neginf_raises():
    with pytest.raises(capi.AsmcError) as e:
        capi.systematic_resample([-np.inf] * 300, 0.5)
    assert e.value.code == abi.ERR_DEGENERATE


@pytest.mark.skipif(not oracle.available("ref", abi.RNG_XOSHIRO), reason="reference not built")
def test_run_smc_fp64_matches_reference_at_scale():
    """End to end at a size where a blocked CDF would have flipped ancestors
    (~40 per event at 2^22; here 2^17 particles, always resampling): the device's
    reference mode reproduces the unmodified reference's run_smc statistics."""
    ref = oracle.load("ref", abi.RNG_XOSHIRO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
    betas = np.linspace(0, 1, 6)
    n = 1 << 17
    a = ref.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, n, policy=abi.POLICY_ALWAYS, seed=3, round=1,
                    workers=8)
    b = capi.run_smc(tg, abi.kernel(abi.KERNEL_RWMH), betas, n, policy=abi.POLICY_ALWAYS, seed=3, round=1,
                     exec_=abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64))
    for k in ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z"):
        x, y = np.asarray(a[k][1:]), np.asarray(b[k][1:])
        assert np.max(np.abs(x - y) / np.maximum(1, np.abs(x))) < 1e-10, k


def test_ancestors_on_exact_slot_ties():
    """Equal log-weights at power-of-two N with u = 0 put CDF values on (or within an ulp of)
    the slot positions (m + u) / N, where the ancestor pass's multiply-by-reciprocal filter
    must defer to the reference's division: the same ancestors as the rule (restatement)."""
    rs = oracle.load("restate")
    g = np.random.default_rng(5)
    cases = [np.zeros(1 << 16), np.zeros((1 << 14) * 3 + 1), np.full(1 << 18, -3.0),
             np.repeat(g.normal(0, 1, 1 << 10), 64)]
    for lw in cases:
        for u in (0.0, 0.5, 0.25, 1.0 - 2.0 ** -53):
            assert (capi.systematic_resample(lw, u) == rs.systematic_resample_u(lw, u)).all(), (len(lw), u)
