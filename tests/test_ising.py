"""Config 5: relaxed Ising model on an L x L torus with HMC (ASMC_TARGET_ISING).

Oracles: the unmodified reference engine running the Ising plugin of
oracle/ref_harness.cpp (RWMH / identity: the reference has no HMC), the
restatement's identical plugin and HMC (oracle/restate.c), and the closed form
Z(1) = (2 pi)^{n/2} |A|^{-1/2} e^{c n/2} Z_Ising(K) with Kaufman's exact finite-torus
Z_Ising (paper_2408_12057_b200/exact.py), itself pinned here against brute-force
enumeration.  Device tolerance: fp32 lattice energies with fp64 block sums agree
with the fp64 oracle to ~3e-8 relative in the per-step log-moments (1e-6 asserted).
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi, exact

PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
KC = exact.K_CRITICAL


def brute_log_z(m, n, K):
    N = m * n
    idx = np.arange(2 ** N, dtype=np.int64)
    s = (((idx[:, None] >> np.arange(N)) & 1) * 2 - 1).reshape(-1, m, n)
    E = (s * np.roll(s, 1, 1)).sum((1, 2)) + (s * np.roll(s, 1, 2)).sum((1, 2))
    a = K * E
    return a.max() + math.log(np.exp(a - a.max()).sum())


@pytest.mark.parametrize("m,n", [(3, 3), (4, 4), (3, 4), (4, 5)])
@pytest.mark.parametrize("K", [0.1, KC, 1.0])
def test_kaufman_matches_enumeration(m, n, K):
    assert abs(exact.ising_log_z(n, K, M=m) - brute_log_z(m, n, K)) < 1e-12 * abs(brute_log_z(m, n, K)) + 1e-12


def test_relaxed_log_z_matches_direct_sum():
    """Z(1) = sum_s exp(s'As/2) (2 pi)^{n/2} |A|^{-1/2} with a dense A (L = 3 and 4)."""
    for L, K, delta in ((3, 0.3, 1.0), (4, KC, 0.5)):
        n = L * L
        A = np.zeros((n, n))
        for a in range(L):
            for b in range(L):
                i = a * L + b
                A[i, i] = delta + 4 * K
                for j in (((a + 1) % L) * L + b, ((a - 1) % L) * L + b, a * L + (b + 1) % L, a * L + (b - 1) % L):
                    A[i, j] += K
        s = np.array(list(itertools.product([-1.0, 1.0], repeat=n)))
        q = 0.5 * np.einsum("ki,ij,kj->k", s, A, s)
        direct = q.max() + math.log(np.exp(q - q.max()).sum()) + 0.5 * n * math.log(2 * math.pi) \
            - 0.5 * np.linalg.slogdet(A)[1]
        assert abs(direct - exact.ising_relaxed_log_z(L, K, delta)) < 1e-9 * abs(direct)


def test_restatement_plugin_matches_reference_plugin():
    if not oracle.available("ref", PH):
        pytest.skip("reference not built here")
    tg = abi.ising(4, KC, 1.0, 1.0)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.3), 1)
    betas = np.linspace(0, 1, 6)
    a = oracle.load("ref", PH).run_smc(tg, k, betas, 256, policy=abi.POLICY_ALWAYS, seed=4)
    b = oracle.load("restate", PH).run_smc(tg, k, betas, 256, policy=abi.POLICY_ALWAYS, seed=4)
    assert a["log_z_hat"] == b["log_z_hat"] and np.array_equal(a["log_g2"], b["log_g2"])


def test_restatement_hmc_estimates_exact_log_z():
    tg = abi.ising(4, 0.3, 1.0, 1.0)
    k = abi.kernel(abi.KERNEL_HMC, (0.3,), 1, leapfrog=8)
    r = oracle.load("restate", PH).run_sais_single(tg, k, np.linspace(0, 1, 41), 2048, seed=1, round=1)
    assert abs(r["log_z_hat"] - exact.ising_relaxed_log_z(4, 0.3, 1.0)) < 0.1


@pytest.mark.gpu
@pytest.mark.parametrize("kname", ["identity", "rwmh", "hmc"])
@pytest.mark.parametrize("L,n", [(8, 512), (32, 256), (64, 64)])  # row kernel (8), 4x4 tiles (32, 64)
def test_ising_device_matches_oracle(kname, L, n):
    tg = abi.ising(L, KC, 1.0, 1.0)
    k = {"identity": abi.kernel(abi.KERNEL_IDENTITY),
         "rwmh": abi.kernel(abi.KERNEL_RWMH, (0.1, 0.3), 1),
         "hmc": abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=6)}[kname]
    o = oracle.load("restate", PH) if kname == "hmc" or not oracle.available("ref", PH) else oracle.load("ref", PH)
    betas = np.linspace(0, 1, 9)
    a = o.run_sais_single(tg, k, betas, n, seed=2, round=1)
    b = capi.run_sais_single(tg, k, betas, n, seed=2, round=1, exec_=abi.execopts(PH, F32))
    for g in ("log_g0", "log_g1", "log_g2"):
        assert np.max(np.abs(a[g][1:] - b[g][1:]) / np.abs(a[g][1:]).clip(1)) < 1e-6, g
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 1e-6 * abs(a["log_z_hat"])


@pytest.mark.gpu
def test_ising_ssmc_matches_oracle_and_exact():
    tg = abi.ising(16, KC, 1.0, 1.0)
    ex = abi.execopts(PH, F32)
    # SSMC machinery (weight kernel, CDF, gather of lattice rows + cached V) against the
    # reference engine: identity kernel, so no MH decision can flip between fp32 and fp64
    k0 = abi.kernel(abi.KERNEL_IDENTITY)
    betas = np.linspace(0, 1, 17)
    o = oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)
    a = o.run_smc(tg, k0, betas, 512, policy=abi.POLICY_ALWAYS, seed=6, round=1)
    b = capi.run_smc(tg, k0, betas, 512, policy=abi.POLICY_ALWAYS, seed=6, round=1, exec_=ex)
    assert a["resample_times"] == b["resample_times"] == list(range(1, 17))
    for g in ("log_g0", "log_g1", "log_g2"):
        assert np.max(np.abs(a[g][1:] - b[g][1:]) / np.abs(a[g][1:]).clip(1)) < 1e-6, g
    # HMC moves under adaptive resampling: an unbiased estimate of the exact log Z(1)
    k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=8)
    exact_lz = exact.ising_relaxed_log_z(16, KC, 1.0)
    r = capi.run_smc(tg, k, np.linspace(0, 1, 129), 1 << 13, policy=abi.POLICY_ADAPTIVE_ESS, seed=4,
                     round=1, exec_=ex)
    assert abs(r["log_z_hat"] - exact_lz) < 0.5
    r = capi.run_sais_single(tg, k, np.linspace(0, 1, 257), 1 << 14, seed=3, round=1, exec_=ex)
    assert abs(r["log_z_hat"] - exact_lz) < 0.5


@pytest.mark.gpu
def test_ising_64_rounds_run_and_reject_bad_modes():
    tg = abi.ising(64, KC, 1.0, 1.0)
    k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=4)
    r = capi.run_rounds(tg, k, abi.MODE_SAIS, 512, 3, seed=1, exec_=abi.execopts(PH, F32))
    assert list(r["steps"]) == [1, 2, 3] and np.all(np.isfinite(r["log_z_hat"]))
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_single(tg, k, [0.0, 1.0], 16, exec_=abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64))
    assert e.value.code == abi.ERR_CAPABILITY
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_single(abi.ising(12, KC), k, [0.0, 1.0], 16, exec_=abi.execopts(PH, F32))
    assert e.value.code == abi.ERR_CAPABILITY


def test_host_api_ising_target_potential():
    import paper_2408_12057_b200 as asmc
    L, K, delta, sigma = 5, KC, 0.7, 1.3
    t = asmc.IsingTarget(L, K, delta, sigma)
    y = np.random.default_rng(0).normal(size=L * L)
    Y = y.reshape(L, L)
    u = (delta + 4 * K) * Y + K * (np.roll(Y, 1, 0) + np.roll(Y, -1, 0) + np.roll(Y, 1, 1) + np.roll(Y, -1, 1))
    log_eta = np.sum(-0.5 * (y / sigma) ** 2 - math.log(sigma) - 0.5 * math.log(2 * math.pi))
    V = np.sum(-0.5 * Y * u + np.logaddexp(u, -u)) - log_eta
    assert t.dim() == L * L and t.side() == L
    assert abs(t.potential(y.tolist()) - V) < 1e-10 * abs(V)
    assert abs(t.log_reference(y.tolist()) - log_eta) < 1e-10 * abs(log_eta)
    with pytest.raises(ValueError):
        asmc.IsingTarget(2, K)
