"""GPU: config 3 as BASELINE.json configures it, against the unmodified reference.

SSMC (run_ssmc, drivers.cpp:186-232) with adaptive-ESS systematic resampling on the
d = 100 bimodal mixture (MixtureTarget(2, 0.5, -1, 0.5, 1, 0.5), exact log Z = 0),
RWMH {0.1, 1, 10}, N1 = 4096, 6 rounds -- the reference (oracle/_ref, Philox shadow
streams, fp64) and the device (fp32 / Philox, the bench's mode) over 20 seeds each.

The two runs share every random number, every resampling rule (the reference's
sequential CDF, csrc/refcdf.cu) and every schedule operation; they differ by fp32
arithmetic, which flips a rare MH decision and then diverges that particle.  Bars:
  * per round, the mean over seeds of log Z-hat and of Lambda-hat agree within
    3 standard errors of the seed-to-seed spread (Monte Carlo error);
  * per seed, the resampling times agree in >= 80 % of rounds and |d log Z-hat| is
    small next to the spread across seeds (median < 0.25 sigma).
"""
import os

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


def lam_total(r):
    steps = [int(v) for v in r["steps"]]
    return np.array([r["lambda_"][i, steps[i]] for i in range(len(steps))])


def test_config3_vs_reference_over_seeds():
    if not oracle.available("ref", PH):
        pytest.skip("reference not built")
    ref = oracle.load("ref", PH)
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 100)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    seeds = range(1, 21)
    A, B = [], []
    same_times, rounds_total = 0, 0
    for s in seeds:
        a = ref.run_rounds(tg, k, abi.MODE_SSMC, 4096, 6, policy=abi.POLICY_ADAPTIVE_ESS, seed=s,
                           workers=os.cpu_count() or 1)
        b = capi.run_rounds(tg, k, abi.MODE_SSMC, 4096, 6, policy=abi.POLICY_ADAPTIVE_ESS, seed=s,
                            exec_=abi.execopts(PH, F32))
        assert list(a["steps"]) == list(b["steps"]) and list(a["n_particles"]) == list(b["n_particles"])
        A.append((a["log_z_hat"].copy(), lam_total(a)))
        B.append((b["log_z_hat"].copy(), lam_total(b)))
        for i in range(6):
            T = int(a["steps"][i])
            rounds_total += 1
            same_times += np.array_equal(a["resampled"][i, :T + 1], b["resampled"][i, :T + 1])
    za, zb = np.array([x[0] for x in A]), np.array([x[0] for x in B])
    la, lb = np.array([x[1] for x in A]), np.array([x[1] for x in B])
    n = len(seeds)
    for name, x, y in (("log_z", za, zb), ("lambda", la, lb)):
        se = np.sqrt((x.var(axis=0, ddof=1) + y.var(axis=0, ddof=1)) / n)
        d = np.abs(x.mean(axis=0) - y.mean(axis=0))
        assert np.all(d <= 3 * se + 1e-9), (name, d, se)
    sigma = za.std(axis=0, ddof=1)
    assert np.all(np.median(np.abs(za - zb), axis=0) < 0.25 * sigma + 1e-9), (np.median(np.abs(za - zb), axis=0), sigma)
    assert same_times >= 0.8 * rounds_total, (same_times, rounds_total)
