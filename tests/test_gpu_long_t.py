"""GPU: long-T SAIS.  The reference's run_sais_single has no cap on T
(drivers.cpp:59-146 keeps (T+1) accumulators per wave slot in heap memory).  The
shared-memory pass keeps per-warp step accumulators for the steps of one launch, so a
long round runs in t-tiles with the particle rows parked in HBM between them
(capi.cu: sais_tile_rows / launch_sais_pass).  Bars:
  * tiling changes nothing: any tile length gives the same bits as one launch;
  * T = 2000, d = 1000 (far beyond the 227 KB of one launch) runs and agrees with the
    unmodified reference (Philox shadow streams) within the fp32 tolerance below;
  * config 2's round loop, continued until T ~ Lambda^2, drives log Z-hat to the exact 0.
"""
import os

import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu
PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
RWMH = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


def sais(tg, betas, n, tile=None, lanes=32, seed=4):
    old = os.environ.pop("ASMC_SAIS_TILE", None)
    if tile is not None:
        os.environ["ASMC_SAIS_TILE"] = str(tile)
    try:
        return capi.run_sais_single(tg, RWMH, betas, n, seed=seed, round=1,
                                    exec_=abi.execopts(PH, F32, lanes=lanes))
    finally:
        os.environ.pop("ASMC_SAIS_TILE", None)
        if old is not None:
            os.environ["ASMC_SAIS_TILE"] = old


@pytest.mark.parametrize("dim,lanes", [(1000, 32), (100, 4), (300, 32)])
def test_tiles_bit_identical_to_one_launch(dim, lanes):
    tg = abi.scale_gaussian(1.0, 2.0, dim) if dim != 100 else abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, dim)
    T = 40
    betas = np.linspace(0, 1, T + 1) ** 2
    one = sais(tg, betas, 3000, tile=T, lanes=lanes)
    for tile in (1, 7, 16):
        got = sais(tg, betas, 3000, tile=tile, lanes=lanes)
        for k in ("log_g0", "log_g1", "log_g2"):
            assert np.array_equal(got[k], one[k]), (tile, k)
        assert got["log_z_hat"] == one["log_z_hat"] and got["elbo_hat"] == one["elbo_hat"]


def test_long_t_2000_d1000_matches_reference():
    """T = 2000 at d = 1000: one launch would need 8 x 2001 x 4 x 16 B = 1 MB of
    per-warp accumulators; the tiles run it.  Reference: the unmodified run_sais_single
    compiled against the Philox shadow streams (fp64); the device computes in fp32, so
    particles whose MH decision flips diverge -- per-step log-moments within 0.05
    absolute, log Z-hat within 0.05 (n = 256)."""
    if not oracle.available("ref", PH):
        pytest.skip("reference not built")
    ref = oracle.load("ref", PH)
    tg = abi.scale_gaussian(1.0, 2.0, 1000)
    T, n = 2000, 256
    betas = np.linspace(0, 1, T + 1)
    b = sais(tg, betas, n)
    a = ref.run_sais_single(tg, RWMH, betas, n, seed=4, round=1, workers=os.cpu_count() or 1)
    for k in ("log_g1",):
        assert np.max(np.abs(a[k][1:] - b[k][1:])) < 0.05, k
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 0.05, (a["log_z_hat"], b["log_z_hat"])


@pytest.mark.parametrize("kname,rounds,tol", [("idealized", 13, 0.1), ("hmc", 15, 3.0)])
def test_config2_round_loop_reaches_exact_log_z(kname, rounds, tol):
    """Config 2's target (d = 1000 scale mismatch, Lambda ~ 31): the doubling round loop
    (drivers.cpp:186-232) from N1 = 2^10 with schedule adaptation drives log Z-hat to the
    exact 0 once T grows past ~Lambda^2 / 10, through the t-tiled long-T pass (T up to
    148 / 297 here; one launch holds ~22 steps at d = 1000).  With the config's RWMH
    {0.1, 1, 10} the same loop stays near -210 at T = 1193: random-walk moves in d = 1000
    barely follow the annealed scale (a kernel property the unmodified reference shares,
    test_long_t_2000_d1000_matches_reference), so convergence is shown with the
    reference's idealized kernel and with HMC."""
    tg = abi.scale_gaussian(1.0, 2.0, 1000)
    k = abi.kernel(abi.KERNEL_IDEALIZED) if kname == "idealized" else abi.kernel(abi.KERNEL_HMC, (0.3,), 1, 5)
    r = capi.run_rounds(tg, k, abi.MODE_SAIS, 1 << 10, rounds, seed=1, exec_=abi.execopts(PH, F32))
    lz = [float(v) for v in r["log_z_hat"]]
    assert int(r["steps"][-1]) >= 148
    assert abs(lz[-1]) < tol, lz
    assert lz[0] < -200  # T = 1: the round loop starts far from the answer
