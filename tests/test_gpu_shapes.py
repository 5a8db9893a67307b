"""Odd and large shapes of the shared-memory pass against the oracle (GPU).

The G = 4 / 32 lanes-per-particle pass handles d % 4 != 0 (the unaligned Philox
path), fewer quads than lanes, the last quad-iteration with only some lanes active,
particle counts that leave the last 256-block partly empty, and d up to the shared
memory budget.  Every shape runs SAIS through the C-ABI and is compared with the
unmodified reference engine on the Philox shadow stream (fp32 tolerance as in
tests/test_gpu_parity.py), and with its own full-evaluation run (early rejection
off) bit for bit.
"""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu

PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
RWMH = abi.kernel(abi.KERNEL_RWMH, (0.05, 0.3, 2.0), 1)


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


def _ref():
    return oracle.load("ref", PH) if oracle.available("ref", PH) else oracle.load("restate", PH)


SHAPES = [  # (target, lanes, n)
    ("scale17_g4", lambda: abi.scale_gaussian(1.0, 2.0, 17), 4, 1000),
    ("gauss33_g4", lambda: abi.gaussian_shift(0.0, 0.5, 1.0, 33), 4, 777),
    ("mix129_g32", lambda: abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 129), 32, 600),
    ("scale1001_g32", lambda: abi.scale_gaussian(1.0, 2.0, 1001), 32, 513),
    ("gauss2048_g32", lambda: abi.gaussian_shift(0.0, 0.05, 1.0, 2048), 32, 300),
]


@pytest.mark.parametrize("name,make,lanes,n", SHAPES)
def test_shape_matches_reference(monkeypatch, name, make, lanes, n):
    tg = make()
    betas = np.linspace(0.0, 1.0, 5)
    a = _ref().run_sais_single(tg, RWMH, betas, n, seed=4, round=2)
    ex = abi.execopts(PH, F32, lanes=lanes)
    b = capi.run_sais_single(tg, RWMH, betas, n, seed=4, round=2, exec_=ex)
    for g in ("log_g0", "log_g1", "log_g2"):
        rel = np.abs(a[g][1:] - b[g][1:]) / np.abs(a[g][1:]).clip(1)
        assert np.max(rel) < 2e-3, (name, g, a[g], b[g])
    assert abs(a["log_z_hat"] - b["log_z_hat"]) < 2e-3 * max(1.0, abs(a["log_z_hat"])), name
    monkeypatch.setenv("ASMC_NO_EARLY_REJECT", "1")
    c = capi.run_sais_single(tg, RWMH, betas, n, seed=4, round=2, exec_=ex)
    monkeypatch.delenv("ASMC_NO_EARLY_REJECT")
    for g in ("log_g0", "log_g1", "log_g2"):
        assert np.array_equal(b[g], c[g]), (name, g)
