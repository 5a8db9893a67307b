"""GPU: batched seeds (asmc_run_sais_seeds).  The seed is an extra launch
dimension of the one-lane pass, the fold, the report and the schedule kernels; every
seed's results must equal its own asmc_run_rounds(SAIS) call bit for bit (reference
arithmetic and throughput mode), and match the unmodified reference's run_sais."""
import numpy as np
import pytest

import oracle
from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu
XO, PH, F64, F32 = abi.RNG_XOSHIRO, abi.RNG_PHILOX, abi.PREC_FP64, abi.PREC_FP32


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if capi.device_count() < 1:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


@pytest.mark.parametrize("rng,prec", [(XO, F64), (PH, F32)])
@pytest.mark.parametrize("tname", ["gauss10", "mix12"])
def test_batched_seeds_equal_single_runs(rng, prec, tname):
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10) if tname == "gauss10" else abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 12)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    seeds = [1, 2, 7, 1000, 123456789]
    ex = abi.execopts(rng, prec, lanes=1)
    b = capi.run_sais_seeds(tg, k, 3000, 4, seeds, exec_=ex)
    for i, s in enumerate(seeds):
        r = capi.run_rounds(tg, k, abi.MODE_SAIS, 3000, 4, seed=s, exec_=ex)
        assert list(b["steps"]) == [int(v) for v in r["steps"]]
        assert np.array_equal(b["log_z_hat"][i], r["log_z_hat"]), (s, b["log_z_hat"][i], r["log_z_hat"])
        assert np.array_equal(b["elbo_hat"][i], r["elbo_hat"])
        lam = np.array([r["lambda_"][j, int(r["steps"][j])] for j in range(4)])
        assert np.array_equal(b["lambda_total"][i], lam)


def test_batched_seeds_match_reference_run_sais():
    if not oracle.available("ref", XO):
        pytest.skip("reference not built")
    ref = oracle.load("ref", XO)
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 10)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    seeds = [3, 4, 5]
    b = capi.run_sais_seeds(tg, k, 2048, 4, seeds, exec_=abi.execopts(XO, F64, lanes=1))
    for i, s in enumerate(seeds):
        a = ref.run_rounds(tg, k, abi.MODE_SAIS, 2048, 4, seed=s, workers=4)
        assert np.max(np.abs(a["log_z_hat"] - b["log_z_hat"][i])) < 1e-9


def test_batched_seeds_rejects_wide_layouts():
    tg = abi.scale_gaussian(1.0, 2.0, 2000)
    with pytest.raises(capi.AsmcError) as e:
        capi.run_sais_seeds(tg, abi.kernel(abi.KERNEL_RWMH), 256, 2, [1, 2], exec_=abi.execopts(PH, F32))
    assert e.value.code == abi.ERR_CAPABILITY
