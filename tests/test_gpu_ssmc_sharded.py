"""Multi-GPU SSMC (asmc_smc_shard_*) on one B200: G shards driven in lockstep by
paper_2408_12057_b200.distributed with VirtualComm (the collectives become
concatenations/slices in rank order, exactly what NCCL delivers).  The sharded
run must be BIT-identical to the single-GPU asmc_run_smc (same fp32/Philox
execution mode): per-step g0/g1/g2, ESS, resampling times, log Z, ELBO, and the
final particles themselves for every world size."""
import numpy as np
import pytest

from paper_2408_12057_b200 import abi, capi, distributed

pytestmark = pytest.mark.gpu

PH, F32 = abi.RNG_PHILOX, abi.PREC_FP32
N = 2 * abi.FOLD_CHUNK + 12345
KEYS = ("log_g0", "log_g1", "log_g2", "ess_trace", "cum_log_z", "resample_times", "resampled")


def _same(a, b):
    for k in KEYS:
        assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    assert a["log_z_hat"] == b["log_z_hat"] and a["elbo_hat"] == b["elbo_hat"]


@pytest.mark.parametrize("policy", [abi.POLICY_ALWAYS, abi.POLICY_ADAPTIVE_ESS])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_ssmc_bit_identical_to_single_gpu(policy, world):
    tg = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 8)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    betas = np.linspace(0, 1, 7)
    ex = abi.execopts(PH, F32)
    ref = capi.run_smc(tg, k, betas, N, policy=policy, seed=5, round=2, exec_=ex)
    reps = distributed.run_smc_multi(tg, k, betas, N, policy=policy, seed=5, round=2, exec_=ex,
                                     world=world)
    assert len(ref["resample_times"]) > 0
    for r in reps:
        _same(r, ref)


def test_sharded_particles_identical_across_world_sizes():
    tg = abi.scale_gaussian(1.0, 2.0, 20)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.5, 1.0), 1)
    betas = np.linspace(0, 1, 6)
    ex = abi.execopts(PH, F32)
    stats = {}
    one = distributed.run_smc_multi(tg, k, betas, N, policy=abi.POLICY_ALWAYS, seed=3, exec_=ex,
                                    world=1, return_state=True)
    three = distributed.run_smc_multi(tg, k, betas, N, policy=abi.POLICY_ALWAYS, seed=3, exec_=ex,
                                      world=3, return_state=True, stats=stats)
    x1 = one[0]["x"]
    x3 = np.concatenate([r["x"] for r in three])
    assert x1.shape == (N, 20) and np.array_equal(x1, x3)
    assert np.array_equal(one[0]["log_w"], np.concatenate([r["log_w"] for r in three]))
    assert len(stats["rows_moved"]) == 5  # one exchange per step (policy always)
    _same(one[0], three[2])


def test_shard_api_rejects_misuse():
    tg = abi.gaussian_shift(0.0, 1.0, 1.0, 4)
    k = abi.kernel(abi.KERNEL_RWMH)
    ex = abi.execopts(PH, F32)
    with pytest.raises(capi.AsmcError) as e:
        capi.SmcShard(tg, k, [0.0, 1.0], 1000, 10, 1000, exec_=ex)
    assert "multiple of ASMC_FOLD_CHUNK" in e.value.msg
    with pytest.raises(capi.AsmcError) as e:
        capi.SmcShard(tg, k, [0.0, 1.0], 1000, 0, 1000, exec_=abi.execopts(abi.RNG_XOSHIRO, abi.PREC_FP64))
    assert e.value.code == abi.ERR_CAPABILITY
    s = capi.SmcShard(tg, k, [0.0, 0.5, 1.0], 1000, 0, 1000, exec_=ex)
    with pytest.raises(capi.AsmcError):
        s.step(2, 0)  # out of order
    with pytest.raises(capi.AsmcError):
        s.report()  # before the last step
    s.close()


@pytest.mark.parametrize("kind", ["logistic", "ising"])
def test_sharded_sais_partials_for_step_outer_targets(kind):
    """SAIS sharding for configs 4 and 5 -- chunk partials of any shard split
    fold to the single-launch statistics (same fixed tree, global particle ids)."""
    if kind == "logistic":
        X, y = abi.logistic_data(2000, 64, 0)
        tg = abi.logistic(X, y, 1.0)
        k = abi.kernel(abi.KERNEL_RWMH, (0.01, 0.03), 1)
    else:
        tg = abi.ising(16, 0.4406868, 1.0, 1.0)
        k = abi.kernel(abi.KERNEL_HMC, (0.25,), 1, leapfrog=4)
    betas = np.linspace(0, 1, 4)
    ex = abi.execopts(PH, F32)
    single = capi.run_sais_single(tg, k, betas, N, seed=7, round=2, exec_=ex)
    for world in (1, 3):
        ranges = distributed.chunk_partition(N, world)
        parts = np.concatenate([capi.sais_partials(tg, k, betas, N, p0, p1, seed=7, round=2, exec_=ex)
                                for p0, p1 in ranges if p1 > p0])
        rep = capi.fold_partials(parts, N)
        for key in ("log_g0", "log_g1", "log_g2"):
            assert np.array_equal(rep[key], single[key]), (kind, world, key)
        assert rep["log_z_hat"] == single["log_z_hat"]


def test_multi_gpu_zja_identical_for_any_shard_count():
    """every bisection probe is an all-gather of per-chunk partials folded
    in chunk order, so 1 and 3 shards choose the same schedule bit for bit; the result
    matches the single-GPU asmc_run_zja (cooperative-grid tree) to fold-order rounding."""
    tg = abi.gaussian_shift(0.0, 2.0, 1.0, 4)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.5, 1.0), 1)
    ex = abi.execopts(PH, F32)
    stats = {}
    one = distributed.run_zja_multi(tg, k, N, 0.05, seed=3, exec_=ex, world=1)
    three = distributed.run_zja_multi(tg, k, N, 0.05, seed=3, exec_=ex, world=3, stats=stats)
    assert np.array_equal(one[0]["betas"], three[1]["betas"]) and one[0]["betas"][-1] == 1.0
    for r in three:
        assert r["log_z_hat"] == one[0]["log_z_hat"] and np.array_equal(r["log_g1"], one[0]["log_g1"])
    single = capi.run_zja(tg, k, N, delta_star=0.05, seed=3, exec_=ex)
    assert single["steps"] == one[0]["steps"]
    assert np.max(np.abs(single["rounds"][-1]["betas"] - one[0]["betas"])) < 1e-6
    assert abs(single["rounds"][-1]["log_z_hat"] - one[0]["log_z_hat"]) < 1e-6
    assert stats["probes"] > 20 * one[0]["steps"]  # the communication the paper's SAIS avoids
    # the device-resident search syncs with the host about once per annealing step
    assert stats["host_syncs"] <= 2 * one[0]["steps"]


@pytest.mark.parametrize("world", [1, 3])
def test_multi_gpu_zja_device_search_matches_host_search(world):
    """asmc_zja_shard_search_* (state machine in HBM, no host round trip per probe) against
    the host-driven search over the same all-gathered partials: the same schedule up to the
    fold's last-ulp libm differences, the same warnings, far fewer host synchronisations."""
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 0.5, 1.0), 1)
    ex = abi.execopts(PH, F32)
    for tg, delta in ((abi.gaussian_shift(0.0, 2.0, 1.0, 4), 0.05),
                      (abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 2), 0.02)):
        sd, sh = {}, {}
        dev = distributed.run_zja_multi(tg, k, N, delta, seed=5, exec_=ex, world=world, stats=sd)
        host = distributed.run_zja_multi(tg, k, N, delta, seed=5, exec_=ex, world=world, stats=sh,
                                         device_search=False)
        assert dev[0]["steps"] == host[0]["steps"] and dev[0]["warning"] == host[0]["warning"]
        assert np.max(np.abs(dev[0]["betas"] - host[0]["betas"])) < 1e-9
        assert abs(dev[0]["log_z_hat"] - host[0]["log_z_hat"]) < 1e-8
        assert sd["host_syncs"] * 10 < sh["host_syncs"]
