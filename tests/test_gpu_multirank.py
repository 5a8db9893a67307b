"""GPU: the multi-rank SAIS path end to end -- two processes (torch.distributed, gloo), both
on cuda:0, each running its particle shard through the device-resident partials
(asmc_sais_partials_dev -> all-gather -> asmc_fold_partials_dev) -- against the single-GPU
round loop (asmc_run_rounds) on the same total particles: identical bits.  The NVLink /
NCCL variant of the same code path is the driver's N > 1 bench."""
import os
import socket

import numpy as np
import pytest

from paper_2408_12057_b200 import abi, capi

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, n1, rounds):
    import torch
    import torch.distributed as dist
    from paper_2408_12057_b200 import distributed
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        tg = abi.scale_gaussian(1.0, 2.0, 200)
        k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
        r = distributed.run_sais(tg, k, n1, rounds, 7, abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, device=0),
                                 rank, world)
        q.put((rank, [float(v) for v in r["log_z_hat"]], [list(map(float, b)) for b in r["betas"]]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_one_rank():
    import torch.multiprocessing as mp
    n1, rounds = 3 * abi.FOLD_CHUNK + 4321, 3
    tg = abi.scale_gaussian(1.0, 2.0, 200)
    k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
    one = capi.run_rounds(tg, k, abi.MODE_SAIS, n1, rounds, seed=7, exec_=abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, n1, rounds)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, lz, betas = q.get(timeout=600)
        got[rank] = (lz, betas)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0] == got[1]
    assert got[0][0] == [float(v) for v in one["log_z_hat"]]
    for r in range(rounds):
        T = int(one["steps"][r])
        assert got[0][1][r] == [float(v) for v in one["betas"][r][: T + 1]]


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist
    from paper_2408_12057_b200 import distributed
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, device=0)
        out = {"backend": dist.get_backend()}
        tg = abi.scale_gaussian(1.0, 2.0, 200)
        k = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1)
        r = distributed.run_sais(tg, k, 2 * abi.FOLD_CHUNK + 999, 3, 7, ex, 0, 1)
        out["sais"] = [float(v) for v in r["log_z_hat"]]
        comm = distributed.TorchComm(0, 1)
        tm = abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 8)
        km = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0), 1)
        betas = np.linspace(0.0, 1.0, 9)
        (rep,) = distributed.run_smc_multi(tm, km, betas, 3 * abi.FOLD_CHUNK + 77, policy=abi.POLICY_ALWAYS, seed=4,
                                           exec_=ex, comm=comm, rank=0, world=1)
        out["smc"] = (float(rep["log_z_hat"]), [int(v) for v in rep["resample_times"]])
        tz = abi.gaussian_shift(0.0, 2.0, 1.0, 4)
        (z,) = distributed.run_zja_multi(tz, km, 2 * abi.FOLD_CHUNK + 5, 0.05, seed=3, exec_=ex, comm=comm, rank=0,
                                         world=1)
        out["zja"] = (float(z["log_z_hat"]), [float(v) for v in z["betas"]])
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_nccl_process_group_paths_equal_single_gpu():
    """The NCCL code paths themselves (device-to-device all-gathers on the library's stream:
    SAIS partials, SSMC step partials + log-weights, ZJA probe partials) in a real NCCL
    process group of one rank -- the most this one-GPU box can run (NCCL refuses two ranks
    on one device) -- against the single-GPU entry points, bit for bit."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0 and out["backend"] == "nccl"
    ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    one = capi.run_rounds(abi.scale_gaussian(1.0, 2.0, 200), abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0, 10.0), 1),
                          abi.MODE_SAIS, 2 * abi.FOLD_CHUNK + 999, 3, seed=7, exec_=ex)
    assert out["sais"] == [float(v) for v in one["log_z_hat"]]
    km = abi.kernel(abi.KERNEL_RWMH, (0.1, 1.0), 1)
    s = capi.run_smc(abi.mixture(2.0, 0.5, -1.0, 0.5, 1.0, 0.5, 8), km, np.linspace(0.0, 1.0, 9),
                     3 * abi.FOLD_CHUNK + 77, policy=abi.POLICY_ALWAYS, seed=4, exec_=ex)
    assert out["smc"][0] == float(s["log_z_hat"]) and out["smc"][1] == [int(v) for v in s["resample_times"]]
    from paper_2408_12057_b200 import distributed
    (z,) = distributed.run_zja_multi(abi.gaussian_shift(0.0, 2.0, 1.0, 4), km, 2 * abi.FOLD_CHUNK + 5, 0.05, seed=3,
                                     exec_=ex, world=1)
    assert out["zja"] == (float(z["log_z_hat"]), [float(v) for v in z["betas"]])
