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
