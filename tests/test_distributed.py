"""Multi-GPU host logic on CPU (gloo, world_size 2): chunk partition, the
chunk-partial allgather and its ordering, and the round loop of
paper_2408_12057_b200.distributed -- with a deterministic stand-in for the
device pass so the collective logic runs without a GPU.  The property tested
is the one the device path relies on: every rank ends with identical results,
equal to the single-rank run, for any world size."""
import os
import socket

import numpy as np
import pytest

from paper_2408_12057_b200 import abi, distributed


def test_chunk_partition_covers_exactly():
    for n in (1, 1000, abi.FOLD_CHUNK, abi.FOLD_CHUNK + 1, 47453135):
        for w in (1, 2, 3, 8):
            parts = distributed.chunk_partition(n, w)
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, _) in zip(parts, parts[1:]):
                assert b == c
            assert all(p0 % abi.FOLD_CHUNK == 0 for p0, _ in parts)


def fake_partials(betas, n, p0, p1, k):
    """Stand-in for asmc_sais_partials: a deterministic function of the GLOBAL chunk index."""
    T = len(betas) - 1
    nch = (p1 - p0 + abi.FOLD_CHUNK - 1) // abi.FOLD_CHUNK
    out = np.zeros((nch, T + 1, 4, 2))
    for i in range(nch):
        c = p0 // abi.FOLD_CHUNK + i
        g = np.random.default_rng(1000 * k + c)
        out[i, 1:, :, 0] = g.normal(0, 1, (T, 4))
        out[i, 1:, :, 1] = g.uniform(1, 2, (T, 4))
        out[i, 0, :, 0] = -np.inf
    return out


def fold(parts, n):
    """Sequential combine over chunks in order (the device final fold's semantics)."""
    T = parts.shape[1] - 1
    acc = np.zeros((T + 1, 4, 2))
    acc[..., 0] = -np.inf
    for c in range(parts.shape[0]):
        for t in range(1, T + 1):
            for a in range(4):
                m, s = acc[t, a]
                om, os_ = parts[c, t, a]
                if om <= m:
                    s += os_ * np.exp(om - m)
                else:
                    s = s * np.exp(m - om) + os_
                    m = om
                acc[t, a] = (m, s)
    tot = acc[..., 0] + np.log(acc[..., 1])
    return {"log_g0": tot[:, 0], "log_g1": tot[:, 1], "log_g2": tot[:, 2],
            "log_z_hat": tot[T, 1] - np.log(n), "elbo_hat": 0.0}


def barrier(rep, betas):
    raw = np.maximum(0.0, rep["log_g2"][1:] - 2 * rep["log_g1"][1:] + rep["log_g0"][1:])
    return np.concatenate([[0.0], np.cumsum(np.sqrt(raw))])


def schedule(lam, betas, t_new):
    return np.interp(np.linspace(0, lam[-1], t_new + 1), lam, betas) if lam[-1] > 0 else \
        np.linspace(0, 1, t_new + 1)


def budget(n, t):
    return int(np.ceil(np.sqrt(2) * n)), int(np.ceil(np.sqrt(2) * t))


def run(rank, world):
    return distributed.run_sais(None, None, 3 * abi.FOLD_CHUNK + 777, 3, 1, None, rank, world,
                                partials_fn=fake_partials, fold_fn=fold, barrier_fn=barrier,
                                schedule_fn=schedule, budget_fn=budget, device="cpu")


def _worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        res = run(rank, world)
        q.put((rank, [float(v) for v in res["log_z_hat"]], [list(map(float, b)) for b in res["betas"]]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_round_loop_matches_single_rank():
    import torch.multiprocessing as mp
    single = run(0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    for _ in procs:
        rank, lz, betas = q.get(timeout=120)
        got[rank] = (lz, betas)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1]
    assert got[0][0] == [float(v) for v in single["log_z_hat"]]


def test_io_bytes_accounting():
    h2d, d2h = distributed.io_bytes([1, 2, 3, 5])
    assert h2d == 16 + 4 * 80
    assert d2h > 0
