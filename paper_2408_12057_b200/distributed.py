"""Multi-GPU SAIS round loop: one process per GPU, particles sharded by fold chunk.

Partition: round k's particles [0, N_k) are cut into fold chunks
of ASMC_FOLD_CHUNK = 262144 particles (1024 reduction blocks); rank r owns the
contiguous chunk range [r C / G, (r+1) C / G).  Each rank runs the fused pass
for its range (asmc_sais_partials), all ranks allgather the per-chunk
accumulator partials (4 log-moments x (T+1) steps x 16 B per chunk -- about
40 KB per GPU per round), and every rank folds all chunks in chunk order
(asmc_fold_partials) -- so the estimates are bit-identical for any GPU count.
The barrier estimate and the next schedule are then computed redundantly on
every rank (device kernels), and the next round starts.  There is no other
data-path collective: SAIS particles never leave the GPU that drew them.

The collective and partition logic is plain Python over torch.distributed so it
runs unchanged on gloo (CPU tests, world_size 2) and NCCL (B200 box).
"""
import math

import numpy as np

from . import abi

SIZEOF_ROUNDDEV = 80
SIZEOF_SMCSTATE = 80


def chunk_partition(n, world, chunk=abi.FOLD_CHUNK):
    """[(p_begin, p_end)] per rank; p_begin is always a multiple of `chunk`."""
    nch = (n + chunk - 1) // chunk
    out = []
    for r in range(world):
        c0, c1 = r * nch // world, (r + 1) * nch // world
        out.append((min(n, c0 * chunk), min(n, c1 * chunk)))
    return out


def chunks_of(rng, chunk=abi.FOLD_CHUNK):
    b, e = rng
    return 0 if e <= b else (e - b + chunk - 1) // chunk


def allgather_partials(local, counts, T, device=None):
    """Concatenate every rank's chunk partials in rank (= chunk) order.

    local: array (c_r, T+1, 4, 2); counts: chunks per rank.  Ranks pad to the
    largest count so a fixed-size all_gather works on both gloo and NCCL."""
    import torch
    import torch.distributed as dist

    cmax = max(max(counts), 1)
    buf = np.zeros((cmax, T + 1, 4, 2))
    if len(local):
        buf[: len(local)] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    outs = [torch.empty_like(t) for _ in counts]
    dist.all_gather(outs, t)
    parts = [o.cpu().numpy()[:c] for o, c in zip(outs, counts)]
    return np.concatenate(parts, axis=0)


def run_sais(target, kernel, n1, rounds, seed, exec_, rank, world, partials_fn=None,
             fold_fn=None, barrier_fn=None, schedule_fn=None, budget_fn=None, device=None):
    """run_sais (drivers.cpp:186-232) sharded over `world` ranks.

    The *_fn hooks default to the C-ABI (capi) and exist so the host logic can
    be exercised on CPU-only gloo tests with a stand-in for the device pass."""
    if partials_fn is None or fold_fn is None:
        from . import capi
        partials_fn = partials_fn or (lambda b, n, p0, p1, k: capi.sais_partials(
            target, kernel, b, n, p0, p1, seed=seed, round=k, exec_=exec_))
        fold_fn = fold_fn or capi.fold_partials
        barrier_fn = barrier_fn or (lambda r, b: capi.barrier_estimate(
            r["log_g0"], r["log_g1"], r["log_g2"], b, device=exec_.device))
        schedule_fn = schedule_fn or (lambda lam, b, tn: capi.generate_schedule(
            lam, b, tn, device=exec_.device))
        budget_fn = budget_fn or (lambda n, t: capi.budget(n, t, target.dim, 4096 << 20,
                                                            abi.MODE_SAIS))
        if device is None:
            device = f"cuda:{exec_.device}"
    betas = np.array([0.0, 1.0])
    n, T = n1, 1
    res = {k: [] for k in ("n_particles", "steps", "betas", "log_g0", "log_g1", "log_g2",
                           "lambda_", "log_z_hat", "elbo_hat", "kernel_applications")}
    for k in range(1, rounds + 1):
        ranges = chunk_partition(n, world)
        counts = [chunks_of(r) for r in ranges]
        p0, p1 = ranges[rank]
        local = partials_fn(betas, n, p0, p1, k) if p1 > p0 else np.zeros((0, T + 1, 4, 2))
        allp = allgather_partials(local, counts, T, device) if world > 1 else local
        rep = fold_fn(allp, n)
        lam = barrier_fn(rep, betas)
        for key, val in (("n_particles", n), ("steps", T), ("betas", betas.copy()),
                         ("log_g0", rep["log_g0"]), ("log_g1", rep["log_g1"]),
                         ("log_g2", rep["log_g2"]), ("lambda_", lam),
                         ("log_z_hat", rep["log_z_hat"]), ("elbo_hat", rep["elbo_hat"]),
                         ("kernel_applications", n * T)):
            res[key].append(val)
        if k < rounds:
            n, T_new = budget_fn(n, T)
            betas = schedule_fn(lam, betas, T_new)
            T = T_new
    return res


def io_bytes(ts):
    """Host<->device bytes one asmc_run_rounds(SAIS) call moves, counted from
    the copies in csrc/capi.cu: H2D = round-1 betas + one RoundDev per round;
    D2H = per round g0,g1,g2,cum_log_z,lambda,betas (8 B x (T+1) each),
    resampled (1 B), resample_times (4 B), scalars (16 B), SmcState."""
    h2d = 16 + SIZEOF_ROUNDDEV * len(ts)
    d2h = 4 + sum(6 * 8 * (t + 1) + (t + 1) + 4 * (t + 1) + 16 + SIZEOF_SMCSTATE for t in ts)
    return h2d, d2h
