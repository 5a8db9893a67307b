"""Multi-GPU SAIS round loop: one process per GPU, particles sharded by fold chunk.

Partition: round k's particles [0, N_k) are cut into fold chunks
of ASMC_FOLD_CHUNK = 262144 particles (1024 reduction blocks); rank r owns the
contiguous chunk range [r C / G, (r+1) C / G).  Each rank runs the fused pass
for its range (asmc_sais_partials), all ranks allgather the per-chunk
accumulator partials (4 log-moments x (T+1) steps x 16 B per chunk -- about
40 KB per GPU per round), and every rank folds all chunks in chunk order
(asmc_fold_partials_dev) -- so the estimates are bit-identical for any GPU count.
The partials never visit the host: the pass writes them into a device tensor
(asmc_sais_partials_dev), the all-gather runs device to device (NCCL), and the fold
runs on the GPU, all on one CUDA stream shared by torch and the library.
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
SIZEOF_SMCSTATE = 88


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

    Default (no hooks): the device path -- partials in device tensors, NCCL all-gather,
    device fold.  The *_fn hooks replace the C-ABI calls with host-array stand-ins so the
    host logic runs on CPU-only gloo tests."""
    device_path = partials_fn is None and fold_fn is None
    if device_path:
        import torch
        import torch.distributed as dist
        from . import capi
        dev = torch.device("cuda", exec_.device)
        # one non-default stream shared by torch (buffers, collectives) and the library:
        # with torch's legacy default stream (handle 0) the library would run on its own
        # non-blocking stream, unordered with torch's zero-fill of the partials buffer
        stream = torch.cuda.Stream(device=dev) if exec_.stream == 0 else \
            torch.cuda.ExternalStream(exec_.stream, device=dev)
        torch.cuda.current_stream(dev).synchronize()
        ex = abi.execopts(exec_.rng, exec_.precision, exec_.device, exec_.lanes, stream.cuda_stream)
        barrier_fn = barrier_fn or (lambda r, b: capi.barrier_estimate(
            r["log_g0"], r["log_g1"], r["log_g2"], b, device=exec_.device))
        schedule_fn = schedule_fn or (lambda lam, b, tn: capi.generate_schedule(
            lam, b, tn, device=exec_.device))
    budget_fn = budget_fn or (lambda n, t: __import__(__package__ + ".capi", fromlist=["budget"]).budget(
        n, t, target.dim, 4096 << 20, abi.MODE_SAIS))
    betas = np.array([0.0, 1.0])
    n, T = n1, 1
    res = {k: [] for k in ("n_particles", "steps", "betas", "log_g0", "log_g1", "log_g2",
                           "lambda_", "log_z_hat", "elbo_hat", "kernel_applications", "cum_log_z",
                           "resampled", "wall_seconds")}
    for k in range(1, rounds + 1):
        ranges = chunk_partition(n, world)
        counts = [chunks_of(r) for r in ranges]
        p0, p1 = ranges[rank]
        if device_path:
            cmax = max(max(counts), 1)
            with torch.cuda.stream(stream):
                local = torch.zeros((cmax, T + 1, 4, 2), dtype=torch.float64, device=dev)
            if p1 > p0:
                capi.sais_partials_dev(target, kernel, betas, n, p0, p1, local.data_ptr(), seed=seed, round=k,
                                       exec_=ex)
            with torch.cuda.stream(stream):
                if dist.is_initialized() and dist.get_backend() == "nccl":  # device to device (any world)
                    outs = [torch.empty_like(local) for _ in counts]
                    dist.all_gather(outs, local)
                elif world > 1:  # gloo (the 2-ranks-on-one-GPU check): staged through the host
                    host = local.cpu()
                    outs = [torch.empty_like(host) for _ in counts]
                    dist.all_gather(outs, host)
                    outs = [o.to(dev) for o in outs]
                else:
                    outs = [local]
                allp = torch.cat([o[:c] for o, c in zip(outs, counts)]).contiguous()
            rep = capi.fold_partials_dev(allp.data_ptr(), allp.shape[0], T, n, exec_=ex)
        else:
            local = partials_fn(betas, n, p0, p1, k) if p1 > p0 else np.zeros((0, T + 1, 4, 2))
            allp = allgather_partials(local, counts, T, device) if world > 1 else local
            rep = fold_fn(allp, n)
        lam = barrier_fn(rep, betas)
        for key, val in (("n_particles", n), ("steps", T), ("betas", betas.copy()),
                         ("log_g0", rep["log_g0"]), ("log_g1", rep["log_g1"]),
                         ("log_g2", rep["log_g2"]), ("lambda_", lam),
                         ("log_z_hat", rep["log_z_hat"]), ("elbo_hat", rep["elbo_hat"]),
                         ("kernel_applications", n * T),
                         ("cum_log_z", rep.get("cum_log_z", np.zeros(T + 1))),
                         ("resampled", rep.get("resampled", np.zeros(T + 1, np.uint8))),
                         ("wall_seconds", 0.0)):
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


# ------------------------------------------------------------------ SSMC
# Multi-GPU run_smc (engine.cpp:97-188).  Shards are the fold-chunk
# ranges of chunk_partition.  Per step every shard all-gathers the chunk partials
# (6 accumulators x 16 B per 262144 particles) and folds them in chunk order, so
# ESS, the resampling decision and the uniform are the same on every rank and
# equal to the single-GPU run.  On a resampling event:
#   * the log-weights (8 B per particle) are all-gathered and every rank builds the
#     reference's sequential CDF over all of them (engine.cpp:61-80, bit for bit, by the
#     parallel exact scan of csrc/refcdf.cu) and the global ancestors a_m;
#   * a_m is non-decreasing, so the slots whose ancestor lies in shard r form one
#     contiguous range; shard r packs those rows in slot order;
#   * one all-to-all-v moves each packed row to the shard owning its slot.
# Weight mass that stays balanced across shards keeps most rows on their GPU
# (the self part of the all-to-all is a local copy).

class VirtualComm:
    """All shards in this process (one GPU, or a CPU test): collectives are
    concatenations and slices, in the same rank order NCCL would use."""

    def __init__(self, world):
        self.world = world

    def allgather(self, tensors, counts):
        import torch
        cat = torch.cat(list(tensors), 0)
        return [cat] + [cat.clone() for _ in tensors[1:]]  # one buffer per rank, as NCCL delivers

    def alltoall(self, sends, send_splits, recv_splits):
        import torch
        offs = [np.concatenate([[0], np.cumsum(s)]).astype(int) for s in send_splits]
        out = []
        for q in range(self.world):
            parts = [sends[r][offs[r][q]:offs[r][q + 1]] for r in range(self.world)]
            out.append(torch.cat(parts, 0))
        return out


class TorchComm:
    """One shard per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group

    def allgather(self, tensors, counts):
        import torch
        import torch.distributed as dist
        (x,) = tensors
        cmax = max(max(counts), 1)
        buf = torch.zeros((cmax,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        buf[: x.shape[0]] = x
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return [torch.cat([o[:c] for o, c in zip(outs, counts)], 0)]

    def alltoall(self, sends, send_splits, recv_splits):
        import torch
        import torch.distributed as dist
        (x,), (ss,), (rs,) = sends, send_splits, recv_splits
        recv = torch.empty((int(sum(rs)),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        dist.all_to_all_single(recv, x, [int(v) for v in rs], [int(v) for v in ss], group=self.group)
        return [recv]


def _overlap(a0, a1, b0, b1):
    return max(0, min(a1, b1) - max(a0, b0))


def exchange_splits(slots, bounds):
    """send[r][q] = rows shard r packs for shard q: |[slots[r], slots[r+1]) & [bounds[q], bounds[q+1])|."""
    G = len(bounds) - 1
    return [[_overlap(slots[r], slots[r + 1], bounds[q], bounds[q + 1]) for q in range(G)]
            for r in range(G)]


class DeviceShard:
    """Tensor-facing adapter over capi.SmcShard (device buffers by data_ptr)."""

    def __init__(self, shard, device):
        self.s, self.device = shard, device
        self.chunks, self.exchange_len, self.row_bytes = shard.chunks, shard.exchange_len, shard.row_bytes
        self.T = shard.T

    def step(self, t, partials):
        self.s.step(t, partials.data_ptr())

    def decide(self, t, all_partials, lw_out):
        return self.s.decide(t, all_partials.data_ptr(), all_partials.shape[0], lw_out.data_ptr())

    def plan(self, all_lw, bounds):
        return self.s.plan(all_lw.data_ptr(), all_lw.shape[0], bounds)

    def pack(self, rows):
        self.s.pack(rows.data_ptr())

    def accept(self, rows):
        self.s.accept(rows.data_ptr())

    def report(self):
        return self.s.report()


def run_smc_sharded(shards, ranks, comm, bounds, stats=None, nacc=abi.SHARD_NACC,
                    chunk=abi.FOLD_CHUNK):
    """Drive local shards (one per process with TorchComm; all of them with
    VirtualComm) through steps 1..T in lockstep; returns each shard's report.

    shards[i] owns particles [bounds[ranks[i]], bounds[ranks[i]+1]).  `stats`
    (dict, optional) collects per-step exchange volumes for the bench."""
    import torch
    G = len(bounds) - 1
    T = shards[0].T
    dev = shards[0].device
    n_chunks = [chunks_of((bounds[r], bounds[r + 1]), chunk) for r in range(G)]
    n_ex = [bounds[r + 1] - bounds[r] for r in range(G)]  # log-weights per shard
    parts = [torch.empty((s.chunks, nacc, 2), dtype=torch.float64, device=dev) for s in shards]
    lws = [torch.empty((max(s.exchange_len, 1),), dtype=torch.float64, device=dev) for s in shards]
    for t in range(1, T + 1):
        for s, p in zip(shards, parts):
            s.step(t, p)
        allp = comm.allgather(parts, n_chunks)
        flags = [s.decide(t, a, b) for s, a, b in zip(shards, allp, lws)]
        if not flags[0]:
            continue
        alll = comm.allgather([b[: s.exchange_len] for s, b in zip(shards, lws)], n_ex)
        slots = [s.plan(a, bounds) for s, a in zip(shards, alll)]
        splits = exchange_splits(slots[0], bounds)
        sends = []
        for s, r, sl in zip(shards, ranks, slots):
            rows = torch.empty((sl[r + 1] - sl[r], s.row_bytes), dtype=torch.uint8, device=dev)
            s.pack(rows)
            sends.append(rows)
        recvs = comm.alltoall(sends, [splits[r] for r in ranks],
                              [[splits[q][r] for q in range(G)] for r in ranks])
        for s, rows in zip(shards, recvs):
            s.accept(rows)
        if stats is not None:
            moved = sum(splits[r][q] for r in range(G) for q in range(G) if q != r)
            stats.setdefault("rows_moved", []).append(moved)
    return [s.report() for s in shards]



def run_smc_multi(target, kernel, betas, n, policy=abi.POLICY_ADAPTIVE_ESS, rho=0.5, seed=0, round=0,
                  exec_=None, comm=None, rank=0, world=1, return_state=False, stats=None):
    """Multi-GPU asmc::run_smc: this process's shard(s) on exec_.device.

    comm = TorchComm(rank, world) drives one shard per process (NCCL on the GPU
    box); comm = None runs all `world` shards in this process (VirtualComm) --
    the single-GPU proof that the sharded result is bit-identical to asmc_run_smc.
    All library work and all torch-side buffers/collectives share one CUDA stream."""
    import torch
    from . import capi
    ex = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    dev = torch.device("cuda", ex.device)
    stream = torch.cuda.Stream(device=dev)
    ex = abi.execopts(ex.rng, ex.precision, ex.device, ex.lanes, stream.cuda_stream)
    bounds = [b for b, _ in chunk_partition(n, world)] + [n]
    ranks = list(range(world)) if comm is None else [rank]
    comm = comm or VirtualComm(world)
    with torch.cuda.device(dev), torch.cuda.stream(stream):
        shards = [DeviceShard(capi.SmcShard(target, kernel, betas, n, bounds[r], bounds[r + 1], policy,
                                            rho, seed, round, ex), dev) for r in ranks]
        reps = run_smc_sharded(shards, ranks, comm, bounds, stats=stats)
        if return_state:
            for rep, s in zip(reps, shards):
                rep["x"], rep["log_w"] = s.s.state()
    stream.synchronize()
    for s in shards:
        s.s.close()
    return reps


# ------------------------------------------------------------------- ZJA
# Multi-GPU run_zja (drivers.cpp:234-341; SURVEY 8e "ZJA: per-step allgathers inside
# the bisection").  Every probe of zja_next_beta's bisection (schedule.cpp:219-264) is
# one all-gather of the shards' per-chunk (m1, m2) partials, folded in chunk order on
# every rank -- so all ranks take the same branches and choose the same beta, and the
# result is the same for any GPU count.  ~50 collectives per annealing step, against
# one per ROUND for SAIS: the paper's argument, made measurable.

def _lacc_combine(a, b):
    """LogAccumulator::combine (logsum.hpp:30-38) on (max, sum) pairs (host doubles)."""
    am, asum = a
    bm, bs = b
    if bm == -math.inf:
        return a
    if bm <= am:
        return (am, asum + bs * math.exp(bm - am))
    return (bm, asum * math.exp(am - bm) + bs)


def _lacc_total(a):
    return -math.inf if a[0] == -math.inf else a[0] + math.log(a[1])


def zja_search(dhat, beta, delta, tol=1e-10):
    """zja_next_beta's search (schedule.cpp:233-263) over a dhat(b2) oracle."""
    if dhat(1.0) <= delta:
        return 1.0, False

    def bisect(lo, hi):
        while hi - lo > tol:
            mid = 0.5 * (lo + hi)
            if dhat(mid) <= delta:
                lo = mid
            else:
                hi = mid
        return lo

    root = bisect(beta, 1.0)
    for i in range(1, 16):
        probe = beta + (root - beta) * float(i) / 16
        if dhat(probe) > delta * (1.0 + 1e-12):
            return bisect(beta, probe), True
    return root, False


def _bisect_probes(beta, tol=1e-10):
    """probes bisect(beta, 1) takes when the interval halves exactly (a lower bound)"""
    k, w = 0, 1.0 - beta
    while w > tol:
        w *= 0.5
        k += 1
    return k


def run_zja_multi(target, kernel, n, delta_star, seed=0, exec_=None, comm=None, rank=0, world=1, max_steps=100000,
                  round=1, stats=None, device_search=True):
    """run_zja's adaptive round (delta_star > 0) sharded over `world` GPUs; returns the
    run report with the chosen schedule (`betas`) on every rank.

    device_search=True keeps the bisection on the device (asmc_zja_shard_search_*):
    probe -> all-gather -> step are stream-ordered with no host round trip; the host
    enqueues a batch of probes sized to the search's expected length (test + bisection
    + 15-point scan) and polls once, adding small batches only for the non-monotone
    fallback.  device_search=False is the host-driven search (one synchronising
    all-gather per probe), kept for A/B."""
    import torch
    from . import capi
    if not delta_star > 0:
        raise ValueError("run_zja_multi needs delta_star > 0 (calibrate with a sharded SAIS pilot)")
    ex = exec_ or abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32)
    dev = torch.device("cuda", ex.device)
    stream = torch.cuda.Stream(device=dev)
    ex = abi.execopts(ex.rng, ex.precision, ex.device, ex.lanes, stream.cuda_stream)
    bounds = [b for b, _ in chunk_partition(n, world)] + [n]
    ranks = list(range(world)) if comm is None else [rank]
    comm = comm or VirtualComm(world)
    n_chunks = [chunks_of((bounds[r], bounds[r + 1])) for r in range(world)]
    probes = 0
    with torch.cuda.device(dev), torch.cuda.stream(stream):
        shards = [capi.ZjaShard(target, kernel, n, bounds[r], bounds[r + 1], seed, round, max_steps, ex) for r in ranks]
        parts = [torch.empty((s.chunks, abi.SHARD_NACC, 2), dtype=torch.float64, device=dev) for s in shards]
        lws = [torch.empty((max(s.exchange_len, 1),), dtype=torch.float64, device=dev) for s in shards]

        def gathered(local):  # all-gather host partials (chunks, 2, 2) in rank (= chunk) order
            ts = [torch.from_numpy(a).to(dev) for a in local]
            return [g.cpu().numpy() for g in comm.allgather(ts, n_chunks)][0]

        def fold(allp, k):
            acc = (-math.inf, 0.0)
            for c in range(allp.shape[0]):
                acc = _lacc_combine(acc, (float(allp[c, k, 0]), float(allp[c, k, 1])))
            return acc

        betas = [0.0]
        warning = False
        t = 0
        launched = polls = 0
        while betas[-1] < 1.0:
            t += 1
            if t > max_steps:
                raise capi.AsmcError(abi.ERR_EVALUATION,
                                     f"online adaptation failed to reach beta = 1 within {max_steps} steps")
            beta = betas[-1]
            for s in shards:
                s.eval()
            log_m0 = None

            def dhat(b2):
                nonlocal probes
                probes += 1
                allp = gathered([s.probe(beta, b2) for s in shards])
                raw = _lacc_total(fold(allp, 1)) - 2.0 * _lacc_total(fold(allp, 0)) + log_m0
                return raw if raw > 0.0 else 0.0

            if device_search:
                for s in shards:
                    s.search_begin(t, delta_star)
                zp = [torch.empty((s.chunks, 2, 2), dtype=torch.float64, device=dev) for s in shards]
                batch = 2 + _bisect_probes(beta) + 15
                while True:
                    for _ in range(batch):
                        for s, z in zip(shards, zp):
                            s.probe_dev(z.data_ptr())
                        allz = comm.allgather(zp, n_chunks)
                        for s, a in zip(shards, allz):
                            s.search_step(a.data_ptr(), a.shape[0])
                        launched += 1
                    polls += 1
                    done, b, w, taken = shards[0].search_poll()
                    if done:
                        break
                    batch = 8
                probes += taken
            else:
                log_m0 = _lacc_total(fold(gathered([s.probe(beta, -1.0) for s in shards]), 0))
                if log_m0 == -math.inf:
                    raise capi.AsmcError(abi.ERR_DEGENERATE, "all log-weights are -inf")
                b, w = zja_search(dhat, beta, delta_star)
                for s in shards:
                    s.set_beta(t, b)
            warning = warning or w
            betas.append(b)
            for s, p in zip(shards, parts):
                s.step(t, p.data_ptr())
            allp = comm.allgather(parts, n_chunks)
            for s, a, bt in zip(shards, allp, lws):  # policy never: no exchange
                s.decide(t, a.data_ptr(), a.shape[0], bt.data_ptr())
        reps = [s.report(t) for s in shards]
    stream.synchronize()
    for s in shards:
        s.close()
    for r in reps:
        r.update(betas=np.array(betas), steps=t, warning=warning, delta_star=delta_star)
    if stats is not None:
        stats["probes"] = probes  # incl. the log_m0 probe on the device path
        if device_search:
            stats["probes_launched"] = launched  # incl. no-op probes after the search ended
            stats["host_syncs"] = polls
            stats["collectives"] = launched + t
        else:
            stats["host_syncs"] = probes + t
            stats["collectives"] = probes + 2 * t  # probes + log_m0 + step partials per step
    return reps
