"""Multi-GPU SSMC host logic (paper_2408_12057_b200/distributed.py run_smc_sharded)
on CPU: the chunk-partial allgather, the block-total allgather, the slot-range
rule and the all-to-all-v of resampled rows -- with a stand-in shard whose
weights and states are deterministic functions of the GLOBAL particle id, so the
only thing that can differ between world sizes is the exchange itself.

The property the device path relies on: systematic resampling over shards
(each shard resolving the output slots whose position falls in its part of the
CDF, engine.cpp:61-80) picks exactly the ancestors of one global lower_bound,
and the rows land in slot order on the shard that owns the slot."""
import bisect
import math
import socket

import numpy as np
import pytest

from paper_2408_12057_b200 import distributed

CHUNK, BLOCK = 64, 8


def pos(m, u, n, total):  # engine.cpp:68-70 operation order (IEEE double, as on device)
    return ((m + u) / n) * total


class FakeShard:
    """Stand-in for asmc_smc_shard_*: state row = (global id of the original particle, generation)."""

    def __init__(self, n, p0, p1, T, seed):
        import torch
        self.torch = torch
        self.n, self.p0, self.p1, self.T, self.seed = n, p0, p1, T, seed
        self.nl = p1 - p0
        self.chunks = -(-self.nl // CHUNK)
        self.blocks = -(-self.nl // BLOCK)
        self.row_bytes = 16
        self.device = "cpu"
        self.state = torch.stack([torch.arange(p0, p1, dtype=torch.float64),
                                  torch.zeros(self.nl, dtype=torch.float64)], 1)
        self.lw = [0.0] * self.nl
        self.resample_times = []

    def step(self, t, partials):
        for j in range(self.nl):
            x = float(self.state[j, 0])
            self.lw[j] += 3.0 * math.sin(0.731 * x + 1.37 * t + self.seed)
        partials.zero_()
        for c in range(self.chunks):
            seg = self.lw[c * CHUNK:(c + 1) * CHUNK]
            partials[c, 0, 0] = max(seg)

    def decide(self, t, allp, btot):
        self.gmax = float(allp[:, 0, 0].max())
        self.u = (math.sin(17.0 * t + self.seed) + 1.0) / 2.0 * 0.999
        fire = t % 2 == 0 or t == self.T
        if fire:
            self.resample_times.append(t)
            self.cum = [0.0] * self.nl
            for b in range(self.blocks):
                s = 0.0
                for j in range(b * BLOCK, min(self.nl, (b + 1) * BLOCK)):
                    s += math.exp(self.lw[j] - self.gmax)
                    self.cum[j] = s
                btot[b] = s
        return fire

    def plan(self, allb, bounds):
        vals = [float(v) for v in allb]
        boff, off = [], 0.0
        for v in vals:  # cdf_scan_kernel: sequential exclusive scan
            boff.append(off)
            off += v
        total = off
        b0 = self.p0 // BLOCK
        self.cum = [c + boff[b0 + j // BLOCK] for j, c in enumerate(self.cum)]
        G = len(bounds) - 1
        slots = [0] * (G + 1)
        slots[G] = self.n
        for r in range(1, G):  # shard_bounds_kernel
            rb = bounds[r] // BLOCK
            thr = boff[rb] if rb < len(boff) else total
            lo, hi = 0, self.n
            while lo < hi:
                mid = (lo + hi) // 2
                if pos(mid, self.u, self.n, total) <= thr:
                    lo = mid + 1
                else:
                    hi = mid
            slots[r] = lo
        self.total, self.slots = total, slots
        self.me = bounds.index(self.p0)
        return slots

    def pack(self, rows):
        lo, hi = self.slots[self.me], self.slots[self.me + 1]
        out = rows.view(self.torch.float64).reshape(-1, 2)
        for i, m in enumerate(range(lo, hi)):
            j = bisect.bisect_left(self.cum, pos(m, self.u, self.n, self.total))
            out[i] = self.state[min(j, self.nl - 1)]
            out[i, 1] += 1

    def accept(self, rows):
        self.state = rows.view(self.torch.float64).reshape(-1, 2).clone()
        self.lw = [0.0] * self.nl

    def report(self):
        return {"state": self.state.numpy().copy(), "resample_times": self.resample_times}


def run(rank, world, n, T, seed, comm=None):
    bounds = [b for b, _ in distributed.chunk_partition(n, world, CHUNK)] + [n]
    if comm is None:  # all shards in this process
        shards = [FakeShard(n, bounds[r], bounds[r + 1], T, seed) for r in range(world)]
        reps = distributed.run_smc_sharded(shards, list(range(world)), distributed.VirtualComm(world),
                                           bounds, chunk=CHUNK, block=BLOCK)
        return np.concatenate([r["state"] for r in reps]), reps[0]["resample_times"]
    shard = FakeShard(n, bounds[rank], bounds[rank + 1], T, seed)
    (rep,) = distributed.run_smc_sharded([shard], [rank], comm, bounds, chunk=CHUNK, block=BLOCK)
    return rep["state"], rep["resample_times"]


def global_reference(n, T, seed):
    """Single-array systematic resampling with the blocked CDF (no shards at all)."""
    state = np.stack([np.arange(n, dtype=np.float64), np.zeros(n)], 1)
    lw = np.zeros(n)
    for t in range(1, T + 1):
        lw = lw + np.array([3.0 * math.sin(0.731 * x + 1.37 * t + seed) for x in state[:, 0]])
        if not (t % 2 == 0 or t == T):
            continue
        gmax = lw.max()
        cum, off = np.zeros(n), 0.0
        for b in range(-(-n // BLOCK)):
            s = 0.0
            for j in range(b * BLOCK, min(n, (b + 1) * BLOCK)):
                s += math.exp(lw[j] - gmax)
                cum[j] = s
            for j in range(b * BLOCK, min(n, (b + 1) * BLOCK)):
                cum[j] = cum[j] + off
            off += s
        u = (math.sin(17.0 * t + seed) + 1.0) / 2.0 * 0.999
        anc = [min(bisect.bisect_left(list(cum), pos(m, u, n, off)), n - 1) for m in range(n)]
        state = state[anc].copy()
        state[:, 1] += 1
        lw = np.zeros(n)
    return state


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_virtual_shards_match_global_resampling(world):
    n, T = 5 * CHUNK + 13, 5
    ref = global_reference(n, T, 0)
    got, times = run(0, world, n, T, 0)
    assert times == [2, 4, 5]
    assert np.array_equal(got, ref)
    assert got[:, 1].max() == 3


def test_exchange_splits_cover_every_slot_once():
    bounds = [0, 64, 128, 200]
    for slots in ([0, 0, 200, 200], [0, 50, 150, 200], [0, 200, 200, 200], [0, 64, 128, 200]):
        sp = distributed.exchange_splits(slots, bounds)
        assert [sum(r) for r in sp] == [slots[r + 1] - slots[r] for r in range(3)]
        assert [sum(sp[r][q] for r in range(3)) for q in range(3)] == [64, 64, 72]


def _worker(rank, world, port, q, n, T):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        state, times = run(rank, world, n, T, 1, distributed.TorchComm(rank, world))
        q.put((rank, state.tolist(), times))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_ssmc_exchange_matches_single_rank():
    import torch.multiprocessing as mp
    n, T = 4 * CHUNK + 29, 4
    ref = global_reference(n, T, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, n, T)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, state, times = q.get(timeout=120)
        got[rank] = (np.array(state), times)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][1] == got[1][1] == [2, 4]
    assert np.array_equal(np.concatenate([got[0][0], got[1][0]]), ref)
