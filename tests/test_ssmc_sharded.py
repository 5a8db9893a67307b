"""Multi-GPU SSMC host logic (paper_2408_12057_b200/distributed.py run_smc_sharded)
on CPU: the chunk-partial allgather, the log-weight allgather, the slot-range rule
and the all-to-all-v of resampled rows -- with a stand-in shard whose weights and
states are deterministic functions of the GLOBAL particle id, so the only thing that
can differ between world sizes is the exchange itself.

The property the device path relies on: every rank builds the same global sequential
CDF (engine.cpp:61-80) from the all-gathered log-weights, the ancestors a_m are
non-decreasing in m, so the slots whose ancestor lies in shard r are one contiguous
range, and the rows land in slot order on the shard that owns the slot."""
import bisect
import math
import socket

import numpy as np
import pytest

from paper_2408_12057_b200 import distributed

CHUNK = 64


def ref_ancestors(lw, u):
    """engine.cpp:61-80 in plain Python floats (IEEE double, sequential order)."""
    n = len(lw)
    mx, sm = -math.inf, 0.0  # LogAccumulator (logsum.hpp:18-45)
    for v in lw:
        if v == -math.inf:
            continue
        if v <= mx:
            sm += math.exp(v - mx)
        else:
            sm = sm * math.exp(mx - v) + 1.0
            mx = v
    l1 = mx + math.log(sm)
    out, cum, j = [], math.exp(lw[0] - l1), 0
    for m in range(n):
        p = (m + u) / n
        while cum < p and j + 1 < n:
            j += 1
            cum += math.exp(lw[j] - l1)
        out.append(j)
    return out


class FakeShard:
    """Stand-in for asmc_smc_shard_*: state row = (global id of the original particle, generation)."""

    def __init__(self, n, p0, p1, T, seed):
        import torch
        self.torch = torch
        self.n, self.p0, self.p1, self.T, self.seed = n, p0, p1, T, seed
        self.nl = p1 - p0
        self.chunks = -(-self.nl // CHUNK)
        self.exchange_len = self.nl
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

    def decide(self, t, allp, lw_out):
        self.u = (math.sin(17.0 * t + self.seed) + 1.0) / 2.0 * 0.999
        fire = t % 2 == 0 or t == self.T
        if fire:
            self.resample_times.append(t)
            for j in range(self.nl):
                lw_out[j] = self.lw[j]
        return fire

    def plan(self, all_lw, bounds):
        self.anc = ref_ancestors([float(v) for v in all_lw], self.u)
        G = len(bounds) - 1
        slots = [bisect.bisect_left(self.anc, bounds[r]) for r in range(G)] + [self.n]
        self.slots = slots
        self.me = bounds.index(self.p0)
        return slots

    def pack(self, rows):
        lo, hi = self.slots[self.me], self.slots[self.me + 1]
        out = rows.view(self.torch.float64).reshape(-1, 2)
        for i, m in enumerate(range(lo, hi)):
            j = self.anc[m] - self.p0
            assert 0 <= j < self.nl
            out[i] = self.state[j]
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
                                           bounds, chunk=CHUNK)
        return np.concatenate([r["state"] for r in reps]), reps[0]["resample_times"]
    shard = FakeShard(n, bounds[rank], bounds[rank + 1], T, seed)
    (rep,) = distributed.run_smc_sharded([shard], [rank], comm, bounds, chunk=CHUNK)
    return rep["state"], rep["resample_times"]


def global_reference(n, T, seed):
    """Single-array systematic resampling, the reference rule (no shards at all)."""
    state = np.stack([np.arange(n, dtype=np.float64), np.zeros(n)], 1)
    lw = np.zeros(n)
    for t in range(1, T + 1):
        lw = lw + np.array([3.0 * math.sin(0.731 * x + 1.37 * t + seed) for x in state[:, 0]])
        if not (t % 2 == 0 or t == T):
            continue
        u = (math.sin(17.0 * t + seed) + 1.0) / 2.0 * 0.999
        anc = ref_ancestors([float(v) for v in lw], u)
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
