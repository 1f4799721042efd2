"""Multi-process (gloo, world_size 2 and 3) tests of the orchestration in
paper_1208_3933_b200/dist.py: incumbent MIN all-reduce, deterministic work
stealing, termination, winner broadcast.  On CPU the per-rank engine is a
host-side step-level B&B over the oracle's bound (test infrastructure)."""
import itertools
import os
import socket

import numpy as np
import pytest

from paper_1208_3933_b200 import dist as fdist


# ------------------------------------------------------------ pure functions

def test_shard_covers_exactly():
    for N in (0, 1, 7, 1000, 1 << 20):
        for R in (1, 2, 3, 8):
            parts = [fdist.shard(N, r, R) for r in range(R)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(R - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


def test_plan_rebalance_properties():
    rng = np.random.default_rng(0)
    for _ in range(300):
        R = int(rng.integers(2, 9))
        sizes = [int(x) for x in rng.integers(0, 1000, R)]
        if rng.random() < 0.3:
            sizes[int(rng.integers(R))] = 0
        plan = fdist.plan_rebalance(sizes, max_chunk=10_000)
        assert plan == fdist.plan_rebalance(list(sizes), max_chunk=10_000)  # deterministic
        after = list(sizes)
        for d, r, k in plan:
            assert d != r and k > 0 and after[d] >= k
            after[d] -= k
            after[r] += k
        assert sum(after) == sum(sizes)
        if sum(sizes) >= 2 * R and min(sizes) == 0:
            assert plan, sizes            # an idle rank gets work
        assert max(after) - min(after) <= max(sizes) - min(sizes)


def test_pack_unpack():
    for inc, r in [(0, 0), (1278, 3), (2**31 - 1, 7)]:
        w = fdist.pack_ub(inc, r)
        assert fdist.unpack_ub(w) == (inc, r)
        assert (w < fdist.pack_ub(inc + 1, 0)) or inc == 2**31 - 1


# ------------------------------------------------ host engine (test double)

class HostEngine:
    """Step-level B&B on the host with the oracle's bound: same interface as
    dist.DeviceEngine, nodes exported as int16 rows [k][n] + depths."""

    def __init__(self, ptm, rank, world, initial_ub=2**31 - 1):
        import oracle
        self.T = oracle.Tables(ptm)
        self.p = ptm
        self.n = ptm.shape[0]
        self.rank = rank
        self.inc = initial_ub + 1 if initial_ub < 2**31 - 1 else 2**31 - 1
        self.best = None
        self.best_ms = None
        self.bounded = 0
        n = self.n
        self.stack = [[]] if world == 1 else [[j] for j in range(n - 1, -1, -1) if j % world == rank]

    def step(self, iters):
        import oracle
        for _ in range(iters):
            if not self.stack:
                return
            node = self.stack.pop()
            rest = [j for j in range(self.n) if j not in node]
            kids = []
            for j in rest:
                child = node + [j]
                lb = self.T.lb(child)
                self.bounded += 1
                if len(child) >= self.n - 1:
                    full = child + [q for q in rest if q != j]
                    ms = oracle.makespan(self.p, full)
                    assert ms == lb
                    if ms < self.inc:
                        self.inc, self.best, self.best_ms = ms, full, ms
                elif lb < self.inc:
                    kids.append((lb, child))
            for lb, child in sorted(kids, key=lambda x: -x[0]):
                self.stack.append(child)

    def pool_size(self):
        return len(self.stack)

    def ub_get(self):
        return fdist.pack_ub(self.best_ms if self.best is not None else 2**31 - 1, self.rank)

    def ub_set(self, word):
        self.inc = min(self.inc, fdist.unpack_ub(word)[0])

    def status_word(self, elapsed_ms, device):
        import torch
        return torch.tensor([self.ub_get(), self.pool_size(), self.bounded, elapsed_ms],
                            dtype=torch.int64, device=device)

    def stats(self):
        return {"bounded": self.bounded}

    def result(self):
        if self.best is None:
            return -5, -1, None
        return 0, self.best_ms, np.array(self.best, np.int32)

    def alloc_node_buffer(self, k):
        import torch
        return torch.zeros(k * (self.n + 1), dtype=torch.int32)

    def export_nodes(self, k):
        import torch
        out = []
        for _ in range(min(k, len(self.stack))):
            out.append(self.stack.pop(0))      # shallowest first
        buf = torch.full((len(out), self.n + 1), -1, dtype=torch.int32)
        for i, nd in enumerate(out):
            buf[i, 0] = len(nd)
            buf[i, 1:1 + len(nd)] = torch.tensor(nd, dtype=torch.int32)
        return buf.flatten(), len(out)

    def import_nodes(self, buf, k):
        rows = buf.view(k, self.n + 1)
        for i in range(k):
            d = int(rows[i, 0])
            self.stack.append([int(x) for x in rows[i, 1:1 + d]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ptm, initial_ub, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = HostEngine(ptm, rank, world, initial_ub)
        res = fdist.distributed_bb(eng, dist, rank=rank, world=world, device="cpu",
                                   sync_every=3, max_chunk=4)
        q.put((rank, res.status, res.makespan, res.perm.tolist(), res.winner, res.moved,
               res.bounded))
    finally:
        dist.destroy_process_group()


def _run(world, ptm, initial_ub=2**31 - 1):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ptm, initial_ub, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def _brute(p):
    best = None
    for q in itertools.permutations(range(p.shape[0])):
        m = p.shape[1]
        C = [0] * m
        for j in q:
            prev = 0
            for k in range(m):
                C[k] = max(C[k], prev) + int(p[j, k])
                prev = C[k]
        best = C[-1] if best is None else min(best, C[-1])
    return best


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_distributed_bb_matches_bruteforce(world, orc):
    rng = np.random.default_rng(world)
    for _ in range(2):
        p = rng.integers(1, 50, (7, 4)).astype(np.int32)
        opt = _brute(p)
        out = _run(world, p)
        ms = {o[2] for o in out}
        perms = {tuple(o[3]) for o in out}
        assert ms == {opt}, (ms, opt)
        assert len(perms) == 1                       # the winner's broadcast
        assert orc.makespan(p, list(perms.pop())) == opt
        assert all(o[1] == 0 for o in out)


def test_gloo_distributed_bb_notfound(orc):
    rng = np.random.default_rng(9)
    p = rng.integers(1, 50, (6, 3)).astype(np.int32)
    opt = _brute(p)
    out = _run(2, p, initial_ub=opt - 1)
    assert all(o[1] == 1 and o[2] == -1 for o in out)
    out = _run(2, p, initial_ub=opt)
    assert all(o[1] == 0 and o[2] == opt for o in out)
