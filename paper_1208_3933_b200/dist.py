"""Multi-GPU orchestration: one process per GPU,
torch.distributed for the collectives, libfsp for every compute step.

* Bounding pools shard with no data-path collective: rank r bounds the
  contiguous slice [r*N/R, (r+1)*N/R) of a pool (``shard``).
* The device B&B shares one scalar, the incumbent: every ``sync_every`` local
  iterations each rank publishes (own best << 32 | rank), a MIN all-reduce
  (NCCL over NVLink on GPUs, gloo on CPU) picks the global one, every rank
  adopts it.  Pool sizes are all-gathered; a deterministic plan pairs donors
  with starving ranks and open nodes move point to point (the shallowest nodes
  of the donor, i.e. the largest subtrees).  The search ends when every pool is
  empty after a synchronisation.  The winner (low 32 bits of the reduced word)
  broadcasts its permutation.

The per-rank engine is anything with the step interface of ``binding.BBState``
(step / pool_size / ub_get / ub_set / export_nodes / import_nodes / result /
stats); tests drive this module on CPU with gloo and a host-side engine.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

INT32_MAX = 2**31 - 1


def shard(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous static shard [lo, hi) of n_items for rank (weak scaling)."""
    lo = n_items * rank // world
    hi = n_items * (rank + 1) // world
    return lo, hi


def plan_rebalance(sizes, max_chunk: int = 1 << 16, slack: float = 0.25, min_give: int = 1):
    """Deterministic donor -> receiver transfers from the all-gathered pool sizes.

    Ranks above mean*(1+slack) donate down to the mean; ranks below
    mean*(1-slack) (in particular empty ones) receive up to the mean.  Donors
    and receivers are matched greedily, largest surplus with largest deficit,
    ties by rank.  Returns [(donor, receiver, count)], count <= max_chunk."""
    sizes = [int(s) for s in sizes]
    R = len(sizes)
    total = sum(sizes)
    if R < 2 or total == 0:
        return []
    mean = total / R
    surplus = {r: sizes[r] - int(mean) for r in range(R) if sizes[r] > mean * (1 + slack)}
    deficit = {r: int(np.ceil(mean)) - sizes[r] for r in range(R)
               if sizes[r] < mean * (1 - slack) or sizes[r] == 0}
    donors = sorted(surplus, key=lambda r: (-surplus[r], r))
    recvs = sorted(deficit, key=lambda r: (-deficit[r], r))
    plan = []
    di = ri = 0
    while di < len(donors) and ri < len(recvs):
        d, r = donors[di], recvs[ri]
        k = min(surplus[d], deficit[r], max_chunk)
        if k >= min_give:
            plan.append((d, r, k))
        surplus[d] -= k
        deficit[r] -= k
        if surplus[d] < min_give:
            di += 1
        if deficit[r] < min_give:
            ri += 1
        if k < min_give:
            break
    return plan


def pack_ub(incumbent: int, rank: int) -> int:
    return (int(incumbent) << 32) | int(rank)


def unpack_ub(word: int) -> tuple[int, int]:
    return int(word) >> 32, int(word) & 0xFFFFFFFF


@dataclass
class DistResult:
    status: int          # 0 optimal, 1 none <= initial_ub, 2 budget exhausted
    makespan: int
    perm: np.ndarray
    winner: int
    bounded: int         # summed over ranks
    rounds: int
    moved: int           # open nodes moved between ranks
    wall_s: float


def _allreduce_min_i64(dist, group, value: int, device) -> int:
    import torch
    t = torch.tensor([value], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


def _allgather_i64(dist, group, value: int, world: int, device) -> list[int]:
    import torch
    t = torch.tensor([value], dtype=torch.int64, device=device)
    out = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def distributed_bb(engine, dist, group=None, *, rank: int, world: int, device="cpu",
                   sync_every: int = 4, time_limit_s: float = 0.0, max_chunk: int = 1 << 16,
                   bounded_budget: int = 0) -> DistResult:
    """Run the device B&B on every rank with incumbent sharing and work
    stealing.  ``engine`` is this rank's step-level B&B; ``device`` is where
    collective tensors live ("cuda" for NCCL, "cpu" for gloo)."""
    import torch
    t0 = time.perf_counter()
    rounds = moved = 0
    stop = False
    while True:
        engine.step(sync_every)
        # ONE collective per round: all-gather of [ub word, pool size, bounded,
        # elapsed ms]; the MIN of the ub words is the global incumbent (low 32
        # bits: its holder), the sums/max drive termination and the budget
        st = engine.status_word(int((time.perf_counter() - t0) * 1e3), device)
        out = torch.empty(world * 4, dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(out, st, group=group)
        rows = out.view(world, 4).cpu().numpy()
        engine.ub_set(int(rows[:, 0].min()))
        sizes = [int(x) for x in rows[:, 1]]
        rounds += 1
        if sum(sizes) == 0:
            break
        # budget: every rank sees the same gathered counters -> same decision
        if (time_limit_s > 0 and int(rows[:, 3].max()) >= time_limit_s * 1e3) or \
                (bounded_budget > 0 and int(rows[:, 2].sum()) >= bounded_budget):
            stop = True
            break
        for donor, recv, k in plan_rebalance(sizes, max_chunk):
            if rank == donor:
                buf, got = engine.export_nodes(k)
                hdr = torch.tensor([got], dtype=torch.int64, device=device)
                dist.send(hdr, recv, group=group)
                if got:
                    dist.send(buf, recv, group=group)
                moved += got
            elif rank == recv:
                hdr = torch.zeros(1, dtype=torch.int64, device=device)
                dist.recv(hdr, donor, group=group)
                got = int(hdr.item())
                if got:
                    buf = engine.alloc_node_buffer(got)
                    dist.recv(buf, donor, group=group)
                    engine.import_nodes(buf, got)
                moved += got
    g = _allreduce_min_i64(dist, group, engine.ub_get(), device)
    inc, winner = unpack_ub(g)
    n = engine.n
    perm = torch.zeros(n, dtype=torch.int32, device=device)
    have = inc < INT32_MAX
    if have and rank == winner:
        rc, ms, p = engine.result()
        assert rc == 0 and ms == inc, (rc, ms, inc)
        perm.copy_(torch.from_numpy(p))
    if have:
        dist.broadcast(perm, winner, group=group)
    total_bounded = sum(_allgather_i64(dist, group, int(engine.stats()["bounded"]), world, device))
    moved_total = sum(_allgather_i64(dist, group, moved, world, device))
    status = 2 if stop else (0 if have else 1)
    return DistResult(status, inc if have else -1, perm.cpu().numpy(), winner if have else -1,
                      total_bounded, rounds, moved_total, time.perf_counter() - t0)


class DeviceEngine:
    """Adapter: binding.BBState on this rank's GPU.  Node buffers are CUDA
    uint8 tensors (NCCL point-to-point over NVLink); with comm_device="cpu"
    (gloo) they are staged through host memory."""

    def __init__(self, state, device, comm_device=None):
        self.state = state
        self.n = state.n
        self.device = device
        self.comm = comm_device or device
        self.node_bytes = state.node_bytes()

    def step(self, iters):
        self.state.step(iters)

    def pool_size(self):
        return self.state.pool_size()

    def ub_get(self):
        return self.state.ub_get()

    def ub_set(self, word):
        self.state.ub_set(word)

    def status_word(self, elapsed_ms, device):
        """[ub word, pool size, bounded, elapsed ms] as an int64 tensor on the
        collective's device; on CUDA the ub word is written device-to-device
        by fsp_bb_ub_publish (stream-ordered before the collective)."""
        import torch
        t = torch.tensor([0, self.pool_size(), int(self.stats()["bounded"]), elapsed_ms],
                         dtype=torch.int64, device=device)
        if t.is_cuda:
            self.state.ub_publish(t[0:1])
        else:
            t[0] = self.ub_get()
        return t

    def stats(self):
        return self.state.stats()

    def result(self):
        return self.state.result()

    def alloc_node_buffer(self, k):
        import torch
        return torch.empty(k * self.node_bytes, dtype=torch.uint8, device=self.comm)

    def export_nodes(self, k):
        import torch
        buf = torch.empty(k * self.node_bytes, dtype=torch.uint8, device=self.device)
        got = self.state.export(k, buf.data_ptr())
        out = buf[:got * self.node_bytes]
        return (out if self.comm == self.device else out.to(self.comm)), got

    def import_nodes(self, buf, k):
        import torch
        if buf.device.type != "cuda":
            buf = buf.to(self.device)
        # an NCCL recv only orders torch's current stream; fsp_bb_import copies
        # on the state's own stream, so the data must have landed first
        torch.cuda.current_stream(buf.device).synchronize()
        self.state.import_(buf.data_ptr(), k)
