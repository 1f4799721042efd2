"""GPU parity of the device B&B (fsp_bb_solve / step API) against the oracle.

The optimum is unique, the permutation is not: checks are makespan(perm) ==
returned makespan == oracle / brute-force optimum."""
import itertools

import numpy as np
import pytest

from paper_1208_3933_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fsp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1208_3933_b200 import binding
    binding.lib()
    return binding


def brute(p):
    n = p.shape[0]
    best = None
    for q in itertools.permutations(range(n)):
        m = p.shape[1]
        C = [0] * m
        for j in q:
            prev = 0
            for k in range(m):
                C[k] = max(C[k], prev) + int(p[j, k])
                prev = C[k]
        best = C[-1] if best is None else min(best, C[-1])
    return best


def test_bb_bruteforce(fsp, orc):
    rng = np.random.default_rng(31)
    for _ in range(40):
        n, m = int(rng.integers(1, 8)), int(rng.integers(2, 6))
        p = rng.integers(1, 40, (n, m)).astype(np.int32)
        opt = brute(p)
        inst = fsp.Instance(p)
        rc, ms, perm, st = inst.bb_solve()
        assert rc == 0 and ms == opt, (p.tolist(), ms, opt)
        assert orc.makespan(p, perm) == opt and sorted(perm.tolist()) == list(range(n))
        rc, ms, perm, _ = inst.bb_solve(opt)             # UB equal to the optimum: found (R9)
        assert rc == 0 and ms == opt
        if opt > 0:
            rc, ms, _, _ = inst.bb_solve(opt - 1)         # below it: none
            assert rc == fsp.FSP_ENOTFOUND


def test_bb_matches_oracle_medium(fsp, orc):
    rng = np.random.default_rng(77)
    for _ in range(6):
        n, m = int(rng.integers(9, 13)), int(rng.integers(3, 6))
        p = rng.integers(1, 99, (n, m)).astype(np.int32)
        orc_rc, orc_ms, _, _ = orc.Tables(p).bb_dfs()
        rc, ms, perm, st = fsp.Instance(p).bb_solve()
        assert rc == 0 and orc_rc == 0 and ms == orc_ms
        assert orc.makespan(p, perm) == ms


def test_bb_m2_johnson(fsp, orc):
    rng = np.random.default_rng(5)
    for _ in range(5):
        n = int(rng.integers(5, 60))
        p = rng.integers(1, 99, (n, 2)).astype(np.int32)
        order = orc.johnson_order(p[:, 0], p[:, 1])
        rc, ms, perm, _ = fsp.Instance(p).bb_solve()
        assert rc == 0 and ms == orc.makespan(p, order) == orc.makespan(p, perm)


@pytest.mark.parametrize("name,opt", [("ta001", 1278), ("ta002", 1359), ("ta003", 1081),
                                      ("ta004", 1293)])
def test_bb_taillard_optimum(fsp, orc, name, opt):
    # BASELINE.json configs[0]: full B&B from the root (no initial UB) to the
    # optimum; ta002-ta004 optima recalled (tests/golden/taillard_optima.txt)
    p = inputs.instance(name)
    rc, ms, perm, st = fsp.Instance(p).bb_solve(2**31 - 1, 0, 120.0)
    assert rc == 0 and ms == opt and orc.makespan(p, perm) == opt
    assert sorted(perm.tolist()) == list(range(p.shape[0]))
    # and the proof: nothing at or below opt - 1
    rc, _, _, _ = fsp.Instance(p).bb_solve(opt - 1, 0, 120.0)
    assert rc == fsp.FSP_ENOTFOUND


def _completion(p, row, d):
    m = p.shape[1]
    C = np.zeros(m, np.int64)
    for j in row[:d]:
        prev = 0
        for k in range(m):
            C[k] = max(C[k], prev) + int(p[j, k])
            prev = C[k]
    return C


@pytest.mark.parametrize("name,snapshots,sample", [("ta001", (1, 2, 5, 20, 60), 0),
                                                   ("ta021", (1, 3, 10, 40), 4000),
                                                   ("ta091", (1, 4, 30, 200), 1500)])
def test_bb_child_pool_lbs_match_oracle(fsp, orc, name, snapshots, sample):
    """Element-wise parity of the device B&B's bounding step: after a number of
    iterations, the last iteration's child pool (prefixes built by expand,
    completion times carried from the parents, LBs from the sparse-walk plan
    with the pool size read on the device) is exported and every child's LB
    (sample = 0) or a random sample of them is recomputed by the oracle."""
    p = inputs.instance(name)
    n = p.shape[0]
    inst = fsp.Instance(p)
    T = orc.Tables(p)
    bb = fsp.BBState(inst)
    rng = np.random.default_rng(7)
    done = 0
    checked = 0
    for it in snapshots:
        bb.step(it - done)
        done = it
        if bb.pool_size() == 0:
            break
        pf, dp, Cc, lb = bb.debug_children()
        k = len(dp)
        if k == 0:      # every popped parent was eliminated at pop (R9)
            continue
        idx = np.arange(k) if sample == 0 or k <= sample else np.sort(
            np.concatenate([rng.choice(k - 32, sample - 32, replace=False), np.arange(k - 32, k)]))
        want = T.lb_eval(pf[idx], dp[idx])
        bad = np.nonzero(want != lb[idx])[0]
        assert bad.size == 0, (name, it, idx[bad[:5]], lb[idx][bad[:5]], want[bad[:5]])
        for i in idx[:: max(1, len(idx) // 200)]:
            d = int(dp[i])
            row = pf[i, :d].astype(np.int64)
            assert len(set(row.tolist())) == d and row.max(initial=0) < n
            assert (Cc[i] == _completion(p, row, d)).all()
        checked += len(idx)
    assert checked > 0


def test_bb_budget(fsp, orc):
    p = inputs.instance("ta021")
    rc, ms, perm, st = fsp.Instance(p).bb_solve(2**31 - 1, 200000, 0.0)
    assert rc in (fsp.FSP_EBUDGET, fsp.FSP_ENOTFOUND)
    assert st["bounded"] >= 200000
    if rc == fsp.FSP_EBUDGET:
        assert orc.makespan(p, perm) == ms


def test_bb_two_ranks_one_gpu(fsp, orc):
    """The step API with world=2 on one device: host-side MIN of the packed
    incumbents stands in for the NCCL all-reduce; the optimum must equal the
    single-rank one; export/import move open nodes between the ranks."""
    import torch
    rng = np.random.default_rng(12)
    for _ in range(4):
        n, m = int(rng.integers(6, 11)), int(rng.integers(3, 6))
        p = rng.integers(1, 60, (n, m)).astype(np.int32)
        opt = orc.Tables(p).bb_dfs()[1]
        inst = fsp.Instance(p)
        ranks = [fsp.BBState(inst, 2**31 - 1, r, 2) for r in range(2)]
        buf = torch.empty(4096 * ranks[0].node_bytes(), dtype=torch.uint8, device="cuda")
        for it in range(100000):
            for s in ranks:
                s.step(2)
            g = min(s.ub_get() for s in ranks)       # the MIN all-reduce, on the host
            for s in ranks:
                s.ub_set(g)
            sizes = [s.pool_size() for s in ranks]
            if sum(sizes) == 0:
                break
            # rebalance: the larger pool donates half of the difference
            a, b = (0, 1) if sizes[0] >= sizes[1] else (1, 0)
            give = min((sizes[a] - sizes[b]) // 2, 4096)
            if give > 0:
                k = ranks[a].export(give, buf.data_ptr())
                ranks[b].import_(buf.data_ptr(), k)
        results = [s.result() for s in ranks]
        best = min(r[1] for r in results if r[0] == 0)
        assert best == opt
        for rc, ms, perm in results:
            if rc == 0:
                assert orc.makespan(p, perm) == ms


def test_distributed_driver_nccl_world1(fsp, orc):
    """dist.distributed_bb over a real NCCL process group (world 1) with the
    device engine: the adapter path bench.py uses on N GPUs."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1208_3933_b200 import dist as fdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(3)
        p = rng.integers(1, 60, (9, 4)).astype(np.int32)
        opt = orc.Tables(p).bb_dfs()[1]
        inst = fsp.Instance(p)
        eng = fdist.DeviceEngine(fsp.BBState(inst, 2**31 - 1, 0, 1), "cuda")
        res = fdist.distributed_bb(eng, dist, rank=0, world=1, device="cuda", sync_every=2)
        assert res.status == 0 and res.makespan == opt
        assert orc.makespan(p, res.perm) == opt
    finally:
        dist.destroy_process_group()


def _gloo_device_worker(rank, world, port, ptm, q):
    import os

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["FSP_BB_MEM_FRAC"] = "0.05"
    os.environ["FSP_BB_CHILDREN"] = str(1 << 16)
    from paper_1208_3933_b200 import binding
    from paper_1208_3933_b200 import dist as fdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = binding.Instance(ptm)
        state = binding.BBState(inst, 2**31 - 1, rank, world)
        eng = fdist.DeviceEngine(state, "cuda", "cpu")
        # forced imbalance: rank 1 hands its whole start pool to rank 0, so
        # the work stealing has to move nodes back
        nb = eng.node_bytes
        if rank == 1:
            buf, got = eng.export_nodes(state.pool_size())
            dist.send(torch.tensor([got]), 0)
            dist.send(buf.cpu(), 0)
        else:
            hdr = torch.zeros(1, dtype=torch.int64)
            dist.recv(hdr, 1)
            k = int(hdr.item())
            buf = torch.empty(k * nb, dtype=torch.uint8)
            dist.recv(buf, 1)
            eng.import_nodes(buf, k)
        sizes0 = state.pool_size()
        res = fdist.distributed_bb(eng, dist, rank=rank, world=world, device="cpu", sync_every=1,
                                   max_chunk=256)
        q.put((rank, sizes0, res.status, res.makespan, res.perm.tolist(), res.moved))
    finally:
        dist.destroy_process_group()


def test_distributed_bb_world2_one_gpu_stealing(fsp, orc):
    """dist.distributed_bb at world 2 (two processes sharing cuda:0, gloo
    collectives, device engines): rank 1 starts empty, nodes must move
    (moved > 0), and both ranks report the oracle optimum."""
    import socket

    import torch.multiprocessing as mp
    rng = np.random.default_rng(21)
    p = rng.integers(1, 99, (13, 6)).astype(np.int32)
    opt = orc.Tables(p).bb_dfs()[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_device_worker, args=(r, 2, port, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert out[1][1] == 0                       # rank 1 started empty
    assert all(o[2] == 0 and o[3] == opt for o in out), (out, opt)
    assert out[0][4] == out[1][4] and orc.makespan(p, out[0][4]) == opt
    assert out[0][5] > 0                        # work stealing moved nodes


def test_bb_family_kernel_optima(fsp, orc, monkeypatch):
    """The B&B with sibling-incremental bounding (FSP_BB_FAMILY=1: batches of
    parents with <= 32 unscheduled jobs bounded by family.cu) reaches the same
    optima; its child pools match the oracle element-wise."""
    monkeypatch.setenv("FSP_BB_FAMILY", "1")
    monkeypatch.setenv("FSP_BB_K", "32")
    for name, opt in (("ta001", 1278), ("ta003", 1081)):
        p = inputs.instance(name)
        rc, ms, perm, _ = fsp.Instance(p).bb_solve(2**31 - 1, 0, 60.0)
        assert rc == 0 and ms == opt and orc.makespan(p, perm) == opt
    rng = np.random.default_rng(8)
    for _ in range(4):
        n, m = int(rng.integers(8, 12)), int(rng.integers(3, 6))
        p = rng.integers(1, 99, (n, m)).astype(np.int32)
        rc, ms, perm, _ = fsp.Instance(p).bb_solve()
        assert rc == 0 and ms == orc.Tables(p).bb_dfs()[1] == orc.makespan(p, perm)
    p = inputs.instance("ta021")
    T = orc.Tables(p)
    bb = fsp.BBState(fsp.Instance(p))
    bb.step(40)
    pf, dp, Cc, lb = bb.debug_children()
    assert len(dp) > 0 and (T.lb_eval(pf, dp) == lb).all()


@pytest.mark.parametrize("threads", [2, 4])
def test_bb_hybrid_threads(fsp, orc, threads):
    """fsp_bb_solve_hybrid (host threads each driving a device B&B state,
    shared incumbent, work stealing): the same optima as the oracle, the
    ENOTFOUND proof below the optimum, budgets honoured."""
    for name, opt in (("ta001", 1278), ("ta002", 1359), ("ta004", 1293)):
        p = inputs.instance(name)
        inst = fsp.Instance(p)
        rc, ms, perm, st = inst.bb_solve_hybrid(threads, 2**31 - 1, 0, 120.0)
        assert rc == 0 and ms == opt and orc.makespan(p, perm) == opt, (name, rc, ms)
        assert sorted(perm.tolist()) == list(range(p.shape[0]))
        rc, _, _, _ = inst.bb_solve_hybrid(threads, opt - 1, 0, 120.0)
        assert rc == fsp.FSP_ENOTFOUND
    rng = np.random.default_rng(threads)
    for _ in range(6):
        n, m = int(rng.integers(1, 11)), int(rng.integers(2, 6))
        p = rng.integers(1, 60, (n, m)).astype(np.int32)
        rc, ms, perm, _ = fsp.Instance(p).bb_solve_hybrid(threads)
        assert rc == 0 and ms == orc.Tables(p).bb_dfs()[1] == orc.makespan(p, perm)
    p = inputs.instance("ta021")
    rc, ms, perm, st = fsp.Instance(p).bb_solve_hybrid(threads, 2**31 - 1, 2_000_000, 0.0)
    assert rc in (fsp.FSP_EBUDGET, fsp.FSP_ENOTFOUND) and st["bounded"] >= 2_000_000
    if rc == fsp.FSP_EBUDGET:
        assert orc.makespan(p, perm) == ms
