"""GPU parity: fsp_lb_eval (CUDA, through the C ABI) vs the CPU oracle.

Bit-exact (integer work, tolerance 0, BASELINE.json north_star) on every node
of seeded pools sized so the oracle finishes in seconds, plus sampled nodes of
the full-size 200x20 pool in the launch configuration bench.py times, plus the
edge cases (empty, ragged, d = 0 / n-1 / n, duplicates, degenerate instances,
malformed nodes).
"""
import numpy as np
import pytest

from paper_1208_3933_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def fsp():
    from paper_1208_3933_b200 import binding
    binding.lib()
    return binding


def dev(torch, a):
    if a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_lb(torch, inst, pf, dp):
    out = inst.lb_eval(dev(torch, pf), dev(torch, dp))
    torch.cuda.synchronize()
    return out.cpu().numpy()


def compare(torch, fsp, orc, ptm, pf, dp):
    inst = fsp.Instance(ptm)
    got = gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_OK
    want = orc.Tables(ptm).lb_eval(pf, dp)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {got[bad[:5]]} want {want[bad[:5]]}"
    return inst


@pytest.mark.parametrize("name,N", [("ta001", 20000), ("ta021", 65536), ("ta051", 16411),
                                    ("ta091", 4133), ("ta111", 1061)])
def test_parity_config_pools(torch, fsp, orc, name, N):
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed(name))
    compare(torch, fsp, orc, ptm, pf, dp)


@pytest.mark.parametrize("d", ["zero", "n-1", "n"])
def test_parity_fixed_depths(torch, fsp, orc, d):
    for name in ("ta021", "ta091"):
        n, m, seed = inputs.TAILLARD_SEEDS[name]
        depth = {"zero": 0, "n-1": n - 1, "n": n}[d]
        pf, dp = inputs.pool_fixed_depth(n, 300, depth, 5)
        compare(torch, fsp, orc, inputs.taillard(n, m, seed), pf, dp)


@pytest.mark.parametrize("m", [2, 3, 7, 11, 13, 17, 25, 32])
def test_parity_machine_counts(torch, fsp, orc, m):
    rng = np.random.default_rng(m)
    n = int(rng.integers(1, 60))
    ptm = rng.integers(0, 99, (n, m)).astype(np.int32)
    pf, dp = inputs.pool_d1(n, 777, 100 + m)
    compare(torch, fsp, orc, ptm, pf, dp)


def test_parity_degenerate_instances(torch, fsp, orc):
    rng = np.random.default_rng(9)
    cases = [np.zeros((17, 6), np.int32),                           # all zero
             np.tile(rng.integers(1, 99, 8), (40, 1)).astype(np.int32),   # identical jobs
             rng.integers(0, 3, (33, 5)).astype(np.int32),           # heavy ties
             rng.integers(0, 32767, (12, 4)).astype(np.int32),       # large times
             np.array([[5, 7]], np.int32)]                           # n = 1
    for ptm in cases:
        n = ptm.shape[0]
        pf, dp = inputs.pool_d1(n, 200, 3)
        pf2, dp2 = inputs.pool_fixed_depth(n, 50, n, 4)
        compare(torch, fsp, orc, ptm, np.concatenate([pf, pf2]), np.concatenate([dp, dp2]))


def test_parity_strides_and_ragged(torch, fsp, orc):
    n, m, seed = inputs.TAILLARD_SEEDS["ta021"]
    ptm = inputs.taillard(n, m, seed)
    for stride in (n, n + 3, 64):
        for N in (1, 31, 33, 257, 1000):
            pf, dp = inputs.pool_d1(n, N, N + stride, stride=stride)
            compare(torch, fsp, orc, ptm, pf, dp)


def test_duplicates_and_empty(torch, fsp, orc):
    n, m, seed = inputs.TAILLARD_SEEDS["ta051"]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 1, 77)
    pf, dp = np.repeat(pf, 999, 0), np.repeat(dp, 999, 0)
    compare(torch, fsp, orc, ptm, pf, dp)
    inst = fsp.Instance(ptm)
    import torch as T
    out = inst.lb_eval(T.zeros((0, 56), dtype=T.int16, device="cuda"),
                       T.zeros(0, dtype=T.int32, device="cuda"))
    assert out.numel() == 0


def test_malformed_nodes_flagged(torch, fsp, orc):
    n, m, seed = inputs.TAILLARD_SEEDS["ta021"]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 500, 8)
    inst = fsp.Instance(ptm)
    gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_OK
    want = orc.Tables(ptm).lb_eval(pf, dp)
    for kind in ("job", "dup", "depth"):
        bad_pf, bad_dp = pf.copy(), dp.copy()
        i = 123
        bad_dp[i] = max(bad_dp[i], 2)
        bad_pf[i, :bad_dp[i]] = np.arange(bad_dp[i])
        if kind == "job":
            bad_pf[i, 0] = n + 5
        elif kind == "dup":
            bad_pf[i, 1] = bad_pf[i, 0]
        else:
            bad_dp[i] = n + 1
        got = gpu_lb(torch, inst, bad_pf, bad_dp)
        assert inst.check() == fsp.FSP_EBADNODE, kind
        assert inst.check() == fsp.FSP_OK           # flag cleared
        keep = np.arange(500) != i
        assert (got[keep] == want[keep]).all(), kind


def test_host_api_matches_device(torch, fsp, orc):
    n, m, seed = inputs.TAILLARD_SEEDS["ta051"]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 300_001, 31)
    inst = fsp.Instance(ptm)
    host = inst.lb_eval_host(pf, dp)
    devv = gpu_lb(torch, inst, pf, dp)
    assert (host == devv).all()
    sample = np.random.default_rng(0).choice(len(dp), 2000, replace=False)
    want = orc.Tables(ptm).lb_eval(pf[sample], dp[sample])
    assert (host[sample] == want).all()


def test_full_size_200x20_sampled(torch, fsp, orc):
    """BASELINE configs[3] at bench size (1M nodes, bench launch config):
    sampled nodes recomputed one by one by the oracle."""
    n, m, seed = inputs.TAILLARD_SEEDS["ta091"]
    ptm = inputs.taillard(n, m, seed)
    N = 1 << 20
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed("ta091"))
    inst = fsp.Instance(ptm)
    got = gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_OK
    rng = np.random.default_rng(1)
    sample = np.concatenate([rng.choice(N, 3000, replace=False), np.arange(N - 40, N)])
    want = orc.Tables(ptm).lb_eval(pf[sample], dp[sample])
    assert (got[sample] == want).all()
    # properties at any size: LB >= prefix-free machine bound, <= (n+m-1)*max p
    assert got.min() >= int(ptm.sum(0).max()) and got.max() <= (n + m - 1) * int(ptm.max())


# ------------------------------------------------ sibling (B&B child) pools

def completion_times(p, pf, dp):
    """C_k of each prefix by event simulation (independent of both sides)."""
    m = p.shape[1]
    out = np.zeros((len(dp), m), np.int32)
    for i in range(len(dp)):
        C = [0] * m
        for j in pf[i, :dp[i]]:
            prev = 0
            for k in range(m):
                C[k] = max(C[k], prev) + int(p[j, k])
                prev = C[k]
        out[i] = C
    return out


@pytest.mark.parametrize("name,depth", [("ta021", 15), ("ta051", 40), ("ta091", 190),
                                        ("ta091", 120), ("ta001", 10), ("ta111", 480),
                                        # live sets around 32 jobs per 128-node block: the
                                        # inverse-position compaction and the scan both run
                                        ("ta091", 168), ("ta091", 172), ("ta091", 176)])
def test_parity_sibling_pools(torch, fsp, orc, name, depth):
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_dfs_frontier(n, 40, depth, depth)
    inst = fsp.Instance(ptm)
    want = orc.Tables(ptm).lb_eval(pf, dp)
    for comp in (False, True):
        C = torch.from_numpy(completion_times(ptm, pf, dp)).cuda() if comp else None
        got = inst.lb_eval_sibling(dev(torch, pf), dev(torch, dp), C)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        assert inst.check() == fsp.FSP_OK
        assert (got == want).all(), (name, depth, comp, int((got != want).sum()))


def test_parity_sibling_api_on_random_pools(torch, fsp, orc):
    """The sparse plan on D1 pools (compaction rarely applies) and on deep
    random pools (it does) still equals the oracle."""
    for name, N in (("ta021", 3001), ("ta091", 1031)):
        n, m, seed = inputs.TAILLARD_SEEDS[name]
        ptm = inputs.taillard(n, m, seed)
        inst = fsp.Instance(ptm)
        T = orc.Tables(ptm)
        for pf, dp in (inputs.pool_d1(n, N, 9), inputs.pool_fixed_depth(n, N, n - 3, 10)):
            got = inst.lb_eval_sibling(dev(torch, pf), dev(torch, dp)).cpu().numpy()
            assert (got == T.lb_eval(pf, dp)).all()


@pytest.mark.parametrize("split", [1, 2, 4, 8, 16])
def test_parity_couple_split(torch, fsp, orc, monkeypatch, split):
    """Every couple split of a tile over `split` warps (LbArgs.split, atomicMax
    combine) gives the oracle's LBs: a 200x20 pool whose 3 couple groups are
    shared out unevenly (64 couples per group, 190 in all) and a ragged tail."""
    monkeypatch.setenv("FSP_LB_SPLIT", str(split))
    n, m, seed = inputs.TAILLARD_SEEDS["ta091"]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 1500, inputs.pool_seed("ta091") + 77)
    compare(torch, fsp, orc, ptm, pf, dp)
    n, m, seed = inputs.TAILLARD_SEEDS["ta021"]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 3001, inputs.pool_seed("ta021") + 77)
    compare(torch, fsp, orc, ptm, pf, dp)


@pytest.mark.parametrize("n,m", [(20, 5), (20, 20), (70, 10)])
def test_parity_walk16_offset_boundary(torch, fsp, orc, n, m):
    """The 16-bit walk carries e + max p unsigned and is taken iff
    (n + m) * max p <= 65535: instances exactly at the largest
    admissible max p (16-bit walk, every value up to its limit) and one above it
    (int32 walk) both match the oracle bit for bit."""
    pmax16 = 65535 // (n + m)
    for pmax, walk16 in [(pmax16, 1), (pmax16 + 1, 0)]:
        rng = np.random.default_rng(1208 + n * m + pmax)
        ptm = rng.integers(pmax // 2, pmax + 1, size=(n, m)).astype(np.int32)
        ptm[rng.integers(n), rng.integers(m)] = pmax
        ptm[0, :] = pmax  # one job at max p on every machine: t2 near its bound
        pf, dp = inputs.pool_d1(n, 3000, 4242 + pmax)
        inst = compare(torch, fsp, orc, ptm, pf, dp)
        assert inst.info["walk16"] == walk16


@pytest.mark.parametrize("n,m", [(20, 20), (41, 10), (200, 20), (20, 5), (33, 5)])
def test_parity_heads_job_pairs_boundary(torch, fsp, orc, n, m):
    """Job-pair heads (lb_kernel.cu jp_heads) push a scheduled job's half to an
    offset M = (65535 - max_j sum_k p_jk) rounded down to 16 and are taken iff
    M > (n + m) * max p: instances at the largest admissible max p (every real
    head, tail and load close to M) and one above it (per-job heads) both match
    the oracle; odd n exercises the padding job of the last pair."""
    def ok(p):
        return ((65535 - m * p) & ~15) > (n + m) * p and ((n + 1) // 2) * p <= 65535
    pmax = max(p for p in range(1, 4000) if ok(p))
    for pm, jp in [(pmax, 1), (pmax + 1, 0)]:
        rng = np.random.default_rng(3933 + n * m + pm)
        ptm = rng.integers(pm // 2, pm + 1, size=(n, m)).astype(np.int32)
        ptm[0, :] = pm  # one job at max p on every machine: the largest row sum
        parts = [inputs.pool_d1(n, 2000, 977 + pm),
                 inputs.pool_fixed_depth(n, 40, n, 978 + pm),  # complete schedules (R6)
                 inputs.pool_fixed_depth(n, 40, n - 1, 979 + pm)]  # one unscheduled job
        pf = np.concatenate([p[0] for p in parts])
        dp = np.concatenate([p[1] for p in parts])
        inst = compare(torch, fsp, orc, ptm, pf, dp)
        assert inst.launch_info(len(dp))["heads_jp"] == jp


@pytest.mark.parametrize("name", ["ta001", "ta021", "ta091"])
def test_c_pass_16bit_rows_ab(torch, fsp, orc, monkeypatch, name):
    """Taillard times fit a byte, so the C pass reads 8-bit PTM rows by
    default; FSP_LB_PTM8=0 forces the 16-bit rows: both match the oracle."""
    monkeypatch.setenv("FSP_LB_PTM8", "0")
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 4000, inputs.pool_seed(name) + 6)
    compare(torch, fsp, orc, ptm, pf, dp)


@pytest.mark.parametrize("name", ["ta001", "ta021", "ta091"])
def test_heads_job_pairs_ab(torch, fsp, orc, monkeypatch, name):
    """The same pool through the job-pair heads and the per-job heads
    (FSP_LB_JP=0, the A/B switch) gives identical LBs, equal to the oracle's."""
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 5000, inputs.pool_seed(name) + 5)
    a = compare(torch, fsp, orc, ptm, pf, dp)
    assert a.launch_info(len(dp))["heads_jp"] == 1
    monkeypatch.setenv("FSP_LB_JP", "0")
    b = compare(torch, fsp, orc, ptm, pf, dp)
    assert b.launch_info(len(dp))["heads_jp"] == 0


# ------------------------------------------- bench launch shapes

def _sampled(torch, fsp, orc, ptm, pf, dp, k, seed):
    inst = fsp.Instance(ptm)
    got = gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_OK
    N = len(dp)
    rng = np.random.default_rng(seed)
    sample = np.concatenate([rng.choice(N - 200, k, replace=False), np.arange(N - 200, N)])
    want = orc.Tables(ptm).lb_eval(pf[sample], dp[sample])
    bad = np.nonzero(got[sample] != want)[0]
    assert bad.size == 0, (sample[bad[:5]], got[sample][bad[:5]], want[bad[:5]])
    return inst, got


@pytest.mark.parametrize("rows", ["planner", "nibble"])
def test_full_size_500x20_bench_shape(torch, fsp, orc, monkeypatch, rows):
    """BASELINE configs[4] (ta111-class 500x20) at the bench's 1,048,576-node D1
    pool plus a ragged tail of 77 nodes: the launch shape is the bench one (no
    couple split, several tile iterations per CTA, every couple group cycling
    through the TMA buffers; the planner's byte rows with 8 warps, and the
    12-warp nibble rows of FSP_LB_ROWS=1), checked on 3,000 random nodes and
    the last 200."""
    if rows == "nibble":
        monkeypatch.setenv("FSP_LB_ROWS", "1")
    n, m, seed = inputs.TAILLARD_SEEDS["ta111"]
    ptm = inputs.taillard(n, m, seed)
    N = (1 << 20) + 77
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed("ta111"))
    inst = fsp.Instance(ptm)
    li = inst.launch_info(N)
    assert li["split"] == 1 and li["iterations"] > 1 and li["groups"] > li["group_buffers"]
    assert li["row_layout"] == (2 if rows == "nibble" else 1) and li["heads_jp"] == 1
    _, got = _sampled(torch, fsp, orc, ptm, pf, dp, 3000, 11)
    assert got.min() >= int(ptm.sum(0).max()) and got.max() <= (n + m - 1) * int(ptm.max())


def test_full_size_50x20_4m_sampled(torch, fsp, orc):
    """BASELINE configs[2] (ta051-class 50x20) at the top of its pool sweep,
    4,194,304 nodes, bench launch shape, sampled."""
    n, m, seed = inputs.TAILLARD_SEEDS["ta051"]
    ptm = inputs.taillard(n, m, seed)
    N = 1 << 22
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed("ta051"))
    inst = fsp.Instance(ptm)
    li = inst.launch_info(N)
    assert li["split"] == 1 and li["iterations"] > 1
    _sampled(torch, fsp, orc, ptm, pf, dp, 4000, 12)


def test_20x5_split1_every_node(torch, fsp, orc, monkeypatch):
    """The m = 5 kernel (lane-major rows, several CTAs per SM) without the
    couple split, on a 65,536-node ta001 pool: every LB against the oracle."""
    monkeypatch.setenv("FSP_LB_SPLIT", "1")
    n, m, seed = inputs.TAILLARD_SEEDS["ta001"]
    ptm = inputs.taillard(n, m, seed)
    N = 1 << 16
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed("ta001") + 5)
    inst = fsp.Instance(ptm)
    li = inst.launch_info(N)
    assert li["split"] == 1 and li["row_layout"] == 0
    compare(torch, fsp, orc, ptm, pf, dp)
    # and the bench-size 1M pool in the default shape, sampled
    monkeypatch.delenv("FSP_LB_SPLIT")
    pf, dp = inputs.pool_d1(n, 1 << 20, inputs.pool_seed("ta001"))
    assert inst.launch_info(1 << 20)["split"] == 1
    _sampled(torch, fsp, orc, ptm, pf, dp, 20000, 13)


@pytest.mark.parametrize("name", ["ta021", "ta091"])
def test_bench_shape_launch_info(fsp, name):
    """The 1M-node bench pools run unsplit with several tile iterations."""
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    inst = fsp.Instance(inputs.taillard(n, m, seed))
    li = inst.launch_info(1 << 20)
    assert li["split"] == 1 and li["iterations"] >= 2 and li["grid"] >= 148


@pytest.mark.parametrize("name,N", [("ta091", 300_007), ("ta021", 70_001), ("ta111", 40_003)])
def test_host_api_pinned_gather_path(torch, fsp, orc, monkeypatch, name, N):
    """fsp_lb_eval_host on pinned buffers takes the zero-copy gather path
    (only 2*depth prefix bytes cross PCIe, several chunks in flight); its LBs
    equal the device path's, the copy path's and, sampled, the oracle's."""
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, N, 4321)
    inst = fsp.Instance(ptm)
    h_pf = torch.from_numpy(pf.view(np.int16)).pin_memory()
    h_dp = torch.from_numpy(dp).pin_memory()
    h_lb = torch.full((N,), -1, dtype=torch.int32).pin_memory()
    inst.lb_eval_host_ptr(h_pf.data_ptr(), pf.shape[1], h_dp.data_ptr(), N, h_lb.data_ptr())
    got = h_lb.numpy().copy()
    assert (got == gpu_lb(torch, inst, pf, dp)).all()
    monkeypatch.setenv("FSP_HOST_COPY", "1")
    h_lb.fill_(-1)
    inst.lb_eval_host_ptr(h_pf.data_ptr(), pf.shape[1], h_dp.data_ptr(), N, h_lb.data_ptr())
    assert (h_lb.numpy() == got).all()
    rng = np.random.default_rng(5)
    sample = np.concatenate([rng.choice(N, 800, replace=False), np.arange(N - 50, N)])
    assert (got[sample] == orc.Tables(ptm).lb_eval(pf[sample], dp[sample])).all()


# ------------------------- sibling-incremental bounding (NEXT-1, family.cu)

def _children_of(pf, dp, n):
    """Every child (parent prefix + unscheduled j, ascending j) of each parent,
    as rows + depths, with (parent, t) of each child (test-side enumeration)."""
    rows, deps, where = [], [], []
    for i in range(len(dp)):
        d = int(dp[i])
        used = set(int(x) for x in pf[i, :d])
        t = 0
        for j in range(n):
            if j in used:
                continue
            r = pf[i].copy()
            r[d] = j
            rows.append(r)
            deps.append(d + 1)
            where.append((i, t))
            t += 1
    return np.stack(rows), np.array(deps, np.int32), where


@pytest.mark.parametrize("name,nparents", [("ta001", 400), ("ta021", 300), ("ta051", 200),
                                           ("ta091", 120)])
def test_parity_children_family(torch, fsp, orc, name, nparents):
    """fsp_lb_eval_children (prefix/suffix compositions per couple) equals the
    oracle on every child of parents with 1..32 unscheduled jobs, with the
    parents' completion times given and recomputed."""
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    rng = np.random.default_rng(17)
    depth = n - rng.integers(1, min(32, n) + 1, nparents)
    pf = inputs.random_prefixes(n, depth.astype(np.int32), 77)
    dp = depth.astype(np.int32)
    inst = fsp.Instance(ptm)
    rows, deps, where = _children_of(pf, dp, n)
    want = orc.Tables(ptm).lb_eval(rows, deps)
    C = torch.from_numpy(completion_times(ptm, pf, dp)).cuda()
    for comp in (None, C):
        got = inst.lb_eval_children(dev(torch, pf), dev(torch, dp), comp)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        vals = np.array([got[i, t] for i, t in where])
        bad = np.nonzero(vals != want)[0]
        assert bad.size == 0, (name, comp is None, bad[:5], vals[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("m", [2, 3, 7, 13, 25, 32])
def test_parity_children_family_machine_counts(torch, fsp, orc, m):
    rng = np.random.default_rng(100 + m)
    n = int(rng.integers(2, 40))
    ptm = rng.integers(0, 99, (n, m)).astype(np.int32)
    depth = (n - rng.integers(1, min(32, n) + 1, 150)).astype(np.int32)
    pf = inputs.random_prefixes(n, depth, 5)
    inst = fsp.Instance(ptm)
    rows, deps, where = _children_of(pf, depth, n)
    want = orc.Tables(ptm).lb_eval(rows, deps)
    got = inst.lb_eval_children(dev(torch, pf), dev(torch, depth)).cpu().numpy()
    vals = np.array([got[i, t] for i, t in where])
    assert (vals == want).all(), (m, n, int((vals != want).sum()))


def test_tune_pool(torch, fsp):
    """fsp_lb_tune_pool (runtime pool-size choice): a power of two
    in range whose measured rate reaches the requested fraction of the best."""
    n, m, seed = inputs.TAILLARD_SEEDS["ta021"]
    inst = fsp.Instance(inputs.taillard(n, m, seed))
    pool, rates = inst.tune_pool(18, 0.9)
    assert pool in rates and all(r > 0 for r in rates.values())
    assert rates[pool] >= 0.9 * max(rates.values())
    assert all(rates[s] < 0.9 * max(rates.values()) for s in rates if s < pool)


@pytest.mark.parametrize("name,N", [("ta021", 20011), ("ta091", 300_000)])
def test_parity_records_in_global_memory(torch, fsp, orc, monkeypatch, name, N):
    """Placement ablation (NEXT-3): the walk reading its couple records from
    global memory (L1/L2) instead of the TMA-staged shared buffers gives the
    same LBs (sampled against the oracle, all against the default kernel)."""
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, N, 99)
    ref = gpu_lb(torch, fsp.Instance(ptm), pf, dp)
    monkeypatch.setenv("FSP_LB_RECS", "global")
    got = gpu_lb(torch, fsp.Instance(ptm), pf, dp)
    assert (got == ref).all()
    sample = np.random.default_rng(3).choice(N, 500, replace=False)
    assert (got[sample] == orc.Tables(ptm).lb_eval(pf[sample], dp[sample])).all()


# ------------------------------ A/B: the north_star's warp-per-sub-problem mapping

@pytest.mark.parametrize("name,N", [("ta001", 5003), ("ta021", 4133), ("ta051", 2001), ("ta091", 1037)])
def test_parity_warp_per_node_mapping(torch, fsp, orc, monkeypatch, name, N):
    """FSP_LB_MAPPING=warp (wpn.cu: one warp per sub-problem, lanes over
    couples, heads/tails by warp reductions) bounds the same pools bit for bit;
    ragged batch tails and d = 0 / n - 1 / n nodes included."""
    monkeypatch.setenv("FSP_LB_MAPPING", "warp")
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    parts = [inputs.pool_d1(n, N, inputs.pool_seed(name) + 9),
             inputs.pool_fixed_depth(n, 33, n, 91), inputs.pool_fixed_depth(n, 35, n - 1, 92),
             inputs.pool_fixed_depth(n, 31, 0, 93)]
    pf = np.concatenate([p[0] for p in parts])
    dp = np.concatenate([p[1] for p in parts])
    inst = compare(torch, fsp, orc, ptm, pf, dp)
    assert inst.launch_info(len(dp))["mapping"] == 1


def test_warp_per_node_mapping_flags_malformed(torch, fsp, monkeypatch):
    """The A/B kernel raises the same malformed-node flag (job >= n, repeated job)."""
    monkeypatch.setenv("FSP_LB_MAPPING", "warp")
    n, m, seed = inputs.TAILLARD_SEEDS["ta021"]
    inst = fsp.Instance(inputs.taillard(n, m, seed))
    pf, dp = inputs.pool_fixed_depth(n, 64, 5, 7)
    pf[3, 1] = pf[3, 0]  # repeated job
    gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_EBADNODE
    pf, dp = inputs.pool_fixed_depth(n, 64, 5, 7)
    pf[9, 2] = n + 3  # job out of range
    gpu_lb(torch, inst, pf, dp)
    assert inst.check() == fsp.FSP_EBADNODE


@pytest.mark.parametrize("name,kc", [("ta021", "0"), ("ta091", "1")])
def test_parity_dense_kcache_switch(torch, fsp, orc, monkeypatch, name, kc):
    """Dense 20-machine walks with R_k/A_k cached across couples (the default
    for n <= 64) and without it (the default above) give the oracle's LBs
    either way: each config run through its non-default variant."""
    monkeypatch.setenv("FSP_LB_KCACHE", kc)
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, 3001, inputs.pool_seed(name) + 31)
    compare(torch, fsp, orc, ptm, pf, dp)
