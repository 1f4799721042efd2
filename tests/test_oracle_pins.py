"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test checks the oracle against something other than itself: worked
examples (SPEC / Taillard), closed forms, brute force over all orders on tiny
inputs, and invariants.  The helpers below are written from the *definitions*
(lattice paths, event simulation, minimum over all completions), never from
Fig. 3, so a dropped term, wrong sign/index or transposed operand in the
oracle fails one of them.  SURVEY.md §8(c) numbers the pins P1..P13.
"""
import itertools
import os

import numpy as np
import pytest

from paper_1208_3933_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------- independent helpers

def cmax_by_paths(p, perm):
    """Makespan as the longest monotone lattice path through the (job, machine)
    grid — the critical-path characterisation, enumerated path by path."""
    n, m = len(perm), p.shape[1]
    best = 0
    # a path is a choice of the n-1 'next job' moves among n+m-2 moves
    for downs in itertools.combinations(range(n + m - 2), n - 1):
        i = k = 0
        s = int(p[perm[0], 0])
        ds = set(downs)
        for step in range(n + m - 2):
            if step in ds:
                i += 1
            else:
                k += 1
            s += int(p[perm[i], k])
        best = max(best, s)
    return best


def simulate(p, perm):
    """Event simulation: per machine, the time it becomes free; per job, the
    time its previous operation ends.  Returns start times [job][machine]."""
    m = p.shape[1]
    free = [0] * m
    start = {}
    for j in perm:
        ready = 0
        for k in range(m):
            s = max(free[k], ready)
            start[(j, k)] = s
            free[k] = s + int(p[j, k])
            ready = free[k]
    return start, free


def cmax_sim(p, perm):
    return simulate(p, perm)[1][-1] if len(perm) else 0


def best_completion(p, prefix):
    n = p.shape[0]
    rest = [j for j in range(n) if j not in prefix]
    return min(cmax_sim(p, list(prefix) + list(q)) for q in itertools.permutations(rest))


def two_machine_lag(order, a, lag, b, start1, start2):
    """Two machines with time lags: M1 processes a_j, the job then waits
    lag_j, then M2 processes b_j; M1 free from start1, M2 from start2."""
    f1, f2 = start1, start2
    for j in order:
        f1 = f1 + a[j]
        f2 = max(f2, f1 + lag[j]) + b[j]
    return f2


def rand_instance(rng, n, m, lo=0, hi=20):
    return rng.integers(lo, hi, (n, m)).astype(np.int32)


# --------------------------------------------------------------------- makespan

def test_makespan_spec_examples(orc):
    # n=1, row [2,3,4] -> 9 (row sum)
    assert orc.makespan(np.array([[2, 3, 4]]), [0]) == 9
    # one job per machine column sums: m=2 with a single machine's work only
    p = np.array([[5, 0], [7, 0], [1, 0]])
    assert orc.makespan(p, [0, 1, 2]) == 13


def test_makespan_vs_lattice_paths(orc):
    rng = np.random.default_rng(7)
    for _ in range(60):
        n, m = int(rng.integers(1, 6)), int(rng.integers(2, 5))
        p = rand_instance(rng, n, m)
        perm = list(rng.permutation(n))
        assert orc.makespan(p, perm) == cmax_by_paths(p, perm)


# --------------------------------------------------------------- Johnson's rule

def test_johnson_spec_example(orc):
    # a=[3,5,1], b=[2,4,4] -> [2,1,0], two-machine makespan 12 = optimum
    order = orc.johnson_order([3, 5, 1], [2, 4, 4])
    assert order.tolist() == [2, 1, 0]
    a, b, z = [3, 5, 1], [2, 4, 4], [0, 0, 0]
    assert two_machine_lag(order, a, z, b, 0, 0) == 12
    assert min(two_machine_lag(q, a, z, b, 0, 0)
               for q in itertools.permutations(range(3))) == 12


def test_johnson_optimal_bruteforce(orc):
    rng = np.random.default_rng(11)
    for _ in range(150):
        n = int(rng.integers(1, 8))
        a, b = rng.integers(0, 15, n), rng.integers(0, 15, n)
        order = orc.johnson_order(a, b).tolist()
        assert sorted(order) == list(range(n))
        z = [0] * n
        best = min(two_machine_lag(q, a, z, b, 0, 0) for q in itertools.permutations(range(n)))
        assert two_machine_lag(order, a, z, b, 0, 0) == best


# ---------------------------------------------------------- tables (Table I, §II-D)

def test_machine_pairs(orc):
    T = orc.Tables(np.ones((4, 3), np.int32))
    assert T.MM.tolist() == [[0, 1], [0, 2], [1, 2]]
    assert orc.Tables(np.ones((2, 20), np.int32)).P == 190    # P9


def test_table_sizes_200x20(orc):
    # P9 / P:420-422: at 200x20, JM and LM have 38,000 entries, PTM 4,000
    p = inputs.taillard(200, 20, 2013025619)
    T = orc.Tables(p)
    assert T.JM.size == 38000 and T.LM.size == 38000 and T.ptm.size == 4000
    assert T.MM.size == 190 * 2 == 20 * 19                      # Table I: m(m-1)
    for col in T.JM.T:                                          # every column a permutation
        assert sorted(col.tolist()) == list(range(200))


def test_lags_closed_forms(orc):
    # row [4,7,2], couple (0,2) -> lag 7; adjacent couples lag 0
    T = orc.Tables(np.array([[4, 7, 2]], np.int32))
    MM = T.MM.tolist()
    assert T.LM[0, MM.index([0, 2])] == 7
    assert T.LM[0, MM.index([0, 1])] == 0 and T.LM[0, MM.index([1, 2])] == 0
    rng = np.random.default_rng(3)
    p = rand_instance(rng, 6, 6)
    T = orc.Tables(p)
    MM = T.MM.tolist()
    for idx, (k, l) in enumerate(MM):
        if l > k + 1:  # lm(k,l) = lm(k,l-1) + p_{l-1}
            assert (T.LM[:, idx] == T.LM[:, MM.index([k, l - 1])] + p[:, l - 1]).all()
    # tails: q_{j,m-1} = 0, q_{j,l} = q_{j,l+1} + p_{j,l+1}
    assert (T.QM[:, -1] == 0).all()
    assert (T.QM[:, :-1] == T.QM[:, 1:] + p[:, 1:]).all()


def test_jm_columns_solve_lag_relaxation(orc):
    # each JM column, simulated on the lag-augmented two-machine
    # problem of its couple, attains the minimum over all orders (n <= 6).
    rng = np.random.default_rng(5)
    for _ in range(25):
        n, m = int(rng.integers(2, 7)), int(rng.integers(3, 6))
        p = rand_instance(rng, n, m)
        T = orc.Tables(p)
        for idx, (k, l) in enumerate(T.MM.tolist()):
            lag = T.LM[:, idx]
            a, b = p[:, k], p[:, l]
            got = two_machine_lag(T.JM[:, idx], a, lag, b, 0, 0)
            best = min(two_machine_lag(q, a, lag, b, 0, 0)
                       for q in itertools.permutations(range(n)))
            assert got == best


# ------------------------------------------------------------------ the bound

def _nodes(rng, n, count):
    for _ in range(count):
        d = int(rng.integers(0, n + 1))
        yield [int(x) for x in rng.permutation(n)[:d]]


def test_P1_admissible_bruteforce(orc):
    rng = np.random.default_rng(101)
    for _ in range(120):
        n, m = int(rng.integers(2, 7)), int(rng.integers(2, 6))
        p = rand_instance(rng, n, m)
        T = orc.Tables(p)
        for pre in _nodes(rng, n, 4):
            assert T.lb(pre) <= best_completion(p, pre)


def test_P2_m2_exact_every_node(orc):
    # Johnson: for m = 2 the bound is the exact best completion
    rng = np.random.default_rng(202)
    for _ in range(120):
        n = int(rng.integers(1, 8))
        p = rand_instance(rng, n, 2)
        T = orc.Tables(p)
        for pre in _nodes(rng, n, 3):
            assert T.lb(pre) == best_completion(p, pre)


def test_P3_per_couple_relaxation_exact(orc):
    """Each couple's value = min over all orders of the unscheduled jobs of the
    two-machine-with-lags schedule started at the heads, plus the tail.  Heads
    are re-derived here as the earliest start of each unscheduled job if it
    were scheduled next (event simulation), tails from their definition."""
    rng = np.random.default_rng(303)
    for _ in range(60):
        n, m = int(rng.integers(2, 7)), int(rng.integers(3, 6))
        p = rand_instance(rng, n, m)
        T = orc.Tables(p)
        for pre in _nodes(rng, n, 3):
            S = [j for j in range(n) if j not in pre]
            if not S:
                continue
            lbv, pv, heads, tails, _ = T.lb(pre, detail=True)
            R = [min(simulate(p, pre + [j])[0][(j, k)] for j in S) for k in range(m)]
            Q = [min(int(p[j, l + 1:].sum()) for j in S) for l in range(m)]
            assert heads.tolist() == R and tails.tolist() == Q
            for idx, (k, l) in enumerate(T.MM.tolist()):
                lag = [int(p[j, k + 1:l].sum()) for j in range(n)]
                best = min(two_machine_lag(q, p[:, k], lag, p[:, l], R[k], R[l])
                           for q in itertools.permutations(S))
                assert pv[idx] == best + Q[l]
            assert lbv == max(pv.max(), 0)


def test_P4_leaves_exact(orc):
    rng = np.random.default_rng(404)
    for _ in range(100):
        n, m = int(rng.integers(1, 9)), int(rng.integers(2, 7))
        p = rand_instance(rng, n, m)
        T = orc.Tables(p)
        perm = [int(x) for x in rng.permutation(n)]
        assert T.lb(perm) == cmax_by_paths(p, perm)            # d = n
        assert T.lb(perm[:-1]) == cmax_by_paths(p, perm)       # d = n-1: forced completion


def test_P5_identical_jobs_closed_form(orc):
    rng = np.random.default_rng(505)
    for _ in range(40):
        n, m = int(rng.integers(1, 30)), int(rng.integers(2, 9))
        r = rng.integers(0, 50, m)
        p = np.tile(r, (n, 1)).astype(np.int32)
        closed = int(r.sum()) + (n - 1) * int(r.max())       # every permutation's makespan
        assert orc.Tables(p).lb([]) == closed == cmax_by_paths(p, list(range(n))) if n <= 6 \
            else orc.Tables(p).lb([]) == closed


def test_P6_relabelling_invariance(orc):
    """Renaming jobs permutes JM ties differently; the bound must not move."""
    rng = np.random.default_rng(606)
    for _ in range(40):
        n, m = int(rng.integers(2, 25)), int(rng.integers(2, 8))
        p = rand_instance(rng, n, m, 0, 6)  # many ties
        sigma = rng.permutation(n)          # new label of old job j = sigma[j]
        p2 = np.empty_like(p)
        p2[sigma] = p
        T, T2 = orc.Tables(p), orc.Tables(p2)
        for pre in _nodes(rng, n, 5):
            assert T.lb(pre) == T2.lb([int(sigma[j]) for j in pre])


def test_P7_envelope(orc):
    rng = np.random.default_rng(707)
    for _ in range(60):
        n, m = int(rng.integers(2, 40)), int(rng.integers(2, 8))
        p = rand_instance(rng, n, m, 0, 99)
        T = orc.Tables(p)
        for pre in _nodes(rng, n, 4):
            S = [j for j in range(n) if j not in pre]
            lbv, _, R, Q, _ = T.lb(pre, detail=True)
            assert lbv <= (n + m - 1) * int(p.max())
            if S:  # dominates the one-machine bound
                one = max(int(R[k]) + int(p[S, k].sum()) + int(Q[k]) for k in range(m))
                assert lbv >= one
            # never below the prefix's own completion on the last machine
            assert lbv >= cmax_sim(p, pre)


def test_P8_table_I_access_counts(orc):
    # Table I: JM n*P, LM n'*P, PTM n'*m(m-1), RM m(m-1), QM P, MM m(m-1)
    rng = np.random.default_rng(808)
    p = rand_instance(rng, 12, 6)
    T = orc.Tables(p)
    P = T.P
    for pre in _nodes(rng, 12, 10):
        if len(pre) == 12:
            continue
        nprime = 12 - len(pre)
        _, _, _, _, c = T.lb(pre, detail=True)
        assert c["jm_reads"] == 12 * P
        assert c["lm_reads"] == nprime * P
        assert c["ptm_reads"] == nprime * 6 * 5
        assert c["rm_reads"] == 6 * 5 and c["mm_reads"] == 6 * 5 and c["qm_reads"] == P


def test_lb_eval_matches_single_and_rejects_bad(orc):
    p = inputs.taillard(20, 5, 873654221)
    T = orc.Tables(p)
    pf, dp = inputs.pool_d1(20, 50, 1)
    lb = T.lb_eval(pf, dp)
    for i in range(50):
        assert lb[i] == T.lb(pf[i, :dp[i]])
    bad = pf.copy()
    bad[0, 0] = 25
    dp2 = dp.copy()
    dp2[0] = max(dp2[0], 1)
    with pytest.raises(ValueError):
        T.lb_eval(bad, dp2)


# --------------------------------------------------------------------- the B&B

def test_bb_vs_bruteforce(orc):
    rng = np.random.default_rng(909)
    for _ in range(40):
        n, m = int(rng.integers(1, 8)), int(rng.integers(2, 6))
        p = rand_instance(rng, n, m, 1, 30)
        T = orc.Tables(p)
        opt = min(cmax_sim(p, list(q)) for q in itertools.permutations(range(n)))
        rc, ms, perm, st = T.bb_dfs()
        assert rc == 0 and ms == opt and cmax_by_paths(p, perm.tolist()) == opt
        assert sorted(perm.tolist()) == list(range(n))
        # initial UB semantics (R9): equal to the optimum -> found; below -> none
        rc, ms, perm, _ = T.bb_dfs(opt)
        assert rc == 0 and ms == opt
        if opt > 0:
            assert T.bb_dfs(opt - 1)[0] == 1


def test_bb_m2_equals_johnson(orc):
    rng = np.random.default_rng(1010)
    for _ in range(20):
        n = int(rng.integers(2, 40))
        p = rand_instance(rng, n, 2, 1, 99)
        order = orc.johnson_order(p[:, 0], p[:, 1])
        rc, ms, _, _ = orc.Tables(p).bb_dfs()
        assert rc == 0 and ms == cmax_sim(p, order.tolist())


def _golden_optima():
    rows = []
    with open(os.path.join(GOLDEN, "taillard_optima.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                name, n, m, seed, opt, _ = line.split()
                rows.append((name, int(n), int(m), int(seed), int(opt)))
    return rows


def test_taillard_generator_ta001_rows():
    with open(os.path.join(GOLDEN, "ta001_first_rows.txt")) as f:
        rows = [list(map(int, l.split())) for l in f if l.strip() and not l.startswith("#")]
    p = inputs.taillard(20, 5, 873654221)
    assert p[:, 0].tolist() == rows[0] and p[:, 1].tolist() == rows[1]
    # seed 1 -> state 16807 -> first time 1
    assert inputs.taillard(1, 1, 1)[0, 0] == 1


@pytest.mark.parametrize("row", range(4), ids=["ta001", "ta002", "ta003", "ta004"])
def test_bb_taillard_optimum(orc, row):
    # P12/P13: the full B&B from the root (no initial UB) reaches the published
    # optimum; ta001's 1278 is BASELINE.json's, ta002-ta004 are recalled, and a
    # seed/optimum match pins both (R19 makes ta001 a 5K-node search)
    name, n, m, seed, opt = _golden_optima()[row]
    p = inputs.taillard(n, m, seed)
    rc, ms, perm, _ = orc.Tables(p).bb_dfs()
    assert rc == 0 and ms == opt and cmax_sim(p, perm.tolist()) == opt
    assert sorted(perm.tolist()) == list(range(n))
    # and nothing below it exists (R9: initial_ub = opt - 1 -> no schedule)
    if row == 0:
        assert orc.Tables(p).bb_dfs(opt - 1)[0] == 1


def test_root_bound_ta001_equals_optimum(orc):
    # the ta001 optimum 1278 (BASELINE.json) is attained by the root bound, so
    # any schedule of makespan 1278 is a certificate of optimality
    p = inputs.instance("ta001")
    assert orc.Tables(p).lb([]) == 1278
