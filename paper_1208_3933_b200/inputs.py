"""Seeded synthetic inputs shared by tests, bench and smoke.

This module holds NO arithmetic of the method (no bound, no makespan, no
Johnson order): only the instance generator and the node-pool generators.
Both the CUDA path and the oracle receive what it produces as plain arrays.

* ``taillard(n, m, seed)`` — Taillard's (1993) benchmark generator: the
  minimal-standard LCG (16807, 2^31-1, Schrage split 127773/2836), times
  ``1 + floor(u * 99)`` drawn machine-major (for each machine, for each job),
  returned job-major ``[n][m]`` as PTM is indexed in Fig. 3.
  SURVEY.md App. A; verified on ta001 (tests/golden/ta001_first_rows.txt).
* ``pool_d1(n, N, seed)`` — recipe D1 of DESIGN.md §5: depth d ~ U{0..n-1},
  prefix = the first d entries of a uniformly random permutation of [0, n),
  built with a counter-based splitmix64 Fisher-Yates so every machine
  reproduces it bit for bit.  Rows are padded to ``stride`` (multiple of 8
  jobs = 16 bytes) with 0xFFFF.
"""
from __future__ import annotations

import numpy as np

# Taillard (1993) seeds.  ta001 is verified by its published first row; the
# others are recalled and UNVERIFIED — instances are labelled
# tai-gen(n, m, seed) rather than claimed to be the published ones.
TAILLARD_SEEDS = {
    "ta001": (20, 5, 873654221),
    "ta002": (20, 5, 379008056),
    "ta003": (20, 5, 1866992158),
    "ta004": (20, 5, 216771124),
    "ta005": (20, 5, 495070989),
    "ta021": (20, 20, 479340445),
    "ta051": (50, 20, 1539989115),
    "c100x20": (100, 20, 1286373166),  # 100x20 class (seed recalled for ta081, unverified)
    "ta091": (200, 20, 2013025619),
    "ta111": (500, 20, 1368624604),
}

# BASELINE.json configs, in order (config_index = position).
CONFIGS = ["ta001", "ta021", "ta051", "ta091", "ta111"]
POOL_SEED_BASE = 12083933

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def taillard(n: int, m: int, seed: int) -> np.ndarray:
    if not (0 < seed < 2147483647):
        raise ValueError("seed must be in (0, 2^31-1)")
    p = np.zeros((n, m), dtype=np.int32)
    s = int(seed)
    for i in range(m):          # machine-major draws
        for j in range(n):
            k = s // 127773
            s = 16807 * (s % 127773) - 2836 * k
            if s < 0:
                s += 2147483647
            p[j, i] = 1 + int((s / 2147483647.0) * 99)
    return p


def instance(name: str) -> np.ndarray:
    n, m, seed = TAILLARD_SEEDS[name]
    return taillard(n, m, seed)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def _draw(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based 64-bit draw for (seed, stream, node index)."""
    with np.errstate(over="ignore"):
        base = _splitmix64(np.array([(seed * 0x100000001B3 + stream) & 0xFFFFFFFFFFFFFFFF],
                                    dtype=np.uint64))[0]
        return _splitmix64(idx.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03) ^ base)


def default_stride(n: int) -> int:
    return (n + 7) // 8 * 8


def random_prefixes(n: int, depth: np.ndarray, seed: int, stride: int | None = None,
                    first: int = 0):
    """Uniformly random d-prefixes (partial Fisher-Yates, counter-based; node i
    of the pool draws with counter first + i, so any slice of a pool can be
    generated on its own)."""
    N = depth.shape[0]
    stride = default_stride(n) if stride is None else stride
    perm = np.tile(np.arange(n, dtype=np.uint16), (N, 1))
    rows = np.arange(N)
    ctr = rows + first
    dmax = int(depth.max()) if N else 0
    for i in range(min(dmax, n - 1)):
        r = _draw(seed, 1 + i, ctr)
        j = (i + (r % np.uint64(n - i))).astype(np.int64)
        a = perm[:, i].copy()
        perm[:, i] = perm[rows, j]
        perm[rows, j] = a
    out = np.full((N, stride), 0xFFFF, dtype=np.uint16)
    cols = np.arange(n)
    keep = cols[None, :] < depth[:, None]
    out[:, :n] = np.where(keep, perm, np.uint16(0xFFFF))
    return out


def pool_d1(n: int, N: int, seed: int, stride: int | None = None, first: int = 0):
    """Recipe D1: returns (prefix uint16[N][stride], depth int32[N]) — nodes
    first .. first+N-1 of the seeded pool (a shard of a larger pool)."""
    rows = np.arange(first, first + N)
    depth = (_draw(seed, 0, rows) % np.uint64(n)).astype(np.int32)
    return random_prefixes(n, depth, seed, stride, first), depth


def pool_fixed_depth(n: int, N: int, d: int, seed: int, stride: int | None = None):
    depth = np.full(N, d, dtype=np.int32)
    return random_prefixes(n, depth, seed, stride), depth


def pool_seed(config_name: str) -> int:
    return POOL_SEED_BASE + CONFIGS.index(config_name)


def pool_children(n: int, parent_pf: np.ndarray, parent_dp: np.ndarray, stride: int | None = None):
    """B&B-shaped pool: every child (prefix + j, j unscheduled, ascending j) of
    each parent, parents in order, children contiguous (the layout of the
    device B&B's child pools)."""
    stride = default_stride(n) if stride is None else stride
    rows, deps = [], []
    for pf, d in zip(parent_pf, parent_dp):
        d = int(d)
        used = set(int(x) for x in pf[:d])
        for j in range(n):
            if j in used:
                continue
            r = np.full(stride, 0xFFFF, dtype=np.uint16)
            r[:d] = pf[:d]
            r[d] = j
            rows.append(r)
            deps.append(d + 1)
    if not rows:
        return np.zeros((0, stride), np.uint16), np.zeros(0, np.int32)
    return np.stack(rows), np.array(deps, dtype=np.int32)


def pool_dfs_frontier(n: int, n_parents: int, depth: int, seed: int, stride: int | None = None):
    """Children of `n_parents` parents that share a random prefix of length
    depth-1 and differ in their last job (siblings and cousins, as in a
    depth-first batch)."""
    base, _ = pool_fixed_depth(n, 1, max(depth - 1, 0), seed, stride)
    d0 = max(depth - 1, 0)
    used = set(int(x) for x in base[0, :d0])
    free = [j for j in range(n) if j not in used]
    rng = np.random.default_rng(seed)
    pick = rng.permutation(free)[:n_parents]
    par = np.repeat(base, len(pick), axis=0)
    for i, j in enumerate(pick):
        par[i, d0] = j
    return pool_children(n, par, np.full(len(pick), d0 + 1, np.int32), stride)
