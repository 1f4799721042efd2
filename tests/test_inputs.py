"""The seeded input generators (paper_1208_3933_b200/inputs.py)."""
import numpy as np

from paper_1208_3933_b200 import inputs


def test_pool_d1_valid_and_deterministic():
    for n in (1, 5, 20, 50):
        pf, dp = inputs.pool_d1(n, 300, 12083933)
        pf2, dp2 = inputs.pool_d1(n, 300, 12083933)
        assert (pf == pf2).all() and (dp == dp2).all()
        assert pf.shape == (300, inputs.default_stride(n)) and pf.dtype == np.uint16
        assert dp.min() >= 0 and dp.max() <= n - 1
        for i in range(300):
            row = pf[i, :dp[i]].tolist()
            assert len(set(row)) == len(row) and all(0 <= j < n for j in row)
            assert (pf[i, dp[i]:] == 0xFFFF).all()


def test_pool_d1_depth_spread():
    pf, dp = inputs.pool_d1(200, 20000, 7)
    assert abs(dp.mean() - 99.5) < 2.0           # d ~ U{0..n-1}
    # first position is close to uniform over jobs
    first = pf[dp > 0, 0]
    counts = np.bincount(first, minlength=200)
    assert counts.min() > 40 and counts.max() < 170


def test_fixed_depth_pools():
    for d in (0, 19, 20):
        pf, dp = inputs.pool_fixed_depth(20, 64, d, 3)
        assert (dp == d).all()
        for i in range(64):
            assert sorted(set(pf[i, :d].tolist())) == sorted(pf[i, :d].tolist())


def test_pool_d1_shards_concatenate():
    # strong scaling (bench.py --strong-total): every rank generates only its
    # shard [lo, hi) of one pool, and the shards concatenate to the pool
    from paper_1208_3933_b200 import dist as fdist
    full_pf, full_dp = inputs.pool_d1(37, 1001, 99)
    parts = [inputs.pool_d1(37, hi - lo, 99, first=lo)
             for lo, hi in (fdist.shard(1001, r, 3) for r in range(3))]
    assert (np.concatenate([p[0] for p in parts]) == full_pf).all()
    assert (np.concatenate([p[1] for p in parts]) == full_dp).all()
