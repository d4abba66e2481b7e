"""CPU: bench.py's workload construction follows the reference semantics."""
import numpy as np

import bench
from keys import key
from py_oracle import Oracle, OracleKey


def test_frontiers_are_a_binary_tree():
    fr = bench.frontiers(1000, 4, seed=1)
    for d, (offs, rows) in enumerate(fr):
        assert len(offs) == (1 << d) + 1 and offs[-1] == 1000
        assert sorted(rows.tolist()) == list(range(1000))
        for i in range(len(offs) - 1):
            seg = rows[offs[i]:offs[i + 1]]
            assert np.all(np.diff(seg.astype(np.int64)) > 0)  # ascending inside a node
            if d:  # children partition the parent
                po, pr = fr[d - 1]
                parent = set(pr[po[i // 2]:po[i // 2 + 1]].tolist())
                assert set(seg.tolist()) <= parent


def test_adds_per_tree_is_the_reference_counter_law():
    n, p, q = key("k512_c0ffee")
    ok = OracleKey(Oracle(), n)
    rng = np.random.default_rng(2)
    R, J, K = 300, 2, 8
    fr = bench.frontiers(R, 3, seed=3)
    bins = rng.integers(0, K, (J, R), dtype=np.uint16)
    cts = bench.rand_words(rng, 2 * R, 2 * ok.nw)
    want = 0
    for offs, rows in fr:
        _, adds = ok.accumulate(cts, bins, offs, rows, K)
        want += adds
    assert bench.adds_per_tree([bins], fr, K) == want
