"""At-scale parity where the CPU reference cannot run: BASELINE
config 3's shape — 3 parties, 285k rows × 30 features (10 each), 256 bins,
2048-bit key — encrypted on the GPU, histogrammed level by level in tree mode
(sibling subtraction) to depth 5, and EVERY slot decrypted.  Checked against
the exact integer-sum oracle: a decrypted slot is
decode_fixed(Σ q_i mod n) with mpz_get_d truncation, q_i the int64
fixed-point gradients; empty slots decode to 0.0; the decryption counter is
the number of occupied slots; the addition counter follows the fold_into law."""
import os
import sys

import numpy as np
import pytest

from keys import key
from paper_2504_03909_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def decode_trunc(v: int, scale: int = 40) -> float:
    """decode_fixed of the signed plaintext v (he.cpp:138-143): mpz_get_d truncates."""
    a = abs(v)
    bl = a.bit_length()
    if bl > 53:
        a = (a >> (bl - 53)) << (bl - 53)
    d = float(a)
    return float(np.ldexp(-d if v < 0 else d, -scale))


def test_config3_shape_integer_sum_oracle():
    import torch

    import bench

    n, p, q = key("k2048_7")
    R, parties, J, K, D = 285_000, 3, 10, 256, 5
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(285)
    # fixed-point gradients on the 2^-40 grid: g in (-1, 1), h in [0, 0.25]
    qg = rng.integers(-(1 << 40) + 1, 1 << 40, R, dtype=np.int64)
    qh = rng.integers(0, 1 << 38, R, dtype=np.int64)
    qf = np.stack([qg, qh], 1).reshape(-1)
    active = _lib.Context(n, p, q)
    ops_a = _lib.DeviceOps(active)
    nw, cw = active.nw, active.ct_words
    r = torch.randint(-(2**31), 2**31 - 1, (2 * R, nw), dtype=torch.int32, device=dev)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((2 * R, cw), dtype=torch.int32, device=dev)
    ops_a.encrypt(torch.from_numpy(qf).to(dev), r, 2 * R, cts)
    fronts = bench.frontiers(R, D, seed=3)
    parents = [np.full(1, -1, np.int32)] + [np.arange(1 << d, dtype=np.int32) // 2 for d in range(1, D)]
    total_dec = 0
    for party in range(parties):
        ctx = _lib.Context(n)  # passive holder: public key only
        ops = _lib.DeviceOps(ctx)
        gh = ops.gh_from_dev(cts, R)
        bins = rng.integers(0, K, (J, R), dtype=np.uint16)
        d_bins = torch.from_numpy(bins.astype(np.int16)).to(dev)
        for d in range(D):
            offs, rows = fronts[d]
            N = len(offs) - 1
            out = torch.empty((N * J * K * 2, cw), dtype=torch.int32, device=dev)
            adds = ops.accumulate_tree(gh, d_bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), offs, N,
                                       torch.from_numpy(rows.astype(np.int32)).to(dev), len(rows), K, parents[d], out)
            vals = torch.empty(N * J * K * 2, dtype=torch.float64, device=dev)
            decs = ops_a.decrypt(out, N * J * K * 2, vals)
            got = vals.cpu().numpy().reshape(N, J, K, 2)
            # integer-sum oracle
            node_of = np.repeat(np.arange(N), np.diff(offs))
            want_adds = want_decs = 0
            for f in range(J):
                key_ = node_of * K + bins[f][rows].astype(np.int64)
                cnt = np.bincount(key_, minlength=N * K)
                want_adds += 2 * int(np.maximum(cnt - 1, 0).sum())
                want_decs += 2 * int((cnt > 0).sum())
                for gi, qv in enumerate((qg, qh)):
                    sums = np.zeros(N * K, dtype=np.int64)  # |Σ| < 2^59: exact in int64
                    np.add.at(sums, key_, qv[rows])
                    exp = np.ldexp(sums.astype(np.float64), -40)  # exact below 2^53
                    big = np.nonzero(np.abs(sums) >= (1 << 53))[0]
                    for i in big:  # mpz_get_d truncation above 53 bits
                        exp[i] = decode_trunc(int(sums[i]))
                    np.testing.assert_array_equal(got[:, f, :, gi], exp.reshape(N, K))
            assert adds == want_adds
            assert decs == want_decs
            total_dec += decs
        gh.free()
    assert total_dec > 100_000


def test_config5_10m_rows_depth8_integer_sum_oracle():
    """BASELINE configs[4] on one GPU (the C ABI's device entry points): one
    party's 50 of the 100 features, 10M rows, 256 bins, 2048-bit key, depth 8
    (histograms at depths 0-7, up to 128 nodes × 50 × 256 × 2 slots), tree mode
    (sibling subtraction from level 1), every slot of every level decrypted and
    compared with the C integer-sum oracle (oracle/paillier_oracle.c
    orc_intsum_hist: Σ q per slot mod n, decode_fixed) — values bit-exact,
    addition and decryption counters equal.  Gradient ciphertexts are drawn
    from a table of 2^18 encryptions of random fixed-point values (encrypting
    all 20M on the GPU would add ≈40 s; the histogram sees 20M independently
    indexed rows either way)."""
    import torch

    import bench
    from py_oracle import Oracle, OracleKey

    n, p, q = key("k2048_7")
    R, J, K, D, P = 10_000_000, 50, 256, 8, 1 << 18
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(510)
    holder = _lib.Context(n, p, q)
    passive = _lib.Context(n)
    ops_h, ops_p = _lib.DeviceOps(holder), _lib.DeviceOps(passive)
    cw, nw = holder.ct_words, holder.nw
    # table of encryptions: G values in (-2^40, 2^40), H values in [0, 2^38)
    tq = np.concatenate([rng.integers(-(1 << 40) + 1, 1 << 40, P // 2), rng.integers(0, 1 << 38, P // 2)])
    r = torch.randint(-(2**31), 2**31 - 1, (P, nw), dtype=torch.int32, device=dev)
    r[:, -1] &= 0x3FFFFFFF
    table = torch.empty((P, cw), dtype=torch.int32, device=dev)
    ops_h.encrypt(torch.from_numpy(tq.astype(np.int64)).to(dev), r, P, table)
    del r
    idx = np.empty(2 * R, np.int64)
    idx[0::2] = rng.integers(0, P // 2, R)
    idx[1::2] = rng.integers(P // 2, P, R)
    qf = tq[idx]
    gh_dev = table[torch.from_numpy(idx).to(dev)]
    gh = ops_p.gh_from_dev(gh_dev, R)
    del gh_dev, table
    torch.cuda.empty_cache()
    bins = rng.integers(0, K, (J, R), dtype=np.uint16)
    d_bins = torch.from_numpy(bins.astype(np.int16)).to(dev)
    fronts = bench.frontiers(R, D, seed=8)
    parents = [np.full(1, -1, np.int32)] + [np.arange(1 << d, dtype=np.int32) // 2 for d in range(1, D)]
    ok = OracleKey(Oracle(), n)
    total_slots = 0
    for d in range(D):
        offs, rows = fronts[d]
        N = len(offs) - 1
        S = N * J * K * 2
        out = torch.empty((S, cw), dtype=torch.int32, device=dev)
        adds = ops_p.accumulate_tree(gh, d_bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), offs, N,
                                     torch.from_numpy(rows.astype(np.int32)).to(dev), len(rows), K, parents[d], out)
        vals = torch.empty(S, dtype=torch.float64, device=dev)
        decs = ops_h.decrypt(out, S, vals)
        del out
        want, want_adds, want_decs = ok.intsum_hist(qf, bins, offs, rows, K)
        got = vals.cpu().numpy()
        bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
        assert bad.size == 0, f"level {d}: {bad.size} of {S} slots differ (first {bad[:5]})"
        assert adds == want_adds, d
        assert decs == want_decs, d
        total_slots += S
    assert total_slots == sum((1 << d) * J * K * 2 for d in range(D))
    assert passive.lib.sfxb_ctx_tree_derived(passive.h) == (1 << (D - 1)) - 1  # one derived child per split
    gh.free()
