"""Device group (sfxb_ctx_create_multi): one key over several GPUs of one
process — the multi-GPU path of the drop-in plugin.

Every result and counter of a group must equal the single-device context's
(which the other GPU tests pin to the oracle and the reference's golden
vectors).  The build box has one GPU, so the group repeats device 0: each
shard still has its own stream, buffers, row shard and slot slice, the
cross-shard reduce reads the other shards' partials through their device
pointers exactly as it reads peers over NVLink, and no kernel ever waits on
another shard's kernel (shards synchronise only through events)."""
import random

import numpy as np
import pytest

from keys import key
from paper_2504_03909_b200 import _lib
from py_oracle import ints_to_words
from test_gpu_histogram import _random_tree, frontier

pytestmark = pytest.mark.gpu


def _group(kname, shards, private=True):
    n, p, q = key(kname)
    if private:
        return _lib.Context(n, p, q, devices=[0] * shards), _lib.Context(n, p, q)
    return _lib.Context(n, devices=[0] * shards), _lib.Context(n)


def _rand_r(rng, n, count, nw):
    return ints_to_words([rng.randrange(2, n) for _ in range(count)], nw)


def test_group_shape_and_single_device_fallback():
    grp, one = _group("k512_c0ffee", 3)
    assert grp.n_shards == 3 and one.n_shards == 1
    assert grp.lib.sfxb_ctx_shard_device(grp.h, 2) == 0
    assert grp.lib.sfxb_ctx_shard_device(grp.h, 3) == -1
    assert grp.key_id == one.key_id
    n, p, q = key("k512_c0ffee")
    assert _lib.Context(n, devices=[0]).n_shards == 1
    with pytest.raises(_lib.SfxbError):
        _lib.Context(n, devices=[0] * 17)
    with pytest.raises(_lib.SfxbError, match="no such CUDA device"):
        _lib.Context(n, devices=[0, 99])


@pytest.mark.parametrize("kname,count", [("k2048_7", 3 * 4096 + 5), ("k512_c0ffee", 100)])
def test_group_encrypt_decrypt_add_equal_single(kname, count):
    grp, one = _group(kname, 3)
    n, p, q = key(kname)
    rng = random.Random(kname)
    r = _rand_r(rng, n, count, one.nw)
    qf = np.array([rng.randrange(-(1 << 40), 1 << 40) for _ in range(count)], np.int64)
    c1 = one.encrypt(qf, r)
    cg = grp.encrypt(qf, r)
    assert np.array_equal(c1, cg)
    v1, d1 = one.decrypt(c1)
    vg, dg = grp.decrypt(cg)
    assert np.array_equal(v1.view(np.int64), vg.view(np.int64)) and d1 == dg == count
    assert np.array_equal(one.add(c1, c1[::-1].copy()), grp.add(cg, cg[::-1].copy()))
    assert grp.launches > 0


def test_group_encrypt_flags_non_coprime_blinding():
    """r sharing a factor with n is flagged element-wise across shards
    (he.cpp:19-28 rejection rule), exactly as on one device."""
    grp, one = _group("k512_c0ffee", 2)
    n, p, q = key("k512_c0ffee")
    rng = random.Random(5)
    count = 2 * 4096 + 3
    rr = [rng.randrange(2, n) for _ in range(count)]
    for i in (7, 4096 + 11, count - 1):
        rr[i] = p * rng.randrange(1, q)
    r = ints_to_words(rr, one.nw)
    qf = np.zeros(count, np.int64)
    f1, fg = np.zeros(count, np.uint8), np.zeros(count, np.uint8)
    import ctypes as C

    outs = []
    for ctx, flags in ((one, f1), (grp, fg)):
        out = np.zeros((count, ctx.ct_words), np.uint32)
        rc = ctx.lib.sfxb_encrypt(ctx.h, qf, r.reshape(-1), count, out.reshape(-1), flags.ctypes.data_as(C.c_void_p))
        assert rc == _lib.SFXB_ERR_COPRIME
        assert "not coprime" in ctx.lib.sfxb_last_error(ctx.h).decode()
        outs.append(out)
    assert np.array_equal(f1, fg) and sorted(np.nonzero(fg)[0].tolist()) == [7, 4096 + 11, count - 1]


@pytest.mark.parametrize("private", [False, True])
@pytest.mark.parametrize("kname,shape,shards", [("k512_c0ffee", (5000, 3, 16, 5), 3),
                                                 ("k2048_7", (700, 2, 8, 4), 2),
                                                 ("k512_c0ffee", (5, 2, 4, 3), 4)])
def test_group_histogram_tree_mode_equals_single(kname, shape, shards, private):
    """Row-sharded partials + cross-shard product over the slot slices +
    sibling subtraction on the slices == the single-device histogram and its
    reference counter, level by level (leaves, an empty child, trivial-zero
    ciphertexts, rows outside the frontier, a shard without rows)."""
    n_samples, J, K, depth = shape
    grp, one = _group(kname, shards, private=private)
    n, _, _ = key(kname)
    rng = random.Random(str(shape))
    cts = [rng.randrange(2, n * n) for _ in range(2 * n_samples)]
    cts[1] = 1
    cts[2 * (n_samples - 1)] = 1
    cw = ints_to_words(cts, one.ct_words)
    bins = np.array([[rng.randrange(K) for _ in range(n_samples)] for _ in range(J)], np.uint16)
    ops1, opsg = _lib.DeviceOps(one), _lib.DeviceOps(grp)
    g1, gg = ops1.gh_upload(cw), opsg.gh_upload(cw)
    levels = _random_tree(rng, n_samples, depth)
    for lvl, (nodes, parents) in enumerate(levels):
        offs, rows = frontier(nodes)
        par = np.array(parents, np.int32)
        want, want_adds = ops1.accumulate_tree_host(g1, bins, offs, rows, K, par)
        got, adds = opsg.accumulate_tree_host(gg, bins, offs, rows, K, par)
        assert np.array_equal(got, want), lvl
        assert adds == want_adds, lvl
        # direct (non-tree) group histogram and the one-shot host call agree too
        got2, adds2 = opsg.accumulate_host(gg, bins, offs, rows, K)
        assert np.array_equal(got2, want) and adds2 == want_adds
        got3, adds3 = grp.accumulate(cw, bins, offs, rows, K)
        assert np.array_equal(got3, want) and adds3 == want_adds
    if depth > 2:
        assert grp.lib.sfxb_ctx_tree_derived(grp.h) > 0


def test_group_histogram_errors():
    grp, _ = _group("k512_c0ffee", 2, private=False)
    n, _, _ = key("k512_c0ffee")
    rng = random.Random(3)
    cw = ints_to_words([rng.randrange(2, n * n) for _ in range(2 * 10)], grp.ct_words)
    ok_bins = np.zeros((1, 10), np.uint16)
    with pytest.raises(_lib.SfxbError, match="row index out of range in accumulate"):
        grp.accumulate(cw, ok_bins, np.array([0, 2], np.uint32), np.array([1, 10], np.uint32), 2)
    bad = ok_bins.copy()
    bad[0, 8] = 5
    with pytest.raises(_lib.SfxbError, match="bin index out of range in accumulate"):
        grp.accumulate(cw, bad, np.array([0, 2], np.uint32), np.array([1, 8], np.uint32), 2)
    with pytest.raises(_lib.AuthorizationError, match="decrypt requested without private key material"):
        grp.decrypt(cw[:2])


def test_group_decrypt_tree_equals_single():
    n_samples, J, K, depth = 600, 2, 8, 4
    kname = "k512_c0ffee"
    grp, one = _group(kname, 3)
    n, _, _ = key(kname)
    rng = random.Random("dt")
    cw = ints_to_words([rng.randrange(2, n * n) for _ in range(2 * n_samples)], one.ct_words)
    bins = np.array([[rng.randrange(K) for _ in range(n_samples)] for _ in range(J)], np.uint16)
    for nodes, parents in _random_tree(rng, n_samples, depth):
        offs, rows = frontier(nodes)
        h, _ = one.accumulate(cw, bins, offs, rows, K)
        par = np.array(parents, np.int32)
        want, wd = one.decrypt_tree(5, h, len(nodes), par)
        got, gd = grp.decrypt_tree(5, h, len(nodes), par)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)) and gd == wd
    assert grp.dec_derived == one.dec_derived > 0


@pytest.mark.parametrize("private", [False, True])
@pytest.mark.parametrize("world,J,K", [(3, 1, 5), (4, 2, 3), (2, 3, 8)])
def test_rank_sliced_histograms_equal_single(world, J, K, private):
    """The one-process-per-GPU entry points (sfxb_accumulate_part_dev, the
    caller's all_to_all + count all_reduce, sfxb_combine_slices_dev) with
    `world` contexts on this GPU standing in for the ranks and the exchange
    done by hand: tree-mode histograms and the reference counter equal one
    context's, level by level, incl. padded column blocks (2·J·K not a
    multiple of world)."""
    import torch

    from paper_2504_03909_b200 import dist as pdist

    kname = "k512_c0ffee"
    n, p, q = key(kname)
    mk = (lambda: _lib.Context(n, p, q)) if private else (lambda: _lib.Context(n))
    one, ranks = mk(), [mk() for _ in range(world)]
    o1, ops = _lib.DeviceOps(one), [_lib.DeviceOps(c) for c in ranks]
    rng = random.Random(f"{world}{J}{K}{private}")
    n_samples, depth = 400, 4
    cts = [rng.randrange(2, n * n) for _ in range(2 * n_samples)]
    cts[3] = 1
    cw = ints_to_words(cts, one.ct_words)
    bins = np.array([[rng.randrange(K) for _ in range(n_samples)] for _ in range(J)], np.uint16)
    dev = torch.device("cuda:0")
    g1 = o1.gh_upload(cw)
    spans = [pdist.row_shard(n_samples, world, r) for r in range(world)]
    ghs = [ops[r].gh_upload(cw[2 * lo:2 * hi]) for r, (lo, hi) in enumerate(spans)]
    d_bins = [torch.from_numpy(bins[:, lo:hi].astype(np.int16).copy()).to(dev) for lo, hi in spans]
    spn = 2 * J * K
    jl = ops[0].slice_width(J, K, world)
    assert jl == (spn + world - 1) // world
    for lvl, (nodes, parents) in enumerate(_random_tree(rng, n_samples, depth)):
        N = len(nodes)
        offs, rows = frontier(nodes)
        par = np.array(parents, np.int32)
        sizes = np.diff(offs).astype(np.uint32)
        want, want_adds = o1.accumulate_tree_host(g1, bins, offs, rows, K, par)
        sends, reals = [], []
        for r, (lo, hi) in enumerate(spans):
            sub = [[x - lo for x in nd if lo <= x < hi] for nd in nodes]
            so, sr = frontier(sub)
            d_off = torch.from_numpy(so.astype(np.int32)).to(dev)
            d_rows = torch.from_numpy(sr.astype(np.int32) if len(sr) else np.zeros(1, np.int32)).to(dev)
            send = torch.zeros((world * N * jl, one.ct_words), dtype=torch.int32, device=dev)
            real = torch.zeros(2 * N * J * K, dtype=torch.int32, device=dev)
            ops[r].accumulate_part(ghs[r], d_bins[r], J, d_off, so, N, d_rows, len(sr), K, par, sizes, world,
                                   send, real)
            sends.append(send.view(world, N * jl, one.ct_words))
            reals.append(real)
        total = sum(reals)
        adds = ops[0].count_additions(total, 2 * N * J * K)
        assert adds == want_adds, lvl
        blocks = []
        for r in range(world):
            recv = torch.stack([sends[k][r] for k in range(world)]).contiguous()  # the all_to_all
            out = torch.zeros((N * jl, one.ct_words), dtype=torch.int32, device=dev)
            ops[r].combine_slices(ghs[r], recv, world, r, N, J, K, par, sizes, out)
            blocks.append(out.cpu().numpy().view(np.uint32).reshape(N, jl, -1))
        got = np.concatenate(blocks, 1)[:, :spn].reshape(N * spn, -1)
        assert np.array_equal(got, want), lvl
    assert sum(c.lib.sfxb_ctx_tree_derived(c.h) for c in ranks) > 0
