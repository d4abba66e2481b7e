"""Helper for tests/test_gpu_switches.py (run in a subprocess, because the
launch-shape switches are read once per process): encrypt, decrypt and
tree-mode histograms of both party kinds through the C ABI on fixed seeded
inputs; prints one SHA-256 over every output byte and counter.

    python tests/ab_driver.py KEYNAME
"""
import hashlib
import os
import random
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
from keys import key  # noqa: E402
from paper_2504_03909_b200 import _lib  # noqa: E402


def frontier(nodes):
    offs = np.cumsum([0] + [len(x) for x in nodes]).astype(np.uint32)
    rows = np.array([r for nd in nodes for r in nd], np.uint32)
    return offs, rows


def main():
    kname = sys.argv[1]
    n, p, q = key(kname)
    h = hashlib.sha256()
    dev = torch.device("cuda:0")
    ctx = _lib.Context(n, p, q)
    ops = _lib.DeviceOps(ctx)
    # encrypt + decrypt: 3 waves of exponentiations and a partial one
    count = 60_000
    g = torch.Generator(device=dev).manual_seed(5)
    qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
    r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
    ops.encrypt(qf, r, count, cts)
    vals = torch.empty(count, dtype=torch.float64, device=dev)
    decs = ops.decrypt(cts, count, vals)
    h.update(cts.cpu().numpy().tobytes())
    h.update(vals.cpu().numpy().tobytes())
    h.update(str(decs).encode())
    # tree-mode histograms: key holder (CRT digits) and passive party (base-n digits)
    rng = random.Random(kname + "ab")
    n_samples, J, K = 3000, 3, 16
    cw = cts[: 2 * n_samples].cpu().numpy().view(np.uint32)
    bins = np.array([[rng.randrange(K) for _ in range(n_samples)] for _ in range(J)], np.uint16)
    levels, nodes = [], [list(range(n_samples))]
    levels.append((nodes, [-1]))
    for _ in range(3):
        nxt, par = [], []
        for pi, rows in enumerate(nodes):
            cut = rng.randrange(len(rows) + 1)
            sh = rows[:]
            rng.shuffle(sh)
            a, b = sorted(sh[:cut]), sorted(sh[cut:])
            nxt += [a, b]
            par += [pi, pi]
        nodes = nxt
        levels.append((nodes, par))
    for c in (ctx, _lib.Context(n)):
        o = _lib.DeviceOps(c)
        gh = o.gh_upload(cw)
        for nds, par in levels:
            offs, rows = frontier(nds)
            got, adds = o.accumulate_tree_host(gh, bins, offs, rows, K, np.array(par, np.int32))
            h.update(got.tobytes())
            h.update(str(adds).encode())
        gh.free()
    print(h.hexdigest())


if __name__ == "__main__":
    main()
