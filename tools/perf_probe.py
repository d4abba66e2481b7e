"""Quick per-kernel throughput probe on one B200 (development tool, not the bench).

    python tools/perf_probe.py [--rows 1000000] [--enc 65536] [--dec 65536]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from keys import key  # noqa: E402
from paper_2504_03909_b200 import _lib  # noqa: E402


def rand_below(gen, bound_words, count, top_mask):
    x = torch.randint(0, 2**31, (count, bound_words), dtype=torch.int64, generator=gen)
    x = (x * 2 + torch.randint(0, 2, (count, bound_words), generator=gen)) & 0xFFFFFFFF
    x[:, -1] &= top_mask
    return x.to(torch.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--feats", type=int, default=14)
    ap.add_argument("--nodes", type=int, default=1)
    ap.add_argument("--enc", type=int, default=65536)
    ap.add_argument("--dec", type=int, default=65536)
    ap.add_argument("--key", default="k2048_7")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    peak, clk = _lib.imad_peak(0)
    print(f"imad peak {peak:.3e} products/s at {clk:.0f} MHz", flush=True)
    n, p, q = key(a.key)
    ctx = _lib.Context(n, p, q)
    ops = _lib.DeviceOps(ctx)
    nw, cw = ctx.nw, ctx.ct_words
    gen = torch.Generator().manual_seed(1)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # ---- encrypt
    cnt = a.enc
    r = rand_below(gen, nw, cnt, 0x3FFFFFFF).to(torch.int32).to(dev)  # < n (top limb bound)
    qf = torch.randint(-(1 << 40), 1 << 40, (cnt,), dtype=torch.int64, generator=gen).to(dev)
    out = torch.zeros((cnt, cw), dtype=torch.int32, device=dev)
    ops.encrypt(qf, r, cnt, out)  # warm-up at the timed size
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ops.encrypt(qf, r, cnt, out)
    dt = time.perf_counter() - t0
    prods = cnt * (2 * 2 * 1030 * (2 * 32 * 32 + 32) + 2 * 1030 * (2 * 64 * 64 + 64))
    print(f"encrypt {cnt}: {dt*1e3:.1f} ms  {cnt/dt:.0f} enc/s  ~{prods/dt:.3e} products/s "
          f"({prods/dt/peak*100:.1f}% of peak)", flush=True)

    # ---- decrypt (random ciphertexts < n^2)
    cnt = a.dec
    cts = rand_below(gen, cw, cnt, 0x3FFFFFFF).to(torch.int32).to(dev)
    vals = torch.zeros(cnt, dtype=torch.float64, device=dev)
    ops.decrypt(cts, cnt, vals)
    t0 = time.perf_counter()
    decs = ops.decrypt(cts, cnt, vals)
    dt = time.perf_counter() - t0
    prods = cnt * 2 * 1230 * (2 * 64 * 64 + 64)
    print(f"decrypt {cnt}: {dt*1e3:.1f} ms  {decs/dt:.0f} dec/s  ~{prods/dt:.3e} products/s "
          f"({prods/dt/peak*100:.1f}% of peak)", flush=True)

    # ---- histogram: rows x feats, K=256, nodes
    R, J, K = a.rows, a.feats, 256
    gh = rand_below(gen, cw, 2 * R, 0x3FFFFFFF).to(torch.int32).to(dev)
    h = ops.gh_from_dev(gh, R)
    bins = torch.randint(0, K, (J, R), dtype=torch.int16, generator=gen).to(dev)
    perm = torch.randperm(R, generator=gen).to(torch.int32)
    N = a.nodes
    offs = torch.linspace(0, R, N + 1).to(torch.int64).to(torch.int32).to(dev)
    rows = perm.to(dev)
    nslots = N * J * K * 2
    outh = torch.zeros((nslots, cw), dtype=torch.int32, device=dev)
    del gh
    ops.accumulate(h, bins, J, offs, N, rows, R, K, outh)  # warm-up (allocations)
    torch.cuda.synchronize()
    ctx.profile(True)
    t0 = time.perf_counter()
    adds = ops.accumulate(h, bins, J, offs, N, rows, R, K, outh)
    dt = time.perf_counter() - t0
    nk, kms = ctx.kernel_time(0)
    ctx.profile(False)
    print(f"  seg_prod launches={nk} kernel_ms={kms:.1f} ({adds*(2*128*128+128)/(kms/1e3)/peak*100:.1f}% of peak "
          f"inside the kernel)", flush=True)
    prods = adds * (2 * 128 * 128 + 128)
    print(f"histogram R={R} J={J} N={N}: {dt*1e3:.1f} ms  adds={adds}  {adds/dt:.3e} adds/s  "
          f"{prods/dt:.3e} products/s ({prods/dt/peak*100:.1f}% of peak)", flush=True)
    print("launches", ctx.launches)


if __name__ == "__main__":
    main()
