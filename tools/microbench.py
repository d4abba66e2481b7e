"""SURVEY §8d config 4 microbenchmark: encrypt / add (fold into 256 bins) /
decrypt throughput over batch sizes and key sizes on one B200.

    python tools/microbench.py [--bits 1024 2048 3072] [--sizes 1024 4096 ... 16777216]
                               [--max-seconds 900] > profiles/rNN_micro.jsonl

One JSON line per (op, bits, size): throughput from CUDA events on the
context stream (inputs resident in HBM, warm-up call at the same size
first), and the fraction of the IMAD.WIDE peak from the multiplications the
kernels executed.  "add" / "add_pub" (key holder / passive party) fold k ciphertexts (k/2 rows × (G, H)) into 256
bins with uniform-random bin ids (seed 1) and counts k − occupied additions,
as the reference's counter does.  Sizes whose estimated time exceeds
--max-seconds (from the previous size's rate) are skipped and reported so.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from keys import key  # noqa: E402
from paper_2504_03909_b200 import _lib  # noqa: E402

KEYS = {512: "k512_c0ffee", 1024: "k1024_7", 2048: "k2048_7", 3072: "k3072_7"}


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=[1024, 2048, 3072])
    ap.add_argument("--sizes", type=int, nargs="+", default=[1 << k for k in range(10, 25, 2)])
    ap.add_argument("--ops", nargs="+", default=["enc", "enc_pub", "add", "add_pub", "dec"])
    ap.add_argument("--max-seconds", type=float, default=900.0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    peak, mhz = _lib.imad_peak(0)
    for bits in a.bits:
        n, p, q = key(KEYS[bits])
        ctx = _lib.Context(n, p, q)
        pub = _lib.Context(n)
        nw, cw = ctx.nw, ctx.ct_words
        s2 = cw // 2  # limbs of p² (CRT modulus)
        prod_p2 = 2 * s2 * s2 + s2
        prod_n2 = 2 * cw * cw + cw
        for op in a.ops:
            # key holder (CRT digits) vs passive party (public key: base-n digits)
            c = pub if op in ("enc_pub", "add_pub") else ctx
            ops = _lib.DeviceOps(c)
            stream = torch.cuda.ExternalStream(c.lib.sfxb_ctx_stream(c.h), device=dev)
            rate = None
            for k in a.sizes:
                rec = {"op": op, "bits": bits, "size": k}
                if rate and k / rate > a.max_seconds:
                    rec["skipped"] = f"estimated {k / rate:.0f} s > --max-seconds"
                    print(json.dumps(rec), flush=True)
                    continue
                g = torch.Generator(device=dev).manual_seed(k)
                if op in ("enc", "enc_pub", "dec"):
                    qf = torch.randint(-(1 << 40), 1 << 40, (k,), dtype=torch.int64, device=dev, generator=g)
                    r = torch.randint(-(2**31), 2**31 - 1, (k, nw), dtype=torch.int32, device=dev, generator=g)
                    r[:, -1] &= 0x3FFFFFFF
                    cts = torch.empty((k, cw), dtype=torch.int32, device=dev)
                    if op == "dec":
                        cts.random_(generator=g)  # random units < 2^(32(cw-1)) < n² stand for ciphertexts
                        cts[:, -1] = 0
                        vals = torch.empty(k, dtype=torch.float64, device=dev)
                        fn = lambda: ops.decrypt(cts, k, vals, sync=False)  # noqa: E731
                        fam, unit_products = 2, prod_p2
                    else:
                        fn = lambda: ops.encrypt(qf, r, k, cts, sync=False)  # noqa: E731
                        fam, unit_products = (1, prod_p2) if op == "enc" else (None, None)
                    if not rate or k / rate < 5:
                        fn()  # warm-up at this size (scratch growth; long runs amortise it)
                    c.profile(True)
                    dt, res = timed(stream, fn)
                    stats = c.kernel_stats(fam) if fam is not None else None
                    c.profile(False)
                    units = res if op == "dec" else k
                else:  # add: fold k ciphertexts into 256 bins
                    rows = k // 2
                    cts = torch.empty((2 * rows, cw), dtype=torch.int32, device=dev)
                    cts.random_(generator=g)  # random units < n² (same cost as ciphertexts)
                    cts[:, -1] = 0
                    gh = ops.gh_from_dev(cts, rows)
                    bins = np.random.default_rng(1).integers(0, 256, (1, rows), dtype=np.uint16)
                    d_bins = torch.from_numpy(bins.astype(np.int16)).to(dev)
                    d_off = torch.tensor([0, rows], dtype=torch.int32, device=dev)
                    d_rows = torch.arange(rows, dtype=torch.int32, device=dev)
                    out = torch.empty((256 * 2, cw), dtype=torch.int32, device=dev)
                    fn = lambda: ops.accumulate(gh, d_bins, 1, d_off, 1, d_rows, rows, 256, out,  # noqa: E731
                                                sync=False)
                    if not rate or k / rate < 5:
                        fn()
                    c.profile(True)
                    dt, res = timed(stream, fn)
                    stats = c.kernel_stats(0)
                    c.profile(False)
                    gh.free()
                    units, unit_products = res, prod_n2
                rate = units / dt if dt > 0 else None
                rec.update({"per_s": rate, "seconds": dt, "units": int(units)})
                if stats and stats[1] > 0:
                    # kernel families count the 32x32->64 products their launches executed
                    rec["roofline_frac"] = stats[2] / (stats[1] / 1e3) / peak
                    rec["kernel_ms"] = stats[1]
                print(json.dumps(rec), flush=True)
    print(json.dumps({"imad_peak_products_per_s": peak, "sm_clock_mhz": mhz}), flush=True)


if __name__ == "__main__":
    main()
