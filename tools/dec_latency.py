"""Latency of decrypt batches of a tree's level sizes (2048-bit, device-resident),
CUDA events, median of 5 after a warm-up: the tail split's lane choice at work.

    [SFXB_DEC_SMALL_TPI=0] python tools/dec_latency.py
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from keys import key  # noqa: E402
from paper_2504_03909_b200 import _lib  # noqa: E402


def main():
    n, p, q = key("k2048_7")
    ctx = _lib.Context(n, p, q)
    ops = _lib.DeviceOps(ctx)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(3)
    big = 114688
    qf = torch.randint(-(1 << 40), 1 << 40, (big,), dtype=torch.int64, device=dev, generator=g)
    r = torch.randint(-(2**31), 2**31 - 1, (big, ctx.nw), dtype=torch.int32, device=dev, generator=g)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((big, ctx.ct_words), dtype=torch.int32, device=dev)
    ops.encrypt(qf, r, big, cts)
    vals = torch.empty(big, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(ctx.lib.sfxb_ctx_stream(ctx.h), device=dev)
    out = {"small_tpi": os.environ.get("SFXB_DEC_SMALL_TPI", "default")}
    for count in (3584, 7168, 14336, 28672, 57344, 114688):
        ops.decrypt(cts, count, vals)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            ops.decrypt(cts, count, vals)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[str(count)] = round(statistics.median(ts), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
