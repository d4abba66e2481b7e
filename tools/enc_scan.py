import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from keys import key
from paper_2504_03909_b200 import _lib
n, p, q = key("k2048_7")
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q); ops = _lib.DeviceOps(ctx)
g = torch.Generator(device=dev).manual_seed(1)
for count in (8192, 32768, 65536, 98304, 131072, 32768):
    qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
    r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
    ops.encrypt(qf, r, count, cts)
    ctx.profile(True)
    t0 = time.perf_counter(); ops.encrypt(qf, r, count, cts); dt = time.perf_counter() - t0
    nl, ms = ctx.kernel_time(1); ctx.profile(False)
    print(f"{count}: {dt*1e3:.1f} ms wall, {count/dt:.0f} enc/s; exp kernels {ms:.1f} ms ({nl} launches)", flush=True)
