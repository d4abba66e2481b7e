import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from keys import key
from paper_2504_03909_b200 import _lib
n, p, q = key("k2048_7")
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q); ops = _lib.DeviceOps(ctx)
count = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = torch.Generator(device=dev).manual_seed(1)
qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
r[:, -1] &= 0x3FFFFFFF
cts = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
for _ in range(2):
    ops.encrypt(qf, r, count, cts)
print("ok")
