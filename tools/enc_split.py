"""One encrypt + one decrypt batch at bench size (for an ncu launch list of
the CRT exponentiation kernels).  Development tool."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from keys import key  # noqa: E402
from paper_2504_03909_b200 import _lib  # noqa: E402

kname = sys.argv[1] if len(sys.argv) > 1 else "k2048_7"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
n, p, q = key(kname)
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q)
ops = _lib.DeviceOps(ctx)
g = torch.Generator(device=dev).manual_seed(1)
qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
r[:, -1] &= 0x3FFFFFFF
cts = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
vals = torch.empty(count, dtype=torch.float64, device=dev)
for _ in range(2):
    ops.encrypt(qf, r, count, cts)
    ops.decrypt(cts, count, vals)
torch.cuda.synchronize()
print("ok")
