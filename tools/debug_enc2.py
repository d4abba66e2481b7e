import sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from keys import key
from paper_2504_03909_b200 import _lib
n, p, q = key("k2048_7")
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q); ops = _lib.DeviceOps(ctx)
nw, cw = ctx.nw, ctx.ct_words
rng = np.random.default_rng(1)
count = 60000
qf = torch.from_numpy(rng.integers(-(1 << 40), 1 << 40, count, dtype=np.int64)).to(dev)
r = torch.randint(-(2**31), 2**31 - 1, (count, nw), dtype=torch.int32, device=dev)
r[:, -1] &= 0x3FFFFFFF
big = torch.empty((count, cw), dtype=torch.int32, device=dev)
ops.encrypt(qf, r, count, big)
small = torch.empty((count, cw), dtype=torch.int32, device=dev)
for s in range(0, count, 1000):
    ops.encrypt(qf[s:s+1000], r[s:s+1000], 1000, small[s:s+1000])
bad = torch.nonzero((big != small).any(dim=1)).flatten().cpu().numpy()
print("bad", len(bad), bad[:40])
big2 = torch.empty((count, cw), dtype=torch.int32, device=dev)
ops.encrypt(qf, r, count, big2)
bad2 = torch.nonzero((big2 != small).any(dim=1)).flatten().cpu().numpy()
print("bad (2nd run)", len(bad2), bad2[:20], "same set:", set(bad.tolist()) == set(bad2.tolist()))
