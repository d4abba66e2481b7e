"""Small multi-warp run of every kernel family (for compute-sanitizer)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from keys import key
from paper_2504_03909_b200 import _lib

n, p, q = key(sys.argv[1] if len(sys.argv) > 1 else "k512_c0ffee")
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q)
ops = _lib.DeviceOps(ctx)
count = 1024
g = torch.Generator(device=dev).manual_seed(1)
qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
r[:, -1] &= 0x3FFFFFFF
cts = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
ops.encrypt(qf, r, count, cts)
R, J, K = count // 2, 2, 8
gh = ops.gh_from_dev(cts, R)
bins = torch.randint(0, K, (J, R), dtype=torch.int16, device=dev, generator=g)
offs = np.array([0, R // 2, R], np.uint32)
rows = torch.arange(R, dtype=torch.int32, device=dev)
out = torch.empty((2 * J * K * 2, ctx.ct_words), dtype=torch.int32, device=dev)
ops.accumulate(gh, bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), 2, rows, R, K, out)
ops.accumulate_tree(gh, bins, J, torch.from_numpy(np.array([0, R], np.int32)).to(dev), np.array([0, R], np.uint32), 1,
                    rows, R, K, np.array([-1], np.int32), out[: J * K * 2])
ops.accumulate_tree(gh, bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), offs, 2, rows, R, K,
                    np.array([0, 0], np.int32), out)
vals = torch.empty(2 * J * K * 2, dtype=torch.float64, device=dev)
ops.decrypt(out, 2 * J * K * 2, vals)
pub = _lib.Context(n)
_lib.DeviceOps(pub).encrypt(qf[:256], r[:256], 256, cts[:256])
print("sanitize smoke ok", ctx.launches + pub.launches, "launches")
