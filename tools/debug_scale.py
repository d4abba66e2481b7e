import sys, os
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from keys import key
from paper_2504_03909_b200 import _lib
n, p, q = key("k2048_7")
dev = torch.device("cuda:0")
R = 1000
rng = np.random.default_rng(285)
qg = rng.integers(-(1 << 40) + 1, 1 << 40, R, dtype=np.int64)
qh = rng.integers(0, 1 << 38, R, dtype=np.int64)
qf = np.stack([qg, qh], 1).reshape(-1)
active = _lib.Context(n, p, q); ops_a = _lib.DeviceOps(active)
nw, cw = active.nw, active.ct_words
r = torch.randint(-(2**31), 2**31 - 1, (2 * R, nw), dtype=torch.int32, device=dev)
r[:, -1] &= 0x3FFFFFFF
cts = torch.empty((2 * R, cw), dtype=torch.int32, device=dev)
ops_a.encrypt(torch.from_numpy(qf).to(dev), r, 2 * R, cts)
vals = torch.empty(2 * R, dtype=torch.float64, device=dev)
ops_a.decrypt(cts, 2 * R, vals)
v = vals.cpu().numpy()
print("direct dec ok:", np.array_equal(v, np.ldexp(qf.astype(np.float64), -40)), v[:4], np.ldexp(qf[:4].astype(np.float64), -40))
# host path
c2 = active.encrypt(qf[:8], r[:8].cpu().numpy().view(np.uint32))
print("host vs dev cts equal:", np.array_equal(c2, cts[:8].cpu().numpy().view(np.uint32)))
v2, _ = active.decrypt(c2)
print("host dec:", v2[:4])
import bench
for R in (1000, 20000, 285000):
    qg = rng.integers(-(1 << 40) + 1, 1 << 40, R, dtype=np.int64)
    qh = rng.integers(0, 1 << 38, R, dtype=np.int64)
    qf = np.stack([qg, qh], 1).reshape(-1)
    r = torch.randint(-(2**31), 2**31 - 1, (2 * R, nw), dtype=torch.int32, device=dev)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((2 * R, cw), dtype=torch.int32, device=dev)
    ops_a.encrypt(torch.from_numpy(qf).to(dev), r, 2 * R, cts)
    vals = torch.empty(2 * R, dtype=torch.float64, device=dev)
    ops_a.decrypt(cts, 2 * R, vals)
    print(R, "enc->dec ok:", np.array_equal(vals.cpu().numpy(), np.ldexp(qf.astype(np.float64), -40)))
    J, K = 2, 256
    ctx = _lib.Context(n); ops = _lib.DeviceOps(ctx)
    gh = ops.gh_from_dev(cts, R)
    bins = rng.integers(0, K, (J, R), dtype=np.uint16)
    d_bins = torch.from_numpy(bins.astype(np.int16)).to(dev)
    offs = np.array([0, R], np.uint32); rows = np.arange(R, dtype=np.uint32)
    out = torch.empty((J * K * 2, cw), dtype=torch.int32, device=dev)
    ops.accumulate(gh, d_bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), 1, torch.from_numpy(rows.astype(np.int32)).to(dev), R, K, out)
    v = torch.empty(J * K * 2, dtype=torch.float64, device=dev)
    ops_a.decrypt(out, J * K * 2, v)
    got = v.cpu().numpy().reshape(J, K, 2)
    for f in range(J):
        sums = np.zeros(K, np.int64); np.add.at(sums, bins[f].astype(np.int64), qg)
        exp = np.ldexp(sums.astype(np.float64), -40)
        print("  f", f, "match", np.sum(got[f, :, 0] == exp), "/", K, got[f, :3, 0], exp[:3])
