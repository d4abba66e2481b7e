import sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
from keys import key
from paper_2504_03909_b200 import _lib
from py_oracle import Oracle, OracleKey, from_words
n, p, q = key(sys.argv[1] if len(sys.argv) > 1 else "k2048_7")
ok = OracleKey(Oracle(), n, p, q)
dev = torch.device("cuda:0")
ctx = _lib.Context(n, p, q); ops = _lib.DeviceOps(ctx)
nw, cw = ctx.nw, ctx.ct_words
rng = np.random.default_rng(1)
for count in (2000, 8000, 20000, 60000):
    qf = rng.integers(-(1 << 40), 1 << 40, count, dtype=np.int64)
    r = torch.randint(-(2**31), 2**31 - 1, (count, nw), dtype=torch.int32, device=dev)
    r[:, -1] &= 0x3FFFFFFF
    cts = torch.empty((count, cw), dtype=torch.int32, device=dev)
    ops.encrypt(torch.from_numpy(qf).to(dev), r, count, cts)
    c = cts.cpu().numpy().view(np.uint32); rr = r.cpu().numpy().view(np.uint32)
    idx = sorted(set([0, 1, count // 2, count - 1] + list(rng.integers(0, count, 12))))
    bad = [int(i) for i in idx if from_words(c[i]) != ok.encrypt_with_r(int(qf[i]) % n, from_words(rr[i]))]
    print(count, "bad idx", bad[:10], "of", len(idx), flush=True)
