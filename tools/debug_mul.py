import sys, random
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
from keys import key
from paper_2504_03909_b200 import _lib
from py_oracle import ints_to_words, words_to_ints
for kname in ("k512_c0ffee", "k1024_7", "k2048_7", "k3072_7"):
    n, p, q = key(kname)
    n2 = n * n
    ctx = _lib.Context(n)
    rng = random.Random(5)
    count = 200000 if kname != "k3072_7" else 60000
    a = [rng.randrange(1, n2) for _ in range(count)]
    b = [rng.randrange(1, n2) for _ in range(count)]
    # adversarial: all-ones words, values near n^2, small values
    for i in range(0, 2000):
        a[i] = n2 - 1 - rng.randrange(0, 1 << 64)
        b[i] = n2 - 1 - rng.randrange(0, 1 << 64)
    out = words_to_ints(ctx.add(ints_to_words(a, ctx.ct_words), ints_to_words(b, ctx.ct_words)))
    bad = [i for i in range(count) if out[i] != a[i] * b[i] % n2]
    print(kname, "bad", len(bad), bad[:5], flush=True)
