"""GPU parity: encrypt / ct-add / decrypt through the C ABI against the oracle
and the reference's golden vectors (bit-exact; decrypted doubles compared
bitwise).  Reference behaviour pinned: he.cpp:87-143, test_he.cpp:22-41."""
import json
import math
import os
import random

import numpy as np
import pytest

from keys import key
from paper_2504_03909_b200 import _lib
from py_oracle import Oracle, OracleKey, from_words, ints_to_words, words_to_ints

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def golden(name):
    with open(os.path.join(HERE, "golden", f"plugin_{name}.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def ctx_for(name, private=True):
    n, p, q = key(name)
    return _lib.Context(n, p, q) if private else _lib.Context(n)


def test_toy_known_answers():
    # test_he.cpp:22-41: n=35, Enc(0, r=2) = 18, Dec(Enc(3,4)·Enc(4,9)) = 7
    ctx = _lib.Context(35, 5, 7)
    c = ctx.encrypt(np.array([0], np.int64), np.array([[2]], np.uint32))
    assert from_words(c[0]) == 18
    c3 = ctx.encrypt(np.array([3], np.int64), np.array([[4]], np.uint32))
    c4 = ctx.encrypt(np.array([4], np.int64), np.array([[9]], np.uint32))
    s = ctx.add(c3, c4)
    assert from_words(s[0]) == (from_words(c3[0]) * from_words(c4[0])) % 1225
    vals, decs, plain = ctx.decrypt(s, scale=0, want_plain=True)
    assert from_words(plain[0]) == 7 and vals[0] == 7.0 and decs == 1
    # Dec(trivial zero) = 0, not counted (secure_processor.cpp:734-738)
    vals, decs = ctx.decrypt(np.array([[1, 0]], np.uint32))
    assert vals[0] == 0.0 and decs == 0
    with pytest.raises(_lib.SfxbError, match="not coprime"):
        ctx.encrypt(np.array([3], np.int64), np.array([[5]], np.uint32))
    with pytest.raises(_lib.SfxbError, match="out of range"):
        ctx.encrypt(np.array([3], np.int64), np.array([[35]], np.uint32))


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k2048_7"])
def test_encrypt_matches_reference_golden(kname):
    g = golden(kname)
    n, p, q = key(kname)
    ctx = _lib.Context(n, p, q)
    nw = ctx.nw
    r = ints_to_words([int(x, 16) for x in g["r_stream"]], nw)
    gh = np.array(g["fixture4"]["inputs"]["gh"], np.float64).reshape(-1)
    qf = np.array([ctx.encode_check(x) for x in gh], np.int64)
    cts = ctx.encrypt(qf, r[: len(qf)])
    want = [int(x, 16) for x in g["fixture4"]["cts"]]
    assert words_to_ints(cts) == want


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k1024_7", "k2048_7", "k3072_7"])
def test_encrypt_random_matches_oracle(oracle, kname):
    n, p, q = key(kname)
    ok = OracleKey(oracle, n, p, q)
    rng = random.Random(kname)
    count = 24
    qs = [rng.randrange(-(1 << 62), 1 << 62) for _ in range(count)]
    qs[:4] = [0, 1, -1, -(1 << 62)]
    rs = [rng.randrange(2, n) for _ in range(count)]
    for pub_only in (False, True):
        ctx = _lib.Context(n) if pub_only else _lib.Context(n, p, q)
        cts = ctx.encrypt(np.array(qs, np.int64), ints_to_words(rs, ctx.nw))
        got = words_to_ints(cts)
        for i in range(count):
            m = qs[i] % n
            assert got[i] == ok.encrypt_with_r(m, rs[i]), (kname, pub_only, i)


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k2048_7"])
def test_add_matches_python(kname):
    n, p, q = key(kname)
    ctx = _lib.Context(n)
    rng = random.Random(5)
    a = [rng.randrange(1, n * n) for _ in range(40)]
    b = [rng.randrange(1, n * n) for _ in range(40)]
    out = ctx.add(ints_to_words(a, ctx.ct_words), ints_to_words(b, ctx.ct_words))
    assert words_to_ints(out) == [(x * y) % (n * n) for x, y in zip(a, b)]


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k1024_7", "k2048_7", "k3072_7"])
def test_decrypt_random_matches_oracle(oracle, kname):
    n, p, q = key(kname)
    ok = OracleKey(oracle, n, p, q)
    ctx = _lib.Context(n, p, q)
    rng = random.Random(kname + "dec")
    cts = []
    for i in range(20):
        while True:
            c = rng.randrange(2, n * n)
            if c % p and c % q:
                break
        cts.append(c)
    vals, decs, plain = ctx.decrypt(ints_to_words(cts, ctx.ct_words), want_plain=True)
    assert decs == len(cts)
    want_m = [ok.decrypt(c) for c in cts]
    assert words_to_ints(plain) == want_m
    for i, m in enumerate(want_m):
        w = ok.decode_fixed(m)
        assert vals[i] == w or (np.isnan(w) and np.isnan(vals[i])), (i, vals[i], w)


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k2048_7"])
def test_decrypt_golden_slots(kname):
    g = golden(kname)
    n, p, q = key(kname)
    ctx = _lib.Context(n, p, q)
    for fx in ("fixture4", "random50"):
        slots = ints_to_words([int(x, 16) for x in g[fx]["slots"]], ctx.ct_words)
        vals, decs = ctx.decrypt(slots)
        want = np.array([float.fromhex(x) for x in g[fx]["values"]])
        assert np.array_equal(vals, want)
        assert decs == g[fx]["counters"][2] - g[fx]["counters_after_accumulate"][2]


def test_decrypt_errors():
    n, p, q = key("k512_c0ffee")
    pub = _lib.Context(n)
    with pytest.raises(_lib.AuthorizationError, match="without private key material"):
        pub.decrypt(np.zeros((1, pub.ct_words), np.uint32))
    ctx = _lib.Context(n, p, q)
    with pytest.raises(_lib.SfxbError, match="out of range"):
        ctx.decrypt(np.zeros((1, ctx.ct_words), np.uint32))
    with pytest.raises(_lib.SfxbError, match="not coprime"):
        ctx.decrypt(_lib.to_words(n, ctx.ct_words)[None, :])


def test_decode_truncates_like_mpz_get_d(oracle):
    # decode_fixed (he.cpp:138-143): mpz_get_d truncates toward zero
    n, p, q = key("k2048_7")
    ok = OracleKey(oracle, n, p, q)
    ctx = _lib.Context(n, p, q)
    rng = random.Random(3)
    ms = [(1 << 60) + 255, n - ((1 << 60) + 255), 0, 1, n - 1, (n - 1) // 2, (n + 1) // 2,
          (1 << 64) - 1, (1 << 64), (1 << 64) + 1, rng.randrange(n), (1 << 200) + 12345]
    rs = [rng.randrange(2, n) for _ in ms]
    cts = [ok.encrypt_with_r(m, r) for m, r in zip(ms, rs)]
    vals, _, plain = ctx.decrypt(ints_to_words(cts, ctx.ct_words), want_plain=True)
    assert words_to_ints(plain) == ms
    for m, v in zip(ms, vals):
        w = ok.decode_fixed(m)
        assert v == w or (np.isinf(v) and np.isinf(w) and (v > 0) == (w > 0)), (m, v, w)


@pytest.mark.parametrize("kname", ["k1024_7", "k2048_7", "k3072_7"])
def test_large_batches_equal_small_batches(oracle, kname):
    """Multi-iteration grid-stride batches (every warp of every kernel busy,
    instances of different warps at different phases) give the same
    ciphertexts and plaintexts as one-wave batches, and match the oracle."""
    import torch

    n, p, q = key(kname)
    ok = OracleKey(oracle, n, p, q)
    ctx = _lib.Context(n, p, q)
    ops = _lib.DeviceOps(ctx)
    dev = torch.device("cuda:0")
    count = {"k1024_7": 120_000, "k2048_7": 60_000, "k3072_7": 16_000}[kname]
    chunk = 1000
    g = torch.Generator(device=dev).manual_seed(9)
    qf = torch.randint(-(1 << 40), 1 << 40, (count,), dtype=torch.int64, device=dev, generator=g)
    r = torch.randint(-(2**31), 2**31 - 1, (count, ctx.nw), dtype=torch.int32, device=dev, generator=g)
    r[:, -1] &= 0x3FFFFFFF
    big = torch.empty((count, ctx.ct_words), dtype=torch.int32, device=dev)
    ops.encrypt(qf, r, count, big)
    small = torch.empty_like(big)
    for s in range(0, count, chunk):
        ops.encrypt(qf[s:s + chunk], r[s:s + chunk], min(chunk, count - s), small[s:s + chunk])
    assert torch.equal(big, small)
    c = big.cpu().numpy().view(np.uint32)
    rr = r.cpu().numpy().view(np.uint32)
    qq = qf.cpu().numpy()
    for i in [0, 1, count // 3, count - 1]:
        assert from_words(c[i]) == ok.encrypt_with_r(int(qq[i]) % n, from_words(rr[i]))
    vals = torch.empty(count, dtype=torch.float64, device=dev)
    decs = ops.decrypt(big, count, vals)
    assert decs == count
    np.testing.assert_array_equal(vals.cpu().numpy(), np.ldexp(qq.astype(np.float64), -40))


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k1024_7", "k2048_7"])
def test_encrypt_plain_words_matches_oracle(oracle, kname):
    """sfxb_encrypt_plain (packed-vector plaintexts, he.cpp:220-232): full-width
    m ∈ [0, n), CRT and public-key contexts, plus the m range check."""
    n, p, q = key(kname)
    ok = OracleKey(oracle, n, p, q)
    rng = random.Random(kname + "plain")
    ms = [0, 1, n - 1, (n - 1) // 2] + [rng.randrange(n) for _ in range(12)]
    rs = [rng.randrange(2, n) for _ in ms]
    for ctx in (_lib.Context(n, p, q), _lib.Context(n)):
        got = words_to_ints(ctx.encrypt_plain(ints_to_words(ms, ctx.nw), ints_to_words(rs, ctx.nw)))
        assert got == [ok.encrypt_with_r(m, r) for m, r in zip(ms, rs)]
        with pytest.raises(_lib.SfxbError, match="plaintext out of range"):
            ctx.encrypt_plain(ints_to_words([n], ctx.nw), ints_to_words([5], ctx.nw))


def _prime(rng, bits):
    """Deterministic random prime (Miller-Rabin, 40 bases) for odd-size keys."""
    while True:
        c = rng.getrandbits(bits) | (3 << (bits - 2)) | 1
        d, r = c - 1, 0
        while d % 2 == 0:
            d //= 2
            r += 1
        ok = True
        for _ in range(40):
            x = pow(rng.randrange(2, c - 1), d, c)
            if x in (1, c - 1):
                continue
            for _ in range(r - 1):
                x = x * x % c
                if x == c - 1:
                    break
            else:
                ok = False
                break
        if ok:
            return c


@pytest.mark.parametrize("pbits", [400, 800, 1200])
def test_primes_short_of_their_size_class_use_the_mod_p2_kernels(pbits):
    """Primes that do not fill their limb class (p < 2^(32s−1)) take the
    mod-p² CIOS exponentiations instead of the base-p digit path; both must
    agree with Python big integers (encrypt_with_r he.cpp:87-99, decrypt :105-115)."""
    rng = random.Random(pbits)
    p, q = _prime(rng, pbits), _prime(rng, pbits)
    n = p * q
    lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
    mu = pow(lam, -1, n)
    ctx = _lib.Context(n, p, q)
    count = 16
    qs = [rng.randrange(-(1 << 60), 1 << 60) for _ in range(count)]
    rs = [rng.randrange(2, n) for _ in range(count)]
    cts = words_to_ints(ctx.encrypt(np.array(qs, np.int64), ints_to_words(rs, ctx.nw)))
    n2 = n * n
    for i in range(count):
        assert cts[i] == (1 + (qs[i] % n) * n) % n2 * pow(rs[i], n, n2) % n2, i
    _, decs, plain = ctx.decrypt(ints_to_words(cts, ctx.ct_words), want_plain=True)
    assert decs == count
    assert words_to_ints(plain) == [((pow(c, lam, n2) - 1) // n) * mu % n for c in cts]


@pytest.mark.parametrize("kname", ["k1024_7", "k2048_7"])
def test_small_batch_decrypt_lanes_equal_one_lane(oracle, kname, monkeypatch):
    """Small decrypt batches, and the last partial wave of large ones, spread
    each exponentiation over 4 or 2 lanes (lower latency); the one-lane
    kernel for everything (SFXB_DEC_SMALL_TPI=0) gives the same plaintexts
    and values, and both match the oracle.  At 2048 bits one wave is ≈37.9K
    (item, prime) jobs: 28,672 items are 1.5 waves, 57,400 are 3.03."""
    n, p, q = key(kname)
    ok = OracleKey(oracle, n, p, q)
    ctx = _lib.Context(n, p, q)
    rng = random.Random(kname + "lanes")
    n2 = n * n
    base_m = [rng.randrange(n) for _ in range(48)]
    base_c = [(1 + m * n) * pow(rng.randrange(2, n), n, n2) % n2 for m in base_m]
    for count in (3, 700, 5000, 14000, 30000) + ((28672, 57400) if kname == "k2048_7" else ()):
        # homomorphic sums of random pairs: valid ciphertexts of known plaintexts
        pairs = [(rng.randrange(48), rng.randrange(48)) for _ in range(count)]
        ms = [(base_m[a] + base_m[b]) % n for a, b in pairs]
        cts = [base_c[a] * base_c[b] % n2 for a, b in pairs]
        words = ints_to_words(cts, ctx.ct_words)
        monkeypatch.delenv("SFXB_DEC_SMALL_TPI", raising=False)
        v1, d1, p1 = ctx.decrypt(words, want_plain=True)
        monkeypatch.setenv("SFXB_DEC_SMALL_TPI", "0")
        v0, d0, p0 = ctx.decrypt(words, want_plain=True)
        assert d1 == d0 == count
        assert np.array_equal(p1, p0)
        assert np.array_equal(v1.view(np.uint64), v0.view(np.uint64))
        assert words_to_ints(p1) == ms
        for i in (0, count // 2, count - 1):
            assert ok.decrypt(cts[i]) == ms[i]


@pytest.mark.parametrize("kname", ["toy35", "k512_c0ffee", "k2048_7"])
def test_encode_batch_equals_encode_check(kname):
    """sfxb_encode_batch (all host threads; encrypt_gh's encode) returns the
    per-value sfxb_encode_check results (encode_fixed, he.cpp:125-136) and
    stops at the first failing value with its message: non-finite, off the
    fixed-point grid, or |q| >= n/2 (reachable with the toy key only)."""
    n, p, q = (35, 5, 7) if kname == "toy35" else key(kname)
    ctx = _lib.Context(n, p, q)
    rng = np.random.default_rng(7)
    if kname == "toy35":
        x = rng.integers(-17, 18, 1000) * 2.0 ** -40
    else:
        x = np.concatenate([rng.uniform(-1, 1, 300_000), rng.uniform(0, 0.25, 300_000)])
    want = np.array([ctx.encode_check(v) for v in x[:2000]], np.int64)
    got, bad = ctx.encode_batch(x)
    assert bad is None and np.array_equal(got[:2000], want)
    cases = [(len(x) // 2 + 3, float("nan"), "finite"), (777 % len(x), 2.0 ** 30, "fixed-point grid"),
             (len(x) - 1, -math.inf, "finite")]
    if kname == "toy35":
        cases.append((500, 18 * 2.0 ** -40, "below n/2"))  # 2·18 >= 35
    for k, v, msg in cases:
        y = x.copy()
        y[k] = v
        if k + 5 < len(y):
            y[k + 5] = float("nan")  # a later failure must not win
        q2, first = _encode_first_bad(ctx, y)
        assert first == k and msg in ctx.lib.sfxb_last_error(ctx.h).decode()
        assert np.array_equal(q2[:k], got[:k])


def _encode_first_bad(ctx, y):
    import ctypes as C

    q = np.zeros(len(y), np.int64)
    bad = C.c_size_t(0)
    rc = ctx.lib.sfxb_encode_batch(ctx.h, np.ascontiguousarray(y), len(y), 40, q, C.byref(bad))
    assert rc == _lib.SFXB_ERR_RANGE
    return q, bad.value


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k2048_7"])
def test_offline_online_encryption_is_bit_identical(oracle, kname):
    """Blinding powers queued ahead (sfxb_blind_append on a low-priority
    second context of the key) and consumed by the online step
    (sfxb_encrypt_blind: c = (1 + m·n)·r^n mod n²) give exactly the
    ciphertexts of sfxb_encrypt with the same r, for fixed-point and word
    plaintexts; the queue is FIFO across appends, pops and partial takes."""
    import ctypes as C

    n, p, q = key(kname)
    ctx = _lib.Context(n, p, q)
    bg = _lib.Context(n, p, q)
    assert bg.lib.sfxb_ctx_set_low_priority(bg.h) == 0
    rng = random.Random(9)
    count = 3000
    qf = np.array([rng.randrange(-(1 << 41), 1 << 41) for _ in range(count)], np.int64)
    r = ints_to_words([rng.randrange(2, n) for _ in range(count)], ctx.nw)
    want = ctx.encrypt(qf, r)
    b = C.c_void_p()
    assert ctx.lib.sfxb_blind_create(bg.h, 2048, C.byref(b)) == 0
    try:
        assert bg.lib.sfxb_blind_append(bg.h, b, np.ascontiguousarray(r[:1500]).reshape(-1), 1500, None) == 0
        got = np.zeros((count, ctx.ct_words), np.uint32)
        assert ctx.lib.sfxb_encrypt_blind(ctx.h, b, qf[:700].ctypes.data, None, 700,
                                          got[:700].reshape(-1)) == 0
        assert ctx.lib.sfxb_blind_size(b) == 800
        # append past the tail (compaction), then take the rest in one go
        assert bg.lib.sfxb_blind_append(bg.h, b, np.ascontiguousarray(r[1500:2700]).reshape(-1), 1200, None) == 0
        assert ctx.lib.sfxb_encrypt_blind(ctx.h, b, qf[700:2700].ctypes.data, None, 2000,
                                          got[700:2700].reshape(-1)) == 0
        assert np.array_equal(got[:2700], want[:2700])
        # capacity and underflow are errors, nothing consumed
        assert bg.lib.sfxb_blind_append(bg.h, b, np.ascontiguousarray(r[:300]).reshape(-1), 2100, None) != 0
        assert ctx.lib.sfxb_encrypt_blind(ctx.h, b, qf.ctypes.data, None, 1, got[:1].reshape(-1)) != 0
        # word plaintexts (the packed path) and pop
        m = ints_to_words([rng.randrange(0, n) for _ in range(200)], ctx.nw)
        want_m = ctx.encrypt_plain(m, r[2700:2900])
        assert bg.lib.sfxb_blind_append(bg.h, b, np.ascontiguousarray(r[2600:2900]).reshape(-1), 300, None) == 0
        assert ctx.lib.sfxb_blind_pop(b, 100) == 0
        got_m = np.zeros((200, ctx.ct_words), np.uint32)
        assert ctx.lib.sfxb_encrypt_blind(ctx.h, b, None, np.ascontiguousarray(m).ctypes.data, 200,
                                          got_m.reshape(-1)) == 0
        assert np.array_equal(got_m, want_m) and ctx.lib.sfxb_blind_size(b) == 0
    finally:
        ctx.lib.sfxb_blind_free(b)


@pytest.mark.parametrize("kname", ["toy35", "k2048_7"])
def test_device_gradients_equal_reference(kname):
    """sfxb_gradients_dev (compute_gradients + quantize_gradients + encode_fixed
    on the device) against the reference's own functions (oracle/_ref
    ref_gradients): the quantized doubles and the fixed-point plaintexts are
    bit-identical, including probabilities at 0 and 1, values on rounding
    boundaries of the 2^-40 grid, and the first failing value with its message
    (NaN, off the grid, |q| >= n/2 for the toy key)."""
    import ctypes as C

    import torch

    import py_oracle as po

    if not po.reference_available():
        pytest.skip("oracle/_ref not built")
    ref = po.Reference()
    n, p, q = (35, 5, 7) if kname == "toy35" else key(kname)
    nw = max(1, (n.bit_length() + 31) // 32)
    ctx = _lib.Context(n, p, q)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(4)
    N = 20000 if kname != "toy35" else 64
    prob = rng.uniform(0, 1, N)
    prob[:6] = [0.0, 1.0, 0.5, 0.5 + 2.0 ** -41, 0.25 + 2.0 ** -42, 1 - 2.0 ** -53]
    if kname == "toy35":
        prob = rng.integers(0, 9, N) * 2.0 ** -40  # |q| tiny, below n/2 = 17
    lab = rng.integers(0, 2, N).astype(np.uint8)
    if kname == "toy35":
        lab[:] = 0

    def run_ref(pr):
        qo, gh, bad = np.zeros(2 * N, np.int64), np.zeros(2 * N), C.c_size_t()
        rc = ref.lib.ref_gradients(pr, lab, N, 40, po.to_words(n, nw), nw, qo, gh, C.byref(bad))
        return rc, qo, gh, bad.value, ref.lib.ref_last_error().decode() if rc else ""

    def run_dev(pr):
        d_q = torch.zeros(2 * N, dtype=torch.int64, device=dev)
        d_gh = torch.zeros(2 * N, dtype=torch.float64, device=dev)
        bad = C.c_size_t()
        d_p, d_l = torch.from_numpy(pr).to(dev), torch.from_numpy(lab).to(dev)  # kept alive over the call
        torch.cuda.synchronize()
        rc = ctx.lib.sfxb_gradients_dev(ctx.h, d_p.data_ptr(), d_l.data_ptr(), N, 40, d_q.data_ptr(),
                                        d_gh.data_ptr(), C.byref(bad))
        torch.cuda.synchronize()
        return rc, d_q.cpu().numpy(), d_gh.cpu().numpy(), bad.value, (
            ctx.lib.sfxb_last_error(ctx.h).decode() if rc else "")

    rc, q_ref, gh_ref, bad_ref, _ = run_ref(prob)
    rc2, q_dev, gh_dev, bad_dev, _ = run_dev(prob)
    assert rc == 0 and rc2 == 0 and bad_ref == bad_dev == 2 * N
    assert np.array_equal(gh_ref.view(np.uint64), gh_dev.view(np.uint64))
    assert np.array_equal(q_ref, q_dev)
    cases = [(N // 2, float("nan")), (N // 3, 1e30)]
    if kname == "toy35":
        cases.append((7, 18 * 2.0 ** -40))  # g = p: q = 18, 2|q| >= 35
    for k, v in cases:
        pr = prob.copy()
        pr[k] = v
        rc, q_ref, gh_ref, bad_ref, msg_ref = run_ref(pr)
        rc2, q_dev, gh_dev, bad_dev, msg_dev = run_dev(pr)
        assert bad_ref == bad_dev and (rc != 0) == (rc2 != 0), (k, v, bad_ref, bad_dev)
        if rc:
            assert msg_ref.split(":")[-1].strip() in msg_dev
            assert np.array_equal(q_ref[:bad_ref], q_dev[:bad_ref])
