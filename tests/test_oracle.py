"""CPU: pin the oracle (oracle/paillier_oracle.c) before trusting it.

* the reference's own known-answer values (test_he.cpp:22-41, :111-121)
* golden vectors produced by the unmodified reference library
  (tests/golden/plugin_*.json, tests/golden/make_golden.py)
* an independent restatement in Python big integers (pow)
* live comparison with oracle/_ref when it is built
* CRT decryption (the GPU algorithm) == the reference's c^λ mod n² decryption
"""
import json
import math
import os
import random
import sys

import numpy as np
import pytest

from keys import key
from py_oracle import (Oracle, OracleError, OracleKey, RefPlugin, Reference, ints_to_words,
                       reference_available, to_words, words_to_ints)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


def golden(name):
    with open(os.path.join(HERE, "golden", f"plugin_{name}.json")) as f:
        return json.load(f)


def test_toy_known_answers(oracle):
    # test_he.cpp:22-41
    k = OracleKey(oracle, 35, 5, 7)
    assert k.encrypt_with_r(0, 2) == 18
    assert k.decrypt(k.encrypt_with_r(3, 4) * k.encrypt_with_r(4, 9) % 1225) == 7
    assert k.decrypt(1) == 0
    with pytest.raises(OracleError, match="out of range"):
        k.encrypt_with_r(35, 2)
    with pytest.raises(OracleError, match="not coprime"):
        k.encrypt_with_r(3, 5)


def test_fixed_point_known_answers(oracle):
    # test_he.cpp:111-121: encode(-0.5, 40) = n − 2^39; toy key rejects |x|·2^s >= n/2
    n, p, q = key("k512_c0ffee")
    k = OracleKey(oracle, n, p, q)
    assert k.encode_fixed(0.0)[0] == 0
    assert k.encode_fixed(-0.5)[0] == n - 2**39
    assert k.decode_fixed(n - 2**39) == -0.5
    toy = OracleKey(oracle, 35, 5, 7)
    with pytest.raises(OracleError, match="below n/2"):
        toy.encode_fixed(1.0, 10)
    with pytest.raises(OracleError, match="finite"):
        k.encode_fixed(float("nan"))
    with pytest.raises(OracleError, match="too large"):
        k.encode_fixed(2.0**22)


def test_decode_truncates_like_mpz_get_d(oracle):
    # mpz_get_d truncates: −(2^60 + 255) -> −2^60
    n, p, q = key("k512_c0ffee")
    k = OracleKey(oracle, n, p, q)
    assert k.decode_fixed(n - (2**60 + 255), 0) == -(2.0**60)
    assert k.decode_fixed(2**60 + 255, 0) == 2.0**60


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k2048_7"])
def test_oracle_reproduces_reference_golden(oracle, kname):
    g = golden(kname)
    n, p, q = key(kname)
    k = OracleKey(oracle, n, p, q)
    seed = int(g["rng_seed"])
    assert words_to_ints(k.rng_draw(seed, len(g["r_stream"]))) == [int(x, 16) for x in g["r_stream"]]
    for fx in ("fixture4", "random50"):
        d = g[fx]
        gh = np.array(d["inputs"]["gh"], np.float64)
        cts, enc = k.encrypt_gh(gh, seed)
        assert words_to_ints(cts) == [int(x, 16) for x in d["cts"]]
        assert enc == d["counters"][0]
        nodes = d["inputs"]["nodes"]
        offs = np.cumsum([0] + [len(x) for x in nodes]).astype(np.uint32)
        rows = np.array([r for nd in nodes for r in nd], np.uint32)
        slots, adds = k.accumulate(cts, np.array(d["inputs"]["bins"], np.uint16), offs, rows, d["inputs"]["n_bins"])
        assert words_to_ints(slots) == [int(x, 16) for x in d["slots"]]
        assert adds == d["counters_after_accumulate"][1]
        vals, decs = k.decrypt_slots(slots)
        assert [float(v).hex() for v in vals] == d["values"]
        assert decs == d["counters"][2]


def test_counter_law_fixture4():
    # test_processor.cpp:383-415: enc 8 / add 8 / dec 16
    d = golden("k512_c0ffee")["fixture4"]
    assert d["counters"][:3] == [8, 8, 16]


def test_oracle_matches_python_bigints(oracle):
    n, p, q = key("k512_c0ffee")
    k = OracleKey(oracle, n, p, q)
    rng = random.Random(4)
    n2 = n * n
    lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
    mu = pow(lam, -1, n)
    for _ in range(20):
        m, r = rng.randrange(n), rng.randrange(2, n)
        c = (1 + m * n) % n2 * pow(r, n, n2) % n2
        assert k.encrypt_with_r(m, r) == c
        assert k.decrypt(c) == ((pow(c, lam, n2) - 1) // n) * mu % n == m


@pytest.mark.parametrize("kname", ["k512_c0ffee", "k1024_7", "k2048_7"])
def test_crt_decrypt_equals_reference_decrypt(oracle, kname):
    n, p, q = key(kname)
    k = OracleKey(oracle, n, p, q)
    rng = random.Random(kname)
    for _ in range(10):
        c = rng.randrange(2, n * n)
        if c % p == 0 or c % q == 0:
            continue
        assert k.decrypt(c, crt=True) == k.decrypt(c)


def test_integer_sum_oracle_matches_paillier(oracle):
    # decrypted slot == decode(Σ q_i mod n) with mpz_get_d truncation
    n, p, q = key("k512_c0ffee")
    k = OracleKey(oracle, n, p, q)
    rng = random.Random(8)
    xs = [rng.uniform(-1, 1) for _ in range(30)]
    qs = [k.encode_fixed(x)[1] for x in xs]
    acc = 1
    for x in xs:
        m, _ = k.encode_fixed(x)
        acc = acc * k.encrypt_with_r(m, rng.randrange(2, n)) % (n * n)
    vals, _ = k.decrypt_slots(ints_to_words([acc], 2 * k.nw))
    assert vals[0] == k.decode_int_sum(np.array(qs, np.int64))


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference(oracle):
    ref = Reference()
    n, p, q = key("k512_acce55")
    assert ref.keygen(512, 0xACCE55) == (n, p, q)
    k = OracleKey(oracle, n, p, q)
    nw = k.nw
    assert ref.key_id(n, nw) == k.key_id
    rng = random.Random(12)
    for _ in range(5):
        m, r = rng.randrange(n), rng.randrange(2, n)
        assert ref.encrypt_with_r(n, nw, m, r) == k.encrypt_with_r(m, r)
    # a random accumulate with empty bins, trivial-zero inputs and a partial frontier
    M, J, K = 120, 4, 16
    plug = RefPlugin(ref, n, nw)
    cts = [rng.randrange(2, n * n) for _ in range(2 * M)]
    cts[5] = cts[17] = 1
    cw = ints_to_words(cts, 2 * nw)
    bins = np.array([[rng.randrange(K) for _ in range(M)] for _ in range(J)], np.uint16)
    nodes = [sorted(rng.sample(range(M), 40)), sorted(rng.sample(range(M), 25))]
    offs = np.cumsum([0] + [len(x) for x in nodes]).astype(np.uint32)
    rows = np.array([r for nd in nodes for r in nd], np.uint32)
    want = plug.accumulate(cw, bins, offs, rows, K)
    got, adds = k.accumulate(cw, bins, offs, rows, K)
    assert np.array_equal(got, want)
    assert adds == plug.counters()[1]


def test_keys_fixture_sizes():
    for name, bits in [("k512_c0ffee", 512), ("k1024_7", 1024), ("k2048_7", 2048), ("k3072_7", 3072)]:
        n, p, q = key(name)
        assert n.bit_length() == bits and p * q == n
        assert p.bit_length() == q.bit_length() == bits // 2


def test_to_words_roundtrip():
    x = (1 << 200) + 12345
    assert words_to_ints(to_words(x, 8)[None, :]) == [x]


# ---- integer-sum oracle plugin (oracle/intsum_plugin.cpp) -----------------


def _scale_libs():
    ref = os.path.join(ROOT, "oracle", "_ref")
    libs = [os.path.join(ref, x) for x in ("libintsum_plugin.so", "librecord_plugin.so", "libsfxb_refcapi.so")]
    for p in libs:
        if not os.path.exists(p):
            pytest.skip(f"{p} not built")
    return libs[0]


@pytest.mark.parametrize("name", ["vertical_toy512", "vertical_threaded_3p"])
def test_intsum_plugin_equals_cpu_paillier(name):
    """The integer-sum oracle plugin reproduces the reference's CPU Paillier
    run: forest, partial models, enc/add/dec counters and every decrypted
    histogram (recording wrapper digests, call by call).  (Also checked on
    BASELINE config 1, 10k × 8 at 1024-bit, when the golden was made.)"""
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import TRAIN_CONFIGS, run_recorded

    intsum = _scale_libs()
    ini, bits, seed = TRAIN_CONFIGS[name]
    a = run_recorded(ini, bits, seed, None)
    b = run_recorded(ini, bits, seed, intsum)
    assert a["forest"] == b["forest"] and a["partials"] == b["partials"]
    assert a["counters"][:3] == b["counters"][:3]
    assert len(a["records"]) == len(b["records"]) >= 2
    for x, y in zip(a["records"], b["records"]):
        for k in ("key", "private", "decrypt_calls", "slots", "per_call", "fnv", "counters"):
            assert x[k] == y[k], k


@pytest.mark.parametrize("name", ["vertical_c2_2048", "vertical_c3_2048"])
def test_intsum_golden_at_scale_reproduces(name):
    """tests/golden/train_<name>_intsum.json is what the oracle plugin
    produces now (configs[1]: 1M × 28, depth 6; configs[2]: 284,807 × 30,
    3 parties threaded, depth 5; 2048-bit, two trees)."""
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import SCALE_CONFIGS, run_recorded

    intsum = _scale_libs()
    want = json.load(open(os.path.join(ROOT, "tests", "golden", f"train_{name}_intsum.json")))
    ini, bits, seed = SCALE_CONFIGS[name]
    got = run_recorded(ini, bits, seed, intsum)
    assert got["forest"] == want["forest"] and got["partials"] == want["partials"]
    assert got["counters"][:3] == want["counters"]
    for x, y in zip(got["records"], want["records"]):
        for k in ("key", "private", "decrypt_calls", "slots", "per_call", "fnv", "counters"):
            assert x[k] == y[k], k
