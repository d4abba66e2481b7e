"""Drop-in parity on the metric's own configuration (BASELINE configs[1], and
configs[2]):
the reference's run_training (report.cpp:132) on 1M rows × 28 features, 256
bins, depth 6, 2048-bit keygen(2048, 7), two trees, with the GPU adapter
interposed on make_paillier_plugin — against the same run with the
integer-sum oracle plugin (oracle/intsum_plugin.cpp), whose
golden was produced in the dev container (tests/golden/make_golden.py scale)
and is itself pinned against the CPU Paillier plugin (tests/test_oracle.py).
Compared: the forest text (every split and leaf), the partial models, the
enc / add / dec counters of the report and of every plugin, and EVERY
decrypted histogram (the recording wrapper oracle/record_plugin.cpp folds
each decrypt_histogram result — node ids, features, the bits of every G and
H — into a digest per call)."""
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PLUGIN = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
REF = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, os.path.join(HERE, "golden"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["vertical_c2_2048", "vertical_c3_2048"])
def test_training_loop_at_scale_matches_integer_sum_oracle(name):
    """configs[1] (1M × 28, two parties) and configs[2] (284,807 × 30, three
    parties called concurrently, fraud-like labels), 2048-bit, two trees."""
    from make_golden import SCALE_CONFIGS, run_recorded

    for p in (PLUGIN, os.path.join(REF, "librecord_plugin.so"), os.path.join(REF, "libsfxb_refcapi.so")):
        if not os.path.exists(p):
            pytest.skip(f"{p} not built")
    want = json.load(open(os.path.join(HERE, "golden", f"train_{name}_intsum.json")))
    ini, bits, seed = SCALE_CONFIGS[name]
    got = run_recorded(ini, bits, seed, PLUGIN, env={"SFXB_PLUGIN_VERBOSE": "1"}, timeout=1800)
    assert got["forest"] == want["forest"]
    assert got["partials"] == want["partials"]
    assert got["counters"][:3] == want["counters"]
    assert len(got["records"]) == len(want["records"]) >= 2
    for g, w in zip(got["records"], want["records"]):
        assert g["key"] == w["key"] and g["private"] == w["private"]
        assert g["counters"] == w["counters"]
        assert g["decrypt_calls"] == w["decrypt_calls"] and g["slots"] == w["slots"]
        assert g["per_call"] == w["per_call"]  # every decrypted histogram, call by call
        assert g["fnv"] == w["fnv"]
    # only the active party decrypts
    assert [r["decrypt_calls"] > 0 for r in got["records"]] == [r["private"] for r in got["records"]]
