"""Parallel wire codec (paper_2504_03909_b200/host/
wire_parallel.cpp): sfxb::serialize_buffer / parse_buffer interposed over the
unmodified reference library must produce the reference's bytes and payloads
(secure_processor.cpp:119-375) — checked directly against the reference's own
definitions (tools/wire_bench.cpp) and through the reference's training loop,
whose transcript (every buffer the Bus carried) must match the golden run
byte for byte.  CPU only: the codec has no device code."""
import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
WIRE = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_wire.so")
PLUGIN = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
BENCH = os.path.join(ROOT, "oracle", "_ref", "wire_bench")

sys.path.insert(0, os.path.join(HERE, "golden"))


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (__graft_entry__.build() in the dev container)")


KINDS = ("gh_pairs_enc", "histogram_enc", "agg_result_enc", "histogram_enc_packed", "agg_result_enc_packed",
         "gh_pairs_enc_small")


def _bench(lib, args, extra_env=None):
    env = dict(os.environ, LD_PRELOAD=lib, SFXB_WIRE_VERBOSE="1", **(extra_env or {}))
    out = subprocess.run([BENCH, *map(str, args)], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1]), out.stderr


@pytest.mark.parametrize("bits,seed", [(1024, 1), (2048, 2), (3072, 3), (512, 4)])
def test_codec_matches_reference(bits, seed):
    """bytes, parsed payloads and malformed-buffer errors (exception type,
    message, byte offset; ≥ 30 malformed inputs per kind: truncations, trailing
    bytes, rewritten header / layout / length fields, bit flips) equal the
    reference's for every ciphertext kind and layout, large and small buffers —
    all handled by the codec itself, none by the reference's functions"""
    _need(WIRE)
    _need(BENCH)
    res, err = _bench(WIRE, [3000, 3, 5, 64, bits, seed])
    assert res["interposed"] and res["ok"]
    for kind in KINDS:
        r = res[kind]
        assert r["bytes_identical"] and r["parse_identical"], kind
        a, b = r["malformed_same_error"].split("/")
        assert a == b and int(b) >= 30, kind
    line = [ln for ln in err.splitlines() if ln.startswith("[sfxb-wire]")][-1]
    assert "serialize native=6 ref=0" in line and " ref=0" in line.split("parse")[1]


@pytest.mark.parametrize("top_pad,walk_test", [("1", None), ("0", None), ("1", "1")])
def test_codec_large_buffer_heap_step(top_pad, walk_test):
    """a gh buffer above 64 MB (140,000 ciphertexts at 2048-bit n) parses with
    glibc's heap-growth step raised (host/parallel.hpp TopPadScope) and without
    it (SFXB_HOST_TOP_PAD=0), its length chain walked on all threads (and with
    SFXB_WIRE_WALK_TEST: wrong range syncs, serial fallback): bytes, payloads
    and errors equal the reference's"""
    _need(WIRE)
    _need(BENCH)
    env = {"SFXB_HOST_TOP_PAD": top_pad, **({"SFXB_WIRE_WALK_TEST": walk_test} if walk_test else {})}
    res, err = _bench(WIRE, [70000, 1, 2, 16, 2048, 5], env)
    r = res["gh_pairs_enc"]
    assert res["ok"] and r["bytes"] >= 64 << 20
    assert r["bytes_identical"] and r["parse_identical"]
    a, b = r["malformed_same_error"].split("/")
    assert a == b


def test_codec_in_the_plugin_library():
    """the GPU adapter library carries the same codec"""
    _need(PLUGIN)
    _need(BENCH)
    res, err = _bench(PLUGIN, [1000, 1, 2, 16, 1024, 9])
    assert res["interposed"] and res["ok"]
    assert "serialize native=6 ref=0" in err


def test_plugin_library_needs_no_reference_symbols():
    """the adapter + codec library resolves nothing from the reference library:
    its only undefined symbols are the C ABI, GMP, libc/libstdc++ (the
    reference's types come from its headers)"""
    _need(PLUGIN)
    out = subprocess.run(["nm", "-D", "--undefined-only", "-C", PLUGIN], capture_output=True, text=True)
    assert out.returncode == 0
    assert not [ln for ln in out.stdout.splitlines() if "sfxb::" in ln], out.stdout


@pytest.mark.parametrize("name", ["vertical_toy512", "vertical_threaded_3p", "horizontal_toy1024"])
def test_training_transcript_with_codec(name):
    """the reference's vertical (and horizontal: packed layouts) training loop
    with the codec on every ciphertext buffer:
    forest, counters and every transcript byte equal the golden CPU run"""
    _need(WIRE)
    from make_golden import TRAIN_CONFIGS

    gpath = os.path.join(HERE, "golden", f"train_{name}.json")
    _need(gpath)
    _need(os.path.join(ROOT, "oracle", "_ref", "libsfxb_refcapi.so"))
    ini, bits, seed = TRAIN_CONFIGS[name]
    env = dict(os.environ, LD_PRELOAD=WIRE, SFXB_WIRE_VERBOSE="1")
    out = subprocess.run([sys.executable, os.path.join(HERE, "train_driver.py"), os.path.join(HERE, "configs", ini),
                          str(bits), str(seed)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stderr.splitlines() if ln.startswith("[sfxb-wire]")][-1]
    assert int(line.split("serialize native=")[1].split()[0]) > 0
    assert int(line.split("parse native=")[1].split()[0]) > 0
    got, want = json.loads(out.stdout), json.load(open(gpath))
    for k in ("forest", "partials", "counters", "transcript_bytes", "transcript_fnv"):
        assert got[k] == want[k], k
