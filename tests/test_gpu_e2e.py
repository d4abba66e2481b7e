"""End-to-end drop-in parity: the reference's own training
loop and unit suites, run with the CUDA EncryptionPlugin interposed on
sfxb::make_paillier_plugin (LD_PRELOAD of libsfxb_cuda_plugin.so), must
reproduce the CPU reference bit-for-bit: forests, partial models, op counters
and every transcript byte (which includes every gradient ciphertext and every
encrypted histogram slot on the wire)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PLUGIN = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
REF = os.path.join(ROOT, "oracle", "_ref")

sys.path.insert(0, os.path.join(HERE, "golden"))


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (built in the dev container, travels with the repo)")


def _train_with_plugin(name, devices=None, extra_env=None):
    from make_golden import TRAIN_CONFIGS

    ini, bits, seed = TRAIN_CONFIGS[name]
    env = dict(os.environ, LD_PRELOAD=PLUGIN, SFXB_PLUGIN_VERBOSE="1")
    if devices:
        env["SFXB_CUDA_DEVICES"] = devices
    env.update(extra_env or {})
    out = subprocess.run([sys.executable, os.path.join(HERE, "train_driver.py"), os.path.join(HERE, "configs", ini),
                          str(bits), str(seed)], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    stats = [ln for ln in out.stderr.splitlines() if ln.startswith("[sfxb-cuda-plugin]")]
    return json.loads(out.stdout), stats


@pytest.mark.parametrize("name", ["vertical_toy512", "vertical_threaded_3p", "vertical_c1_1024",
                                  "vertical_toy2048", "horizontal_toy1024"])
def test_reference_training_loop_with_gpu_plugin(name):
    _need(PLUGIN)
    _need(os.path.join(REF, "libsfxb_refcapi.so"))
    gpath = os.path.join(HERE, "golden", f"train_{name}.json")
    _need(gpath)
    want = json.load(open(gpath))
    got, stats = _train_with_plugin(name)
    # every party's plugin was the GPU adapter
    assert len(stats) >= 2
    if name.startswith("vertical"):
        # sibling subtraction derived histogram nodes, and the active party
        # decrypted sibling slots by verified reuse
        assert sum(int(s.split("derived_nodes=")[1].split()[0]) for s in stats) > 0
        assert sum(int(s.split("derived_slots=")[1].split()[0]) for s in stats) > 0
    else:
        # the packed vectors went through the GPU (no reference plugin is involved)
        assert sum(int(s.split("launches=")[1].split()[0]) for s in stats) > 0
    assert got["forest"] == want["forest"]
    assert got["partials"] == want["partials"]
    assert got["counters"] == want["counters"]
    assert got["transcript_bytes"] == want["transcript_bytes"]
    assert got["transcript_fnv"] == want["transcript_fnv"]


@pytest.mark.parametrize("name", ["vertical_c1_1024", "vertical_threaded_3p"])
def test_training_loop_with_device_group_plugin(name):
    """The same drop-in run with every plugin spread over a device group
    (SFXB_CUDA_DEVICES; sfxb_ctx_create_multi).  One GPU here, so the group
    repeats device 0 with 3 shards: row-sharded histograms reduced across
    shards, element-sharded encrypt/decrypt, sliced decrypt_tree."""
    _need(PLUGIN)
    _need(os.path.join(REF, "libsfxb_refcapi.so"))
    gpath = os.path.join(HERE, "golden", f"train_{name}.json")
    _need(gpath)
    want = json.load(open(gpath))
    got, stats = _train_with_plugin(name, devices="0,0,0")
    assert stats and all("shards=3" in s for s in stats)
    assert sum(int(s.split("derived_nodes=")[1].split()[0]) for s in stats) > 0
    for k in ("forest", "partials", "counters", "transcript_bytes", "transcript_fnv"):
        assert got[k] == want[k], k


@pytest.mark.parametrize("chunk", ["997", "61"])
@pytest.mark.parametrize("name", ["vertical_c1_1024", "vertical_threaded_3p"])
def test_training_loop_with_pipelined_encrypt_gh(name, chunk):
    """encrypt_gh's pipelined path (blinding factors of chunk k+1 drawn while
    the GPU encrypts chunk k, output marshalled one chunk behind) with the
    chunk shrunk to 997 or 61 so the small golden runs go through it (61: many
    chunks, a ragged last one): the same r stream, ciphertexts and transcript
    bytes."""
    _need(PLUGIN)
    _need(os.path.join(REF, "libsfxb_refcapi.so"))
    gpath = os.path.join(HERE, "golden", f"train_{name}.json")
    _need(gpath)
    want = json.load(open(gpath))
    got, _ = _train_with_plugin(name, extra_env={"SFXB_ENC_CHUNK": chunk})
    for k in ("forest", "partials", "counters", "transcript_bytes", "transcript_fnv"):
        assert got[k] == want[k], k


@pytest.mark.parametrize("pre_chunk,enc_chunk,policy", [("97", "61", None), ("5000", None, None), ("0", None, None),
                                                        ("97", "61", "always"), ("97", None, "between")])
@pytest.mark.parametrize("name", ["vertical_c1_1024", "vertical_threaded_3p", "horizontal_toy1024"])
def test_training_loop_with_precomputed_blinding(name, pre_chunk, enc_chunk, policy):
    """The offline phase (blinding powers of the next encrypt_gh drawn and
    exponentiated in the background, consumed by the online step) in small
    chunks, so later calls find partly filled queues and draw the rest
    (pipelined with a 61-value encrypt chunk), in whole chunks, and switched
    off (SFXB_ENC_PRECOMPUTE=0); launched except during decrypt calls
    (default), also during them (always) or between calls only (between):
    the same r stream, ciphertexts and transcript bytes."""
    _need(PLUGIN)
    _need(os.path.join(REF, "libsfxb_refcapi.so"))
    gpath = os.path.join(HERE, "golden", f"train_{name}.json")
    _need(gpath)
    want = json.load(open(gpath))
    env = {"SFXB_ENC_PRECOMPUTE_CHUNK": pre_chunk} if pre_chunk != "0" else {"SFXB_ENC_PRECOMPUTE": "0"}
    if policy:
        env["SFXB_ENC_PRECOMPUTE"] = policy
    if enc_chunk:
        env["SFXB_ENC_CHUNK"] = enc_chunk
    got, _ = _train_with_plugin(name, extra_env=env)
    for k in ("forest", "partials", "counters", "transcript_bytes", "transcript_fnv"):
        assert got[k] == want[k], k


@pytest.mark.parametrize("suite", ["test_processor", "test_federation"])
def test_reference_suites_with_gpu_plugin(suite):
    """The reference's own doctest suites (oracle/_ref, doctest shim) pass with
    every Paillier plugin they create coming from the GPU adapter."""
    _need(PLUGIN)
    binary = os.path.join(REF, suite)
    _need(binary)
    _need(os.path.join(REF, "golden"))
    env = dict(os.environ, LD_PRELOAD=PLUGIN)
    out = subprocess.run([binary], cwd=REF, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-1500:], out.stderr[-3000:])
    assert "failed: 0" in out.stdout
