"""The launch-shape and kernel-choice switches change how the work is laid out
on the GPU, never the results: encrypt, decrypt and tree-mode histograms of
both party kinds hash identically under each (tests/ab_driver.py in a fresh
process per setting, since each switch is read once per process).  The
default results are themselves pinned by the parity tests."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

SWITCHES = [
    {"SFXB_P2_WAVES": "0"},          # one launch per exponentiation batch
    {"SFXB_P2_WAVES": "3"},          # three waves per launch
    {"SFXB_STEP1_WAVES": "1"},       # encrypt step 1 one wave per launch
    {"SFXB_DEC_SMALL_TPI": "0"},     # no 2/4-lane tail split in decrypt
    {"SFXB_PAIR_WIDE": "0"},         # batch inversion at the class's lanes on every tree level
    {"SFXB_GH_ND_DIRECT": "0"},      # passive gh conversion as mod-n² Montgomery + split
]


def _run(kname, extra):
    env = dict(os.environ, **extra)
    out = subprocess.run([sys.executable, os.path.join(HERE, "ab_driver.py"), kname], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("kname", ["k1024_7", "k2048_7"])
def test_switches_give_identical_results(kname):
    base = _run(kname, {})
    for sw in SWITCHES:
        assert _run(kname, sw) == base, sw


@pytest.mark.parametrize("kname", ["k1024_7", "k2048_7", "k3072_7"])
def test_encryption_wave_is_a_whole_number_of_blocks(kname):
    """sfxb_ctx_enc_wave (the adapter sizes its encrypt and offline-phase
    chunks by it): positive, a whole number of blocks' instances per prime row,
    the public-key context's wave its own."""
    sys.path.insert(0, os.path.dirname(HERE))
    from keys import key
    from paper_2504_03909_b200 import _lib

    n, p, q = key(kname)
    priv, pub = _lib.Context(n, p, q), _lib.Context(n)
    w, wp = priv.lib.sfxb_ctx_enc_wave(priv.h), pub.lib.sfxb_ctx_enc_wave(pub.h)
    assert w > 0 and wp > 0
    assert w % 16 == 0 and wp % 4 == 0


def test_encryption_wave_of_a_device_group_sums_its_shards():
    """A device group (device 0 listed twice) reports the sum of its shards'
    waves (the group context is its own shard 0)."""
    sys.path.insert(0, os.path.dirname(HERE))
    from keys import key
    from paper_2504_03909_b200 import _lib

    n, p, q = key("k2048_7")
    one = _lib.Context(n, p, q)
    grp = _lib.Context(n, p, q, devices=[0, 0])
    assert grp.lib.sfxb_ctx_enc_wave(grp.h) == 2 * one.lib.sfxb_ctx_enc_wave(one.h)
