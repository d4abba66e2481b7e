"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the dev container after `make -C oracle ref` (it needs oracle/_ref,
built from /root/reference/proj/src).  Everything written here is produced by
the reference library itself (oracle/ref_capi.cpp over libsfxb_ref.so):

  keys.json     keygen(bits, seed) / keypair_from_primes(5, 7) outputs
  plugin_*.json PaillierPlugin runs: r stream, encrypt_gh ciphertexts,
                accumulate_rows residues, decrypt_histogram values, counters

    python tests/golden/make_golden.py
"""
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from py_oracle import Reference, RefPlugin, from_words, words_to_ints  # noqa: E402

ACTIVE_SEED = (1 ^ (0x9E3779B97F4A7C15 * 1)) & (2**64 - 1)  # federation.cpp:82, party 0 salt


def hexs(xs):
    return [format(int(x), "x") for x in xs]


def main():
    ref = Reference()
    keys = {"toy": {"n": "23", "p": "5", "q": "7"}}
    specs = {
        "k512_c0ffee": (512, 0xC0FFEE),   # test_he.cpp:16-19, test_processor.cpp:18-21
        "k512_acce55": (512, 0xACCE55),   # acceptance.cpp:49-52
        "k1024_7": (1024, 7),             # SURVEY §8d keygen(bits, 7)
        "k2048_7": (2048, 7),
        "k3072_7": (3072, 7),
    }
    for name, (bits, seed) in specs.items():
        n, p, q = ref.keygen(bits, seed)
        keys[name] = {"n": format(n, "x"), "p": format(p, "x"), "q": format(q, "x")}
        print(name, n.bit_length(), flush=True)
    with open(os.path.join(HERE, "keys.json"), "w") as f:
        json.dump(keys, f, indent=1)

    # Plugin runs: the test_processor.cpp:56-62 fixture and a randomized
    # M=50, J=3, K=8 fixture in the style of test_processor.cpp:442-486.
    rnd = random.Random(99)
    M, J, K = 50, 3, 8
    bins_r = [[rnd.randrange(K) for _ in range(M)] for _ in range(J)]
    gh_r = [[(rnd.randrange(2048) - 1024) / 1024.0, rnd.randrange(1024) / 1024.0] for _ in range(M)]
    nodes_r = [[r for r in range(M) if r % 2 == 0], [r for r in range(M) if r % 2 == 1]]
    fixtures = {
        "fixture4": {
            "gh": [[1.0, 0.5], [-2.0, 1.0], [4.0, 0.25], [8.0, 2.0]],
            "bins": [[0, 1, 0, 1], [1, 1, 0, 0]],
            "feature_ids": [0, 2],
            "nodes": [[0, 1, 2, 3], [1, 2]],
            "n_bins": 2,
        },
        "random50": {"gh": gh_r, "bins": bins_r, "feature_ids": [0, 1, 2], "nodes": nodes_r, "n_bins": K},
    }
    for kname in ["k512_c0ffee", "k2048_7"]:
        kd = keys[kname]
        n, p, q = (int(kd[c], 16) for c in "npq")
        nw = (n.bit_length() + 31) // 32
        out = {"key": kname, "rng_seed": str(ACTIVE_SEED)}
        out["r_stream"] = hexs(words_to_ints(ref.rng_draw(ACTIVE_SEED, n, nw, 8)))
        for fname, fx in fixtures.items():
            plug = RefPlugin(ref, n, nw, p, q, rng_seed=ACTIVE_SEED)
            gh = np.array(fx["gh"], np.float64)
            cts = plug.encrypt_gh(gh)
            bins = np.array(fx["bins"], np.uint16)
            offs = np.cumsum([0] + [len(x) for x in fx["nodes"]]).astype(np.uint32)
            rows = np.array([r for nd in fx["nodes"] for r in nd], np.uint32)
            slots = plug.accumulate(cts, bins, offs, rows, fx["n_bins"], feature_ids=fx["feature_ids"])
            c_after_acc = plug.counters()
            vals = plug.decrypt_slots(slots, len(fx["nodes"]), bins.shape[0], fx["n_bins"])
            out[fname] = {
                "inputs": fx,
                "cts": hexs(words_to_ints(cts)),
                "slots": hexs(words_to_ints(slots)),
                "values": [float(v).hex() for v in vals],
                "counters_after_accumulate": c_after_acc,
                "counters": plug.counters(),
            }
        path = os.path.join(HERE, f"plugin_{kname}.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print("wrote", path, os.path.getsize(path), flush=True)


TRAIN_CONFIGS = {
    # name: (ini under tests/configs, key bits, key seed)
    "vertical_toy512": ("vertical_toy512.ini", 512, 0xACCE55),
    "vertical_threaded_3p": ("vertical_threaded_3p.ini", 512, 0xC0FFEE),
    "vertical_c1_1024": ("vertical_c1_1024.ini", 1024, 7),
    "horizontal_toy1024": ("horizontal_toy1024.ini", 1024, 7),
    "vertical_toy2048": ("vertical_toy2048.ini", 2048, 7),
}

# Runs too large for the CPU Paillier plugin: the reference training loop with
# the integer-sum oracle plugin (oracle/intsum_plugin.cpp, pinned against the
# CPU Paillier plugin on vertical_toy512 and vertical_c1_1024 by
# tests/test_oracle.py) under the recording wrapper (oracle/record_plugin.cpp).
SCALE_CONFIGS = {
    "vertical_c2_2048": ("vertical_c2_2048.ini", 2048, 7),
    "vertical_c3_2048": ("vertical_c3_2048.ini", 2048, 7),
}


def record_lines(stderr):
    """the recording wrapper's per-plugin JSON lines, in plugin destruction order"""
    return [json.loads(ln.split("] ", 1)[1]) for ln in stderr.splitlines() if ln.startswith("[sfxb-record]")]


def run_recorded(ini, bits, seed, preload_after, env=None, timeout=3600):
    """run_training through tests/train_driver.py with the recording wrapper
    ahead of `preload_after` (a plugin library or None = the reference's own)"""
    import subprocess

    rec = os.path.join(ROOT, "oracle", "_ref", "librecord_plugin.so")
    pre = rec + (" " + preload_after if preload_after else "")
    e = dict(os.environ, **(env or {}))
    e["LD_PRELOAD"] = pre
    drv = os.path.join(ROOT, "tests", "train_driver.py")
    out = subprocess.run([sys.executable, drv, os.path.join(ROOT, "tests", "configs", ini), str(bits), str(seed)],
                         capture_output=True, text=True, env=e, timeout=timeout)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-3000:])
    res = json.loads(out.stdout)
    res["records"] = record_lines(out.stderr)
    return res


def scale_goldens(names=None):
    """integer-sum oracle runs -> tests/golden/train_<name>_intsum.json"""
    intsum = os.path.join(ROOT, "oracle", "_ref", "libintsum_plugin.so")
    for name, (ini, bits, seed) in SCALE_CONFIGS.items():
        if names and name not in names:
            continue
        res = run_recorded(ini, bits, seed, intsum)
        keep = {k: res[k] for k in ("forest", "partials", "counters")}
        keep["counters"] = keep["counters"][:3]  # bytes differ (shorter values on the wire)
        keep["records"] = [{k: r[k] for k in ("key", "private", "decrypt_calls", "slots", "fnv", "per_call", "counters")}
                           for r in res["records"]]
        path = os.path.join(HERE, f"train_{name}_intsum.json")
        with open(path, "w") as f:
            json.dump(keep, f, indent=1)
        print("wrote", path, flush=True)


def train_goldens(names=None):
    """run_training with the reference CPU plugin -> tests/golden/train_<name>.json"""
    import subprocess

    drv = os.path.join(ROOT, "tests", "train_driver.py")
    for name, (ini, bits, seed) in TRAIN_CONFIGS.items():
        if names and name not in names:
            continue
        out = subprocess.run([sys.executable, drv, os.path.join(ROOT, "tests", "configs", ini), str(bits), str(seed)],
                             check=True, capture_output=True, text=True).stdout
        path = os.path.join(HERE, f"train_{name}.json")
        with open(path, "w") as f:
            f.write(out)
        print("wrote", path, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "train":
        train_goldens(sys.argv[2:] or None)
    elif len(sys.argv) > 1 and sys.argv[1] == "scale":
        scale_goldens(sys.argv[2:] or None)
    else:
        main()
