"""Wall time of whole reference training runs (run_training, report.cpp:132)
with the GPU plugin interposed, per variant of the offline phase of
encryption: except during decrypt calls (default), also during them
(SFXB_ENC_PRECOMPUTE=always), between plugin calls only (=between; listed
as "nodecrypt" before it became the default) or off (=0).  The recording
wrapper (oracle/record_plugin.cpp) adds the plugin's own per-call seconds, so
the host-only share of a tree (the reference's Bus, gradients, splits) is
visible next to it.  Forests and counters must agree across variants.

    python tools/train_timing.py tests/configs/vertical_c2_2048.ini 2048 7 [trees]
"""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLUGIN = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
RECORD = os.path.join(ROOT, "oracle", "_ref", "librecord_plugin.so")


def run(ini_text, bits, seed, env_extra):
    with tempfile.NamedTemporaryFile("w", suffix=".ini", delete=False) as f:
        f.write(ini_text)
        path = f.name
    env = dict(os.environ, LD_PRELOAD=f"{RECORD} {PLUGIN}", **env_extra)
    t0 = time.perf_counter()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "train_driver.py"), path, str(bits), str(seed)],
                         capture_output=True, text=True, env=env, timeout=7200)
    wall = time.perf_counter() - t0
    os.unlink(path)
    if out.returncode != 0:
        return {"error": out.stderr[-2000:]}
    res = json.loads(out.stdout)
    rec = [json.loads(ln.split("] ", 1)[1]) for ln in out.stderr.splitlines() if ln.startswith("[sfxb-record]")]
    names = ["cuts", "gradient", "encrypt", "aggregate", "decrypt", "split"]
    return {"env": env_extra, "wall_s": wall, "phases_s": dict(zip(names, res["phases"])),
            "plugin_seconds": [r["seconds"] for r in rec], "counters": res["counters"][:3],
            "forest": res["forest"]}


def main():
    ini, bits, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    text = open(ini).read()
    if len(sys.argv) > 4:
        import re

        text = re.sub(r"num_trees = \d+", f"num_trees = {sys.argv[4]}", text)
    variants = [{}, {"SFXB_ENC_PRECOMPUTE": "always"}, {"SFXB_ENC_PRECOMPUTE": "between"}, {"SFXB_ENC_PRECOMPUTE": "0"}]
    runs = [run(text, bits, seed, v) for v in variants]
    forests = {r.get("forest") for r in runs}
    for r in runs:
        r.pop("forest", None)
    print(json.dumps({"config": ini, "trees": sys.argv[4] if len(sys.argv) > 4 else "as in the file",
                      "host_cores": os.cpu_count(), "runs": runs, "forests_identical": len(forests) == 1}, indent=1))


if __name__ == "__main__":
    main()
