"""Whole training runs at BASELINE configs[0] (vertical 2-party 10k × 8, 64
bins, 1024-bit, depth 3, 5 trees): the reference's run_training as shipped
(CPU PaillierPlugin, threaded = false and threaded = true) and with the GPU
plugin interposed (same two modes).  Wall time of the run and the
reference's own phase split (report.cpp PhaseTimes: cuts, gradient, encrypt,
aggregate, decrypt, split), plus the host's core count; forests and counters
must agree across all four runs.

    python tools/c1_timing.py > profiles/r02_c1_training.json
"""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLUGIN = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
INI = os.path.join(ROOT, "tests", "configs", "vertical_c1_1024.ini")


def run(threaded: bool, gpu: bool):
    text = open(INI).read()
    if threaded:
        text = text.replace("max_bin = 64", "max_bin = 64\nthreads = true")
    with tempfile.NamedTemporaryFile("w", suffix=".ini", delete=False) as f:
        f.write(text)
        path = f.name
    env = dict(os.environ)
    if gpu:
        env["LD_PRELOAD"] = PLUGIN
    t0 = time.perf_counter()
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "train_driver.py"), path, "1024", "7"],
                         capture_output=True, text=True, env=env, timeout=3600)
    wall = time.perf_counter() - t0
    os.unlink(path)
    if out.returncode != 0:
        return {"error": out.stderr[-2000:]}
    res = json.loads(out.stdout)
    names = ["cuts", "gradient", "encrypt", "aggregate", "decrypt", "split"]
    return {"threaded": threaded, "plugin": "gpu (LD_PRELOAD libsfxb_cuda_plugin.so)" if gpu else "reference CPU",
            "wall_s": wall, "phases_s": dict(zip(names, res["phases"])), "counters": res["counters"],
            "forest": res["forest"]}


def main():
    runs = [run(False, True), run(True, True), run(False, False), run(True, False)]
    forests = {r.get("forest") for r in runs}
    counters = {tuple(r.get("counters", [])[:3]) for r in runs}
    for r in runs:
        r.pop("forest", None)
    print(json.dumps({"config": "BASELINE configs[0]: vertical 2-party 10k x 8, 64 bins, 1024-bit keygen(1024, 7), "
                                "depth 3, 5 trees (tests/configs/vertical_c1_1024.ini)",
                      "host_cores": os.cpu_count(), "runs": runs, "forests_identical": len(forests) == 1,
                      "counters_identical": len(counters) == 1}, indent=1))


if __name__ == "__main__":
    main()
