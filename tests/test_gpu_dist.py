"""N>1 data path of bench.py on real kernels: two ranks row-shard the HIGGS-
shaped workload, build Montgomery-form partial histograms (tree mode),
exchange slices (all_to_all) and reduce them with K4; rank 0 then recomputes
every level from all rows on one GPU and requires bit-exact equality
(bench.py --check).  Only one GPU exists in this build, so both ranks share
it and exchange through host memory (gloo) — the ranks' kernels never wait on
each other; this checks the sharding/exchange/reduce logic, not NVLink."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ranks,tree", [(2, True), (2, False), (3, True)])
def test_sharded_histograms_equal_one_gpu(ranks, tree):
    env = dict(os.environ, SFXB_DIST_BACKEND="gloo", SFXB_BENCH_SAME_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr=127.0.0.1", f"--master-port={29517 + 2 * ranks + int(tree)}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(ranks), "--steps", "1", "--warmup", "3", "--rows", "30001", "--feats", "3", "--bins", "32",
           "--depth", "4", "--key", "k1024_7", "--enc-sample", "4096", "--dec-sample", "4096", "--e2e-steps", "1",
           "--no-cpu", "--check"] + ([] if tree else ["--no-tree"])
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == ranks
    assert line["check"]["ok"] and line["check"]["slots_compared"] > 0
