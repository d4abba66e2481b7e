"""Run the reference's training loop (run_training, report.cpp:132) through
oracle/ref_capi on one INI config and print the artifacts as JSON.  Used by
tests/golden/make_golden.py (CPU plugin) and by the GPU end-to-end test with
LD_PRELOAD=paper_2504_03909_b200/lib/libsfxb_cuda_plugin.so (GPU plugin
interposed on sfxb::make_paillier_plugin)."""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
from py_oracle import Reference  # noqa: E402


def main(ini_path, bits, seed):
    ref = Reference()
    with tempfile.TemporaryDirectory() as d:
        rc = ref.lib.ref_write_private_key(int(bits), int(seed), os.path.join(d, "key.priv").encode(),
                                           os.path.join(d, "key.pub").encode())
        ref._check(rc)
        os.environ["SFXB_KEY_DIR"] = d
        out = ref.train(open(ini_path).read())
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:4])
