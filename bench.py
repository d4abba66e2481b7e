#!/usr/bin/env python
"""bench.py — encrypted-histogram s/tree + Paillier enc/s on B200 (BASELINE.json).

Workload (BASELINE.json configs[1]): vertical 2-party HIGGS-shaped synthetic
data, 1M rows × 28 features (14 per party), 256 bins, depth 6 (histograms at
depths 0-5), 2048-bit key keygen(2048, 7).  One STEP = one tree's encrypted
histogram build: accumulate_rows for every level × party (12 calls), each row
of the frontier folded into its (node, feature, bin) slot for G and H.
Synthetic inputs: uniform bins, balanced binary frontiers (every row stays in
the frontier to depth 5), random ciphertexts < n² (the kernel cost does not
depend on the plaintexts).  The gradient ciphertexts (1 GB) exceed L2.

Reported (one JSON line, rank 0):
  value       device-resident s/tree (CUDA events on the kernels' stream,
              max over ranks); lower is better.  Each step starts from the
              tree's gradient ciphertexts in HBM and converts them to every
              party's resident form (CRT / base-n digits) inside the step
  e2e         the same through the C ABI with HOST buffers: per tree and party
              the gh ciphertexts and the bin columns are uploaded once
              (sfxb_gh_upload, sfxb_bins_upload), every level uploads its
              frontier and downloads its slots (sfxb_accumulate_tree_bins) —
              the C++ adapter's call pattern; median of --e2e-steps (5) trees
              after one warm-up tree, per-step times in `e2e_steps_s`
  enc_per_s / dec_per_s / adds_per_s: Paillier encrypt (CRT), decrypt (CRT)
              and ciphertext-add throughput, each from its own timed sample
  roofline    dominant kernel K2 (segmented Montgomery product): `achieved` =
              the 32×32→64 products its launches executed (per multiplication:
              5S²+2S at the passive party on base-n digits, 2(5s²+2s) at the
              key holder on CRT digits; sibling subtraction builds only the
              smaller children) ÷ its CUDA-event time; `peak` = the
              IMAD.WIDE.U32 carry-chain microbenchmark run in this process.
              `reference_equivalent` = the reference's work for the same tree
              (ciphertext_additions × (2s²+s), s = 128 limbs: SURVEY §8d's
              unit) ÷ the same time — it exceeds the peak because the kernels
              do fewer products than the reference algorithm, not more work
  check       (default on) bit-exact self-check of the timed pass: every
              level of every party rebuilt without sibling subtraction on this
              GPU, plus sampled slots recomputed as Python big-integer products
              mod n² (N>1: rank 0 recomputes the sharded result on one GPU)
  cpu_baseline the reference PaillierPlugin (oracle/_ref, built from the
              unmodified sources) on one host core, bounded sample,
              extrapolated with the exact per-tree addition count; plus the
              reference's encrypt and decrypt rates on all host threads

Multi-GPU (torchrun): rows are sharded contiguously; partial histograms are
exchanged with all_to_all and reduced by the K4 kernel (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "encrypted-histogram s/tree + Paillier enc/s, 1M×28, 2048-bit n, 1/2/4/8 B200"
UNIT = "s/tree"
S_LIMBS = 128  # 2048-bit n: ciphertexts mod n² are 128 u32 limbs
PRODUCTS_PER_ADD = 2 * S_LIMBS * S_LIMBS + S_LIMBS  # Montgomery modmul mod n²


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--feats", type=int, default=14, help="features per party")
    ap.add_argument("--parties", type=int, default=2)
    ap.add_argument("--bins", type=int, default=256)
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--key", default="k2048_7")
    ap.add_argument("--enc-sample", type=int, default=1 << 18)
    ap.add_argument("--dec-sample", type=int, default=1 << 18)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-sample-rows", type=int, default=12000, help="per host thread (reference arm)")
    ap.add_argument("--cpu-rows", type=int, default=40000, help="single-core cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-plugin-e2e", action="store_true", help="skip the reference-facing plugin timing")
    ap.add_argument("--no-tree", action="store_true", help="disable sibling subtraction (direct histograms)")
    ap.add_argument("--check", dest="check", action="store_true", default=True, help="(default) the self-check")
    ap.add_argument("--no-check", dest="check", action="store_false",
                    help="skip the bit-exact self-check (N=1: direct histograms of every level + sampled big-integer "
                         "slot products; N>1: rank 0 recomputes the sharded result from all rows on one GPU)")
    return ap.parse_args()


def config(a, world):
    return {
        "workload": f"vertical {a.parties}-party HIGGS-shaped synthetic {a.rows}x{a.feats * a.parties}, "
                    f"{a.bins} bins, depth {a.depth}, 2048-bit n (configs[1])",
        "rows": a.rows, "features": a.feats * a.parties, "parties": a.parties, "bins": a.bins,
        "depth": a.depth, "key": "keygen(2048, 7)", "parallelism": f"row-shard x{world}",
        "histogram": "direct per-node products" if a.no_tree else
                     "sibling subtraction: levels >= 1 build the smaller child, larger = parent * smaller^-1 mod n^2",
        "l2": "inputs > L2 (gh ciphertexts 1 GB)",
    }


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ synthetic frontier


def frontiers(n_rows: int, depth: int, seed: int):
    """Balanced binary frontiers: node(depth d) = top d bits of a per-row key;
    rows ascending inside a node (the reference's NodeRows order)."""
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, 2**32, n_rows, dtype=np.uint64)
    out = []
    for d in range(depth):
        node = (keys >> np.uint64(32 - d)).astype(np.int64) if d else np.zeros(n_rows, np.int64)
        order = np.argsort(node, kind="stable").astype(np.uint32)
        counts = np.bincount(node, minlength=1 << d)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint32)
        out.append((offs, order))
    return out


def adds_per_tree(bins_per_party, fronts, K):
    """The reference's ciphertext_additions for one tree (fold_into law)."""
    total = 0
    for offs, rows in fronts:
        N = len(offs) - 1
        node_of = np.repeat(np.arange(N), np.diff(offs))
        for bins in bins_per_party:
            for f in range(bins.shape[0]):
                key = node_of * K + bins[f][rows].astype(np.int64)
                c = np.bincount(key, minlength=N * K)
                total += 2 * int(np.maximum(c - 1, 0).sum())
    return total


def rand_words(rng, count, words, top_mask=0x3FFFFFFF):
    x = rng.integers(0, 2**32, (count, words), dtype=np.uint64).astype(np.uint32)
    x[:, -1] &= np.uint32(top_mask)  # < 2^(32·words − 2) <= n² (n has exactly 2048 bits)
    return x


# ------------------------------------------------------------------ CPU baseline


def cpu_baseline(a, n, nw, adds_tree, threads: int = 1):
    """Reference PaillierPlugin::accumulate_rows on a bounded level-0 sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import py_oracle as po

    S = min(a.cpu_rows if threads <= 1 else a.cpu_sample_rows * threads, a.rows)
    rng = np.random.default_rng(11)
    cts = rand_words(rng, 2 * S, 2 * nw)
    bins = rng.integers(0, a.bins, (a.feats, S), dtype=np.uint16)
    offs = np.array([0, S], np.uint32)
    rows = np.arange(S, dtype=np.uint32)
    if po.reference_available():
        ref = po.Reference()
        t0 = time.perf_counter()
        if threads <= 1:
            plug = po.RefPlugin(ref, n, nw)
            plug.accumulate(cts, bins, offs, rows, a.bins)
            adds = plug.counters()[1]
        else:
            import ctypes as C

            out = C.c_uint64(0)
            ref._check(ref.lib.ref_accumulate_threaded(
                po.to_words(n, nw), nw, cts.reshape(-1), S, bins.reshape(-1), a.feats, offs, 1, rows, a.bins,
                threads, C.byref(out)))
            adds = out.value
        dt = time.perf_counter() - t0
        kind = "reference"
    else:  # oracle port (C restatement)
        ok = po.OracleKey(po.Oracle(), n)
        t0 = time.perf_counter()
        _, adds = ok.accumulate(cts, bins, offs, rows, a.bins)
        dt = time.perf_counter() - t0
        kind, threads = "port", 1
    rate = adds / dt
    return {
        "value": adds_tree / rate, "unit": UNIT, "cores": threads, "kind": kind,
        "sample": f"accumulate_rows level-0, {S} rows x {a.feats} features x {a.bins} bins, 2048-bit n: "
                  f"{adds} ciphertext additions in {dt:.2f} s ({rate:.3e} adds/s), extrapolated to "
                  f"{adds_tree} additions/tree",
        "adds_per_s": rate,
    }


def cpu_rates(n, p, q, nw, slots, threads, pairs_per_thread=32, dec_per_thread=64):
    """The reference's encrypt_gh and decrypt_histogram rates on all host
    threads (one plugin instance per thread; bounded samples): enc/s, dec/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import py_oracle as po

    if not po.reference_available():
        return None
    ref = po.Reference()
    e, es = C.c_uint64(0), C.c_double(0)
    ref._check(ref.lib.ref_encrypt_threaded(po.to_words(n, nw), nw, pairs_per_thread, threads, C.byref(e),
                                            C.byref(es)))
    cnt = min(len(slots), dec_per_thread * threads)
    d, ds = C.c_uint64(0), C.c_double(0)
    ref._check(ref.lib.ref_decrypt_threaded(po.to_words(p, nw), po.to_words(q, nw), nw,
                                            np.ascontiguousarray(slots[:cnt]).reshape(-1), cnt, threads, C.byref(d),
                                            C.byref(ds)))
    return {"enc_per_s": e.value / es.value, "dec_per_s": d.value / ds.value, "cores": threads, "kind": "reference",
            "sample": f"PaillierPlugin::encrypt_gh of {pairs_per_thread} pairs and decrypt_histogram of "
                      f"{cnt // threads} slots per thread, one plugin per host thread, 2048-bit n "
                      f"({e.value} encryptions in {es.value:.2f} s, {d.value} decryptions in {ds.value:.2f} s)"}


# ------------------------------------------------------------------ reference arm


def wire_codec(a):
    """The processor buffers one tree puts on the reference's Bus (SURVEY
    §8f rank 1; Bus::send = serialize_buffer + parse_buffer,
    federation.cpp:96-102): the gh_pairs_enc buffer (2 x rows ciphertexts)
    and the deepest level's scalar histogram (2^(depth-1) nodes), serialized
    and parsed by the reference's implementation and by the parallel codec
    LD_PRELOADed with the GPU adapter (host/wire_parallel.cpp); bytes and
    payloads compared (tools/wire_bench.cpp)."""
    import subprocess

    exe = os.path.join(ROOT, "oracle", "_ref", "wire_bench")
    plugin = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
    if not (os.path.exists(exe) and os.path.exists(plugin)):
        return {"unavailable": "oracle/_ref/wire_bench or the plugin library not built"}
    bits = {"k512_c0ffee": 512, "k1024_7": 1024, "k2048_7": 2048, "k3072_7": 3072}.get(a.key, 2048)
    env = dict(os.environ, LD_PRELOAD=plugin)
    try:
        out = subprocess.run([exe, str(a.rows), str(1 << (a.depth - 1)), str(a.feats), str(a.bins), str(bits), "1",
                              "0"], env=env, capture_output=True, text=True, timeout=600)
        res = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"wire_bench failed: {e}"}
    res["host_threads"] = os.cpu_count()
    return res


def plugin_e2e(a, devices=None, env_extra=None):
    """The reference-facing end to end: tools/plugin_bench.cpp drives the
    reference's EncryptionPlugin calls of one tree (encrypt_gh, accumulate_rows
    per level and party, decrypt_histogram per level and party) with the GPU
    adapter LD_PRELOADed over the unmodified reference library — host
    marshalling of the reference's mpz payloads included.  Four trees, the
    last reported (steady state: the first grows buffers; with the offline
    phase each tree's blinding powers are precomputed during the previous
    tree).  tree_wall_s includes the untimed host copies of the gradient
    payload between the calls (the Bus's share of the reference loop)."""
    import subprocess

    exe = os.path.join(ROOT, "oracle", "_ref", "plugin_bench")
    plugin = os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda_plugin.so")
    if not (os.path.exists(exe) and os.path.exists(plugin)):
        return {"unavailable": "oracle/_ref/plugin_bench or the plugin library not built"}
    bits = {"k512_c0ffee": 512, "k1024_7": 1024, "k2048_7": 2048, "k3072_7": 3072}.get(a.key, 2048)
    env = dict(os.environ, LD_PRELOAD=plugin, **(env_extra or {}))
    if devices:
        # the drop-in plugin spread over a device group (sfxb_ctx_create_multi):
        # row-sharded histograms reduced over NVLink peer memory in one kernel
        env["SFXB_CUDA_DEVICES"] = devices
    try:
        # four trees, the last reported: with the offline phase of encryption
        # the last tree is in steady state (each tree's blinding powers are
        # computed during the previous tree, sharing the GPU with it)
        out = subprocess.run([exe, str(a.rows), str(a.feats), str(a.bins), str(a.depth), str(bits), str(a.parties),
                              "4"], env=env, capture_output=True, text=True, timeout=900)
        res = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"plugin_bench failed: {e}"}
    res["pattern"] = ("reference EncryptionPlugin calls of one tree through the GPU adapter (LD_PRELOAD over "
                      "oracle/_ref/libsfxb_ref.so): encrypt_gh (2 x rows ciphertexts), accumulate_rows per level "
                      "and party, decrypt_histogram of every party's histograms; keygen(bits, 7)")
    return res


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from keys import key

    n, p, q = key(a.key)
    nw = (n.bit_length() + 31) // 32
    fronts = frontiers(a.rows, a.depth, seed=5)
    rng = np.random.default_rng(3)
    bins_pp = [rng.integers(0, a.bins, (a.feats, a.rows), dtype=np.uint16) for _ in range(a.parties)]
    adds_tree = adds_per_tree(bins_pp, fronts, a.bins)
    threads = os.cpu_count() or 1
    vals = []
    last = None
    for i in range(a.warmup + a.steps):
        last = cpu_baseline(a, n, nw, adds_tree, threads=threads)
        if i >= a.warmup:
            vals.append(last["value"])
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": dict(config(a, world), histogram="reference PaillierPlugin::accumulate_rows (direct folds)",
                       parallelism=f"{last['cores']} host threads, one plugin instance each, feature-sliced"),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "adds_per_s": last["adds_per_s"],
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm


def check_sharded(a, ops, ctxs, h_out, fronts_full, bins_pp, world, dev, cw):
    """Rank 0: rebuild every rank's gradient shard (same generators), histogram
    all rows on this GPU level by level (direct products) and compare with the
    row-sharded, exchanged and K4-reduced result of the e2e pass."""
    import torch

    from paper_2504_03909_b200 import dist as pdist

    shards = []
    for r in range(world):
        lo, hi = pdist.row_shard(a.rows, world, r)
        g = torch.Generator(device=dev).manual_seed(1000 + r)
        x = torch.randint(-(2**31), 2**31 - 1, (2 * (hi - lo), cw), dtype=torch.int32, device=dev, generator=g)
        x[:, -1] &= 0x3FFFFFFF
        shards.append(x)
    full = torch.cat(shards, 0)
    slots = 0
    for pi in range(a.parties):
        gh = ops[pi].gh_from_dev(full, a.rows)
        d_bins = torch.from_numpy(bins_pp[pi].astype(np.int16)).to(dev)
        for d, (offs, rows) in enumerate(fronts_full):
            N = len(offs) - 1
            out = torch.empty((N * a.feats * a.bins * 2, cw), dtype=torch.int32, device=dev)
            ops[pi].accumulate(gh, d_bins, a.feats, torch.from_numpy(offs.astype(np.int32)).to(dev), N,
                               torch.from_numpy(rows.astype(np.int32)).to(dev), len(rows), a.bins, out)
            want = out.cpu().numpy().view(np.uint32)
            if not np.array_equal(want, h_out[pi][d]):
                bad = int((want != h_out[pi][d]).any(axis=1).sum())
                raise SystemExit(f"--check: party {pi} level {d}: {bad} slots differ from the one-GPU histogram")
            slots += want.shape[0]
        gh.free()
    return {"ok": True, "slots_compared": slots,
            "against": "direct one-GPU histogram of all rows, bit-exact"}


def check_single(a, ops, h_out, fronts, bins_pp, parents, gh_np, n, dev, cw, samples=12):
    """N=1: the timed configuration's histograms (tree mode: the larger sibling
    derived as parent · smaller⁻¹ mod n²) against (i) every level of every
    party rebuilt with direct products on this GPU, bit-exact, and (ii)
    `samples` random slots per party at the root and the deepest level
    recomputed as Python big-integer products mod n² of the slot's gradient
    ciphertexts (empty slot = 1)."""
    import torch

    rng = np.random.default_rng(77)
    n2 = n * n
    K, J = a.bins, a.feats
    compared = 0
    for pi in range(a.parties):
        g = ops[pi].gh_upload(gh_np)
        d_bins = torch.from_numpy(bins_pp[pi].astype(np.int16)).to(dev)
        for d, (offs, rows) in enumerate(fronts):
            N = len(offs) - 1
            out = torch.empty((N * J * K * 2, cw), dtype=torch.int32, device=dev)
            ops[pi].accumulate(g, d_bins, J, torch.from_numpy(offs.astype(np.int32)).to(dev), N,
                               torch.from_numpy(rows.astype(np.int32)).to(dev), len(rows), K, out)
            direct = out.cpu().numpy().view(np.uint32)
            if not np.array_equal(direct, h_out[pi][d]):
                bad = int((direct != h_out[pi][d]).any(axis=1).sum())
                raise SystemExit(f"--check: party {pi} level {d}: {bad} slots differ from the direct histogram")
            compared += direct.shape[0]
            if d in (0, len(fronts) - 1):
                for s in rng.integers(0, N * J * K * 2, samples):
                    node, rest = divmod(int(s), J * K * 2)
                    f, rest = divmod(rest, K * 2)
                    b, w = divmod(rest, 2)
                    rr = rows[offs[node]:offs[node + 1]]
                    sel = rr[bins_pp[pi][f][rr] == b]
                    prod = 1
                    for r in sel:
                        prod = prod * int.from_bytes(gh_np[2 * int(r) + w].tobytes(), "little") % n2
                    if int.from_bytes(h_out[pi][d][s].tobytes(), "little") != prod:
                        raise SystemExit(f"--check: party {pi} level {d} slot {s} differs from the big-integer product")
        g.free()
    return {"ok": True, "slots_compared": compared, "bigint_slots": 2 * samples * a.parties,
            "against": "direct (no sibling subtraction) one-GPU histograms of every level, bit-exact; sampled "
                       "slots of the root and deepest level as Python big-integer products mod n^2"}


def run_ours(a):
    import torch
    import torch.distributed as dist

    from keys import key
    from paper_2504_03909_b200 import _lib
    from paper_2504_03909_b200 import dist as pdist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knobs: SFXB_DIST_BACKEND=gloo + SFXB_BENCH_SAME_GPU=1 run the N>1
    # data path (sharding, exchange, K4 reduce) with several ranks on one GPU,
    # exchanging through host memory — a logic check, not a performance run
    if os.environ.get("SFXB_BENCH_SAME_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SFXB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # communicator setup lines on stderr (nRanks per communicator)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    peak, peak_clk = _lib.imad_peak(local)
    n, p, q = key(a.key)
    ctxs = [_lib.Context(n, p, q, device=local)] + [_lib.Context(n, device=local) for _ in range(a.parties - 1)]
    ops = [_lib.DeviceOps(c) for c in ctxs]
    nw, cw = ctxs[0].nw, ctxs[0].ct_words
    lo, hi = pdist.row_shard(a.rows, world, rank)
    R = hi - lo
    K, J, D = a.bins, a.feats, a.depth

    # ---- synthetic inputs (identical on every rank; each keeps its rows)
    fronts_full = frontiers(a.rows, D, seed=5)
    rng = np.random.default_rng(3)
    bins_pp = [rng.integers(0, K, (J, a.rows), dtype=np.uint16) for _ in range(a.parties)]
    adds_tree_ref = adds_per_tree(bins_pp, fronts_full, K) if rank == 0 else 0
    fronts = []
    for offs, rows in fronts_full:
        # local frontier: rows of this shard, renumbered, node order kept
        N = len(offs) - 1
        node_of = np.repeat(np.arange(N), np.diff(offs))
        keep = (rows >= lo) & (rows < hi)
        lrows = (rows[keep] - lo).astype(np.uint32)
        lcount = np.bincount(node_of[keep], minlength=N)
        loffs = np.concatenate([[0], np.cumsum(lcount)]).astype(np.uint32)
        fronts.append((loffs, lrows))
    d_bins = [torch.from_numpy(b[:, lo:hi].astype(np.int16).copy()).to(dev) for b in bins_pp]
    d_front = [(torch.from_numpy(o.astype(np.int32)).to(dev), torch.from_numpy(r.astype(np.int32)).to(dev))
               for o, r in fronts]
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    gh_dev = torch.randint(-(2**31), 2**31 - 1, (2 * R, cw), dtype=torch.int32, device=dev, generator=gen)
    gh_dev[:, -1] &= 0x3FFFFFFF
    gh = [ops[pi].gh_from_dev(gh_dev, R) for pi in range(a.parties)]
    gh_host = torch.empty((2 * R, cw), dtype=torch.int32, pin_memory=True)
    gh_host.copy_(gh_dev)
    n_slots = [(1 << d) * J * K * 2 for d in range(D)]
    pad = [pdist.padded_slots(s, world) for s in n_slots]
    outs = [[torch.empty((pad[d], cw), dtype=torch.int32, device=dev) for _ in range(a.parties)] for d in range(D)]
    finals = [[None] * a.parties for _ in range(D)]
    # tree mode on N>1 ranks: column slices (sfxb_accumulate_part_dev / all_to_all /
    # sfxb_combine_slices_dev); global node sizes pick the same smaller sibling everywhere
    sliced = world > 1 and not a.no_tree
    sizes = [np.diff(o).astype(np.uint32) for o, _ in fronts_full]
    jl = ops[0].slice_width(J, K, world)
    if sliced:
        sends = [[torch.empty((world * (1 << d) * jl, cw), dtype=torch.int32, device=dev) for _ in range(a.parties)]
                 for d in range(D)]
        reals = [[torch.zeros(2 * (1 << d) * J * K, dtype=torch.int32, device=dev) for _ in range(a.parties)]
                 for d in range(D)]
        slices = [[torch.empty(((1 << d) * jl, cw), dtype=torch.int32, device=dev) for _ in range(a.parties)]
                  for d in range(D)]

    def sliced_level(pi, g, d, N):
        """One level of one party on N>1 ranks (tree mode): partial slices,
        all_to_all, count all_reduce, product + sibling subtraction per slice.
        Returns the reference addition count (on rank 0; 0 elsewhere)."""
        offs, rows = d_front[d]
        ops[pi].accumulate_part(g, d_bins[pi], J, offs, fronts[d][0], N, rows, rows.shape[0], K, parents[d],
                                sizes[d], world, sends[d][pi], reals[d][pi], sync=False)
        ctxs[pi].lib.sfxb_ctx_sync(ctxs[pi].h)
        recv = pdist.exchange(sends[d][pi], world)
        pdist.all_reduce_counts(reals[d][pi])
        adds = ops[pi].count_additions(reals[d][pi], 2 * N * J * K) if rank == 0 else 0
        # sync=True: torch's stream (the collectives) drains before the context
        # stream reads the received blocks
        ops[pi].combine_slices(g, recv, world, rank, N, J, K, parents[d], sizes[d], slices[d][pi])
        return adds
    stream = torch.cuda.ExternalStream(ctxs[0].lib.sfxb_ctx_stream(ctxs[0].h), device=dev)

    # parent of node i at depth d is node i // 2 of depth d−1 (frontiers() builds
    # a binary tree); level 0 has none
    parents = [np.full(1, -1, np.int32)] + [np.arange(1 << d, dtype=np.int32) // 2 for d in range(1, D)]

    def one_tree(sync_each=True):
        adds = 0
        # a new tree brings new gradient ciphertexts: every party converts them
        # to its resident form (digits / Montgomery) inside the step
        for pi in range(a.parties):
            gh[pi].free()
            gh[pi] = ops[pi].gh_from_dev(gh_dev, R)
        for d in range(D):
            offs, rows = d_front[d]
            N = offs.shape[0] - 1
            for pi in range(a.parties):
                if sliced:
                    adds += sliced_level(pi, gh[pi], d, N)
                    continue
                if a.no_tree:
                    adds += ops[pi].accumulate(gh[pi], d_bins[pi], J, offs, N, rows, rows.shape[0], K, outs[d][pi],
                                               mont_out=world > 1, sync=False)
                else:
                    adds += ops[pi].accumulate_tree(gh[pi], d_bins[pi], J, offs, fronts[d][0], N, rows,
                                                    rows.shape[0], K, parents[d], outs[d][pi],
                                                    mont_out=world > 1, sync=False)
                if world > 1:
                    ctxs[pi].lib.sfxb_ctx_sync(ctxs[pi].h)
                    recv = pdist.exchange(outs[d][pi], world)
                    # reduce_partials syncs torch's stream (the NCCL op) before enqueueing
                    finals[d][pi] = pdist.reduce_slice(
                        recv, lambda parts, k, sl, out: ops[pi].reduce_partials(parts, k, sl, out))
        for c in ctxs:
            c._check(c.lib.sfxb_ctx_sync(c.h))
        return adds

    # ---- warm-up
    for _ in range(a.warmup):
        one_tree()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region (device events on the kernels' stream; all parties'
    # contexts are drained before the end event)
    for c in ctxs:
        c.profile(True)
    launches0 = sum(c.launches for c in ctxs)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    adds_timed = 0
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(a.steps):
            adds_timed += one_tree()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = sum(c.launches for c in ctxs) - launches0
    k2 = [c.kernel_stats(0) for c in ctxs]
    k2_launches = sum(x[0] for x in k2)
    k2_ms = sum(x[1] for x in k2)
    k2_modmuls = sum(x[2] for x in k2)
    kt = [c.kernel_stats(3) for c in ctxs]  # sibling-subtraction inversion/derivation
    kt_ms = sum(x[1] for x in kt)
    kt_modmuls = sum(x[2] for x in kt)
    for c in ctxs:
        c.profile(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    adds_t = torch.tensor([adds_timed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(adds_t, op=dist.ReduceOp.SUM)
    ms_step = t.item() / a.steps
    adds_step = adds_t.item() / a.steps

    # ---- e2e through the C ABI with host buffers
    h_bins = [torch.from_numpy(b[:, lo:hi].copy()).pin_memory().numpy() for b in bins_pp]
    h_front = [(o, torch.from_numpy(r.astype(np.int32)).pin_memory().numpy().view(np.uint32)) for o, r in fronts]
    h2d = d2h = 0
    e2e_times = []
    gh_np = gh_host.numpy().view(np.uint32)
    def e2e_party(pi, counters):
        # one party's calls for one tree (the adapter's pattern: gh up once,
        # then per level bins + frontier up, slots down)
        tg = time.perf_counter()
        g = ops[pi].gh_upload(gh_np)
        e2e_phase["gh_upload"] += time.perf_counter() - tg
        h2d_p, d2h_p = gh_np.nbytes, 0
        bh = None
        if world == 1 and not a.no_tree:
            # the bin columns go up once per tree (the adapter keeps them on the
            # device for the whole run; counted here per tree, conservatively)
            tb = time.perf_counter()
            bh = ops[pi].bins_upload(h_bins[pi])
            e2e_phase["bins_upload"] += time.perf_counter() - tb
            h2d_p += h_bins[pi].nbytes
        for d in range(D):
            offs, rows = h_front[d]
            if sliced:
                N = len(offs) - 1
                sliced_level(pi, g, d, N)
                ctxs[pi].lib.sfxb_ctx_sync(ctxs[pi].h)
                full = pdist.gather_columns(slices[d][pi], N, 2 * J * K, world)
                if rank == 0:
                    h_out[pi][d][:] = full.cpu().numpy().view(np.uint32)
                    d2h_p += h_out[pi][d].nbytes
            elif world > 1:
                outp = outs[d][pi]
                ops[pi].accumulate(g, d_bins[pi], J, d_front[d][0], len(offs) - 1, d_front[d][1], len(rows), K,
                                   outp, mont_out=True)
                recv = pdist.exchange(outp, world)
                fin = pdist.reduce_slice(recv, lambda parts, k, sl, out: ops[pi].reduce_partials(parts, k, sl, out))
                full = pdist.gather_slices(fin, n_slots[d], world)
                if rank == 0:
                    h_out[pi][d][:] = full.cpu().numpy().view(np.uint32)
                    d2h_p += h_out[pi][d].nbytes
            elif a.no_tree:
                ops[pi].accumulate_host(g, h_bins[pi], offs, rows, K, out=h_out[pi][d])
                d2h_p += h_out[pi][d].nbytes
            else:
                ta = time.perf_counter()
                ops[pi].accumulate_tree_bins(g, bh, J, offs, rows, K, parents[d], out=h_out[pi][d])
                e2e_phase[f"level{d}"] += time.perf_counter() - ta
                d2h_p += h_out[pi][d].nbytes
            h2d_p += offs.nbytes + rows.nbytes + (0 if bh is not None else h_bins[pi].nbytes)
        tf = time.perf_counter()
        if bh is not None:
            ops[pi].bins_free(bh)
        tf2 = time.perf_counter()
        g.free()
        e2e_phase["bins_free"] += tf2 - tf
        e2e_phase["gh_free"] += time.perf_counter() - tf2
        counters[pi] = (h2d_p, d2h_p)

    e2e_phase = collections.defaultdict(float)
    h_out = [[torch.empty((n_slots[d], cw), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
              for d in range(D)] for _ in range(a.parties)]
    # parties one after the other (the reference's default threaded=false order;
    # concurrent parties on one GPU only contend for the same SMs)
    concurrent = False
    for it in range(1 + max(1, a.e2e_steps)):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        counters = [None] * a.parties
        t0 = time.perf_counter()
        if concurrent:
            ths = [threading.Thread(target=e2e_party, args=(pi, counters)) for pi in range(a.parties)]
            for th in ths:
                th.start()
            for th in ths:
                th.join()
        else:
            for pi in range(a.parties):
                e2e_party(pi, counters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        h2d = sum(c[0] for c in counters)
        d2h = sum(c[1] for c in counters)
        if it > 0:  # first iteration is a warm-up
            e2e_times.append(dt)
        else:
            e2e_phase.clear()
    e2e = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
    check = None
    if a.check and world > 1 and rank == 0:
        check = check_sharded(a, ops, ctxs, h_out, fronts_full, bins_pp, world, dev, cw)
    elif a.check and world == 1 and not a.no_tree:
        check = check_single(a, ops, h_out, fronts, bins_pp, parents, gh_np, n, dev, cw)
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)

    # ---- enc/s and dec/s samples (per GPU, rank-local; whole-job = × world)
    E = a.enc_sample
    r_dev = torch.randint(-(2**31), 2**31 - 1, (E, nw), dtype=torch.int32, device=dev, generator=gen)
    r_dev[:, -1] &= 0x3FFFFFFF
    q_dev = torch.randint(-(1 << 41), 1 << 41, (E,), dtype=torch.int64, device=dev, generator=gen)
    enc_out = torch.empty((E, cw), dtype=torch.int32, device=dev)
    ops[0].encrypt(q_dev, r_dev, E, enc_out)  # warm-up at the timed size (scratch growth)
    ctxs[0].profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    ops[0].encrypt(q_dev, r_dev, E, enc_out, sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    enc_s = e0.elapsed_time(e1) / 1e3
    k1 = ctxs[0].kernel_stats(1)
    ctxs[0].profile(False)
    # the same batch end to end through the C ABI with host buffers (sfxb_encrypt:
    # range checks, r up, ciphertexts down), as encrypt_gh drives it
    q_host = q_dev.cpu().numpy()
    r_host = r_dev.cpu().numpy().view(np.uint32)
    ctxs[0].encrypt(q_host, r_host)  # warm-up at the timed size (staging growth)
    t0 = time.perf_counter()
    ctxs[0].encrypt(q_host, r_host)
    enc_e2e_s = time.perf_counter() - t0
    Dn = min(a.dec_sample, n_slots[D - 1])
    dec_in = outs[D - 1][0][:Dn] if world == 1 else enc_out[:Dn]
    dec_vals = torch.empty(Dn, dtype=torch.float64, device=dev)
    ops[0].decrypt(dec_in, Dn, dec_vals)  # warm-up at the timed size
    ctxs[0].profile(True)
    torch.cuda.synchronize()
    e0.record(stream)
    decs = ops[0].decrypt(dec_in, Dn, dec_vals, sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    dec_s = e0.elapsed_time(e1) / 1e3
    k3 = ctxs[0].kernel_stats(2)
    ctxs[0].profile(False)

    # ---- per-tree decryption as the active party's plugin does it: every
    # level of every party's histograms through sfxb_decrypt_tree (host
    # buffers; verified sibling reuse against the previous level)
    dec_tree = None
    if world == 1 and not a.no_tree and ctxs[0].has_private:
        def dec_pass():
            n_dec = 0
            t0 = time.perf_counter()
            for pi in range(a.parties):
                for d in range(D):
                    N = len(fronts[d][0]) - 1
                    _, dd = ctxs[0].decrypt_tree(pi, h_out[pi][d], N, parents[d] if d else None)
                    n_dec += dd
            return time.perf_counter() - t0, n_dec
        dec_pass()
        der0 = ctxs[0].dec_derived
        ctxs[0].profile(True)
        dt_s, n_dec = dec_pass()
        k3t = ctxs[0].kernel_stats(2)
        ctxs[0].profile(False)
        dec_tree = {"s_per_tree": dt_s, "decryptions": n_dec, "derived_by_sibling_reuse": ctxs[0].dec_derived - der0,
                    "crt_kernel_ms": k3t[1],
                    "pattern": "sfxb_decrypt_tree per party per level, host buffers (slots up, doubles down)"}

    if world > 1:
        # every rank is done with the GPUs: the other ranks leave, so rank 0's
        # device-group plugin arm below has all GPUs to itself
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    enc_per_s = E / enc_s * world
    dec_per_s = decs / dec_s * world
    # products the K2 launches actually executed (sibling subtraction builds only
    # the smaller children, so this is below the reference addition count)
    # family 0 counts the 32x32->64 products its launches executed (mod n^2 CIOS for the
    # passive party, CRT on base-p/q digits for the key holder)
    achieved = k2_modmuls / (k2_ms / 1e3) if k2_ms > 0 else 0.0
    # CRT exponentiations: families 1 and 2 count the 32x32->64 products their
    # launches executed (Montgomery passes mod p on base-p digits, padic.cuh)
    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config(a, world),
        "enc_per_s": enc_per_s, "dec_per_s": dec_per_s, "adds_per_s": adds_step / (ms_step / 1e3),
        "enc_e2e_per_s": E / enc_e2e_s * world,
        "ciphertext_additions_per_tree": adds_step,
        "plugin_s_per_tree_extrapolated": {
            "encrypt_2M": 2 * a.rows / enc_per_s, "histogram": ms_step / 1e3,
            "decrypt_occupied": sum(n_slots) * a.parties / dec_per_s,
            "decrypt_tree_measured": dec_tree["s_per_tree"] if dec_tree else None,
        },
        "e2e": {"value": e2e.item(), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "pattern": "C ABI with pinned host buffers: per party sfxb_gh_upload and sfxb_bins_upload once per "
                           "tree, then per level sfxb_accumulate_tree_bins (frontier up, slots down), parties in "
                           "sequence"
                           if world == 1 else
                           "per party gh up, device histograms, all_to_all + K4, slots gathered to rank 0"},
        "e2e_phase_s": {k: v / max(1, len(e2e_times)) for k, v in e2e_phase.items()},
        "e2e_steps_s": e2e_times,
        "gpu_launches": int(launches),
        "roofline": {
            "bound": "imad", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tproducts/s",
            "frac": achieved / peak if peak else None,
            # dram__bytes_read.sum + dram__bytes_write.sum of one K2 launch from the round's
            # ncu --set full capture at the bench size (profiles/r02_nd.raw.csv: k_seg_prod_nd,
            # level 0 pass 1, 1M rows): read 14.204 GB + wrote 0.231 GB, against the launch's
            # algorithmic bytes — every (row, feature) gathers its G and H digits once
            # (1M x 14 x 2 x 512 B = 14.336 GB) and writes one partial per piece (0.224 GB)
            "traffic": 14.435e9, "traffic_algorithmic": 14.56e9,
            "traffic_launch": "k_seg_prod_nd<64,4,64> level 0 pass 1 at 1M rows (ncu, profiles/r02_nd.raw.csv)",
            "kernel": "K2 segmented product: k_seg_prod_nd (passive party) + k_seg_prod_p2 (key holder)",
            "work": f"K2 executed {k2_modmuls:.4g} 32x32->64 products in the timed steps: passive party "
                    f"5S^2+2S = {5 * (cw // 2) ** 2 + 2 * (cw // 2)} per ciphertext multiplication (base-n "
                    f"digits, S = {cw // 2} limbs of n), key holder 2*(5s^2+2s) = "
                    f"{2 * (5 * (cw // 4) ** 2 + 2 * (cw // 4))} (CRT mod p^2, q^2 on base-p digits), vs "
                    f"{PRODUCTS_PER_ADD} for the reference's multiplication mod n^2; {int(adds_timed)} reference "
                    f"additions (+{kt_modmuls} multiplications mod n^2 in the sibling-subtraction inversion, "
                    f"{kt_ms:.1f} ms)",
            "kernel_launches": k2_launches, "kernel_ms": k2_ms, "kernel_share_of_step": k2_ms / ms,
            "reference_equivalent": {
                "achieved": adds_timed * PRODUCTS_PER_ADD / (k2_ms / 1e3) / 1e12 if k2_ms > 0 else None,
                "frac": adds_timed * PRODUCTS_PER_ADD / (k2_ms / 1e3) / peak if k2_ms > 0 and peak else None,
                "unit": "Tproducts/s",
                "definition": f"SURVEY 8(d) unit: reference ciphertext_additions x (2s^2+s) = {PRODUCTS_PER_ADD} "
                              "products per addition (one multiplication mod n^2), over the same K2 time; above 1 "
                              "because the kernels execute fewer products than the reference algorithm "
                              "(sibling subtraction, digit arithmetic), not more",
            },
            "peak_source": "sfxb_imad_peak: IMAD.WIDE.U32(.X) carry chains on all SMs, measured in this process "
                           "before the timed region (SM clock: see clocks)",
        },
        "roofline_encrypt": {"achieved": k1[2] / (k1[1] / 1e3) / 1e12 if k1[1] else None,
                             "peak": peak / 1e12, "unit": "Tproducts/s",
                             "frac": k1[2] / (k1[1] / 1e3) / peak if k1[1] else None,
                             "products_per_encryption": k1[2] / E if E else None,
                             "kernel": "k_enc_step1 (r^(q mod p-1) mod p) + k_p2_pow<MODE 0> (x^p mod p^2 on "
                                       "base-p digits) + k_enc_post, both primes"},
        "roofline_decrypt": {"achieved": k3[2] / (k3[1] / 1e3) / 1e12 if k3[1] else None,
                             "peak": peak / 1e12, "unit": "Tproducts/s",
                             "frac": k3[2] / (k3[1] / 1e3) / peak if k3[1] else None,
                             "products_per_decryption": k3[2] / decs if decs else None,
                             "kernel": "k_dec_pre + k_p2_pow<MODE 1> (c^(p-1) mod p^2 on base-p digits), both primes"},
        "decrypt_tree": dec_tree,
        "check": check,
        "clocks": clk.summary(),
    }
    if world == 1 and not a.no_plugin_e2e:
        line["plugin_e2e"] = plugin_e2e(a)
        # the same without the offline phase of encryption (blinding powers
        # of the next encrypt_gh precomputed in the background)
        off = plugin_e2e(a, env_extra={"SFXB_ENC_PRECOMPUTE": "0"})
        line["plugin_e2e_no_precompute"] = {k: off.get(k) for k in (
            "encrypt_gh_s", "accumulate_rows_s", "decrypt_histogram_s", "plugin_s_per_tree", "tree_wall_s",
            "unavailable")}
        line["wire"] = wire_codec(a)
    elif world > 1 and not a.no_plugin_e2e and os.environ.get("SFXB_DIST_BACKEND", "nccl") == "nccl":
        # the drop-in plugin's own multi-GPU path: one process, the N GPUs of
        # this job as a device group (the other ranks have finished)
        torch.cuda.synchronize()
        line["plugin_e2e_group"] = plugin_e2e(a, devices=",".join(str(i) for i in range(world)))
    if world == 1 and not a.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(a, n, nw, adds_tree_ref, threads=1)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)}
        try:
            line["cpu_baseline"]["paillier_rates_all_threads"] = cpu_rates(
                n, p, q, nw, h_out[0][D - 1], os.cpu_count() or 1)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"]["paillier_rates_all_threads"] = {"unavailable": str(e)}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
