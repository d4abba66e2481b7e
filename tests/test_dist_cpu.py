"""CPU: the multi-GPU row-shard exchange (paper_2504_03909_b200/dist.py) with
gloo, world size 2: partial histograms of each rank's rows, all_to_all of slot
slices, element-wise modular product of the slices, gathered — equals the
single-process histogram (oracle)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03909_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _words_to_int(w):
    return int.from_bytes(np.ascontiguousarray(w, np.uint32).tobytes(), "little")


def _int_to_words(x, words):
    return np.frombuffer(x.to_bytes(4 * words, "little"), np.uint32)


def _worker(rank, world, port, n, cts, bins, offs, rows, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n2 = n * n
    R = bins.shape[1]
    lo, hi = pdist.row_shard(R, world, rank)
    J = bins.shape[0]
    N = len(offs) - 1
    n_slots = N * J * K * 2
    cw = cts.shape[1]
    # partial: product over this rank's rows (plain ints here; Montgomery on GPU)
    part = [1] * pdist.padded_slots(n_slots, world)
    for nd in range(N):
        for r in rows[offs[nd]:offs[nd + 1]]:
            if not (lo <= r < hi):
                continue
            for f in range(J):
                for g in range(2):
                    s = ((nd * J + f) * K + int(bins[f][r])) * 2 + g
                    part[s] = part[s] * _words_to_int(cts[2 * r + g]) % n2
    t = torch.from_numpy(np.stack([_int_to_words(x, cw) for x in part]).astype(np.int64))
    recv = pdist.exchange(t, world)

    def reduce_fn(parts, k, sl, out):
        for i in range(sl):
            acc = 1
            for pp in range(k):
                acc = acc * _words_to_int(parts[pp, i].numpy().astype(np.uint32)) % n2
            out[i] = torch.from_numpy(_int_to_words(acc, cw).astype(np.int64))

    mine = pdist.reduce_slice(recv, reduce_fn)
    full = pdist.gather_slices(mine, n_slots, world)
    if rank == 0:
        q.put(full.numpy().astype(np.uint32))
    dist.barrier()
    dist.destroy_process_group()


def test_row_shard_partition():
    for R in (0, 1, 7, 100):
        for W in (1, 2, 3, 8):
            spans = [pdist.row_shard(R, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == R
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))


def test_gloo_world2_exchange_equals_single_process():
    from keys import key
    from py_oracle import Oracle, OracleKey

    n, _, _ = key("k512_c0ffee")
    ok = OracleKey(Oracle(), n)
    rng = np.random.default_rng(5)
    R, J, K = 40, 2, 4
    cts = rng.integers(0, 2**32, (2 * R, 2 * ok.nw), dtype=np.uint64).astype(np.uint32)
    cts[:, -1] &= 0x3FFFFFFF
    bins = rng.integers(0, K, (J, R), dtype=np.uint16)
    nodes = [list(range(0, R, 2)), list(range(1, R, 3))]
    offs = np.cumsum([0] + [len(x) for x in nodes]).astype(np.uint32)
    rows = np.array([r for nd in nodes for r in nd], np.uint32)
    want, _ = ok.accumulate(cts, bins, offs, rows, K)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, cts, bins, offs, rows, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(got, want)


def _worker_columns(rank, world, port, n, cts, bins, offs, rows, K, q):
    """The tree-mode N>1 layout: column-block slices of every node
    (sfxb_accumulate_part_dev), all_to_all, per-block product, SUM of the
    real-ciphertext counts, gather_columns — with plain big-int products."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n2 = n * n
    R = bins.shape[1]
    lo, hi = pdist.row_shard(R, world, rank)
    J = bins.shape[0]
    N = len(offs) - 1
    spn = J * K * 2
    cw = cts.shape[1]
    part = [1] * (N * spn)
    real = np.zeros(N * spn, np.int32)
    for nd in range(N):
        for r in rows[offs[nd]:offs[nd + 1]]:
            if not (lo <= r < hi):
                continue
            for f in range(J):
                for g in range(2):
                    s = nd * spn + ((f * K + int(bins[f][r])) * 2 + g)
                    part[s] = part[s] * _words_to_int(cts[2 * r + g]) % n2
                    real[s] += 1
    p = np.stack([_int_to_words(x, cw) for x in part]).astype(np.int64)
    send = torch.from_numpy(pdist.to_column_slices(p, N, spn, world).reshape(-1, cw))
    recv = pdist.exchange(send, world)  # [world, N*jl, cw]
    jl, _ = pdist.column_blocks(spn, world)
    mine = torch.zeros((N * jl, cw), dtype=torch.int64)
    for i in range(N * jl):
        acc = 1
        for k in range(world):
            acc = acc * _words_to_int(recv[k, i].numpy().astype(np.uint32)) % n2
        mine[i] = torch.from_numpy(_int_to_words(acc, cw).astype(np.int64))
    full = pdist.gather_columns(mine, N, spn, world)
    counts = pdist.all_reduce_counts(torch.from_numpy(real))
    if rank == 0:
        adds = int(torch.clamp(counts - 1, min=0).sum())
        q.put((full.numpy().astype(np.uint32), adds))
    dist.barrier()
    dist.destroy_process_group()


def test_column_slices_layout_roundtrip():
    rng = np.random.default_rng(1)
    for N, spn, world in ((3, 10, 4), (1, 8, 8), (2, 7, 3), (4, 6, 1)):
        part = rng.integers(0, 1000, (N * spn, 2))
        sl = pdist.to_column_slices(part, N, spn, world)
        jl, blocks = pdist.column_blocks(spn, world)
        assert sl.shape == (world, N * jl, 2)
        back = np.concatenate([sl[k].reshape(N, jl, 2) for k in range(world)], 1)[:, :spn].reshape(-1, 2)
        assert np.array_equal(back, part)
        assert blocks[0][0] == 0 and blocks[-1][1] == spn


def test_gloo_world3_column_slices_equal_single_process():
    from keys import key
    from py_oracle import Oracle, OracleKey

    n, _, _ = key("k512_c0ffee")
    ok = OracleKey(Oracle(), n)
    rng = np.random.default_rng(9)
    R, J, K = 30, 1, 5  # 2·J·K = 10 slots per node: not a multiple of 3 (padded last block)
    cts = rng.integers(0, 2**32, (2 * R, 2 * ok.nw), dtype=np.uint64).astype(np.uint32)
    cts[:, -1] &= 0x3FFFFFFF
    bins = rng.integers(0, K, (J, R), dtype=np.uint16)
    nodes = [list(range(0, R, 2)), list(range(1, R, 3)), []]
    offs = np.cumsum([0] + [len(x) for x in nodes]).astype(np.uint32)
    rows = np.array([r for nd in nodes for r in nd], np.uint32)
    want, want_adds = ok.accumulate(cts, bins, offs, rows, K)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_columns, args=(r, 3, port, n, cts, bins, offs, rows, K, q))
             for r in range(3)]
    for p in procs:
        p.start()
    got, adds = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(got, want)
    assert adds == want_adds
