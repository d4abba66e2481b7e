"""Row-sharded multi-GPU encrypted histogram.

One process per GPU.  Each rank holds the gradient ciphertexts and bin
columns of a contiguous row range and builds PARTIAL histograms (Montgomery
form, every slot a product over its own rows only).  Homomorphic addition is a
modular product, so the partials cannot be combined by an NCCL sum; instead

  1. the slot axis is cut into `world` equal slices (padded),
  2. ``all_to_all_single`` sends slice s of every rank's partial to rank s
     (each rank receives world × slice, moving (world−1)/world of one partial
     instead of the (world−1) partials of an all-gather),
  3. rank s multiplies its world slices element-wise with the K4 kernel
     (sfxb_reduce_partials_dev) into the plain-form result for its slice.

The collective and the layout logic are independent of the reduce, so the
CPU tests drive the same functions with the gloo backend and an oracle
reduce (tests/test_dist_cpu.py).

Tree mode (sibling subtraction) uses column slices instead (the device
group's order, include/sfxb_cuda.h "rank-sliced histograms"): every node's
2·J·K slots are cut into `world` column blocks of jl, rank k owns block k of
every node, builds only the smaller siblings' partials, and derives the
larger ones on its own block after the exchange — the batch inversion and
the per-slot work shard with the ranks.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def row_shard(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_rows, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slice_len(n_slots: int, world: int) -> int:
    return (n_slots + world - 1) // world


def padded_slots(n_slots: int, world: int) -> int:
    return slice_len(n_slots, world) * world


def exchange(partial: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """partial: [padded_slots, ct_words] on this rank -> [world, slice, ct_words]
    holding slice `rank` of every rank's partial (rank-major)."""
    assert partial.shape[0] % world == 0
    recv = torch.empty_like(partial)
    if world == 1:
        recv.copy_(partial)
    elif partial.is_cuda and dist.get_backend(group) == "gloo":
        # host-staged path (gloo has no CUDA all_to_all): used by the
        # several-ranks-on-one-GPU logic check only
        host = torch.empty(partial.shape, dtype=partial.dtype)
        dist.all_to_all_single(host, partial.cpu().contiguous(), group=group)
        recv.copy_(host)
    else:
        dist.all_to_all_single(recv, partial.contiguous(), group=group)
    return recv.view(world, partial.shape[0] // world, partial.shape[1])


def reduce_slice(recv: torch.Tensor, reduce_fn) -> torch.Tensor:
    """Combine the world partial slices element-wise with `reduce_fn(parts,
    n_parts, n_slots, out)` (the K4 kernel on GPU)."""
    world, sl, cw = recv.shape
    out = torch.empty((sl, cw), dtype=recv.dtype, device=recv.device)
    reduce_fn(recv, world, sl, out)
    return out


def gather_slices(local: torch.Tensor, n_slots: int, world: int, group=None) -> torch.Tensor:
    """All ranks' reduced slices -> the full [n_slots, ct_words] histogram
    (what the active party collects)."""
    if world == 1:
        return local[:n_slots]
    if local.is_cuda and dist.get_backend(group) == "gloo":
        parts = [torch.empty(local.shape, dtype=local.dtype) for _ in range(world)]
        dist.all_gather(parts, local.cpu().contiguous(), group=group)
        return torch.cat(parts, 0)[:n_slots].to(local.device)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, 0)[:n_slots]


def column_blocks(spn: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Slot-column blocks of every node: width jl = ceil(spn / world) and the
    [lo, hi) columns of block k (the last may be short or empty)."""
    jl = (spn + world - 1) // world
    return jl, [(min(k * jl, spn), min((k + 1) * jl, spn)) for k in range(world)]


def to_column_slices(part, n_nodes: int, spn: int, world: int):
    """Reference layout of sfxb_accumulate_part_dev's output: [n_nodes*spn, cw]
    -> [world, n_nodes*jl, cw], block k = columns of block k of every node
    (zero padding past spn).  Used by the CPU tests."""
    import numpy as np

    jl, blocks = column_blocks(spn, world)
    cw = part.shape[1]
    p3 = np.asarray(part).reshape(n_nodes, spn, cw)
    out = np.zeros((world, n_nodes, jl, cw), dtype=p3.dtype)
    for k, (lo, hi) in enumerate(blocks):
        out[k, :, : hi - lo] = p3[:, lo:hi]
    return out.reshape(world, n_nodes * jl, cw)


def gather_columns(local: torch.Tensor, n_nodes: int, spn: int, world: int, group=None) -> torch.Tensor:
    """Every rank's plain block [n_nodes*jl, cw] -> the full [n_nodes*spn, cw]
    histogram (node-major, as accumulate_rows returns it)."""
    jl = (spn + world - 1) // world
    cw = local.shape[1]
    if world == 1:
        parts = [local]
    elif local.is_cuda and dist.get_backend(group) == "gloo":
        parts = [torch.empty(local.shape, dtype=local.dtype) for _ in range(world)]
        dist.all_gather(parts, local.cpu().contiguous(), group=group)
        parts = [x.to(local.device) for x in parts]
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
    full = torch.stack([x.view(n_nodes, jl, cw) for x in parts], 1)  # [n_nodes, world, jl, cw]
    return full.reshape(n_nodes, world * jl, cw)[:, :spn].reshape(n_nodes * spn, cw)


def all_reduce_counts(real: torch.Tensor, group=None) -> torch.Tensor:
    """SUM of the per-slot real-ciphertext counts over ranks (int32)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if real.is_cuda and dist.get_backend(group) == "gloo":
            host = real.cpu()
            dist.all_reduce(host, group=group)
            real.copy_(host)
        else:
            dist.all_reduce(real, group=group)
    return real
