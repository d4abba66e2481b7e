// K2: encrypted histogram (PaillierPlugin::accumulate_rows,
// secure_processor.cpp:587-620) as a segmented modular product.
//
//   1. key(i, f) = (node(i)·J + f)·K + bins[f][rows[i]]   (slot pair index)
//      counting sort of the frontier's (row, feature) items by key
//   2. pass 1: every key's rows are cut into pieces of ≤ C items; one
//      instance multiplies a piece (Montgomery form, gathered from the
//      resident gh ciphertexts), for G and H separately
//   3. pass k>1: the same over the previous pass's partials until each key
//      has one partial
//   4. finalize: plain form (or Montgomery for multi-GPU partials); empty
//      slots are the literal 1 (trivial_zero, he.cpp:123)
// Products mod n² are unique residues, so any grouping/order is bit-exact.
#pragma once
#include "kernels.cuh"

namespace sfxb {
namespace dev {

// position -> frontier node (one block per node)
__global__ void k_node_of(const uint32_t *offsets, uint32_t *node_of) {
    const uint32_t nd = blockIdx.x;
    for (uint32_t i = offsets[nd] + threadIdx.x; i < offsets[nd + 1]; i += blockDim.x) node_of[i] = nd;
}

// per (gh row) flags: bit0 = Enc(g) == 1, bit1 = Enc(h) == 1 (trivial zeros are
// skipped by fold_into and not counted, secure_processor.cpp:724-732)
template <int S4>
__global__ void k_gh_flags(const uint32_t *gh_plain, uint32_t n_samples, int ct_words, uint8_t *flags) {
    for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_samples; r += (size_t)gridDim.x * blockDim.x) {
        uint8_t f = 0;
        for (int g = 0; g < 2; ++g) {
            const uint32_t *c = gh_plain + (2 * r + g) * S4;
            bool one = c[0] == 1u;
            for (int k = 1; k < ct_words; ++k) one &= c[k] == 0u;
            f |= one ? (uint8_t)(1u << g) : (uint8_t)0;
        }
        flags[r] = f;
    }
}

struct HistArgs {
    const uint32_t *rows;
    uint32_t n_rows;
    const uint32_t *node_of;
    const uint16_t *bins;
    uint32_t n_samples;
    uint32_t J, K;
    const uint8_t *gh_flags; // may be null
    uint32_t *count;         // N·J·K
    uint32_t *ones;          // N·J·K·2 (may be null)
    uint32_t *cursor;        // N·J·K
    const uint32_t *seg_start;
    uint32_t *sorted;        // n_rows·J
    uint32_t *status;        // bit0 bin out of range, bit1 row out of range
    const uint8_t *derived;  // per frontier node: 1 = derived by sibling subtraction (may be null)
};

__global__ void k_hist_count(HistArgs a) {
    const size_t total = (size_t)a.n_rows * a.J;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const uint32_t f = (uint32_t)(t / a.n_rows), i = (uint32_t)(t % a.n_rows);
        const uint32_t row = a.rows[i];
        if (row >= a.n_samples) {
            atomicOr(a.status, 2u);
            continue;
        }
        const uint32_t b = a.bins[(size_t)f * a.n_samples + row];
        if (b >= a.K) {
            atomicOr(a.status, 1u);
            continue;
        }
        const size_t key = ((size_t)a.node_of[i] * a.J + f) * a.K + b;
        atomicAdd(a.count + key, 1u);
        if (a.gh_flags) {
            const uint8_t fl = a.gh_flags[row];
            if (fl & 1u) atomicAdd(a.ones + 2 * key, 1u);
            if (fl & 2u) atomicAdd(a.ones + 2 * key + 1, 1u);
        }
    }
}

__global__ void k_hist_scatter(HistArgs a) {
    const size_t total = (size_t)a.n_rows * a.J;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        const uint32_t f = (uint32_t)(t / a.n_rows), i = (uint32_t)(t % a.n_rows);
        const uint32_t row = a.rows[i];
        if (a.derived && a.derived[a.node_of[i]]) continue;
        const uint32_t b = a.bins[(size_t)f * a.n_samples + row];
        const size_t key = ((size_t)a.node_of[i] * a.J + f) * a.K + b;
        const uint32_t pos = a.seg_start[key] + atomicAdd(a.cursor + key, 1u);
        a.sorted[pos] = row;
    }
}

// Σ_keys,g max(count − ones − 1, 0)
__global__ void k_hist_adds(const uint32_t *count, const uint32_t *ones, size_t nkeys,
                            unsigned long long *adds) {
    unsigned long long local = 0;
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nkeys; k += (size_t)gridDim.x * blockDim.x) {
        const uint32_t c = count[k];
        for (int g = 0; g < 2; ++g) {
            const uint32_t real = c - (ones ? ones[2 * k + g] : 0u);
            local += real > 0 ? real - 1 : 0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(adds, local);
}

// pieces of ≤ C items per segment: npieces[k] = ceil(len[k] / C)
__global__ void k_npieces(const uint32_t *seg_len, size_t nkeys, uint32_t C, uint32_t *np) {
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nkeys; k += (size_t)gridDim.x * blockDim.x)
        np[k] = (seg_len[k] + C - 1) / C;
}

struct Piece {
    uint32_t start, len;
};

__global__ void k_emit_pieces(const uint32_t *seg_start, const uint32_t *seg_len, const uint32_t *piece_start,
                              size_t nkeys, uint32_t C, Piece *pieces) {
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nkeys; k += (size_t)gridDim.x * blockDim.x) {
        const uint32_t len = seg_len[k], s0 = seg_start[k], p0 = piece_start[k];
        for (uint32_t j = 0; j * C < len; ++j) pieces[p0 + j] = Piece{s0 + j * C, min(C, len - j * C)};
    }
}

// Segmented product pass.  Job j = 2·piece + gh.  Item k of a piece is
//   pass 1: gh[(2·sorted[start+k] + gh)·S]      (gather by row id)
//   pass>1: prev[(start+k)·2 + gh]·S            (contiguous partials)
// Every instance of a warp runs the same number of Montgomery products
// (shorter pieces keep their accumulator), exiting when the warp is done.
// Pieces are visited in `order` (sorted by length, longest first) so that the
// instances of a warp run pieces of (nearly) equal length; partial j is
// written at the piece's own index, keeping each key's partials contiguous.
// Work distribution: each warp claims its next NIW = 32/TPI jobs from a
// global counter (warp-uniform trip counts; no block-level rounds, so the
// tail is at most one piece).
template <int S, int TPI, int C>
__global__ void __launch_bounds__(kBlock) k_seg_prod(ModArg M, const Piece *pieces, const uint32_t *order,
                                                     size_t n_pieces, const uint32_t *sorted,
                                                     const uint32_t *src, uint32_t *dst,
                                                     unsigned long long *next_job) {
    constexpr int L = S / TPI, NI = kBlock / TPI, NIW = 32 / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    const size_t total = 2 * n_pieces;
    for (;;) {
        unsigned long long base = 0;
        if ((threadIdx.x & 31) == 0) base = atomicAdd(next_job, (unsigned long long)NIW);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= total) break;
        const size_t mine = base + (threadIdx.x & 31) / TPI;
        const bool active = mine < total;
        const size_t job = active ? mine : total - 1;
        const uint32_t pidx = order[job >> 1];
        const Piece pc = pieces[pidx];
        const uint32_t g = (uint32_t)(job & 1);
        auto item_ptr = [&](uint32_t k) -> const uint32_t * {
            const size_t idx = sorted ? (2 * (size_t)sorted[pc.start + k] + g) : (2 * (size_t)(pc.start + k) + g);
            return src + idx * S;
        };
        uint32_t acc[L], x[L];
        load_lane<S, TPI>(acc, item_ptr(0));
        for (int k = 1; k < C; ++k) {
            const bool more = active && (uint32_t)k < pc.len;
            if (!__any_sync(0xffffffffu, more)) break; // warp-uniform exit
            load_lane<S, TPI>(x, item_ptr(more ? (uint32_t)k : 0u));
            uint32_t r[L];
            mmul<S, TPI>(r, acc, x, st, N, M.np);
#pragma unroll
            for (int w = 0; w < L; ++w) acc[w] = more ? r[w] : acc[w];
        }
        if (active) store_lane<S, TPI>(dst + (2 * (size_t)pidx + g) * S, acc);
    }
}

// sort keys for the pieces: (length, index)
__global__ void k_piece_keys(const Piece *pieces, size_t n, uint32_t *len, uint32_t *idx) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        len[i] = pieces[i].len;
        idx[i] = (uint32_t)i;
    }
}

// Finalize outputs shared by the K2 variants: the Montgomery form (tree cache
// / partials) and/or the plain residue of every slot.  Slots of nodes flagged
// in `skip_node` (derived later by sibling subtraction) are not computed when
// the whole warp's instances belong to such nodes (their values are rewritten
// by k_derive, so computing them anyway is harmless).
struct FinOut {
    uint32_t *mont;          // may be null
    uint32_t *plain;         // may be null
    const uint8_t *skip_node; // may be null
    uint32_t slots_per_node; // 2·J·K
};
__device__ __forceinline__ bool fin_skip(const FinOut &o, size_t slot) {
    const bool sk = o.skip_node != nullptr && o.skip_node[slot / o.slots_per_node];
    return __all_sync(0xffffffffu, sk);
}

// Output slot (key, gh): count == 0 -> literal 1 (Montgomery one for the
// Montgomery output); else the key's single final partial.
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_hist_finalize(ModArg M, const uint32_t *count, const uint32_t *final_idx,
                                                          size_t nkeys, const uint32_t *partial, FinOut o) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L], one_m[L];
    load_const<S, TPI>(N, mr, kMod);
    load_const<S, TPI>(one_m, mr, kOne);
    SFXB_UNIFORM_LOOP(slot, active, 2 * nkeys) {
        if (fin_skip(o, slot)) continue;
        const size_t key = slot >> 1;
        const uint32_t g = (uint32_t)(slot & 1);
        const bool empty = count[key] == 0;
        uint32_t v[L];
        if (!empty) load_lane<S, TPI>(v, partial + (2 * (size_t)final_idx[key] + g) * S);
        else
#pragma unroll
            for (int w = 0; w < L; ++w) v[w] = one_m[w];
        if (o.mont && active) store_lane<S, TPI>(o.mont + slot * S, v);
        if (o.plain) {
            from_mont<S, TPI>(v, v, st, N, M.np); // Montgomery one -> 1
            if (active) store_lane<S, TPI>(o.plain + slot * S, v);
        }
    }
}

// ---------------------------------------------------------------- sibling subtraction
//
// Level d ≥ 1 of a tree: for siblings (a, b) whose parent P was histogrammed
// at level d−1, only the child with fewer rows is built directly and the other
// is derived as hist(P)·hist(small)⁻¹ mod n² (residues are unique, so this is
// bit-identical to the direct product).  The inverses of all small-child slots
// come from one Montgomery batch inversion: a pairwise product tree (up),
// one inversion of the root on the host, and the tree walked back down.

// out[i] = in[2i]·in[2i+1] (Montgomery form), or in[2i] when 2i+1 == n_in
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_pair_up(ModArg M, const uint32_t *in, size_t n_in, uint32_t *out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L], one_m[L];
    load_const<S, TPI>(N, mr, kMod);
    load_const<S, TPI>(one_m, mr, kOne);
    const size_t n_out = (n_in + 1) / 2;
    SFXB_UNIFORM_LOOP(i, active, n_out) {
        uint32_t a[L], b[L];
        load_lane<S, TPI>(a, in + 2 * i * S);
        if (2 * i + 1 < n_in) load_lane<S, TPI>(b, in + (2 * i + 1) * S);
        else
#pragma unroll
            for (int k = 0; k < L; ++k) b[k] = one_m[k];
        mmul<S, TPI>(a, a, b, st, N, M.np);
        if (active) store_lane<S, TPI>(out + i * S, a);
    }
}

// inv_out[i] = inv_parent[i/2]·in[i^1] (or inv_parent[i/2] without a sibling)
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_pair_down(ModArg M, const uint32_t *inv_parent, const uint32_t *in,
                                                      size_t n_in, uint32_t *inv_out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L], one_m[L];
    load_const<S, TPI>(N, mr, kMod);
    load_const<S, TPI>(one_m, mr, kOne);
    SFXB_UNIFORM_LOOP(i, active, n_in) {
        uint32_t a[L], b[L];
        load_lane<S, TPI>(a, inv_parent + (i / 2) * S);
        if ((i ^ 1) < n_in) load_lane<S, TPI>(b, in + (i ^ 1) * S);
        else
#pragma unroll
            for (int k = 0; k < L; ++k) b[k] = one_m[k];
        mmul<S, TPI>(a, a, b, st, N, M.np);
        if (active) store_lane<S, TPI>(inv_out + i * S, a);
    }
}

struct Derived {
    uint32_t derived, small, parent; // node indices: this level, this level, previous level
};

// gather the slots of the small siblings: v[d·spn + k] = hist[small_d·spn + k]
__global__ void k_gather_small(const uint32_t *hist, const Derived *dv, size_t n_derived, size_t spn, int S,
                               uint32_t *v) {
    const size_t words = n_derived * spn * (size_t)S;
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (size_t)gridDim.x * blockDim.x) {
        const size_t slot = w / S, k = w % S;
        const size_t d = slot / spn, j = slot % spn;
        v[w] = hist[((size_t)dv[d].small * spn + j) * S + k];
    }
}

// hist[derived_d·spn + k] = parent_hist[parent_d·spn + k] · inv_small[d·spn + k]
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_derive(ModArg M, const uint32_t *parent_hist, const uint32_t *inv_small,
                                                   const Derived *dv, size_t n_derived, size_t spn, uint32_t *hist) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(j, active, n_derived * spn) {
        const Derived d = dv[j / spn];
        const size_t k = j % spn;
        uint32_t a[L], b[L];
        load_lane<S, TPI>(a, parent_hist + ((size_t)d.parent * spn + k) * S);
        load_lane<S, TPI>(b, inv_small + j * S);
        mmul<S, TPI>(a, a, b, st, N, M.np);
        if (active) store_lane<S, TPI>(hist + ((size_t)d.derived * spn + k) * S, a);
    }
}

// out[d·spn + k] = from_mont(hist[d·spn + k]) for the derived nodes d
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_from_mont_nodes(ModArg M, const uint32_t *hist, const Derived *dv,
                                                            size_t n_derived, size_t spn, uint32_t *out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(j, active, n_derived * spn) {
        const size_t e = (size_t)dv[j / spn].derived * spn + j % spn;
        uint32_t v[L];
        load_lane<S, TPI>(v, hist + e * S);
        from_mont<S, TPI>(v, v, st, N, M.np);
        if (active) store_lane<S, TPI>(out + e * S, v);
    }
}

// out = from_mont(in) element-wise
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_from_mont_copy(ModArg M, const uint32_t *in, size_t count, uint32_t *out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(e, active, count) {
        uint32_t v[L];
        load_lane<S, TPI>(v, in + e * S);
        from_mont<S, TPI>(v, v, st, N, M.np);
        if (active) store_lane<S, TPI>(out + e * S, v);
    }
}

// x -> x·R mod M (any x < R)
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_to_mont(ModArg M, uint32_t *x, size_t count) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(e, active, count) {
        uint32_t v[L];
        load_lane<S, TPI>(v, x + e * S);
        to_mont<S, TPI>(v, v, mr, st, N);
        if (active) store_lane<S, TPI>(x + e * S, v);
    }
}

// K4: out[i] = from_mont(∏_p parts[p][i]) for Montgomery-form partials
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_reduce_parts(ModArg M, const uint32_t *parts, uint32_t n_parts,
                                                         size_t n_slots, uint32_t *out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(e, active, n_slots) {
        uint32_t acc[L], x[L];
        load_lane<S, TPI>(acc, parts + e * S);
        for (uint32_t p = 1; p < n_parts; ++p) {
            load_lane<S, TPI>(x, parts + ((size_t)p * n_slots + e) * S);
            mmul<S, TPI>(acc, acc, x, st, N, M.np);
        }
        from_mont<S, TPI>(acc, acc, st, N, M.np);
        if (active) store_lane<S, TPI>(out + e * S, acc);
    }
}

// ---------------------------------------------------------------- multi-GPU (one process)
//
// A device group holds the gh rows in contiguous row shards, one per GPU.
// Each shard builds Montgomery-form partial histograms of its own rows; shard k
// then owns slot slice [j0, j0 + jl) of every node and multiplies the partials
// of all shards for that slice, reading the peers' buffers directly over
// NVLink (P2P loads; no staging copy, no NCCL: homomorphic addition is a
// modular product, which no NCCL reduction op computes).

constexpr int kMaxShards = 16;
struct PeerSet {
    const uint32_t *p[kMaxShards];
    uint32_t n;
};

// out[node·jl + j] = ∏_shards part[node·spn + j0 + j]   (Montgomery form)
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_reduce_peer(ModArg M, PeerSet parts, size_t n_nodes, size_t spn,
                                                        size_t j0, size_t jl, uint32_t *out) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, mr, kMod);
    SFXB_UNIFORM_LOOP(e, active, n_nodes * jl) {
        const size_t src = (e / jl) * spn + j0 + e % jl;
        uint32_t acc[L], x[L];
        load_lane<S, TPI>(acc, parts.p[0] + src * S);
        for (uint32_t p = 1; p < parts.n; ++p) {
            load_lane<S, TPI>(x, parts.p[p] + src * S);
            mmul<S, TPI>(acc, acc, x, st, N, M.np);
        }
        if (active) store_lane<S, TPI>(out + e * S, acc);
    }
}

// Columns past the slots of a node in rank-sliced blocks (2·J·K not a
// multiple of world) hold the Montgomery one, so that the cross-rank product
// and the batch inversion of sibling subtraction see units there.
__global__ void k_fill_pad(uint32_t *send, uint32_t world, size_t n_nodes, size_t jl, size_t spn, int S,
                           const uint32_t *one) {
    const size_t total = (size_t)world * n_nodes * jl * S;
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (size_t)gridDim.x * blockDim.x) {
        const size_t slot = w / S, k = slot / (n_nodes * jl), j = slot % jl;
        if (k * jl + j >= spn) send[w] = one[w % S];
    }
}

// per (key, gh): real (non-trivial-zero) ciphertexts folded into the slot
__global__ void k_hist_real(const uint32_t *count, const uint32_t *ones, size_t nkeys, uint32_t *real) {
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < nkeys; k += (size_t)gridDim.x * blockDim.x) {
        const uint32_t c = count[k];
        real[2 * k] = c - (ones ? ones[2 * k] : 0u);
        real[2 * k + 1] = c - (ones ? ones[2 * k + 1] : 0u);
    }
}

// the reference counter over the whole group: Σ_slots max(Σ_shards real − 1, 0)
__global__ void k_adds_multi(PeerSet real, size_t n, unsigned long long *adds) {
    unsigned long long local = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long t = 0;
        for (uint32_t p = 0; p < real.n; ++p) t += real.p[p][i];
        local += t > 0 ? t - 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(adds, local);
}

} // namespace dev
} // namespace sfxb
