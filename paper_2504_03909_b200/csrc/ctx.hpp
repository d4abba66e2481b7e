// Host-side key context shared by the translation units of libsfxb_cuda.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "bignum_host.hpp"

struct sfxb_ctx;

namespace sfxb {

// Device copy of a Montgomery modulus: 4·S words [m | R mod m | R² | R³].
struct DevMod {
    uint32_t *w = nullptr;
    uint32_t np = 0;
    int S = 0;
};

// Size class: s = limbs of a prime; mod-p² and mod-n values use 2s limbs,
// ciphertexts (mod n²) 4s limbs.  s ∈ {4 (n ≤ 256 bits, tests), 8 (512),
// 16 (1024), 32 (2048), 48 (3072)}.
struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
};

struct CtxState {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sms = 148;
    int s = 0;          // size class
    uint32_t nw = 0;    // exact limbs of n as given
    bool has_priv = false;
    uint64_t key_id = 0;
    uint64_t launches = 0;
    std::string err;

    host::Big n, p, q, n2;
    DevMod mod_n2, mod_n, mod_pq[2], mod_pq2[2];
    // device constants (each padded to its modulus size)
    uint32_t *d_n = nullptr;          // n, 2s limbs
    uint32_t *d_n4 = nullptr;         // n, 4s limbs
    uint32_t *d_n2w = nullptr;        // n², 4s limbs
    uint32_t *d_nR_n2 = nullptr;      // n·R mod n²            (4s)
    uint32_t *d_q2R_n2 = nullptr;     // q²·R mod n²           (4s)
    uint32_t *d_qq_inv_m = nullptr;   // (q²)^-1·R mod p²      (2s)
    uint32_t *d_pinv[2] = {nullptr, nullptr};  // p^-1 mod 2^(32s), q^-1 mod 2^(32s)   (s)
    uint32_t *d_hR[2] = {nullptr, nullptr};    // h_p·R mod p, h_q·R mod q            (s)
    uint32_t *d_qinvR_p = nullptr;    // q^-1·R mod p          (s)
    uint32_t *d_qR_n = nullptr;       // q·R mod n             (2s)
    // exponent window digits (device) and their counts
    uint8_t *d_dig_n = nullptr;
    int nd_n = 0;
    uint8_t *d_dig_e1[2] = {nullptr, nullptr}; // q mod (p−1), p mod (q−1)
    int nd_e1[2] = {0, 0};
    uint8_t *d_dig_pq[2] = {nullptr, nullptr}; // p, q
    int nd_pq[2] = {0, 0};
    uint8_t *d_dig_m1[2] = {nullptr, nullptr}; // p−1, q−1
    int nd_m1[2] = {0, 0};
    // sliding-window programs (host::sliding_ops) for the digit exponentiations
    uint8_t *d_ops_pq[2] = {nullptr, nullptr}, *d_ops_m1[2] = {nullptr, nullptr}, *d_ops_e1[2] = {nullptr, nullptr};
    int nops_pq[2] = {0, 0}, nops_m1[2] = {0, 0}, nops_e1[2] = {0, 0};

    // optional per-kernel-family CUDA-event timing (bench roofline):
    // family 0 = K2 segmented product, 1 = K1 encrypt exps, 2 = K3 decrypt exp
    bool profile = false;
    struct Prof {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
        uint64_t launches = 0;
        uint64_t modmuls = 0; // Montgomery multiplications the launches executed
        double ms_done = 0;
    } prof[4];

    // sibling-subtraction parent cache: the last tree-mode call's histograms
    // (Montgomery form, node-major), double-buffered
    Buf tree_buf[2];
    int tree_cur = 0;
    bool tree_valid = false;
    const void *tree_gh = nullptr;
    uint32_t tree_J = 0, tree_K = 0, tree_N = 0;
    uint64_t tree_derived_nodes = 0; // nodes obtained by sibling subtraction so far
    std::unique_ptr<host::MontHost> mh_n2;

    // decrypt-side sibling reuse: previous level per histogram stream (tag)
    struct DecCache {
        Buf cts[2], plain[2]; // [cur] = previous level, [cur ^ 1] = this call
        int cur = 0;
        uint32_t n_nodes = 0, spn = 0; // spn: slots of this context's slice per node
        uint32_t spn_total = 0, j0 = 0; // the caller's slots per node and the slice start
        bool valid = false;
    };
    std::map<uint64_t, DecCache> dec_cache;
    uint64_t dec_derived = 0;         // slots decrypted by verified sibling reuse
    // per-item 32×32 products of the CRT exponentiations (profiling units of
    // kernel families 1 and 2)
    uint64_t prod_dec = 0, prod_enc = 0;
    // mod-p² exponentiations on base-p digits (padic.cuh): both primes fill
    // their size class (p > 2^(32s−1)); otherwise the CIOS mod-p² kernels
    bool p2_digits = false;
    uint32_t *d_cdec[2] = {nullptr, nullptr}; // h_p·R⁻¹ mod p, h_q·R⁻¹ mod q   (s)
    uint32_t *d_negR[2] = {nullptr, nullptr}; // p − R mod p, q − R mod q          (s)
    uint32_t *d_one_p2[2] = {nullptr, nullptr}; // digits of 1̃ mod p², q²: [R mod p | R mod p]  (2s)
    // passive-party K2 on base-n digits (padic.cuh): n fills its 2s limbs
    bool n_digits = false;
    uint32_t *d_negR_n = nullptr; // n − R mod n, R = 2^(64s)   (2s)
    uint32_t *d_one_nd = nullptr; // digits of 1̃ [R mod n | R mod n]  (4s)
    uint32_t *d_r4_nd = nullptr;  // digits of R⁴ mod n² (k_gh_nd_direct)  (4s)

    // scratch (grown on demand, freed with the context)
    Buf scratch_table, tmp[4], host_pinned[2], io[6]; // io: host-API staging (grow-only)
    std::vector<void *> owned; // device allocations of constants
    void *hist = nullptr;      // K2 work buffers (HistBufs, sfxb_cuda.cu), grown on demand

    // device group (sfxb_ctx_create_multi): shard contexts, shards[0] == this;
    // empty for a single-device context
    std::vector<::sfxb_ctx *> shards;
    cudaEvent_t ev_part = nullptr; // this shard's partial histograms are complete
    cudaStream_t copy_stream = nullptr; // pipelined gh upload (sfxb_gh_upload)
    cudaEvent_t ev_chunk[8] = {};
    uint32_t tree_j0 = 0, tree_jl = 0, tree_G = 0; // group tree cache: this shard's slot slice
    // one spare gh allocation (limbs + flags), recycled by the next upload
    void *spare_gh = nullptr, *spare_flags = nullptr;
    size_t spare_gh_bytes = 0, spare_flags_bytes = 0;
};

constexpr int kWindow = 5; // fixed exponent window for the 1024-bit CRT exponents
constexpr int kWindowN = 5;

} // namespace sfxb
