// Paillier kernels (sm_100a).  Every kernel runs 128-thread blocks of
// NI = 128/TPI instances and strides over its work items; per-instance
// exponentiation tables live in a global scratch slice (blockIdx·NI + inst).
//
//   K1 encrypt   k_enc_step1 / k_enc_step2 / k_enc_combine   (CRT, he.cpp:87-99)
//                k_pow_n2 + k_enc_combine(crt=false)          (public-key only)
//   K2 histogram hist.cu
//   K3 decrypt   k_dec_scan / k_dec_step / k_dec_combine      (CRT, he.cpp:105-115)
//   K0 modmul    k_mulmod                                     (he.cpp:117-121)
#pragma once
#include "modexp.cuh"

namespace sfxb {
namespace dev {

constexpr int kBlock = 128;

struct ModArg {
    const uint32_t *w;
    uint32_t np;
    __device__ __forceinline__ ModRef ref() const { return ModRef{w, np}; }
};

// Plain word i of the instance's staging area: the low/high half of pair
// i/2 in the swizzled b_slot layout (so staging never aliases another
// instance's slots, see mont.cuh).
template <int TPI>
__device__ __forceinline__ uint32_t *staged_ptr(const Stage &st, int i) {
    constexpr int NIc = kBlock / TPI;
    return reinterpret_cast<uint32_t *>(st.sB + b_slot<NIc>(i >> 1, st.inst)) + (i & 1);
}

// Redistribute a value between two lane layouts of the same TPI through the
// instance's staging buffer: `src` has Ssrc limbs (Ssrc/TPI per lane), the
// result has Sdst limbs (zero-extended or truncated).
template <int Ssrc, int Sdst, int TPI>
__device__ __forceinline__ void relayout(uint32_t (&dst)[Sdst / TPI], const uint32_t (&src)[Ssrc / TPI],
                                         const Stage &st) {
    constexpr int Ls = Ssrc / TPI, Ld = Sdst / TPI;
    const int t = inst_lane<TPI>();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < Ls; ++k) {
        const int i = t * Ls + k;
        if (i < Sdst) *staged_ptr<TPI>(st, i) = src[k];
    }
    if constexpr (Sdst > Ssrc) {
#pragma unroll
        for (int k = 0; k < Ld; ++k) {
            const int i = t * Ld + k;
            if (i >= Ssrc) *staged_ptr<TPI>(st, i) = 0u;
        }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < Ld; ++k) dst[k] = *staged_ptr<TPI>(st, t * Ld + k);
    __syncwarp();
}

// word i of the value last written by relayout (all lanes may read)
template <int TPI>
__device__ __forceinline__ uint32_t staged_word(const Stage &st, int i) {
    return *staged_ptr<TPI>(st, i);
}

// Grid-stride loop in which every instance of a block runs the same number
// of iterations (the shuffles/ballots use full-warp masks).  Past the end,
// an instance recomputes the last item with `active == false` (no stores).
#define SFXB_UNIFORM_LOOP(var, active, total)                                                      \
    for (size_t sfxb_base_ = (size_t)blockIdx.x * (kBlock / TPI), sfxb_tot_ = (total);            \
         sfxb_base_ < sfxb_tot_; sfxb_base_ += (size_t)gridDim.x * (kBlock / TPI))                 \
        for (bool sfxb_once_ = true; sfxb_once_; sfxb_once_ = false)                               \
            for (const size_t var = (sfxb_base_ + threadIdx.x / TPI < sfxb_tot_)                   \
                                        ? sfxb_base_ + threadIdx.x / TPI                           \
                                        : sfxb_tot_ - 1;                                           \
                 sfxb_once_; sfxb_once_ = false)                                                   \
                for (const bool active = sfxb_base_ + threadIdx.x / TPI < sfxb_tot_; sfxb_once_;   \
                     sfxb_once_ = false)

template <int TPI>
__device__ __forceinline__ Stage make_stage(uint2 *sB) {
    return Stage{sB, kBlock / TPI, (int)(threadIdx.x / TPI)};
}

// ------------------------------------------------------------------ K0

// out = a·b mod M  (a, b < M).  MontMul(MontMul(a, b), R²).
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_mulmod(ModArg M, const uint32_t *a, const uint32_t *b,
                                                   uint32_t *out, size_t count) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L], x[L], y[L], c[L];
    load_const<S, TPI>(N, mr, kMod);
    load_const<S, TPI>(c, mr, kR2);
    SFXB_UNIFORM_LOOP(e, active, count) {
        load_lane<S, TPI>(x, a + e * S);
        load_lane<S, TPI>(y, b + e * S);
        mmul<S, TPI>(x, x, y, st, N, M.np);
        mmul<S, TPI>(x, c, x, st, N, M.np);
        if (active) store_lane<S, TPI>(out + e * S, x);
    }
}

// ------------------------------------------------------------------ K1 encrypt (CRT)

struct EncArgs {
    const uint32_t *r;      // count × 2s
    const int64_t *qfix;    // count (fixed-point plaintexts), or null when mw is set
    const uint32_t *mw;     // count × 2s plaintext words m < n (packed vectors), or null
    size_t count;
    ModArg mod_pq[2];       // S = s
    ModArg mod_pq2[2];      // S = 2s
    ModArg mod_n2;          // S = 4s
    const uint8_t *dig_e1[2];
    int nd_e1[2];
    const uint8_t *ops_e1[2]; // sliding-window programs of e1 (preferred when set)
    int nops_e1[2];
    const uint8_t *dig_pq[2];
    int nd_pq[2];
    const uint8_t *dig_n;
    int nd_n;
    const uint32_t *n4;      // n zero-extended to 4s limbs
    const uint32_t *nR_n2;   // 4s
    const uint32_t *q2R_n2;  // 4s
    const uint32_t *qq_inv_m; // 2s
    uint32_t *x;            // count × 2 × 2s   (step1 -> step2)
    uint32_t *y;            // count × 2 × 2s   (step2 -> combine) or count × 4s (no CRT)
    uint32_t *out;          // count × 4s
    uint8_t *flags;         // count, may be null
    uint32_t *status;       // device word: bit0 = some r not coprime
    uint32_t *scratch;      // tables
};

// x = (r mod prime)^(e1) mod prime, e1 = other prime mod (prime − 1); flags p | r.
template <int S, int TPI, int W>
__global__ void __launch_bounds__(kBlock) k_enc_step1(EncArgs a) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    // one prime per block row (blockIdx.y): the exponent digits, hence the
    // control flow of mont_pow, must be uniform across a warp
    const int which = (int)blockIdx.y;
    const size_t gi = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * NI + st.inst;
    uint32_t *table = a.scratch + gi * ((size_t)S << W);
    SFXB_UNIFORM_LOOP(e, active, a.count) {
        const ModRef M = a.mod_pq[which].ref();
        uint32_t N[L], lo[L], hi[L], x[L];
        load_const<S, TPI>(N, M, kMod);
        load_lane<S, TPI>(lo, a.r + e * 2 * S);
        load_lane<S, TPI>(hi, a.r + e * 2 * S + S);
        to_mont_wide<S, TPI>(x, lo, hi, M, st, N);
        if (eq_small<L, TPI>(x, 0u) && active && inst_lane<TPI>() == 0) {
            atomicOr(a.status, 1u);
            if (a.flags) a.flags[e] = 1;
        }
        if (a.ops_e1[which]) mont_pow_ops<S, TPI>(x, a.ops_e1[which], a.nops_e1[which], W, table, M, st, N);
        else mont_pow<S, TPI>(x, a.dig_e1[which], a.nd_e1[which], W, table, M, st, N);
        from_mont<S, TPI>(x, x, st, N, M.np);
        if (active) {
            uint32_t *dst = a.x + (e * 2 + which) * 2 * S;
            store_lane<S, TPI>(dst, x);
            uint32_t z[L];
#pragma unroll
            for (int k = 0; k < L; ++k) z[k] = 0;
            store_lane<S, TPI>(dst + S, z);
        }
    }
}

// y = x^prime mod prime²   (= r^n mod prime², K1)
template <int S, int TPI, int W>
__global__ void __launch_bounds__(kBlock) k_enc_step2(EncArgs a) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const int which = (int)blockIdx.y; // see k_enc_step1
    const size_t gi = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * NI + st.inst;
    uint32_t *table = a.scratch + gi * ((size_t)S << W);
    SFXB_UNIFORM_LOOP(e, active, a.count) {
        const ModRef M = a.mod_pq2[which].ref();
        uint32_t N[L], x[L];
        load_const<S, TPI>(N, M, kMod);
        load_lane<S, TPI>(x, a.x + (e * 2 + which) * S);
        to_mont<S, TPI>(x, x, M, st, N);
        mont_pow<S, TPI>(x, a.dig_pq[which], a.nd_pq[which], W, table, M, st, N);
        from_mont<S, TPI>(x, x, st, N, M.np);
        if (active) store_lane<S, TPI>(a.y + (e * 2 + which) * S, x);
    }
}

// Public-key-only path: y = r^n mod n² directly (S = 4s).
template <int S, int TPI, int W>
__global__ void __launch_bounds__(kBlock) k_pow_n2(EncArgs a) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const size_t gi = (size_t)blockIdx.x * NI + st.inst;
    uint32_t *table = a.scratch + gi * ((size_t)S << W);
    const ModRef M = a.mod_n2.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, M, kMod);
    SFXB_UNIFORM_LOOP(e, active, a.count) {
        uint32_t x[L], r2s[S / 2 / TPI];
        load_lane<S / 2, TPI>(r2s, a.r + e * (S / 2));
        relayout<S / 2, S, TPI>(x, r2s, st);
        to_mont<S, TPI>(x, x, M, st, N);
        mont_pow<S, TPI>(x, a.dig_n, a.nd_n, W, table, M, st, N);
        from_mont<S, TPI>(x, x, st, N, M.np);
        if (active) store_lane<S, TPI>(a.y + e * S, x);
    }
}

// c = (1 + m·n)·Y mod n², Y = r^n mod n² (CRT-combined from y_p, y_q when crt).
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_enc_combine(EncArgs a, int crt) {
    constexpr int S2 = 2 * s, S4 = 4 * s, L2 = S2 / TPI, L4 = S4 / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S4 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M4 = a.mod_n2.ref();
    uint32_t N4[L4];
    load_const<S4, TPI>(N4, M4, kMod);
    SFXB_UNIFORM_LOOP(e, active, a.count) {
        uint32_t Y[L4], C4[L4], t4[L4];
        if (crt) {
            const ModRef M2 = a.mod_pq2[0].ref();
            uint32_t N2[L2], yp[L2], yq[L2], d[L2], C2[L2], h[L2];
            load_const<S2, TPI>(N2, M2, kMod);
            load_lane<S2, TPI>(yp, a.y + (e * 2 + 0) * S2);
            load_lane<S2, TPI>(yq, a.y + (e * 2 + 1) * S2);
            reduce_once<S2, TPI>(d, yq, N2); // y_q mod p² (y_q < q² < 2p²)
            mod_sub<S2, TPI>(d, yp, d, N2);
            load_lane<S2, TPI>(C2, a.qq_inv_m);
            mmul<S2, TPI>(h, C2, d, st, N2, M2.np); // h = (y_p − y_q)·q⁻² mod p²
            uint32_t h4[L4], yq4[L4];
            relayout<S2, S4, TPI>(h4, h, st);
            relayout<S2, S4, TPI>(yq4, yq, st);
            load_lane<S4, TPI>(C4, a.q2R_n2);
            mmul<S4, TPI>(t4, C4, h4, st, N4, M4.np); // q²·h (< n², exact)
            mod_add<S4, TPI>(Y, t4, yq4, N4);         // Y = y_q + q²·h = r^n mod n²
        } else {
            load_lane<S4, TPI>(Y, a.y + e * S4);
        }
        uint32_t m[L4];
        if (a.mw) {
            // plaintext given as words (packed vectors, he.cpp:220-225)
            uint32_t m2[L2];
            load_lane<S2, TPI>(m2, a.mw + e * S2);
            relayout<S2, S4, TPI>(m, m2, st);
        } else {
            // m = q mod n: q >= 0 -> q ; q < 0 -> n − |q|
            const int64_t qv = a.qfix[e];
            const uint64_t mag = qv < 0 ? (uint64_t)(-(qv + 1)) + 1u : (uint64_t)qv;
            uint32_t mq[L4];
            set_small<L4, TPI>(mq, 0u);
            if (inst_lane<TPI>() == 0) {
                mq[0] = (uint32_t)mag;
                mq[1] = (uint32_t)(mag >> 32);
            }
            uint32_t n4[L4];
            load_lane<S4, TPI>(n4, a.n4);
            sub_full<S4, TPI>(m, n4, mq); // warp-uniform; selected below
#pragma unroll
            for (int k = 0; k < L4; ++k) m[k] = qv < 0 ? m[k] : mq[k];
        }
        load_lane<S4, TPI>(C4, a.nR_n2);
        mmul<S4, TPI>(t4, C4, m, st, N4, M4.np); // m·n (< n², exact)
        uint32_t one[L4];
        set_small<L4, TPI>(one, 1u);
        mod_add<S4, TPI>(t4, t4, one, N4);        // 1 + m·n
        mmul<S4, TPI>(t4, t4, Y, st, N4, M4.np);  // (1+mn)·Y·R⁻¹
        load_const<S4, TPI>(C4, M4, kR2);
        mmul<S4, TPI>(t4, C4, t4, st, N4, M4.np); // ·R² ·R⁻¹
        if (active) store_lane<S4, TPI>(a.out + e * S4, t4);
    }
}

// ------------------------------------------------------------------ gradients on the device
//
// compute_gradients (gbdt.cpp:69-80): g = p − y, h = p·(1 − p); quantize_gradients
// (:82-87) = fixed_round (fixed_point.hpp:22-24) on the 2^-scale grid; then
// encode_fixed's checks (he.cpp:125-136) and q = llround(ldexp(x, scale)) —
// the plaintexts sfxb_encrypt_dev takes, G and H interleaved.  Every step is
// one correctly rounded IEEE operation (explicit _rn intrinsics: no FMA
// contraction), ldexp and llround are exact, so q is bit-identical to the
// reference's host arithmetic.  The sigmoid that turns margins into p stays
// with the caller (the reference's federation loop, federation.cpp:460-461):
// libm exp is not reproducible bit for bit on the device.
// status[0]: lowest failing index (count when none); status[1]: failure kind
// (1 non-finite, 2 off the grid, 3 |q| >= n/2).
struct GradArgs {
    const double *prob;
    const uint8_t *label;
    size_t n;
    int scale;
    double lim;        // 2^(62 − scale)
    uint64_t n64;      // n when n < 2^64 (toy keys), else 0 (no bound reachable)
    int64_t *q;        // 2n
    double *gh;        // optional 2n quantized (g, h)
    unsigned long long *status;
};

__device__ __forceinline__ int encode_one(const GradArgs &a, double x, int64_t &q) {
    if (!isfinite(x)) return 1;
    if (fabs(x) >= a.lim) return 2;
    q = llround(ldexp(x, a.scale));
    const uint64_t mag = q < 0 ? (uint64_t)(-(q + 1)) + 1u : (uint64_t)q;
    if (a.n64 && 2 * mag >= a.n64) return 3;
    return 0;
}

// fixed_round (fixed_point.hpp:22-24) = ldexp((double)llround(ldexp(x, s)), −s),
// with the host's llround for values outside int64 (NaN, |x|·2^s ≥ 2^63: the
// x86-64 conversion yields INT64_MIN) so even garbage inputs fail the same way
__device__ __forceinline__ double fixed_round_dev(double x, int s) {
    const double y = ldexp(x, s);
    const long long q = (isfinite(y) && fabs(y) < 9.223372036854775808e18) ? llround(y) : (long long)(1ull << 63);
    return ldexp((double)q, -s);
}

__global__ void k_gradients(GradArgs a) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n; i += (size_t)gridDim.x * blockDim.x) {
        const double p = a.prob[i];
        const double g = __dsub_rn(p, (double)a.label[i]);
        const double h = __dmul_rn(p, __dsub_rn(1.0, p));
        const double gq = fixed_round_dev(g, a.scale), hq = fixed_round_dev(h, a.scale);
        if (a.gh) {
            a.gh[2 * i] = gq;
            a.gh[2 * i + 1] = hq;
        }
        int64_t q0 = 0, q1 = 0;
        const int e0 = encode_one(a, gq, q0), e1 = e0 ? 0 : encode_one(a, hq, q1);
        if (e0 || e1) {
            const unsigned long long idx = e0 ? 2 * i : 2 * i + 1;
            if (atomicMin(&a.status[0], idx) > idx) a.status[1] = (unsigned long long)(e0 ? e0 : e1);
        }
        a.q[2 * i] = q0;
        a.q[2 * i + 1] = q1;
    }
}

// ------------------------------------------------------------------ K3 decrypt (CRT)

// decode_fixed (he.cpp:138-143) before the final ldexp: v = m − n if 2m > n,
// converted like mpz_get_d (truncation toward zero).  word(k) = limb k of m.
template <typename W>
__device__ __forceinline__ double decode_words(int Sn, W word, const uint32_t *nw) {
    // 2m > n  <=>  m > n >> 1 (n odd)
    int cmpv = 0;
    for (int k = Sn - 1; k >= 0 && cmpv == 0; --k) {
        const uint32_t hn_k = (nw[k] >> 1) | (k + 1 < Sn ? (nw[k + 1] << 31) : 0u);
        const uint32_t mk = word(k);
        cmpv = mk > hn_k ? 1 : (mk < hn_k ? -1 : 0);
    }
    const bool neg = cmpv > 0;
    // |v| = neg ? n − m : m, scanned from limb 0 keeping the highest
    // nonzero limb and the two limbs below it.
    uint32_t w_top = 0, w_1 = 0, w_2 = 0, prev1 = 0, prev2 = 0, bw = 0;
    int topk = -1;
    for (int k = 0; k < Sn; ++k) {
        const uint32_t mk = word(k);
        uint32_t vk = mk;
        if (neg) {
            const uint64_t diff = (uint64_t)nw[k] - mk - bw;
            vk = (uint32_t)diff;
            bw = (uint32_t)(diff >> 63);
        }
        if (vk != 0) {
            topk = k;
            w_top = vk;
            w_1 = prev1;
            w_2 = prev2;
        }
        prev2 = prev1;
        prev1 = vk;
    }
    double val = 0.0;
    if (topk >= 0) {
        const int lz = __clz(w_top);
        const int bits = topk * 32 + (32 - lz);
        if (bits <= 64) {
            const unsigned long long w64 =
                topk == 0 ? (unsigned long long)w_top : ((unsigned long long)w_top << 32) | w_1;
            val = __ull2double_rz(w64); // truncation == mpz_get_d
        } else {
            unsigned long long w64 = ((unsigned long long)w_top << 32) | w_1;
            if (lz) w64 = (w64 << lz) | (w_2 >> (32 - lz));
            val = ldexp(__ull2double_rz(w64), bits - 64);
        }
        if (neg) val = -val;
    }
    return val;
}

struct DecArgs {
    const uint32_t *cts;     // count × 4s
    size_t count;
    uint32_t *idx;           // compacted indices of non-trivial slots
    uint32_t *n_idx;         // device counter
    ModArg mod_pq[2];        // s
    ModArg mod_pq2[2];       // 2s
    ModArg mod_n;            // 2s
    const uint8_t *dig_m1[2];
    int nd_m1[2];
    const uint32_t *pinv[2]; // s
    const uint32_t *hR[2];   // s
    const uint32_t *qinvR_p; // s
    const uint32_t *qR_n;    // 2s
    const uint32_t *n2w;     // n² limbs, 4s
    const uint32_t *nw;      // n limbs, 2s
    uint32_t *mpq;           // count × 2 × s
    double *values;          // count
    uint32_t *plain;         // count × 2s (may be null)
    uint32_t *status;        // bit1 = out of range, bit2 = not coprime
    uint32_t scale;
    uint32_t *scratch;
    const uint8_t *skip;     // optional: 1 = plaintext derived elsewhere (sibling reuse)
    uint32_t *n_skipped;     // non-trivial slots skipped (still counted as decryptions)
};

// Flag trivial slots (== 1 -> 0.0, uncounted), range-check the rest and
// compact their indices.  One thread per slot.
template <int S4>
__global__ void k_dec_scan(DecArgs a) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.count;
         e += (size_t)gridDim.x * blockDim.x) {
        const uint32_t *c = a.cts + e * S4;
        bool one = c[0] == 1u, zero = c[0] == 0u;
        for (int k = 1; k < S4; ++k) {
            one &= c[k] == 0u;
            zero &= c[k] == 0u;
        }
        if (one) {
            a.values[e] = 0.0;
            if (a.plain)
                for (int k = 0; k < S4 / 2; ++k) a.plain[e * (S4 / 2) + k] = 0u;
            continue;
        }
        // c >= n² ?
        bool ge = true;
        for (int k = S4 - 1; k >= 0; --k) {
            if (c[k] != a.n2w[k]) {
                ge = c[k] > a.n2w[k];
                break;
            }
        }
        if (zero || ge) atomicOr(a.status, 2u);
        if (a.skip && a.skip[e]) {
            atomicAdd(a.n_skipped, 1u);
            continue;
        }
        const uint32_t slot = atomicAdd(a.n_idx, 1u);
        a.idx[slot] = (uint32_t)e;
    }
}

// m_prime = L_prime(c^(prime−1) mod prime²)·h_prime mod prime
template <int s, int TPI, int W>
__global__ void __launch_bounds__(kBlock) k_dec_step(DecArgs a, uint32_t n_items) {
    constexpr int S2 = 2 * s, L2 = S2 / TPI, L1 = s / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S2 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const int which = (int)blockIdx.y; // see k_enc_step1
    const size_t gi = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * NI + st.inst;
    uint32_t *table = a.scratch + gi * ((size_t)S2 << W);
    SFXB_UNIFORM_LOOP(item, active, (size_t)n_items) {
        const uint32_t e = a.idx[item];
        const ModRef M2 = a.mod_pq2[which].ref();
        uint32_t N2[L2], lo[L2], hi[L2], u[L2];
        load_const<S2, TPI>(N2, M2, kMod);
        load_lane<S2, TPI>(lo, a.cts + (size_t)e * 2 * S2);
        load_lane<S2, TPI>(hi, a.cts + (size_t)e * 2 * S2 + S2);
        to_mont_wide<S2, TPI>(u, lo, hi, M2, st, N2);
        mont_pow<S2, TPI>(u, a.dig_m1[which], a.nd_m1[which], W, table, M2, st, N2);
        from_mont<S2, TPI>(u, u, st, N2, M2.np);
        if (eq_small<L2, TPI>(u, 0u) && active && inst_lane<TPI>() == 0) atomicOr(a.status, 4u);
        // ℓ = (u − 1)/prime = ((u − 1) mod 2^(32s))·prime⁻¹ mod 2^(32s); every
        // lane computes it redundantly from the staged words (s²/2 products).
        uint32_t tmp[L2];
        relayout<S2, S2, TPI>(tmp, u, st);
        const uint32_t *pinv = a.pinv[which];
        uint32_t lw[s];
#pragma unroll
        for (int k = 0; k < s; ++k) lw[k] = 0u;
        uint32_t borrow = 1u;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const uint32_t ui = staged_word<TPI>(st, i);
            const uint32_t xi = ui - borrow;
            borrow = ui < borrow ? 1u : 0u;
            uint32_t c = 0;
#pragma unroll
            for (int j = 0; j < s - i; ++j) {
                const uint64_t t = (uint64_t)xi * __ldg(pinv + j) + lw[i + j] + c;
                lw[i + j] = (uint32_t)t;
                c = (uint32_t)(t >> 32);
            }
        }
        uint32_t ell[L1];
        const int t = inst_lane<TPI>();
#pragma unroll
        for (int k = 0; k < L1; ++k) {
            uint32_t v = 0;
#pragma unroll
            for (int tt = 0; tt < TPI; ++tt) v = (t == tt) ? lw[tt * L1 + k] : v;
            ell[k] = v;
        }
        const ModRef M1 = a.mod_pq[which].ref();
        uint32_t N1[L1], C1[L1], mp[L1];
        load_const<s, TPI>(N1, M1, kMod);
        load_lane<s, TPI>(C1, a.hR[which]);
        mmul<s, TPI>(mp, C1, ell, st, N1, M1.np); // ℓ·h_prime mod prime
        if (active) store_lane<s, TPI>(a.mpq + ((size_t)e * 2 + which) * s, mp);
    }
}

// m = m_q + q·((m_p − m_q)·q⁻¹ mod p); decode_fixed with mpz_get_d truncation.
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_dec_combine(DecArgs a, uint32_t n_items) {
    constexpr int Sn = 2 * s, L1 = s / TPI, Ln = Sn / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[Sn / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M1 = a.mod_pq[0].ref(), Mn = a.mod_n.ref();
    uint32_t N1[L1], Nn[Ln];
    load_const<s, TPI>(N1, M1, kMod);
    load_const<Sn, TPI>(Nn, Mn, kMod);
    SFXB_UNIFORM_LOOP(item, active, (size_t)n_items) {
        const uint32_t e = a.idx[item];
        uint32_t mp[L1], mq[L1], d[L1], C1[L1], h[L1];
        load_lane<s, TPI>(mp, a.mpq + ((size_t)e * 2 + 0) * s);
        load_lane<s, TPI>(mq, a.mpq + ((size_t)e * 2 + 1) * s);
        reduce_once<s, TPI>(d, mq, N1); // m_q mod p (m_q < q < 2p)
        mod_sub<s, TPI>(d, mp, d, N1);
        load_lane<s, TPI>(C1, a.qinvR_p);
        mmul<s, TPI>(h, C1, d, st, N1, M1.np);
        uint32_t hn[Ln], mqn[Ln], Cn[Ln], m[Ln];
        relayout<s, Sn, TPI>(hn, h, st);
        relayout<s, Sn, TPI>(mqn, mq, st);
        load_lane<Sn, TPI>(Cn, a.qR_n);
        mmul<Sn, TPI>(m, Cn, hn, st, Nn, Mn.np); // q·h (< n, exact)
        mod_add<Sn, TPI>(m, m, mqn, Nn);
        if (a.plain && active) store_lane<Sn, TPI>(a.plain + (size_t)e * Sn, m);
        // decode_fixed (he.cpp:138-143): v = m − n if 2m > n; mpz_get_d truncates.
        uint32_t tmp[Ln];
        relayout<Sn, Sn, TPI>(tmp, m, st);
        const double val = decode_words(Sn, [&](int k) { return staged_word<TPI>(st, k); }, a.nw);
        if (active && inst_lane<TPI>() == 0) a.values[e] = ldexp(val, -(int)a.scale);
    }
}

// ------------------------------------------------------------------ K3 sibling reuse

// flag[j] = 1 when ct_a·ct_b ≡ ct_parent (mod n²) for derived slot j; then
// m_b = m_parent − m_a (mod n) by the homomorphism and b need not be decrypted.
struct SibArgs {
    const uint32_t *cts;      // this call, node-major, n_nodes × spn × 4s
    const uint32_t *prev_cts; // previous call (same tag)
    const uint32_t *pairs;    // per derived node: (b, a, parent)
    size_t n_pairs, spn;
    uint8_t *skip;            // per slot of this call
};

template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_sib_verify(ModArg M, SibArgs a) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef mr = M.ref();
    uint32_t N[L], R2[L];
    load_const<S, TPI>(N, mr, kMod);
    load_const<S, TPI>(R2, mr, kR2);
    SFXB_UNIFORM_LOOP(j, active, a.n_pairs * a.spn) {
        const uint32_t *pr = a.pairs + 3 * (j / a.spn);
        const size_t k = j % a.spn;
        uint32_t x[L], y[L], z[L];
        load_lane<S, TPI>(x, a.cts + ((size_t)pr[1] * a.spn + k) * S);
        load_lane<S, TPI>(y, a.cts + ((size_t)pr[0] * a.spn + k) * S);
        load_lane<S, TPI>(z, a.prev_cts + ((size_t)pr[2] * a.spn + k) * S);
        // x·y mod n² = MontMul(MontMul(x, y), R²); x, y < n² (range-checked by the scan)
        mmul<S, TPI>(x, x, y, st, N, M.np);
        mmul<S, TPI>(x, R2, x, st, N, M.np);
        bool eq = true;
#pragma unroll
        for (int w = 0; w < L; ++w) eq &= x[w] == z[w];
        const bool all = inst_ballot<TPI>(!eq) == 0;
        if (active && inst_lane<TPI>() == 0) a.skip[(size_t)pr[0] * a.spn + k] = all ? 1 : 0;
    }
}

// m_b = (m_parent − m_a) mod n for the skipped slots, then decode_fixed.
template <int Sn>
__global__ void k_sib_derive(const uint32_t *pairs, size_t n_pairs, size_t spn, const uint8_t *skip,
                             const uint32_t *plain, const uint32_t *prev_plain, const uint32_t *nw,
                             uint32_t scale, uint32_t *plain_out, double *values) {
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_pairs * spn;
         j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t *pr = pairs + 3 * (j / spn);
        const size_t k = j % spn, eb = (size_t)pr[0] * spn + k;
        if (!skip[eb]) continue;
        const uint32_t *ma = plain + ((size_t)pr[1] * spn + k) * Sn;
        const uint32_t *mp = prev_plain + ((size_t)pr[2] * spn + k) * Sn;
        uint32_t m[Sn];
        uint32_t br = 0;
        for (int w = 0; w < Sn; ++w) {
            const uint64_t d = (uint64_t)mp[w] - ma[w] - br;
            m[w] = (uint32_t)d;
            br = (uint32_t)(d >> 63);
        }
        if (br) { // add n back
            uint32_t c = 0;
            for (int w = 0; w < Sn; ++w) {
                const uint64_t t = (uint64_t)m[w] + nw[w] + c;
                m[w] = (uint32_t)t;
                c = (uint32_t)(t >> 32);
            }
        }
        for (int w = 0; w < Sn; ++w) plain_out[eb * Sn + w] = m[w];
        values[eb] = ldexp(decode_words(Sn, [&](int w) { return m[w]; }, nw), -(int)scale);
    }
}

} // namespace dev
} // namespace sfxb
