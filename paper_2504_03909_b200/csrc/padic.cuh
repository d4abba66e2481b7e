// Exponentiation mod p² on base-p digits with Montgomery arithmetic mod p
// (K1 encrypt step 2 and K3 decrypt: x^p mod p², c^(p−1) mod p²).
//
// R = 2^(32s) (s = limbs of p, p > R/2).  An element X of Z/p² is carried by
// its Montgomery representative X̃ = X·R² mod p² (R² = the Montgomery radix
// of the s'=2s-limb modulus p²), written on base-p digits
//     X̃ ≡ A·R + B·p (mod p²),   A, B ∈ [0, p).
// The Montgomery product X̃1·X̃2·R⁻² mod p² is then
//     A1A2 + p·(A1B2 + A2B1)·R⁻¹            (the B1B2·p² term vanishes)
// and with one CIOS pass mod p on A1·A2, which yields t and the quotient
// digits m with A1A2 = (t + ge·p)·R − m·p (mont_mul_m),
//     A' = t,   B' = MM(A1, B2) + MM(A2, B1) − m + ge·R   (mod p),
// MM(x, y) = x·y·R⁻¹ mod p.  A multiplication costs 3 CIOS passes mod p
// (3·(2s²+s) 32×32 products) and a squaring 2 (B' = 2·MM(A, B) − m + ge·R),
// against 2(2s)²+2s products for one CIOS pass mod p² — 48% fewer products
// for a windowed exponentiation.  Results are canonical residues, so they are
// bit-identical to the mod-p² CIOS path (and to GMP).
//
// The identity 1̃ = R² mod p² has digits (R mod p, R mod p) when p > R/2.
#pragma once
#include "hist.cuh"

namespace sfxb {
namespace dev {

// Stage operand b of the next CIOS pass: from registers
template <int S, int TPI>
__device__ __forceinline__ void stage_regs(const Stage &st, const uint32_t (&v)[S / TPI]) {
    stage_b<S, TPI>(st, v);
}

// mont_sqr for the digit squarings at one lane per instance (
// -DSFXB_NO_SQR_P2 builds the two-CIOS-pass squaring instead)
#if !defined(SFXB_NO_SQR_P2) || defined(SFXB_SQR)
constexpr bool kSqrP2 = true;
#else
constexpr bool kSqrP2 = false;
#endif

// K2 job claiming: the block takes 4·NIW jobs at once from the global
// counter between two barriers, so the warps of a block start every job batch
// in step (they then run the same fully unrolled multiply body together:
// fewer instruction-fetch stalls) — K2 399.8 -> 396 ms/tree at the bench
// size, frac 0.883 -> 0.89 (profiles/r02_ab_blockjobs.jsonl).  Built with
// -DSFXB_K2_WARPJOBS, each warp claims its own NIW jobs instead.
#ifndef SFXB_K2_WARPJOBS
#define SFXB_K2_JOB_STATE __shared__ unsigned long long sfxb_jb_
#define SFXB_K2_CLAIM(base, NIW, total)                                                                      \
    __syncthreads();                                                                                         \
    if (threadIdx.x == 0) sfxb_jb_ = atomicAdd(next_job, (unsigned long long)(NIW) * (kBlock / 32));        \
    __syncthreads();                                                                                         \
    if (sfxb_jb_ >= (total)) break;                                                                          \
    base = sfxb_jb_ + (unsigned long long)(threadIdx.x >> 5) * (NIW)
#else
#define SFXB_K2_JOB_STATE (void)0
#define SFXB_K2_CLAIM(base, NIW, total)                                                                      \
    if ((threadIdx.x & 31) == 0) base = atomicAdd(next_job, (unsigned long long)(NIW));                     \
    base = __shfl_sync(0xffffffffu, base, 0);                                                                \
    if (base >= (total)) break
#endif

// One Montgomery product mod p² on digits: (A, B) <- (A, B) ⊛ (A2, B2),
// or the square when `square` (A2, B2 unused).  Two CIOS passes:
//   pass 0: square:   v = 2·MM(A, B)
//           multiply: v = MM2(A·B2 + A2·B)   (one two-product pass, mont_mul2)
//   pass 1: t, ge = MM(A, A | A2), v -= m on the fly (borrow bw);  A <- t
// then B <- v − m + ge·R (mod p): v − m + (ge − bw)·R with v − m (mod R)
// < R < 2p.  Rmod = R mod p, negR = p − R mod p (global).  Products: square
// 2·(2s²+s), multiply (3s²+s) + (2s²+s).  One inlined copy of each CIOS body.
template <int s, int TPI>
__device__ __forceinline__ void p2_mul(uint32_t (&A)[s / TPI], uint32_t (&B)[s / TPI], const uint32_t *g2,
                                       bool square, const Stage &st, uint2 *sD, const uint32_t (&N)[s / TPI],
                                       uint32_t np, const uint32_t *Rmod, const uint32_t *negR) {
    constexpr int L = s / TPI;
    uint32_t v[L], x[L];
    bool ge = false;
    uint32_t bw = 0;
    constexpr bool kSqr = kSqrP2 && TPI == 1;
    if constexpr (kSqr) {
        if (square) {
            // pass 0: v = 2·MM(A, B)
            stage_b<s, TPI>(st, B);
            {
                uint32_t r[L], b;
                mont_mul_sub<s, TPI>(r, v, A, st.sB, st.inst, N, np, false, b);
                mod_add<s, TPI>(v, r, r, N);
            }
            // pass 1 squares A' = min(A, p − A) (mont_sqr_sub): t is the same,
            // and its quotient m' satisfies ge·R − m ≡ ge'·R − m' + 2A (mod p)
            // [A² = A'² + 2pA − p²], so 2A joins v when A was flipped
            {
                uint32_t t[L];
                if (sqr_operand<s>(t, A, N)) {
                    mod_add<s, TPI>(v, v, A, N);
                    mod_add<s, TPI>(v, v, A, N);
                }
            }
            uint32_t r[L], b;
            bool fl;
            ge = mont_sqr_sub<s>(r, v, A, N, np, true, b, fl);
            bw = b;
#pragma unroll
            for (int k = 0; k < L; ++k) A[k] = r[k];
        }
    }
    const bool generic = !kSqr || !square;
#pragma unroll 1
    for (int c = 0; c < (generic ? 2 : 0); ++c) {
        if (c == 0 && !square) {
            {
                uint32_t tmp[L];
                load_lane<s, TPI>(tmp, g2 + s); // B2
                stage_b<s, TPI>(st, tmp);
            }
            stage_b<s, TPI>(Stage{sD, st.NI, st.inst}, B);
            load_lane<s, TPI>(x, g2); // A2 (register operand, and pass 1's scanned operand)
            mont_mul2<s, TPI>(v, A, x, st.sB, sD, st.inst, N, np);
        } else {
            {
                uint32_t tmp[L];
#pragma unroll
                for (int k = 0; k < L; ++k) tmp[k] = c == 0 ? B[k] : (square ? A[k] : x[k]);
                stage_b<s, TPI>(st, tmp);
            }
            uint32_t r[L], b;
            const bool g = mont_mul_sub<s, TPI>(r, v, A, st.sB, st.inst, N, np, c == 1, b);
            if (c == 0) {
                mod_add<s, TPI>(v, r, r, N);
            } else {
                ge = g;
                bw = b;
#pragma unroll
                for (int k = 0; k < L; ++k) A[k] = r[k];
            }
        }
    }
    reduce_once<s, TPI>(v, v, N);
    {
        // + (ge − bw)·R  (mod p)
        const int delta = (ge ? 1 : 0) - (int)bw;
        uint32_t tmp[L];
        load_lane<s, TPI>(tmp, delta > 0 ? Rmod : negR);
#pragma unroll
        for (int k = 0; k < L; ++k) tmp[k] = delta ? tmp[k] : 0u;
        mod_add<s, TPI>(v, v, tmp, N);
    }
#pragma unroll
    for (int k = 0; k < L; ++k) B[k] = v[k];
}

// (A, B) <- (A, B)^e, e as a sliding-window program (host::sliding_ops:
// n_ops byte pairs (squarings, odd digit)).  `table` = this instance's
// scratch of 2^(w−1) + 1 entries of 2s words ([A | B]): x^1, x^3, …,
// x^(2^w − 1), then x².
template <int s, int TPI>
__device__ __forceinline__ void p2_pow(uint32_t (&A)[s / TPI], uint32_t (&B)[s / TPI], const uint8_t *ops,
                                       int n_ops, int w, uint32_t *table, const Stage &st, uint2 *sD,
                                       const uint32_t (&N)[s / TPI], uint32_t np, const uint32_t *Rmod,
                                       const uint32_t *negR) {
    const int T = 1 << (w - 1);
    uint32_t *x2 = table + 2 * s * T;
    store_lane<s, TPI>(table, A);
    store_lane<s, TPI>(table + s, B);
    // op sequence: x² (one squaring), T−1 multiplies by x² for the odd
    // powers, then the program; ONE p2_mul call site (one inlined copy of the
    // CIOS body in the loop)
    int j = -1, oi = 0, sq = 0;
    bool started = false;
    for (;;) {
        bool square;
        const uint32_t *g2 = nullptr;
        if (j < T - 1) {
            square = j < 0;
            g2 = x2;
        } else {
            if (!started) {
                const int d0 = ops[1];
                load_lane<s, TPI>(A, table + 2 * s * (d0 >> 1));
                load_lane<s, TPI>(B, table + 2 * s * (d0 >> 1) + s);
                oi = 1;
                sq = n_ops > 1 ? ops[2] : 0;
                started = true;
            }
            if (sq > 0) {
                square = true;
            } else {
                if (oi >= n_ops) break;
                const int d = ops[2 * oi + 1];
                ++oi;
                sq = oi < n_ops ? ops[2 * oi] : 0;
                if (d == 0) continue;
                square = false;
                g2 = table + 2 * s * (d >> 1);
            }
        }
        p2_mul<s, TPI>(A, B, g2, square, st, sD, N, np, Rmod, negR);
        if (j < T - 1) {
            if (j < 0) {
                store_lane<s, TPI>(x2, A);
                store_lane<s, TPI>(x2 + s, B);
                load_lane<s, TPI>(A, table);
                load_lane<s, TPI>(B, table + s);
            } else {
                store_lane<s, TPI>(table + 2 * s * (j + 1), A);
                store_lane<s, TPI>(table + 2 * s * (j + 1) + s, B);
            }
            ++j;
        } else if (square) {
            --sq;
        }
    }
}

// 32×32 products of p2_pow for a sliding-window program at s limbs
// (p2_mul: square 2·(2s²+s), multiply (3s²+s) + (2s²+s)).
// `sqr`: squarings by mont_sqr (one lane per instance, kSqrP2): the pass
// v = 2·MM(A, B) plus s(s+1)/2 + s² + s for A², instead of 2·(2s²+s)
inline unsigned long long p2_pow_products(const uint8_t *ops, int n_ops, int w, int s, bool sqr) {
    const unsigned long long sq = sqr ? (2ull * s * s + s) + (s * (s + 1ull) / 2 + 1ull * s * s + s)
                                      : 2ull * (2ull * s * s + s),
                             mul = (3ull * s * s + s) + (2ull * s * s + s);
    unsigned long long prod = sq + mul * ((1ull << (w - 1)) - 1);
    for (int i = 1; i < n_ops; ++i) prod += sq * ops[2 * i] + (ops[2 * i + 1] ? mul : 0ull);
    return prod;
}

// Digits of X̃ (a canonical residue mod p², 2s limbs: hi·R + lo, hi < p):
// MM_m(1, lo) gives lo = (t + ge·p)·R − m·p, so A = hi + t (mod p, flag ge2)
// and B = (ge + ge2)·R − m (mod p).
template <int s, int TPI>
__device__ __forceinline__ void p2_split(uint32_t (&A)[s / TPI], uint32_t (&B)[s / TPI], const uint32_t (&lo)[s / TPI],
                                         const uint32_t (&hi)[s / TPI], const Stage &st,
                                         const uint32_t (&N)[s / TPI], uint32_t np, const uint32_t *Rmod) {
    constexpr int L = s / TPI;
    uint32_t q[L], t[L], one[L], x[L];
    set_small<L, TPI>(one, 1u);
    stage_b<s, TPI>(st, lo);
    const bool ge = mont_mul_m<s, TPI>(t, q, one, st.sB, st.inst, N, np);
    uint32_t Rsum[L];
    Rsum[0] = add_cc(hi[0], t[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) Rsum[k] = addc_cc(hi[k], t[k]);
    uint32_t cc = addc(0u, 0u), over;
    if constexpr (TPI == 1) {
        over = cc;
    } else {
        bool all_ones = true;
#pragma unroll
        for (int k = 0; k < L; ++k) all_ones &= (Rsum[k] == 0xffffffffu);
        const uint32_t G = inst_ballot<TPI>(cc != 0);
        const uint32_t P = inst_ballot<TPI>(all_ones);
        const uint64_t sum = (uint64_t)P + ((uint64_t)G << 1);
        const uint32_t cin = (uint32_t)(sum ^ P);
        if ((cin >> inst_lane<TPI>()) & 1u) {
            Rsum[0] = add_cc(Rsum[0], 1u);
#pragma unroll
            for (int k = 1; k < L; ++k) Rsum[k] = addc_cc(Rsum[k], 0u);
        }
        over = (uint32_t)(sum >> TPI) & 1u;
    }
    const bool ge2 = final_sub<L, TPI>(Rsum, over, N);
#pragma unroll
    for (int k = 0; k < L; ++k) A[k] = Rsum[k];
    const int nge = (ge ? 1 : 0) + (ge2 ? 1 : 0);
    uint32_t Rp[L], y[L];
    load_lane<s, TPI>(Rp, Rmod);
#pragma unroll
    for (int k = 0; k < L; ++k) {
        x[k] = nge ? Rp[k] : 0u;
        y[k] = nge == 2 ? Rp[k] : 0u;
    }
    mod_add<s, TPI>(x, x, y, N);
    reduce_once<s, TPI>(q, q, N);
    mod_sub<s, TPI>(B, x, q, N);
}

// ------------------------------------------------------------------ kernels

struct P2Args {
    ModArg mod_p[2];          // S = s
    const uint32_t *pinv[2];  // p⁻¹ mod 2^(32s)
    const uint32_t *cdec[2];  // h_p·R⁻¹ mod p (decrypt output)
    const uint32_t *negR[2];  // p − R mod p
    const uint8_t *ops[2];    // sliding-window programs (host::sliding_ops)
    int n_ops[2];             // byte pairs
    const uint32_t *in;       // per (item, prime): 2s words
    uint32_t *out;            // per (item or element, prime)
    const uint32_t *idx;      // decrypt: item -> element (compaction), else null
    size_t count;             // items [first, first + count) of this launch
    size_t first;
    uint32_t *status;         // decrypt: bit2 = not coprime
    uint32_t *scratch;        // tables
};

// Encrypt step 2 / decrypt exponentiation on digits.
//   MODE 0 (encrypt): in = x < p plain at [x | 0]; X̃ = x·R² mod p² has
//     A = x·R mod p and B = k·R mod p with k = (x·R − A)/p = (−A)·p⁻¹ mod R.
//     out = [A | B] of x^p (k_enc_post makes it plain).
//   MODE 1 (decrypt): in = X̃ = c·R² mod p² (k_dec_pre); lo = X̃ mod R,
//     hi = X̃ div R; MM_m(1, lo) gives lo = (t + ge·p)·R − m·p, so
//     A = hi + t (mod p, flag ge2) and B = (ge + ge2)·R − m (mod p).
//     u = c^(p−1) = 1 + p·ℓ has digits (R mod p, R mod p + ℓ·R²), so the CRT
//     share m_p = ℓ·h_p = MM(B − R mod p, h_p·R⁻¹) goes to out (s words per
//     (element, prime)); A = 0 flags c ≡ 0 (mod p).
#ifndef SFXB_P2_MINB
#define SFXB_P2_MINB 1
#endif
template <int s, int TPI, int W, int MODE>
__global__ void __launch_bounds__(kBlock, SFXB_P2_MINB) k_p2_pow(P2Args a) {
    constexpr int L = s / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[s / 2 * NI], sD[s / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const int which = (int)blockIdx.y; // one prime per block row: uniform digits
    const size_t gi = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * NI + st.inst;
    uint32_t *table = a.scratch + gi * ((size_t)(2 * s) << W);
    const ModRef M = a.mod_p[which].ref();
    uint32_t N[L];
    load_const<s, TPI>(N, M, kMod);
    SFXB_UNIFORM_LOOP(local, active, a.count) {
        const size_t item = a.first + local;
        const uint32_t *src = a.in + (item * 2 + which) * 2 * s;
        uint32_t A[L], B[L], x[L];
        if constexpr (MODE == 0) {
            load_lane<s, TPI>(x, src);
            uint32_t C[L];
            load_const<s, TPI>(C, M, kR2);
            stage_regs<s, TPI>(st, C);
            uint32_t q[L];
            mont_mul_m<s, TPI>(A, q, x, st.sB, st.inst, N, M.np); // A = x·R mod p
            // k = (−A)·p⁻¹ mod 2^(32s) (exact division), every lane redundantly
            // from the staged words of A
            uint32_t tmp[L];
            relayout<s, s, TPI>(tmp, A, st);
            const uint32_t *pinv = a.pinv[which];
            uint32_t kw[s];
#pragma unroll
            for (int k = 0; k < s; ++k) kw[k] = 0u;
            uint32_t carry_neg = 1u; // −A = ~A + 1
#pragma unroll
            for (int i = 0; i < s; ++i) {
                const uint32_t ai = ~staged_word<TPI>(st, i);
                const uint32_t ni = ai + carry_neg;
                carry_neg = (carry_neg && ni == 0u) ? 1u : 0u;
                uint32_t c = 0;
#pragma unroll
                for (int j = 0; j < s - i; ++j) {
                    const uint64_t t = (uint64_t)ni * __ldg(pinv + j) + kw[i + j] + c;
                    kw[i + j] = (uint32_t)t;
                    c = (uint32_t)(t >> 32);
                }
            }
            const int tl = inst_lane<TPI>();
#pragma unroll
            for (int k = 0; k < L; ++k) {
                uint32_t v = 0;
#pragma unroll
                for (int tt = 0; tt < TPI; ++tt) v = (tl == tt) ? kw[tt * L + k] : v;
                tmp[k] = v;
            }
            // B = k·R mod p = MM(R² mod p, k)   (register operand < p, k any)
            stage_regs<s, TPI>(st, tmp);
            mont_mul_m<s, TPI>(B, q, C, st.sB, st.inst, N, M.np);
        } else {
            uint32_t lo[L], hi[L];
            load_lane<s, TPI>(lo, src);
            load_lane<s, TPI>(hi, src + s);
            p2_split<s, TPI>(A, B, lo, hi, st, N, M.np, M.w + kOne * s);
        }
        p2_pow<s, TPI>(A, B, a.ops[which], a.n_ops[which], W, table, st, sD, N, M.np, M.w + kOne * s,
                       a.negR[which]);
        if constexpr (MODE == 0) {
            uint32_t *dst = a.out + (item * 2 + which) * 2 * s;
            if (active) {
                store_lane<s, TPI>(dst, A);
                store_lane<s, TPI>(dst + s, B);
            }
        } else {
            const uint32_t e = a.idx[item];
            if (eq_small<L, TPI>(A, 0u) && active && inst_lane<TPI>() == 0) atomicOr(a.status, 4u);
            uint32_t C[L], mp[L], q[L];
            load_const<s, TPI>(C, M, kOne);
            mod_sub<s, TPI>(x, B, C, N);
            load_lane<s, TPI>(C, a.cdec[which]);
            stage_regs<s, TPI>(st, C);
            mont_mul_m<s, TPI>(mp, q, x, st.sB, st.inst, N, M.np); // ℓ·h_p mod p
            if (active) store_lane<s, TPI>(a.out + ((size_t)e * 2 + which) * s, mp);
        }
    }
}

// Encrypt: [A | B] digits of Ũ = u·R² mod p² -> plain u = x^p mod p² in place:
//   u = Ũ·R⁻² = MM2(A, R) + MM2(B, p)  (mod p²), MM2 = Montgomery product mod p².
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_enc_post(EncArgs a) {
    constexpr int S2 = 2 * s, L2 = S2 / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S2 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const int which = (int)blockIdx.y;
    const ModRef M2 = a.mod_pq2[which].ref();
    uint32_t N2[L2];
    load_const<S2, TPI>(N2, M2, kMod);
    const int tl = inst_lane<TPI>();
    // lane limbs [tl·L2, tl·L2 + L2): the low half (limbs < s) or the high half
    const bool low = tl * L2 < s;
    SFXB_UNIFORM_LOOP(e, active, a.count) {
        uint32_t *yp = a.y + (e * 2 + which) * S2;
        uint32_t ab[L2], bb[L2], Rc[L2], pc[L2], u[L2], v[L2];
        load_lane<S2, TPI>(ab, yp);
        // B moved to the low half through the staging buffer
        relayout<S2, S2, TPI>(bb, ab, st);
#pragma unroll
        for (int k = 0; k < L2; ++k) {
            const int limb = tl * L2 + k;
            bb[k] = limb < s ? staged_word<TPI>(st, limb + s) : 0u;
            ab[k] = low ? ab[k] : 0u;
            Rc[k] = limb == s ? 1u : 0u;
        }
        __syncwarp();
        const ModRef Mp = a.mod_pq[which].ref();
#pragma unroll
        for (int k = 0; k < L2; ++k) {
            const int limb = tl * L2 + k;
            pc[k] = limb < s ? __ldg(Mp.w + limb) : 0u;
        }
        mmul<S2, TPI>(u, ab, Rc, st, N2, M2.np);
        mmul<S2, TPI>(v, bb, pc, st, N2, M2.np);
        mod_add<S2, TPI>(u, u, v, N2);
        if (active) store_lane<S2, TPI>(yp, u);
    }
}

// Decrypt: X̃ = c·R² mod p² (Montgomery form of c mod p², c < n²) per
// (item, prime) for k_p2_pow<MODE 1>.
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_dec_pre(DecArgs a, uint32_t n_items, uint32_t *xt) {
    constexpr int S2 = 2 * s, L2 = S2 / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S2 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const int which = (int)blockIdx.y;
    const ModRef M2 = a.mod_pq2[which].ref();
    uint32_t N2[L2];
    load_const<S2, TPI>(N2, M2, kMod);
    SFXB_UNIFORM_LOOP(item, active, (size_t)n_items) {
        const uint32_t e = a.idx[item];
        uint32_t lo[L2], hi[L2], u[L2];
        load_lane<S2, TPI>(lo, a.cts + (size_t)e * 2 * S2);
        load_lane<S2, TPI>(hi, a.cts + (size_t)e * 2 * S2 + S2);
        to_mont_wide<S2, TPI>(u, lo, hi, M2, st, N2);
        if (active) store_lane<S2, TPI>(xt + (item * 2 + which) * S2, u);
    }
}


// ------------------------------------------------------------------ K2 at the key holder
//
// The active party holds p and q (federation.cpp:83-85), so its encrypted
// histogram can multiply ciphertexts by CRT: mod p² and mod q² on base-p/q
// digits (2 × 3 CIOS passes of 2s²+s products = 12,480 at 2048-bit n against
// one mod-n² pass of 2(4s)²+4s = 32,896), recombined to the unique residue
// mod n² per output slot — bit-identical to the mod-n² product.
// gh ciphertexts live as [A_p | B_p | A_q | B_q] (4s words, the ciphertext's
// own footprint).

struct CrtArgs {
    ModArg mod_p[2];      // s
    ModArg mod_p2[2];     // 2s
    ModArg mod_n2;        // 4s
    const uint32_t *qq_inv_m; // (q²)⁻¹·R2 mod p²       (2s)
    const uint32_t *q2R_n2;   // q²·R4 mod n²           (4s)
    const uint32_t *negR[2];  // p − R mod p            (s)
    const uint32_t *one[2];   // digits of 1̃ mod p²: [R mod p | R mod p]  (2s)
};

// plain ciphertexts (4s words each, in place) -> digits of c mod p², c mod q²
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_gh_digits(CrtArgs a, uint32_t *gh, size_t count) {
    constexpr int S2 = 2 * s, L2 = S2 / TPI, L = s / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S2 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    SFXB_UNIFORM_LOOP(e, active, count) {
        uint32_t *c = gh + e * 4 * s;
        uint32_t lo[L2], hi[L2], X[2][L2];
        load_lane<S2, TPI>(lo, c);
        load_lane<S2, TPI>(hi, c + S2);
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
            const ModRef M2 = a.mod_p2[pr].ref();
            uint32_t N2[L2], u[L2];
            load_const<S2, TPI>(N2, M2, kMod);
            to_mont_wide<S2, TPI>(u, lo, hi, M2, st, N2); // c·R2 mod p² (R2 = 2^(64s) = R²)
#pragma unroll
            for (int k = 0; k < L2; ++k) X[pr][k] = u[k];
        }
        __syncwarp();
        if (active) {
            store_lane<S2, TPI>(c, X[0]);
            store_lane<S2, TPI>(c + S2, X[1]);
        }
        __syncwarp();
#pragma unroll 1
        for (int pr = 0; pr < 2; ++pr) {
            const ModRef M = a.mod_p[pr].ref();
            uint32_t N[L], xl[L], xh[L], A[L], B[L];
            load_const<s, TPI>(N, M, kMod);
            load_lane<s, TPI>(xl, c + pr * S2);
            load_lane<s, TPI>(xh, c + pr * S2 + s);
            p2_split<s, TPI>(A, B, xl, xh, st, N, M.np, M.w + kOne * s);
            __syncwarp();
            if (active) {
                store_lane<s, TPI>(c + pr * S2, A);
                store_lane<s, TPI>(c + pr * S2 + s, B);
            }
            __syncwarp();
        }
    }
}

// Segmented product pass on digits (the k_seg_prod protocol).  Job j =
// 4·rank + 2·gh + prime over the length-sorted pieces; TPI lanes per job (the
// prime may differ between the instances of a warp: each loads its own
// modulus).  An instance past the end of its piece multiplies by the digits
// of 1̃, so every instance of a warp runs the same passes.
#ifndef SFXB_ND_MINB
#define SFXB_ND_MINB 1
#endif
#ifndef SFXB_ND_PREFETCH
#define SFXB_ND_PREFETCH 0
#endif
#ifndef SFXB_K_MINB
#define SFXB_K_MINB 1
#endif
template <int s, int TPI, int C>
__global__ void __launch_bounds__(kBlock, (TPI > 1 ? SFXB_K_MINB : 1)) k_seg_prod_p2(CrtArgs a, const Piece *pieces, const uint32_t *order,
                                                        size_t n_pieces, const uint32_t *sorted, const uint32_t *src,
                                                        uint32_t *dst, unsigned long long *next_job) {
    constexpr int L = s / TPI, NI = kBlock / TPI, NIW = 32 / TPI;
    __shared__ uint2 sB[s / 2 * NI], sD[s / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const size_t total = 4 * n_pieces;
    SFXB_K2_JOB_STATE;
    for (;;) {
        unsigned long long base = 0;
        SFXB_K2_CLAIM(base, NIW, total);
        const size_t mine = base + (threadIdx.x & 31) / TPI;
        const bool active = mine < total;
        const size_t job = active ? mine : total - 1;
        const uint32_t pidx = order[job >> 2];
        const Piece pc = pieces[pidx];
        const uint32_t g = (uint32_t)((job >> 1) & 1), pr = (uint32_t)(job & 1);
        // (selects, not a dynamic index into the parameter arrays: no local copy)
        const ModRef M = (pr ? a.mod_p[1] : a.mod_p[0]).ref();
        const uint32_t *one = pr ? a.one[1] : a.one[0], *negR = pr ? a.negR[1] : a.negR[0];
        uint32_t N[L], A[L], B[L];
        load_const<s, TPI>(N, M, kMod);
        auto item_ptr = [&](uint32_t k) -> const uint32_t * {
            const size_t idx = sorted ? (2 * (size_t)sorted[pc.start + k] + g) : (2 * (size_t)(pc.start + k) + g);
            return src + idx * 4 * s + pr * 2 * s;
        };
        const uint32_t *p0 = item_ptr(0);
        load_lane<s, TPI>(A, p0);
        load_lane<s, TPI>(B, p0 + s);
        for (int k = 1; k < C; ++k) {
            const bool more = active && (uint32_t)k < pc.len;
            if (!__any_sync(0xffffffffu, more)) break; // warp-uniform exit
            // the rows are gathered at random from a gh buffer far larger
            // than L2: fetch the next item while this one is multiplied
            if (more && (uint32_t)k + 1 < pc.len && inst_lane<TPI>() == 0) {
                const uint32_t *nx = item_ptr((uint32_t)k + 1);
#pragma unroll
                for (int o = 0; o < 2 * s; o += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + o));
            }
            p2_mul<s, TPI>(A, B, more ? item_ptr((uint32_t)k) : one, false, st, sD, N, M.np, M.w + kOne * s, negR);
        }
        if (active) {
            uint32_t *d = dst + (2 * (size_t)pidx + g) * 4 * s + pr * 2 * s;
            store_lane<s, TPI>(d, A);
            store_lane<s, TPI>(d + s, B);
        }
    }
}

// digits [A | B] of Ũ = u·R2 mod p² (this lane's layout at S2) -> plain u:
//   u = MM2(A, R) + MM2(B, p)  (mod p²)
template <int s, int TPI>
__device__ __forceinline__ void p2_digits_plain(uint32_t (&u)[2 * s / TPI], const uint32_t *ab, const ModRef &M2,
                                                const ModRef &Mp, const Stage &st, const uint32_t (&N2)[2 * s / TPI]) {
    constexpr int S2 = 2 * s, L2 = S2 / TPI;
    const int tl = inst_lane<TPI>();
    const bool low = tl * L2 < s;
    uint32_t av[L2], bv[L2], Rc[L2], pc[L2], v[L2];
    load_lane<S2, TPI>(av, ab);
    relayout<S2, S2, TPI>(bv, av, st);
#pragma unroll
    for (int k = 0; k < L2; ++k) {
        const int limb = tl * L2 + k;
        bv[k] = limb < s ? staged_word<TPI>(st, limb + s) : 0u;
        av[k] = low ? av[k] : 0u;
        Rc[k] = limb == s ? 1u : 0u;
        pc[k] = limb < s ? __ldg(Mp.w + limb) : 0u;
    }
    __syncwarp();
    mmul<S2, TPI>(u, av, Rc, st, N2, M2.np);
    mmul<S2, TPI>(v, bv, pc, st, N2, M2.np);
    mod_add<S2, TPI>(u, u, v, N2);
}

// Output slot (key, gh): count == 0 -> 1 (Montgomery one for partials); else
// CRT of the key's final digit partial: c = c_q + q²·((c_p − c_q)·q⁻² mod p²).
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_hist_finalize_p2(CrtArgs a, const uint32_t *count,
                                                             const uint32_t *final_idx, size_t nkeys,
                                                             const uint32_t *partial, FinOut o) {
    constexpr int S2 = 2 * s, S4 = 4 * s, L2 = S2 / TPI, L4 = S4 / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S4 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M4 = a.mod_n2.ref();
    uint32_t N4[L4];
    load_const<S4, TPI>(N4, M4, kMod);
    SFXB_UNIFORM_LOOP(slot, active, 2 * nkeys) {
        if (fin_skip(o, slot)) continue;
        const size_t key = slot >> 1;
        const uint32_t g = (uint32_t)(slot & 1);
        uint32_t c4[L4];
        // warp-uniform: every instance runs the CRT (empty keys on a dummy but
        // valid operand) and selects afterwards
        const bool empty = count[key] == 0;
        {
            // (an empty key reads its own output slot: valid memory, result discarded)
            const uint32_t *pp = empty ? (o.mont ? o.mont : o.plain) + slot * S4
                                       : partial + (2 * (size_t)final_idx[key] + g) * S4;
            const ModRef M2 = a.mod_p2[0].ref(), Q2 = a.mod_p2[1].ref();
            uint32_t N2[L2], yp[L2], yq[L2], d[L2], C2[L2], h[L2];
            load_const<S2, TPI>(N2, Q2, kMod);
            p2_digits_plain<s, TPI>(yq, pp + S2, Q2, a.mod_p[1].ref(), st, N2);
            load_const<S2, TPI>(N2, M2, kMod);
            p2_digits_plain<s, TPI>(yp, pp, M2, a.mod_p[0].ref(), st, N2);
            reduce_once<S2, TPI>(d, yq, N2); // c_q mod p² (c_q < q² < 2p²)
            mod_sub<S2, TPI>(d, yp, d, N2);
            load_lane<S2, TPI>(C2, a.qq_inv_m);
            mmul<S2, TPI>(h, C2, d, st, N2, M2.np);
            uint32_t h4[L4], yq4[L4], C4[L4];
            relayout<S2, S4, TPI>(h4, h, st);
            relayout<S2, S4, TPI>(yq4, yq, st);
            load_lane<S4, TPI>(C4, a.q2R_n2);
            mmul<S4, TPI>(c4, C4, h4, st, N4, M4.np); // q²·h (< n², exact)
            mod_add<S4, TPI>(c4, c4, yq4, N4);
        }
        if (empty) set_small<L4, TPI>(c4, 1u);
        if (o.plain && active) store_lane<S4, TPI>(o.plain + slot * S4, c4);
        if (o.mont) {
            uint32_t C4[L4];
            load_const<S4, TPI>(C4, M4, kR2);
            mmul<S4, TPI>(c4, C4, c4, st, N4, M4.np); // 1 -> Montgomery one
            if (active) store_lane<S4, TPI>(o.mont + slot * S4, c4);
        }
    }
}


// ------------------------------------------------------------------ K2 at a passive party
//
// Without the factorisation the same digit arithmetic works with n in the
// role of p (nothing above needs primality, only n odd and n > R/2 for
// R = 2^(64s)): X̃ = X·R² mod n² ≡ A·R + B·n, a multiplication mod n² is 3
// CIOS passes mod n, 3·(2(2s)²+2s) = 24,768 products at 2048-bit n against
// 2(4s)²+4s = 32,896 for one CIOS pass mod n².  The gh ciphertexts are
// already in Montgomery form mod n² (= X̃); k_gh_split_n splits them into
// [A | B] in place.

struct NdArgs {
    ModArg mod_n;            // 2s
    ModArg mod_n2;           // 4s
    const uint32_t *negR;    // n − R mod n              (2s)
    const uint32_t *one;     // digits of 1̃: [R mod n | R mod n]   (4s)
    const uint32_t *n4;      // n zero-extended           (4s)
    const uint32_t *r4;      // digits of R⁴ mod n² (the representative of R² mod n²)  (4s)
};

template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_gh_split_n(NdArgs a, uint32_t *gh, size_t count) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M = a.mod_n.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, M, kMod);
    SFXB_UNIFORM_LOOP(e, active, count) {
        uint32_t *c = gh + e * 2 * S;
        uint32_t lo[L], hi[L], A[L], B[L];
        load_lane<S, TPI>(lo, c);
        load_lane<S, TPI>(hi, c + S);
        p2_split<S, TPI>(A, B, lo, hi, st, N, M.np, M.w + kOne * S);
        if (active) { // each lane rewrites exactly the limbs it read
            store_lane<S, TPI>(c, A);
            store_lane<S, TPI>(c + S, B);
        }
    }
}

// Plain ciphertexts X < n² (2S words each, in place) -> digits of X̃ = X·R² mod
// n² in one kernel: the digits (A0, B0) of X itself (p2_split; as a
// representative X stands for X·R⁻²) times the digits of R⁴ mod n² give
// X·R⁴·R⁻² = X̃ — a split plus one digit multiplication, 2·S² + 5·S² + … fewer
// products than a mod-n² Montgomery conversion (2(2S)² + 2S) followed by the
// split (k_to_mont + k_gh_split_n).
template <int S, int TPI>
__global__ void __launch_bounds__(kBlock) k_gh_nd_direct(NdArgs a, uint32_t *gh, size_t count) {
    constexpr int L = S / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S / 2 * NI], sD[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M = a.mod_n.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, M, kMod);
    SFXB_UNIFORM_LOOP(e, active, count) {
        uint32_t *c = gh + e * 2 * S;
        uint32_t lo[L], hi[L], A[L], B[L];
        load_lane<S, TPI>(lo, c);
        load_lane<S, TPI>(hi, c + S);
        p2_split<S, TPI>(A, B, lo, hi, st, N, M.np, M.w + kOne * S);
        __syncwarp();
        p2_mul<S, TPI>(A, B, a.r4, false, st, sD, N, M.np, M.w + kOne * S, a.negR);
        if (active) { // each lane rewrites exactly the limbs it read
            store_lane<S, TPI>(c, A);
            store_lane<S, TPI>(c + S, B);
        }
    }
}

// Segmented product pass on base-n digits (the k_seg_prod protocol; an
// instance past the end of its piece multiplies by the digits of 1̃, which
// leaves (A, B) unchanged, so every instance runs the same passes).
template <int S, int TPI, int C>
__global__ void __launch_bounds__(kBlock, SFXB_ND_MINB) k_seg_prod_nd(NdArgs a, const Piece *pieces, const uint32_t *order,
                                                        size_t n_pieces, const uint32_t *sorted, const uint32_t *src,
                                                        uint32_t *dst, unsigned long long *next_job) {
    constexpr int L = S / TPI, NI = kBlock / TPI, NIW = 32 / TPI;
    __shared__ uint2 sB[S / 2 * NI], sD[S / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M = a.mod_n.ref();
    uint32_t N[L];
    load_const<S, TPI>(N, M, kMod);
    const size_t total = 2 * n_pieces;
    SFXB_K2_JOB_STATE;
    for (;;) {
        unsigned long long base = 0;
        SFXB_K2_CLAIM(base, NIW, total);
        const size_t mine = base + (threadIdx.x & 31) / TPI;
        const bool active = mine < total;
        const size_t job = active ? mine : total - 1;
        const uint32_t pidx = order[job >> 1];
        const Piece pc = pieces[pidx];
        const uint32_t g = (uint32_t)(job & 1);
        auto item_ptr = [&](uint32_t k) -> const uint32_t * {
            const size_t idx = sorted ? (2 * (size_t)sorted[pc.start + k] + g) : (2 * (size_t)(pc.start + k) + g);
            return src + idx * 2 * S;
        };
        uint32_t A[L], B[L];
        const uint32_t *p0 = item_ptr(0);
        load_lane<S, TPI>(A, p0);
        load_lane<S, TPI>(B, p0 + S);
        for (int k = 1; k < C; ++k) {
            const bool more = active && (uint32_t)k < pc.len;
            if (!__any_sync(0xffffffffu, more)) break; // warp-uniform exit
#if SFXB_ND_PREFETCH
            if (more && (uint32_t)k + 1 < pc.len && inst_lane<TPI>() == 0) {
                const uint32_t *nx = item_ptr((uint32_t)k + 1);
#pragma unroll
                for (int o = 0; o < 2 * S; o += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + o));
            }
#endif
            p2_mul<S, TPI>(A, B, more ? item_ptr((uint32_t)k) : a.one, false, st, sD, N, M.np, M.w + kOne * S,
                           a.negR);
        }
        if (active) {
            uint32_t *d = dst + (2 * (size_t)pidx + g) * 2 * S;
            store_lane<S, TPI>(d, A);
            store_lane<S, TPI>(d + S, B);
        }
    }
}

// Output slot: count == 0 -> 1 (Montgomery one for partials); else the
// key's final digits [A | B] -> plain c = MM4(A, R) + MM4(B, n) (mod n²),
// Montgomery form c·R4 for partials.
template <int s, int TPI>
__global__ void __launch_bounds__(kBlock) k_hist_finalize_nd(NdArgs a, const uint32_t *count,
                                                             const uint32_t *final_idx, size_t nkeys,
                                                             const uint32_t *partial, FinOut o) {
    constexpr int S2 = 2 * s, S4 = 4 * s, L4 = S4 / TPI, NI = kBlock / TPI;
    __shared__ uint2 sB[S4 / 2 * NI];
    const Stage st = make_stage<TPI>(sB);
    const ModRef M4 = a.mod_n2.ref();
    uint32_t N4[L4];
    load_const<S4, TPI>(N4, M4, kMod);
    const int tl = inst_lane<TPI>();
    const bool low = tl * L4 < S2;
    SFXB_UNIFORM_LOOP(slot, active, 2 * nkeys) {
        if (fin_skip(o, slot)) continue;
        const size_t key = slot >> 1;
        const uint32_t g = (uint32_t)(slot & 1);
        const bool empty = count[key] == 0;
        const uint32_t *pp = empty ? (o.mont ? o.mont : o.plain) + slot * S4
                                   : partial + (2 * (size_t)final_idx[key] + g) * S4;
        uint32_t av[L4], bv[L4], Rc[L4], nc[L4], u[L4], v[L4];
        load_lane<S4, TPI>(av, pp);
        relayout<S4, S4, TPI>(bv, av, st);
#pragma unroll
        for (int k = 0; k < L4; ++k) {
            const int limb = tl * L4 + k;
            bv[k] = limb < S2 ? staged_word<TPI>(st, limb + S2) : 0u;
            av[k] = low ? av[k] : 0u;
            Rc[k] = limb == S2 ? 1u : 0u;
        }
        __syncwarp();
        load_lane<S4, TPI>(nc, a.n4);
        mmul<S4, TPI>(u, av, Rc, st, N4, M4.np);
        mmul<S4, TPI>(v, bv, nc, st, N4, M4.np);
        mod_add<S4, TPI>(u, u, v, N4);
        if (empty) set_small<L4, TPI>(u, 1u);
        if (o.plain && active) store_lane<S4, TPI>(o.plain + slot * S4, u);
        if (o.mont) {
            load_const<S4, TPI>(v, M4, kR2);
            mmul<S4, TPI>(u, v, u, st, N4, M4.np); // 1 -> Montgomery one
            if (active) store_lane<S4, TPI>(o.mont + slot * S4, u);
        }
    }
}

} // namespace dev
} // namespace sfxb
