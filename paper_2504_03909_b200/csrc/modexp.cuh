// Modular toolbox on top of mont.cuh: modulus descriptors, modular add/sub,
// fixed-window Montgomery exponentiation, reduction of double-width values.
#pragma once
#include "mont.cuh"

namespace sfxb {
namespace dev {

// A Montgomery modulus in device memory: words [m | one | r2 | r3], each S
// limbs (one = R mod m, r2 = R² mod m, r3 = R³ mod m, R = 2^(32S)), and np.
struct ModRef {
    const uint32_t *w; // 4·S words
    uint32_t np;
};

template <int S, int TPI>
struct Lane {
    static constexpr int L = S / TPI;
};

template <int S, int TPI>
__device__ __forceinline__ void load_const(uint32_t (&v)[S / TPI], const ModRef &M, int which) {
    load_lane<S, TPI>(v, M.w + which * S);
}
enum : int { kMod = 0, kOne = 1, kR2 = 2, kR3 = 3 };

// Shared-memory staging for operand b of the instances of one block.
struct Stage {
    uint2 *sB;
    int NI;
    int inst;
};

// (one lane per instance: the slots are private to the thread, so program
// order suffices and the staging is safe in divergent code)
template <int S, int TPI>
__device__ __forceinline__ void stage_b(const Stage &st, const uint32_t (&v)[S / TPI]) {
    if constexpr (TPI > 1) __syncwarp();
    store_b<S, TPI>(st.sB, st.NI, st.inst, v);
    if constexpr (TPI > 1) __syncwarp();
}

// r = A·B·R⁻¹ mod M with B given in lane limbs (staged through shared memory)
template <int S, int TPI>
__device__ __forceinline__ void mmul(uint32_t (&r)[S / TPI], const uint32_t (&A)[S / TPI],
                                     const uint32_t (&B)[S / TPI], const Stage &st,
                                     const uint32_t (&N)[S / TPI], uint32_t np) {
    stage_b<S, TPI>(st, B);
    mont_mul<S, TPI>(r, A, st.sB, st.NI, st.inst, N, np);
}

// r = (a + b) mod M for a, b < M (distributed, carry/borrow lookahead)
template <int S, int TPI>
__device__ __forceinline__ void mod_add(uint32_t (&r)[S / TPI], const uint32_t (&a)[S / TPI],
                                        const uint32_t (&b)[S / TPI], const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t R[L];
    R[0] = add_cc(a[0], b[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) R[k] = addc_cc(a[k], b[k]);
    uint32_t c = addc(0u, 0u);
    uint32_t over;
    if constexpr (TPI == 1) {
        over = c;
    } else {
        // carry into lane t+1; lookahead with propagate = all ones
        bool all_ones = true;
#pragma unroll
        for (int k = 0; k < L; ++k) all_ones &= (R[k] == 0xffffffffu);
        const uint32_t G = inst_ballot<TPI>(c != 0);
        const uint32_t P = inst_ballot<TPI>(all_ones);
        const uint64_t sum = (uint64_t)P + ((uint64_t)G << 1);
        const uint32_t cin = (uint32_t)(sum ^ P);
        if ((cin >> inst_lane<TPI>()) & 1u) {
            R[0] = add_cc(R[0], 1u);
#pragma unroll
            for (int k = 1; k < L; ++k) R[k] = addc_cc(R[k], 0u);
        }
        over = (uint32_t)(sum >> TPI) & 1u;
    }
    final_sub<L, TPI>(R, over, N);
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = R[k];
}

// r = a − b (full width, wraps mod 2^(32S)); returns 1 when a < b.
template <int S, int TPI>
__device__ __forceinline__ uint32_t sub_full(uint32_t (&r)[S / TPI], const uint32_t (&a)[S / TPI],
                                             const uint32_t (&b)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t D[L];
    D[0] = sub_cc(a[0], b[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) D[k] = subc_cc(a[k], b[k]);
    uint32_t bout = subc(0u, 0u) & 1u;
    uint32_t top;
    if constexpr (TPI == 1) {
        top = bout;
    } else {
        bool zero = true;
#pragma unroll
        for (int k = 0; k < L; ++k) zero &= (D[k] == 0u);
        const uint32_t G = inst_ballot<TPI>(bout != 0);
        const uint32_t P = inst_ballot<TPI>(zero);
        const uint64_t sum = (uint64_t)P + ((uint64_t)G << 1);
        const uint32_t bin = (uint32_t)(sum ^ P);
        if ((bin >> inst_lane<TPI>()) & 1u) {
            D[0] = sub_cc(D[0], 1u);
#pragma unroll
            for (int k = 1; k < L; ++k) D[k] = subc_cc(D[k], 0u);
        }
        top = (uint32_t)(sum >> TPI) & 1u;
    }
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = D[k];
    return top;
}

// r = (a − b) mod M for a, b < M
template <int S, int TPI>
__device__ __forceinline__ void mod_sub(uint32_t (&r)[S / TPI], const uint32_t (&a)[S / TPI],
                                        const uint32_t (&b)[S / TPI], const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t D[L];
    const uint32_t neg = sub_full<S, TPI>(D, a, b);
    // add M back when a < b; computed unconditionally (warp-uniform
    // collectives), selected per instance
    uint32_t T[L];
    T[0] = add_cc(D[0], N[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) T[k] = addc_cc(D[k], N[k]);
    uint32_t c = addc(0u, 0u);
    if constexpr (TPI > 1) {
        bool all_ones = true;
#pragma unroll
        for (int k = 0; k < L; ++k) all_ones &= (T[k] == 0xffffffffu);
        const uint32_t G = inst_ballot<TPI>(c != 0);
        const uint32_t P = inst_ballot<TPI>(all_ones);
        const uint64_t sum = (uint64_t)P + ((uint64_t)G << 1);
        const uint32_t cin = (uint32_t)(sum ^ P);
        if ((cin >> inst_lane<TPI>()) & 1u) {
            T[0] = add_cc(T[0], 1u);
#pragma unroll
            for (int k = 1; k < L; ++k) T[k] = addc_cc(T[k], 0u);
        }
    }
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = neg ? T[k] : D[k];
}

// r = x mod M for x < 2M (one conditional subtraction)
template <int S, int TPI>
__device__ __forceinline__ void reduce_once(uint32_t (&r)[S / TPI], const uint32_t (&x)[S / TPI],
                                            const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t R[L];
#pragma unroll
    for (int k = 0; k < L; ++k) R[k] = x[k];
    final_sub<L, TPI>(R, 0u, N);
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = R[k];
}

// Montgomery form of a 2S-limb value T = hi·2^(32S) + lo (any value):
//   T·R mod M = MontMul(R³, hi) + MontMul(R², lo)   (the scanned operand may
// be any S-limb value as long as the register operand is < M).
template <int S, int TPI>
__device__ __forceinline__ void to_mont_wide(uint32_t (&r)[S / TPI], const uint32_t (&lo)[S / TPI],
                                             const uint32_t (&hi)[S / TPI], const ModRef &M,
                                             const Stage &st, const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t C[L], a[L], b[L];
    load_const<S, TPI>(C, M, kR3);
    mmul<S, TPI>(a, C, hi, st, N, M.np);
    load_const<S, TPI>(C, M, kR2);
    mmul<S, TPI>(b, C, lo, st, N, M.np);
    mod_add<S, TPI>(r, a, b, N);
}

// Montgomery form of an S-limb value x (any value < 2^(32S))
template <int S, int TPI>
__device__ __forceinline__ void to_mont(uint32_t (&r)[S / TPI], const uint32_t (&x)[S / TPI],
                                        const ModRef &M, const Stage &st,
                                        const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t C[L];
    load_const<S, TPI>(C, M, kR2);
    mmul<S, TPI>(r, C, x, st, N, M.np);
}

// plain value of a Montgomery-form x
template <int S, int TPI>
__device__ __forceinline__ void from_mont(uint32_t (&r)[S / TPI], const uint32_t (&x)[S / TPI],
                                          const Stage &st, const uint32_t (&N)[S / TPI], uint32_t np) {
    constexpr int L = S / TPI;
    uint32_t one[L];
    set_small<L, TPI>(one, 1u);
    mmul<S, TPI>(r, x, one, st, N, np);
}

// squarings of the mod-p exponentiation (encrypt step 1) by mont_sqr (one
// lane per instance) in an SFXB_SQR / SFXB_SQR_POW build; the default build
// squares with mont_mul(x, x): measured faster on the B200.
// The digit squarings of k_p2_pow do use mont_sqr (padic.cuh p2_mul).
#if defined(SFXB_SQR) || defined(SFXB_SQR_POW)
template <int TPI>
constexpr bool kSqrPow = TPI == 1;
#else
template <int TPI>
constexpr bool kSqrPow = false;
#endif

// Fixed-window exponentiation in the Montgomery domain:
//   x <- x^e, e given as `nd` window digits of `w` bits, most significant first.
// `table` = this instance's 2^w·S-word scratch in global memory (L2-resident).
// The table build and the main loop share ONE Montgomery multiply call site
// (the operand is either acc itself — a squaring — or a table entry / x), so
// the hot loop is a single inlined copy of the unrolled CIOS body.
template <int S, int TPI>
__device__ __forceinline__ void mont_pow(uint32_t (&x)[S / TPI], const uint8_t *digits, int nd, int w,
                                         uint32_t *table, const ModRef &M, const Stage &st,
                                         const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    const int T = 1 << w;
    uint32_t one[L];
    load_const<S, TPI>(one, M, kOne);
    store_lane<S, TPI>(table, one);
    store_lane<S, TPI>(table + S, x);
    // op sequence: table build (T−2 multiplies by x), then for each digit
    // after the first: w squarings and one multiply by table[d] (skipped for d == 0)
    uint32_t acc[L];
#pragma unroll
    for (int k = 0; k < L; ++k) acc[k] = x[k];
    int j = 2;          // next table entry to build (build phase while j < T)
    int i = 1, sq = 0;  // digit index and squarings done for it (main phase)
    bool started = false;
    for (;;) {
        bool square;
        const uint32_t *bsrc = nullptr;
        if (j < T) {
            square = false;
            bsrc = table + S; // x
        } else {
            if (!started) {
                load_lane<S, TPI>(acc, table + (int)digits[0] * S);
                started = true;
            }
            if (i >= nd) break;
            if (sq < w) {
                square = true;
            } else {
                const int d = digits[i];
                ++i;
                sq = 0;
                if (d == 0) continue;
                square = false;
                bsrc = table + d * S;
            }
        }
        if constexpr (kSqrPow<TPI>) {
            if (square) {
                // symmetric products once (mont_sqr: 24% fewer at S = 32)
                mont_sqr<S>(acc, acc, N, M.np);
            } else {
                uint32_t b[L];
                load_lane<S, TPI>(b, bsrc);
                mmul<S, TPI>(acc, acc, b, st, N, M.np);
            }
        } else {
            uint32_t b[L];
            if (square) {
#pragma unroll
                for (int k = 0; k < L; ++k) b[k] = acc[k];
            } else {
                load_lane<S, TPI>(b, bsrc);
            }
            mmul<S, TPI>(acc, acc, b, st, N, M.np);
        }
        if (j < T) {
            store_lane<S, TPI>(table + j * S, acc);
            ++j;
        } else if (square) {
            ++sq;
        }
    }
#pragma unroll
    for (int k = 0; k < L; ++k) x[k] = acc[k];
}

// Sliding-window exponentiation in the Montgomery domain: x <- x^e with e as
// a host::sliding_ops program (n_ops byte pairs: squarings, odd digit).
// `table` = this instance's scratch of 2^(w−1) + 1 entries of S words: x^1,
// x^3, …, x^(2^w − 1), then x².  One Montgomery multiply call site.
template <int S, int TPI>
__device__ __forceinline__ void mont_pow_ops(uint32_t (&x)[S / TPI], const uint8_t *ops, int n_ops, int w,
                                             uint32_t *table, const ModRef &M, const Stage &st,
                                             const uint32_t (&N)[S / TPI]) {
    constexpr int L = S / TPI;
    const int T = 1 << (w - 1);
    uint32_t *x2 = table + S * T;
    store_lane<S, TPI>(table, x);
    uint32_t acc[L];
#pragma unroll
    for (int k = 0; k < L; ++k) acc[k] = x[k];
    int j = -1, oi = 0, sq = 0;
    bool started = false;
    for (;;) {
        bool square;
        const uint32_t *bsrc = nullptr;
        if (j < T - 1) {
            square = j < 0;
            bsrc = x2;
        } else {
            if (!started) {
                load_lane<S, TPI>(acc, table + S * (ops[1] >> 1));
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
                bsrc = table + S * (d >> 1);
            }
        }
        if constexpr (kSqrPow<TPI>) {
            if (square) {
                // symmetric products once (mont_sqr: 24% fewer at S = 32)
                mont_sqr<S>(acc, acc, N, M.np);
            } else {
                uint32_t b[L];
                load_lane<S, TPI>(b, bsrc);
                mmul<S, TPI>(acc, acc, b, st, N, M.np);
            }
        } else {
            uint32_t b[L];
            if (square) {
#pragma unroll
                for (int k = 0; k < L; ++k) b[k] = acc[k];
            } else {
                load_lane<S, TPI>(b, bsrc);
            }
            mmul<S, TPI>(acc, acc, b, st, N, M.np);
        }
        if (j < T - 1) {
            if (j < 0) {
                store_lane<S, TPI>(x2, acc);
                load_lane<S, TPI>(acc, table);
            } else {
                store_lane<S, TPI>(table + S * (j + 1), acc);
            }
            ++j;
        } else if (square) {
            --sq;
        }
    }
#pragma unroll
    for (int k = 0; k < L; ++k) x[k] = acc[k];
}

} // namespace dev
} // namespace sfxb
