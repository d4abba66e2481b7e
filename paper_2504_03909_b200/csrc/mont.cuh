// Warp-cooperative CIOS Montgomery arithmetic on 32-bit limbs for sm_100a.
//
// One big-integer "instance" (an S-limb value mod M, S = 32·k bits / 32) is
// spread over TPI consecutive lanes of a warp; lane t owns limbs
// [t·L, t·L+L), L = S/TPI (even).  The multiply
//     MontMul(a, b) = a·b·2^(−32S) mod M        (a, b < M, result < M)
// is CIOS (coarsely integrated operand scanning): S iterations, each adds
// a·b_i and q_i·M (q_i = acc_0·(−M⁻¹) mod 2^32) and shifts the accumulator
// down one limb.
//
// Instruction shape: every 32×32 product is ONE
// IMAD.WIDE.U32(.X) — the PTX pair `mad{c}.lo.cc / madc.hi.cc` on the same
// operands with a 64-bit addend in an aligned register pair fuses into one
// wide multiply-add with carry-in/carry-out predicate on sm_100a.  To keep the
// addend pairs aligned the accumulator is held as two arrays (sppark-style):
// E (pairs at even limb positions) and O (pairs at odd positions); a limb
// shift turns O into the next E, and the old E becomes the next O by a MAD
// that reads its addend two registers up (the shift costs no moves).  Carries
// that leave a lane's window are kept in one word Z and folded into the lane's
// top limb one step later; the one-limb shift across lanes is two
// __shfl_down_sync per iteration, q_i is one __shfl_sync.  Operand b is read
// limb-pair by limb-pair (LDS.64) from shared memory.
//
// Exactness: with a, b < M the CIOS accumulator stays < 2M, so after the last
// iteration one cross-lane carry resolution (ballot carry-lookahead) and one
// conditional subtraction give the canonical residue in [0, M) — the residues
// are unique, so results are bit-identical to GMP's `a*b % M` path.
#pragma once
#include <cstdint>

namespace sfxb {
namespace dev {

// ---------------------------------------------------------------- PTX carry primitives

__device__ __forceinline__ uint32_t add_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t addc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t addc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("addc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t sub_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t subc_cc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t subc(uint32_t a, uint32_t b) {
    uint32_t r;
    asm volatile("subc.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// (d0,d1) = a·b + (c0,c1), carry out          -> IMAD.WIDE.U32 (P out)
__device__ __forceinline__ void mad_w_cc(uint32_t &d0, uint32_t &d1, uint32_t a, uint32_t b,
                                         uint32_t c0, uint32_t c1) {
    asm volatile("mad.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.cc.u32 %1, %2, %3, %5;"
                 : "=r"(d0), "=r"(d1)
                 : "r"(a), "r"(b), "r"(c0), "r"(c1));
}
// (d0,d1) = a·b + (c0,c1) + carry in, carry out -> IMAD.WIDE.U32.X (P in/out)
__device__ __forceinline__ void madc_w_cc(uint32_t &d0, uint32_t &d1, uint32_t a, uint32_t b,
                                          uint32_t c0, uint32_t c1) {
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.cc.u32 %1, %2, %3, %5;"
                 : "=r"(d0), "=r"(d1)
                 : "r"(a), "r"(b), "r"(c0), "r"(c1));
}
// (d0,d1) = a·b (no carries)
__device__ __forceinline__ void mul_w(uint32_t &d0, uint32_t &d1, uint32_t a, uint32_t b) {
    uint64_t p = (uint64_t)a * b;
    d0 = (uint32_t)p;
    d1 = (uint32_t)(p >> 32);
}

// ---------------------------------------------------------------- instance geometry

template <int S_, int TPI_>
struct Geom {
    static constexpr int S = S_;
    static constexpr int TPI = TPI_;
    static constexpr int L = S / TPI;
    static_assert(S % TPI == 0, "TPI must divide S");
    static_assert(L % 2 == 0 && L >= 2, "limbs per lane must be even");
    static_assert(TPI == 1 || TPI == 2 || TPI == 4 || TPI == 8 || TPI == 16 || TPI == 32, "TPI");
};

// Lane index inside the instance and the instance's base lane in the warp.
template <int TPI>
__device__ __forceinline__ int inst_lane() {
    return (int)(threadIdx.x & 31) & (TPI - 1);
}
template <int TPI>
__device__ __forceinline__ uint32_t inst_mask_shift() {
    return (threadIdx.x & 31) & ~(uint32_t)(TPI - 1);
}

// broadcast from lane `src` of the instance
template <int TPI>
__device__ __forceinline__ uint32_t inst_bcast(uint32_t v, int src) {
    if constexpr (TPI == 1) return v;
    else return __shfl_sync(0xffffffffu, v, src, TPI);
}
// value of lane t+1 (0 for the top lane)
template <int TPI>
__device__ __forceinline__ uint32_t from_above(uint32_t v) {
    if constexpr (TPI == 1) return 0u;
    else {
        uint32_t r = __shfl_down_sync(0xffffffffu, v, 1, TPI);
        return inst_lane<TPI>() == TPI - 1 ? 0u : r;
    }
}
// value of lane t−1 (0 for lane 0)
template <int TPI>
__device__ __forceinline__ uint32_t from_below(uint32_t v) {
    if constexpr (TPI == 1) return 0u;
    else {
        uint32_t r = __shfl_up_sync(0xffffffffu, v, 1, TPI);
        return inst_lane<TPI>() == 0 ? 0u : r;
    }
}
// per-instance bit masks of a warp-wide predicate (bit t = lane t of this instance)
template <int TPI>
__device__ __forceinline__ uint32_t inst_ballot(bool pred) {
    if constexpr (TPI == 1) return pred ? 1u : 0u;
    else {
        uint32_t b = __ballot_sync(0xffffffffu, pred);
        return (b >> inst_mask_shift<TPI>()) & ((TPI == 32) ? 0xffffffffu : ((1u << TPI) - 1u));
    }
}

// ---------------------------------------------------------------- shared-memory operand b
//
// Operand b of an instance lives in shared memory as limb pairs: pair p of
// instance k at sB[p·NI + (k ^ ((p >> 3) mod NI))] (uint2), NI = instances per
// block (a power of two).  The TPI lanes of an instance read the same pair
// (broadcast) and the instances of a warp read distinct 8-byte words
// (conflict-free LDS.64).  The XOR swizzle spreads the writes of the lanes of
// one instance (lane t owns pairs [t·L/2, (t+1)·L/2)) over distinct banks.
// It depends on the pair index ONLY, so for every operand size and for the
// plain word staging (relayout) an instance always owns the same slots —
// instances of different warps never alias.

template <int NI>
__device__ __forceinline__ int b_slot(int pair, int inst) {
    return pair * NI + (inst ^ ((pair >> 3) & (NI - 1)));
}

template <int S, int TPI>
__device__ __forceinline__ void store_b(uint2 *sB, int NI, int inst, const uint32_t (&v)[S / TPI]) {
    constexpr int L = S / TPI, NIc = 128 / TPI;
    const int t = inst_lane<TPI>();
#pragma unroll
    for (int j = 0; j < L / 2; ++j) sB[b_slot<NIc>(t * (L / 2) + j, inst)] = make_uint2(v[2 * j], v[2 * j + 1]);
    (void)NI;
}

// ---------------------------------------------------------------- CIOS core

// One CIOS step for limb pair (b_lo at iteration i, b_hi at i+1) is written
// as two calls of `step` with the E/O roles swapped.
// Returns q_i (the Montgomery quotient digit of this step).
template <int L, int TPI>
__device__ __forceinline__ uint32_t cios_step(uint32_t (&E)[L], uint32_t (&Q)[L], uint32_t &Z,
                                          const uint32_t (&A)[L], const uint32_t (&N)[L],
                                          uint32_t bi, uint32_t np, bool first) {
    const int t = inst_lane<TPI>();
    uint32_t Zn;
    if (first) {
        // E = A_even·b_i, O(Q) = A_odd·b_i
#pragma unroll
        for (int k = 0; k < L / 2; ++k) {
            mul_w(Q[2 * k], Q[2 * k + 1], A[2 * k + 1], bi);
            mul_w(E[2 * k], E[2 * k + 1], A[2 * k], bi);
        }
        Zn = 0;
    } else {
        // The one-limb shift of the previous step: the old E (now in Q) moves
        // down; its two lowest words belong to lane t−1's window.
        const uint32_t u0 = from_above<TPI>(Q[0]);
        const uint32_t u1 = from_above<TPI>(Q[1]);
        const uint32_t x = (t == 0) ? Q[1] : 0u; // lane 0: limb 0 of the new window
        E[0] = add_cc(E[0], x);
        // O = A_odd·b_i + (old E >> 2 limbs): fused shift, carry chain from E[0]
#pragma unroll
        for (int k = 0; k < L / 2 - 1; ++k)
            madc_w_cc(Q[2 * k], Q[2 * k + 1], A[2 * k + 1], bi, Q[2 * k + 2], Q[2 * k + 3]);
        madc_w_cc(Q[L - 2], Q[L - 1], A[L - 1], bi, u0, u1);
        Zn = addc(0u, 0u);
        Q[L - 1] = add_cc(Q[L - 1], Z); // old Z now sits at the top of the window
        Zn = addc(Zn, 0u);
        // E += A_even·b_i
        mad_w_cc(E[0], E[1], A[0], bi, E[0], E[1]);
#pragma unroll
        for (int k = 1; k < L / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], A[2 * k], bi, E[2 * k], E[2 * k + 1]);
        Q[L - 1] = addc_cc(Q[L - 1], 0u);
        Zn = addc(Zn, 0u);
    }
    // q_i from limb 0 (lane 0 only holds it), broadcast to the instance
    const uint32_t q = inst_bcast<TPI>(E[0] * np, 0);
    // O += N_odd·q
    mad_w_cc(Q[0], Q[1], N[1], q, Q[0], Q[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(Q[2 * k], Q[2 * k + 1], N[2 * k + 1], q, Q[2 * k], Q[2 * k + 1]);
    Zn = addc(Zn, 0u);
    // E += N_even·q   (limb 0 of lane 0 becomes 0)
    mad_w_cc(E[0], E[1], N[0], q, E[0], E[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], N[2 * k], q, E[2 * k], E[2 * k + 1]);
    Q[L - 1] = addc_cc(Q[L - 1], 0u);
    Z = addc(Zn, 0u);
    return q;
}

// CIOS step of the two-product pass: acc += A·b_i + C·d_i, then q_i·M and
// the shift (cios_step with a second E/O chain pair; the accumulator stays
// below 3M, its extra bit lives in Z).
template <int L, int TPI>
__device__ __forceinline__ void cios_step2(uint32_t (&E)[L], uint32_t (&Q)[L], uint32_t &Z,
                                           const uint32_t (&A)[L], const uint32_t (&C)[L], const uint32_t (&N)[L],
                                           uint32_t bi, uint32_t di, uint32_t np) {
    const int t = inst_lane<TPI>();
    uint32_t Zn;
    const uint32_t u0 = from_above<TPI>(Q[0]);
    const uint32_t u1 = from_above<TPI>(Q[1]);
    const uint32_t x = (t == 0) ? Q[1] : 0u;
    E[0] = add_cc(E[0], x);
#pragma unroll
    for (int k = 0; k < L / 2 - 1; ++k)
        madc_w_cc(Q[2 * k], Q[2 * k + 1], A[2 * k + 1], bi, Q[2 * k + 2], Q[2 * k + 3]);
    madc_w_cc(Q[L - 2], Q[L - 1], A[L - 1], bi, u0, u1);
    Zn = addc(0u, 0u);
    Q[L - 1] = add_cc(Q[L - 1], Z);
    Zn = addc(Zn, 0u);
    // O += C_odd·d_i
    mad_w_cc(Q[0], Q[1], C[1], di, Q[0], Q[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(Q[2 * k], Q[2 * k + 1], C[2 * k + 1], di, Q[2 * k], Q[2 * k + 1]);
    Zn = addc(Zn, 0u);
    // E += A_even·b_i
    mad_w_cc(E[0], E[1], A[0], bi, E[0], E[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], A[2 * k], bi, E[2 * k], E[2 * k + 1]);
    Q[L - 1] = addc_cc(Q[L - 1], 0u);
    Zn = addc(Zn, 0u);
    // E += C_even·d_i
    mad_w_cc(E[0], E[1], C[0], di, E[0], E[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], C[2 * k], di, E[2 * k], E[2 * k + 1]);
    Q[L - 1] = addc_cc(Q[L - 1], 0u);
    Zn = addc(Zn, 0u);
    const uint32_t q = inst_bcast<TPI>(E[0] * np, 0);
    mad_w_cc(Q[0], Q[1], N[1], q, Q[0], Q[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(Q[2 * k], Q[2 * k + 1], N[2 * k + 1], q, Q[2 * k], Q[2 * k + 1]);
    Zn = addc(Zn, 0u);
    mad_w_cc(E[0], E[1], N[0], q, E[0], E[1]);
#pragma unroll
    for (int k = 1; k < L / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], N[2 * k], q, E[2 * k], E[2 * k + 1]);
    Q[L - 1] = addc_cc(Q[L - 1], 0u);
    Z = addc(Zn, 0u);
}

// Carry-lookahead across the instance's lanes: lane t adds 1 if a carry
// reaches it.  g = lane generates a carry out, p = lane propagates (all ones).
// Returns the carry out of the top lane.
template <int L, int TPI>
__device__ __forceinline__ uint32_t resolve_carries(uint32_t (&R)[L], uint32_t g) {
    if constexpr (TPI == 1) {
        return g;
    } else {
        bool all_ones = true;
#pragma unroll
        for (int k = 0; k < L; ++k) all_ones &= (R[k] == 0xffffffffu);
        const uint32_t G = inst_ballot<TPI>(g != 0);
        const uint32_t P = inst_ballot<TPI>(all_ones);
        const uint64_t sum = (uint64_t)P + ((uint64_t)G << 1);
        const uint32_t cin = (uint32_t)(sum ^ P);
        if ((cin >> inst_lane<TPI>()) & 1u) {
            R[0] = add_cc(R[0], 1u);
#pragma unroll
            for (int k = 1; k < L; ++k) R[k] = addc_cc(R[k], 0u);
        }
        return (uint32_t)(sum >> TPI) & 1u;
    }
}

// Canonicalise: V = R + over·2^(32S) with V < 2M; return V mod M in R.
// Returns whether M was subtracted (instance-uniform).
template <int L, int TPI>
__device__ __forceinline__ bool final_sub(uint32_t (&R)[L], uint32_t over, const uint32_t (&N)[L]) {
    uint32_t D[L];
    D[0] = sub_cc(R[0], N[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) D[k] = subc_cc(R[k], N[k]);
    uint32_t bout = subc(0u, 0u) & 1u; // 1 when this lane borrowed
    uint32_t top_borrow;
    if constexpr (TPI == 1) {
        top_borrow = bout;
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
        top_borrow = (uint32_t)(sum >> TPI) & 1u;
    }
    // V >= M  <=>  overflow word set, or R − N did not borrow out of the top
    const bool ge = over != 0 || top_borrow == 0;
#pragma unroll
    for (int k = 0; k < L; ++k) R[k] = ge ? D[k] : R[k];
    return ge;
}

// V = R + over·2^(32S) (over small): subtract M once when V >= M, keeping
// the overflow word (the two-product pass ends below 3M).
template <int L, int TPI>
__device__ __forceinline__ void cond_sub_wide(uint32_t (&R)[L], uint32_t &over, const uint32_t (&N)[L]) {
    uint32_t D[L];
    D[0] = sub_cc(R[0], N[0]);
#pragma unroll
    for (int k = 1; k < L; ++k) D[k] = subc_cc(R[k], N[k]);
    uint32_t bout = subc(0u, 0u) & 1u;
    uint32_t top_borrow;
    if constexpr (TPI == 1) {
        top_borrow = bout;
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
        top_borrow = (uint32_t)(sum >> TPI) & 1u;
    }
    const bool ge = over != 0 || top_borrow == 0;
#pragma unroll
    for (int k = 0; k < L; ++k) R[k] = ge ? D[k] : R[k];
    over = ge ? over - top_borrow : over;
}

// The end of a CIOS pass: after the last step E = Y (the old even array,
// still unshifted) and X holds the odd-aligned array, which becomes the
// even-aligned window; Y shifts down one limb: window limb k = X[k] + Y[k+1]
// (+ lane t+1's Y[0]).  Then carries across lanes and the final conditional
// subtraction; returns whether M was subtracted.
template <int L, int TPI, bool WIDE = false>
__device__ __forceinline__ bool mont_tail(uint32_t (&r)[L], const uint32_t (&X)[L], const uint32_t (&Y)[L],
                                          uint32_t Z, const uint32_t (&N)[L]) {
    const uint32_t u0 = from_above<TPI>(Y[0]);
    uint32_t R[L];
    R[0] = add_cc(X[0], Y[1]);
#pragma unroll
    for (int k = 1; k < L - 1; ++k) R[k] = addc_cc(X[k], Y[k + 1]);
    R[L - 1] = addc_cc(X[L - 1], u0);
    uint32_t C = addc(Z, 0u); // carry word at position t·L+L (into lane t+1)
    uint32_t over;
    if constexpr (TPI == 1) {
        over = C;
    } else {
        const uint32_t cin = from_below<TPI>(C);
        const uint32_t ctop = inst_bcast<TPI>(C, TPI - 1);
        R[0] = add_cc(R[0], cin);
#pragma unroll
        for (int k = 1; k < L; ++k) R[k] = addc_cc(R[k], 0u);
        uint32_t c2 = addc(0u, 0u);
        uint32_t ripple = resolve_carries<L, TPI>(R, c2);
        over = ctop + ripple;
    }
    if constexpr (WIDE) cond_sub_wide<L, TPI>(R, over, N); // < 3M -> < 2M
    const bool ge = final_sub<L, TPI>(R, over, N);
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = R[k];
    return ge;
}

// r = A·B·2^(−32S) mod M.  A, N: this lane's L limbs; B: instance operand in
// shared memory (store_b layout); np = −M⁻¹ mod 2^32.  r may alias A.
//
// All S iterations run the same (non-peeled) step on a zero-initialised
// accumulator, and the pair loop is unrolled by L/2: one trip of the
// unrolled body rotates both accumulator arrays through all L/2 register
// pairs, so the per-step limb shift is pure register renaming (no MOVs
// competing with IMAD.WIDE for the FMA-heavy pipe).
template <int S, int TPI>
__device__ __forceinline__ void mont_mul(uint32_t (&r)[S / TPI], const uint32_t (&A)[S / TPI],
                                         const uint2 *sB, int NI, int inst,
                                         const uint32_t (&N)[S / TPI], uint32_t np) {
    constexpr int L = S / TPI;
    constexpr int U = (L / 2 <= S / 2 && (S / 2) % (L / 2) == 0) ? L / 2 : 1;
    uint32_t X[L], Y[L], Z = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) X[k] = Y[k] = 0;
    constexpr int NIc = 128 / TPI;
#pragma unroll U
    for (int i = 0; i < S / 2; ++i) {
        const uint2 b = sB[b_slot<NIc>(i, inst)];
        cios_step<L, TPI>(X, Y, Z, A, N, b.x, np, false);
        cios_step<L, TPI>(Y, X, Z, A, N, b.y, np, false);
    }
    mont_tail<L, TPI>(r, X, Y, Z, N);
}

// mont_mul that also returns the quotient m = Σ q_i·2^(32i) of the pass
// (lane t receives limbs [t·L, t·L+L) in Mq) and whether the final
// subtraction happened:  A·B = (r + ge·M)·2^(32S) − m·M  exactly.
// With capture == false, Mq is left untouched (one call site can serve
// passes with and without the quotient).
template <int S, int TPI>
__device__ __forceinline__ bool mont_mul_m(uint32_t (&r)[S / TPI], uint32_t (&Mq)[S / TPI],
                                           const uint32_t (&A)[S / TPI], const uint2 *sB, int inst,
                                           const uint32_t (&N)[S / TPI], uint32_t np, bool capture = true) {
    constexpr int L = S / TPI, NIc = 128 / TPI;
    const int t = inst_lane<TPI>();
    uint32_t X[L], Y[L], Z = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) X[k] = Y[k] = 0;
    for (int tr = 0; tr < TPI; ++tr) {
#pragma unroll
        for (int j = 0; j < L / 2; ++j) {
            const uint2 b = sB[b_slot<NIc>(tr * (L / 2) + j, inst)];
            const uint32_t q0 = cios_step<L, TPI>(X, Y, Z, A, N, b.x, np, false);
            const uint32_t q1 = cios_step<L, TPI>(Y, X, Z, A, N, b.y, np, false);
            if (capture && tr == t) {
                Mq[2 * j] = q0;
                Mq[2 * j + 1] = q1;
            }
        }
    }
    return mont_tail<L, TPI>(r, X, Y, Z, N);
}

// mont_mul that, when `sub`, also subtracts the pass's quotient
// m = Σ q_i·2^(32i) from V in place (V − m mod 2^(32S), final borrow in
// `borrow`) instead of storing m: A·B = (r + ge·M)·2^(32S) − m·M exactly.
// Returns ge.  (The digit arithmetic of padic.cuh only needs V − m.)
template <int S, int TPI>
__device__ __forceinline__ bool mont_mul_sub(uint32_t (&r)[S / TPI], uint32_t (&V)[S / TPI],
                                             const uint32_t (&A)[S / TPI], const uint2 *sB, int inst,
                                             const uint32_t (&N)[S / TPI], uint32_t np, bool sub,
                                             uint32_t &borrow) {
    constexpr int L = S / TPI, NIc = 128 / TPI;
    const int t = inst_lane<TPI>();
    uint32_t X[L], Y[L], Z = 0, bw = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) X[k] = Y[k] = 0;
    for (int tr = 0; tr < TPI; ++tr) {
#pragma unroll
        for (int j = 0; j < L / 2; ++j) {
            const uint2 b = sB[b_slot<NIc>(tr * (L / 2) + j, inst)];
            const uint32_t q0 = cios_step<L, TPI>(X, Y, Z, A, N, b.x, np, false);
            const uint32_t q1 = cios_step<L, TPI>(Y, X, Z, A, N, b.y, np, false);
            if (sub && tr == t) {
                const uint64_t d0 = (uint64_t)V[2 * j] - q0 - bw;
                V[2 * j] = (uint32_t)d0;
                const uint64_t d1 = (uint64_t)V[2 * j + 1] - q1 - (uint32_t)(d0 >> 63);
                V[2 * j + 1] = (uint32_t)d1;
                bw = (uint32_t)(d1 >> 63);
            }
        }
        if constexpr (TPI > 1) bw = __shfl_sync(0xffffffffu, bw, tr, TPI); // lane tr's borrow moves on
    }
    borrow = bw;
    return mont_tail<L, TPI>(r, X, Y, Z, N);
}

// r = (A·B + C·D)·2^(−32S) mod M with A, C < M in registers and B, D staged
// in shared memory (sB, sD; store_b layout): one CIOS pass with two products
// per step — 3S²+S products instead of 2·(2S²+S) for two passes.
template <int S, int TPI>
__device__ __forceinline__ void mont_mul2(uint32_t (&r)[S / TPI], const uint32_t (&A)[S / TPI],
                                          const uint32_t (&C)[S / TPI], const uint2 *sB, const uint2 *sD, int inst,
                                          const uint32_t (&N)[S / TPI], uint32_t np) {
    constexpr int L = S / TPI, NIc = 128 / TPI;
    constexpr int U = L / 2;
    uint32_t X[L], Y[L], Z = 0;
#pragma unroll
    for (int k = 0; k < L; ++k) X[k] = Y[k] = 0;
#pragma unroll U
    for (int i = 0; i < S / 2; ++i) {
        const uint2 b = sB[b_slot<NIc>(i, inst)];
        const uint2 d = sD[b_slot<NIc>(i, inst)];
        cios_step2<L, TPI>(X, Y, Z, A, C, N, b.x, d.x, np);
        cios_step2<L, TPI>(Y, X, Z, A, C, N, b.y, d.y, np);
    }
    mont_tail<L, TPI, true>(r, X, Y, Z, N);
}

// ---------------------------------------------------------------- squaring (one lane per instance)
//
// r = a²·2^(−32S) mod M, CIOS with the symmetric products taken once: step i
// adds a_i·(a_i·B^i + 2·Σ_{j>i} a_j·B^j) (relative positions j ≥ i of the
// shifted accumulator) instead of a·a_i, then q_i·M and the shift as in
// cios_step.  Requires a < M/2 (sqr_operand flips a to M − a otherwise:
// (M − a)² ≡ a²), so 2a fits S limbs and each row stays below M·B — the
// CIOS bound acc < 2M holds and the result is the same canonical residue as
// mont_mul(a, a).  Products: S(S+1)/2 + S² + S instead of 2S² + S (24% fewer
// at S = 32).  Positions j < i carry no product; there the shift of the odd
// array is plain moves with carry (ALU pipe).  Fully unrolled (the row start
// is a compile-time constant in every step).
//
// D[j] = limb j of 2a = (a_j << 1) | (a_{j−1} >> 31); the row's limb at
// j = i + 1 is a_{i+1} << 1 (a_i's top bit belongs to position i... of 2a but
// to no term of the row: 2·a_{i+1}·B^{i+1} has only a_{i+1}'s bits).
template <int S>
__device__ __forceinline__ uint32_t sqr_step(uint32_t (&E)[S], uint32_t (&Q)[S], uint32_t &Z, const uint32_t (&a)[S],
                                             const uint32_t (&D)[S], const uint32_t (&N)[S], uint32_t np, const int i) {
    const uint32_t bi = a[i];
    auto op = [&](int j) -> uint32_t { return j == i ? a[i] : (j == i + 1 ? (a[j] << 1) : D[j]); };
    uint32_t Zn;
    // shift of the previous step fused with the odd products (j odd)
    E[0] = add_cc(E[0], Q[1]);
#pragma unroll
    for (int k = 0; k < S / 2 - 1; ++k) {
        if (2 * k + 1 < i) {
            Q[2 * k] = addc_cc(Q[2 * k + 2], 0u);
            Q[2 * k + 1] = addc_cc(Q[2 * k + 3], 0u);
        } else {
            madc_w_cc(Q[2 * k], Q[2 * k + 1], op(2 * k + 1), bi, Q[2 * k + 2], Q[2 * k + 3]);
        }
    }
    madc_w_cc(Q[S - 2], Q[S - 1], op(S - 1), bi, 0u, 0u);
    Zn = addc(0u, 0u);
    Q[S - 1] = add_cc(Q[S - 1], Z);
    Zn = addc(Zn, 0u);
    // even products (j even, j >= i)
    const int k0 = (i + 1) / 2;
    if (k0 < S / 2) {
        mad_w_cc(E[2 * k0], E[2 * k0 + 1], op(2 * k0), bi, E[2 * k0], E[2 * k0 + 1]);
#pragma unroll
        for (int k = k0 + 1; k < S / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], op(2 * k), bi, E[2 * k], E[2 * k + 1]);
        Q[S - 1] = addc_cc(Q[S - 1], 0u);
        Zn = addc(Zn, 0u);
    }
    const uint32_t q = E[0] * np;
    mad_w_cc(Q[0], Q[1], N[1], q, Q[0], Q[1]);
#pragma unroll
    for (int k = 1; k < S / 2; ++k) madc_w_cc(Q[2 * k], Q[2 * k + 1], N[2 * k + 1], q, Q[2 * k], Q[2 * k + 1]);
    Zn = addc(Zn, 0u);
    mad_w_cc(E[0], E[1], N[0], q, E[0], E[1]);
#pragma unroll
    for (int k = 1; k < S / 2; ++k) madc_w_cc(E[2 * k], E[2 * k + 1], N[2 * k], q, E[2 * k], E[2 * k + 1]);
    Q[S - 1] = addc_cc(Q[S - 1], 0u);
    Z = addc(Zn, 0u);
    return q;
}

// a' = min(a, M − a) for a < M (same square mod M, a' < M/2); returns
// whether a was replaced
template <int S>
__device__ __forceinline__ bool sqr_operand(uint32_t (&r)[S], const uint32_t (&a)[S], const uint32_t (&N)[S]) {
    uint32_t d[S];
    d[0] = sub_cc(N[0], a[0]);
#pragma unroll
    for (int k = 1; k < S; ++k) d[k] = subc_cc(N[k], a[k]);
    // M − a < a  <=>  a − (M − a) does not borrow and is nonzero; M odd, so
    // a − (M − a) = 2a − M is never 0
    uint32_t t = sub_cc(a[0], d[0]);
#pragma unroll
    for (int k = 1; k < S; ++k) t = subc_cc(a[k], d[k]);
    const bool flip = (subc(0u, 0u) & 1u) == 0;
    (void)t;
#pragma unroll
    for (int k = 0; k < S; ++k) r[k] = flip ? d[k] : a[k];
    return flip;
}

// r = a²·2^(−32S) mod M (a < M); with `sub`, also V −= m (mod 2^(32S),
// final borrow in `borrow`), m = Σ q_i·2^(32i) the pass's quotient, as
// mont_mul_sub — for the operand actually squared (a or M − a, *flipped).
// Returns ge (M subtracted at the end): a'·a' = (r + ge·M)·2^(32S) − m·M.
template <int S>
__device__ __forceinline__ bool mont_sqr_sub(uint32_t (&r)[S], uint32_t (&V)[S], const uint32_t (&a_in)[S],
                                             const uint32_t (&N)[S], uint32_t np, bool sub, uint32_t &borrow,
                                             bool &flipped) {
    uint32_t a[S], D[S];
    flipped = sqr_operand<S>(a, a_in, N);
    D[0] = a[0] << 1;
#pragma unroll
    for (int k = 1; k < S; ++k) D[k] = (a[k] << 1) | (a[k - 1] >> 31);
    uint32_t X[S], Y[S], Z = 0, bw = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) X[k] = Y[k] = 0;
#pragma unroll
    for (int i = 0; i < S; i += 2) {
        const uint32_t q0 = sqr_step<S>(X, Y, Z, a, D, N, np, i);
        const uint32_t q1 = sqr_step<S>(Y, X, Z, a, D, N, np, i + 1);
        if (sub) {
            const uint64_t d0 = (uint64_t)V[i] - q0 - bw;
            V[i] = (uint32_t)d0;
            const uint64_t d1 = (uint64_t)V[i + 1] - q1 - (uint32_t)(d0 >> 63);
            V[i + 1] = (uint32_t)d1;
            bw = (uint32_t)(d1 >> 63);
        }
    }
    borrow = bw;
    return mont_tail<S, 1>(r, X, Y, Z, N);
}

template <int S>
__device__ __forceinline__ void mont_sqr(uint32_t (&r)[S], const uint32_t (&a)[S], const uint32_t (&N)[S],
                                         uint32_t np) {
    uint32_t V[S], bw;
    bool fl;
    mont_sqr_sub<S>(r, V, a, N, np, false, bw, fl);
}

// ---------------------------------------------------------------- global <-> lane limbs

template <int S, int TPI>
__device__ __forceinline__ void load_lane(uint32_t (&v)[S / TPI], const uint32_t *g) {
    constexpr int L = S / TPI;
    const uint32_t *p = g + inst_lane<TPI>() * L;
    if constexpr (L % 4 == 0) {
#pragma unroll
        for (int k = 0; k < L / 4; ++k) {
            uint4 w = reinterpret_cast<const uint4 *>(p)[k];
            v[4 * k] = w.x;
            v[4 * k + 1] = w.y;
            v[4 * k + 2] = w.z;
            v[4 * k + 3] = w.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < L / 2; ++k) {
            uint2 w = reinterpret_cast<const uint2 *>(p)[k];
            v[2 * k] = w.x;
            v[2 * k + 1] = w.y;
        }
    }
}

template <int S, int TPI>
__device__ __forceinline__ void store_lane(uint32_t *g, const uint32_t (&v)[S / TPI]) {
    constexpr int L = S / TPI;
    uint32_t *p = g + inst_lane<TPI>() * L;
    if constexpr (L % 4 == 0) {
#pragma unroll
        for (int k = 0; k < L / 4; ++k)
            reinterpret_cast<uint4 *>(p)[k] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < L / 2; ++k) reinterpret_cast<uint2 *>(p)[k] = make_uint2(v[2 * k], v[2 * k + 1]);
    }
}

// lane limbs of a small constant (value v at limb 0)
template <int L, int TPI>
__device__ __forceinline__ void set_small(uint32_t (&r)[L], uint32_t v) {
#pragma unroll
    for (int k = 0; k < L; ++k) r[k] = 0;
    if (inst_lane<TPI>() == 0) r[0] = v;
}

// instance-wide equality with a small constant
template <int L, int TPI>
__device__ __forceinline__ bool eq_small(const uint32_t (&r)[L], uint32_t v) {
    bool ok = true;
    const bool l0 = inst_lane<TPI>() == 0;
#pragma unroll
    for (int k = 0; k < L; ++k) ok &= (r[k] == ((l0 && k == 0) ? v : 0u));
    return inst_ballot<TPI>(!ok) == 0;
}

} // namespace dev
} // namespace sfxb
