// libsfxb_cuda.so: key contexts, launch logic and the C ABI (include/sfxb_cuda.h).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>

#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/sfxb_cuda.h"
#include "bignum_host.hpp"
#include "ctx.hpp"
#include "hist.cuh"
#include "kernels.cuh"
#include "padic.cuh"

#include <cub/cub.cuh>

using namespace sfxb;
using sfxb::host::Big;

namespace sfxb {
namespace host {
namespace {
// the GMP ABI subset used for inversion (x86-64 GMP 6: 64-bit limbs)
struct GmpMpz {
    int alloc, size;
    void *d;
};
struct GmpApi {
    void (*init)(GmpMpz *) = nullptr;
    void (*clear)(GmpMpz *) = nullptr;
    void (*import_)(GmpMpz *, size_t, int, size_t, int, size_t, const void *) = nullptr;
    void *(*export_)(void *, size_t *, int, size_t, int, size_t, const GmpMpz *) = nullptr;
    int (*invert)(GmpMpz *, const GmpMpz *, const GmpMpz *) = nullptr;
    bool ok = false;
    GmpApi() {
        void *h = dlopen("libgmp.so.10", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        init = (decltype(init))dlsym(h, "__gmpz_init");
        clear = (decltype(clear))dlsym(h, "__gmpz_clear");
        import_ = (decltype(import_))dlsym(h, "__gmpz_import");
        export_ = (decltype(export_))dlsym(h, "__gmpz_export");
        invert = (decltype(invert))dlsym(h, "__gmpz_invert");
        ok = init && clear && import_ && export_ && invert;
    }
};
const GmpApi &gmp() {
    static GmpApi api;
    return api;
}
} // namespace

bool inv_mod_fast(const Big &x, const Big &M, Big &out) {
    const GmpApi &g = gmp();
    if (!g.ok) return inv_mod_odd(x, M, out);
    GmpMpz a, m, r;
    g.init(&a);
    g.init(&m);
    g.init(&r);
    g.import_(&a, x.size(), -1, 4, 0, 0, x.data());
    g.import_(&m, M.size(), -1, 4, 0, 0, M.data());
    const int ok = g.invert(&r, &a, &m);
    if (ok) {
        out.assign(M.size() + 1, 0);
        size_t cnt = 0;
        g.export_(out.data(), &cnt, -1, 4, 0, 0, &r);
        trim(out);
    }
    g.clear(&a);
    g.clear(&m);
    g.clear(&r);
    return ok != 0;
}
} // namespace host
} // namespace sfxb

struct sfxb_ctx : CtxState {};
// Queue of precomputed blinding powers r^n mod n² (device, 4s-limb stride),
// in the order their r were drawn.
struct sfxb_blind {
    int device = 0;
    uint32_t s = 0, nw = 0;
    uint64_t key_id = 0;
    uint32_t *d = nullptr;
    size_t cap = 0, head = 0, size = 0; // live entries [head, head + size)
};
// Device-resident bin columns (n_features × n_samples u16, column-major)
struct sfxb_bins {
    const sfxb_ctx *ctx = nullptr;
    uint32_t J = 0, n = 0;
    uint16_t *d = nullptr;
};
struct sfxb_gh {
    sfxb_ctx *ctx = nullptr;
    uint32_t *d = nullptr;     // 2·n_samples × 4s limbs, Montgomery form
    uint8_t *flags = nullptr;  // per row: bit0 Enc(g) == 1, bit1 Enc(h) == 1
    uint32_t n_samples = 0;
    bool digits = false;       // key holder: [A_p | B_p | A_q | B_q] digits instead (padic.cuh K2)
    bool digits_n = false;     // passive party: [A | B] base-n digits of the Montgomery form
    size_t bytes = 0, fbytes = 0;
    // device group: one handle per shard holding rows [row_lo[k], row_lo[k+1])
    std::vector<sfxb_gh *> parts;
    std::vector<uint32_t> row_lo;
};

namespace {

thread_local std::string g_create_err;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess)                                                                     \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                      \
    } while (0)

// NVTX range over one C ABI call (visible in Nsight Systems / ncu NVTX
// filters; header-only NVTX 3, no cost without an attached tool)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

template <typename F>
int guard(sfxb_ctx *ctx, F &&f) {
    try {
        f();
        return SFXB_OK;
    } catch (const ApiError &e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const CudaError &e) {
        if (ctx) ctx->err = e.what();
        return SFXB_ERR_CUDA;
    } catch (const std::exception &e) {
        if (ctx) ctx->err = e.what();
        return SFXB_ERR_ARG;
    }
}

// --------------------------------------------------------------- device memory helpers

template <typename T>
T *dev_upload(CtxState &c, const T *h, size_t n) {
    T *d = nullptr;
    CK(cudaMalloc(&d, n * sizeof(T) + 16));
    CK(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice));
    c.owned.push_back(d);
    return d;
}
uint32_t *dev_big(CtxState &c, const Big &v, size_t words) {
    Big p = host::pad(v, words);
    return dev_upload(c, p.data(), words);
}
DevMod dev_mod(CtxState &c, const Big &m, int S) {
    host::MontHost mh(m, S);
    std::vector<uint32_t> w(4 * (size_t)S);
    std::copy(mh.m.begin(), mh.m.end(), w.begin());
    std::copy(mh.r1.begin(), mh.r1.end(), w.begin() + S);
    std::copy(mh.r2.begin(), mh.r2.end(), w.begin() + 2 * S);
    std::copy(mh.r3.begin(), mh.r3.end(), w.begin() + 3 * S);
    DevMod d;
    d.w = dev_upload(c, w.data(), w.size());
    d.np = mh.np;
    d.S = S;
    return d;
}
uint8_t *dev_digits(CtxState &c, const Big &e, int w, int &nd) {
    std::vector<uint8_t> d = host::window_digits(e, w);
    nd = (int)d.size();
    return dev_upload(c, d.data(), d.size());
}
// Montgomery multiplications of mont_pow for exponent e at window w (modexp.cuh:206):
// table build, w squarings per digit after the first, one multiply per non-zero digit
uint64_t pow_mmuls(const Big &e, int w) {
    std::vector<uint8_t> d = host::window_digits(e, w);
    uint64_t m = (1u << w) - 2 + (uint64_t)(d.size() - 1) * w;
    for (size_t i = 1; i < d.size(); ++i) m += d[i] != 0;
    return m;
}
// Grow-only device buffer.  The old allocation is released first (the new
// one is usually larger than what is left); the size is recorded only once
// the new allocation exists, so a failed cudaMalloc (OOM) leaves an empty
// buffer that the next call allocates again, never a null pointer that
// claims capacity.
void *grow(Buf &b, size_t bytes) {
    if (b.bytes < bytes) {
        void *old = b.p;
        b.p = nullptr;
        b.bytes = 0;
        if (old) CK(cudaFree(old));
        void *p = nullptr;
        const cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            (void)cudaGetLastError(); // an allocation failure is not sticky: clear it
            throw CudaError(std::string("cudaMalloc of ") + std::to_string(bytes) + " bytes: " + cudaGetErrorString(e));
        }
        b.p = p;
        b.bytes = bytes;
    }
    return b.p;
}

dev::ModArg arg(const DevMod &m) { return dev::ModArg{m.w, m.np}; }

// --------------------------------------------------------------- size classes
//
// Tuned TPI (lanes per instance) per kernel and class.  S = limbs of the
// modulus of that kernel: step1 s, step2 2s, histogram / ct-add 4s.
template <int s>
struct Cls;
// TP: p2_pow (mod-p² exponentiation on base-p digits, S = s); TQ: its
// mod-p² pre/post conversions (S = 2s)
template <>
struct Cls<4> {
    static constexpr int T1 = 1, T2 = 1, TC = 1, TD = 1, TE = 1, TH = 1, TN = 1, TP = 1, TQ = 1, TND = 1, TK = 1;
};
template <>
struct Cls<8> {
    static constexpr int T1 = 1, T2 = 1, TC = 2, TD = 1, TE = 1, TH = 2, TN = 2, TP = 1, TQ = 2, TND = 1, TK = 1;
};
template <>
struct Cls<16> {
    static constexpr int T1 = 1, T2 = 2, TC = 4, TD = 2, TE = 2, TH = 4, TN = 4, TP = 1, TQ = 4, TND = 2, TK = 1;
};
#ifndef SFXB_T1_32
#define SFXB_T1_32 1
#endif
#ifndef SFXB_T2_32
#define SFXB_T2_32 4
#endif
#ifndef SFXB_TD_32
#define SFXB_TD_32 2
#endif
#ifndef SFXB_TH_32
#define SFXB_TH_32 4
#endif
#ifndef SFXB_TP_32
#define SFXB_TP_32 1
#endif
#ifndef SFXB_TK_32
#define SFXB_TK_32 1
#endif
#ifndef SFXB_TND_32
#define SFXB_TND_32 4
#endif
template <>
struct Cls<32> { // 2048-bit keys (tuned on B200, profiles/)
    static constexpr int T1 = SFXB_T1_32, T2 = SFXB_T2_32, TC = 8, TD = SFXB_TD_32, TE = 4, TH = SFXB_TH_32, TN = 8,
                         TP = SFXB_TP_32, TQ = 4, TND = SFXB_TND_32, TK = SFXB_TK_32;
};
// 3072-bit: encrypt step 1 at one lane and the digit exponentiation at two
// lanes per instance — 123K → 142K enc/s and 176K → 197K dec/s against 2 / 4
// lanes (profiles/r02_ab_3072.jsonl)
#ifndef SFXB_T1_48
#define SFXB_T1_48 1
#endif
#ifndef SFXB_TP_48
#define SFXB_TP_48 2
#endif
template <>
struct Cls<48> { // 3072-bit keys
    static constexpr int T1 = SFXB_T1_48, T2 = 4, TC = 8, TD = 4, TE = 8, TH = 8, TN = 8, TP = SFXB_TP_48, TQ = 8,
                         TND = 4, TK = 4;
};

// lanes per instance of the gh conversions (key holder's CRT digits, passive
// party's base-n digits): the class's TQ / TND, 2 at 2048 bits (bench A/B,
// 0.4579 -> 0.4554 / 0.4562 s/tree: fewer lanes, fewer shuffles, some spills)
template <typename C>
constexpr int kTG = C::TQ;
template <typename C>
constexpr int kTGN = C::TND;
#ifndef SFXB_TG_32
#define SFXB_TG_32 2
#endif
#ifndef SFXB_TGN_32
#define SFXB_TGN_32 2
#endif
template <>
constexpr int kTG<Cls<32>> = SFXB_TG_32;
template <>
constexpr int kTGN<Cls<32>> = SFXB_TGN_32;

// grid.x for `items` work items spread over `rows` block rows (grid.y)
template <typename K>
int occupancy_grid(CtxState &c, K kernel, size_t items, int NI, int rows = 1) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, dev::kBlock, 0));
    if (per_sm < 1) per_sm = 1;
    size_t want = (items + (size_t)NI * rows - 1) / ((size_t)NI * rows);
    size_t cap = std::max<size_t>(1, (size_t)c.sms * per_sm / rows);
    if (want < 1) want = 1;
    return (int)std::min(want, cap);
}

template <typename Fn>
void dispatch_class(int s, Fn &&fn) {
    switch (s) {
    case 4: fn(std::integral_constant<int, 4>{}); break;
    case 8: fn(std::integral_constant<int, 8>{}); break;
    case 16: fn(std::integral_constant<int, 16>{}); break;
    case 32: fn(std::integral_constant<int, 32>{}); break;
    case 48: fn(std::integral_constant<int, 48>{}); break;
    default: throw ApiError(SFXB_ERR_UNSUPPORTED, "unsupported key size class");
    }
}

void check_launch(CtxState &c) {
    CK(cudaGetLastError());
    c.launches++;
}

// Brackets a launch with events on the context stream when profiling is on.
struct ProfScope {
    CtxState &c;
    int fam;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(CtxState &c_, int fam_, uint64_t modmuls = 0) : c(c_), fam(fam_) {
        if (!c.profile) return;
        c.prof[fam].modmuls += modmuls;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, c.stream));
    }
    ~ProfScope() {
        if (!c.profile || !a) return;
        cudaEventRecord(b, c.stream);
        c.prof[fam].ev.emplace_back(a, b);
        c.prof[fam].launches++;
    }
};

// --------------------------------------------------------------- encrypt

// Items per k_p2_pow launch: SFXB_P2_WAVES whole waves (default 1; a wave =
// the items one launch of `grid` resident blocks holds at once; 0 = a single
// launch).  Every warp of a launch then runs the same exponentiation program
// once, in step: with many items per thread the warps of an SM drift apart
// into different parts of the (fully unrolled, ~100 KB) program, and the
// instruction cache no longer holds what they execute — one launch over 4M
// encryptions ran 14% slower per item than one-wave launches
// (profiles/r02_ab_chunk.jsonl).
size_t p2_chunk(size_t count, size_t wave) {
    static const long v = std::getenv("SFXB_P2_WAVES") ? std::atol(std::getenv("SFXB_P2_WAVES")) : 1;
    return v > 0 ? (size_t)v * std::max<size_t>(wave, 1) : std::max<size_t>(count, 1);
}

void encrypt_dev(sfxb_ctx *c, const int64_t *d_q, const uint32_t *d_r, size_t count,
                 uint32_t *d_out, uint8_t *d_flags, const uint32_t *d_m = nullptr) {
    if (count == 0) return;
    const int s = c->s;
    const size_t S2 = 2 * (size_t)s, S4 = 4 * (size_t)s;
    dev::EncArgs a{};
    a.r = d_r;
    a.qfix = d_q;
    a.mw = d_m;
    a.count = count;
    a.mod_n2 = arg(c->mod_n2);
    a.dig_n = c->d_dig_n;
    a.nd_n = c->nd_n;
    a.n4 = c->d_n4;
    a.nR_n2 = c->d_nR_n2;
    a.out = d_out;
    a.flags = d_flags;
    uint32_t *status = (uint32_t *)grow(c->tmp[3], 64);
    CK(cudaMemsetAsync(status, 0, 4, c->stream));
    a.status = status;
    if (c->has_priv) {
        for (int i = 0; i < 2; ++i) {
            a.mod_pq[i] = arg(c->mod_pq[i]);
            a.mod_pq2[i] = arg(c->mod_pq2[i]);
            a.dig_e1[i] = c->d_dig_e1[i];
            a.nd_e1[i] = c->nd_e1[i];
            a.ops_e1[i] = c->d_ops_e1[i];
            a.nops_e1[i] = c->nops_e1[i];
            a.dig_pq[i] = c->d_dig_pq[i];
            a.nd_pq[i] = c->nd_pq[i];
        }
        a.q2R_n2 = c->d_q2R_n2;
        a.qq_inv_m = c->d_qq_inv_m;
        a.x = (uint32_t *)grow(c->tmp[0], count * 2 * S2 * 4);
        a.y = (uint32_t *)grow(c->tmp[1], count * 2 * S2 * 4);
    } else {
        a.y = (uint32_t *)grow(c->tmp[1], count * S4 * 4);
    }
    dispatch_class(s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        if (c->has_priv) {
            {
                auto k = dev::k_enc_step1<cs, C::T1, kWindow>;
                constexpr int NI = dev::kBlock / C::T1;
                int grid = occupancy_grid(*c, k, 2 * count, NI, 2);
                a.scratch = (uint32_t *)grow(c->scratch_table, 2 * (size_t)grid * NI * ((size_t)cs << kWindow) * 4);
                ProfScope prof_(*c, 1, c->prod_enc * count);
                // whole waves per launch as for k_p2_pow (SFXB_STEP1_WAVES)
                static const long waves1 =
                    std::getenv("SFXB_STEP1_WAVES") ? std::atol(std::getenv("SFXB_STEP1_WAVES")) : 0;
                const size_t chunk = waves1 > 0 ? (size_t)waves1 * grid * NI : count;
                for (size_t f = 0; f < count; f += chunk) {
                    dev::EncArgs ac = a;
                    ac.r = a.r + f * S2;
                    ac.x = a.x + f * 2 * S2;
                    ac.flags = a.flags ? a.flags + f : nullptr;
                    ac.count = std::min(chunk, count - f);
                    k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(ac);
                    check_launch(*c);
                }
            }
            if (c->p2_digits) {
                // y = x^prime mod prime² on base-prime digits (padic.cuh), then plain
                dev::P2Args pa{};
                for (int i = 0; i < 2; ++i) {
                    pa.mod_p[i] = arg(c->mod_pq[i]);
                    pa.pinv[i] = c->d_pinv[i];
                    pa.negR[i] = c->d_negR[i];
                    pa.ops[i] = c->d_ops_pq[i];
                    pa.n_ops[i] = c->nops_pq[i];
                }
                pa.in = a.x;
                pa.out = a.y;
                pa.count = count;
                {
                    auto k = dev::k_p2_pow<cs, C::TP, kWindow, 0>;
                    constexpr int NI = dev::kBlock / C::TP;
                    int grid = occupancy_grid(*c, k, 2 * count, NI, 2);
                    pa.scratch = (uint32_t *)grow(c->scratch_table,
                                                  2 * (size_t)grid * NI * ((size_t)(2 * cs) << kWindow) * 4);
                    ProfScope prof_(*c, 1);
                    const size_t chunk = p2_chunk(count, (size_t)grid * NI);
                    for (size_t f = 0; f < count; f += chunk) {
                        pa.first = f;
                        pa.count = std::min(chunk, count - f);
                        k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(pa);
                        check_launch(*c);
                    }
                }
                {
                    auto k = dev::k_enc_post<cs, C::TQ>;
                    constexpr int NI = dev::kBlock / C::TQ;
                    int grid = occupancy_grid(*c, k, 2 * count, NI, 2);
                    k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(a);
                    check_launch(*c);
                }
            } else {
                auto k = dev::k_enc_step2<2 * cs, C::T2, kWindow>;
                constexpr int NI = dev::kBlock / C::T2;
                int grid = occupancy_grid(*c, k, 2 * count, NI, 2);
                a.scratch = (uint32_t *)grow(c->scratch_table, 2 * (size_t)grid * NI * ((size_t)(2 * cs) << kWindow) * 4);
                ProfScope prof_(*c, 1);
                k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(a);
                check_launch(*c);
            }
        } else {
            auto k = dev::k_pow_n2<4 * cs, C::TN, kWindowN>;
            constexpr int NI = dev::kBlock / C::TN;
            int grid = occupancy_grid(*c, k, count, NI);
            a.scratch = (uint32_t *)grow(c->scratch_table, (size_t)grid * NI * ((size_t)(4 * cs) << kWindowN) * 4);
            k<<<grid, dev::kBlock, 0, c->stream>>>(a);
            check_launch(*c);
        }
        {
            auto k = dev::k_enc_combine<cs, C::TC>;
            constexpr int NI = dev::kBlock / C::TC;
            int grid = occupancy_grid(*c, k, count, NI);
            k<<<grid, dev::kBlock, 0, c->stream>>>(a, c->has_priv ? 1 : 0);
            check_launch(*c);
        }
    });
    uint32_t st = 0;
    CK(cudaMemcpyAsync(&st, status, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (st & 1u) throw ApiError(SFXB_ERR_COPRIME, "encrypt: blinding factor not coprime to modulus");
}

// --------------------------------------------------------------- decrypt

void decrypt_dev(sfxb_ctx *c, const uint32_t *d_cts, size_t count, uint32_t scale, double *d_values,
                 uint32_t *d_plain, uint64_t *decryptions, const uint8_t *d_skip = nullptr) {
    if (!c->has_priv) throw ApiError(SFXB_ERR_AUTH, "decrypt requested without private key material");
    if (count == 0) return;
    if (count > 0xffffffffull) throw ApiError(SFXB_ERR_ARG, "decrypt: too many slots in one call");
    const int s = c->s;
    dev::DecArgs a{};
    a.cts = d_cts;
    a.count = count;
    a.idx = (uint32_t *)grow(c->tmp[2], count * 4 + 64);
    uint32_t *misc = (uint32_t *)grow(c->tmp[3], 64);
    a.n_idx = misc + 1;
    a.status = misc;
    a.n_skipped = misc + 2;
    a.skip = d_skip;
    CK(cudaMemsetAsync(misc, 0, 12, c->stream));
    for (int i = 0; i < 2; ++i) {
        a.mod_pq[i] = arg(c->mod_pq[i]);
        a.mod_pq2[i] = arg(c->mod_pq2[i]);
        a.dig_m1[i] = c->d_dig_m1[i];
        a.nd_m1[i] = c->nd_m1[i];
        a.pinv[i] = c->d_pinv[i];
        a.hR[i] = c->d_hR[i];
    }
    a.mod_n = arg(c->mod_n);
    a.qinvR_p = c->d_qinvR_p;
    a.qR_n = c->d_qR_n;
    a.n2w = c->d_n2w;
    a.nw = c->d_n;
    a.mpq = (uint32_t *)grow(c->tmp[0], count * 2 * (size_t)s * 4);
    a.values = d_values;
    a.plain = d_plain;
    a.scale = scale;
    dispatch_class(s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        {
            int grid = (int)std::min<size_t>((count + 255) / 256, (size_t)c->sms * 8);
            dev::k_dec_scan<4 * cs><<<grid, 256, 0, c->stream>>>(a);
            check_launch(*c);
        }
        uint32_t hst[3];
        CK(cudaMemcpyAsync(hst, misc, 12, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (hst[0] & 2u) throw ApiError(SFXB_ERR_RANGE, "decrypt: ciphertext out of range");
        const uint32_t n_items = hst[1];
        // the reference's counter: every non-trivial slot (decrypted or derived)
        if (decryptions) *decryptions += (uint64_t)n_items + hst[2];
        c->dec_derived += hst[2];
        if (n_items == 0) return;
        if (c->p2_digits) {
            // X̃ = c·R² mod prime², then c^(prime−1) on base-prime digits -> m_prime
            uint32_t *xt = (uint32_t *)grow(c->tmp[1], (size_t)n_items * 2 * (2 * cs) * 4 + 64);
            ProfScope prof_(*c, 2, c->prod_dec * n_items);
            {
                auto k = dev::k_dec_pre<cs, C::TQ>;
                constexpr int NI = dev::kBlock / C::TQ;
                int grid = occupancy_grid(*c, k, 2 * (size_t)n_items, NI, 2);
                k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(a, n_items, xt);
                check_launch(*c);
            }
            dev::P2Args pa{};
            for (int i = 0; i < 2; ++i) {
                pa.mod_p[i] = arg(c->mod_pq[i]);
                pa.pinv[i] = c->d_pinv[i];
                pa.cdec[i] = c->d_cdec[i];
                pa.negR[i] = c->d_negR[i];
                pa.ops[i] = c->d_ops_m1[i];
                pa.n_ops[i] = c->nops_m1[i];
            }
            pa.in = xt;
            pa.out = a.mpq;
            pa.idx = a.idx;
            pa.count = n_items;
            pa.status = a.status;
            // items [first, first + cnt) at TPv lanes per instance
            auto launch = [&](auto tp, size_t first, size_t cnt) {
                constexpr int TPv = decltype(tp)::value;
                if (cnt == 0) return;
                auto k = dev::k_p2_pow<cs, TPv, kWindow, 1>;
                constexpr int NI = dev::kBlock / TPv;
                int grid = occupancy_grid(*c, k, 2 * cnt, NI, 2);
                pa.scratch =
                    (uint32_t *)grow(c->scratch_table, 2 * (size_t)grid * NI * ((size_t)(2 * cs) << kWindow) * 4);
                const size_t chunk = p2_chunk(cnt, (size_t)grid * NI);
                for (size_t f = 0; f < cnt; f += chunk) {
                    pa.first = first + f;
                    pa.count = std::min(chunk, cnt - f);
                    k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(pa);
                    check_launch(*c);
                }
            };
            // Whole waves of exponentiations at one lane per instance; what
            // does not fill a wave — a small batch (a tree's first levels), or
            // the last partial wave of a large one — may finish sooner at 2 or
            // 4 lanes per instance.  A one-lane wave takes ≈0.75–1.1 of a full
            // wave's time however few its jobs (latency); at 4 lanes time
            // follows the job count (≈1.15 µs per job at 2048 bits); at 2
            // lanes a wave holds half as many jobs and takes ≈0.66 of a
            // one-lane wave.  Measured at 2048 bits (tools/dec_latency.py,
            // profiles/r02_dec_latency.jsonl): 3,584 / 7,168 / 14,336 items
            // take 9.2 / 15.5 / 22.7 ms with this choice against 17.3 / 17.7 /
            // 22.7 at one lane, 9.2 / 19.7 / 32.5 at 4 lanes and 11.4 / 15.5 /
            // 30.9 at 2 lanes; 28,672 items (a wave + 51% of one) 46 ms with
            // the tail at 4 lanes against 49.5 at one and 50.9 at two.  Same
            // results in every case (SFXB_DEC_SMALL_TPI=0: one lane for all).
            bool split = false;
            if constexpr (C::TP == 1 && (cs == 16 || cs == 32)) {
                const char *e = std::getenv("SFXB_DEC_SMALL_TPI");
                if (!e || std::atoi(e) != 0) {
                    auto instances = [&](auto k, int tpv) { // concurrent (item, prime) jobs of kernel k
                        int per_sm = 0;
                        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, dev::kBlock, 0));
                        return (size_t)std::max(per_sm, 1) * c->sms * (dev::kBlock / tpv);
                    };
                    const size_t S1 = instances(dev::k_p2_pow<cs, 1, kWindow, 1>, 1);
                    const size_t S2 = instances(dev::k_p2_pow<cs, 2, kWindow, 1>, 2);
                    const size_t S4 = instances(dev::k_p2_pow<cs, 4, kWindow, 1>, 4);
                    // jobs are (item, prime); full waves of one-lane instances first
                    const size_t jobs = 2 * (size_t)n_items, full = jobs / S1 * S1;
                    const size_t bulk = full / 2, tail = n_items - bulk, J = 2 * tail;
                    int lanes = 1;
                    if (tail) {
                        if (4 * J <= 3 * S4) lanes = 4;             // a small batch: 4 lanes
                        else if (5 * J <= 4 * S2) lanes = 2;        // within one 2-lane wave
                        else if (5 * J <= 3 * S1) lanes = 4;        // up to 60% of a one-lane wave
                    }
                    if (lanes > 1) {
                        split = true;
                        launch(std::integral_constant<int, 1>{}, 0, bulk);
                        if (lanes == 4) launch(std::integral_constant<int, 4>{}, bulk, tail);
                        else launch(std::integral_constant<int, 2>{}, bulk, tail);
                    }
                }
            }
            if (!split) launch(std::integral_constant<int, C::TP>{}, 0, n_items);
        } else {
            auto k = dev::k_dec_step<cs, C::TD, kWindow>;
            constexpr int NI = dev::kBlock / C::TD;
            int grid = occupancy_grid(*c, k, 2 * (size_t)n_items, NI, 2);
            a.scratch = (uint32_t *)grow(c->scratch_table, 2 * (size_t)grid * NI * ((size_t)(2 * cs) << kWindow) * 4);
            ProfScope prof_(*c, 2, c->prod_dec * n_items);
            k<<<dim3(grid, 2), dev::kBlock, 0, c->stream>>>(a, n_items);
            check_launch(*c);
        }
        {
            auto k = dev::k_dec_combine<cs, C::TE>;
            constexpr int NI = dev::kBlock / C::TE;
            int grid = occupancy_grid(*c, k, n_items, NI);
            k<<<grid, dev::kBlock, 0, c->stream>>>(a, n_items);
            check_launch(*c);
        }
        CK(cudaMemcpyAsync(hst, misc, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (hst[0] & 4u) throw ApiError(SFXB_ERR_COPRIME, "decrypt: ciphertext not coprime to modulus");
    });
}

// --------------------------------------------------------------- ct add

void add_dev(sfxb_ctx *c, const uint32_t *d_a, const uint32_t *d_b, size_t count, uint32_t *d_out) {
    if (count == 0) return;
    dispatch_class(c->s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        auto k = dev::k_mulmod<4 * cs, C::TH>;
        constexpr int NI = dev::kBlock / C::TH;
        int grid = occupancy_grid(*c, k, count, NI);
        k<<<grid, dev::kBlock, 0, c->stream>>>(arg(c->mod_n2), d_a, d_b, d_out, count);
        check_launch(*c);
    });
}


// --------------------------------------------------------------- histogram (K2)

// items per segmented-product piece: long segments use kPieceLong (fewer
// partials / passes), short ones kPiece (less tail work)
#ifndef SFXB_PIECE_LONG
#define SFXB_PIECE_LONG 64
#endif
#ifndef SFXB_PIECE
#define SFXB_PIECE 16
#endif
constexpr int kPiece = SFXB_PIECE, kPieceLong = SFXB_PIECE_LONG;

struct HistBufs {
    Buf node_of, count, ones, cursor, seg_start, sorted, np, piece_start, pieces, part[2], cub, misc, plen, pord,
        derived, pairs, tree_up, tree_dn,
        // device group: bins slice, local frontier, partials, real counts, slice staging
        g_bins, g_offs, g_rows, g_part, g_real, g_hist, g_plain, g_misc;
    Buf *all() { return &node_of; }
    static constexpr int kCount = 27;
};
static_assert(sizeof(HistBufs) == HistBufs::kCount * sizeof(Buf), "HistBufs is a plain array of Buf");
// per context (a context is used by one host thread at a time)
HistBufs &hist_bufs(sfxb_ctx *c) {
    if (!c->hist) c->hist = new HistBufs();
    return *static_cast<HistBufs *>(c->hist);
}
void free_hist_bufs(sfxb_ctx *c) {
    if (!c->hist) return;
    HistBufs *B = static_cast<HistBufs *>(c->hist);
    for (int i = 0; i < HistBufs::kCount; ++i)
        if (B->all()[i].p) cudaFree(B->all()[i].p);
    delete B;
    c->hist = nullptr;
}

// The key holder's histograms multiply by CRT on base-p/q digits (2.6× fewer
// products than mod n²); SFXB_NO_CRT_HISTOGRAM=1 forces the mod-n² path.
bool crt_histogram(const sfxb_ctx *c) {
    static const bool off = std::getenv("SFXB_NO_CRT_HISTOGRAM") != nullptr;
    return c->has_priv && c->p2_digits && !off;
}
dev::CrtArgs crt_args(const sfxb_ctx *c) {
    dev::CrtArgs a{};
    for (int i = 0; i < 2; ++i) {
        a.mod_p[i] = arg(c->mod_pq[i]);
        a.mod_p2[i] = arg(c->mod_pq2[i]);
        a.negR[i] = c->d_negR[i];
        a.one[i] = c->d_one_p2[i];
    }
    a.mod_n2 = arg(c->mod_n2);
    a.qq_inv_m = c->d_qq_inv_m;
    a.q2R_n2 = c->d_q2R_n2;
    return a;
}

// A passive party's histograms multiply on base-n digits (3 CIOS passes mod
// n per multiplication, 25% fewer products than one mod-n² pass);
// SFXB_NO_NDIGIT_HISTOGRAM=1 forces the mod-n² CIOS path.
bool nd_histogram(const sfxb_ctx *c) {
    static const bool off = std::getenv("SFXB_NO_NDIGIT_HISTOGRAM") != nullptr;
    return c->n_digits && !off;
}
dev::NdArgs nd_args(const sfxb_ctx *c) {
    dev::NdArgs a{};
    a.mod_n = arg(c->mod_n);
    a.mod_n2 = arg(c->mod_n2);
    a.negR = c->d_negR_n;
    a.one = c->d_one_nd;
    a.r4 = c->d_r4_nd;
    a.n4 = c->d_n4;
    return a;
}

void h2d_padded(sfxb_ctx *c, uint32_t *d, const uint32_t *h, size_t count, size_t words, size_t stride);

// Trivial-zero flags and the resident form (digits / Montgomery) of gh rows
// [lo, hi), on the context stream.
void gh_prepare_range(sfxb_ctx *c, sfxb_gh *g, size_t lo, size_t hi) {
    if (hi <= lo) return;
    const size_t S4 = 4 * (size_t)c->s, rows = hi - lo, n2 = 2 * rows;
    uint32_t *d = g->d + 2 * lo * S4;
    dispatch_class(c->s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        int grid = (int)std::min<size_t>((rows + 255) / 256, (size_t)c->sms * 8);
        dev::k_gh_flags<4 * cs><<<grid, 256, 0, c->stream>>>(d, (uint32_t)rows, 2 * c->nw, g->flags + lo);
        check_launch(*c);
        if (g->digits) {
            // key holder: CRT digits mod p², q² (padic.cuh "K2 at the key holder")
            auto k = dev::k_gh_digits<cs, kTG<C>>;
            constexpr int NI = dev::kBlock / kTG<C>;
            k<<<occupancy_grid(*c, k, n2, NI), dev::kBlock, 0, c->stream>>>(crt_args(c), d, n2);
            check_launch(*c);
        } else {
            static const bool two_step = std::getenv("SFXB_GH_ND_DIRECT") && std::atoi(std::getenv("SFXB_GH_ND_DIRECT")) == 0;
            if (g->digits_n && !two_step) {
                // digits of X̃ straight from X (padic.cuh k_gh_nd_direct)
                auto kd = dev::k_gh_nd_direct<2 * cs, kTGN<C>>;
                constexpr int NId = dev::kBlock / kTGN<C>;
                kd<<<occupancy_grid(*c, kd, n2, NId), dev::kBlock, 0, c->stream>>>(nd_args(c), d, n2);
                check_launch(*c);
                return;
            }
            auto k = dev::k_to_mont<4 * cs, C::TH>;
            constexpr int NI = dev::kBlock / C::TH;
            k<<<occupancy_grid(*c, k, n2, NI), dev::kBlock, 0, c->stream>>>(arg(c->mod_n2), d, n2);
            check_launch(*c);
            if (g->digits_n) {
                auto ks = dev::k_gh_split_n<2 * cs, C::TND>;
                constexpr int NIs = dev::kBlock / C::TND;
                ks<<<occupancy_grid(*c, ks, n2, NIs), dev::kBlock, 0, c->stream>>>(nd_args(c), d, n2);
                check_launch(*c);
            }
        }
    });
}

void gh_choose_form(sfxb_ctx *c, sfxb_gh *g) {
    g->digits = crt_histogram(c);
    g->digits_n = !g->digits && nd_histogram(c);
}

void gh_prepare(sfxb_ctx *c, sfxb_gh *g) {
    gh_choose_form(c, g);
    gh_prepare_range(c, g, 0, g->n_samples);
}

// Host gh rows -> device, pipelined: chunk k's copy (copy stream) overlaps
// the conversion of chunk k−1 (context stream).
void gh_upload_pipelined(sfxb_ctx *c, sfxb_gh *g, const uint32_t *gh_cts) {
    const size_t S4 = 4 * (size_t)c->s, cw = 2 * (size_t)c->nw, n = g->n_samples;
    gh_choose_form(c, g);
    if (cw != S4 || n < 65536) { // padded layout or small: one shot
        if (n) h2d_padded(c, g->d, gh_cts, 2 * n, cw, S4);
        gh_prepare_range(c, g, 0, n);
        return;
    }
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    constexpr int kChunks = 8;
    if (!c->ev_chunk[0])
        for (int k = 0; k < kChunks; ++k) CK(cudaEventCreateWithFlags(&c->ev_chunk[k], cudaEventDisableTiming));
    // the copy stream must not overwrite rows still read by earlier work
    CK(cudaEventRecord(c->ev_chunk[0], c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_chunk[0], 0));
    for (int k = 0; k < kChunks; ++k) {
        const size_t lo = n * k / kChunks, hi = n * (k + 1) / kChunks;
        CK(cudaMemcpyAsync(g->d + 2 * lo * S4, gh_cts + 2 * lo * cw, 2 * (hi - lo) * S4 * 4, cudaMemcpyHostToDevice,
                           c->copy_stream));
        CK(cudaEventRecord(c->ev_chunk[k], c->copy_stream));
        CK(cudaStreamWaitEvent(c->stream, c->ev_chunk[k], 0));
        gh_prepare_range(c, g, lo, hi);
    }
}

sfxb_gh *gh_alloc(sfxb_ctx *c, uint32_t n_samples) {
    auto g = std::make_unique<sfxb_gh>();
    g->ctx = c;
    g->n_samples = n_samples;
    const size_t bytes = (size_t)n_samples * 2 * 4 * c->s * 4 + 16, fbytes = (size_t)n_samples + 16;
    if (c->spare_gh && c->spare_gh_bytes >= bytes && c->spare_flags_bytes >= fbytes) {
        // recycle the spare allocation (one gh per tree: avoids a 1 GB free + malloc)
        g->d = (uint32_t *)c->spare_gh;
        g->flags = (uint8_t *)c->spare_flags;
        g->bytes = c->spare_gh_bytes;
        g->fbytes = c->spare_flags_bytes;
        c->spare_gh = c->spare_flags = nullptr;
        return g.release();
    }
    CK(cudaMalloc(&g->d, bytes));
    CK(cudaMalloc(&g->flags, fbytes));
    g->bytes = bytes;
    g->fbytes = fbytes;
    return g.release();
}

template <typename T>
T *bget(Buf &b, size_t n) {
    return (T *)grow(b, n * sizeof(T) + 64);
}

// Sibling subtraction on a level's Montgomery-form histograms `hist`
// (n_nodes × spn slots, node-major): for every pair, slots of `derived` =
// parent_hist[parent] · hist[small]⁻¹ mod n², all inverses from one batch
// inversion (product tree up on the GPU, root inverse on the host, tree down).
// Returns false (nothing written) when some small-child slot is not a unit.
template <int cs>
bool derive_siblings(sfxb_ctx *c, HistBufs &B, uint32_t *hist, const uint32_t *parent_hist,
                     const dev::Derived *d_pairs, size_t n_pairs, size_t spn) {
    using C = Cls<cs>;
    constexpr int S4 = 4 * cs, NI = dev::kBlock / C::TH;
    cudaStream_t st = c->stream;
    const size_t m = n_pairs * spn; // values to invert
    // level sizes of the product tree
    std::vector<size_t> lvl_n{m}, lvl_off{0};
    while (lvl_n.back() > 1) {
        lvl_off.push_back(lvl_off.back() + lvl_n.back());
        lvl_n.push_back((lvl_n.back() + 1) / 2);
    }
    const size_t total = lvl_off.back() + lvl_n.back();
    uint32_t *tr = bget<uint32_t>(B.tree_up, total * S4);
    uint32_t *inv = bget<uint32_t>(B.tree_dn, total * S4);
    {
        const size_t words = m * S4;
        const int gg = (int)std::min<size_t>((words + 255) / 256, (size_t)c->sms * 16);
        dev::k_gather_small<<<gg, 256, 0, st>>>(hist, d_pairs, n_pairs, spn, S4, tr);
        check_launch(*c);
    }
    // Lanes per instance per tree level: the product tree's upper levels are
    // a few hundred to a few thousand multiplications each, one after the
    // other — latency, not throughput.  Where the level's instances would
    // not fill a wave at C::TH lanes, more lanes per instance (up to 32)
    // shorten each multiplication's dependent chain (same products, same
    // residues); the big bottom levels keep C::TH.
    size_t wave_threads = 0;
    {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_pair_up<S4, C::TH>, dev::kBlock, 0));
        wave_threads = (size_t)std::max(per_sm, 1) * c->sms * dev::kBlock;
    }
    static const bool wide = !(std::getenv("SFXB_PAIR_WIDE") && std::atoi(std::getenv("SFXB_PAIR_WIDE")) == 0);
    auto lanes_for = [&](size_t instances) {
        int t = C::TH;
        while (wide && t < 32 && S4 / (2 * t) >= 2 && instances * 2 * t <= wave_threads) t *= 2;
        return t;
    };
    // f(std::integral_constant<int, TPI>) for the runtime lane count t
    auto with_lanes = [&](int t, auto f) {
        auto one = [&](auto tp) {
            constexpr int T = decltype(tp)::value;
            if constexpr (T >= C::TH && S4 % T == 0 && S4 / T >= 2 && (S4 / T) % 2 == 0) f(tp);
        };
        switch (t) {
        case 32: one(std::integral_constant<int, 32>{}); break;
        case 16: one(std::integral_constant<int, 16>{}); break;
        case 8: one(std::integral_constant<int, 8>{}); break;
        default: one(std::integral_constant<int, C::TH>{}); break;
        }
    };
    for (size_t l = 0; l + 1 < lvl_n.size(); ++l) {
        ProfScope prof_(*c, 3, lvl_n[l] / 2);
        with_lanes(lanes_for(lvl_n[l + 1]), [&](auto tp) {
            constexpr int T = decltype(tp)::value;
            auto kup = dev::k_pair_up<S4, T>;
            const int gu = occupancy_grid(*c, kup, lvl_n[l + 1], dev::kBlock / T);
            kup<<<gu, dev::kBlock, 0, st>>>(arg(c->mod_n2), tr + lvl_off[l] * S4, lvl_n[l],
                                            tr + lvl_off[l + 1] * S4);
        });
        check_launch(*c);
    }
    // invert the root on the host (GMP mpz_invert, or binary extended Euclid)
    std::vector<uint32_t> root(S4);
    CK(cudaMemcpyAsync(root.data(), tr + lvl_off.back() * S4, S4 * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    host::Big plain = c->mh_n2->from_mont(host::from_words(root.data(), S4)), rinv;
    if (!host::inv_mod_fast(plain, c->n2, rinv)) return false;
    host::Big rinv_m = host::pad(c->mh_n2->to_mont(rinv), S4);
    CK(cudaMemcpyAsync(inv + lvl_off.back() * S4, rinv_m.data(), S4 * 4, cudaMemcpyHostToDevice, st));
    for (size_t l = lvl_n.size() - 1; l-- > 0;) {
        ProfScope prof_(*c, 3, lvl_n[l]);
        with_lanes(lanes_for(lvl_n[l]), [&](auto tp) {
            constexpr int T = decltype(tp)::value;
            auto kdn = dev::k_pair_down<S4, T>;
            const int gd = occupancy_grid(*c, kdn, lvl_n[l], dev::kBlock / T);
            kdn<<<gd, dev::kBlock, 0, st>>>(arg(c->mod_n2), inv + lvl_off[l + 1] * S4, tr + lvl_off[l] * S4,
                                            lvl_n[l], inv + lvl_off[l] * S4);
        });
        check_launch(*c);
    }
    CK(cudaStreamSynchronize(st)); // rinv_m is a host temporary
    auto kd = dev::k_derive<S4, C::TH>;
    const int gdv = occupancy_grid(*c, kd, m, NI);
    ProfScope prof_(*c, 3, m);
    kd<<<gdv, dev::kBlock, 0, st>>>(arg(c->mod_n2), parent_hist, inv, d_pairs, n_pairs, spn, hist);
    check_launch(*c);
    return true;
}

// Tree mode (h_parent != nullptr): h_parent[i] is the index of frontier node
// i's parent in the PREVIOUS tree-mode call on this context (−1: none).  The
// context keeps that call's histograms (Montgomery form) as parents; siblings
// (exactly two children of one cached parent) are split into a directly built
// small child and a derived large child.
//
// Device-group shards (accumulate_group) pass h_skip (nodes not built here:
// their slots stay the identity, as the group derives them after the
// cross-shard product) and d_real (2·N·J·K per-slot counts of non-trivial
// ciphertexts, for the group-wide reference counter).
void accumulate_dev(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *d_bins, uint32_t J, const uint32_t *d_offsets,
                    uint32_t N, const uint32_t *d_rows, uint32_t R, uint32_t K, uint32_t *d_out, int mont_out,
                    uint64_t *additions, const int32_t *h_parent = nullptr, const uint32_t *h_offsets = nullptr,
                    const uint8_t *h_skip = nullptr, uint32_t *d_real = nullptr) {
    if (!g || g->ctx != c) throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
    if (K == 0 || K > 65536) throw ApiError(SFXB_ERR_ARG, "accumulate: n_bins out of range");
    const size_t nkeys = (size_t)N * J * K;
    const bool tree = h_parent != nullptr;
    if (nkeys == 0) {
        if (tree) c->tree_valid = false;
        return;
    }
    const size_t spn = (size_t)J * K * 2; // slots per node
    // ---- sibling pairs whose parent histogram is cached
    std::vector<dev::Derived> pairs;
    std::vector<uint8_t> derived_flag;
    size_t derived_rows = 0;
    if (tree && c->tree_valid && c->tree_gh == g && c->tree_J == J && c->tree_K == K) {
        std::vector<uint32_t> offs(N + 1);
        if (h_offsets) std::copy(h_offsets, h_offsets + N + 1, offs.begin());
        else {
            CK(cudaMemcpyAsync(offs.data(), d_offsets, (N + 1) * 4, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        std::vector<std::vector<uint32_t>> kids(c->tree_N);
        for (uint32_t i = 0; i < N; ++i)
            if (h_parent[i] >= 0 && (uint32_t)h_parent[i] < c->tree_N) kids[h_parent[i]].push_back(i);
        derived_flag.assign(N, 0);
        for (uint32_t pnode = 0; pnode < c->tree_N; ++pnode) {
            if (kids[pnode].size() != 2) continue;
            const uint32_t a = kids[pnode][0], b = kids[pnode][1];
            const uint32_t na = offs[a + 1] - offs[a], nb = offs[b + 1] - offs[b];
            const uint32_t small = na <= nb ? a : b, large = na <= nb ? b : a;
            pairs.push_back(dev::Derived{large, small, pnode});
            derived_flag[large] = 1;
            derived_rows += std::max(na, nb);
        }
    }
    if (h_skip && !tree) {
        if (!h_offsets) throw ApiError(SFXB_ERR_ARG, "accumulate: skip mask needs host offsets");
        derived_flag.assign(h_skip, h_skip + N);
        for (uint32_t i = 0; i < N; ++i)
            if (h_skip[i]) derived_rows += h_offsets[i + 1] - h_offsets[i];
    }
    const bool any_skip = std::find(derived_flag.begin(), derived_flag.end(), (uint8_t)1) != derived_flag.end();
    if (nkeys >= 0xffffffffull || (size_t)R * J >= 0xffffffffull)
        throw ApiError(SFXB_ERR_ARG, "accumulate: frontier too large for one call");
    HistBufs &B = hist_bufs(c);
    cudaStream_t st = c->stream;
    uint32_t *count = bget<uint32_t>(B.count, nkeys), *ones = bget<uint32_t>(B.ones, 2 * nkeys);
    uint32_t *cursor = bget<uint32_t>(B.cursor, nkeys), *seg_start = bget<uint32_t>(B.seg_start, nkeys);
    uint32_t *misc = bget<uint32_t>(B.misc, 16); // [0] status, [4] max count, [8..9] adds, [12..13] job counter
    CK(cudaMemsetAsync(count, 0, nkeys * 4, st));
    CK(cudaMemsetAsync(ones, 0, 2 * nkeys * 4, st));
    CK(cudaMemsetAsync(cursor, 0, nkeys * 4, st));
    CK(cudaMemsetAsync(misc, 0, 64, st));
    dev::HistArgs a{};
    a.rows = d_rows;
    a.n_rows = R;
    a.bins = d_bins;
    a.n_samples = g->n_samples;
    a.J = J;
    a.K = K;
    a.gh_flags = g->flags;
    a.count = count;
    a.ones = ones;
    a.cursor = cursor;
    a.seg_start = seg_start;
    a.status = misc;
    uint8_t *d_derived = nullptr;
    dev::Derived *d_pairs = nullptr;
    if (any_skip) {
        d_derived = bget<uint8_t>(B.derived, N);
        CK(cudaMemcpyAsync(d_derived, derived_flag.data(), N, cudaMemcpyHostToDevice, st));
        a.derived = d_derived;
    }
    if (!pairs.empty()) {
        d_pairs = bget<dev::Derived>(B.pairs, pairs.size());
        CK(cudaMemcpyAsync(d_pairs, pairs.data(), pairs.size() * sizeof(dev::Derived), cudaMemcpyHostToDevice, st));
    }
    if (R > 0) {
        uint32_t *node_of = bget<uint32_t>(B.node_of, R);
        a.node_of = node_of;
        dev::k_node_of<<<N, 256, 0, st>>>(d_offsets, node_of);
        check_launch(*c);
        const size_t items = (size_t)R * J;
        int grid = (int)std::min<size_t>((items + 255) / 256, (size_t)c->sms * 16);
        dev::k_hist_count<<<grid, 256, 0, st>>>(a);
        check_launch(*c);
        uint32_t status = 0;
        CK(cudaMemcpyAsync(&status, misc, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (status & 2u) throw ApiError(SFXB_ERR_ARG, "row index out of range in accumulate");
        if (status & 1u) throw ApiError(SFXB_ERR_ARG, "bin index out of range in accumulate");
    }
    // reference counter over ALL nodes (derived ones included)
    unsigned long long *adds_d = reinterpret_cast<unsigned long long *>(misc + 8);
    {
        int grid = (int)std::min<size_t>((nkeys + 255) / 256, (size_t)c->sms * 8);
        dev::k_hist_adds<<<grid, 256, 0, st>>>(count, ones, nkeys, adds_d);
        check_launch(*c);
        if (d_real) {
            dev::k_hist_real<<<grid, 256, 0, st>>>(count, ones, nkeys, d_real);
            check_launch(*c);
        }
    }
    // derived / skipped nodes are not built directly
    for (uint32_t i = 0; i < (uint32_t)derived_flag.size(); ++i)
        if (derived_flag[i]) CK(cudaMemsetAsync(count + (size_t)i * J * K, 0, (size_t)J * K * 4, st));
    // scan counts -> segment starts; max count -> number of passes
    size_t tmp_bytes = 0, tmp2 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, count, seg_start, (int)nkeys, st));
    CK(cub::DeviceReduce::Max(nullptr, tmp2, count, misc + 4, (int)nkeys, st));
    void *cubtmp = grow(B.cub, std::max(tmp_bytes, tmp2) + 256);
    CK(cub::DeviceScan::ExclusiveSum(cubtmp, tmp_bytes, count, seg_start, (int)nkeys, st));
    CK(cub::DeviceReduce::Max(cubtmp, tmp2, count, misc + 4, (int)nkeys, st));
    if (R > 0) {
        const size_t items = (size_t)R * J;
        uint32_t *sorted = bget<uint32_t>(B.sorted, items);
        a.sorted = sorted;
        int grid = (int)std::min<size_t>((items + 255) / 256, (size_t)c->sms * 16);
        dev::k_hist_scatter<<<grid, 256, 0, st>>>(a);
        check_launch(*c);
    }
    uint32_t maxc = 0;
    unsigned long long adds_h = 0;
    CK(cudaMemcpyAsync(&maxc, misc + 4, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&adds_h, adds_d, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (additions) *additions += adds_h;

    // Passes of the segmented product.  Pass i reads segments (starts S_i,
    // lengths L_i) and writes per-key piece counts np and piece starts ps;
    // then S_{i+1} = ps, L_{i+1} = np.  Two (np, ps) and two partial buffers
    // alternate.
    uint32_t *npb[2] = {bget<uint32_t>(B.np, 2 * nkeys), nullptr};
    npb[1] = npb[0] + nkeys;
    uint32_t *psb[2] = {bget<uint32_t>(B.piece_start, 2 * nkeys), nullptr};
    psb[1] = psb[0] + nkeys;
    const uint32_t *cur_start = seg_start, *cur_len = count;
    const uint32_t *src = g->d;
    const uint32_t *sorted = R ? (const uint32_t *)B.sorted.p : nullptr;
    const uint32_t *final_idx = seg_start, *final_part = g->d;
    dispatch_class(c->s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        constexpr int S4 = 4 * cs;
        const int g1 = (int)std::min<size_t>((nkeys + 255) / 256, (size_t)c->sms * 8);
        // items of the current pass (pass 1: frontier rows of directly built nodes)
        size_t items = ((size_t)R - derived_rows) * J;
        uint32_t m = maxc;
        for (int pass = 0; m > 0; ++pass) {
            // piece length for this pass: long pieces when segments are long
            const size_t avg = items / std::max<size_t>(1, std::min<size_t>(nkeys, items));
            const uint32_t Cp = (avg >= 2 * (size_t)kPieceLong && m > (uint32_t)kPieceLong) ? kPieceLong : kPiece;
            uint32_t *np = npb[pass & 1], *ps = psb[pass & 1];
            dev::k_npieces<<<g1, 256, 0, st>>>(cur_len, nkeys, Cp, np);
            check_launch(*c);
            CK(cub::DeviceScan::ExclusiveSum(cubtmp, tmp_bytes, np, ps, (int)nkeys, st));
            uint32_t tail[2];
            CK(cudaMemcpyAsync(&tail[0], ps + nkeys - 1, 4, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(&tail[1], np + nkeys - 1, 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const size_t P = (size_t)tail[0] + tail[1];
            dev::Piece *pieces = bget<dev::Piece>(B.pieces, P);
            dev::k_emit_pieces<<<g1, 256, 0, st>>>(cur_start, cur_len, ps, nkeys, Cp, pieces);
            check_launch(*c);
            // order pieces by length, longest first (warp-uniform trip counts)
            uint32_t *plen = bget<uint32_t>(B.plen, 2 * P), *pidx = bget<uint32_t>(B.pord, 2 * P);
            {
                const int gp = (int)std::min<size_t>((P + 255) / 256, (size_t)c->sms * 8);
                dev::k_piece_keys<<<gp, 256, 0, st>>>(pieces, P, plen, pidx);
                check_launch(*c);
                size_t sort_bytes = 0;
                CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, plen, plen + P, pidx, pidx + P,
                                                             (int)P, 0, 8, st));
                cubtmp = grow(B.cub, std::max({tmp_bytes, tmp2, sort_bytes}) + 256);
                CK(cub::DeviceRadixSort::SortPairsDescending(cubtmp, sort_bytes, plen, plen + P, pidx, pidx + P,
                                                             (int)P, 0, 8, st));
            }
            const uint32_t *order = pidx + P;
            uint32_t *dst = bget<uint32_t>(B.part[pass & 1], P * 2 * S4);
            constexpr int NI = dev::kBlock / C::TH;
            unsigned long long *next_job = reinterpret_cast<unsigned long long *>(misc + 12);
            CK(cudaMemsetAsync(next_job, 0, 8, st));
            // each piece: len − 1 multiplications, G and H; profiling counts 32×32 products
            const uint64_t mults = 2 * (items - P);
            if (g->digits) {
                // CRT on digits: 2 primes × (two-product pass + one pass) mod p per multiplication
                const uint64_t pp = 5ull * cs * cs + 2 * cs;
                ProfScope prof_(*c, 0, mults * 2 * pp);
                constexpr int NIp = dev::kBlock / C::TK;
                if (Cp == (uint32_t)kPieceLong) {
                    auto k = dev::k_seg_prod_p2<cs, C::TK, kPieceLong>;
                    k<<<occupancy_grid(*c, k, 4 * P, NIp), dev::kBlock, 0, st>>>(
                        crt_args(c), pieces, order, P, pass == 0 ? sorted : nullptr, src, dst, next_job);
                } else {
                    auto k = dev::k_seg_prod_p2<cs, C::TK, kPiece>;
                    k<<<occupancy_grid(*c, k, 4 * P, NIp), dev::kBlock, 0, st>>>(
                        crt_args(c), pieces, order, P, pass == 0 ? sorted : nullptr, src, dst, next_job);
                }
            } else if (g->digits_n) {
                // base-n digits: two-product pass + one pass mod n per multiplication
                const uint64_t pn = 5ull * (2 * cs) * (2 * cs) + 2 * (2 * cs);
                ProfScope prof_(*c, 0, mults * pn);
                constexpr int NIn = dev::kBlock / C::TND;
                if (Cp == (uint32_t)kPieceLong) {
                    auto k = dev::k_seg_prod_nd<2 * cs, C::TND, kPieceLong>;
                    k<<<occupancy_grid(*c, k, 2 * P, NIn), dev::kBlock, 0, st>>>(
                        nd_args(c), pieces, order, P, pass == 0 ? sorted : nullptr, src, dst, next_job);
                } else {
                    auto k = dev::k_seg_prod_nd<2 * cs, C::TND, kPiece>;
                    k<<<occupancy_grid(*c, k, 2 * P, NIn), dev::kBlock, 0, st>>>(
                        nd_args(c), pieces, order, P, pass == 0 ? sorted : nullptr, src, dst, next_job);
                }
            } else if (Cp == (uint32_t)kPieceLong) {
                auto k = dev::k_seg_prod<S4, C::TH, kPieceLong>;
                const int grid = occupancy_grid(*c, k, 2 * P, NI);
                ProfScope prof_(*c, 0, mults * (2ull * S4 * S4 + S4));
                k<<<grid, dev::kBlock, 0, st>>>(arg(c->mod_n2), pieces, order, P, pass == 0 ? sorted : nullptr, src,
                                                dst, next_job);
            } else {
                auto k = dev::k_seg_prod<S4, C::TH, kPiece>;
                const int grid = occupancy_grid(*c, k, 2 * P, NI);
                ProfScope prof_(*c, 0, mults * (2ull * S4 * S4 + S4));
                k<<<grid, dev::kBlock, 0, st>>>(arg(c->mod_n2), pieces, order, P, pass == 0 ? sorted : nullptr, src,
                                                dst, next_job);
            }
            check_launch(*c);
            final_idx = ps;
            final_part = dst;
            cur_start = ps;
            cur_len = np;
            src = dst;
            items = P;
            if (m <= Cp) break;
            m = (m + Cp - 1) / Cp;
        }
        auto kf = dev::k_hist_finalize<S4, C::TH>;
        constexpr int NI = dev::kBlock / C::TH;
        auto kfd = dev::k_hist_finalize_p2<cs, C::TC>;
        auto kfn = dev::k_hist_finalize_nd<cs, C::TC>;
        auto finalize = [&](dev::FinOut o) {
            o.slots_per_node = (uint32_t)spn;
            if (g->digits_n) {
                kfn<<<occupancy_grid(*c, kfn, 2 * nkeys, dev::kBlock / C::TC), dev::kBlock, 0, st>>>(
                    nd_args(c), count, final_idx, nkeys, final_part, o);
            } else if (g->digits) {
                // digits -> CRT residue mod n² (a key without rows keeps the literal 1)
                kfd<<<occupancy_grid(*c, kfd, 2 * nkeys, dev::kBlock / C::TC), dev::kBlock, 0, st>>>(
                    crt_args(c), count, final_idx, nkeys, final_part, o);
            } else {
                kf<<<occupancy_grid(*c, kf, 2 * nkeys, NI), dev::kBlock, 0, st>>>(arg(c->mod_n2), count, final_idx,
                                                                                 nkeys, final_part, o);
            }
            check_launch(*c);
        };
        if (!tree) {
            finalize(mont_out ? dev::FinOut{d_out, nullptr, nullptr, 0} : dev::FinOut{nullptr, d_out, nullptr, 0});
            return;
        }
        // tree mode: all nodes in Montgomery form in the context's current
        // buffer (the parents of the next level); directly built nodes also
        // go to the plain output now, derived nodes after k_derive
        uint32_t *hist = (uint32_t *)grow(c->tree_buf[c->tree_cur ^ 1], (size_t)N * spn * S4 * 4 + 64);
        finalize(dev::FinOut{hist, mont_out ? nullptr : d_out, pairs.empty() ? nullptr : d_derived, 0});
        const bool derived_ok = pairs.empty() ||
            derive_siblings<cs>(c, B, hist, (const uint32_t *)c->tree_buf[c->tree_cur].p, d_pairs, pairs.size(), spn);
        if (!derived_ok) {
            // exact fallback: rebuild this level without sibling subtraction
            c->tree_valid = false;
            std::vector<int32_t> none(N, -1);
            accumulate_dev(c, g, d_bins, J, d_offsets, N, d_rows, R, K, d_out, mont_out, nullptr, none.data(),
                           h_offsets);
            return;
        }
        if (mont_out) {
            CK(cudaMemcpyAsync(d_out, hist, (size_t)N * spn * S4 * 4, cudaMemcpyDeviceToDevice, st));
        } else if (!pairs.empty()) {
            auto kc = dev::k_from_mont_nodes<S4, C::TH>;
            const int gc = occupancy_grid(*c, kc, pairs.size() * spn, NI);
            kc<<<gc, dev::kBlock, 0, st>>>(arg(c->mod_n2), hist, d_pairs, pairs.size(), spn, d_out);
            check_launch(*c);
        }
        c->tree_derived_nodes += pairs.size();
        c->tree_cur ^= 1;
        c->tree_valid = true;
        c->tree_gh = g;
        c->tree_J = J;
        c->tree_K = K;
        c->tree_N = N;
    });
}

void reduce_parts_dev(sfxb_ctx *c, const uint32_t *d_parts, uint32_t parts, size_t n_slots, uint32_t *d_out) {
    if (n_slots == 0) return;
    if (parts == 0) throw ApiError(SFXB_ERR_ARG, "reduce_partials: no inputs");
    dispatch_class(c->s, [&](auto sc) {
        constexpr int cs = decltype(sc)::value;
        using C = Cls<cs>;
        auto k = dev::k_reduce_parts<4 * cs, C::TH>;
        constexpr int NI = dev::kBlock / C::TH;
        const int grid = occupancy_grid(*c, k, n_slots, NI);
        k<<<grid, dev::kBlock, 0, c->stream>>>(arg(c->mod_n2), d_parts, parts, n_slots, d_out);
        check_launch(*c);
    });
}

// --------------------------------------------------------------- host <-> padded layouts

// copy `count` values of `words` limbs into a padded device layout of `stride`
void h2d_padded(sfxb_ctx *c, uint32_t *d, const uint32_t *h, size_t count, size_t words, size_t stride) {
    if (words == stride) {
        CK(cudaMemcpyAsync(d, h, count * words * 4, cudaMemcpyHostToDevice, c->stream));
        return;
    }
    std::vector<uint32_t> tmp(count * stride, 0u);
    for (size_t i = 0; i < count; ++i) std::memcpy(&tmp[i * stride], h + i * words, words * 4);
    CK(cudaMemcpyAsync(d, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
}
void d2h_padded(sfxb_ctx *c, uint32_t *h, const uint32_t *d, size_t count, size_t words, size_t stride) {
    if (words == stride) {
        CK(cudaMemcpyAsync(h, d, count * words * 4, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return;
    }
    std::vector<uint32_t> tmp(count * stride);
    CK(cudaMemcpyAsync(tmp.data(), d, tmp.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < count; ++i) std::memcpy(h + i * words, &tmp[i * stride], words * 4);
}

// view of a grow-only per-context staging buffer
template <typename T>
struct IoBuf {
    T *p;
    IoBuf(Buf &b, size_t n) : p((T *)grow(b, n * sizeof(T) + 64)) {}
};

template <typename T>
struct DevBuf {
    T *p = nullptr;
    explicit DevBuf(size_t n) { CK(cudaMalloc(&p, n * sizeof(T) + 16)); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
};

// --------------------------------------------------------------- host-buffer operations (one device)

// sfxb_encrypt / sfxb_encrypt_plain: q_fixed xor m_words (count × n_words)
void encrypt_host(sfxb_ctx *c, const int64_t *q_fixed, const uint32_t *m_words, const uint32_t *r, size_t count,
                  uint32_t *out_cts, uint8_t *r_flags) {
    CK(cudaSetDevice(c->device));
    if (count == 0) return;
    const size_t Sn = 2 * (size_t)c->s, S4 = 4 * (size_t)c->s;
    // range checks of encrypt_with_r (he.cpp:88-89), in its order per element
    // (word-wise compares against n, no allocation per element)
    const std::vector<uint32_t> nw_words = host::pad(c->n, c->nw);
    auto lt_n = [&](const uint32_t *x) {
        for (uint32_t k = c->nw; k-- > 0;)
            if (x[k] != nw_words[k]) return x[k] < nw_words[k];
        return false; // equal
    };
    for (size_t i = 0; i < count; ++i) {
        if (m_words && !lt_n(m_words + i * c->nw))
            throw ApiError(SFXB_ERR_RANGE, "encrypt: plaintext out of range [0, n)");
        const uint32_t *ri = r + i * c->nw;
        bool small = true;
        for (uint32_t k = 1; k < c->nw; ++k) small &= ri[k] == 0;
        if (small && ri[0] < 1) throw ApiError(SFXB_ERR_RANGE, "encrypt: blinding factor out of range");
        if (!lt_n(ri)) throw ApiError(SFXB_ERR_RANGE, "encrypt: blinding factor out of range");
    }
    IoBuf<int64_t> dq(c->io[0], m_words ? 1 : count);
    IoBuf<uint32_t> dr(c->io[1], count * Sn), dout(c->io[2], count * S4);
    IoBuf<uint8_t> dflags(c->io[3], count);
    IoBuf<uint32_t> dm(c->io[4], m_words ? count * Sn : 1);
    CK(cudaMemsetAsync(dflags.p, 0, count, c->stream));
    if (m_words) h2d_padded(c, dm.p, m_words, count, c->nw, Sn);
    else CK(cudaMemcpyAsync(dq.p, q_fixed, count * 8, cudaMemcpyHostToDevice, c->stream));
    h2d_padded(c, dr.p, r, count, c->nw, Sn);
    int st = SFXB_OK;
    try {
        encrypt_dev(c, m_words ? nullptr : dq.p, dr.p, count, dout.p, dflags.p, m_words ? dm.p : nullptr);
    } catch (const ApiError &e) {
        if (e.code != SFXB_ERR_COPRIME) throw;
        st = e.code;
        c->err = e.what();
    }
    if (r_flags) {
        CK(cudaMemcpyAsync(r_flags, dflags.p, count, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    if (st != SFXB_OK) throw ApiError(st, c->err);
    d2h_padded(c, out_cts, dout.p, count, 2 * c->nw, S4);
}

// rows × cols values of `words` limbs, taken from column col0 of a host matrix
// with `pitch` values per row, into a dense device layout of `stride` limbs
void h2d_cols(sfxb_ctx *c, uint32_t *d, const uint32_t *h, size_t rows, size_t pitch, size_t col0, size_t cols,
              size_t words, size_t stride) {
    if (!rows || !cols) return;
    if (words == stride) {
        CK(cudaMemcpy2DAsync(d, cols * stride * 4, h + col0 * words, pitch * words * 4, cols * words * 4, rows,
                             cudaMemcpyHostToDevice, c->stream));
        return;
    }
    std::vector<uint32_t> tmp(rows * cols * stride, 0u);
    for (size_t r = 0; r < rows; ++r)
        for (size_t j = 0; j < cols; ++j)
            std::memcpy(&tmp[(r * cols + j) * stride], h + (r * pitch + col0 + j) * words, words * 4);
    CK(cudaMemcpyAsync(d, tmp.data(), tmp.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
}
// the inverse of h2d_cols (synchronous)
void d2h_cols(sfxb_ctx *c, uint32_t *h, const uint32_t *d, size_t rows, size_t pitch, size_t col0, size_t cols,
              size_t words, size_t stride) {
    if (!rows || !cols) return;
    if (words == stride) {
        CK(cudaMemcpy2DAsync(h + col0 * words, pitch * words * 4, d, cols * stride * 4, cols * words * 4, rows,
                             cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return;
    }
    std::vector<uint32_t> tmp(rows * cols * stride);
    CK(cudaMemcpyAsync(tmp.data(), d, tmp.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (size_t r = 0; r < rows; ++r)
        for (size_t j = 0; j < cols; ++j)
            std::memcpy(h + (r * pitch + col0 + j) * words, &tmp[(r * cols + j) * stride], words * 4);
}

void add_host(sfxb_ctx *c, const uint32_t *a, const uint32_t *b, size_t count, uint32_t *out) {
    CK(cudaSetDevice(c->device));
    if (count == 0) return;
    const size_t S4 = 4 * (size_t)c->s, cw = 2 * c->nw;
    const std::vector<uint32_t> n2w = host::pad(c->n2, cw);
    auto lt_n2 = [&](const uint32_t *x) {
        for (size_t k = cw; k-- > 0;)
            if (x[k] != n2w[k]) return x[k] < n2w[k];
        return false;
    };
    for (size_t i = 0; i < count; ++i)
        if (!lt_n2(a + i * cw) || !lt_n2(b + i * cw))
            throw ApiError(SFXB_ERR_RANGE, "add_ciphertexts: ciphertext out of range");
    IoBuf<uint32_t> da(c->io[0], count * S4), db(c->io[1], count * S4), dout(c->io[2], count * S4);
    h2d_padded(c, da.p, a, count, cw, S4);
    h2d_padded(c, db.p, b, count, cw, S4);
    add_dev(c, da.p, db.p, count, dout.p);
    d2h_padded(c, out, dout.p, count, cw, S4);
}

void decrypt_host(sfxb_ctx *c, const uint32_t *cts, size_t count, uint32_t scale, double *out_values,
                  uint32_t *out_plain, uint64_t *decryptions) {
    CK(cudaSetDevice(c->device));
    if (!c->has_priv) throw ApiError(SFXB_ERR_AUTH, "decrypt requested without private key material");
    if (count == 0) return;
    const size_t Sn = 2 * (size_t)c->s, S4 = 4 * (size_t)c->s;
    IoBuf<uint32_t> dc(c->io[0], count * S4), dplain(c->io[1], out_plain ? count * Sn : 1);
    IoBuf<double> dv(c->io[2], count);
    h2d_padded(c, dc.p, cts, count, 2 * c->nw, S4);
    decrypt_dev(c, dc.p, count, scale, dv.p, out_plain ? dplain.p : nullptr, decryptions);
    CK(cudaMemcpyAsync(out_values, dv.p, count * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (out_plain) d2h_padded(c, out_plain, dplain.p, count, c->nw, Sn);
}

// SFXB_TRACE=1: per-phase wall times of one call (stream synchronized at each lap)
struct TraceT {
    cudaStream_t st;
    bool on;
    std::chrono::steady_clock::time_point t;
    std::string line;
    TraceT(cudaStream_t s_) : st(s_), on(std::getenv("SFXB_TRACE") != nullptr), t(std::chrono::steady_clock::now()) {}
    void lap(const char *ph) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        char b[64];
        std::snprintf(b, sizeof b, " %s=%.1fms", ph, std::chrono::duration<double, std::milli>(now - t).count());
        line += b;
        t = now;
    }
    ~TraceT() {
        if (on) std::fprintf(stderr, "[sfxb-trace]%s\n", line.c_str());
    }
};

// sfxb_decrypt_tree on slot slice [j0, j0 + jl) of every node (the whole node
// for a single-device context).  The slice's cache entry is this level's
// ciphertexts and plaintexts; sibling checks compare slot j of a, b and P, so
// they never leave the slice.
void decrypt_tree_impl(sfxb_ctx *c, uint64_t tag, const uint32_t *cts, uint32_t n_nodes, uint32_t spn_total,
                       uint32_t j0, uint32_t jl, const int32_t *parent, uint32_t scale, double *out_values,
                       uint64_t *decryptions) {
    CK(cudaSetDevice(c->device));
    if (!c->has_priv) throw ApiError(SFXB_ERR_AUTH, "decrypt requested without private key material");
    const uint32_t spn = jl;
    const size_t count = (size_t)n_nodes * spn;
    const size_t Sn = 2 * (size_t)c->s, S4 = 4 * (size_t)c->s;
    TraceT tr(c->stream);
    CtxState::DecCache &prev = c->dec_cache[tag];
    // sibling pairs (two children of one cached parent): b = second child
    std::vector<uint32_t> pairs;
    if (parent && prev.valid && prev.spn == spn && prev.spn_total == spn_total && prev.j0 == j0) {
        std::vector<std::vector<uint32_t>> kids(prev.n_nodes);
        for (uint32_t i = 0; i < n_nodes; ++i)
            if (parent[i] >= 0 && (uint32_t)parent[i] < prev.n_nodes) kids[parent[i]].push_back(i);
        for (uint32_t pnode = 0; pnode < prev.n_nodes; ++pnode)
            if (kids[pnode].size() == 2) {
                pairs.push_back(kids[pnode][1]);
                pairs.push_back(kids[pnode][0]);
                pairs.push_back(pnode);
            }
    }
    const int nx = prev.cur ^ 1;
    uint32_t *dc = (uint32_t *)grow(prev.cts[nx], count * S4 * 4 + 64);
    uint32_t *dplain = (uint32_t *)grow(prev.plain[nx], count * Sn * 4 + 64);
    IoBuf<double> dv(c->io[2], count ? count : 1);
    tr.lap("alloc");
    if (count) h2d_cols(c, dc, cts, n_nodes, spn_total, j0, jl, 2 * c->nw, S4);
    tr.lap("h2d");
    uint8_t *skip = nullptr;
    const size_t np = pairs.size() / 3;
    uint32_t *dpairs = nullptr;
    if (np && spn) {
        skip = (uint8_t *)grow(c->io[4], count + 64);
        dpairs = (uint32_t *)grow(c->io[5], pairs.size() * 4 + 64);
        CK(cudaMemsetAsync(skip, 0, count, c->stream));
        CK(cudaMemcpyAsync(dpairs, pairs.data(), pairs.size() * 4, cudaMemcpyHostToDevice, c->stream));
        dev::SibArgs sa{dc, (const uint32_t *)prev.cts[prev.cur].p, dpairs, np, spn, skip};
        dispatch_class(c->s, [&](auto sc) {
            constexpr int cs = decltype(sc)::value;
            using C = Cls<cs>;
            auto k = dev::k_sib_verify<4 * cs, C::TH>;
            constexpr int NI = dev::kBlock / C::TH;
            const int grid = occupancy_grid(*c, k, np * spn, NI);
            k<<<grid, dev::kBlock, 0, c->stream>>>(arg(c->mod_n2), sa);
            check_launch(*c);
        });
    }
    tr.lap("verify");
    if (count) decrypt_dev(c, dc, count, scale, dv.p, dplain, decryptions, skip);
    tr.lap("decrypt");
    if (skip) {
        dispatch_class(c->s, [&](auto sc) {
            constexpr int cs = decltype(sc)::value;
            const int grid = (int)std::min<size_t>((np * spn + 127) / 128, (size_t)c->sms * 8);
            dev::k_sib_derive<2 * cs><<<grid, 128, 0, c->stream>>>(
                dpairs, np, spn, skip, dplain, (const uint32_t *)prev.plain[prev.cur].p, c->d_n, scale, dplain, dv.p);
            check_launch(*c);
        });
    }
    if (count)
        CK(cudaMemcpy2DAsync(out_values + j0, (size_t)spn_total * 8, dv.p, (size_t)jl * 8, (size_t)jl * 8, n_nodes,
                             cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    tr.lap("derive_d2h");
    if (tr.on) {
        char b[96];
        std::snprintf(b, sizeof b, " tag=%llu nodes=%u spn=%u pairs=%zu", (unsigned long long)tag, n_nodes, spn, np);
        tr.line += b;
    }
    // this level becomes the parent level of the tag
    prev.cur = nx;
    prev.n_nodes = n_nodes;
    prev.spn = spn;
    prev.spn_total = spn_total;
    prev.j0 = j0;
    prev.valid = true;
}

// =================================================================== device group
//
// sfxb_ctx_create_multi: one key on several GPUs of this process (SURVEY §8e
// inside the reference's single-process plugin).  Encrypt, add and decrypt
// split their elements into contiguous ranges; decrypt_tree splits every
// node's slots into per-GPU slices; the histogram is row-sharded with a
// cross-GPU modular-product reduce over NVLink peer memory (accumulate_group).
// Every shard runs on its own host thread and stream.

bool is_group(const sfxb_ctx *c) { return c->shards.size() > 1; }

// f(k, shard) for k < n on one host thread per shard (shard 0 on the caller's
// thread); rethrows the error of the lowest failing shard after all finish
template <typename F>
void for_shards(sfxb_ctx *c, size_t n, F &&f) {
    std::vector<std::exception_ptr> errs(n);
    std::vector<std::thread> th;
    th.reserve(n);
    auto run = [&](size_t k) {
        try {
            CK(cudaSetDevice(c->shards[k]->device));
            f(k, c->shards[k]);
        } catch (...) {
            errs[k] = std::current_exception();
        }
    };
    for (size_t k = 1; k < n; ++k) th.emplace_back(run, k);
    run(0);
    for (auto &t : th) t.join();
    CK(cudaSetDevice(c->device));
    for (auto &e : errs)
        if (e) std::rethrow_exception(e);
}

// bounds of `parts` near-equal contiguous ranges of `count` items
std::vector<size_t> split_even(size_t count, size_t parts) {
    std::vector<size_t> lo(parts + 1, 0);
    const size_t base = count / parts, extra = count % parts;
    for (size_t k = 0; k < parts; ++k) lo[k + 1] = lo[k] + base + (k < extra ? 1 : 0);
    return lo;
}
// element-wise batches: no shard gets fewer than `grain` items
std::vector<size_t> split_batch(size_t count, size_t shards, size_t grain) {
    return split_even(count, std::max<size_t>(1, std::min(shards, count / std::max<size_t>(1, grain))));
}
constexpr size_t kGrainExp = 4096;   // encrypt / decrypt: one exponentiation per item
constexpr size_t kGrainAdd = 65536;  // ct-add: one multiplication per item

void encrypt_group(sfxb_ctx *c, const int64_t *q, const uint32_t *m, const uint32_t *r, size_t count,
                   uint32_t *out, uint8_t *flags) {
    const std::vector<size_t> lo = split_batch(count, c->shards.size(), kGrainExp);
    const size_t nw = c->nw, cw = 2 * nw;
    for_shards(c, lo.size() - 1, [&](size_t k, sfxb_ctx *sh) {
        const size_t a = lo[k], n = lo[k + 1] - a;
        encrypt_host(sh, q ? q + a : nullptr, m ? m + a * nw : nullptr, r + a * nw, n, out + a * cw,
                     flags ? flags + a : nullptr);
    });
}

void add_group(sfxb_ctx *c, const uint32_t *x, const uint32_t *y, size_t count, uint32_t *out) {
    const std::vector<size_t> lo = split_batch(count, c->shards.size(), kGrainAdd);
    const size_t cw = 2 * (size_t)c->nw;
    for_shards(c, lo.size() - 1, [&](size_t k, sfxb_ctx *sh) {
        const size_t a = lo[k];
        add_host(sh, x + a * cw, y + a * cw, lo[k + 1] - a, out + a * cw);
    });
}

void decrypt_group(sfxb_ctx *c, const uint32_t *cts, size_t count, uint32_t scale, double *vals, uint32_t *plain,
                   uint64_t *decryptions) {
    if (!c->has_priv) throw ApiError(SFXB_ERR_AUTH, "decrypt requested without private key material");
    const std::vector<size_t> lo = split_batch(count, c->shards.size(), kGrainExp);
    const size_t nw = c->nw, cw = 2 * nw;
    std::vector<uint64_t> decs(lo.size() - 1, 0);
    for_shards(c, lo.size() - 1, [&](size_t k, sfxb_ctx *sh) {
        const size_t a = lo[k];
        decrypt_host(sh, cts + a * cw, lo[k + 1] - a, scale, vals + a, plain ? plain + a * nw : nullptr, &decs[k]);
    });
    if (decryptions)
        for (uint64_t d : decs) *decryptions += d;
}

void decrypt_tree_group(sfxb_ctx *c, uint64_t tag, const uint32_t *cts, uint32_t n_nodes, uint32_t spn,
                        const int32_t *parent, uint32_t scale, double *vals, uint64_t *decryptions) {
    if (!c->has_priv) throw ApiError(SFXB_ERR_AUTH, "decrypt requested without private key material");
    const size_t G = c->shards.size();
    const std::vector<size_t> jlo = split_even(spn, G);
    std::vector<uint64_t> decs(G, 0);
    for_shards(c, G, [&](size_t k, sfxb_ctx *sh) {
        decrypt_tree_impl(sh, tag, cts, n_nodes, spn, (uint32_t)jlo[k], (uint32_t)(jlo[k + 1] - jlo[k]), parent,
                          scale, vals, &decs[k]);
    });
    if (decryptions)
        for (uint64_t d : decs) *decryptions += d;
}

sfxb_gh *gh_upload_group(sfxb_ctx *c, const uint32_t *gh_cts, uint32_t n_samples) {
    const size_t G = c->shards.size(), cw = 2 * (size_t)c->nw, S4 = 4 * (size_t)c->s;
    const std::vector<size_t> lo = split_even(n_samples, G);
    auto g = std::make_unique<sfxb_gh>();
    g->ctx = c;
    g->n_samples = n_samples;
    g->parts.assign(G, nullptr);
    for (size_t k = 0; k <= G; ++k) g->row_lo.push_back((uint32_t)lo[k]);
    try {
        for_shards(c, G, [&](size_t k, sfxb_ctx *sh) {
            const size_t n = lo[k + 1] - lo[k];
            g->parts[k] = gh_alloc(sh, (uint32_t)n);
            if (n) h2d_padded(sh, g->parts[k]->d, gh_cts + 2 * lo[k] * cw, 2 * n, cw, S4);
            gh_prepare(sh, g->parts[k]);
            CK(cudaStreamSynchronize(sh->stream));
        });
    } catch (...) {
        for (sfxb_gh *p : g->parts)
            if (p) sfxb_gh_free(p);
        throw;
    }
    return g.release();
}

// Sibling pairs of a level against the context's cached parent level (valid
// for gradient handle g, J, K and slice geometry G), the smaller child (by
// the callers' GLOBAL row counts `sizes`) built directly, the larger derived.
// Every shard / rank computes the same plan from the same inputs.
void plan_pairs(const sfxb_ctx *c, const sfxb_gh *g, uint32_t J, uint32_t K, uint32_t G, const int32_t *parent,
                const uint32_t *sizes, uint32_t N, std::vector<dev::Derived> &pairs, std::vector<uint8_t> &skip) {
    pairs.clear();
    skip.assign(N, 0);
    if (!parent || !(c->tree_valid && c->tree_gh == g && c->tree_J == J && c->tree_K == K && c->tree_G == G)) return;
    std::vector<std::vector<uint32_t>> kids(c->tree_N);
    for (uint32_t i = 0; i < N; ++i)
        if (parent[i] >= 0 && (uint32_t)parent[i] < c->tree_N) kids[parent[i]].push_back(i);
    for (uint32_t pnode = 0; pnode < c->tree_N; ++pnode) {
        if (kids[pnode].size() != 2) continue;
        const uint32_t a = kids[pnode][0], b = kids[pnode][1];
        const uint32_t small = sizes[a] <= sizes[b] ? a : b, large = sizes[a] <= sizes[b] ? b : a;
        pairs.push_back(dev::Derived{large, small, pnode});
        skip[large] = 1;
    }
}

// ---- rank-sliced histograms (one process per GPU, bench.py under torchrun)
//
// The device group's algorithm with the peer reads replaced by a collective
// the caller runs (NCCL all_to_all): sfxb_accumulate_part_dev builds this
// rank's Montgomery partials (nodes to be derived skipped) already cut into
// `world` slot slices, rank-major; after the exchange sfxb_combine_slices_dev
// multiplies the received slices, derives the larger siblings on the slice
// against the slice cached at the previous level and writes the plain slice.

// slice width: every node's 2·J·K slots in `world` column blocks of jl
uint32_t slice_width(uint32_t J, uint32_t K, uint32_t world) {
    const uint32_t spn = 2 * J * K;
    return (spn + world - 1) / world;
}

void accumulate_part(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *d_bins, uint32_t J, const uint32_t *d_offs,
                     const uint32_t *h_offs, uint32_t N, const uint32_t *d_rows, uint32_t R, uint32_t K,
                     const int32_t *h_parent, const uint32_t *h_sizes, uint32_t world, uint32_t *d_send,
                     uint32_t *d_real) {
    if (!g || g->ctx != c || !g->parts.empty())
        throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
    if (world == 0 || world > (uint32_t)dev::kMaxShards) throw ApiError(SFXB_ERR_ARG, "accumulate: bad world size");
    const size_t S4 = 4 * (size_t)c->s, spn = 2 * (size_t)J * K, jl = slice_width(J, K, world);
    std::vector<dev::Derived> pairs;
    std::vector<uint8_t> skip;
    plan_pairs(c, g, J, K, world, h_parent, h_sizes, N, pairs, skip);
    HistBufs &B = hist_bufs(c);
    uint32_t *part = bget<uint32_t>(B.g_part, (size_t)N * spn * S4);
    accumulate_dev(c, g, d_bins, J, d_offs, N, d_rows, R, K, part, 1, nullptr, nullptr, h_offs, skip.data(), d_real);
    cudaStream_t st = c->stream;
    if (jl * world != spn && N) {
        const size_t words = (size_t)world * N * jl * S4;
        const int grid = (int)std::min<size_t>((words + 255) / 256, (size_t)c->sms * 16);
        dev::k_fill_pad<<<grid, 256, 0, st>>>(d_send, world, N, jl, spn, (int)S4, c->mod_n2.w + S4); // R mod n²
        check_launch(*c);
    }
    for (uint32_t k = 0; k < world && N; ++k) {
        const size_t lo = (size_t)k * jl, w = lo < spn ? std::min<size_t>(jl, spn - lo) : 0;
        if (w)
            CK(cudaMemcpy2DAsync(d_send + (size_t)k * N * jl * S4, jl * S4 * 4, part + lo * S4, spn * S4 * 4,
                                 w * S4 * 4, N, cudaMemcpyDeviceToDevice, st));
    }
}

void combine_slices(sfxb_ctx *c, const sfxb_gh *g, const uint32_t *d_recv, uint32_t world, uint32_t rank, uint32_t N,
                    uint32_t J, uint32_t K, const int32_t *h_parent, const uint32_t *h_sizes, uint32_t *d_out) {
    if (world == 0 || world > (uint32_t)dev::kMaxShards || rank >= world)
        throw ApiError(SFXB_ERR_ARG, "combine: bad world size or rank");
    const size_t S4 = 4 * (size_t)c->s, jl = slice_width(J, K, world), cnt = (size_t)N * jl;
    const bool tree = h_parent != nullptr;
    std::vector<dev::Derived> pairs;
    std::vector<uint8_t> skip;
    plan_pairs(c, g, J, K, world, h_parent, h_sizes, N, pairs, skip);
    HistBufs &B = hist_bufs(c);
    cudaStream_t st = c->stream;
    uint32_t *hist = tree ? (uint32_t *)grow(c->tree_buf[c->tree_cur ^ 1], cnt * S4 * 4 + 64)
                          : bget<uint32_t>(B.g_hist, cnt * S4);
    dev::PeerSet parts{};
    parts.n = world;
    for (uint32_t k = 0; k < world; ++k) parts.p[k] = d_recv + (size_t)k * cnt * S4;
    if (cnt) {
        dispatch_class(c->s, [&](auto sc) {
            constexpr int cs = decltype(sc)::value;
            using C = Cls<cs>;
            constexpr int NI = dev::kBlock / C::TH;
            auto kr = dev::k_reduce_peer<4 * cs, C::TH>;
            kr<<<occupancy_grid(*c, kr, cnt, NI), dev::kBlock, 0, st>>>(arg(c->mod_n2), parts, N, jl, 0, jl, hist);
            check_launch(*c);
            if (!pairs.empty()) {
                dev::Derived *d_pairs = bget<dev::Derived>(B.pairs, pairs.size());
                CK(cudaMemcpyAsync(d_pairs, pairs.data(), pairs.size() * sizeof(dev::Derived), cudaMemcpyHostToDevice,
                                   st));
                if (!derive_siblings<cs>(c, B, hist, (const uint32_t *)c->tree_buf[c->tree_cur].p, d_pairs,
                                         pairs.size(), jl)) {
                    c->tree_valid = false;
                    throw ApiError(SFXB_ERR_COPRIME, "accumulate: a histogram slot shares a factor with n; "
                                                     "rerun the level without sibling subtraction");
                }
            }
            auto kc = dev::k_from_mont_copy<4 * cs, C::TH>;
            kc<<<occupancy_grid(*c, kc, cnt, NI), dev::kBlock, 0, st>>>(arg(c->mod_n2), hist, cnt, d_out);
            check_launch(*c);
        });
    }
    if (tree) {
        c->tree_cur ^= 1;
        c->tree_valid = true;
        c->tree_gh = g;
        c->tree_J = J;
        c->tree_K = K;
        c->tree_N = N;
        c->tree_G = world;
        c->tree_j0 = rank * (uint32_t)jl;
        c->tree_jl = (uint32_t)jl;
        c->tree_derived_nodes += pairs.size();
    }
}

// Row-sharded histogram over the group (sfxb_accumulate_gh /
// sfxb_accumulate_tree_gh on a multi-device context).
//   phase 1, every shard: its rows of the frontier, its bin columns, partial
//     histograms of its rows in Montgomery form (nodes derived by sibling
//     subtraction are skipped), per-slot real-ciphertext counts;
//   phase 2, shard k: slot slice k of every node = product of all shards'
//     partials, read over NVLink (k_reduce_peer); sibling subtraction on the
//     slice against the slice cached from the previous level; plain form
//     straight into the caller's output rows.  Shard 0 also forms the
//     reference counter from all shards' counts (k_adds_multi).
void accumulate_group(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *bins, uint32_t J, const uint32_t *offs,
                      uint32_t N, const uint32_t *rows, uint32_t K, const int32_t *parent, uint32_t *out_slots,
                      uint64_t *additions) {
    if (!g || g->ctx != c || g->parts.size() != c->shards.size())
        throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
    if (K == 0 || K > 65536) throw ApiError(SFXB_ERR_ARG, "accumulate: n_bins out of range");
    const size_t G = c->shards.size(), S4 = 4 * (size_t)c->s, cw = 2 * (size_t)c->nw;
    const size_t spn = 2 * (size_t)J * K, nkeys = (size_t)N * J * K;
    const bool tree = parent != nullptr;
    if (nkeys == 0) {
        if (tree)
            for (sfxb_ctx *sh : c->shards) sh->tree_valid = false;
        return;
    }
    if (nkeys >= 0xffffffffull || (size_t)offs[N] * J >= 0xffffffffull)
        throw ApiError(SFXB_ERR_ARG, "accumulate: frontier too large for one call");
    // sibling pairs, chosen on global row counts (identical on every shard)
    std::vector<dev::Derived> pairs;
    std::vector<uint8_t> skip;
    {
        std::vector<uint32_t> sizes(N);
        for (uint32_t i = 0; i < N; ++i) sizes[i] = offs[i + 1] - offs[i];
        plan_pairs(c, g, J, K, (uint32_t)G, parent, sizes.data(), N, pairs, skip);
    }
    const std::vector<size_t> jlo = split_even(spn, G);
    const uint32_t n_samples = g->n_samples;
    // The reference lists each node's rows ascending (gbdt.cpp:157-180): then
    // a shard's rows of a node are one contiguous run, found by two binary
    // searches, and each shard touches only its own rows.  Otherwise every
    // shard filters the whole frontier.
    bool ascending = true;
    for (uint32_t i = 0; i < N && ascending; ++i)
        for (uint32_t t = offs[i] + 1; t < offs[i + 1]; ++t)
            if (rows[t] <= rows[t - 1]) {
                ascending = false;
                break;
            }
    for (uint32_t i = 0; i < N && ascending; ++i)
        if (offs[i + 1] > offs[i] && rows[offs[i + 1] - 1] >= n_samples)
            throw ApiError(SFXB_ERR_ARG, "row index out of range in accumulate");
    // ---- phase 1: partial histograms of each shard's rows
    std::vector<const uint32_t *> part_ptr(G), real_ptr(G);
    for_shards(c, G, [&](size_t k, sfxb_ctx *sh) {
        const uint32_t lo = g->row_lo[k], hi = g->row_lo[k + 1];
        std::vector<uint32_t> loffs(N + 1, 0), lrows;
        lrows.reserve((size_t)offs[N] / G + 1024);
        for (uint32_t i = 0; i < N; ++i) {
            if (ascending) {
                const uint32_t *b = rows + offs[i], *e = rows + offs[i + 1];
                for (const uint32_t *r = std::lower_bound(b, e, lo), *re = std::lower_bound(b, e, hi); r < re; ++r)
                    lrows.push_back(*r - lo);
            } else {
                for (uint32_t t = offs[i]; t < offs[i + 1]; ++t) {
                    const uint32_t row = rows[t];
                    if (row >= n_samples) throw ApiError(SFXB_ERR_ARG, "row index out of range in accumulate");
                    if (row >= lo && row < hi) lrows.push_back(row - lo);
                }
            }
            loffs[i + 1] = (uint32_t)lrows.size();
        }
        HistBufs &B = hist_bufs(sh);
        const size_t nr = hi - lo, R = lrows.size();
        uint16_t *db = bget<uint16_t>(B.g_bins, (size_t)J * nr);
        if (nr)
            CK(cudaMemcpy2DAsync(db, nr * 2, bins + lo, (size_t)n_samples * 2, nr * 2, J, cudaMemcpyHostToDevice,
                                 sh->stream));
        uint32_t *doffs = bget<uint32_t>(B.g_offs, N + 1), *drows = bget<uint32_t>(B.g_rows, R ? R : 1);
        CK(cudaMemcpyAsync(doffs, loffs.data(), (N + 1) * 4, cudaMemcpyHostToDevice, sh->stream));
        if (R) CK(cudaMemcpyAsync(drows, lrows.data(), R * 4, cudaMemcpyHostToDevice, sh->stream));
        uint32_t *part = bget<uint32_t>(B.g_part, (size_t)N * spn * S4);
        uint32_t *real = bget<uint32_t>(B.g_real, 2 * nkeys);
        accumulate_dev(sh, g->parts[k], db, J, doffs, N, drows, (uint32_t)R, K, part, 1, nullptr, nullptr,
                       loffs.data(), skip.data(), real);
        CK(cudaEventRecord(sh->ev_part, sh->stream));
        // host staging (loffs, lrows) must outlive the async copies
        CK(cudaStreamSynchronize(sh->stream));
        part_ptr[k] = part;
        real_ptr[k] = real;
    });
    // ---- phase 2: cross-shard product of slot slices, sibling subtraction, output
    dev::PeerSet parts{}, reals{};
    parts.n = reals.n = (uint32_t)G;
    for (size_t k = 0; k < G; ++k) {
        parts.p[k] = part_ptr[k];
        reals.p[k] = real_ptr[k];
    }
    std::vector<char> ok(G, 1);
    unsigned long long adds = 0;
    for_shards(c, G, [&](size_t k, sfxb_ctx *sh) {
        for (size_t j = 0; j < G; ++j) CK(cudaStreamWaitEvent(sh->stream, c->shards[j]->ev_part, 0));
        HistBufs &B = hist_bufs(sh);
        cudaStream_t st = sh->stream;
        const size_t j0 = jlo[k], jl = jlo[k + 1] - jlo[k], cnt = (size_t)N * jl;
        uint32_t *hist = tree ? (uint32_t *)grow(sh->tree_buf[sh->tree_cur ^ 1], cnt * S4 * 4 + 64)
                              : bget<uint32_t>(B.g_hist, cnt * S4);
        if (k == 0) {
            unsigned long long *d_adds = reinterpret_cast<unsigned long long *>(bget<uint32_t>(B.g_misc, 4));
            CK(cudaMemsetAsync(d_adds, 0, 8, st));
            const int grid = (int)std::min<size_t>((2 * nkeys + 255) / 256, (size_t)sh->sms * 8);
            dev::k_adds_multi<<<grid, 256, 0, st>>>(reals, 2 * nkeys, d_adds);
            check_launch(*sh);
            CK(cudaMemcpyAsync(&adds, d_adds, 8, cudaMemcpyDeviceToHost, st));
        }
        if (cnt) {
            dispatch_class(sh->s, [&](auto sc) {
                constexpr int cs = decltype(sc)::value;
                using C = Cls<cs>;
                constexpr int NI = dev::kBlock / C::TH;
                auto kr = dev::k_reduce_peer<4 * cs, C::TH>;
                kr<<<occupancy_grid(*sh, kr, cnt, NI), dev::kBlock, 0, st>>>(arg(sh->mod_n2), parts, N, spn, j0, jl,
                                                                            hist);
                check_launch(*sh);
                if (!pairs.empty()) {
                    dev::Derived *d_pairs = bget<dev::Derived>(B.pairs, pairs.size());
                    CK(cudaMemcpyAsync(d_pairs, pairs.data(), pairs.size() * sizeof(dev::Derived),
                                       cudaMemcpyHostToDevice, st));
                    ok[k] = derive_siblings<cs>(sh, B, hist, (const uint32_t *)sh->tree_buf[sh->tree_cur].p, d_pairs,
                                                pairs.size(), jl);
                }
                if (!ok[k]) return;
                uint32_t *plain = bget<uint32_t>(B.g_plain, cnt * S4);
                auto kc = dev::k_from_mont_copy<4 * cs, C::TH>;
                kc<<<occupancy_grid(*sh, kc, cnt, NI), dev::kBlock, 0, st>>>(arg(sh->mod_n2), hist, cnt, plain);
                check_launch(*sh);
                d2h_cols(sh, out_slots, plain, N, spn, j0, jl, cw, S4);
            });
        }
        CK(cudaStreamSynchronize(st));
    });
    if (std::find(ok.begin(), ok.end(), 0) != ok.end()) {
        // some small-child slot is not a unit: rebuild this level directly
        for (sfxb_ctx *sh : c->shards) sh->tree_valid = false;
        std::vector<int32_t> none(N, -1);
        accumulate_group(c, g, bins, J, offs, N, rows, K, none.data(), out_slots, additions);
        return;
    }
    if (additions) *additions += adds;
    if (tree) {
        for (size_t k = 0; k < G; ++k) {
            sfxb_ctx *sh = c->shards[k];
            sh->tree_cur ^= 1;
            sh->tree_valid = true;
            sh->tree_gh = g;
            sh->tree_J = J;
            sh->tree_K = K;
            sh->tree_N = N;
            sh->tree_G = (uint32_t)G;
            sh->tree_j0 = (uint32_t)jlo[k];
            sh->tree_jl = (uint32_t)(jlo[k + 1] - jlo[k]);
        }
        c->tree_derived_nodes += pairs.size();
    }
}

} // namespace

// =================================================================== C ABI

extern "C" {

const char *sfxb_create_error(void) { return g_create_err.c_str(); }

int sfxb_ctx_create(sfxb_ctx **out, int device, const uint32_t *n, uint32_t n_words, const uint32_t *p,
                    const uint32_t *q, uint32_t pq_words) {
    if (!out || !n || n_words == 0) {
        g_create_err = "sfxb_ctx_create: bad arguments";
        return SFXB_ERR_ARG;
    }
    auto c = std::make_unique<sfxb_ctx>();
    int rc = guard(c.get(), [&] {
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) throw ApiError(SFXB_ERR_CUDA, "no such CUDA device");
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw ApiError(SFXB_ERR_CUDA, "libsfxb_cuda is built for sm_100a only");
        CK(cudaSetDevice(device));
        c->device = device;
        c->sms = prop.multiProcessorCount;
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));

        Big N = host::from_words(n, n_words);
        if ((N[0] & 1u) == 0 || host::bit_length(N) < 3) throw ApiError(SFXB_ERR_ARG, "modulus must be odd and > 4");
        const uint32_t nw = (uint32_t)((host::bit_length(N) + 31) / 32);
        int s = nw <= 8 ? 4 : nw <= 16 ? 8 : nw <= 32 ? 16 : nw <= 64 ? 32 : nw <= 96 ? 48 : 0;
        if (!s) throw ApiError(SFXB_ERR_UNSUPPORTED, "modulus wider than 3072 bits");
        c->s = s;
        c->nw = nw;
        c->n = N;
        c->n2 = host::mul(N, N);
        // key_id_of(n): FNV-1a over lower-case hex (he.cpp:30-38)
        {
            static const char *hex = "0123456789abcdef";
            std::string digits;
            size_t nb = host::bit_length(N);
            for (size_t i = (nb + 3) / 4; i-- > 0;) {
                uint32_t v = (N[i / 8] >> (4 * (i % 8))) & 0xf;
                digits.push_back(hex[v]);
            }
            uint64_t h = 14695981039346656037ULL;
            for (unsigned char ch : digits) {
                h ^= ch;
                h *= 1099511628211ULL;
            }
            c->key_id = h;
        }
        c->mod_n2 = dev_mod(*c, c->n2, 4 * s);
        c->mod_n = dev_mod(*c, N, 2 * s);
        c->d_n = dev_big(*c, N, 2 * s);
        c->d_n4 = dev_big(*c, N, 4 * s);
        c->d_n2w = dev_big(*c, c->n2, 4 * s);
        host::MontHost mn2(c->n2, 4 * s);
        c->mh_n2 = std::make_unique<host::MontHost>(c->n2, 4 * s);
        c->d_nR_n2 = dev_big(*c, mn2.to_mont(N), 4 * s);
        c->d_dig_n = dev_digits(*c, N, kWindowN, c->nd_n);
        // base-n digit constants (passive-party K2, padic.cuh)
        c->n_digits = host::bit_length(N) == 64u * s;
        {
            host::MontHost mnn(N, 2 * s);
            c->d_negR_n = dev_big(*c, host::sub(N, mnn.r1), 2 * s);
            std::vector<uint32_t> one(4 * (size_t)s);
            std::copy(mnn.r1.begin(), mnn.r1.end(), one.begin());
            std::copy(mnn.r1.begin(), mnn.r1.end(), one.begin() + 2 * s);
            c->d_one_nd = dev_upload(*c, one.data(), one.size());
            // digits (A, B) of V = R⁴ mod n² (R = 2^(32·2s); mn2's R² is R⁴):
            // V ≡ A·R + B·n (mod n²), A = V·R⁻¹ mod n, B = (V − A·R mod n²)/n
            // (exact, by the 2-adic inverse of n)
            const Big V = mn2.r2;
            const Big A = host::mod(mnn.mont_mul(host::mod(V, N), host::from_u64(1)), N);
            Big AR(4 * (size_t)s + 1, 0);
            for (size_t i = 0; i < A.size() && i < 2 * (size_t)s; ++i) AR[2 * s + i] = A[i];
            const Big x = host::mod(AR, c->n2);
            const Big T = host::cmp(V, x) >= 0 ? host::sub(V, x) : host::sub(host::add(V, c->n2), x);
            const Big B = host::low(host::mul(host::low(T, 2 * s), host::inv_pow2(N, 2 * s)), 2 * s);
            Big chk = host::mod(host::add(AR, host::mul(B, N)), c->n2);
            host::trim(chk);
            Big Vt = V;
            host::trim(Vt);
            if (host::cmp(chk, Vt) != 0 || host::cmp(B, N) >= 0)
                throw ApiError(SFXB_ERR_ARG, "base-n digits of R^4 mod n^2 (modulus outside the digit class)");
            std::vector<uint32_t> r4(4 * (size_t)s, 0u);
            const Big Ap = host::pad(A, 2 * s), Bp = host::pad(B, 2 * s);
            std::copy(Ap.begin(), Ap.begin() + 2 * s, r4.begin());
            std::copy(Bp.begin(), Bp.begin() + 2 * s, r4.begin() + 2 * s);
            c->d_r4_nd = dev_upload(*c, r4.data(), r4.size());
        }
        if (p && q && pq_words) {
            Big P = host::from_words(p, pq_words), Q = host::from_words(q, pq_words);
            if (host::cmp(host::mul(P, Q), N) != 0) throw ApiError(SFXB_ERR_ARG, "private key inconsistent: p·q != n");
            if (host::cmp(P, Q) == 0) throw ApiError(SFXB_ERR_ARG, "primes must be distinct");
            if ((P[0] & 1u) == 0 || (Q[0] & 1u) == 0) throw ApiError(SFXB_ERR_ARG, "primes must be odd");
            if (host::bit_length(P) > 32u * s || host::bit_length(Q) > 32u * s)
                throw ApiError(SFXB_ERR_UNSUPPORTED, "unbalanced primes are outside the CRT size class");
            // q < 2p and p < 2q keep the single conditional subtractions of the CRT combine exact
            if (host::cmp(Q, host::add(P, P)) >= 0 || host::cmp(P, host::add(Q, Q)) >= 0)
                throw ApiError(SFXB_ERR_UNSUPPORTED, "primes differ by more than a factor of two");
            c->has_priv = true;
            c->p = P;
            c->q = Q;
            const Big PQ[2] = {P, Q};
            struct Win {
                uint64_t e1, pr, pm1;
                std::vector<uint8_t> dig_pr, dig_pm1;
            } host_window[2];
            c->p2_digits = host::bit_length(P) == 32u * s && host::bit_length(Q) == 32u * s;
            for (int i = 0; i < 2; ++i) {
                const Big &pr = PQ[i], &ot = PQ[1 - i];
                Big pr2 = host::mul(pr, pr);
                c->mod_pq[i] = dev_mod(*c, pr, s);
                c->mod_pq2[i] = dev_mod(*c, pr2, 2 * s);
                Big pm1 = host::sub(pr, host::from_u64(1));
                c->d_dig_e1[i] = dev_digits(*c, host::mod(ot, pm1), kWindow, c->nd_e1[i]);
                c->d_dig_pq[i] = dev_digits(*c, pr, kWindow, c->nd_pq[i]);
                c->d_dig_m1[i] = dev_digits(*c, pm1, kWindow, c->nd_m1[i]);
                // profiling units: multiplications mod p² (step 1 runs mod p: 1/4 of the products)
                host_window[i] = {pow_mmuls(host::mod(ot, pm1), kWindow), pow_mmuls(pr, kWindow),
                                  pow_mmuls(pm1, kWindow), host::sliding_ops(pr, kWindow),
                                  host::sliding_ops(pm1, kWindow)};
                c->d_ops_pq[i] = dev_upload(*c, host_window[i].dig_pr.data(), host_window[i].dig_pr.size());
                c->nops_pq[i] = (int)host_window[i].dig_pr.size() / 2;
                c->d_ops_m1[i] = dev_upload(*c, host_window[i].dig_pm1.data(), host_window[i].dig_pm1.size());
                c->nops_m1[i] = (int)host_window[i].dig_pm1.size() / 2;
                {
                    const std::vector<uint8_t> e1ops = host::sliding_ops(host::mod(ot, pm1), kWindow);
                    c->d_ops_e1[i] = dev_upload(*c, e1ops.data(), e1ops.size());
                    c->nops_e1[i] = (int)e1ops.size() / 2;
                    // step 1 (mod p, s limbs) runs the sliding program
                    uint64_t m1 = 1 + ((1ull << (kWindow - 1)) - 1);
                    for (size_t k = 1; k < e1ops.size() / 2; ++k) m1 += e1ops[2 * k] + (e1ops[2 * k + 1] ? 1 : 0);
                    host_window[i].e1 = m1;
                }
                c->d_pinv[i] = dev_big(*c, host::inv_pow2(pr, s), s);
                // h = (−other mod prime)^-1 mod prime, in Montgomery form
                Big negot = host::sub(pr, host::mod(ot, pr));
                Big h = host::inv_mod_prime(negot, pr, s);
                host::MontHost mp(pr, s);
                c->d_hR[i] = dev_big(*c, mp.to_mont(h), s);
                c->d_cdec[i] = dev_big(*c, mp.from_mont(h), s);
                c->d_negR[i] = dev_big(*c, host::sub(pr, mp.r1), s); // p − (R mod p)
                {
                    std::vector<uint32_t> one(2 * (size_t)s);
                    std::copy(mp.r1.begin(), mp.r1.end(), one.begin());
                    std::copy(mp.r1.begin(), mp.r1.end(), one.begin() + s);
                    c->d_one_p2[i] = dev_upload(*c, one.data(), one.size());
                }
            }
            // profiling units: 32×32 products per item of the exponentiation kernels
            const uint64_t pp = 2ull * s * s + s, pp2 = 2ull * (2 * s) * (2 * s) + 2 * s;
            int p2_tp = 0;
            dispatch_class(s, [&](auto sc) { p2_tp = Cls<decltype(sc)::value>::TP; });
            const bool sqr = dev::kSqrP2 && p2_tp == 1;
            for (int i = 0; i < 2; ++i) {
                const Win &w = host_window[i];
                c->prod_enc += w.e1 * pp; // step 1 mod p
                if (c->p2_digits) {
                    c->prod_enc += dev::p2_pow_products(w.dig_pr.data(), (int)w.dig_pr.size() / 2, kWindow, s, sqr) + 2 * pp;
                    c->prod_dec += dev::p2_pow_products(w.dig_pm1.data(), (int)w.dig_pm1.size() / 2, kWindow, s, sqr) + 2 * pp;
                } else {
                    c->prod_enc += w.pr * pp2;
                    c->prod_dec += w.pm1 * pp2;
                }
            }
            host::MontHost mp(P, s), mp2(host::mul(P, P), 2 * s), mn(N, 2 * s);
            Big P2 = host::mul(P, P), Q2 = host::mul(Q, Q);
            // (q²)^-1 mod p² = q²^(p(p−1)−1) mod p²  (Euler)
            Big phi = host::mul(P, host::sub(P, host::from_u64(1)));
            Big qq_inv = mp2.pow(host::mod(Q2, P2), host::sub(phi, host::from_u64(1)));
            c->d_qq_inv_m = dev_big(*c, mp2.to_mont(qq_inv), 2 * s);
            c->d_q2R_n2 = dev_big(*c, mn2.to_mont(Q2), 4 * s);
            Big qinv = host::inv_mod_prime(host::mod(Q, P), P, s);
            c->d_qinvR_p = dev_big(*c, mp.to_mont(qinv), s);
            c->d_qR_n = dev_big(*c, mn.to_mont(Q), 2 * s);
        }
        CK(cudaDeviceSynchronize());
    });
    if (rc != SFXB_OK) {
        g_create_err = c->err;
        for (void *d : c->owned) cudaFree(d);
        if (c->stream) cudaStreamDestroy(c->stream);
        return rc;
    }
    *out = c.release();
    return SFXB_OK;
}

int sfxb_ctx_create_multi(sfxb_ctx **out, const int *devices, uint32_t n_devices, const uint32_t *n,
                          uint32_t n_words, const uint32_t *p, const uint32_t *q, uint32_t pq_words) {
    if (!out || !devices || n_devices == 0 || n_devices > (uint32_t)dev::kMaxShards) {
        g_create_err = "sfxb_ctx_create_multi: bad arguments (1 to 16 devices)";
        return SFXB_ERR_ARG;
    }
    if (n_devices == 1) return sfxb_ctx_create(out, devices[0], n, n_words, p, q, pq_words);
    std::vector<sfxb_ctx *> sh(n_devices, nullptr);
    auto undo = [&] {
        for (sfxb_ctx *x : sh)
            if (x) {
                x->shards.clear();
                sfxb_ctx_destroy(x);
            }
    };
    for (uint32_t k = 0; k < n_devices; ++k) {
        const int rc = sfxb_ctx_create(&sh[k], devices[k], n, n_words, p, q, pq_words);
        if (rc != SFXB_OK) {
            std::string e = g_create_err;
            undo();
            g_create_err = e;
            return rc;
        }
    }
    sfxb_ctx *c = sh[0];
    const int rc = guard(c, [&] {
        // the cross-shard reduce reads peer memory directly: every pair of
        // distinct devices needs P2P access (NVLink / NVSwitch on a B200 box)
        for (uint32_t i = 0; i < n_devices; ++i) {
            CK(cudaSetDevice(devices[i]));
            for (uint32_t j = 0; j < n_devices; ++j) {
                if (devices[j] == devices[i]) continue;
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
                if (!can)
                    throw ApiError(SFXB_ERR_UNSUPPORTED, "device group: no peer access from device " +
                                                             std::to_string(devices[i]) + " to " +
                                                             std::to_string(devices[j]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
                else CK(e);
            }
            CK(cudaEventCreateWithFlags(&sh[i]->ev_part, cudaEventDisableTiming));
        }
        CK(cudaSetDevice(devices[0]));
        c->shards = sh;
    });
    if (rc != SFXB_OK) {
        g_create_err = c->err;
        undo();
        return rc;
    }
    *out = c;
    return SFXB_OK;
}

void *sfxb_host_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    return p;
}

void sfxb_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

int sfxb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}

uint32_t sfxb_ctx_n_shards(const sfxb_ctx *c) { return c->shards.empty() ? 1u : (uint32_t)c->shards.size(); }

// encryptions per wave on one shard's device (shards[0] is the group itself)
static size_t enc_wave_one(const sfxb_ctx *c) {
    size_t items = 0;
    try {
        CK(cudaSetDevice(c->device));
        dispatch_class(c->s, [&](auto sc) {
            constexpr int cs = decltype(sc)::value;
            using C = Cls<cs>;
            // the widest exponentiation of the path encrypt_dev takes; one
            // block row per prime, so a wave holds per_sm·SMs/2 blocks per prime
            auto wave = [&](auto k, int tpi, int rows) {
                int per_sm = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, dev::kBlock, 0));
                return (size_t)std::max(per_sm, 1) * c->sms * (dev::kBlock / tpi) / rows;
            };
            if (!c->has_priv) items = wave(dev::k_pow_n2<4 * cs, C::TN, kWindowN>, C::TN, 1);
            else if (c->p2_digits) items = wave(dev::k_p2_pow<cs, C::TP, kWindow, 0>, C::TP, 2);
            else items = wave(dev::k_enc_step2<2 * cs, C::T2, kWindow>, C::T2, 2);
        });
    } catch (...) {
        return 0;
    }
    return items;
}

size_t sfxb_ctx_enc_wave(const sfxb_ctx *c) {
    if (!c) return 0;
    if (c->shards.empty()) return enc_wave_one(c);
    size_t t = 0;
    for (const sfxb_ctx *sh : c->shards) t += enc_wave_one(sh);
    return t;
}
int sfxb_ctx_shard_device(const sfxb_ctx *c, uint32_t k) {
    if (c->shards.empty()) return k == 0 ? c->device : -1;
    return k < c->shards.size() ? c->shards[k]->device : -1;
}

void sfxb_ctx_destroy(sfxb_ctx *c) {
    if (!c) return;
    if (!c->shards.empty()) {
        std::vector<sfxb_ctx *> sh;
        sh.swap(c->shards);
        for (size_t k = 1; k < sh.size(); ++k) sfxb_ctx_destroy(sh[k]);
    }
    cudaSetDevice(c->device);
    if (c->ev_part) cudaEventDestroy(c->ev_part);
    for (auto &e : c->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    free_hist_bufs(c);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (void *d : c->owned) cudaFree(d);
    if (c->scratch_table.p) cudaFree(c->scratch_table.p);
    for (auto &b : c->tree_buf)
        if (b.p) cudaFree(b.p);
    if (c->spare_gh) cudaFree(c->spare_gh);
    if (c->spare_flags) cudaFree(c->spare_flags);
    for (auto &b : c->tmp)
        if (b.p) cudaFree(b.p);
    for (auto &b : c->io)
        if (b.p) cudaFree(b.p);
    for (auto &kv : c->dec_cache)
        for (int i = 0; i < 2; ++i) {
            if (kv.second.cts[i].p) cudaFree(kv.second.cts[i].p);
            if (kv.second.plain[i].p) cudaFree(kv.second.plain[i].p);
        }
    for (auto &b : c->host_pinned)
        if (b.p) cudaFreeHost(b.p);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char *sfxb_last_error(const sfxb_ctx *c) { return c ? c->err.c_str() : "null context"; }
uint32_t sfxb_ctx_n_words(const sfxb_ctx *c) { return c->nw; }
uint32_t sfxb_ctx_ct_words(const sfxb_ctx *c) { return 2 * c->nw; }
int sfxb_ctx_has_private(const sfxb_ctx *c) { return c->has_priv ? 1 : 0; }
uint64_t sfxb_ctx_key_id(const sfxb_ctx *c) { return c->key_id; }
uint64_t sfxb_ctx_launches(const sfxb_ctx *c) {
    uint64_t t = c->launches;
    for (size_t k = 1; k < c->shards.size(); ++k) t += c->shards[k]->launches;
    return t;
}
uint64_t sfxb_ctx_dec_derived(const sfxb_ctx *c) {
    uint64_t t = c->dec_derived;
    for (size_t k = 1; k < c->shards.size(); ++k) t += c->shards[k]->dec_derived;
    return t;
}
void *sfxb_ctx_stream(sfxb_ctx *c) { return (void *)c->stream; }
int sfxb_ctx_profile(sfxb_ctx *c, int enable) {
    return guard(c, [&] {
        const size_t G = std::max<size_t>(1, c->shards.size());
        for (size_t k = 0; k < G; ++k) {
            sfxb_ctx *x = G > 1 ? c->shards[k] : c;
            CK(cudaSetDevice(x->device));
            CK(cudaStreamSynchronize(x->stream));
            for (auto &p : x->prof) {
                for (auto &e : p.ev) {
                    cudaEventDestroy(e.first);
                    cudaEventDestroy(e.second);
                }
                p = CtxState::Prof{};
            }
            x->profile = enable != 0;
        }
        CK(cudaSetDevice(c->device));
    });
}

// kernel-family totals over the context (all shards of a device group: the
// times are summed GPU time, not wall time)
int sfxb_ctx_kernel_stats(sfxb_ctx *c, int family, uint64_t *launches, double *ms, uint64_t *modmuls) {
    return guard(c, [&] {
        if (family < 0 || family >= 4) throw ApiError(SFXB_ERR_ARG, "kernel family out of range");
        const size_t G = std::max<size_t>(1, c->shards.size());
        uint64_t nl = 0, mm = 0;
        double t_ms = 0;
        for (size_t k = 0; k < G; ++k) {
            sfxb_ctx *x = G > 1 ? c->shards[k] : c;
            CK(cudaSetDevice(x->device));
            CK(cudaStreamSynchronize(x->stream));
            auto &p = x->prof[family];
            for (auto &e : p.ev) {
                float t = 0;
                CK(cudaEventElapsedTime(&t, e.first, e.second));
                p.ms_done += t;
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
            p.ev.clear();
            nl += p.launches;
            t_ms += p.ms_done;
            mm += p.modmuls;
        }
        CK(cudaSetDevice(c->device));
        if (launches) *launches = nl;
        if (ms) *ms = t_ms;
        if (modmuls) *modmuls = mm;
    });
}

int sfxb_ctx_kernel_time(sfxb_ctx *c, int family, uint64_t *launches, double *ms) {
    return sfxb_ctx_kernel_stats(c, family, launches, ms, nullptr);
}

int sfxb_ctx_sync(sfxb_ctx *c) {
    return guard(c, [&] {
        for (size_t k = 1; k < c->shards.size(); ++k) {
            CK(cudaSetDevice(c->shards[k]->device));
            CK(cudaStreamSynchronize(c->shards[k]->stream));
        }
        CK(cudaSetDevice(c->device));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int sfxb_encode_check(sfxb_ctx *c, double x, uint32_t scale, int64_t *q_out) {
    return guard(c, [&] {
        // encode_fixed (he.cpp:125-136) + fixed_encode_ll (fixed_point.hpp:13-15)
        if (!std::isfinite(x)) throw ApiError(SFXB_ERR_RANGE, "encode_fixed: value must be finite");
        if (std::abs(x) >= std::ldexp(1.0, (int)(62 - scale)))
            throw ApiError(SFXB_ERR_RANGE, "encode_fixed: value too large for the fixed-point grid");
        int64_t qv = std::llround(std::ldexp(x, (int)scale));
        uint64_t mag = qv < 0 ? (uint64_t)(-(qv + 1)) + 1u : (uint64_t)qv;
        Big twice = host::add(host::from_u64(mag), host::from_u64(mag));
        if (host::cmp(twice, c->n) >= 0)
            throw ApiError(SFXB_ERR_RANGE, "encode_fixed: |x|·2^scale_bits must stay below n/2");
        *q_out = qv;
    });
}

int sfxb_gradients_dev(sfxb_ctx *c, const double *d_prob, const uint8_t *d_labels, size_t n, uint32_t scale,
                       int64_t *d_q, double *d_gh, size_t *first_bad) {
    const NvtxRange nvtx_("sfxb_gradients_dev");
    return guard(c, [&] {
        if (scale > 62) throw ApiError(SFXB_ERR_ARG, "gradients: scale_bits above 62");
        CK(cudaSetDevice(c->device));
        dev::GradArgs a{};
        a.prob = d_prob;
        a.label = d_labels;
        a.n = n;
        a.scale = (int)scale;
        a.lim = std::ldexp(1.0, (int)(62 - scale));
        a.n64 = host::bit_length(c->n) > 64
                    ? 0
                    : (uint64_t)(c->n.size() > 0 ? c->n[0] : 0) | ((uint64_t)(c->n.size() > 1 ? c->n[1] : 0) << 32);
        a.q = d_q;
        a.gh = d_gh;
        unsigned long long *st = (unsigned long long *)grow(c->tmp[3], 64);
        const unsigned long long init[2] = {2ull * n, 0ull};
        CK(cudaMemcpyAsync(st, init, 16, cudaMemcpyHostToDevice, c->stream));
        a.status = st;
        if (n) {
            const int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)c->sms * 8);
            dev::k_gradients<<<grid, 256, 0, c->stream>>>(a);
            check_launch(*c);
        }
        unsigned long long h[2];
        CK(cudaMemcpyAsync(h, st, 16, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (first_bad) *first_bad = (size_t)h[0];
        if (h[0] < 2ull * n)
            throw ApiError(SFXB_ERR_RANGE, h[1] == 1   ? "encode_fixed: value must be finite"
                                           : h[1] == 2 ? "encode_fixed: value too large for the fixed-point grid"
                                                       : "encode_fixed: |x|·2^scale_bits must stay below n/2");
    });
}

int sfxb_encode_batch(sfxb_ctx *c, const double *x, size_t count, uint32_t scale, int64_t *q_out,
                      size_t *first_bad) {
    const NvtxRange nvtx_("sfxb_encode_batch");
    return guard(c, [&] {
        // encode_fixed's checks (he.cpp:125-136) per value, on all host
        // threads; |q| <= 2^62 after the grid check, so 2|q| fits 64 bits and
        // the n/2 bound is one compare against n's low word (or none when n
        // is wider than 64 bits).
        if (scale > 62) throw ApiError(SFXB_ERR_ARG, "encode: scale_bits above 62");
        const double lim = std::ldexp(1.0, (int)(62 - scale));
        const bool wide = host::bit_length(c->n) > 64;
        const uint64_t n64 = wide ? ~0ull
                                  : (uint64_t)(c->n.size() > 0 ? c->n[0] : 0) |
                                        ((uint64_t)(c->n.size() > 1 ? c->n[1] : 0) << 32);
        const unsigned T = (unsigned)std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(),
                                                                          count / 65536));
        std::vector<size_t> bad(T, count);
        std::vector<int> why(T, 0);
        auto run = [&](unsigned t) {
            const size_t lo = count * t / T, hi = count * (t + 1) / T;
            for (size_t i = lo; i < hi; ++i) {
                const double v = x[i];
                if (!std::isfinite(v)) { bad[t] = i; why[t] = 1; return; }
                if (std::abs(v) >= lim) { bad[t] = i; why[t] = 2; return; }
                const int64_t qv = std::llround(std::ldexp(v, (int)scale));
                const uint64_t mag = qv < 0 ? (uint64_t)(-(qv + 1)) + 1u : (uint64_t)qv;
                if (!wide && 2 * mag >= n64) { bad[t] = i; why[t] = 3; return; }
                q_out[i] = qv;
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < T; ++t) pool.emplace_back(run, t);
        run(0);
        for (auto &th : pool) th.join();
        size_t first = count;
        int w = 0;
        for (unsigned t = 0; t < T; ++t)
            if (bad[t] < first) {
                first = bad[t];
                w = why[t];
            }
        if (first_bad) *first_bad = first;
        if (first < count)
            throw ApiError(SFXB_ERR_RANGE, w == 1   ? "encode_fixed: value must be finite"
                                           : w == 2 ? "encode_fixed: value too large for the fixed-point grid"
                                                    : "encode_fixed: |x|·2^scale_bits must stay below n/2");
    });
}

int sfxb_ctx_set_low_priority(sfxb_ctx *c) {
    return guard(c, [&] {
        if (is_group(c)) throw ApiError(SFXB_ERR_UNSUPPORTED, "stream priority: single-device contexts only");
        CK(cudaSetDevice(c->device));
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        CK(cudaStreamSynchronize(c->stream));
        cudaStream_t st = nullptr;
        CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, least));
        CK(cudaStreamDestroy(c->stream));
        c->stream = st;
    });
}

int sfxb_blind_create(sfxb_ctx *c, size_t capacity, sfxb_blind **out) {
    return guard(c, [&] {
        if (is_group(c)) throw ApiError(SFXB_ERR_UNSUPPORTED, "blinding queue: single-device contexts only");
        CK(cudaSetDevice(c->device));
        auto b = std::make_unique<sfxb_blind>();
        b->device = c->device;
        b->s = (uint32_t)c->s;
        b->nw = c->nw;
        b->key_id = c->key_id;
        b->cap = capacity;
        CK(cudaMalloc(&b->d, std::max<size_t>(capacity, 1) * 4 * (size_t)c->s * 4));
        *out = b.release();
    });
}

void sfxb_blind_free(sfxb_blind *b) {
    if (!b) return;
    cudaSetDevice(b->device);
    cudaFree(b->d);
    delete b;
}

size_t sfxb_blind_size(const sfxb_blind *b) { return b ? b->size : 0; }

int sfxb_blind_append(sfxb_ctx *c, sfxb_blind *b, const uint32_t *r, size_t count, uint8_t *r_flags) {
    const NvtxRange nvtx_("sfxb_blind_append");
    return guard(c, [&] {
        if (!b || b->key_id != c->key_id || b->device != c->device || is_group(c))
            throw ApiError(SFXB_ERR_ARG, "blinding queue: another key or device");
        if (count == 0) return;
        // compact: live entries to the front when the tail has no room
        const size_t S4 = 4 * (size_t)c->s;
        CK(cudaSetDevice(c->device));
        if (b->head + b->size + count > b->cap) {
            if (b->size + count > b->cap) throw ApiError(SFXB_ERR_ARG, "blinding queue: capacity exceeded");
            if (b->size)
                CK(cudaMemcpyAsync(b->d, b->d + b->head * S4, b->size * S4 * 4, cudaMemcpyDeviceToDevice, c->stream));
            b->head = 0;
        }
        // r^n mod n² = Enc(0, r): the encryption pipeline with plaintext 0
        IoBuf<int64_t> dq(c->io[0], count);
        CK(cudaMemsetAsync(dq.p, 0, count * 8, c->stream));
        const size_t Sn = 2 * (size_t)c->s;
        IoBuf<uint32_t> dr(c->io[1], count * Sn);
        IoBuf<uint8_t> dflags(c->io[3], count);
        CK(cudaMemsetAsync(dflags.p, 0, count, c->stream));
        h2d_padded(c, dr.p, r, count, c->nw, Sn);
        int st = SFXB_OK;
        try {
            encrypt_dev(c, dq.p, dr.p, count, b->d + (b->head + b->size) * S4, dflags.p);
        } catch (const ApiError &e) {
            if (e.code != SFXB_ERR_COPRIME) throw;
            st = e.code;
            c->err = e.what();
        }
        if (r_flags) {
            CK(cudaMemcpyAsync(r_flags, dflags.p, count, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        if (st != SFXB_OK) throw ApiError(st, c->err); // nothing appended
        b->size += count;
    });
}

int sfxb_blind_pop(sfxb_blind *b, size_t count) {
    if (!b || count > b->size) return SFXB_ERR_ARG;
    b->head += count;
    b->size -= count;
    if (b->size == 0) b->head = 0;
    return SFXB_OK;
}

int sfxb_encrypt_blind(sfxb_ctx *c, sfxb_blind *b, const int64_t *q_fixed, const uint32_t *m_words, size_t count,
                       uint32_t *out_cts) {
    const NvtxRange nvtx_("sfxb_encrypt_blind");
    return guard(c, [&] {
        if (!b || b->key_id != c->key_id || b->device != c->device || is_group(c))
            throw ApiError(SFXB_ERR_ARG, "blinding queue: another key or device");
        if (count > b->size) throw ApiError(SFXB_ERR_ARG, "blinding queue: fewer precomputed powers than requested");
        if (!q_fixed == !m_words) throw ApiError(SFXB_ERR_ARG, "encrypt: exactly one of q_fixed / m_words");
        if (count == 0) return;
        CK(cudaSetDevice(c->device));
        const size_t Sn = 2 * (size_t)c->s, S4 = 4 * (size_t)c->s;
        if (m_words) {
            const std::vector<uint32_t> nw_words = host::pad(c->n, c->nw);
            for (size_t i = 0; i < count; ++i) {
                const uint32_t *x = m_words + i * c->nw;
                bool lt = false;
                for (uint32_t k = c->nw; k-- > 0;)
                    if (x[k] != nw_words[k]) {
                        lt = x[k] < nw_words[k];
                        break;
                    }
                if (!lt) throw ApiError(SFXB_ERR_RANGE, "encrypt: plaintext out of range [0, n)");
            }
        }
        IoBuf<int64_t> dq(c->io[0], m_words ? 1 : count);
        IoBuf<uint32_t> dm(c->io[4], m_words ? count * Sn : 1), dout(c->io[2], count * S4);
        if (m_words) h2d_padded(c, dm.p, m_words, count, c->nw, Sn);
        else CK(cudaMemcpyAsync(dq.p, q_fixed, count * 8, cudaMemcpyHostToDevice, c->stream));
        // online step: c = (1 + m·n)·Y mod n² with Y the queued r^n mod n²
        dev::EncArgs a{};
        a.qfix = m_words ? nullptr : dq.p;
        a.mw = m_words ? dm.p : nullptr;
        a.count = count;
        a.mod_n2 = arg(c->mod_n2);
        a.n4 = c->d_n4;
        a.nR_n2 = c->d_nR_n2;
        a.y = b->d + b->head * S4;
        a.out = dout.p;
        dispatch_class(c->s, [&](auto sc) {
            constexpr int cs = decltype(sc)::value;
            using C = Cls<cs>;
            auto k = dev::k_enc_combine<cs, C::TC>;
            constexpr int NI = dev::kBlock / C::TC;
            k<<<occupancy_grid(*c, k, count, NI), dev::kBlock, 0, c->stream>>>(a, 0);
            check_launch(*c);
        });
        d2h_padded(c, out_cts, dout.p, count, 2 * c->nw, S4);
        b->head += count;
        b->size -= count;
        if (b->size == 0) b->head = 0;
    });
}

int sfxb_encrypt_dev(sfxb_ctx *c, const int64_t *d_q, const uint32_t *d_r, size_t count, uint32_t *d_out,
                     uint8_t *d_flags) {
    const NvtxRange nvtx_("sfxb_encrypt_dev");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        encrypt_dev(c, d_q, d_r, count, d_out, d_flags);
    });
}


int sfxb_encrypt(sfxb_ctx *c, const int64_t *q_fixed, const uint32_t *r, size_t count, uint32_t *out_cts,
                 uint8_t *r_flags) {
    const NvtxRange nvtx_("sfxb_encrypt");
    return guard(c, [&] {
        if (is_group(c)) encrypt_group(c, q_fixed, nullptr, r, count, out_cts, r_flags);
        else encrypt_host(c, q_fixed, nullptr, r, count, out_cts, r_flags);
    });
}

int sfxb_encrypt_plain(sfxb_ctx *c, const uint32_t *m_words, const uint32_t *r, size_t count, uint32_t *out_cts,
                       uint8_t *r_flags) {
    const NvtxRange nvtx_("sfxb_encrypt_plain");
    return guard(c, [&] {
        if (is_group(c)) encrypt_group(c, nullptr, m_words, r, count, out_cts, r_flags);
        else encrypt_host(c, nullptr, m_words, r, count, out_cts, r_flags);
    });
}

int sfxb_add(sfxb_ctx *c, const uint32_t *a, const uint32_t *b, size_t count, uint32_t *out) {
    const NvtxRange nvtx_("sfxb_add");
    return guard(c, [&] {
        if (is_group(c)) add_group(c, a, b, count, out);
        else add_host(c, a, b, count, out);
    });
}

int sfxb_decrypt_dev(sfxb_ctx *c, const uint32_t *d_cts, size_t count, uint32_t scale, double *d_values,
                     uint32_t *d_plain, uint64_t *decryptions) {
    const NvtxRange nvtx_("sfxb_decrypt_dev");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        decrypt_dev(c, d_cts, count, scale, d_values, d_plain, decryptions);
    });
}

int sfxb_decrypt_tree(sfxb_ctx *c, uint64_t tag, const uint32_t *cts, uint32_t n_nodes, uint32_t spn,
                      const int32_t *parent, uint32_t scale, double *out_values, uint64_t *decryptions) {
    const NvtxRange nvtx_("sfxb_decrypt_tree");
    return guard(c, [&] {
        if (is_group(c)) decrypt_tree_group(c, tag, cts, n_nodes, spn, parent, scale, out_values, decryptions);
        else decrypt_tree_impl(c, tag, cts, n_nodes, spn, 0, spn, parent, scale, out_values, decryptions);
    });
}

int sfxb_decrypt(sfxb_ctx *c, const uint32_t *cts, size_t count, uint32_t scale, double *out_values,
                 uint32_t *out_plain, uint64_t *decryptions) {
    const NvtxRange nvtx_("sfxb_decrypt");
    return guard(c, [&] {
        if (is_group(c)) decrypt_group(c, cts, count, scale, out_values, out_plain, decryptions);
        else decrypt_host(c, cts, count, scale, out_values, out_plain, decryptions);
    });
}

int sfxb_gh_upload(sfxb_ctx *c, const uint32_t *gh_cts, uint32_t n_samples, sfxb_gh **out) {
    const NvtxRange nvtx_("sfxb_gh_upload");
    return guard(c, [&] {
        if (is_group(c)) {
            *out = gh_upload_group(c, gh_cts, n_samples);
            return;
        }
        CK(cudaSetDevice(c->device));
        std::unique_ptr<sfxb_gh> g(gh_alloc(c, n_samples));
        gh_upload_pipelined(c, g.get(), gh_cts);
        CK(cudaStreamSynchronize(c->stream));
        *out = g.release();
    });
}

int sfxb_gh_from_dev(sfxb_ctx *c, const uint32_t *d_gh, uint32_t n_samples, sfxb_gh **out) {
    const NvtxRange nvtx_("sfxb_gh_from_dev");
    return guard(c, [&] {
        if (is_group(c)) throw ApiError(SFXB_ERR_UNSUPPORTED, "gh_from_dev: device-pointer entry points are single-device");
        CK(cudaSetDevice(c->device));
        std::unique_ptr<sfxb_gh> g(gh_alloc(c, n_samples));
        const size_t S4 = 4 * (size_t)c->s;
        CK(cudaMemcpyAsync(g->d, d_gh, 2 * (size_t)n_samples * S4 * 4, cudaMemcpyDeviceToDevice, c->stream));
        gh_prepare(c, g.get());
        CK(cudaStreamSynchronize(c->stream));
        *out = g.release();
    });
}

void sfxb_gh_free(sfxb_gh *g) {
    if (!g) return;
    sfxb_ctx *c = g->ctx;
    if (c->tree_gh == g) c->tree_valid = false;
    if (!g->parts.empty()) { // device group: one handle per shard
        for (sfxb_gh *p : g->parts)
            if (p) sfxb_gh_free(p);
        cudaSetDevice(c->device);
        delete g;
        return;
    }
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (!c->spare_gh) { // keep as the context's spare
        c->spare_gh = g->d;
        c->spare_flags = g->flags;
        c->spare_gh_bytes = g->bytes;
        c->spare_flags_bytes = g->fbytes;
    } else {
        cudaFree(g->d);
        cudaFree(g->flags);
    }
    delete g;
}

int sfxb_accumulate_dev(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *d_bins, uint32_t n_features,
                        const uint32_t *d_node_offsets, uint32_t n_nodes, const uint32_t *d_rows, uint32_t n_rows,
                        uint32_t n_bins, uint32_t *d_out, int mont_out, uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate_dev");
    return guard(c, [&] {
        if (g && !g->parts.empty())
            throw ApiError(SFXB_ERR_UNSUPPORTED, "accumulate: device-pointer entry points take a single-device handle");
        CK(cudaSetDevice(c->device));
        accumulate_dev(c, g, d_bins, n_features, d_node_offsets, n_nodes, d_rows, n_rows, n_bins, d_out, mont_out,
                       additions);
    });
}

int sfxb_accumulate(sfxb_ctx *c, const uint32_t *gh_cts, uint32_t n_samples, const uint16_t *bins, uint32_t J,
                    const uint32_t *node_offsets, uint32_t N, const uint32_t *rows, uint32_t K, uint32_t *out_slots,
                    uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        for (uint32_t i = 0; i < N; ++i)
            if (node_offsets[i + 1] < node_offsets[i]) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets decrease");
        const uint32_t R = N ? node_offsets[N] - node_offsets[0] : 0;
        if (N && node_offsets[0] != 0) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets must start at 0");
        std::unique_ptr<sfxb_gh, void (*)(sfxb_gh *)> g(nullptr, sfxb_gh_free);
        {
            sfxb_gh *gp = nullptr;
            int rc = sfxb_gh_upload(c, gh_cts, n_samples, &gp);
            if (rc != SFXB_OK) throw ApiError(rc, c->err);
            g.reset(gp);
        }
        if (is_group(c)) {
            accumulate_group(c, g.get(), bins, J, node_offsets, N, rows, K, nullptr, out_slots, additions);
            return;
        }
        const size_t S4 = 4 * (size_t)c->s, nslots = 2ull * N * J * K;
        IoBuf<uint16_t> db(c->io[0], (size_t)J * n_samples);
        IoBuf<uint32_t> doff(c->io[1], (size_t)N + 1), drows(c->io[2], R ? R : 1), dout(c->io[3], nslots * S4);
        if ((size_t)J * n_samples)
            CK(cudaMemcpyAsync(db.p, bins, (size_t)J * n_samples * 2, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(doff.p, node_offsets, ((size_t)N + 1) * 4, cudaMemcpyHostToDevice, c->stream));
        if (R) CK(cudaMemcpyAsync(drows.p, rows, (size_t)R * 4, cudaMemcpyHostToDevice, c->stream));
        accumulate_dev(c, g.get(), db.p, J, doff.p, N, drows.p, R, K, dout.p, 0, additions);
        d2h_padded(c, out_slots, dout.p, nslots, 2 * c->nw, S4);
    });
}

int sfxb_accumulate_gh(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *bins, uint32_t J, const uint32_t *node_offsets,
                       uint32_t N, const uint32_t *rows, uint32_t K, uint32_t *out_slots, uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate_gh");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!g || g->ctx != c) throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
        for (uint32_t i = 0; i < N; ++i)
            if (node_offsets[i + 1] < node_offsets[i]) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets decrease");
        if (N && node_offsets[0] != 0) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets must start at 0");
        if (is_group(c)) {
            accumulate_group(c, g, bins, J, node_offsets, N, rows, K, nullptr, out_slots, additions);
            return;
        }
        const uint32_t R = N ? node_offsets[N] : 0;
        const size_t S4 = 4 * (size_t)c->s, nslots = 2ull * N * J * K, n_samples = g->n_samples;
        IoBuf<uint16_t> db(c->io[0], (size_t)J * n_samples);
        IoBuf<uint32_t> doff(c->io[1], (size_t)N + 1), drows(c->io[2], R ? R : 1), dout(c->io[3], nslots * S4);
        if ((size_t)J * n_samples)
            CK(cudaMemcpyAsync(db.p, bins, (size_t)J * n_samples * 2, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(doff.p, node_offsets, ((size_t)N + 1) * 4, cudaMemcpyHostToDevice, c->stream));
        if (R) CK(cudaMemcpyAsync(drows.p, rows, (size_t)R * 4, cudaMemcpyHostToDevice, c->stream));
        accumulate_dev(c, g, db.p, J, doff.p, N, drows.p, R, K, dout.p, 0, additions);
        d2h_padded(c, out_slots, dout.p, nslots, 2 * c->nw, S4);
    });
}

int sfxb_accumulate_tree_dev(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *d_bins, uint32_t n_features,
                             const uint32_t *d_node_offsets, const uint32_t *h_node_offsets, uint32_t n_nodes,
                             const uint32_t *d_rows, uint32_t n_rows, uint32_t n_bins, const int32_t *h_parent,
                             uint32_t *d_out, int mont_out, uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate_tree_dev");
    return guard(c, [&] {
        if (g && !g->parts.empty())
            throw ApiError(SFXB_ERR_UNSUPPORTED, "accumulate: device-pointer entry points take a single-device handle");
        CK(cudaSetDevice(c->device));
        if (!h_parent) throw ApiError(SFXB_ERR_ARG, "accumulate_tree: parent indices required");
        accumulate_dev(c, g, d_bins, n_features, d_node_offsets, n_nodes, d_rows, n_rows, n_bins, d_out, mont_out,
                       additions, h_parent, h_node_offsets);
    });
}

int sfxb_accumulate_tree_gh(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *bins, uint32_t J,
                            const uint32_t *node_offsets, uint32_t N, const uint32_t *rows, uint32_t K,
                            const int32_t *parent, uint32_t *out_slots, uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate_tree_gh");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!g || g->ctx != c) throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
        if (!parent) throw ApiError(SFXB_ERR_ARG, "accumulate_tree: parent indices required");
        for (uint32_t i = 0; i < N; ++i)
            if (node_offsets[i + 1] < node_offsets[i]) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets decrease");
        if (N && node_offsets[0] != 0) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets must start at 0");
        if (is_group(c)) {
            accumulate_group(c, g, bins, J, node_offsets, N, rows, K, parent, out_slots, additions);
            return;
        }
        const uint32_t R = N ? node_offsets[N] : 0;
        const size_t S4 = 4 * (size_t)c->s, nslots = 2ull * N * J * K, n_samples = g->n_samples;
        IoBuf<uint16_t> db(c->io[0], (size_t)J * n_samples);
        IoBuf<uint32_t> doff(c->io[1], (size_t)N + 1), drows(c->io[2], R ? R : 1), dout(c->io[3], nslots * S4);
        if ((size_t)J * n_samples)
            CK(cudaMemcpyAsync(db.p, bins, (size_t)J * n_samples * 2, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(doff.p, node_offsets, ((size_t)N + 1) * 4, cudaMemcpyHostToDevice, c->stream));
        if (R) CK(cudaMemcpyAsync(drows.p, rows, (size_t)R * 4, cudaMemcpyHostToDevice, c->stream));
        accumulate_dev(c, g, db.p, J, doff.p, N, drows.p, R, K, dout.p, 0, additions, parent, node_offsets);
        d2h_padded(c, out_slots, dout.p, nslots, 2 * c->nw, S4);
    });
}

// the default memory pool of `device` keeps what is freed into it
static void retain_pool(int device) {
    static std::mutex m;
    static std::vector<bool> done;
    std::lock_guard<std::mutex> lk(m);
    if ((size_t)device >= done.size()) done.resize(device + 1, false);
    if (done[device]) return;
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    done[device] = true;
}

int sfxb_bins_upload(sfxb_ctx *c, const uint16_t *bins, uint32_t n_features, uint32_t n_samples, sfxb_bins **out) {
    const NvtxRange nvtx_("sfxb_bins_upload");
    return guard(c, [&] {
        if (is_group(c)) throw ApiError(SFXB_ERR_UNSUPPORTED, "bins handle: single-device contexts only");
        CK(cudaSetDevice(c->device));
        auto b = std::make_unique<sfxb_bins>();
        b->ctx = c;
        b->J = n_features;
        b->n = n_samples;
        const size_t bytes = (size_t)n_features * n_samples * 2;
        // stream-ordered allocation from the device's default pool, which
        // keeps freed blocks (release threshold raised once per process):
        // a tree-by-tree upload/free pattern then never reaches cudaFree,
        // whose implicit device synchronisation and unmapping took up to
        // 0.8 s on the box
        retain_pool(c->device);
        CK(cudaMallocAsync(&b->d, bytes + 16, c->stream));
        if (bytes) {
            CK(cudaMemcpyAsync(b->d, bins, bytes, cudaMemcpyHostToDevice, c->stream));
            CK(cudaStreamSynchronize(c->stream));
        }
        *out = b.release();
    });
}

void sfxb_bins_free(sfxb_bins *b) {
    if (!b) return;
    cudaSetDevice(b->ctx->device);
    cudaFreeAsync(b->d, b->ctx->stream);
    delete b;
}

int sfxb_accumulate_tree_bins(sfxb_ctx *c, const sfxb_gh *g, const sfxb_bins *b, const uint32_t *node_offsets,
                              uint32_t N, const uint32_t *rows, uint32_t K, const int32_t *parent,
                              uint32_t *out_slots, uint64_t *additions) {
    const NvtxRange nvtx_("sfxb_accumulate_tree_bins");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!g || g->ctx != c) throw ApiError(SFXB_ERR_ARG, "accumulate: gradient handle belongs to another context");
        if (!b || b->ctx != c) throw ApiError(SFXB_ERR_ARG, "accumulate: bins handle belongs to another context");
        if (b->n != g->n_samples) throw ApiError(SFXB_ERR_ARG, "row-count mismatch between bins and gradients");
        if (!parent) throw ApiError(SFXB_ERR_ARG, "accumulate_tree: parent indices required");
        for (uint32_t i = 0; i < N; ++i)
            if (node_offsets[i + 1] < node_offsets[i]) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets decrease");
        if (N && node_offsets[0] != 0) throw ApiError(SFXB_ERR_ARG, "accumulate: node offsets must start at 0");
        const uint32_t R = N ? node_offsets[N] : 0, J = b->J;
        const size_t S4 = 4 * (size_t)c->s, nslots = 2ull * N * J * K;
        IoBuf<uint32_t> doff(c->io[1], (size_t)N + 1), drows(c->io[2], R ? R : 1), dout(c->io[3], nslots * S4);
        CK(cudaMemcpyAsync(doff.p, node_offsets, ((size_t)N + 1) * 4, cudaMemcpyHostToDevice, c->stream));
        if (R) CK(cudaMemcpyAsync(drows.p, rows, (size_t)R * 4, cudaMemcpyHostToDevice, c->stream));
        accumulate_dev(c, g, b->d, J, doff.p, N, drows.p, R, K, dout.p, 0, additions, parent, node_offsets);
        d2h_padded(c, out_slots, dout.p, nslots, 2 * c->nw, S4);
    });
}

uint64_t sfxb_ctx_tree_derived(const sfxb_ctx *c) { return c->tree_derived_nodes; }

int sfxb_tree_reset(sfxb_ctx *c) {
    return guard(c, [&] {
        c->tree_valid = false;
        for (sfxb_ctx *x : c->shards) x->tree_valid = false;
    });
}

int sfxb_accumulate_part_dev(sfxb_ctx *c, const sfxb_gh *g, const uint16_t *d_bins, uint32_t n_features,
                             const uint32_t *d_node_offsets, const uint32_t *h_node_offsets, uint32_t n_nodes,
                             const uint32_t *d_rows, uint32_t n_rows, uint32_t n_bins, const int32_t *h_parent,
                             const uint32_t *h_node_sizes, uint32_t world, uint32_t *d_send, uint32_t *d_real) {
    const NvtxRange nvtx_("sfxb_accumulate_part_dev");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (!h_node_offsets) throw ApiError(SFXB_ERR_ARG, "accumulate_part: host node offsets required");
        if (h_parent && !h_node_sizes) throw ApiError(SFXB_ERR_ARG, "accumulate_part: node sizes required");
        accumulate_part(c, g, d_bins, n_features, d_node_offsets, h_node_offsets, n_nodes, d_rows, n_rows, n_bins,
                        h_parent, h_node_sizes, world, d_send, d_real);
    });
}

int sfxb_combine_slices_dev(sfxb_ctx *c, const sfxb_gh *g, const uint32_t *d_recv, uint32_t world, uint32_t rank,
                            uint32_t n_nodes, uint32_t n_features, uint32_t n_bins, const int32_t *h_parent,
                            const uint32_t *h_node_sizes, uint32_t *d_out) {
    const NvtxRange nvtx_("sfxb_combine_slices_dev");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        if (h_parent && !h_node_sizes) throw ApiError(SFXB_ERR_ARG, "combine_slices: node sizes required");
        combine_slices(c, g, d_recv, world, rank, n_nodes, n_features, n_bins, h_parent, h_node_sizes, d_out);
    });
}

uint32_t sfxb_slice_width(uint32_t n_features, uint32_t n_bins, uint32_t world) {
    return world ? slice_width(n_features, n_bins, world) : 0;
}

int sfxb_count_additions_dev(sfxb_ctx *c, const uint32_t *d_real, size_t n, uint64_t *additions) {
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        unsigned long long *d_adds = reinterpret_cast<unsigned long long *>(bget<uint32_t>(hist_bufs(c).g_misc, 4));
        CK(cudaMemsetAsync(d_adds, 0, 8, c->stream));
        dev::PeerSet one{};
        one.p[0] = d_real;
        one.n = 1;
        if (n) {
            const int grid = (int)std::min<size_t>((n + 255) / 256, (size_t)c->sms * 8);
            dev::k_adds_multi<<<grid, 256, 0, c->stream>>>(one, n, d_adds);
            check_launch(*c);
        }
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, d_adds, 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (additions) *additions += h;
    });
}

int sfxb_reduce_partials_dev(sfxb_ctx *c, const uint32_t *d_parts, uint32_t parts, size_t n_slots, uint32_t *d_out) {
    const NvtxRange nvtx_("sfxb_reduce_partials_dev");
    return guard(c, [&] {
        CK(cudaSetDevice(c->device));
        reduce_parts_dev(c, d_parts, parts, n_slots, d_out);
    });
}

} // extern "C"
