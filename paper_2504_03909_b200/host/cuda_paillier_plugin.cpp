// CudaPaillierPlugin: the reference's sfxb::EncryptionPlugin backed by the
// B200 kernels through the C ABI (include/sfxb_cuda.h).
//
// Drop-in: this library defines both sfxb::make_paillier_plugin overloads
// (secure_processor.hpp:155-158).  Loaded ahead of the reference library
// (link order or LD_PRELOAD) it takes over every plugin the reference creates,
// including make_plugin in run_vertical_histogram (federation.cpp:76-86) —
// INTEGRATION.md.  Behaviour mirrors PaillierPlugin (secure_processor.cpp:
// 553-746) exactly:
//   * encrypt_gh draws the blinding factors from the same GMP Mersenne-Twister
//     stream as HeRng (he.cpp:11-28: seed via mpz_import, mpz_urandomm,
//     reject r <= 1 and gcd(r, n) != 1) in the same order (g0, h0, g1, ...),
//     so ciphertexts are byte-identical; encode_fixed checks and counters
//     advance exactly as the reference would, including on failure;
//   * accumulate_rows / decrypt_histogram keep the reference's validation
//     order, messages, slot layout, trivial-zero handling and counter laws;
//   * the packed (horizontal) vector path (encrypt_histogram, add_histograms,
//     packed decrypt) packs and unpacks on the host exactly as the reference's
//     packing layer does (PackedLayout::validate / pack_plain / unpack_plain,
//     he.cpp:145-213, restated below) and uses the GPU for every encryption,
//     ciphertext product and decryption, with the reference's r order, checks,
//     error order and vector-granularity counters.
#include <gmp.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <atomic>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "sfxb/errors.hpp"
#include "sfxb/secure_processor.hpp"
#include "sfxb_cuda.h"
#include "parallel.hpp"

namespace sfxb {
namespace {

// ------------------------------------------------------------ helpers

using hostpar::host_threads;
using hostpar::parallel_for;

// mpz <-> little-endian u32 limbs (x86-64 GMP limbs are 64-bit little endian,
// byte-identical to pairs of u32 limbs): raw limb copies, no mpz_import.
static_assert(sizeof(mp_limb_t) == 8, "64-bit GMP limbs expected");

// SFXB_PLUGIN_PROFILE=1: per-call phase times on stderr (host-side costs of
// the reference's payload types vs the GPU call)
struct PhaseTimer {
    const char *name;
    bool on;
    std::chrono::steady_clock::time_point t;
    std::string line;
    explicit PhaseTimer(const char *n)
        : name(n), on(std::getenv("SFXB_PLUGIN_PROFILE") != nullptr), t(std::chrono::steady_clock::now()) {}
    void lap(const char *phase) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        std::snprintf(buf, sizeof buf, " %s=%.1fms", phase, std::chrono::duration<double, std::milli>(now - t).count());
        line += buf;
        t = now;
    }
    ~PhaseTimer() {
        if (on) std::fprintf(stderr, "[sfxb-cuda-plugin] %s%s\n", name, line.c_str());
    }
};

// Grow-only page-locked buffer (sfxb_host_alloc) for the marshalled limbs the
// C ABI copies to / from the device: full-speed DMA, no per-call allocation.
class PinnedBuf {
public:
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf &) = delete;
    PinnedBuf &operator=(const PinnedBuf &) = delete;
    ~PinnedBuf() { sfxb_host_free(p_); }
    template <typename T>
    T *get(size_t n) {
        const size_t need = std::max<size_t>(n * sizeof(T), 1);
        if (need > bytes_) {
            sfxb_host_free(p_);
            p_ = sfxb_host_alloc(need);
            bytes_ = p_ ? need : 0;
            if (!p_) throw sfxb::Error("CUDA Paillier plugin: page-locked host allocation failed");
        }
        return static_cast<T *>(p_);
    }
    template <typename T>
    const T *peek() const {
        return static_cast<const T *>(p_);
    }

private:
    void *p_ = nullptr;
    size_t bytes_ = 0;
};

void to_words(const mpz_class &z, uint32_t *out, size_t words) {
    const size_t used = mpz_size(z.get_mpz_t());
    if (used * 2 > words + 1 || mpz_sgn(z.get_mpz_t()) < 0) {
        // does not fit (or negative): caller reports a range error
        std::memset(out, 0xff, words * 4);
        return;
    }
    std::memset(out, 0, words * 4);
    const mp_limb_t *l = mpz_limbs_read(z.get_mpz_t());
    const size_t bytes = std::min(used * 8, words * 4);
    std::memcpy(out, l, bytes);
    if (used * 8 > words * 4 && (l[used - 1] >> 32) != 0) std::memset(out, 0xff, words * 4);
}

bool fits(const mpz_class &z, size_t words) {
    if (mpz_sgn(z.get_mpz_t()) < 0) return false;
    // whole 64-bit limbs: the header alone decides (no load of the limbs)
    if (words % 2 == 0) return mpz_size(z.get_mpz_t()) <= words / 2;
    return mpz_sizeinbase(z.get_mpz_t(), 2) <= 32 * words;
}

void from_words(mpz_class &z, const uint32_t *w, size_t words) {
    size_t n64 = (words + 1) / 2;
    while (n64 > 0) {
        const uint32_t lo = w[2 * (n64 - 1)], hi = 2 * (n64 - 1) + 1 < words ? w[2 * (n64 - 1) + 1] : 0;
        if (lo | hi) break;
        --n64;
    }
    mp_limb_t *l = mpz_limbs_write(z.get_mpz_t(), (mp_size_t)std::max<size_t>(n64, 1));
    for (size_t i = 0; i < n64; ++i) {
        const uint32_t lo = w[2 * i], hi = 2 * i + 1 < words ? w[2 * i + 1] : 0;
        l[i] = (mp_limb_t)lo | ((mp_limb_t)hi << 32);
    }
    mpz_limbs_finish(z.get_mpz_t(), (mp_size_t)n64);
}

// the reference implementation, for the out-of-scope packed path

// ------------------------------------------------------------ foreground calls
//
// Plugin calls in flight in this process (every instance: the parties'
// plugins share the GPU).  The offline phase launches its next chunk only
// when precompute_may_run(): by default not while a decrypt_histogram call
// (exponentiations competing for the same SMs) is in flight — it fills the
// host's gaps between calls (the reference's Bus, gradients, splits) and the
// idle SMs of accumulate_rows' host phases and transfers.
std::atomic<int> g_foreground{0};
// decrypt_histogram calls in flight (SFXB_ENC_PRECOMPUTE=nodecrypt pauses
// the offline phase only for these: they are exponentiations themselves)
std::atomic<int> g_exclusive{0};

// (also one NVTX range per plugin call: the reference's call names in Nsight)
struct ForegroundCall {
    explicit ForegroundCall(const char *name, bool exclusive = false) : excl(exclusive) {
        g_foreground.fetch_add(1);
        if (excl) g_exclusive.fetch_add(1);
        nvtxRangePushA(name);
    }
    ~ForegroundCall() {
        nvtxRangePop();
        if (excl) g_exclusive.fetch_sub(1);
        g_foreground.fetch_sub(1);
    }
    const bool excl;
    ForegroundCall(const ForegroundCall &) = delete;
    ForegroundCall &operator=(const ForegroundCall &) = delete;
};

// ------------------------------------------------------------ packed vectors
//
// The horizontal path's plaintext packing (he.cpp:145-213), restated so the
// adapter needs nothing from the reference library but its headers: k =
// ⌊(modulus_bits − 1) / slot_bits⌋ slots per plaintext, slot s of a plaintext
// holds q + bias at bit s·slot_bits with q = llround(x·2^scale) and bias =
// 2^(slot_bits − guard_bits − 1); unpacking subtracts bias·addend_count per
// slot and decodes with mpz_get_d truncation.  Checks, messages and their
// order are the reference's.
namespace packing {

unsigned slots(const PackedLayout &l) { // PackedLayout::slots_per_ciphertext, he.cpp:145-148
    if (l.slot_bits == 0) throw ConfigError("slot_bits", "must be positive");
    return (l.modulus_bits - 1) / l.slot_bits;
}

mpz_class bias(const PackedLayout &l) { // PackedLayout::slot_bias, he.cpp:150-154
    mpz_class b;
    mpz_setbit(b.get_mpz_t(), l.slot_bits - l.guard_bits - 1);
    return b;
}

void validate(const PackedLayout &l) { // PackedLayout::validate, he.cpp:156-164
    if (l.slot_bits < 8) throw ConfigError("slot_bits", "must be >= 8");
    if (l.guard_bits + 2 > l.slot_bits) throw ConfigError("guard_bits", "must leave at least one magnitude bit per slot");
    if (l.scale_bits == 0 || l.scale_bits > 52) throw ConfigError("scale_bits", "must be in [1, 52]");
    if (slots(l) < 1) throw ConfigError("slot_bits", "too large for the modulus (zero slots per ciphertext)");
}

// pack_plain, he.cpp:166-193
std::vector<mpz_class> pack(const PackedLayout &l, const std::vector<double> &values) {
    validate(l);
    const size_t k = slots(l);
    const mpz_class b = bias(l);
    const double limit = std::ldexp(1.0, static_cast<int>(62 - l.scale_bits));
    std::vector<mpz_class> out;
    out.reserve((values.size() + k - 1) / k);
    mpz_class q, t;
    for (size_t i = 0; i < values.size(); i += k) {
        mpz_class m = 0;
        for (size_t s = 0; s < std::min(k, values.size() - i); ++s) {
            const double x = values[i + s];
            if (!std::isfinite(x)) throw Error("pack_vector: value must be finite");
            if (std::abs(x) >= limit) throw Error("pack_vector: value too large for the fixed-point grid");
            mpz_set_si(q.get_mpz_t(), static_cast<long>(std::llround(std::ldexp(x, static_cast<int>(l.scale_bits)))));
            if (mpz_cmpabs(q.get_mpz_t(), b.get_mpz_t()) >= 0)
                throw Error("pack_vector: slot overflow at index " + std::to_string(i + s));
            mpz_add(t.get_mpz_t(), q.get_mpz_t(), b.get_mpz_t());
            mpz_mul_2exp(t.get_mpz_t(), t.get_mpz_t(), static_cast<unsigned long>(s) * l.slot_bits);
            mpz_add(m.get_mpz_t(), m.get_mpz_t(), t.get_mpz_t());
        }
        out.push_back(std::move(m));
    }
    return out;
}

// unpack_plain, he.cpp:195-213
std::vector<double> unpack(const PackedLayout &l, const std::vector<mpz_class> &packed, size_t logical_length,
                           std::uint32_t addend_count) {
    validate(l);
    if (addend_count < 1) throw Error("unpack_vector: addend count must be >= 1");
    const size_t k = slots(l);
    if (packed.size() != (logical_length + k - 1) / k)
        throw Error("unpack_vector: ciphertext count does not match logical length");
    mpz_class offset = bias(l);
    mpz_mul_ui(offset.get_mpz_t(), offset.get_mpz_t(), addend_count);
    std::vector<double> out;
    out.reserve(logical_length);
    mpz_class slot;
    for (size_t i = 0; i < logical_length; ++i) {
        // (m >> s·slot_bits) & (2^slot_bits − 1), floor shift as mpz_class's >>
        mpz_fdiv_q_2exp(slot.get_mpz_t(), packed[i / k].get_mpz_t(), static_cast<unsigned long>(i % k) * l.slot_bits);
        mpz_fdiv_r_2exp(slot.get_mpz_t(), slot.get_mpz_t(), l.slot_bits);
        mpz_sub(slot.get_mpz_t(), slot.get_mpz_t(), offset.get_mpz_t());
        out.push_back(std::ldexp(mpz_get_d(slot.get_mpz_t()), -static_cast<int>(l.scale_bits)));
    }
    return out;
}

} // namespace packing

// ------------------------------------------------------------ the plugin

// previous decrypted level of one histogram stream (one sender's tree)
// std::vector without value-initialisation of new elements (the limb buffers
// are overwritten completely; zeroing 100+ MB per call is measurable)
template <typename T>
struct NoInitAlloc : std::allocator<T> {
    template <typename U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <typename U>
    NoInitAlloc(const NoInitAlloc<U> &) {}
    template <typename U>
    void construct(U *p) {
        ::new (static_cast<void *>(p)) U;
    }
    template <typename U, typename... A>
    void construct(U *p, A &&...a) {
        ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
    }
};
using LimbVec = std::vector<uint32_t, NoInitAlloc<uint32_t>>;

struct DecStream {
    uint64_t tag = 0; // sfxb_decrypt_tree cache tag
    LimbVec cts;
    uint32_t n_nodes = 0;
    size_t spn = 0;
    uint64_t last_use = 0;
    uint32_t continued = 0; // levels appended after this stream's root level
};
constexpr size_t kStreams = 8;

// PaillierPlugin's packed layout (secure_processor.cpp:553-558)
PackedLayout packed_layout(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg) {
    PackedLayout l = cfg.packed;
    l.modulus_bits = pk.modulus_bits;
    l.scale_bits = cfg.scale_bits;
    return l;
}

class CudaPaillierPlugin final : public EncryptionPlugin {
public:
    CudaPaillierPlugin(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg)
        : pub_(pk), has_priv_(false), scale_bits_(cfg.scale_bits), layout_(packed_layout(pk, cfg)) {
        init_rng(cfg.rng_seed);
        open_ctx(nullptr);
    }
    CudaPaillierPlugin(const PaillierKeypair &kp, const PaillierPluginConfig &cfg)
        : pub_(kp.pub), priv_(kp.priv), has_priv_(true), scale_bits_(cfg.scale_bits),
          layout_(packed_layout(kp.pub, cfg)) {
        init_rng(cfg.rng_seed);
        open_ctx(&kp);
    }
    ~CudaPaillierPlugin() override {
        if (std::getenv("SFXB_PLUGIN_VERBOSE") && ctx_)
            std::fprintf(stderr, "[sfxb-cuda-plugin] key=%016llx enc=%llu adds=%llu dec=%llu derived_nodes=%llu "
                         "derived_slots=%llu launches=%llu shards=%u\n",
                         (unsigned long long)pub_.key_id, (unsigned long long)counters_.encryptions,
                         (unsigned long long)counters_.ciphertext_additions,
                         (unsigned long long)counters_.decryptions,
                         (unsigned long long)sfxb_ctx_tree_derived(ctx_), (unsigned long long)sfxb_ctx_dec_derived(ctx_),
                         (unsigned long long)sfxb_ctx_launches(ctx_), sfxb_ctx_n_shards(ctx_));
        stop_precompute();
        if (blind_) sfxb_blind_free(blind_);
        if (bg_ctx_) sfxb_ctx_destroy(bg_ctx_);
        if (gh_) sfxb_gh_free(gh_);
        if (bins_h_) sfxb_bins_free(bins_h_);
        if (ctx_) sfxb_ctx_destroy(ctx_);
        gmp_randclear(rng_);
    }

    std::string name() const override { return "paillier"; }
    bool is_passthrough() const override { return false; }
    bool holds_private_key() const override { return has_priv_; }
    std::uint64_t key_id() const override { return pub_.key_id; }

    // ---- encrypt_gh (secure_processor.cpp:574-585)
    GhPayload encrypt_gh(std::span<const GHPair> gh) override {
        const ForegroundCall fg("sfxb::encrypt_gh");
        GhPayload out;
        out.encrypted = true;
        out.n_samples = static_cast<std::uint32_t>(gh.size());
        const size_t count = 2 * gh.size();
        std::vector<int64_t> q(count);
        // encode_fixed checks in the reference's order (g0, h0, g1, ...): the
        // index of the first failure; the reference has drawn one r per
        // successful encryption before it
        std::vector<double> xs(count);
        for (size_t i = 0; i < gh.size(); ++i) {
            xs[2 * i] = gh[i].g;
            xs[2 * i + 1] = gh[i].h;
        }
        size_t ok = count;
        std::string fail_msg;
        if (count && sfxb_encode_batch(ctx_, xs.data(), count, scale_bits_, q.data(), &ok) != SFXB_OK)
            fail_msg = sfxb_last_error(ctx_);
        PhaseTimer pt("encrypt_gh");
        pt.lap("encode");
        const size_t nw = n_words_;
        // blinding powers precomputed since the previous call (offline phase)
        stop_precompute();
        const size_t have = blind_ ? sfxb_blind_size(blind_) : 0;
        pt.lap("join_precompute");
        if (ok < count) {
            // the reference drew one r per successful encryption before the failure
            consume_draws(ok);
            counters_.encryptions += 2 * (ok / 2); // pairs completed before the failure
            throw Error(fail_msg);
        }
        out.cts.resize(count);
        const size_t take = std::min(have, count);
        uint32_t *cts = pin_cts_.get<uint32_t>(count * ct_words_);
        const hostpar::TopPadScope pad(count * ct_words_ * 4);
        auto marshal = [&](size_t lo, size_t hi) {
            parallel_for(hi - lo, [&](size_t a, size_t b) {
                for (size_t i = lo + a; i < lo + b; ++i) {
                    from_words(out.cts[i].value, &cts[i * ct_words_], ct_words_);
                    out.cts[i].key_id = pub_.key_id;
                }
            });
        };
        if (take) {
            // online phase: c = (1 + m·n)·r^n mod n² with the queued powers
            check(sfxb_encrypt_blind(ctx_, blind_, q.data(), nullptr, take, cts));
            pt.lap("online");
        }
        if (take < count && has_priv_ && count - take >= 2 * enc_chunk()) {
            std::thread m0;
            if (take) m0 = std::thread(marshal, 0, take);
            encrypt_gh_pipelined(q, out, take, pt);
            if (m0.joinable()) m0.join();
        } else {
            if (take < count) {
                const size_t rest = count - take;
                uint32_t *r = pin_r_.get<uint32_t>(rest * nw);
                draw_blinding(r, rest);
                pt.lap("draw_r");
                std::vector<uint8_t> flags(rest, 0);
                int rc = sfxb_encrypt(ctx_, q.data() + take, r, rest, cts + take * ct_words_, flags.data());
                if (rc == SFXB_ERR_COPRIME) {
                    // some r shares a factor with n (probability ~2^-1000): redo the
                    // draw with the reference's exact rejection rule from the saved state
                    gmp_randclear(rng_);
                    gmp_randinit_set(rng_, rng_snapshot_);
                    draw_blinding(r, rest, /*exact_gcd=*/true);
                    rc = sfxb_encrypt(ctx_, q.data() + take, r, rest, cts + take * ct_words_, nullptr);
                }
                check(rc);
                pt.lap("gpu");
            }
            marshal(0, count);
        }
        counters_.encryptions += count;
        pt.lap("marshal");
        // offline phase for the next call (the next tree encrypts as many)
        start_precompute(count);
        return out;
    }

    // ---- accumulate_rows (secure_processor.cpp:587-620)
    //
    // The histogram products run on the GPU over the device copy of gh.  Inputs
    // the reference treats specially keep its semantics exactly:
    //   * ciphertexts equal to 1 are skipped (fold_into, :724-732) whatever
    //     their key id;
    //   * "irregular" ciphertexts — a foreign key id, or a value outside
    //     [0, n²) (negative, ≥ n², wider than the ciphertext) — are not
    //     ciphertexts of this key.  They go to the device as the identity and
    //     every slot they land in is folded again on the host with the
    //     reference's rules (assign into an empty slot keeping the value and
    //     key id as they are; a·b tdiv n² otherwise; add_ciphertexts' key
    //     check, he.cpp:117-121).  A foreign key therefore fails only where
    //     the reference's loop multiplies it, with the reference's counter at
    //     that point (replay_folds);
    //   * a bad bin index fails at the reference's loop position, with the
    //     additions it counted before it.
    // Known deviation (not replayed): if a running slot product other than the
    // last becomes exactly 1 (c·c⁻¹ inside one slot — never the case for
    // honest encryptions), the reference's next fold is an uncounted assign;
    // the GPU counts Σ max(k − 1, 0).  Residues are identical either way.
    HistogramPayload accumulate_rows(const GhPayload &gh, const std::vector<std::vector<std::uint16_t>> &bins,
                                     const std::vector<int> &feature_ids, const std::vector<NodeRows> &nodes,
                                     int n_bins) override {
        const ForegroundCall fg("sfxb::accumulate_rows");
        if (!gh.encrypted) throw Error("paillier accumulate expects encrypted gradients");
        if (gh.cts.size() != 2ull * gh.n_samples)
            throw Error("row-count mismatch: ciphertext count is not 2·n_samples");
        for (const auto &col : bins)
            if (col.size() != gh.n_samples) throw Error("row-count mismatch between bins and gradients");
        if (bins.size() < feature_ids.size()) throw Error("row-count mismatch between bins and gradients");
        HistogramPayload out;
        out.layout = HistLayout::enc_scalar;
        const size_t J = feature_ids.size(), K = (size_t)std::max(n_bins, 0), N = nodes.size();
        PhaseTimer pt("accumulate_rows");
        // header-only pass over gh: key ids, signs, sizes, the value 1
        const GhScan scan = scan_gh(gh);
        pt.lap("scan");
        // bins are checked per visited row, as the reference loop does: a
        // parallel scan, and on a hit the reference's loop is replayed for its
        // exception and counter
        {
            std::atomic<bool> bad{false};
            parallel_for(N * J, [&](size_t lo, size_t hi) {
                for (size_t t = lo; t < hi && !bad; ++t) {
                    const NodeRows &nd = nodes[t / J];
                    const std::vector<std::uint16_t> &col = bins[t % J];
                    for (std::uint32_t row : nd.rows)
                        if (row >= gh.n_samples || col[row] >= static_cast<std::uint16_t>(n_bins)) {
                            bad = true;
                            break;
                        }
                }
            }, /*grain=*/1);
            if (bad) fail_with_replay(gh, scan, bins, J, nodes, n_bins);
        }
        pt.lap("validate");
        const bool candidate = gh_ && gh_scan_key_ == scan.key && gh_count_ == gh.cts.size();
        if (!candidate) upload_gh(gh, scan.key);
        pt.lap("ensure_gh");
        // bins: exact change detection against the previous call's staged copy
        const size_t nb_elems = J * gh.n_samples;
        const void *before = pin_bins_.peek<void>();
        uint16_t *flat = pin_bins_.get<uint16_t>(nb_elems);
        const bool same_layout = flat == before && staged_J_ == J && staged_n_ == gh.n_samples && nb_elems;
        const bool bins_changed = stage_bins(bins, J, gh.n_samples, flat, same_layout);
        staged_J_ = J;
        staged_n_ = gh.n_samples;
        const bool same_bins = !bins_changed && staged_fids_ == feature_ids && staged_K_ == n_bins;
        staged_fids_ = feature_ids;
        staged_K_ = n_bins;
        // the columns stay on the device across calls (the reference's bins are
        // fixed for a training run); re-uploaded only when they change
        const bool use_bins_handle = sfxb_ctx_n_shards(ctx_) == 1 && nb_elems;
        if (use_bins_handle && (!bins_h_ || bins_changed || bins_h_J_ != J || bins_h_n_ != gh.n_samples)) {
            if (bins_h_) sfxb_bins_free(bins_h_);
            bins_h_ = nullptr;
            check(sfxb_bins_upload(ctx_, flat, (uint32_t)J, gh.n_samples, &bins_h_));
            bins_h_J_ = J;
            bins_h_n_ = gh.n_samples;
        }
        std::vector<uint32_t> offs(N + 1, 0), rows;
        for (size_t i = 0; i < N; ++i) offs[i + 1] = offs[i] + (uint32_t)nodes[i].rows.size();
        rows.reserve(offs[N]);
        for (const NodeRows &nd : nodes) rows.insert(rows.end(), nd.rows.begin(), nd.rows.end());
        pt.lap("flatten");
        uint32_t *slots = pin_slots_.get<uint32_t>(N * J * K * 2 * ct_words_);
        uint64_t adds = 0;
        auto run_gpu = [&](bool allow_parents) -> int {
            // Sibling subtraction: the reference's next frontier lists the two
            // children of each split node consecutively, in parent order
            // (federation.cpp:591-592).  A parent is accepted only when the
            // merged rows of the pair equal its rows exactly and the features,
            // bins and gradients are those of the previous call.
            std::vector<int32_t> parent(N, -1);
            if (allow_parents && prev_valid_ && same_bins && prev_gh_ == gh_) {
                size_t p = 0;
                for (size_t i = 0; i + 1 < N && p < prev_rows_.size();) {
                    const auto &ra = nodes[i].rows, &rb = nodes[i + 1].rows;
                    size_t q = p;
                    while (q < prev_rows_.size() && prev_rows_[q].size() != ra.size() + rb.size()) ++q;
                    if (q < prev_rows_.size() && merged_equals(ra, rb, prev_rows_[q])) {
                        parent[i] = parent[i + 1] = (int32_t)q;
                        p = q + 1;
                        i += 2;
                    } else {
                        ++i;
                    }
                }
            }
            adds = 0;
            if (!(N && J && K)) return SFXB_OK;
            if (use_bins_handle)
                return sfxb_accumulate_tree_bins(ctx_, gh_, bins_h_, offs.data(), (uint32_t)N, rows.data(),
                                                 (uint32_t)K, parent.data(), slots, &adds);
            return sfxb_accumulate_tree_gh(ctx_, gh_, flat, (uint32_t)J, offs.data(), (uint32_t)N, rows.data(),
                                           (uint32_t)K, parent.data(), slots, &adds);
        };
        int rc;
        if (candidate) {
            // Same limb buffers as the resident copy: the GPU starts on it while
            // the host compares every limb (and every irregular value) with what
            // was uploaded.  A difference discards the result and reruns on a
            // fresh upload — the device copy is never trusted on a sampled key.
            bool same = false;
            std::thread verify([&] {
                try {
                    same = verify_gh(gh);
                } catch (...) {
                    same = false; // treated as a difference: fresh upload below
                }
            });
            try {
                rc = run_gpu(true);
            } catch (...) {
                verify.join();
                throw;
            }
            verify.join();
            pt.lap("gpu+verify");
            if (!same) {
                upload_gh(gh, scan.key);
                rc = run_gpu(false);
                pt.lap("reupload+gpu");
            }
        } else {
            rc = run_gpu(true);
            pt.lap("gpu");
        }
        check(rc);
        prev_valid_ = N && J && K;
        prev_gh_ = gh_;
        prev_rows_.resize(N);
        for (size_t i = 0; i < N; ++i) prev_rows_[i] = nodes[i].rows;
        const size_t per_node = 2 * J * K;
        out.nodes.resize(N);
        for (size_t i = 0; i < N; ++i) {
            NodeHistogram &nh = out.nodes[i];
            nh.node_id = nodes[i].node_id;
            nh.feature_ids = feature_ids;
            nh.n_bins = n_bins;
            nh.scalar_cts.resize(per_node);
        }
        pt.lap("out_alloc");
        {
            const hostpar::TopPadScope pad(N * per_node * ct_words_ * 4);
            parallel_for(N * per_node, [&](size_t lo, size_t hi) {
                for (size_t s = lo; s < hi; ++s) {
                    Ciphertext &c = out.nodes[s / per_node].scalar_cts[s % per_node];
                    from_words(c.value, &slots[s * ct_words_], ct_words_);
                    c.key_id = pub_.key_id;
                }
            });
        }
        pt.lap("out_marshal");
        // slots holding irregular ciphertexts: the reference's folds on the host
        if (!irr_.empty()) adds = refold_irregular(gh, scan, bins, J, nodes, n_bins, out, adds);
        counters_.ciphertext_additions += adds;
        return out;
    }

    // ---- decrypt_histogram (secure_processor.cpp:679-719)
    std::vector<std::pair<std::uint32_t, Histogram>> decrypt_histogram(const HistogramPayload &payload) override {
        const ForegroundCall fg("sfxb::decrypt_histogram", true);
        if (!has_priv_) throw AuthorizationError("decrypt requested without private key material");
        if (payload.layout != HistLayout::enc_scalar) {
            if (payload.layout == HistLayout::enc_packed) return decrypt_packed(payload);
            throw Error("paillier decrypt expects encrypted layouts");
        }
        std::vector<std::pair<std::uint32_t, Histogram>> out;
        PhaseTimer pt("decrypt_histogram");
        size_t total = 0;
        for (const NodeHistogram &node : payload.nodes)
            total += 2 * node.feature_ids.size() * (size_t)std::max(node.n_bins, 0);
        LimbVec cts(total * ct_words_);
        pt.lap("alloc");
        // the reference decrypts slot by slot: key and range errors surface at
        // the first offending non-trivial slot in that order.  Marshalled in
        // parallel; on a bad slot the serial scan below reports the first one.
        size_t base = 0;
        std::vector<std::pair<const NodeHistogram *, size_t>> node_base;
        for (const NodeHistogram &node : payload.nodes) {
            const size_t cnt = 2 * node.feature_ids.size() * (size_t)std::max(node.n_bins, 0);
            if (node.scalar_cts.size() < cnt) throw Error("decrypt_histogram: scalar slot count mismatch");
            node_base.emplace_back(&node, base);
            base += cnt;
        }
        std::atomic<bool> bad{false};
        parallel_for(node_base.size(), [&](size_t lo, size_t hi) {
            for (size_t i = lo; i < hi && !bad; ++i) {
                const NodeHistogram &node = *node_base[i].first;
                const size_t b0 = node_base[i].second;
                const size_t cnt = 2 * node.feature_ids.size() * (size_t)std::max(node.n_bins, 0);
                for (size_t s = 0; s < cnt; ++s) {
                    const Ciphertext &c = node.scalar_cts[s];
                    uint32_t *w = &cts[(b0 + s) * ct_words_];
                    if (c.value == 1) {
                        std::memset(w, 0, ct_words_ * 4);
                        w[0] = 1;
                        continue;
                    }
                    if (c.key_id != pub_.key_id || c.value < 1 || c.value >= pub_.n2 || !fits(c.value, ct_words_)) {
                        bad = true;
                        break;
                    }
                    to_words(c.value, w, ct_words_);
                }
            }
        }, /*grain=*/1);
        if (bad) fail_decrypt(payload, /*coprime_error=*/false);
        pt.lap("marshal_in");
        std::vector<double> vals(total);
        uint64_t decs = 0;
        if (total) {
            try {
                decrypt_level(payload, cts, vals, &decs, pt);
            } catch (const Error &) {
                // the GPU found a slot sharing a factor with n
                if (std::string(sfxb_last_error(ctx_)).find("not coprime") != std::string::npos)
                    fail_decrypt(payload, /*coprime_error=*/true);
                throw;
            }
        }
        counters_.decryptions += decs;
        base = 0;
        for (const NodeHistogram &node : payload.nodes) {
            Histogram hist;
            hist.n_bins = node.n_bins;
            hist.feature_ids = node.feature_ids;
            hist.feats.assign(node.feature_ids.size(), std::vector<GHPair>(static_cast<std::size_t>(node.n_bins)));
            for (std::size_t f = 0; f < node.feature_ids.size(); ++f)
                for (int b = 0; b < node.n_bins; ++b) {
                    const size_t s = base + 2 * (f * (size_t)node.n_bins + (size_t)b);
                    hist.feats[f][b] = GHPair{vals[s], vals[s + 1]};
                }
            base += 2 * node.feature_ids.size() * (size_t)std::max(node.n_bins, 0);
            out.emplace_back(node.node_id, std::move(hist));
        }
        pt.lap("marshal_out");
        return out;
    }

    // ---- packed (horizontal) path: encrypt_histogram (secure_processor.cpp:622-645)
    // = pack_plain (packing layer below, he.cpp:166-193) + one GPU
    // batch of encrypt_with_r over every packed plaintext, r drawn in the
    // reference's order (node: G vector, then H vector).
    HistogramPayload encrypt_histogram(const std::vector<std::pair<std::uint32_t, Histogram>> &node_hists) override {
        const ForegroundCall fg("sfxb::encrypt_histogram");
        packing::validate(layout_);
        HistogramPayload out;
        out.layout = HistLayout::enc_packed;
        std::vector<mpz_class> plains;
        std::vector<size_t> first(1, 0);
        std::vector<std::uint32_t> lengths;
        size_t done_nodes = 0;
        try {
            for (const auto &[node_id, hist] : node_hists) {
                std::vector<double> gs, hs;
                gs.reserve(hist.feats.size() * hist.n_bins);
                hs.reserve(hist.feats.size() * hist.n_bins);
                for (const auto &slots : hist.feats)
                    for (const GHPair &b : slots) {
                        gs.push_back(b.g);
                        hs.push_back(b.h);
                    }
                for (const std::vector<double> *v : {&gs, &hs}) {
                    std::vector<mpz_class> p = packing::pack(layout_, *v);
                    for (mpz_class &m : p) plains.push_back(std::move(m));
                    first.push_back(plains.size());
                    lengths.push_back(static_cast<std::uint32_t>(v->size()));
                }
                ++done_nodes;
            }
        } catch (...) {
            // the reference encrypted (drew r for) every vector packed before the failure
            consume_draws(plains.size());
            counters_.encryptions += 2 * done_nodes;
            throw;
        }
        const size_t count = plains.size();
        std::vector<uint32_t> m(count * n_words_), cts(count * ct_words_);
        for (size_t i = 0; i < count; ++i) to_words(plains[i], &m[i * n_words_], n_words_);
        // queued blinding powers first (the stream order), then fresh draws
        stop_precompute();
        const size_t take = std::min(blind_ ? sfxb_blind_size(blind_) : 0, count);
        if (take) check(sfxb_encrypt_blind(ctx_, blind_, nullptr, m.data(), take, cts.data()));
        if (count > take) {
            const size_t rest = count - take;
            std::vector<uint32_t> r(rest * n_words_);
            draw_blinding(r.data(), rest);
            int rc = sfxb_encrypt_plain(ctx_, &m[take * n_words_], r.data(), rest, &cts[take * ct_words_], nullptr);
            if (rc == SFXB_ERR_COPRIME) {
                gmp_randclear(rng_);
                gmp_randinit_set(rng_, rng_snapshot_);
                draw_blinding(r.data(), rest, /*exact_gcd=*/true);
                rc = sfxb_encrypt_plain(ctx_, &m[take * n_words_], r.data(), rest, &cts[take * ct_words_], nullptr);
            }
            check(rc);
        }
        size_t v = 0;
        for (const auto &[node_id, hist] : node_hists) {
            NodeHistogram nh;
            nh.node_id = node_id;
            nh.feature_ids = hist.feature_ids;
            nh.n_bins = hist.n_bins;
            for (PackedVector *pv : {&nh.packed_g, &nh.packed_h}) {
                pv->logical_length = lengths[v];
                pv->addend_count = 1;
                pv->slot_bits = layout_.slot_bits;
                pv->guard_bits = layout_.guard_bits;
                pv->scale_bits = layout_.scale_bits;
                pv->cts.resize(first[v + 1] - first[v]);
                for (size_t k = 0; k < pv->cts.size(); ++k) {
                    from_words(pv->cts[k].value, &cts[(first[v] + k) * ct_words_], ct_words_);
                    pv->cts[k].key_id = pub_.key_id;
                }
                ++v;
            }
            counters_.encryptions += 2; // vector granularity
            out.nodes.push_back(std::move(nh));
        }
        start_precompute(count); // offline phase for the next call
        return out;
    }

    // ---- add_histograms (secure_processor.cpp:647-676): validation, fold
    // rules and counters in the reference's order; the ciphertext products of
    // each part run as one GPU batch (sfxb_add).
    HistogramPayload add_histograms(const std::vector<HistogramPayload> &parts) override {
        const ForegroundCall fg("sfxb::add_histograms");
        if (parts.empty()) throw Error("add_histograms: no inputs");
        HistogramPayload acc = parts[0];
        for (std::size_t p = 1; p < parts.size(); ++p) {
            const HistogramPayload &cur = parts[p];
            if (cur.layout != acc.layout || cur.nodes.size() != acc.nodes.size())
                throw Error("add_histograms: shape mismatch");
            std::vector<std::pair<Ciphertext *, const Ciphertext *>> work; // lhs ⊗= rhs
            uint64_t adds = 0;
            try {
                for (std::size_t i = 0; i < acc.nodes.size(); ++i) {
                    NodeHistogram &a = acc.nodes[i];
                    const NodeHistogram &b = cur.nodes[i];
                    if (a.node_id != b.node_id || a.feature_ids != b.feature_ids || a.n_bins != b.n_bins)
                        throw Error("add_histograms: shape mismatch");
                    if (acc.layout == HistLayout::enc_packed) {
                        plan_add_packed(a.packed_g, b.packed_g, work);
                        plan_add_packed(a.packed_h, b.packed_h, work);
                        adds += 2; // vector granularity
                    } else if (acc.layout == HistLayout::enc_scalar) {
                        if (a.scalar_cts.size() != b.scalar_cts.size()) throw Error("add_histograms: shape mismatch");
                        for (std::size_t s = 0; s < a.scalar_cts.size(); ++s) {
                            Ciphertext &lhs = a.scalar_cts[s];
                            const Ciphertext &rhs = b.scalar_cts[s];
                            if (is_trivial_zero(rhs)) continue; // fold_into (:724-732)
                            if (is_trivial_zero(lhs)) {
                                lhs = rhs;
                                continue;
                            }
                            if (lhs.key_id != rhs.key_id || lhs.key_id != pub_.key_id)
                                throw Error("add_ciphertexts: key mismatch");
                            work.emplace_back(&lhs, &rhs);
                            ++adds;
                        }
                    } else {
                        throw Error("paillier add_histograms expects encrypted layouts");
                    }
                }
            } catch (...) {
                counters_.ciphertext_additions += adds;
                throw;
            }
            multiply_into(work);
            counters_.ciphertext_additions += adds;
        }
        return acc;
    }

private:
    // SFXB_CUDA_DEVICES="0,1,...,7" spreads the plugin over a device group
    // (sfxb_ctx_create_multi: row-sharded histograms, element-sharded
    // encrypt/decrypt); "all" = every visible GPU.  Otherwise one device,
    // SFXB_CUDA_DEVICE (default 0).
    static std::vector<int> devices_from_env() {
        std::vector<int> devs;
        const char *e = std::getenv("SFXB_CUDA_DEVICES");
        if (e && std::string(e) == "all") {
            for (int i = 0, n = sfxb_device_count(); i < n; ++i) devs.push_back(i);
        } else if (e && *e) {
            std::string s(e);
            size_t pos = 0;
            while (pos <= s.size()) {
                size_t end = s.find(',', pos);
                if (end == std::string::npos) end = s.size();
                if (end > pos) devs.push_back(std::atoi(s.substr(pos, end - pos).c_str()));
                pos = end + 1;
            }
        }
        if (devs.empty()) devs.push_back(std::getenv("SFXB_CUDA_DEVICE") ? std::atoi(std::getenv("SFXB_CUDA_DEVICE")) : 0);
        return devs;
    }

    void open_ctx(const PaillierKeypair *kp) {
        const std::vector<int> devs = devices_from_env();
        n_words_ = (mpz_sizeinbase(pub_.n.get_mpz_t(), 2) + 31) / 32;
        std::vector<uint32_t> n(n_words_);
        to_words(pub_.n, n.data(), n_words_);
        int rc;
        if (kp) {
            size_t pw = (std::max(mpz_sizeinbase(kp->priv.p.get_mpz_t(), 2), mpz_sizeinbase(kp->priv.q.get_mpz_t(), 2)) + 31) / 32;
            std::vector<uint32_t> p(pw), q(pw);
            to_words(kp->priv.p, p.data(), pw);
            to_words(kp->priv.q, q.data(), pw);
            rc = sfxb_ctx_create_multi(&ctx_, devs.data(), (uint32_t)devs.size(), n.data(), (uint32_t)n_words_,
                                       p.data(), q.data(), (uint32_t)pw);
        } else {
            rc = sfxb_ctx_create_multi(&ctx_, devs.data(), (uint32_t)devs.size(), n.data(), (uint32_t)n_words_,
                                       nullptr, nullptr, 0);
        }
        if (rc != SFXB_OK) throw Error(std::string("CUDA Paillier plugin: ") + sfxb_create_error());
        ct_words_ = sfxb_ctx_ct_words(ctx_);
        enc_wave_ = sfxb_ctx_enc_wave(ctx_);
    }

    // HeRng(seed) (he.cpp:11-15)
    void init_rng(std::uint64_t seed) {
        gmp_randinit_mt(rng_);
        mpz_class s;
        mpz_import(s.get_mpz_t(), 1, 1, sizeof seed, 0, 0, &seed);
        gmp_randseed(rng_, s.get_mpz_t());
        gmp_randinit_mt(rng_snapshot_);
    }

    // encrypt_gh for large batches with the host's sequential work off the
    // GPU's critical path: a helper thread draws the blinding factors of chunk
    // k+1 (the reference's MT stream, in order) while the GPU encrypts chunk k,
    // and the ciphertexts of chunk k are marshalled into the payload while the
    // GPU encrypts chunk k+1.  If chunk k holds an r sharing a factor with n
    // (probability ≈ 2^-1000), the stream is rewound to the state before chunk
    // k and the rest is redrawn with the reference's exact rejection rule.
    // chunk size (SFXB_ENC_CHUNK overrides; the tests shrink it to exercise
    // the pipeline on small runs)
    // (default: the multiple of the GPU's encryption wave nearest 256K, so no
    // chunk but a call's last ends in a partial wave)
    size_t enc_chunk() const {
        static const long env = std::getenv("SFXB_ENC_CHUNK") ? std::max(1L, std::atol(std::getenv("SFXB_ENC_CHUNK"))) : 0;
        return env ? (size_t)env : wave_multiple(262144);
    }
    // the multiple of sfxb_ctx_enc_wave nearest `target` (at least one wave)
    size_t wave_multiple(size_t target) const {
        const size_t w = enc_wave_;
        if (w == 0) return target;
        return std::max<size_t>(1, (target + w / 2) / w) * w;
    }
    void encrypt_gh_pipelined(const std::vector<int64_t> &q, GhPayload &out, size_t first, PhaseTimer &pt) {
        // elements [first, count); out.cts already sized, pin_cts_ holds the
        // ciphertexts before `first`
        const size_t kEncChunk = enc_chunk();
        const size_t count = q.size(), nw = n_words_, nch = (count - first + kEncChunk - 1) / kEncChunk;
        uint32_t *r = pin_r_.get<uint32_t>(count * nw); // indexed by element
        uint32_t *cts = pin_cts_.get<uint32_t>(count * ct_words_);
        std::vector<uint8_t> flags(count, 0);
        struct Snap {
            gmp_randstate_t s;
            Snap() { gmp_randinit_mt(s); }
            ~Snap() { gmp_randclear(s); }
        };
        std::vector<std::unique_ptr<Snap>> snap(nch);
        for (auto &x : snap) x = std::make_unique<Snap>();
        std::mutex mu;
        std::condition_variable cv;
        size_t drawn = 0;
        std::atomic<bool> stop{false};
        std::thread drawer([&] {
            mpz_class rv;
            for (size_t k = 0; k < nch && !stop; ++k) {
                gmp_randclear(snap[k]->s);
                gmp_randinit_set(snap[k]->s, rng_);
                const size_t lo = first + k * kEncChunk, hi = std::min(count, lo + kEncChunk);
                for (size_t i = lo; i < hi; ++i) {
                    do mpz_urandomm(rv.get_mpz_t(), rng_, pub_.n.get_mpz_t());
                    while (rv <= 1); // gcd(r, n) is tested on the device
                    to_words(rv, r + i * nw, nw);
                }
                std::lock_guard<std::mutex> lk(mu);
                drawn = k + 1;
                cv.notify_one();
            }
        });
        auto marshal = [&](size_t lo, size_t hi) {
            parallel_for(hi - lo, [&](size_t a, size_t b) {
                for (size_t i = lo + a; i < lo + b; ++i) {
                    from_words(out.cts[i].value, &cts[i * ct_words_], ct_words_);
                    out.cts[i].key_id = pub_.key_id;
                }
            });
        };
        std::thread marshaller;
        auto join_marshal = [&] {
            if (marshaller.joinable()) marshaller.join();
        };
        try {
            for (size_t k = 0; k < nch; ++k) {
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return drawn > k; });
                }
                const size_t lo = first + k * kEncChunk, n = std::min(count, lo + kEncChunk) - lo;
                int rc = sfxb_encrypt(ctx_, &q[lo], r + lo * nw, n, cts + lo * ct_words_, flags.data() + lo);
                if (rc == SFXB_ERR_COPRIME) {
                    stop = true;
                    drawer.join();
                    gmp_randclear(rng_);
                    gmp_randinit_set(rng_, snap[k]->s);
                    draw_blinding(r + lo * nw, count - lo, /*exact_gcd=*/true);
                    check(sfxb_encrypt(ctx_, &q[lo], r + lo * nw, count - lo, cts + lo * ct_words_, nullptr));
                    join_marshal();
                    marshal(lo, count);
                    break;
                }
                check(rc);
                join_marshal();
                marshaller = std::thread(marshal, lo, lo + n);
            }
        } catch (...) {
            stop = true;
            if (drawer.joinable()) drawer.join();
            join_marshal();
            throw;
        }
        if (drawer.joinable()) drawer.join();
        join_marshal();
        pt.lap("pipelined");
    }

    // ---------------------------------------------------------------- offline phase
    //
    // Blinding powers r^n mod n² do not depend on the plaintexts: after a
    // call that encrypted `target` values, a background thread keeps drawing
    // the next r of the HeRng stream (he.cpp:11-28, same rejection rules) and
    // has a low-priority context on the same GPU append r^n mod n² to a
    // device queue, chunk by chunk, until the queue holds `target` powers or
    // the next call arrives.  The next call joins the thread (at a chunk
    // boundary: the stream position then matches the queue exactly), encrypts
    // the first min(queued, needed) values by the online step only, and draws
    // the rest as before.  Every consumer of the stream (encrypt_gh,
    // encrypt_histogram, the draws of a failing call) takes queued powers
    // first, so the r sequence — and every ciphertext — is the reference's.
    // SFXB_ENC_PRECOMPUTE=0 disables it; SFXB_ENC_PRECOMPUTE_CHUNK sets the
    // chunk (default 16384).
    static bool precompute_enabled() {
        static const bool on = [] {
            const char *e = std::getenv("SFXB_ENC_PRECOMPUTE");
            return !(e && std::string(e) == "0");
        }();
        return on;
    }
    // when the next chunk may launch: 2 = except during decrypt_histogram
    // (default, "nodecrypt": between calls and under accumulate_rows, whose
    // host phases and transfers leave SMs idle), 0 = between plugin calls
    // only ("between"), 1 = also during decrypt ("always").  Measured through
    // the plugin (profiles/r02_precompute_policy.md): 4.46–4.58 s/tree vs
    // 4.70 between calls only, 4.54–4.63 always.
    static int precompute_mode() {
        static const int m = [] {
            const char *e = std::getenv("SFXB_ENC_PRECOMPUTE");
            const std::string v = e ? e : "";
            return v == "always" ? 1 : v == "between" ? 0 : 2;
        }();
        return m;
    }
    static bool precompute_may_run() {
        switch (precompute_mode()) {
        case 1: return true;
        case 2: return g_exclusive.load() == 0;
        default: return g_foreground.load() == 0;
        }
    }
    // (default: one encryption wave — 18,944 at 2048 bits on a B200 — so each
    // background launch fills the GPU once)
    size_t precompute_chunk() const {
        static const long env = std::getenv("SFXB_ENC_PRECOMPUTE_CHUNK")
                                    ? std::max(1L, std::atol(std::getenv("SFXB_ENC_PRECOMPUTE_CHUNK")))
                                    : 0;
        return env ? (size_t)env : wave_multiple(16384);
    }

    // queue capacity in blinding powers (SFXB_ENC_PRECOMPUTE_MAX, default 4M:
    // 2 GB of device memory at 2048-bit n — two HIGGS trees' worth)
    static size_t precompute_max() {
        static const size_t m = std::getenv("SFXB_ENC_PRECOMPUTE_MAX")
                                    ? (size_t)std::max(0L, std::atol(std::getenv("SFXB_ENC_PRECOMPUTE_MAX")))
                                    : (size_t)4 << 20;
        return m;
    }

    void start_precompute(size_t target) {
        target = std::min(target, precompute_max());
        if (!precompute_enabled() || !has_priv_ || target == 0 || sfxb_ctx_n_shards(ctx_) != 1) return;
        if (!bg_ctx_) {
            // a second context of the same key on the same device, low priority
            std::vector<uint32_t> n(n_words_);
            to_words(pub_.n, n.data(), n_words_);
            size_t pw = (std::max(mpz_sizeinbase(priv_.p.get_mpz_t(), 2), mpz_sizeinbase(priv_.q.get_mpz_t(), 2)) + 31) / 32;
            std::vector<uint32_t> p(pw), qq(pw);
            to_words(priv_.p, p.data(), pw);
            to_words(priv_.q, qq.data(), pw);
            if (sfxb_ctx_create(&bg_ctx_, sfxb_ctx_shard_device(ctx_, 0), n.data(), (uint32_t)n_words_, p.data(),
                                qq.data(), (uint32_t)pw) != SFXB_OK) {
                bg_ctx_ = nullptr;
                return;
            }
            sfxb_ctx_set_low_priority(bg_ctx_);
        }
        if (blind_ && sfxb_blind_size(blind_) == 0 && target > blind_cap_) {
            sfxb_blind_free(blind_);
            blind_ = nullptr;
        }
        if (!blind_) {
            if (sfxb_blind_create(bg_ctx_, target, &blind_) != SFXB_OK) {
                blind_ = nullptr;
                return;
            }
            blind_cap_ = target;
        }
        const size_t goal = std::min(target, blind_cap_);
        if (sfxb_blind_size(blind_) >= goal) return;
        bg_stop_ = false;
        bg_ = std::thread([this, goal] { precompute_loop(goal); });
    }

    void stop_precompute() {
        if (!bg_.joinable()) return;
        bg_stop_ = true;
        bg_.join();
        bg_stop_ = false;
    }

    // background thread: owns rng_ until joined
    void precompute_loop(size_t goal) {
        const size_t chunk = precompute_chunk(), nw = n_words_;
        std::vector<uint32_t> r(chunk * nw);
        std::vector<uint8_t> flags(chunk);
        gmp_randstate_t snap;
        gmp_randinit_mt(snap);
        mpz_class rv, g;
        while (!bg_stop_) {
            const size_t have = sfxb_blind_size(blind_);
            if (have >= goal) break;
            // SFXB_ENC_PRECOMPUTE policy (precompute_mode)
            while (!precompute_may_run() && !bg_stop_)
                std::this_thread::sleep_for(std::chrono::microseconds(500));
            if (bg_stop_) break;
            const size_t k = std::min(chunk, goal - have);
            gmp_randclear(snap);
            gmp_randinit_set(snap, rng_);
            for (size_t i = 0; i < k; ++i) {
                do mpz_urandomm(rv.get_mpz_t(), rng_, pub_.n.get_mpz_t());
                while (rv <= 1); // gcd(r, n) on the device
                to_words(rv, &r[i * nw], nw);
            }
            int rc = sfxb_blind_append(bg_ctx_, blind_, r.data(), k, flags.data());
            if (rc == SFXB_ERR_COPRIME) {
                // redraw the chunk with the reference's exact rejection rule
                gmp_randclear(rng_);
                gmp_randinit_set(rng_, snap);
                for (size_t i = 0; i < k; ++i) {
                    for (;;) {
                        mpz_urandomm(rv.get_mpz_t(), rng_, pub_.n.get_mpz_t());
                        if (rv <= 1) continue;
                        mpz_gcd(g.get_mpz_t(), rv.get_mpz_t(), pub_.n.get_mpz_t());
                        if (g == 1) break;
                    }
                    to_words(rv, &r[i * nw], nw);
                }
                rc = sfxb_blind_append(bg_ctx_, blind_, r.data(), k, nullptr);
            }
            if (rc != SFXB_OK) {
                // leave the stream where the queue ends; the next call draws on
                gmp_randclear(rng_);
                gmp_randinit_set(rng_, snap);
                break;
            }
        }
        gmp_randclear(snap);
    }

    // `count` draws of the stream taken and discarded (queued powers first)
    void consume_draws(size_t count) {
        stop_precompute();
        const size_t have = blind_ ? sfxb_blind_size(blind_) : 0, take = std::min(have, count);
        if (take) sfxb_blind_pop(blind_, take);
        if (count > take) {
            std::vector<uint32_t> r((count - take) * n_words_);
            draw_blinding(r.data(), count - take);
        }
    }

    // `count` draws of HeRng::unit_below(n) (he.cpp:19-28).  With p, q the
    // gcd test is done on the device (p | r or q | r, SFXB_ERR_COPRIME) and the
    // state before the batch is kept for an exact replay; without them the
    // gcd runs here.
    void draw_blinding(uint32_t *out, size_t count, bool exact_gcd = false) {
        gmp_randclear(rng_snapshot_);
        gmp_randinit_set(rng_snapshot_, rng_);
        const bool host_gcd = exact_gcd || !has_priv_;
        mpz_class r, g;
        for (size_t i = 0; i < count; ++i) {
            for (;;) {
                mpz_urandomm(r.get_mpz_t(), rng_, pub_.n.get_mpz_t());
                if (r <= 1) continue;
                if (host_gcd) {
                    mpz_gcd(g.get_mpz_t(), r.get_mpz_t(), pub_.n.get_mpz_t());
                    if (g != 1) continue;
                }
                break;
            }
            to_words(r, out + i * n_words_, n_words_);
        }
    }

    static bool merged_equals(const std::vector<std::uint32_t> &a, const std::vector<std::uint32_t> &b,
                              const std::vector<std::uint32_t> &p) {
        if (a.size() + b.size() != p.size()) return false;
        size_t i = 0, j = 0;
        for (std::uint32_t v : p) {
            if (i < a.size() && a[i] == v) ++i;
            else if (j < b.size() && b[j] == v) ++j;
            else return false;
        }
        return i == a.size() && j == b.size();
    }

    // The call's bin columns (J × n u16, column-major) staged in the
    // page-locked buffer `flat`, which still holds the previous call's
    // columns: each block of kBinsBlock rows of one feature is compared with
    // its staged copy on all host threads and copied only where it differs.
    // Returns whether anything differs (exact: no hash) — `same_layout` says
    // whether `flat` holds a previous call of the same J × n.
    static constexpr size_t kBinsBlock = size_t(1) << 18;
    static bool stage_bins(const std::vector<std::vector<uint16_t>> &bins, size_t J, size_t n, uint16_t *flat,
                           bool same_layout) {
        const size_t per_f = (n + kBinsBlock - 1) / kBinsBlock, nb = J * per_f;
        std::atomic<bool> changed{!same_layout};
        parallel_for(nb, [&](size_t lo, size_t hi) {
            for (size_t b = lo; b < hi; ++b) {
                const size_t f = b / per_f, i0 = (b % per_f) * kBinsBlock, cnt = std::min(kBinsBlock, n - i0);
                const uint16_t *src = bins[f].data() + i0;
                uint16_t *dst = flat + f * n + i0;
                if (!same_layout || std::memcmp(dst, src, cnt * 2) != 0) {
                    std::memcpy(dst, src, cnt * 2);
                    changed = true;
                }
            }
        }, /*grain=*/2);
        return changed;
    }

    // ---------------------------------------------------------------- gh residency
    //
    // Per ciphertext of a GhPayload: trivial (value 1: skipped by fold_into),
    // regular (this key, 0 ≤ value < n²: multiplied on the GPU) or irregular
    // (anything else: uploaded as the identity, its slots refolded on the host).
    enum : uint8_t { kRegular = 0, kTrivial = 1, kForeign = 2, kOffRange = 3 };

    struct GhScan {
        uint64_t key = 0;          // buffer addresses, sizes and key ids: the residency pre-filter
        std::vector<uint8_t> cls;  // per ciphertext, header-level class (kOffRange needs the limbs)
    };

    // header-only pass: key id, sign, size, and the value 1
    GhScan scan_gh(const GhPayload &gh) const {
        const size_t count = gh.cts.size();
        constexpr size_t kChunk = 8192;
        const size_t nchunks = (count + kChunk - 1) / kChunk;
        GhScan sc;
        sc.cls.resize(count);
        std::vector<uint64_t> part(nchunks, 0);
        parallel_for(nchunks, [&](size_t lo, size_t hi) {
            for (size_t ch = lo; ch < hi; ++ch) {
                uint64_t h = 14695981039346656037ULL;
                for (size_t i = ch * kChunk; i < std::min(count, (ch + 1) * kChunk); ++i) {
                    const Ciphertext &c = gh.cts[i];
                    const mpz_srcptr z = c.value.get_mpz_t();
                    uint8_t k = kRegular;
                    if (z->_mp_size == 1 && mpz_limbs_read(z)[0] == 1) k = kTrivial;
                    else if (c.key_id != pub_.key_id) k = kForeign;
                    else if (z->_mp_size < 0 || (size_t)z->_mp_size * 2 > ct_words_) k = kOffRange;
                    sc.cls[i] = k;
                    h = (h ^ reinterpret_cast<uintptr_t>(mpz_limbs_read(z))) * 1099511628211ULL;
                    h = (h ^ ((uint64_t)(uint32_t)z->_mp_size << 8 ^ k)) * 1099511628211ULL;
                    h = (h ^ c.key_id) * 1099511628211ULL;
                }
                part[ch] = h;
            }
        }, /*grain=*/1);
        sc.key = (uint64_t)count * 0x9E3779B97F4A7C15ull;
        for (uint64_t x : part) sc.key = (sc.key ^ x) * 1099511628211ULL;
        return sc;
    }

    // full class of ciphertext c (reads the top limbs for the n² bound)
    uint8_t classify(const Ciphertext &c) const {
        const mpz_srcptr z = c.value.get_mpz_t();
        if (z->_mp_size == 1 && mpz_limbs_read(z)[0] == 1) return kTrivial;
        if (c.key_id != pub_.key_id) return kForeign;
        if (z->_mp_size < 0 || (size_t)z->_mp_size * 2 > ct_words_) return kOffRange;
        if (mpz_cmp(z, pub_.n2.get_mpz_t()) >= 0) return kOffRange;
        return kRegular;
    }

    // marshal every ciphertext into the page-locked staging buffer (regular:
    // its limbs; trivial and irregular: the identity), record the irregular
    // ones, upload (sfxb_gh_upload)
    void upload_gh(const GhPayload &gh, uint64_t scan_key) {
        if (gh_) sfxb_gh_free(gh_);
        gh_ = nullptr;
        prev_valid_ = false; // a new resident copy: no cached parents (the handle address may repeat)
        const size_t count = gh.cts.size(), cw = ct_words_;
        uint32_t *limbs = pin_limbs_.get<uint32_t>(count * cw);
        constexpr size_t kChunk = 8192;
        const size_t nchunks = (count + kChunk - 1) / kChunk;
        std::vector<std::vector<uint32_t>> irr(nchunks);
        parallel_for(nchunks, [&](size_t lo, size_t hi) {
            for (size_t ch = lo; ch < hi; ++ch)
                for (size_t i = ch * kChunk; i < std::min(count, (ch + 1) * kChunk); ++i) {
                    uint32_t *w = &limbs[i * cw];
                    const uint8_t k = classify(gh.cts[i]);
                    if (k == kRegular) {
                        to_words(gh.cts[i].value, w, cw);
                    } else {
                        std::memset(w, 0, cw * 4);
                        w[0] = 1;
                        if (k != kTrivial) irr[ch].push_back((uint32_t)i);
                    }
                }
        }, /*grain=*/1);
        irr_.clear();
        for (const auto &v : irr)
            for (uint32_t i : v) irr_.push_back(IrrCt{i, gh.cts[i]});
        check(sfxb_gh_upload(ctx_, limbs, gh.n_samples, &gh_));
        gh_scan_key_ = scan_key;
        gh_count_ = count;
    }

    // every limb of gh equals the resident copy (staging buffer) and the
    // irregular ciphertexts are the recorded ones
    bool verify_gh(const GhPayload &gh) const {
        const size_t count = gh.cts.size(), cw = ct_words_;
        const uint32_t *limbs = pin_limbs_.peek<uint32_t>();
        constexpr size_t kChunk = 8192;
        const size_t nchunks = (count + kChunk - 1) / kChunk;
        std::atomic<bool> same{true};
        std::vector<std::vector<uint32_t>> irr(nchunks);
        parallel_for(nchunks, [&](size_t lo, size_t hi) {
            for (size_t ch = lo; ch < hi && same; ++ch)
                for (size_t i = ch * kChunk; i < std::min(count, (ch + 1) * kChunk); ++i) {
                    const uint32_t *w = &limbs[i * cw];
                    const uint8_t k = classify(gh.cts[i]);
                    bool ok;
                    if (k == kRegular) {
                        const mpz_srcptr z = gh.cts[i].value.get_mpz_t();
                        const size_t used = (size_t)z->_mp_size, bytes = used * 8;
                        ok = std::memcmp(w, mpz_limbs_read(z), bytes) == 0;
                        for (size_t j = bytes / 4; ok && j < cw; ++j) ok = w[j] == 0;
                    } else {
                        ok = w[0] == 1;
                        for (size_t j = 1; ok && j < cw; ++j) ok = w[j] == 0;
                        if (k != kTrivial) irr[ch].push_back((uint32_t)i);
                    }
                    if (!ok) {
                        same = false;
                        break;
                    }
                }
        }, /*grain=*/1);
        if (!same) return false;
        size_t j = 0;
        for (const auto &v : irr)
            for (uint32_t i : v) {
                if (j >= irr_.size() || irr_[j].index != i || irr_[j].ct.key_id != gh.cts[i].key_id ||
                    mpz_cmp(irr_[j].ct.value.get_mpz_t(), gh.cts[i].value.get_mpz_t()) != 0)
                    return false;
                ++j;
            }
        return j == irr_.size();
    }

    // The reference's loop (secure_processor.cpp:603-618 with fold_into
    // :724-732 and add_ciphertexts' key check, he.cpp:117-121) replayed on
    // ciphertext classes only: the first exception it raises and the
    // additions it counted before.  Used on the error paths (bad bin, key
    // mismatch), where the call fails exactly where the reference's would.
    [[noreturn]] void fail_with_replay(const GhPayload &gh, const GhScan &scan,
                                       const std::vector<std::vector<std::uint16_t>> &bins, size_t J,
                                       const std::vector<NodeRows> &nodes, int n_bins) {
        const size_t K = (size_t)std::max(n_bins, 0);
        std::vector<uint8_t> st; // per slot: 0 empty (trivial), 1 this key, 2 foreign
        uint64_t adds = 0;
        auto fail = [&](const char *msg) {
            counters_.ciphertext_additions += adds;
            throw Error(msg);
        };
        for (const NodeRows &nd : nodes) {
            st.assign(2 * J * K, 0);
            for (size_t f = 0; f < J; ++f)
                for (std::uint32_t row : nd.rows) {
                    if (row >= gh.n_samples) fail("row index out of range in accumulate");
                    const std::uint16_t b = bins[f][row];
                    if (b >= static_cast<std::uint16_t>(n_bins)) fail("bin index out of range in accumulate");
                    for (size_t w = 0; w < 2; ++w) {
                        const uint8_t k = scan.cls[2 * (size_t)row + w];
                        if (k == kTrivial) continue;
                        uint8_t &s = st[2 * (f * K + b) + w];
                        if (s == 0) {
                            s = k == kForeign ? 2 : 1;
                            continue;
                        }
                        if (s == 2 || k == kForeign) fail("add_ciphertexts: key mismatch");
                        ++adds;
                        s = 1;
                    }
                }
        }
        // not reached on the paths that call this (they saw a failure)
        counters_.ciphertext_additions += adds;
        throw Error("accumulate: internal replay found no failure");
    }

    // Slots holding irregular ciphertexts, folded again on the host with the
    // reference's rules over all of their entries in row order; returns the
    // call's reference addition count (the GPU counted those slots without
    // their irregular entries).
    uint64_t refold_irregular(const GhPayload &gh, const GhScan &scan,
                              const std::vector<std::vector<std::uint16_t>> &bins, size_t J,
                              const std::vector<NodeRows> &nodes, int n_bins, HistogramPayload &out, uint64_t adds) {
        const size_t K = (size_t)std::max(n_bins, 0);
        std::vector<uint8_t> is_irr_row(gh.n_samples, 0);
        for (const IrrCt &x : irr_) is_irr_row[x.index / 2] = 1;
        for (size_t i = 0; i < nodes.size(); ++i) {
            const NodeRows &nd = nodes[i];
            // (feature, slot) pairs of this node touched by an irregular entry
            std::vector<std::pair<size_t, size_t>> hit;
            for (std::uint32_t row : nd.rows)
                if (is_irr_row[row])
                    for (size_t f = 0; f < J; ++f)
                        for (size_t w = 0; w < 2; ++w) {
                            const size_t ci = 2 * (size_t)row + w;
                            const uint8_t k = scan.cls[ci] == kRegular ? classify(gh.cts[ci]) : scan.cls[ci];
                            if (k == kForeign || k == kOffRange) hit.emplace_back(f, 2 * (f * K + bins[f][row]) + w);
                        }
            std::sort(hit.begin(), hit.end());
            hit.erase(std::unique(hit.begin(), hit.end()), hit.end());
            for (const auto &[f, slot] : hit) {
                const size_t b = (slot / 2) % K, w = slot & 1;
                Ciphertext acc{mpz_class(1), pub_.key_id}; // trivial_zero (he.cpp:123)
                uint64_t ref_adds = 0, gpu_entries = 0;
                for (std::uint32_t row : nd.rows) {
                    if (bins[f][row] != b) continue;
                    const Ciphertext &c = gh.cts[2 * (size_t)row + w];
                    if (c.value == 1) continue;                      // fold_into: rhs trivial
                    if (classify(c) == kRegular) ++gpu_entries;
                    if (acc.value == 1) {                            // lhs trivial: assign
                        acc = c;
                        continue;
                    }
                    if (acc.key_id != c.key_id || acc.key_id != pub_.key_id)
                        fail_with_replay(gh, scan, bins, J, nodes, n_bins);
                    mpz_mul(acc.value.get_mpz_t(), acc.value.get_mpz_t(), c.value.get_mpz_t());
                    mpz_tdiv_r(acc.value.get_mpz_t(), acc.value.get_mpz_t(), pub_.n2.get_mpz_t());
                    acc.key_id = pub_.key_id;
                    ++ref_adds;
                }
                adds = adds - (gpu_entries ? gpu_entries - 1 : 0) + ref_adds;
                out.nodes[i].scalar_cts[slot] = std::move(acc);
            }
        }
        return adds;
    }

    void check(int rc) {
        if (rc == SFXB_OK) return;
        std::string msg = sfxb_last_error(ctx_);
        if (rc == SFXB_ERR_AUTH) throw AuthorizationError(msg);
        throw Error(msg);
    }

    // Error path of decrypt_histogram: the reference decrypts slot by slot
    // (secure_processor.cpp:687-696, decrypt_slot :734-738, decrypt he.cpp:
    // 105-115) and stops at the first non-trivial slot with a foreign key,
    // a value outside [1, n²) or a common factor with n — in that order per
    // slot — having counted every non-trivial slot up to and including it.
    // Locate that slot (gcd on all host threads, only here) and fail there.
    [[noreturn]] void fail_decrypt(const HistogramPayload &payload, bool coprime_error) {
        std::vector<const Ciphertext *> nt; // non-trivial slots in the reference's order
        for (const NodeHistogram &node : payload.nodes) {
            const size_t cnt = 2 * node.feature_ids.size() * (size_t)std::max(node.n_bins, 0);
            for (size_t s = 0; s < cnt && s < node.scalar_cts.size(); ++s)
                if (!(node.scalar_cts[s].value == 1)) nt.push_back(&node.scalar_cts[s]);
        }
        auto header_err = [&](const Ciphertext &c) -> const char * {
            if (c.key_id != pub_.key_id) return "decrypt: ciphertext key mismatch";
            if (c.value < 1 || c.value >= pub_.n2) return "decrypt: ciphertext out of range";
            return nullptr;
        };
        size_t first = nt.size();
        const char *msg = nullptr;
        if (!coprime_error)
            for (size_t k = 0; k < nt.size(); ++k)
                if ((msg = header_err(*nt[k]))) {
                    first = k;
                    break;
                }
        // an earlier slot not coprime to n fails first
        std::vector<uint8_t> nc(first, 0);
        parallel_for(first, [&](size_t lo, size_t hi) {
            mpz_class g;
            for (size_t k = lo; k < hi; ++k) {
                if (header_err(*nt[k])) continue;
                mpz_gcd(g.get_mpz_t(), nt[k]->value.get_mpz_t(), pub_.n.get_mpz_t());
                nc[k] = g != 1;
            }
        }, /*grain=*/256);
        for (size_t k = 0; k < first; ++k)
            if (nc[k]) {
                first = k;
                msg = "decrypt: ciphertext not coprime to modulus";
                break;
            }
        if (!msg) throw Error("decrypt_histogram: GPU reported an error no slot reproduces");
        counters_.decryptions += first + 1;
        throw Error(msg);
    }

    // One tree level of one sender's histograms: sibling nodes (ids k, k+1 with
    // k odd, federation.cpp:331-345) whose parent is found in a previously
    // decrypted level are decrypted by verified reuse (sfxb_decrypt_tree);
    // everything else decrypts slot by slot as before.  Senders are not
    // named in the payload, so up to kStreams previous levels are kept and a
    // level continues the stream its first sibling pair matches.
    bool find_parent(const DecStream &st, const NodeHistogram &a, const NodeHistogram &b, uint32_t from,
                     uint32_t *out) {
        mpz_class P, t;
        for (uint32_t tries = 0; tries < st.n_nodes; ++tries) {
            const uint32_t pc = (from + tries) % st.n_nodes;
            const uint32_t *pw = &st.cts[(size_t)pc * st.spn * ct_words_];
            size_t s = 0;
            auto trivial = [&](size_t k) {
                const uint32_t *w = pw + k * ct_words_;
                return w[0] == 1 && std::all_of(w + 1, w + ct_words_, [](uint32_t x) { return x == 0; });
            };
            while (s < st.spn && trivial(s)) ++s;
            if (s == st.spn) continue;
            // one non-trivial slot selects the candidate; the GPU verifies every slot
            mpz_import(P.get_mpz_t(), ct_words_, -1, 4, 0, 0, pw + s * ct_words_);
            t = a.scalar_cts[s].value * b.scalar_cts[s].value;
            mpz_mod(t.get_mpz_t(), t.get_mpz_t(), pub_.n2.get_mpz_t());
            if (t == P) {
                *out = pc;
                return true;
            }
        }
        return false;
    }

    void decrypt_level(const HistogramPayload &payload, LimbVec &cts, std::vector<double> &vals,
                       uint64_t *decs, PhaseTimer &pt) {
        const auto &nodes = payload.nodes;
        const size_t spn = 2 * nodes[0].feature_ids.size() * (size_t)std::max(nodes[0].n_bins, 0);
        bool uniform = spn > 0;
        for (const NodeHistogram &nd : nodes)
            uniform &= nd.feature_ids == nodes[0].feature_ids && nd.n_bins == nodes[0].n_bins;
        if (!uniform) {
            check(sfxb_decrypt(ctx_, cts.data(), vals.size(), scale_bits_, vals.data(), nullptr, decs));
            return;
        }
        std::vector<size_t> pairs; // index of the first node of each sibling pair
        for (size_t i = 0; i + 1 < nodes.size(); ++i)
            if ((nodes[i].node_id & 1u) && nodes[i + 1].node_id == nodes[i].node_id + 1) pairs.push_back(i++);
        // the stream this level continues
        DecStream *st = nullptr;
        uint32_t first = 0;
        if (!pairs.empty())
            for (DecStream &c : dec_streams_)
                if (c.spn == spn && c.n_nodes &&
                    find_parent(c, nodes[pairs[0]], nodes[pairs[0] + 1], 0, &first)) {
                    st = &c;
                    break;
                }
        std::vector<int32_t> parent(nodes.size(), -1);
        const bool continues = st != nullptr;
        if (st) {
            uint32_t cand = first;
            for (size_t i : pairs) {
                uint32_t pc;
                if (find_parent(*st, nodes[i], nodes[i + 1], cand, &pc)) {
                    parent[i] = parent[i + 1] = (int32_t)pc;
                    cand = pc + 1;
                }
            }
        } else {
            // a level without sibling pairs is a sender's root level: the
            // trees of every sender advance level by level together
            // (federation.cpp:456-534), so a stream that already continued
            // past its root belongs to a finished tree.  Recycling the least
            // recently used of those keeps one cache tag (and its device
            // buffers, grown to the deepest level) per sender across trees.
            DecStream *done = nullptr;
            if (pairs.empty())
                for (DecStream &c : dec_streams_)
                    if (c.continued && (!done || c.last_use < done->last_use)) done = &c;
            if (done) {
                st = done;
            } else if (dec_streams_.size() < kStreams) {
                dec_streams_.emplace_back();
                dec_streams_.back().tag = dec_streams_.size();
                st = &dec_streams_.back();
            } else {
                st = &*std::min_element(dec_streams_.begin(), dec_streams_.end(),
                                        [](const DecStream &x, const DecStream &y) { return x.last_use < y.last_use; });
            }
        }
        pt.lap("parents");
        check(sfxb_decrypt_tree(ctx_, st->tag, cts.data(), (uint32_t)nodes.size(), (uint32_t)spn, parent.data(),
                                scale_bits_, vals.data(), decs));
        pt.lap("gpu");
        st->cts.swap(cts);
        st->continued = continues ? st->continued + 1 : 0;
        st->n_nodes = (uint32_t)nodes.size();
        st->spn = spn;
        st->last_use = ++dec_clock_;
    }

    // add_packed (he.cpp:234-253): shape and guard-capacity checks, key checks
    // of add_ciphertexts per element; a becomes the sum's descriptor
    void plan_add_packed(PackedVector &a, const PackedVector &b,
                         std::vector<std::pair<Ciphertext *, const Ciphertext *>> &work) {
        if (a.logical_length != b.logical_length || a.slot_bits != b.slot_bits || a.guard_bits != b.guard_bits ||
            a.scale_bits != b.scale_bits || a.cts.size() != b.cts.size())
            throw Error("add_packed: shape mismatch");
        const std::uint64_t count = std::uint64_t(a.addend_count) + b.addend_count;
        if (count > (std::uint64_t(1) << a.guard_bits)) throw Error("add_packed: addend capacity exceeded (guard bits)");
        for (std::size_t i = 0; i < a.cts.size(); ++i)
            if (a.cts[i].key_id != b.cts[i].key_id || a.cts[i].key_id != pub_.key_id)
                throw Error("add_ciphertexts: key mismatch");
        a.addend_count = static_cast<std::uint32_t>(count);
        for (std::size_t i = 0; i < a.cts.size(); ++i) work.emplace_back(&a.cts[i], &b.cts[i]);
    }

    // lhs = lhs·rhs mod n² for every pair: one GPU batch; values outside
    // [0, n²) (never produced by an encryption) take GMP's a·b % n² exactly
    void multiply_into(const std::vector<std::pair<Ciphertext *, const Ciphertext *>> &work) {
        std::vector<size_t> dev;
        for (size_t i = 0; i < work.size(); ++i) {
            const mpz_class &x = work[i].first->value, &y = work[i].second->value;
            if (x >= 0 && x < pub_.n2 && y >= 0 && y < pub_.n2 && fits(x, ct_words_) && fits(y, ct_words_))
                dev.push_back(i);
            else
                work[i].first->value = x * y % pub_.n2;
        }
        if (dev.empty()) return;
        std::vector<uint32_t> A(dev.size() * ct_words_), B(dev.size() * ct_words_), C(dev.size() * ct_words_);
        parallel_for(dev.size(), [&](size_t lo, size_t hi) {
            for (size_t k = lo; k < hi; ++k) {
                to_words(work[dev[k]].first->value, &A[k * ct_words_], ct_words_);
                to_words(work[dev[k]].second->value, &B[k * ct_words_], ct_words_);
            }
        });
        check(sfxb_add(ctx_, A.data(), B.data(), dev.size(), C.data()));
        parallel_for(dev.size(), [&](size_t lo, size_t hi) {
            for (size_t k = lo; k < hi; ++k) {
                from_words(work[dev[k]].first->value, &C[k * ct_words_], ct_words_);
                work[dev[k]].first->key_id = pub_.key_id;
            }
        });
    }

    // packed decrypt_histogram (secure_processor.cpp:697-712) = unpack_decrypt
    // (he.cpp:255-259) per vector: the CRT decryptions of every ciphertext run
    // as one GPU batch; key/range/coprime errors and unpack_plain errors
    // surface in the reference's order.
    std::vector<std::pair<std::uint32_t, Histogram>> decrypt_packed(const HistogramPayload &payload) {
        std::vector<const PackedVector *> vecs;
        for (const NodeHistogram &node : payload.nodes) {
            vecs.push_back(&node.packed_g);
            vecs.push_back(&node.packed_h);
        }
        size_t total = 0;
        for (const PackedVector *v : vecs) total += v->cts.size();
        std::vector<uint32_t> cts(total * ct_words_);
        size_t bad = total;
        std::string bad_msg;
        {
            size_t i = 0;
            for (const PackedVector *v : vecs) {
                for (const Ciphertext &c : v->cts) {
                    if (c.key_id != pub_.key_id) bad_msg = "decrypt: ciphertext key mismatch";
                    else if (c.value < 1 || c.value >= pub_.n2 || !fits(c.value, ct_words_))
                        bad_msg = "decrypt: ciphertext out of range";
                    if (!bad_msg.empty()) break;
                    to_words(c.value, &cts[i * ct_words_], ct_words_);
                    ++i;
                }
                if (!bad_msg.empty()) break;
            }
            bad = i;
        }
        std::vector<uint32_t> plain(std::max<size_t>(bad, 1) * n_words_);
        std::vector<double> vals(std::max<size_t>(bad, 1));
        uint64_t decs = 0;
        if (bad) {
            int rc = sfxb_decrypt(ctx_, cts.data(), bad, scale_bits_, vals.data(), plain.data(), &decs);
            if (rc == SFXB_ERR_COPRIME) {
                // locate the first ciphertext sharing a factor with n, as the reference would meet it
                mpz_class g;
                size_t k = 0;
                for (const PackedVector *v : vecs) {
                    for (const Ciphertext &c : v->cts) {
                        if (k == bad) break;
                        mpz_gcd(g.get_mpz_t(), c.value.get_mpz_t(), pub_.n.get_mpz_t());
                        if (g != 1) break;
                        ++k;
                    }
                    if (k == bad || g != 1) break;
                }
                bad = k;
                bad_msg = "decrypt: ciphertext not coprime to modulus";
                rc = bad ? sfxb_decrypt(ctx_, cts.data(), bad, scale_bits_, vals.data(), plain.data(), &decs) : SFXB_OK;
            }
            check(rc);
        }
        std::vector<std::pair<std::uint32_t, Histogram>> out;
        size_t idx = 0, vi = 0;
        for (const NodeHistogram &node : payload.nodes) {
            std::vector<double> gh[2];
            for (int w = 0; w < 2; ++w, ++vi) {
                const PackedVector &v = *vecs[vi];
                if (bad < idx + v.cts.size()) throw Error(bad_msg);
                std::vector<mpz_class> m(v.cts.size());
                for (size_t k = 0; k < m.size(); ++k) from_words(m[k], &plain[(idx + k) * n_words_], n_words_);
                const PackedLayout layout{pub_.modulus_bits, v.slot_bits, v.guard_bits, v.scale_bits};
                gh[w] = packing::unpack(layout, m, v.logical_length, v.addend_count);
                idx += v.cts.size();
            }
            counters_.decryptions += 2; // vector granularity
            const std::size_t expect = node.feature_ids.size() * static_cast<std::size_t>(node.n_bins);
            if (gh[0].size() != expect || gh[1].size() != expect)
                throw Error("decrypt_histogram: packed length mismatch");
            Histogram hist;
            hist.n_bins = node.n_bins;
            hist.feature_ids = node.feature_ids;
            for (std::size_t f = 0; f < node.feature_ids.size(); ++f) {
                std::vector<GHPair> slots(static_cast<std::size_t>(node.n_bins));
                for (int b = 0; b < node.n_bins; ++b) {
                    const std::size_t i = f * static_cast<std::size_t>(node.n_bins) + static_cast<std::size_t>(b);
                    slots[static_cast<std::size_t>(b)] = {gh[0][i], gh[1][i]};
                }
                hist.feats.push_back(std::move(slots));
            }
            out.emplace_back(node.node_id, std::move(hist));
        }
        return out;
    }

    PaillierPublicKey pub_;
    PaillierPrivateKey priv_;
    bool has_priv_;
    unsigned scale_bits_;
    PackedLayout layout_; // validated lazily, as the reference does
    gmp_randstate_t rng_, rng_snapshot_;
    sfxb_ctx *ctx_ = nullptr;
    size_t n_words_ = 0, ct_words_ = 0;
    size_t enc_wave_ = 0; // sfxb_ctx_enc_wave: encryptions per GPU wave
    sfxb_gh *gh_ = nullptr;
    PinnedBuf pin_r_, pin_cts_, pin_slots_, pin_limbs_, pin_bins_; // page-locked marshalling buffers
    // offline phase: background context, queue of blinding powers, worker
    sfxb_ctx *bg_ctx_ = nullptr;
    sfxb_blind *blind_ = nullptr;
    size_t blind_cap_ = 0;
    std::thread bg_;
    std::atomic<bool> bg_stop_{false};
    // previous accumulate call (sibling-subtraction parents)
    bool prev_valid_ = false;
    // staged bin columns (pin_bins_) and their device copy
    size_t staged_J_ = 0, staged_n_ = 0;
    std::vector<int> staged_fids_;
    int staged_K_ = -1;
    sfxb_bins *bins_h_ = nullptr;
    size_t bins_h_J_ = 0, bins_h_n_ = 0;
    const sfxb_gh *prev_gh_ = nullptr;
    std::vector<std::vector<std::uint32_t>> prev_rows_;
    // resident gh: pre-filter key, count, and its irregular ciphertexts
    struct IrrCt {
        uint32_t index;
        Ciphertext ct;
    };
    uint64_t gh_scan_key_ = 0;
    size_t gh_count_ = 0;
    std::vector<IrrCt> irr_;
    std::vector<DecStream> dec_streams_;
    uint64_t dec_clock_ = 0;
};

} // namespace

// ------------------------------------------------------------ the factories (interposed)

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg) {
    return std::make_unique<CudaPaillierPlugin>(pk, cfg);
}

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierKeypair &kp, const PaillierPluginConfig &cfg) {
    return std::make_unique<CudaPaillierPlugin>(kp, cfg);
}

} // namespace sfxb
