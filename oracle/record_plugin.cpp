// TEST INFRASTRUCTURE ONLY.
//
// Recording wrapper around whatever make_paillier_plugin comes next in the
// symbol search order (the GPU adapter, the integer-sum oracle or the
// reference itself): LD_PRELOAD="librecord_plugin.so <plugin>.so".  Every
// call is forwarded unchanged; every decrypt_histogram result (node ids,
// feature ids, bin count, the bits of every decoded G and H) is folded into an
// FNV-1a digest per plugin instance, and per call, and the per-call wall
// times of the three scalar entry points are summed.  At destruction one line
// goes to stderr:
//   [sfxb-record] {"key": ..., "private": ..., "decrypt_calls": ..., "slots": ...,
//                  "fnv": ..., "per_call": [...], "counters": [...], "seconds": {...}}
// so two training runs can be compared decrypted histogram by decrypted
// histogram (tests/test_gpu_scale_parity.py).
#include <dlfcn.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sfxb/errors.hpp"
#include "sfxb/secure_processor.hpp"

namespace sfxb {
namespace {

using PubFactory = std::unique_ptr<EncryptionPlugin> (*)(const PaillierPublicKey &, const PaillierPluginConfig &);
using PairFactory = std::unique_ptr<EncryptionPlugin> (*)(const PaillierKeypair &, const PaillierPluginConfig &);

template <typename Fn>
Fn next(const char *mangled) {
    void *p = dlsym(RTLD_NEXT, mangled);
    if (!p) throw Error(std::string("record plugin: no next definition of ") + mangled);
    return reinterpret_cast<Fn>(p);
}

struct Fnv {
    uint64_t h = 14695981039346656037ULL;
    void add(const void *p, size_t n) {
        const unsigned char *c = static_cast<const unsigned char *>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ULL;
    }
    template <typename T>
    void add(const T &v) {
        add(&v, sizeof v);
    }
};

class Recorder final : public EncryptionPlugin {
public:
    explicit Recorder(std::unique_ptr<EncryptionPlugin> in) : in_(std::move(in)) {}
    ~Recorder() override {
        std::string pc;
        for (size_t i = 0; i < per_call_.size(); ++i) {
            char b[24];
            std::snprintf(b, sizeof b, "%s\"%016llx\"", i ? ", " : "", (unsigned long long)per_call_[i]);
            pc += b;
        }
        const OpCounters &c = in_->counters();
        std::fprintf(stderr,
                     "[sfxb-record] {\"key\": \"%016llx\", \"private\": %s, \"decrypt_calls\": %zu, \"slots\": %llu, "
                     "\"fnv\": \"%016llx\", \"per_call\": [%s], \"counters\": [%llu, %llu, %llu], \"seconds\": "
                     "{\"encrypt_gh\": %.6f, \"accumulate_rows\": %.6f, \"decrypt_histogram\": %.6f}}\n",
                     (unsigned long long)in_->key_id(), in_->holds_private_key() ? "true" : "false",
                     per_call_.size(), (unsigned long long)slots_, (unsigned long long)all_.h, pc.c_str(),
                     (unsigned long long)c.encryptions, (unsigned long long)c.ciphertext_additions,
                     (unsigned long long)c.decryptions, t_enc_, t_acc_, t_dec_);
    }
    std::string name() const override { return in_->name(); }
    bool is_passthrough() const override { return in_->is_passthrough(); }
    bool holds_private_key() const override { return in_->holds_private_key(); }
    std::uint64_t key_id() const override { return in_->key_id(); }

    GhPayload encrypt_gh(std::span<const GHPair> gh) override {
        return timed(t_enc_, [&] { return in_->encrypt_gh(gh); });
    }
    HistogramPayload accumulate_rows(const GhPayload &gh, const std::vector<std::vector<std::uint16_t>> &bins,
                                     const std::vector<int> &feature_ids, const std::vector<NodeRows> &nodes,
                                     int n_bins) override {
        return timed(t_acc_, [&] { return in_->accumulate_rows(gh, bins, feature_ids, nodes, n_bins); });
    }
    HistogramPayload encrypt_histogram(const std::vector<std::pair<std::uint32_t, Histogram>> &h) override {
        return timed(t_other_, [&] { return in_->encrypt_histogram(h); });
    }
    HistogramPayload add_histograms(const std::vector<HistogramPayload> &parts) override {
        return timed(t_other_, [&] { return in_->add_histograms(parts); });
    }
    std::vector<std::pair<std::uint32_t, Histogram>> decrypt_histogram(const HistogramPayload &payload) override {
        auto res = timed(t_dec_, [&] { return in_->decrypt_histogram(payload); });
        Fnv call;
        for (const auto &[id, h] : res) {
            call.add(id);
            call.add(h.n_bins);
            for (int f : h.feature_ids) call.add(f);
            for (const auto &bins : h.feats)
                for (const GHPair &b : bins) {
                    call.add(b.g);
                    call.add(b.h);
                    slots_ += 2;
                }
        }
        per_call_.push_back(call.h);
        all_.add(call.h);
        return res;
    }

private:
    template <typename F>
    auto timed(double &acc, F &&f) -> decltype(f()) {
        struct Sync { // counters follow the inner plugin even when the call throws
            Recorder *r;
            double &acc;
            std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
            ~Sync() {
                acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                r->counters_ = r->in_->counters();
            }
        } s{this, acc};
        return f();
    }

    std::unique_ptr<EncryptionPlugin> in_;
    Fnv all_;
    std::vector<uint64_t> per_call_;
    uint64_t slots_ = 0;
    double t_enc_ = 0, t_acc_ = 0, t_dec_ = 0, t_other_ = 0;
};

} // namespace

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg) {
    static PubFactory f = next<PubFactory>(
        "_ZN4sfxb20make_paillier_pluginERKNS_17PaillierPublicKeyERKNS_20PaillierPluginConfigE");
    return std::make_unique<Recorder>(f(pk, cfg));
}

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierKeypair &kp, const PaillierPluginConfig &cfg) {
    static PairFactory f = next<PairFactory>(
        "_ZN4sfxb20make_paillier_pluginERKNS_15PaillierKeypairERKNS_20PaillierPluginConfigE");
    return std::make_unique<Recorder>(f(kp, cfg));
}

} // namespace sfxb
