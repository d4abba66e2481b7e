// TEST INFRASTRUCTURE ONLY.
//
// Integer-sum oracle plugin (SURVEY §8c "exact integer-sum oracle for large
// configs").  An EncryptionPlugin whose "ciphertexts" carry the fixed-point
// plaintexts themselves, so the reference's vertical training loop runs at
// the HIGGS scale (1M rows, 2048-bit key) in seconds while producing exactly
// the decrypted histograms, splits, trees and op counters a Paillier run
// produces:
//   * encrypt_gh: m = encode_fixed(x) (he.cpp:125-136, the reference's own
//     function and checks), stored as value m + 2 (never the trivial zero 1);
//     encryptions += 2 per pair (secure_processor.cpp:574-585).
//   * accumulate_rows: Paillier decryption is a homomorphism, Dec(∏ c_i) =
//     Σ m_i mod n, and m_i ≡ q_i (mod n) with q_i the signed fixed-point
//     integer; so every slot is Σ q_i in 128-bit integers (|Σ| < 2^63 at 10M
//     rows), reduced mod n at the end.  Validation, the slot layout
//     2(f·K+b)+{G,H}, the trivial zero and the addition counter follow
//     secure_processor.cpp:587-620 and fold_into :724-732 (one counted
//     addition per non-trivial entry after a slot's first).
//   * decrypt_histogram: trivial slots → 0.0 uncounted; otherwise
//     decryptions += 1 and decode_fixed(value − 2) (he.cpp:138-143, the
//     reference's own function: mpz_get_d truncation).
// Loaded with LD_PRELOAD ahead of the reference library it replaces both
// make_paillier_plugin overloads, like the GPU adapter.  The wire bytes differ
// from a Paillier run (shorter values); everything decrypted is identical.
#include <gmp.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sfxb/errors.hpp"
#include "sfxb/secure_processor.hpp"

namespace sfxb {
namespace {

class IntSumPlugin final : public EncryptionPlugin {
public:
    IntSumPlugin(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg, bool priv)
        : pub_(pk), priv_(priv), scale_(cfg.scale_bits) {
        half_ = pub_.n / 2;
    }
    std::string name() const override { return "paillier"; }
    bool is_passthrough() const override { return false; }
    bool holds_private_key() const override { return priv_; }
    std::uint64_t key_id() const override { return pub_.key_id; }

    GhPayload encrypt_gh(std::span<const GHPair> gh) override {
        GhPayload out;
        out.encrypted = true;
        out.n_samples = static_cast<std::uint32_t>(gh.size());
        out.cts.reserve(2 * gh.size());
        for (const GHPair &p : gh) {
            for (double x : {p.g, p.h}) out.cts.push_back(Ciphertext{encode_fixed(pub_, x, scale_) + 2, pub_.key_id});
            counters_.encryptions += 2;
        }
        return out;
    }

    HistogramPayload accumulate_rows(const GhPayload &gh, const std::vector<std::vector<std::uint16_t>> &bins,
                                     const std::vector<int> &feature_ids, const std::vector<NodeRows> &nodes,
                                     int n_bins) override {
        if (!gh.encrypted) throw Error("paillier accumulate expects encrypted gradients");
        if (gh.cts.size() != 2ull * gh.n_samples) throw Error("row-count mismatch: ciphertext count is not 2·n_samples");
        for (const auto &col : bins)
            if (col.size() != gh.n_samples) throw Error("row-count mismatch between bins and gradients");
        // signed plaintext of every ciphertext (value − 2 = m; m > n/2 is negative)
        std::vector<__int128> q(gh.cts.size());
        std::vector<uint8_t> trivial(gh.cts.size());
        mpz_class m;
        for (size_t i = 0; i < gh.cts.size(); ++i) {
            const Ciphertext &c = gh.cts[i];
            trivial[i] = c.value == 1;
            if (trivial[i]) continue;
            if (c.key_id != pub_.key_id) throw Error("add_ciphertexts: key mismatch");
            m = c.value - 2;
            const bool neg = m > half_;
            if (neg) m = pub_.n - m;
            if (mpz_sizeinbase(m.get_mpz_t(), 2) > 100) throw Error("intsum oracle: plaintext beyond 100 bits");
            unsigned __int128 v = 0;
            size_t cnt = 0;
            uint64_t w[2] = {0, 0};
            mpz_export(w, &cnt, -1, 8, 0, 0, m.get_mpz_t());
            v = ((unsigned __int128)w[1] << 64) | w[0];
            q[i] = neg ? -(__int128)v : (__int128)v;
        }
        HistogramPayload out;
        out.layout = HistLayout::enc_scalar;
        const size_t K = static_cast<size_t>(n_bins);
        std::vector<__int128> sum;
        std::vector<uint32_t> cnt;
        for (const NodeRows &node : nodes) {
            NodeHistogram nh;
            nh.node_id = node.node_id;
            nh.feature_ids = feature_ids;
            nh.n_bins = n_bins;
            sum.assign(2 * feature_ids.size() * K, 0);
            cnt.assign(2 * feature_ids.size() * K, 0);
            for (size_t f = 0; f < feature_ids.size(); ++f) {
                const std::vector<std::uint16_t> &col = bins[f];
                for (std::uint32_t row : node.rows) {
                    const std::uint16_t b = col[row];
                    if (b >= static_cast<std::uint16_t>(n_bins)) throw Error("bin index out of range in accumulate");
                    for (size_t w = 0; w < 2; ++w) {
                        const size_t i = 2 * (size_t)row + w, s = 2 * (f * K + b) + w;
                        if (trivial[i]) continue;
                        if (cnt[s]++) ++counters_.ciphertext_additions;
                        sum[s] += q[i];
                    }
                }
            }
            nh.scalar_cts.assign(sum.size(), Ciphertext{mpz_class(1), pub_.key_id});
            for (size_t s = 0; s < sum.size(); ++s) {
                if (!cnt[s]) continue;
                const bool neg = sum[s] < 0;
                const unsigned __int128 a = neg ? (unsigned __int128)(-sum[s]) : (unsigned __int128)sum[s];
                const uint64_t w[2] = {(uint64_t)a, (uint64_t)(a >> 64)};
                mpz_import(m.get_mpz_t(), 2, -1, 8, 0, 0, w);
                if (neg && m != 0) m = pub_.n - m; // Σ mod n (|Σ| < n/2)
                nh.scalar_cts[s].value = m + 2;
            }
            out.nodes.push_back(std::move(nh));
        }
        return out;
    }

    HistogramPayload encrypt_histogram(const std::vector<std::pair<std::uint32_t, Histogram>> &) override {
        throw Error("intsum oracle: the packed (horizontal) path is not modelled");
    }
    HistogramPayload add_histograms(const std::vector<HistogramPayload> &) override {
        throw Error("intsum oracle: the packed (horizontal) path is not modelled");
    }

    std::vector<std::pair<std::uint32_t, Histogram>> decrypt_histogram(const HistogramPayload &payload) override {
        if (!priv_) throw AuthorizationError("decrypt requested without private key material");
        if (payload.layout != HistLayout::enc_scalar) throw Error("intsum oracle: scalar layout only");
        std::vector<std::pair<std::uint32_t, Histogram>> out;
        for (const NodeHistogram &node : payload.nodes) {
            Histogram hist;
            hist.n_bins = node.n_bins;
            hist.feature_ids = node.feature_ids;
            hist.feats.assign(node.feature_ids.size(), std::vector<GHPair>(static_cast<size_t>(node.n_bins)));
            for (size_t f = 0; f < node.feature_ids.size(); ++f)
                for (int b = 0; b < node.n_bins; ++b) {
                    const size_t base = 2 * (f * static_cast<size_t>(node.n_bins) + static_cast<size_t>(b));
                    hist.feats[f][b].g = slot(node.scalar_cts[base]);
                    hist.feats[f][b].h = slot(node.scalar_cts[base + 1]);
                }
            out.emplace_back(node.node_id, std::move(hist));
        }
        return out;
    }

private:
    double slot(const Ciphertext &c) {
        if (c.value == 1) return 0.0;
        counters_.decryptions += 1;
        if (c.key_id != pub_.key_id) throw Error("decrypt: ciphertext key mismatch");
        return decode_fixed(pub_, c.value - 2, scale_);
    }

    PaillierPublicKey pub_;
    bool priv_;
    unsigned scale_;
    mpz_class half_;
};

} // namespace

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierPublicKey &pk, const PaillierPluginConfig &cfg) {
    return std::make_unique<IntSumPlugin>(pk, cfg, false);
}

std::unique_ptr<EncryptionPlugin> make_paillier_plugin(const PaillierKeypair &kp, const PaillierPluginConfig &cfg) {
    return std::make_unique<IntSumPlugin>(kp.pub, cfg, true);
}

} // namespace sfxb
