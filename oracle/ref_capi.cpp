// TEST INFRASTRUCTURE ONLY.
//
// extern "C" driver over the UNMODIFIED reference library (oracle/_ref/
// libsfxb_ref.so, built by oracle/Makefile from /root/reference/proj/src).
// It exposes the reference's own public API to ctypes so that
//   * tests/golden/make_golden.py can dump golden vectors produced by the
//     reference itself (keys, r stream, ciphertexts, histogram residues,
//     decrypted histograms, counters, forests);
//   * bench.py's cpu_baseline leg / `--impl reference` can time the
//     reference PaillierPlugin on the host cores;
//   * the end-to-end parity test can run the reference's vertical training
//     loop (run_training, report.cpp:132) with the CPU plugin and with the
//     GPU adapter interposed on make_paillier_plugin.
// Numbers cross this boundary as little-endian u32 limbs (the device format).
#include <gmp.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "sfxb/config.hpp"
#include "sfxb/errors.hpp"
#include "sfxb/gbdt.hpp"
#include "sfxb/he.hpp"
#include "sfxb/inference.hpp"
#include "sfxb/report.hpp"
#include "sfxb/secure_processor.hpp"

using namespace sfxb;

namespace {
thread_local std::string g_err;

mpz_class from_words(const std::uint32_t *w, std::size_t words) {
    mpz_class z;
    mpz_import(z.get_mpz_t(), words, -1, 4, 0, 0, w);
    return z;
}
void to_words(const mpz_class &z, std::uint32_t *out, std::size_t words) {
    std::memset(out, 0, words * 4);
    if (mpz_sizeinbase(z.get_mpz_t(), 2) > 32 * words && z != 0) throw Error("value wider than buffer");
    std::size_t cnt = 0;
    mpz_export(out, &cnt, -1, 4, 0, 0, z.get_mpz_t());
}

struct RefPlugin {
    std::unique_ptr<EncryptionPlugin> plugin;
    PaillierPublicKey pub;
    std::size_t nw = 0;
};

template <typename F>
int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const AuthorizationError &e) {
        g_err = e.what();
        return -2;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}
} // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

// keygen(bits, seed) (he.cpp:58-85); n in nw words, p/q in nw words (zero padded).
int ref_keygen(unsigned bits, std::uint64_t seed, std::uint32_t *n, std::uint32_t *p,
               std::uint32_t *q, std::size_t nw) {
    return guarded([&] {
        PaillierKeypair kp = keygen(bits, seed);
        to_words(kp.pub.n, n, nw);
        to_words(kp.priv.p, p, nw);
        to_words(kp.priv.q, q, nw);
    });
}

int ref_keypair_from_primes(const std::uint32_t *p, const std::uint32_t *q, std::size_t nw,
                            std::uint32_t *n_out, std::uint32_t *lambda_out, std::uint32_t *mu_out) {
    return guarded([&] {
        PaillierKeypair kp = keypair_from_primes(from_words(p, nw), from_words(q, nw));
        to_words(kp.pub.n, n_out, nw);
        to_words(kp.priv.lambda, lambda_out, nw);
        to_words(kp.priv.mu, mu_out, nw);
    });
}

std::uint64_t ref_key_id(const std::uint32_t *n, std::size_t nw) { return key_id_of(from_words(n, nw)); }

// Private key file bytes (he.cpp:263-357) for run_training's key directory.
int ref_write_private_key(unsigned bits, std::uint64_t seed, const char *path_priv,
                          const char *path_pub) {
    return guarded([&] {
        PaillierKeypair kp = keygen(bits, seed);
        std::ofstream(path_priv, std::ios::binary) << serialize_private_key(kp);
        std::ofstream(path_pub, std::ios::binary) << serialize_public_key(kp.pub);
    });
}

// HeRng(seed).unit_below(n) × count (he.cpp:19-28).
int ref_rng_draw(std::uint64_t seed, const std::uint32_t *n, std::size_t nw, std::size_t count,
                 std::uint32_t *out) {
    return guarded([&] {
        HeRng rng(seed);
        mpz_class zn = from_words(n, nw);
        for (std::size_t i = 0; i < count; ++i) to_words(rng.unit_below(zn), out + i * nw, nw);
    });
}

int ref_encrypt_with_r(const std::uint32_t *n, std::size_t nw, const std::uint32_t *m,
                       const std::uint32_t *r, std::uint32_t *out_c) {
    return guarded([&] {
        PaillierPublicKey pk;
        pk.n = from_words(n, nw);
        pk.n2 = pk.n * pk.n;
        Ciphertext c = encrypt_with_r(pk, from_words(m, nw), from_words(r, nw));
        to_words(c.value, out_c, 2 * nw);
    });
}

// compute_gradients + quantize_gradients (gbdt.cpp:69-87) + encode_fixed
// (he.cpp:125-136) for each row, as the reference's loop feeds encrypt_gh:
// q_out[2i], q_out[2i+1] = the signed fixed-point plaintexts of g_i, h_i
// (m − n when m > n/2), gh_out = the quantized doubles.  Stops at the first
// value encode_fixed rejects: returns -1 with the message, *first_bad = its index.
int ref_gradients(const double *prob, const std::uint8_t *labels, std::size_t n, unsigned scale,
                  const std::uint32_t *nwords, std::size_t nw, std::int64_t *q_out, double *gh_out,
                  std::size_t *first_bad) {
    *first_bad = 2 * n;
    return guarded([&] {
        PaillierPublicKey pk;
        pk.n = from_words(nwords, nw);
        pk.n2 = pk.n * pk.n;
        std::vector<std::uint8_t> lab(labels, labels + n);
        std::vector<double> pr(prob, prob + n);
        std::vector<GHPair> gh = compute_gradients(lab, pr);
        quantize_gradients(gh, scale);
        const mpz_class half = pk.n / 2;
        for (std::size_t i = 0; i < 2 * n; ++i) {
            const double x = (i & 1) ? gh[i / 2].h : gh[i / 2].g;
            gh_out[i] = x;
            mpz_class m;
            try {
                m = encode_fixed(pk, x, scale);
            } catch (...) {
                *first_bad = i;
                throw;
            }
            if (m > half) m -= pk.n;
            q_out[i] = mpz_get_si(m.get_mpz_t());
        }
    });
}

// make_paillier_plugin (secure_processor.cpp:754-762); p == nullptr -> public half only.
void *ref_plugin_new(const std::uint32_t *n, const std::uint32_t *p, const std::uint32_t *q,
                     std::size_t nw, std::uint64_t rng_seed, unsigned scale_bits) {
    RefPlugin *rp = nullptr;
    int rc = guarded([&] {
        auto h = std::make_unique<RefPlugin>();
        PaillierPluginConfig cfg;
        cfg.rng_seed = rng_seed;
        cfg.scale_bits = scale_bits;
        h->nw = nw;
        if (p && q) {
            PaillierKeypair kp = keypair_from_primes(from_words(p, nw), from_words(q, nw));
            h->pub = kp.pub;
            h->plugin = make_paillier_plugin(kp, cfg);
        } else {
            h->pub.n = from_words(n, nw);
            h->pub.n2 = h->pub.n * h->pub.n;
            h->pub.modulus_bits = static_cast<unsigned>(mpz_sizeinbase(h->pub.n.get_mpz_t(), 2));
            h->pub.key_id = key_id_of(h->pub.n);
            h->plugin = make_paillier_plugin(h->pub, cfg);
        }
        rp = h.release();
    });
    return rc == 0 ? rp : nullptr;
}

void ref_plugin_free(void *h) { delete static_cast<RefPlugin *>(h); }

void ref_plugin_counters(void *h, std::uint64_t out[4]) {
    const OpCounters &c = static_cast<RefPlugin *>(h)->plugin->counters();
    out[0] = c.encryptions;
    out[1] = c.ciphertext_additions;
    out[2] = c.decryptions;
    out[3] = c.bytes_transferred;
}

const char *ref_plugin_name(void *h) {
    static thread_local std::string s;
    s = static_cast<RefPlugin *>(h)->plugin->name();
    return s.c_str();
}

// encrypt_gh (secure_processor.cpp:574-585): gh = count (g,h) pairs.
int ref_encrypt_gh(void *h, const double *gh, std::size_t count, std::uint32_t *out_cts) {
    RefPlugin *rp = static_cast<RefPlugin *>(h);
    return guarded([&] {
        std::vector<GHPair> v(count);
        for (std::size_t i = 0; i < count; ++i) v[i] = GHPair{gh[2 * i], gh[2 * i + 1]};
        GhPayload out = rp->plugin->encrypt_gh(v);
        for (std::size_t i = 0; i < out.cts.size(); ++i)
            to_words(out.cts[i].value, out_cts + i * 2 * rp->nw, 2 * rp->nw);
    });
}

namespace {
GhPayload gh_from_words(const RefPlugin *rp, const std::uint32_t *cts, std::uint32_t n_samples) {
    GhPayload gh;
    gh.encrypted = true;
    gh.n_samples = n_samples;
    gh.cts.resize(2ull * n_samples);
    for (std::size_t i = 0; i < gh.cts.size(); ++i) {
        gh.cts[i].value = from_words(cts + i * 2 * rp->nw, 2 * rp->nw);
        gh.cts[i].key_id = rp->pub.key_id;
    }
    return gh;
}
} // namespace

// accumulate_rows (secure_processor.cpp:587-620).  Output layout: node-major,
// then the reference's own slot order 2(f·K+b)+{0:G,1:H}.
int ref_accumulate(void *h, const std::uint32_t *cts, std::uint32_t n_samples,
                   const std::uint16_t *bins, std::uint32_t n_features, const int *feature_ids,
                   const std::uint32_t *node_offsets, const std::uint32_t *node_ids,
                   std::uint32_t n_nodes, const std::uint32_t *rows, std::uint32_t n_bins,
                   std::uint32_t *out) {
    RefPlugin *rp = static_cast<RefPlugin *>(h);
    return guarded([&] {
        GhPayload gh = gh_from_words(rp, cts, n_samples);
        std::vector<std::vector<std::uint16_t>> b(n_features);
        for (std::uint32_t f = 0; f < n_features; ++f)
            b[f].assign(bins + std::size_t(f) * n_samples, bins + std::size_t(f + 1) * n_samples);
        std::vector<int> fids(feature_ids, feature_ids + n_features);
        std::vector<NodeRows> nodes(n_nodes);
        for (std::uint32_t i = 0; i < n_nodes; ++i) {
            nodes[i].node_id = node_ids[i];
            nodes[i].rows.assign(rows + node_offsets[i], rows + node_offsets[i + 1]);
        }
        HistogramPayload hp = rp->plugin->accumulate_rows(gh, b, fids, nodes, int(n_bins));
        std::size_t per_node = 2ull * n_features * n_bins;
        for (std::uint32_t i = 0; i < n_nodes; ++i)
            for (std::size_t s = 0; s < per_node; ++s)
                to_words(hp.nodes[i].scalar_cts[s].value, out + (i * per_node + s) * 2 * rp->nw,
                         2 * rp->nw);
    });
}

// decrypt_histogram (secure_processor.cpp:679-719) on enc_scalar slots laid out
// as ref_accumulate writes them; out = node × f × b × {g,h} doubles.
int ref_decrypt_slots(void *h, const std::uint32_t *slots, std::uint32_t n_nodes,
                      std::uint32_t n_features, std::uint32_t n_bins, double *out) {
    RefPlugin *rp = static_cast<RefPlugin *>(h);
    return guarded([&] {
        HistogramPayload hp;
        hp.layout = HistLayout::enc_scalar;
        std::size_t per_node = 2ull * n_features * n_bins;
        for (std::uint32_t i = 0; i < n_nodes; ++i) {
            NodeHistogram nh;
            nh.node_id = i;
            nh.n_bins = int(n_bins);
            for (std::uint32_t f = 0; f < n_features; ++f) nh.feature_ids.push_back(int(f));
            nh.scalar_cts.resize(per_node);
            for (std::size_t s = 0; s < per_node; ++s) {
                nh.scalar_cts[s].value = from_words(slots + (i * per_node + s) * 2 * rp->nw, 2 * rp->nw);
                nh.scalar_cts[s].key_id = rp->pub.key_id;
            }
            hp.nodes.push_back(std::move(nh));
        }
        auto res = rp->plugin->decrypt_histogram(hp);
        for (std::uint32_t i = 0; i < n_nodes; ++i)
            for (std::uint32_t f = 0; f < n_features; ++f)
                for (std::uint32_t b = 0; b < n_bins; ++b) {
                    std::size_t o = ((std::size_t(i) * n_features + f) * n_bins + b) * 2;
                    out[o] = res[i].second.feats[f][b].g;
                    out[o + 1] = res[i].second.feats[f][b].h;
                }
    });
}

// CPU baseline with all host threads: `threads` independent plugin instances
// (the plugin is stateless apart from keys and counters, secure_processor.hpp:111)
// claim work items (feature f, row range k) from a shared counter; an item is
// accumulate_rows over the frontier restricted to the range's rows for one
// feature (J × threads items, so every thread stays busy whatever J is).
// Returns the additions performed (each instance's counter) and the wall time.
int ref_accumulate_threaded(const std::uint32_t *n, std::size_t nw, const std::uint32_t *cts,
                            std::uint32_t n_samples, const std::uint16_t *bins,
                            std::uint32_t n_features, const std::uint32_t *node_offsets,
                            std::uint32_t n_nodes, const std::uint32_t *rows, std::uint32_t n_bins,
                            int threads, std::uint64_t *additions) {
    return guarded([&] {
        std::vector<std::unique_ptr<RefPlugin>> ps;
        for (int t = 0; t < threads; ++t) {
            auto rp = std::unique_ptr<RefPlugin>(
                static_cast<RefPlugin *>(ref_plugin_new(n, nullptr, nullptr, nw, 1, 40)));
            if (!rp) throw Error(g_err);
            ps.push_back(std::move(rp));
        }
        GhPayload gh = gh_from_words(ps[0].get(), cts, n_samples);
        // the frontier cut into `threads` contiguous row ranges
        const std::uint32_t chunks = static_cast<std::uint32_t>(threads);
        std::vector<std::vector<NodeRows>> part(chunks, std::vector<NodeRows>(n_nodes));
        for (std::uint32_t i = 0; i < n_nodes; ++i)
            for (std::uint32_t t = node_offsets[i]; t < node_offsets[i + 1]; ++t) {
                const std::uint32_t k = static_cast<std::uint32_t>(std::uint64_t(rows[t]) * chunks / n_samples);
                part[k][i].node_id = i;
                part[k][i].rows.push_back(rows[t]);
            }
        std::vector<std::vector<std::uint16_t>> cols(n_features);
        for (std::uint32_t f = 0; f < n_features; ++f)
            cols[f].assign(bins + std::size_t(f) * n_samples, bins + std::size_t(f + 1) * n_samples);
        std::atomic<std::uint32_t> next{0};
        const std::uint32_t items = n_features * chunks;
        std::vector<std::thread> pool;
        std::vector<std::string> errs(threads);
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    std::vector<std::vector<std::uint16_t>> b(1);
                    for (std::uint32_t it; (it = next.fetch_add(1)) < items;) {
                        const std::uint32_t f = it % n_features, k = it / n_features;
                        b[0] = cols[f];
                        ps[t]->plugin->accumulate_rows(gh, b, {int(f)}, part[k], int(n_bins));
                    }
                } catch (const std::exception &e) {
                    errs[t] = e.what();
                }
            });
        for (auto &th : pool) th.join();
        for (auto &e : errs)
            if (!e.empty()) throw Error(e);
        std::uint64_t adds = 0;
        for (auto &p : ps) adds += p->plugin->counters().ciphertext_additions;
        *additions = adds;
    });
}

// Reference encrypt_gh (secure_processor.cpp:574-585) on all host threads:
// one plugin per thread (rng seed t + 1), `pairs` (g, h) pairs each.
// Returns the encryptions performed and the wall seconds.
int ref_encrypt_threaded(const std::uint32_t *n, std::size_t nw, std::uint32_t pairs, int threads,
                         std::uint64_t *encryptions, double *seconds) {
    return guarded([&] {
        std::vector<std::unique_ptr<RefPlugin>> ps;
        for (int t = 0; t < threads; ++t) {
            auto rp = std::unique_ptr<RefPlugin>(
                static_cast<RefPlugin *>(ref_plugin_new(n, nullptr, nullptr, nw, 1 + t, 40)));
            if (!rp) throw Error(g_err);
            ps.push_back(std::move(rp));
        }
        std::vector<GHPair> gh(pairs);
        for (std::uint32_t i = 0; i < pairs; ++i)
            gh[i] = GHPair{(i % 2 ? -0.37 : 0.41) + 1e-3 * (i % 97), 0.2 - 1e-4 * (i % 89)};
        std::vector<std::thread> pool;
        const auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < threads; ++t) pool.emplace_back([&, t] { (void)ps[t]->plugin->encrypt_gh(gh); });
        for (auto &th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::uint64_t e = 0;
        for (auto &p : ps) e += p->plugin->counters().encryptions;
        *encryptions = e;
    });
}

// Reference decrypt_histogram (secure_processor.cpp:679-719) on all host
// threads: the `count` ciphertexts (2·nw limbs each) split into one slice per
// thread, each slice one node × one feature × slice/2 bins of the key
// holder's plugin.  Returns the decryptions performed and the wall seconds.
int ref_decrypt_threaded(const std::uint32_t *p, const std::uint32_t *q, std::size_t nw,
                         const std::uint32_t *cts, std::uint32_t count, int threads,
                         std::uint64_t *decryptions, double *seconds) {
    return guarded([&] {
        std::vector<std::unique_ptr<RefPlugin>> ps;
        std::vector<HistogramPayload> hp(threads);
        const std::uint32_t per = (count / threads) & ~1u;
        for (int t = 0; t < threads; ++t) {
            auto rp = std::unique_ptr<RefPlugin>(static_cast<RefPlugin *>(ref_plugin_new(nullptr, p, q, nw, 1, 40)));
            if (!rp) throw Error(g_err);
            hp[t].layout = HistLayout::enc_scalar;
            NodeHistogram nh;
            nh.node_id = 0;
            nh.n_bins = int(per / 2);
            nh.feature_ids = {0};
            for (std::uint32_t i = 0; i < per; ++i) {
                const std::uint32_t *w = cts + (std::size_t(t) * per + i) * 2 * nw;
                nh.scalar_cts.push_back(Ciphertext{from_words(w, 2 * nw), rp->pub.key_id});
            }
            hp[t].nodes.push_back(std::move(nh));
            ps.push_back(std::move(rp));
        }
        std::vector<std::thread> pool;
        std::vector<std::string> errs(threads);
        const auto t0 = std::chrono::steady_clock::now();
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&, t] {
                try {
                    (void)ps[t]->plugin->decrypt_histogram(hp[t]);
                } catch (const std::exception &e) {
                    errs[t] = e.what();
                }
            });
        for (auto &th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (auto &e : errs)
            if (!e.empty()) throw Error(e);
        std::uint64_t d = 0;
        for (auto &pp : ps) d += pp->plugin->counters().decryptions;
        *decryptions = d;
    });
}

// run_training (report.cpp:132) on an INI config text; the key directory is
// taken from SFXB_KEY_DIR or the config.  Outputs the serialized forest, the
// concatenated partial models, report counters and an FNV-1a digest of every
// transcript entry's exact bytes (plus the byte total).
int ref_train(const char *ini_text, char *forest_out, std::size_t forest_cap, char *partials_out,
              std::size_t partials_cap, std::uint64_t counters[4], std::uint64_t *transcript_fnv,
              std::uint64_t *transcript_bytes, double phases[6]) {
    return guarded([&] {
        RunConfig cfg = parse_run_config(ini_text);
        TrainOutput out = run_training(cfg);
        std::string f = serialize_forest(out.forest);
        if (f.size() + 1 > forest_cap) throw Error("forest buffer too small");
        std::memcpy(forest_out, f.c_str(), f.size() + 1);
        std::string parts;
        for (const PartialModel &pm : out.partials) parts += serialize_partial(pm) + "\n---\n";
        if (parts.size() + 1 > partials_cap) throw Error("partials buffer too small");
        std::memcpy(partials_out, parts.c_str(), parts.size() + 1);
        counters[0] = out.report.counters.encryptions;
        counters[1] = out.report.counters.ciphertext_additions;
        counters[2] = out.report.counters.decryptions;
        counters[3] = out.report.counters.bytes_transferred;
        std::uint64_t hsh = 14695981039346656037ULL, total = 0;
        for (const TranscriptEntry &e : out.transcript.entries) {
            for (unsigned char c : e.bytes) {
                hsh ^= c;
                hsh *= 1099511628211ULL;
            }
            total += e.bytes.size();
        }
        *transcript_fnv = hsh;
        *transcript_bytes = total;
        const PhaseTimes &p = out.report.phases;
        double ph[6] = {p.cuts, p.gradient, p.encrypt, p.aggregate, p.decrypt, p.split};
        std::memcpy(phases, ph, sizeof ph);
    });
}

} // extern "C"
