// TEST INFRASTRUCTURE ONLY.
//
// Edge-case scenarios of the scalar plugin path, driven through the
// reference's public API (EncryptionPlugin from make_paillier_plugin,
// secure_processor.hpp:112-158).  Run as is, the plugin is the reference's
// PaillierPlugin; run with LD_PRELOAD=libsfxb_cuda_plugin.so it is the GPU
// adapter.  tests/test_gpu_edges.py compares the two outputs.  One JSON
// object per scenario on stdout: output slots (hex value, key id) or the
// exception (type, message), plus the plugin's counters.
//
// Scenarios follow the reference's semantics in secure_processor.cpp:587-620
// (accumulate_rows), :724-732 (fold_into), :679-738 (decrypt_histogram) and
// he.cpp:105-121 (decrypt, add_ciphertexts).
#include <gmp.h>

#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "sfxb/errors.hpp"
#include "sfxb/he.hpp"
#include "sfxb/secure_processor.hpp"

using namespace sfxb;

namespace {

std::string hex(const mpz_class &v) {
    if (v < 0) return "-" + mpz_class(-v).get_str(16);
    return v.get_str(16);
}

struct Fixture {
    PaillierKeypair kp;
    HeRng rng{7};
    std::mt19937_64 mt{12345};
    explicit Fixture(unsigned bits) : kp(keygen(bits, 0xC0FFEE)) {}

    Ciphertext enc(std::int64_t q) {
        mpz_class m(static_cast<long>(q));
        if (m < 0) m += kp.pub.n;
        return encrypt(kp.pub, m, rng);
    }
    // M rows of encrypted (g, h) with small random integers
    GhPayload gh(std::uint32_t M) {
        GhPayload g;
        g.encrypted = true;
        g.n_samples = M;
        for (std::uint32_t i = 0; i < 2 * M; ++i) g.cts.push_back(enc((std::int64_t)(mt() % 2001) - 1000));
        return g;
    }
    std::vector<std::vector<std::uint16_t>> bins(std::uint32_t J, std::uint32_t M, int K) {
        std::vector<std::vector<std::uint16_t>> b(J, std::vector<std::uint16_t>(M));
        for (auto &col : b)
            for (auto &x : col) x = (std::uint16_t)(mt() % K);
        return b;
    }
};

void print_counters(const EncryptionPlugin &p) {
    const OpCounters &c = p.counters();
    std::printf("\"counters\": [%llu, %llu, %llu]", (unsigned long long)c.encryptions,
                (unsigned long long)c.ciphertext_additions, (unsigned long long)c.decryptions);
}

void print_hist(const HistogramPayload &hp) {
    std::printf("\"slots\": [");
    bool first = true;
    for (const NodeHistogram &nd : hp.nodes)
        for (const Ciphertext &c : nd.scalar_cts) {
            std::printf("%s[\"%s\", \"%016llx\"]", first ? "" : ", ", hex(c.value).c_str(),
                        (unsigned long long)c.key_id);
            first = false;
        }
    std::printf("]");
}

void print_dec(const std::vector<std::pair<std::uint32_t, Histogram>> &res) {
    std::printf("\"values\": [");
    bool first = true;
    for (const auto &[id, h] : res)
        for (const auto &f : h.feats)
            for (const GHPair &b : f) {
                std::printf("%s\"%a\", \"%a\"", first ? "" : ", ", b.g, b.h);
                first = false;
            }
    std::printf("]");
}

// run `body` as scenario `name`: prints slots/values or the exception
void scenario(const char *name, EncryptionPlugin &p, const std::function<void()> &body) {
    std::printf("{\"name\": \"%s\", ", name);
    try {
        body();
        std::printf("\"ok\": true, ");
    } catch (const AuthorizationError &e) {
        std::printf("\"ok\": false, \"type\": \"AuthorizationError\", \"msg\": \"%s\", ", e.what());
    } catch (const Error &e) {
        std::printf("\"ok\": false, \"type\": \"Error\", \"msg\": \"%s\", ", e.what());
    }
    print_counters(p);
    std::printf("}\n");
    std::fflush(stdout);
}

std::vector<NodeRows> two_nodes(std::uint32_t M) {
    // rows 0..M-1 minus a few (out of the frontier), split in two ascending nodes
    std::vector<NodeRows> nodes(2);
    nodes[0].node_id = 1;
    nodes[1].node_id = 2;
    for (std::uint32_t r = 0; r < M; ++r) {
        if (r % 7 == 3) continue;
        nodes[r % 3 == 0 ? 1 : 0].rows.push_back(r);
    }
    return nodes;
}

} // namespace

int main(int argc, char **argv) {
    const unsigned bits = argc > 1 ? (unsigned)std::atoi(argv[1]) : 512;
    Fixture fx(bits);
    PaillierPluginConfig cfg;
    const std::uint32_t M = 60, J = 3;
    const int K = 8;
    const std::vector<int> fids = {0, 1, 2};

    // --- accumulate_rows at the passive party (public key only) and the key holder
    for (int holder = 0; holder < 2; ++holder) {
        auto plugin = holder ? make_paillier_plugin(fx.kp, cfg) : make_paillier_plugin(fx.kp.pub, cfg);
        EncryptionPlugin &p = *plugin;
        const std::string tag = holder ? "holder_" : "passive_";
        GhPayload gh = fx.gh(M);
        auto bins = fx.bins(J, M, K);
        auto nodes = two_nodes(M);
        HistogramPayload out;
        auto run = [&](const char *name) {
            scenario((tag + name).c_str(), p, [&] {
                out = p.accumulate_rows(gh, bins, fids, nodes, K);
                print_hist(out);
                std::printf(", ");
            });
        };
        run("plain");
        // in-place rewrite of one ciphertext's limbs (same mpz buffer, same
        // size): the next call must see it (the resident copy is keyed on
        // content, never on a sample)
        {
            Ciphertext fresh = fx.enc(4242);
            while (mpz_size(fresh.value.get_mpz_t()) != mpz_size(gh.cts[37].value.get_mpz_t())) fresh = fx.enc(4242);
            const void *before = mpz_limbs_read(gh.cts[37].value.get_mpz_t());
            mpz_set(gh.cts[37].value.get_mpz_t(), fresh.value.get_mpz_t());
            if (mpz_limbs_read(gh.cts[37].value.get_mpz_t()) != before) std::fprintf(stderr, "buffer moved\n");
            run("mutated_in_place");
            mpz_set_ui(gh.cts[2 * 40].value.get_mpz_t(), 1); // a trivial zero appears
            run("mutated_trivial");
        }
        // foreign key on rows outside the frontier: never folded, no error
        gh.cts[2 * 3].key_id ^= 0xdeadbeef;
        gh.cts[2 * 10 + 1].key_id ^= 0xdeadbeef;
        run("foreign_key_outside_frontier");
        // trivial zero with a foreign key: skipped by fold_into
        gh.cts[2 * 5] = Ciphertext{mpz_class(1), 99};
        run("trivial_foreign_key");
        // a foreign-key row alone in every slot it lands in: copied with its key
        {
            auto b2 = bins;
            const std::uint32_t r = 1; // node 1 (id 1)
            for (std::uint32_t f = 0; f < J; ++f) {
                for (std::uint32_t row = 0; row < M; ++row)
                    if (b2[f][row] == K - 1) b2[f][row] = K - 2;
                b2[f][r] = K - 1;
            }
            std::swap(bins, b2);
            gh.cts[2 * r].key_id ^= 0x1234;
            run("foreign_key_alone_in_slot");
            // values outside [0, n²) alone in their slots: copied unchanged
            gh.cts[2 * r].key_id ^= 0x1234;
            gh.cts[2 * r].value += fx.kp.pub.n2;
            gh.cts[2 * r + 1].value = -gh.cts[2 * r + 1].value;
            run("off_range_alone_in_slot");
            std::swap(bins, b2);
        }
        // values outside [0, n²) in shared slots: a·b tdiv n², sign included
        gh.cts[2 * 7].value += 3 * fx.kp.pub.n2;
        gh.cts[2 * 8 + 1].value = -gh.cts[2 * 8 + 1].value;
        gh.cts[2 * 11 + 1].value <<= 2 * bits + 70; // wider than a ciphertext
        run("off_range_shared");
        // a zero residue in a shared slot (products become 0)
        gh.cts[2 * 13].value = 0;
        run("zero_shared");
        // next level: children of node 1 (sibling subtraction at the GPU)
        {
            auto parent = nodes;
            std::vector<NodeRows> kids(4);
            for (int c = 0; c < 4; ++c) kids[c].node_id = 3 + c;
            for (int pi = 0; pi < 2; ++pi)
                for (std::uint32_t r : parent[pi].rows) kids[2 * pi + ((r / 2) % 3 == 0 ? 1 : 0)].rows.push_back(r);
            nodes = kids;
            run("next_level_children");
            nodes = parent;
        }
        // a foreign key in a shared slot: fails at the reference's fold
        gh.cts[2 * 14 + 1].key_id ^= 0xfeed;
        run("foreign_key_shared");
        gh.cts[2 * 14 + 1].key_id ^= 0xfeed;
        // a bad bin index after some folds
        {
            auto b2 = bins;
            b2[1][nodes[1].rows[2]] = (std::uint16_t)K;
            std::swap(bins, b2);
            run("bin_out_of_range");
            std::swap(bins, b2);
        }
        // c · c⁻¹ inside one slot followed by another entry (documented
        // counter deviation: the reference's third fold is an uncounted assign)
        {
            GhPayload g2 = fx.gh(3);
            mpz_class inv;
            mpz_invert(inv.get_mpz_t(), g2.cts[0].value.get_mpz_t(), fx.kp.pub.n2.get_mpz_t());
            g2.cts[2].value = inv;
            std::vector<std::vector<std::uint16_t>> b3(1, std::vector<std::uint16_t>(3, 0));
            std::vector<NodeRows> n3(1);
            n3[0].node_id = 0;
            n3[0].rows = {0, 1, 2};
            scenario((tag + "inverse_pair_in_slot").c_str(), p, [&] {
                print_hist(p.accumulate_rows(g2, b3, {0}, n3, 1));
                std::printf(", ");
            });
        }
    }

    // --- decrypt_histogram error order (key holder)
    {
        auto plugin = make_paillier_plugin(fx.kp, cfg);
        EncryptionPlugin &p = *plugin;
        GhPayload gh = fx.gh(M);
        auto bins = fx.bins(J, M, K);
        auto nodes = two_nodes(M);
        HistogramPayload hp = p.accumulate_rows(gh, bins, fids, nodes, K);
        scenario("decrypt_ok", p, [&] {
            print_dec(p.decrypt_histogram(hp));
            std::printf(", ");
        });
        auto with = [&](const char *name, const std::function<void(HistogramPayload &)> &edit) {
            HistogramPayload h2 = hp;
            edit(h2);
            scenario(name, p, [&] {
                print_dec(p.decrypt_histogram(h2));
                std::printf(", ");
            });
        };
        auto nth_nontrivial = [](HistogramPayload &h, size_t k) -> Ciphertext & {
            for (NodeHistogram &nd : h.nodes)
                for (Ciphertext &c : nd.scalar_cts)
                    if (!(c.value == 1) && k-- == 0) return c;
            throw Error("fixture: not enough slots");
        };
        with("decrypt_key_mismatch", [&](HistogramPayload &h) { nth_nontrivial(h, 20).key_id ^= 1; });
        with("decrypt_out_of_range", [&](HistogramPayload &h) { nth_nontrivial(h, 9).value += fx.kp.pub.n2; });
        with("decrypt_not_coprime", [&](HistogramPayload &h) { nth_nontrivial(h, 15).value = fx.kp.priv.p * 3; });
        with("decrypt_not_coprime_before_range", [&](HistogramPayload &h) {
            nth_nontrivial(h, 5).value = fx.kp.priv.q;
            nth_nontrivial(h, 30).value = 0;
        });
        with("decrypt_range_before_not_coprime", [&](HistogramPayload &h) {
            nth_nontrivial(h, 31).value = fx.kp.priv.q;
            nth_nontrivial(h, 6).value = -7;
        });
        auto pub = make_paillier_plugin(fx.kp.pub, cfg);
        scenario("decrypt_without_key", *pub, [&] { pub->decrypt_histogram(hp); });
    }
    return 0;
}
