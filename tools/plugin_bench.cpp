// Per-tree timing of the plugin calls exactly as the reference's vertical
// loop makes them (federation.cpp:456-534): encrypt_gh once per tree at the
// active party, then per level accumulate_rows at every party and
// decrypt_histogram of every party's histograms at the active party.
// Built against the unmodified reference library (oracle/Makefile
// `plugin-bench`); run with LD_PRELOAD=paper_2504_03909_b200/lib/
// libsfxb_cuda_plugin.so the calls go to the GPU adapter — this is the
// end-to-end cost a reference user sees, host marshalling of the reference's
// mpz payloads included.  Without LD_PRELOAD it times the CPU plugin.
//
//   plugin_bench [rows=1000000] [features_per_party=14] [bins=256] [depth=6] [bits=2048] [parties=2] [trees=1]
// (with trees > 1 the last tree is reported; every tree encrypts afresh)
// tree_wall_s: the reported tree from encrypt_gh to its last decrypt,
// including the untimed host copies of the gradient payload to the passive
// parties (the Bus's share of the reference loop) — the GPU adapter's
// offline phase for the next encrypt_gh runs in the background meanwhile.
//
// Prints one JSON object.  Synthetic inputs: gh on the 2^-40 grid
// (g in (-1, 1), h in [0, 0.25]), uniform bins, a full binary tree whose
// children split their parent's rows at random, listed consecutively in
// parent order with heap node ids (2k+1, 2k+2) as the reference does.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "sfxb/he.hpp"
#include "sfxb/secure_processor.hpp"

using namespace sfxb;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

int main(int argc, char **argv) {
    const uint32_t rows = argc > 1 ? (uint32_t)std::atol(argv[1]) : 1000000u;
    const int J = argc > 2 ? std::atoi(argv[2]) : 14;
    const int K = argc > 3 ? std::atoi(argv[3]) : 256;
    const int D = argc > 4 ? std::atoi(argv[4]) : 6;
    const unsigned bits = argc > 5 ? (unsigned)std::atoi(argv[5]) : 2048u;
    const int parties = argc > 6 ? std::atoi(argv[6]) : 2;
    const int trees = argc > 7 ? std::max(1, std::atoi(argv[7])) : 1;

    const PaillierKeypair kp = keygen(bits, 7);
    std::vector<std::unique_ptr<EncryptionPlugin>> plug;
    for (int pi = 0; pi < parties; ++pi) {
        PaillierPluginConfig cfg;
        cfg.scale_bits = 40;
        cfg.rng_seed = 1ull ^ (0x9E3779B97F4A7C15ull * (uint64_t)(pi + 1)); // federation.cpp:82
        plug.push_back(pi == 0 ? make_paillier_plugin(kp, cfg) : make_paillier_plugin(kp.pub, cfg));
    }

    std::mt19937_64 rng(42);
    std::vector<GHPair> gh(rows);
    for (auto &x : gh) {
        x.g = std::ldexp((double)((int64_t)(rng() % (2ull << 40)) - (int64_t)(1ull << 40)), -40);
        x.h = std::ldexp((double)(rng() % (1ull << 38)), -40);
    }
    std::vector<std::vector<std::vector<uint16_t>>> bins(parties, std::vector<std::vector<uint16_t>>(J));
    for (auto &pb : bins)
        for (auto &col : pb) {
            col.resize(rows);
            for (auto &b : col) b = (uint16_t)(rng() % (uint64_t)K);
        }
    std::vector<std::vector<int>> fids(parties);
    for (int pi = 0; pi < parties; ++pi)
        for (int f = 0; f < J; ++f) fids[pi].push_back(pi + f * parties); // alternating split
    // frontiers of a full binary tree
    std::vector<std::vector<NodeRows>> levels(D);
    levels[0].resize(1);
    levels[0][0].node_id = 0;
    for (uint32_t r = 0; r < rows; ++r) levels[0][0].rows.push_back(r);
    for (int d = 1; d < D; ++d)
        for (const NodeRows &p : levels[d - 1]) {
            NodeRows a, b;
            a.node_id = 2 * p.node_id + 1;
            b.node_id = 2 * p.node_id + 2;
            const uint64_t cut = rng() % (1ull << 20);
            for (uint32_t r : p.rows) ((rng() % (1ull << 21)) < (1ull << 20) + cut / 4 ? a : b).rows.push_back(r);
            levels[d].push_back(std::move(a));
            levels[d].push_back(std::move(b));
        }

    // warm-up on a small slice (context creation, kernel loading)
    {
        std::vector<GHPair> small(gh.begin(), gh.begin() + std::min<uint32_t>(rows, 4096));
        GhPayload w = plug[0]->encrypt_gh(small);
        (void)w;
    }

    double enc_s = 0, acc = 0, dec = 0, tree_wall = 0;
    std::string la, ld;
    uint64_t adds = 0, decs = 0;
    for (int tree = 0; tree < trees; ++tree) {
    adds = decs = 0;
    const auto t0 = Clock::now();
    GhPayload enc = plug[0]->encrypt_gh(gh); // active party, once per tree
    const auto t1 = Clock::now();
    // the passive parties hold a copy (what the Bus delivers; not timed)
    std::vector<GhPayload> held(parties, enc);
    std::vector<double> t_acc(D, 0.0), t_dec(D, 0.0);
    for (int d = 0; d < D; ++d) {
        std::vector<HistogramPayload> hist(parties);
        for (int pi = 0; pi < parties; ++pi) {
            const uint64_t a0 = plug[pi]->counters().ciphertext_additions;
            const auto s = Clock::now();
            hist[pi] = plug[pi]->accumulate_rows(held[pi], bins[pi], fids[pi], levels[d], K);
            t_acc[d] += secs(s, Clock::now());
            adds += plug[pi]->counters().ciphertext_additions - a0;
        }
        for (int pi = 0; pi < parties; ++pi) {
            const uint64_t d0 = plug[0]->counters().decryptions;
            const auto s = Clock::now();
            auto res = plug[0]->decrypt_histogram(hist[pi]);
            t_dec[d] += secs(s, Clock::now());
            decs += plug[0]->counters().decryptions - d0;
            (void)res;
        }
    }
    acc = dec = 0;
    la = "[";
    ld = "[";
    for (int d = 0; d < D; ++d) {
        acc += t_acc[d];
        dec += t_dec[d];
        la += (d ? "," : "") + std::to_string(t_acc[d]);
        ld += (d ? "," : "") + std::to_string(t_dec[d]);
    }
    la += "]";
    ld += "]";
    enc_s = secs(t0, t1);
    tree_wall = secs(t0, Clock::now());
    }
    std::printf("{\"plugin\": \"%s\", \"rows\": %u, \"features_per_party\": %d, \"parties\": %d, \"bins\": %d, "
                "\"depth\": %d, \"bits\": %u, \"encrypt_gh_s\": %.6f, \"encryptions_per_s\": %.1f, "
                "\"accumulate_rows_s\": %.6f, \"accumulate_rows_s_per_level\": %s, \"ciphertext_additions\": %llu, "
                "\"decrypt_histogram_s\": %.6f, \"decrypt_histogram_s_per_level\": %s, \"decryptions\": %llu, "
                "\"plugin_s_per_tree\": %.6f, \"tree_wall_s\": %.6f, \"trees\": %d}\n",
                plug[0]->name().c_str(), rows, J, parties, K, D, bits, enc_s, 2.0 * rows / enc_s, acc, la.c_str(),
                (unsigned long long)adds, dec, ld.c_str(), (unsigned long long)decs, enc_s + acc + dec, tree_wall, trees);
    return 0;
}
