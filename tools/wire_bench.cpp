// Parity and timing of the processor-buffer wire codec: sfxb::serialize_buffer
// / sfxb::parse_buffer as this process binds them (with LD_PRELOAD of
// libsfxb_cuda_plugin.so: the parallel codec, host/wire_parallel.cpp) against
// the reference library's own definitions (secure_processor.cpp:119-375,
// looked up in libsfxb_ref.so directly).
//
//   wire_bench [samples=200000] [nodes=8] [feats=14] [bins=256] [bits=2048] [seed=1] [malformed=1]
//
// Payloads: gh_pairs_enc with 2·samples ciphertexts and a scalar
// histogram_enc of `nodes` nodes; values uniform below n² (n of `bits`)
// with random leading-zero lengths, plus 0 and the trivial zero 1.
// Checks: identical bytes, identical parsed payloads (values and key ids),
// and for truncated / extended buffers the same exception message.  Prints
// one JSON object; exit 1 on any mismatch.
#include <dlfcn.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "sfxb/errors.hpp"
#include "sfxb/secure_processor.hpp"

using namespace sfxb;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); }

using SerializeFn = std::string (*)(const ProcessorBuffer &);
using ParseFn = ProcessorBuffer (*)(const std::string &);

static void random_ct(Ciphertext &c, std::mt19937_64 &rng, unsigned bits2, uint64_t key_id) {
    const unsigned kind = rng() % 64;
    if (kind == 0) {
        c.value = 0;
    } else if (kind == 1) {
        c.value = 1;
    } else {
        // uniform limbs below 2^(bits2 - shift): every byte length occurs
        const unsigned shift = kind < 8 ? (unsigned)(rng() % 72) : 0;
        const unsigned b = bits2 - shift;
        const size_t nl = (b + 63) / 64;
        mpz_t z;
        mpz_init(z);
        mp_limb_t *l = mpz_limbs_write(z, (mp_size_t)nl);
        for (size_t i = 0; i < nl; ++i) l[i] = rng();
        if (b % 64) l[nl - 1] &= (~0ull) >> (64 - b % 64);
        mpz_limbs_finish(z, (mp_size_t)nl);
        c.value = mpz_class(z);
        mpz_clear(z);
    }
    c.key_id = key_id;
}

static void le32w(char *p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = (char)((v >> (8 * i)) & 0xFF);
}
static uint32_t rd32r(const char *p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= (uint32_t)(uint8_t)p[i] << (8 * i);
    return v;
}

static bool same_cts(const std::vector<Ciphertext> &a, const std::vector<Ciphertext> &b) {
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a[i].value != b[i].value || a[i].key_id != b[i].key_id) return false;
    return true;
}

static bool same_packed(const PackedVector &a, const PackedVector &b) {
    return a.logical_length == b.logical_length && a.addend_count == b.addend_count && a.slot_bits == b.slot_bits &&
           a.guard_bits == b.guard_bits && a.scale_bits == b.scale_bits && same_cts(a.cts, b.cts);
}

static bool same(const ProcessorBuffer &x, const ProcessorBuffer &y) {
    if (x.version != y.version || x.kind != y.kind || x.payload.index() != y.payload.index()) return false;
    for (int i = 0; i < 3; ++i)
        if (x.header[i] != y.header[i]) return false;
    if (const auto *a = std::get_if<GhPayload>(&x.payload)) {
        const auto &b = std::get<GhPayload>(y.payload);
        return a->encrypted == b.encrypted && a->n_samples == b.n_samples && a->plain.size() == b.plain.size() &&
               same_cts(a->cts, b.cts);
    }
    if (const auto *a = std::get_if<HistogramPayload>(&x.payload)) {
        const auto &b = std::get<HistogramPayload>(y.payload);
        if (a->layout != b.layout || a->nodes.size() != b.nodes.size()) return false;
        for (size_t i = 0; i < a->nodes.size(); ++i) {
            const NodeHistogram &p = a->nodes[i], &q = b.nodes[i];
            if (p.node_id != q.node_id || p.n_bins != q.n_bins || p.feature_ids != q.feature_ids ||
                !same_cts(p.scalar_cts, q.scalar_cts) || !p.plain.feature_ids.empty() ||
                !q.plain.feature_ids.empty() || !same_packed(p.packed_g, q.packed_g) ||
                !same_packed(p.packed_h, q.packed_h))
                return false;
        }
        return true;
    }
    return false;
}

// exception type and message (the message carries the byte offset), or the
// parsed payload's identity when the input happens to be well-formed
static std::string error_of(ParseFn f, const std::string &s, const ProcessorBuffer **parsed = nullptr) {
    try {
        static thread_local ProcessorBuffer keep;
        keep = f(s);
        if (parsed) *parsed = &keep;
    } catch (const ParseError &e) {
        return std::string("ParseError: ") + e.what();
    } catch (const Error &e) {
        return std::string("Error: ") + e.what();
    } catch (const std::exception &e) {
        return std::string("std::exception: ") + e.what();
    }
    return "<no error>";
}

int main(int argc, char **argv) {
    const uint32_t samples = argc > 1 ? (uint32_t)std::atol(argv[1]) : 200000u;
    const uint32_t nodes = argc > 2 ? (uint32_t)std::atol(argv[2]) : 8u;
    const uint32_t feats = argc > 3 ? (uint32_t)std::atol(argv[3]) : 14u;
    const uint32_t bins = argc > 4 ? (uint32_t)std::atol(argv[4]) : 256u;
    const unsigned bits = argc > 5 ? (unsigned)std::atoi(argv[5]) : 2048u;
    const uint64_t seed = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 1;
    const bool malformed = argc > 7 ? std::atoi(argv[7]) != 0 : true;

    void *ref = dlopen("libsfxb_ref.so", RTLD_NOW | RTLD_NOLOAD);
    if (!ref) {
        std::fprintf(stderr, "libsfxb_ref.so not loaded\n");
        return 2;
    }
    auto ref_ser = reinterpret_cast<SerializeFn>(
        dlsym(ref, "_ZN4sfxb16serialize_bufferB5cxx11ERKNS_15ProcessorBufferE"));
    auto ref_par = reinterpret_cast<ParseFn>(
        dlsym(ref, "_ZN4sfxb12parse_bufferERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEE"));
    SerializeFn our_ser = &serialize_buffer;
    ParseFn our_par = &parse_buffer;
    const bool interposed = (void *)our_ser != (void *)ref_ser && (void *)our_par != (void *)ref_par;

    std::mt19937_64 rng(seed);
    const uint64_t kid = 0x5eed0000ull + seed; // serialized buffers drop key ids; parsed ones carry 0
    ProcessorBuffer gh;
    gh.kind = BufferKind::gh_pairs_enc;
    gh.header[0] = samples;
    {
        GhPayload p;
        p.encrypted = true;
        p.n_samples = samples;
        p.cts.resize(2ull * samples);
        for (Ciphertext &c : p.cts) random_ct(c, rng, 2 * bits, kid);
        gh.payload = std::move(p);
    }
    ProcessorBuffer hist;
    hist.kind = BufferKind::histogram_enc;
    hist.header[0] = feats;
    hist.header[1] = bins;
    hist.header[2] = nodes;
    {
        HistogramPayload hp;
        hp.layout = HistLayout::enc_scalar;
        for (uint32_t k = 0; k < nodes; ++k) {
            NodeHistogram nd;
            nd.node_id = 2 * k + 1;
            nd.n_bins = (int)bins;
            for (uint32_t f = 0; f < feats; ++f) nd.feature_ids.push_back((int)(2 * f + (k & 1)));
            nd.scalar_cts.resize(2ull * feats * bins);
            for (Ciphertext &c : nd.scalar_cts) random_ct(c, rng, 2 * bits, kid);
            hp.nodes.push_back(std::move(nd));
        }
        hist.payload = std::move(hp);
    }
    // packed layouts (horizontal mode's histogram_enc / agg_result_enc)
    auto packed = [&](BufferKind kind) {
        ProcessorBuffer b;
        b.kind = kind;
        b.header[0] = feats;
        b.header[1] = bins;
        b.header[2] = nodes;
        HistogramPayload hp;
        hp.layout = HistLayout::enc_packed;
        for (uint32_t k = 0; k < nodes; ++k) {
            NodeHistogram nd;
            nd.node_id = k;
            nd.n_bins = (int)bins;
            for (uint32_t f = 0; f < feats; ++f) nd.feature_ids.push_back((int)f);
            for (PackedVector *v : {&nd.packed_g, &nd.packed_h}) {
                v->logical_length = feats * bins;
                v->addend_count = 1 + (uint32_t)(rng() % 5);
                v->slot_bits = 128;
                v->guard_bits = 10;
                v->scale_bits = 40;
                v->cts.resize((feats * bins + 14) / 15);
                for (Ciphertext &c : v->cts) random_ct(c, rng, 2 * bits, kid);
            }
            hp.nodes.push_back(std::move(nd));
        }
        b.payload = std::move(hp);
        return b;
    };
    ProcessorBuffer hist_packed = packed(BufferKind::histogram_enc);
    ProcessorBuffer agg_packed = packed(BufferKind::agg_result_enc);
    ProcessorBuffer agg_scalar = hist;
    agg_scalar.kind = BufferKind::agg_result_enc;
    // small buffers (a handful of ciphertexts)
    ProcessorBuffer gh_small = gh;
    {
        GhPayload p = std::get<GhPayload>(gh.payload);
        p.n_samples = 3;
        p.cts.resize(6);
        gh_small.header[0] = 3;
        gh_small.payload = std::move(p);
    }

    struct Case {
        const char *name;
        const ProcessorBuffer *b;
        bool timed;
    };
    const Case cases[] = {{"gh_pairs_enc", &gh, true},         {"histogram_enc", &hist, true},
                          {"agg_result_enc", &agg_scalar, false}, {"histogram_enc_packed", &hist_packed, false},
                          {"agg_result_enc_packed", &agg_packed, false}, {"gh_pairs_enc_small", &gh_small, false}};
    bool ok = true;
    std::string report;
    char line[768];
    for (const Case &cs : cases) {
        const ProcessorBuffer &b = *cs.b;
        auto t0 = Clock::now();
        const std::string rb = ref_ser(b);
        auto t1 = Clock::now();
        const std::string ob = our_ser(b);
        auto t2 = Clock::now();
        const ProcessorBuffer rp = ref_par(rb);
        auto t3 = Clock::now();
        const ProcessorBuffer op = our_par(ob);
        auto t4 = Clock::now();
        const bool bytes_eq = rb == ob, parse_eq = same(rp, op);
        // malformed inputs: cuts (inside the header, the layout byte, the
        // first and last entries, random points), one trailing byte, header
        // bytes rewritten (magic, version, kind, layout, counts), entry
        // lengths rewritten (past the end, shorter), random byte flips
        std::vector<std::string> bad;
        if (malformed) {
            for (size_t cut : {size_t(0), size_t(3), size_t(4), size_t(5), size_t(6), size_t(17), size_t(18),
                               size_t(19), size_t(22), size_t(23), rb.size() / 2, rb.size() - 1})
                if (cut < rb.size()) bad.push_back(rb.substr(0, cut));
            for (int i = 0; i < 6; ++i) bad.push_back(rb.substr(0, rng() % rb.size()));
            bad.push_back(rb + '\0');
            bad.push_back(rb + "SFXB");
            auto edit = [&](size_t at, uint8_t v) {
                std::string t = rb;
                if (at < t.size()) t[at] = (char)v;
                bad.push_back(t);
            };
            edit(0, 'X');
            edit(4, 2);
            edit(5, 0);
            edit(5, 9);
            edit(18, 2);               // layout byte of histograms (first entry length byte of gh)
            edit(6, 0xff);             // header[0] low byte
            edit(9, 0x7f);             // header[0] high byte
            edit(10, 0xff);            // header[1]
            edit(14, 0xff);            // header[2]
            edit(17, 0x40);            // header[2] high byte
            edit(rb.size() - 5, 0xff); // inside the last entry
            for (int i = 0; i < 6; ++i) {
                std::string t = rb;
                const size_t at = 18 + rng() % (t.size() - 18);
                t[at] = (char)(t[at] ^ (1u << (rng() % 8)));
                bad.push_back(t);
            }
            // an entry length rewritten: past the end, and one byte short
            const size_t first = (b.kind == BufferKind::gh_pairs_enc) ? 18 : 0;
            if (first) {
                std::string t = rb;
                le32w(&t[first], 0xfffffff0u);
                bad.push_back(t);
                t = rb;
                le32w(&t[first], rd32r(&rb[first]) - 1);
                bad.push_back(t);
            }
        }
        int err_eq = 0;
        for (const std::string &t : bad) {
            const ProcessorBuffer *pr = nullptr, *po = nullptr;
            const std::string er = error_of(ref_par, t, &pr);
            ProcessorBuffer keep_r;
            if (pr) keep_r = *pr;
            const std::string eo = error_of(our_par, t, &po);
            bool eq = er == eo;
            if (eq && er == "<no error>") eq = same(keep_r, *po);
            err_eq += eq;
            if (std::getenv("WIRE_BENCH_LIST")) std::fprintf(stderr, "[%s] %s\n", cs.name, er.c_str());
            if (!eq && std::getenv("WIRE_BENCH_VERBOSE"))
                std::fprintf(stderr, "[%s] ref: %s | ours: %s\n", cs.name, er.c_str(), eo.c_str());
        }
        const int err_cases = (int)bad.size();
        ok &= bytes_eq && parse_eq && err_eq == err_cases;
        size_t n_cts = 0;
        if (const auto *g = std::get_if<GhPayload>(&b.payload)) n_cts = g->cts.size();
        if (const auto *h = std::get_if<HistogramPayload>(&b.payload))
            for (const NodeHistogram &nd : h->nodes) n_cts += nd.scalar_cts.size() + nd.packed_g.cts.size() + nd.packed_h.cts.size();
        std::snprintf(line, sizeof line,
                      "%s\"%s\": {\"ciphertexts\": %zu, \"bytes\": %zu, \"serialize_ref_s\": %.4f, "
                      "\"serialize_s\": %.4f, \"parse_ref_s\": %.4f, \"parse_s\": %.4f, \"bytes_identical\": %s, "
                      "\"parse_identical\": %s, \"malformed_same_error\": \"%d/%d\"}",
                      report.empty() ? "" : ", ", cs.name, n_cts, rb.size(), secs(t0, t1), secs(t1, t2), secs(t2, t3),
                      secs(t3, t4), bytes_eq ? "true" : "false", parse_eq ? "true" : "false", err_eq, err_cases);
        report += line;
    }
    std::printf("{\"interposed\": %s, \"bits\": %u, %s, \"ok\": %s}\n", interposed ? "true" : "false", bits,
                report.c_str(), ok ? "true" : "false");
    return ok ? 0 : 1;
}
