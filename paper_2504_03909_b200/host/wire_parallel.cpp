// Parallel wire codec for the ciphertext-carrying processor buffers (SURVEY
// §8f rank 1): sfxb::serialize_buffer / sfxb::parse_buffer
// (secure_processor.hpp:171-172, secure_processor.cpp:119-375) for the
// gh_pairs_enc and scalar histogram_enc / agg_result_enc kinds, the ≈1 GB
// per tree that Bus::send (federation.cpp:96-102) serializes and re-parses.
//
// Interposed the same way as make_paillier_plugin: this library is loaded
// ahead of the reference library, whose call sites reach both functions
// through the PLT.  Every other kind, the packed layout, small buffers and
// every malformed input go to the reference's own implementation
// (dlsym(RTLD_NEXT)), so error types, messages and offsets are the
// reference's.  Output bytes and parsed payloads are identical:
//   * put_ct (secure_processor.cpp:39-45) writes u32 LE byte count, then
//     |value| big-endian without leading zero bytes (count 0 for value 0);
//     here: count from the limb header, bytes by byte-swapped limb stores;
//   * WireReader::ct (:71-79) imports count bytes big-endian, key_id 0;
//     here: a walk over the length prefixes finds every entry's offset (and
//     every truncation, which the reference then reports) — for gh buffers on
//     all host threads (walk_entries) — then the imports run on all host
//     threads into limbs directly.
// SFXB_WIRE_MIN_CTS (default 4096): buffers with fewer ciphertexts use the
// reference path unchanged.  SFXB_WIRE_VERBOSE=1: call counts at exit.
#include <gmp.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "parallel.hpp"
#include "sfxb/errors.hpp"
#include "sfxb/secure_processor.hpp"

namespace sfxb {
namespace {

struct Stats {
    std::atomic<unsigned long long> ser_fast{0}, ser_ref{0}, parse_fast{0}, parse_ref{0};
    ~Stats() {
        if (std::getenv("SFXB_WIRE_VERBOSE"))
            std::fprintf(stderr, "[sfxb-wire] serialize fast=%llu ref=%llu parse fast=%llu ref=%llu\n",
                         ser_fast.load(), ser_ref.load(), parse_fast.load(), parse_ref.load());
    }
} stats;

using SerializeFn = std::string (*)(const ProcessorBuffer &);
using ParseFn = ProcessorBuffer (*)(const std::string &);

template <typename Fn>
Fn next_symbol(const char *mangled) {
    void *p = dlsym(RTLD_NEXT, mangled);
    if (!p) throw Error(std::string("sfxb wire codec: reference symbol not found: ") + mangled);
    return reinterpret_cast<Fn>(p);
}

std::string ref_serialize(const ProcessorBuffer &b) {
    ++stats.ser_ref;
    static SerializeFn f = next_symbol<SerializeFn>("_ZN4sfxb16serialize_bufferB5cxx11ERKNS_15ProcessorBufferE");
    return f(b);
}

ProcessorBuffer ref_parse(const std::string &s) {
    ++stats.parse_ref;
    static ParseFn f =
        next_symbol<ParseFn>("_ZN4sfxb12parse_bufferERKNSt7__cxx1112basic_stringIcSt11char_traitsIcESaIcEEE");
    return f(s);
}

size_t min_cts() {
    static size_t n = [] {
        const char *e = std::getenv("SFXB_WIRE_MIN_CTS");
        return e ? (size_t)std::strtoull(e, nullptr, 10) : (size_t)4096;
    }();
    return n;
}


constexpr char kMagic[4] = {'S', 'F', 'X', 'B'};

void le32(char *p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<char>((v >> (8 * i)) & 0xFF);
}

uint32_t rd32(const char *p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(static_cast<uint8_t>(p[i])) << (8 * i);
    return v;
}

// bytes put_ct writes for |v| (mpz_export count)
size_t ct_len(const mpz_class &v) {
    const size_t n = mpz_size(v.get_mpz_t());
    if (n == 0) return 0;
    const mp_limb_t top = mpz_limbs_read(v.get_mpz_t())[n - 1];
    return 8 * (n - 1) + (size_t)((64 - __builtin_clzll(top) + 7) / 8);
}

// u32 LE len, then |v| big-endian (len bytes)
void put_ct_at(char *dst, const mpz_class &v, size_t len) {
    le32(dst, static_cast<uint32_t>(len));
    dst += 4;
    if (!len) return;
    const mp_limb_t *l = mpz_limbs_read(v.get_mpz_t());
    const size_t full = len / 8, rb = len % 8;
    for (size_t k = 0; k < full; ++k) {
        const uint64_t be = __builtin_bswap64(l[k]);
        std::memcpy(dst + len - 8 * (k + 1), &be, 8);
    }
    if (rb) {
        const uint64_t top = l[full];
        for (size_t j = 0; j < rb; ++j) dst[j] = static_cast<char>((top >> (8 * (rb - 1 - j))) & 0xFF);
    }
}

// mpz_import(v, len, 1, 1, 1, 0, src)
void get_ct_at(mpz_class &v, const char *src, size_t len) {
    if (len == 0) {
        v = 0;
        return;
    }
    const size_t nl = (len + 7) / 8;
    mp_limb_t *l = mpz_limbs_write(v.get_mpz_t(), (mp_size_t)nl);
    const size_t full = len / 8, rb = len % 8;
    for (size_t k = 0; k < full; ++k) {
        uint64_t be;
        std::memcpy(&be, src + len - 8 * (k + 1), 8);
        l[k] = __builtin_bswap64(be);
    }
    if (rb) {
        uint64_t top = 0;
        for (size_t j = 0; j < rb; ++j) top = (top << 8) | static_cast<uint8_t>(src[j]);
        l[full] = top;
    }
    mpz_limbs_finish(v.get_mpz_t(), (mp_size_t)nl);
}

// Ciphertext runs of one buffer in wire order: (first ciphertext, count)
using Runs = std::vector<std::pair<const Ciphertext *, size_t>>;

// A buffer as fixed bytes around ciphertext runs: prefix, run 0, between[0],
// run 1, between[1], ...  One pass sizes every entry; the fixed bytes are
// copied in order and the ciphertexts written on all host threads.
struct Layout {
    std::string prefix;
    std::vector<std::string> between; // bytes after run r
};

std::string emit(const Layout &lay, const Runs &runs) {
    ++stats.ser_fast;
    size_t total = 0;
    for (const auto &r : runs) total += r.second;
    std::vector<const Ciphertext *> ct(total);
    for (size_t r = 0, k = 0; r < runs.size(); ++r)
        for (size_t i = 0; i < runs[r].second; ++i) ct[k++] = runs[r].first + i;
    std::vector<size_t> len(total), off(total);
    hostpar::parallel_for(total, [&](size_t lo, size_t hi) {
        for (size_t k = lo; k < hi; ++k) len[k] = ct_len(ct[k]->value);
    });
    std::vector<size_t> gap_at(runs.size());
    size_t pos = lay.prefix.size();
    for (size_t r = 0, k = 0; r < runs.size(); ++r) {
        for (size_t i = 0; i < runs[r].second; ++i, ++k) {
            off[k] = pos;
            pos += 4 + len[k];
        }
        gap_at[r] = pos;
        pos += lay.between[r].size();
    }
    std::string out;
    out.resize_and_overwrite(pos, [&](char *p, size_t n) {
        std::memcpy(p, lay.prefix.data(), lay.prefix.size());
        for (size_t r = 0; r < runs.size(); ++r)
            std::memcpy(p + gap_at[r], lay.between[r].data(), lay.between[r].size());
        hostpar::parallel_for(total, [&](size_t lo, size_t hi) {
            for (size_t k = lo; k < hi; ++k) put_ct_at(p + off[k], ct[k]->value, len[k]);
        }, 1024);
        return n;
    });
    return out;
}

void put_u32(std::string &s, uint32_t v) {
    char b[4];
    le32(b, v);
    s.append(b, 4);
}

std::string head_bytes(const ProcessorBuffer &b) {
    std::string s(kMagic, 4);
    s.push_back(static_cast<char>(b.version));
    s.push_back(static_cast<char>(static_cast<uint8_t>(b.kind)));
    for (uint32_t h : b.header) put_u32(s, h);
    return s;
}

bool enc_hist_kind(BufferKind k) { return k == BufferKind::histogram_enc || k == BufferKind::agg_result_enc; }

// Offsets of the length-prefixed entries of d[start, size) in wire order, as
// the serial walk from `start` finds them; true iff that walk reads exactly n
// valid entries ending at `size` (the serial condition).  The buffer is cut
// into one byte range per host thread; each thread past the first finds a
// plausible entry start in its range (kSync consecutive lengths ≤ kSyncLen
// that stay inside the buffer) and walks from there to the end of its range.
// The true chain is then followed range by range: where it lands on a
// position a thread recorded, that thread's list is the true continuation
// (the walk from a position is deterministic); otherwise the range is walked
// serially.  A wrong sync therefore costs time, never a different result.
bool walk_entries(const char *d, size_t size, size_t start, uint64_t n, std::vector<size_t> &off) {
    // SFXB_WIRE_WALK_TEST=1 (tests): accept the first in-buffer length as an
    // entry start, so most ranges sync wrongly and take the serial fallback
    static const bool loose = std::getenv("SFXB_WIRE_WALK_TEST") != nullptr;
    const size_t kSync = loose ? 1 : 16, kSyncLen = loose ? SIZE_MAX : 4096;
    constexpr size_t kMinRange = size_t(1) << 20;
    const unsigned T = std::min<size_t>(hostpar::host_threads(), (size - start) / kMinRange);
    // one entry at p: its end, or 0 when the length runs past the buffer
    auto next = [&](size_t p) -> size_t {
        if (size - p < 4) return 0;
        const uint32_t len = rd32(d + p);
        return len > size - p - 4 ? 0 : p + 4 + (size_t)len;
    };
    auto serial = [&](size_t p, size_t stop, std::vector<size_t> &out) -> size_t { // 0 = invalid entry
        while (p < stop) {
            const size_t q = next(p);
            if (!q) return 0;
            __builtin_prefetch(d + q + 16 * (q - p));
            out.push_back(p);
            p = q;
        }
        return p;
    };
    off.clear();
    if (T < 2) {
        off.reserve(n);
        return serial(start, size, off) == size && off.size() == n;
    }
    std::vector<size_t> lo(T + 1);
    for (unsigned t = 0; t <= T; ++t) lo[t] = start + (size - start) / T * t;
    lo[T] = size;
    std::vector<std::vector<size_t>> lists(T);
    std::vector<size_t> ends(T, 0);
    hostpar::parallel_for(T, [&](size_t a, size_t b) {
        for (size_t t = a; t < b; ++t) {
            size_t s = lo[t];
            if (t > 0) {
                for (; s < lo[t + 1]; ++s) {
                    size_t p = s, k = 0;
                    for (; k < kSync && p < size; ++k) {
                        if (size - p < 4 || rd32(d + p) > kSyncLen) break;
                        const size_t q = next(p);
                        if (!q) break;
                        p = q;
                    }
                    if (k == kSync || (p == size && k > 0)) break;
                }
                if (s >= lo[t + 1]) continue; // no plausible start: walked serially below
            }
            lists[t].reserve((lo[t + 1] - s) / 256 + 16);
            ends[t] = serial(s, lo[t + 1], lists[t]);
        }
    }, 1);
    off.reserve(n);
    size_t p = start;
    for (unsigned t = 0; t < T && p < size; ++t) {
        if (p >= lo[t + 1]) continue;
        const auto &L = lists[t];
        auto it = std::lower_bound(L.begin(), L.end(), p);
        if (it != L.end() && *it == p) {
            if (!ends[t]) return false;
            off.insert(off.end(), it, L.end());
            p = ends[t];
        } else if (!(p = serial(p, lo[t + 1], off))) {
            return false;
        }
        if (off.size() > n) return false;
    }
    return p == size && off.size() == n;
}

} // namespace

// secure_processor.cpp:119-215 (fast path: gh_pairs_enc, scalar encrypted histograms)
std::string serialize_buffer(const ProcessorBuffer &buffer) {
    if (buffer.kind == BufferKind::gh_pairs_enc) {
        const auto *gh = std::get_if<GhPayload>(&buffer.payload);
        if (!gh || gh->cts.size() < min_cts()) return ref_serialize(buffer);
        Layout lay{head_bytes(buffer), {std::string()}};
        return emit(lay, Runs{{gh->cts.data(), gh->cts.size()}});
    }
    if (enc_hist_kind(buffer.kind)) {
        const auto *hp = std::get_if<HistogramPayload>(&buffer.payload);
        if (!hp || hp->layout != HistLayout::enc_scalar) return ref_serialize(buffer);
        size_t n = 0;
        for (const NodeHistogram &nd : hp->nodes) n += nd.scalar_cts.size();
        if (n < min_cts()) return ref_serialize(buffer);
        Layout lay;
        lay.prefix = head_bytes(buffer);
        lay.prefix.push_back(static_cast<char>(static_cast<uint8_t>(hp->layout)));
        Runs runs;
        std::string *gap = &lay.prefix;
        for (const NodeHistogram &nd : hp->nodes) {
            put_u32(*gap, nd.node_id);
            put_u32(*gap, static_cast<uint32_t>(nd.feature_ids.size()));
            for (int fid : nd.feature_ids) put_u32(*gap, static_cast<uint32_t>(fid));
            runs.emplace_back(nd.scalar_cts.data(), nd.scalar_cts.size());
            lay.between.emplace_back();
            gap = &lay.between.back();
        }
        if (runs.empty()) return ref_serialize(buffer);
        return emit(lay, runs);
    }
    return ref_serialize(buffer);
}

// secure_processor.cpp:221-375 (fast path: gh_pairs_enc, scalar encrypted histograms)
ProcessorBuffer parse_buffer(const std::string &bytes) {
    const size_t size = bytes.size();
    const char *d = bytes.data();
    if (size < 18 || std::memcmp(d, kMagic, 4) != 0 || static_cast<uint8_t>(d[4]) != 1) return ref_parse(bytes);
    const uint8_t kind = static_cast<uint8_t>(d[5]);
    const bool gh = kind == static_cast<uint8_t>(BufferKind::gh_pairs_enc);
    const bool hist = enc_hist_kind(static_cast<BufferKind>(kind));
    if (!gh && !hist) return ref_parse(bytes);
    const hostpar::TopPadScope pad(size); // the limb arrays total ≈ the wire bytes
    ProcessorBuffer buf;
    buf.version = 1;
    buf.kind = static_cast<BufferKind>(kind);
    for (int i = 0; i < 3; ++i) buf.header[i] = rd32(d + 6 + 4 * i);
    size_t pos = 18;
    // entry offsets of every ciphertext, in wire order; any truncation or
    // trailing byte hands the buffer to the reference (which reports it)
    std::vector<size_t> off;
    auto walk = [&](uint64_t count) -> bool {
        if (count > (size - pos) / 4) return false;
        for (uint64_t i = 0; i < count; ++i) {
            if (size - pos < 4) return false;
            const uint32_t len = rd32(d + pos);
            if (len > size - pos - 4) return false;
            // the length chain is serially dependent: prefetch where the
            // entry 16 ahead lands if the lengths repeat (they almost all
            // do: full-size residues mod n²)
            __builtin_prefetch(d + pos + 16 * (4 + (size_t)len));
            off.push_back(pos);
            pos += 4 + (size_t)len;
        }
        return true;
    };
    if (gh) {
        const uint64_t n = 2ull * buf.header[0];
        if (n < min_cts()) return ref_parse(bytes);
        if (n > (size - pos) / 4) return ref_parse(bytes); // cannot hold n length prefixes
        // the payload's n empty ciphertexts are constructed on a second thread
        // while the length chain is walked (walk_entries, all host threads)
        GhPayload p;
        p.encrypted = true;
        p.n_samples = buf.header[0];
        std::thread alloc([&] { p.cts.resize(n); });
        const bool ok = walk_entries(d, size, pos, n, off);
        alloc.join();
        if (!ok) return ref_parse(bytes);
        hostpar::parallel_for(n, [&](size_t lo, size_t hi) {
            for (size_t k = lo; k < hi; ++k) get_ct_at(p.cts[k].value, d + off[k] + 4, rd32(d + off[k]));
        }, 1024);
        buf.payload = std::move(p);
        ++stats.parse_fast;
        return buf;
    }
    if (size - pos < 1 || static_cast<uint8_t>(d[pos]) != 0) return ref_parse(bytes); // packed / bad layout
    ++pos;
    const uint32_t n_bins = buf.header[1];
    HistogramPayload hp;
    hp.layout = HistLayout::enc_scalar;
    std::vector<std::pair<size_t, size_t>> node_runs; // (first entry, count)
    for (uint32_t ni = 0; ni < buf.header[2]; ++ni) {
        if (size - pos < 8) return ref_parse(bytes);
        NodeHistogram node;
        node.node_id = rd32(d + pos);
        node.n_bins = static_cast<int>(n_bins);
        const uint32_t n_feats = rd32(d + pos + 4);
        pos += 8;
        if (n_feats > (size - pos) / 4) return ref_parse(bytes);
        node.feature_ids.reserve(n_feats);
        for (uint32_t f = 0; f < n_feats; ++f, pos += 4) node.feature_ids.push_back(static_cast<int>(rd32(d + pos)));
        const uint64_t cnt = 2ull * n_feats * n_bins;
        const size_t first = off.size();
        if (!walk(cnt)) return ref_parse(bytes);
        node_runs.emplace_back(first, (size_t)cnt);
        hp.nodes.push_back(std::move(node));
    }
    if (pos != size || off.size() < min_cts()) return ref_parse(bytes);
    for (size_t i = 0; i < hp.nodes.size(); ++i) hp.nodes[i].scalar_cts.resize(node_runs[i].second);
    std::vector<Ciphertext *> dst(off.size());
    for (size_t i = 0, k = 0; i < hp.nodes.size(); ++i)
        for (Ciphertext &c : hp.nodes[i].scalar_cts) dst[k++] = &c;
    hostpar::parallel_for(off.size(), [&](size_t lo, size_t hi) {
        for (size_t k = lo; k < hi; ++k) get_ct_at(dst[k]->value, d + off[k] + 4, rd32(d + off[k]));
    }, 1024);
    buf.payload = std::move(hp);
    ++stats.parse_fast;
    return buf;
}

} // namespace sfxb
