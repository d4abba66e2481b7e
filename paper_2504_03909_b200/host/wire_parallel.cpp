// Wire codec for the ciphertext-carrying processor buffers (SURVEY §8f rank
// 1): sfxb::serialize_buffer / sfxb::parse_buffer (secure_processor.hpp:
// 171-172, secure_processor.cpp:119-375) for the gh_pairs_enc,
// histogram_enc and agg_result_enc kinds (scalar and packed layouts) — the
// ≈1 GB per tree that Bus::send (federation.cpp:96-102) serializes and
// re-parses — written here, for every buffer size and every malformed input.
//
// Interposed the same way as make_paillier_plugin: this library is loaded
// ahead of the reference library, whose call sites reach both functions
// through the PLT.  The other kinds (plain gradients / histograms, cut_sync,
// tree_sync: no ciphertexts, outside the hot path) are handed to the
// reference's definitions (dlsym(RTLD_NEXT)) after the common header checks.
//
// Format (the reference's, reproduced byte for byte):
//   header  "SFXB", u8 version 1, u8 kind, 3 × u32 LE
//   put_ct  (:39-45) u32 LE byte count, then |value| big-endian without
//           leading zero bytes (count 0 for value 0); here the count comes
//           from the limb header and the bytes from byte-swapped limb stores,
//           ciphertexts written on all host threads into one pre-sized buffer;
//   reading (:52-90, :221-375) WireReader: a missing byte is
//           ParseError("truncated buffer", size); a length running past the
//           end is ParseError("truncated ciphertext entry", offset after the
//           length); a surplus is ParseError("trailing bytes in buffer", pos);
//           parsed ciphertexts carry key id 0.  Here the length chain is
//           walked first (for gh buffers on all host threads, walk_entries),
//           the payload's vectors are reserved exactly where the reference
//           reserves them, and the limb imports run on all host threads.
//           Errors come from the same walk, so type, message and offset are
//           the reference's.
// SFXB_WIRE_VERBOSE=1: how many buffers each path handled, at exit.
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
    std::atomic<unsigned long long> ser_native{0}, ser_ref{0}, parse_native{0}, parse_ref{0};
    ~Stats() {
        if (std::getenv("SFXB_WIRE_VERBOSE"))
            std::fprintf(stderr, "[sfxb-wire] serialize native=%llu ref=%llu parse native=%llu ref=%llu\n",
                         ser_native.load(), ser_ref.load(), parse_native.load(), parse_ref.load());
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

// kinds without ciphertexts (outside the hot path): the reference's codec
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

// ---------------------------------------------------------------- serialize

// Ciphertext runs of one buffer in wire order: (first ciphertext, count)
using Runs = std::vector<std::pair<const Ciphertext *, size_t>>;

// A buffer as fixed bytes around ciphertext runs: prefix, run 0, between[0],
// run 1, between[1], ...  One pass sizes every entry; the fixed bytes are
// copied in order and the ciphertexts written on all host threads.
struct Layout {
    std::string prefix;
    std::vector<std::string> between; // bytes after run r
    Runs runs;
    std::string *gap() { return between.empty() ? &prefix : &between.back(); }
    void run(const std::vector<Ciphertext> &v) {
        runs.emplace_back(v.data(), v.size());
        between.emplace_back();
    }
};

std::string emit(const Layout &lay) {
    ++stats.ser_native;
    const Runs &runs = lay.runs;
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

void put_u8(std::string &s, uint8_t v) { s.push_back(static_cast<char>(v)); }

void put_u32(std::string &s, uint32_t v) {
    char b[4];
    le32(b, v);
    s.append(b, 4);
}

std::string head_bytes(const ProcessorBuffer &b) {
    std::string s(kMagic, 4);
    put_u8(s, b.version);
    put_u8(s, static_cast<uint8_t>(b.kind));
    for (uint32_t h : b.header) put_u32(s, h);
    return s;
}

bool enc_hist_kind(BufferKind k) { return k == BufferKind::histogram_enc || k == BufferKind::agg_result_enc; }

// put_packed (secure_processor.cpp:92-100): six u32 descriptors, then the run
void packed_into(Layout &lay, const PackedVector &v) {
    std::string *g = lay.gap();
    put_u32(*g, v.logical_length);
    put_u32(*g, v.addend_count);
    put_u32(*g, v.slot_bits);
    put_u32(*g, v.guard_bits);
    put_u32(*g, v.scale_bits);
    put_u32(*g, static_cast<uint32_t>(v.cts.size()));
    lay.run(v.cts);
}

// ---------------------------------------------------------------- parse

// WireReader (secure_processor.cpp:52-90) positions and errors
struct Cursor {
    const char *d;
    size_t size, pos;
    [[noreturn]] void truncated() const { throw ParseError("truncated buffer", size); }
    uint8_t u8() {
        if (pos >= size) truncated();
        return static_cast<uint8_t>(d[pos++]);
    }
    uint32_t u32() {
        if (size - pos < 4) truncated(); // the reference reads byte by byte up to the end
        const uint32_t v = rd32(d + pos);
        pos += 4;
        return v;
    }
    // one ciphertext entry: its offset (of the length prefix)
    size_t ct() {
        const size_t at = pos;
        const uint32_t len = u32();
        if (pos + len > size) throw ParseError("truncated ciphertext entry", pos);
        pos += len;
        return at;
    }
    void done() const {
        if (pos != size) throw ParseError("trailing bytes in buffer", pos);
    }
};

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

// imports of every recorded entry into its destination, on all host threads
void import_entries(const char *d, const std::vector<size_t> &off, const std::vector<Ciphertext *> &dst) {
    hostpar::parallel_for(off.size(), [&](size_t lo, size_t hi) {
        for (size_t k = lo; k < hi; ++k) get_ct_at(dst[k]->value, d + off[k] + 4, rd32(d + off[k]));
    }, 1024);
}

// gh_pairs_enc body (secure_processor.cpp:238-246)
GhPayload parse_gh(Cursor &r, uint32_t n_samples) {
    GhPayload gh;
    gh.encrypted = true;
    gh.n_samples = n_samples;
    const uint64_t n = 2ull * n_samples;
    std::vector<size_t> off;
    bool ok = false;
    if (n <= (r.size - r.pos) / 4) {
        // the n empty ciphertexts are constructed on a second thread while the
        // length chain is walked on all host threads
        std::thread alloc([&] { gh.cts.resize(n); });
        ok = walk_entries(r.d, r.size, r.pos, n, off);
        alloc.join();
    }
    if (!ok) {
        // malformed (or cannot hold n length prefixes): the reference's own
        // sequence — reserve, read entry by entry, then the trailing check —
        // raises the error at its offset
        gh.cts.clear();
        gh.cts.shrink_to_fit();
        gh.cts.reserve(n);
        for (uint64_t i = 0; i < n; ++i) r.ct();
        r.done();
        throw Error("wire codec: gh walk disagrees with the serial reader"); // not reached
    }
    std::vector<Ciphertext *> dst(n);
    for (uint64_t i = 0; i < n; ++i) dst[i] = &gh.cts[i];
    import_entries(r.d, off, dst);
    r.pos = r.size;
    return gh;
}

// read_packed (secure_processor.cpp:102-113): descriptors, then the entries;
// returns the entry count
size_t read_packed(Cursor &r, PackedVector &v, std::vector<size_t> &off) {
    v.logical_length = r.u32();
    v.addend_count = r.u32();
    v.slot_bits = r.u32();
    v.guard_bits = r.u32();
    v.scale_bits = r.u32();
    const uint32_t n = r.u32();
    v.cts.reserve(n);
    for (uint32_t i = 0; i < n; ++i) off.push_back(r.ct());
    return n;
}

// histogram_enc / agg_result_enc body (secure_processor.cpp:272-299)
HistogramPayload parse_hist(Cursor &r, const uint32_t header[3]) {
    HistogramPayload hp;
    const uint8_t layout = r.u8();
    if (layout > 1) throw ParseError("unknown encrypted histogram layout", r.pos - 1);
    hp.layout = static_cast<HistLayout>(layout);
    const uint32_t n_bins = header[1];
    std::vector<size_t> off; // every entry in wire order
    struct Run {
        size_t node;
        int vec; // 0 scalar_cts, 1 packed_g, 2 packed_h
        size_t count;
    };
    std::vector<Run> runs;
    for (uint32_t ni = 0; ni < header[2]; ++ni) {
        NodeHistogram node;
        node.node_id = r.u32();
        node.n_bins = static_cast<int>(n_bins);
        const uint32_t n_feats = r.u32();
        for (uint32_t f = 0; f < n_feats; ++f) node.feature_ids.push_back(static_cast<int>(r.u32()));
        if (hp.layout == HistLayout::enc_scalar) {
            const uint64_t cnt = 2ull * n_feats * n_bins;
            node.scalar_cts.reserve(cnt);
            for (uint64_t i = 0; i < cnt; ++i) off.push_back(r.ct());
            runs.push_back(Run{hp.nodes.size(), 0, (size_t)cnt});
        } else {
            runs.push_back(Run{hp.nodes.size(), 1, read_packed(r, node.packed_g, off)});
            runs.push_back(Run{hp.nodes.size(), 2, read_packed(r, node.packed_h, off)});
        }
        hp.nodes.push_back(std::move(node));
    }
    r.done();
    // destinations in wire order, then the imports on all host threads
    std::vector<Ciphertext *> dst;
    dst.reserve(off.size());
    for (const Run &run : runs) {
        NodeHistogram &nd = hp.nodes[run.node];
        std::vector<Ciphertext> &v = run.vec == 0 ? nd.scalar_cts : run.vec == 1 ? nd.packed_g.cts : nd.packed_h.cts;
        v.resize(run.count);
        for (Ciphertext &c : v) dst.push_back(&c);
    }
    const hostpar::TopPadScope pad(r.size); // the limb arrays total ≈ the wire bytes
    import_entries(r.d, off, dst);
    return hp;
}

} // namespace

// secure_processor.cpp:119-215 for the ciphertext kinds
std::string serialize_buffer(const ProcessorBuffer &buffer) {
    if (buffer.kind == BufferKind::gh_pairs_enc) {
        const auto &gh = std::get<GhPayload>(buffer.payload);
        Layout lay;
        lay.prefix = head_bytes(buffer);
        lay.run(gh.cts);
        return emit(lay);
    }
    if (enc_hist_kind(buffer.kind)) {
        const auto &hp = std::get<HistogramPayload>(buffer.payload);
        Layout lay;
        lay.prefix = head_bytes(buffer);
        put_u8(lay.prefix, static_cast<uint8_t>(hp.layout));
        for (const NodeHistogram &nd : hp.nodes) {
            std::string *g = lay.gap();
            put_u32(*g, nd.node_id);
            put_u32(*g, static_cast<uint32_t>(nd.feature_ids.size()));
            for (int fid : nd.feature_ids) put_u32(*g, static_cast<uint32_t>(fid));
            if (hp.layout == HistLayout::enc_scalar) {
                lay.run(nd.scalar_cts);
            } else {
                packed_into(lay, nd.packed_g);
                packed_into(lay, nd.packed_h);
            }
        }
        return emit(lay);
    }
    return ref_serialize(buffer);
}

// secure_processor.cpp:221-375 for the ciphertext kinds
ProcessorBuffer parse_buffer(const std::string &bytes) {
    Cursor r{bytes.data(), bytes.size(), 0};
    if (r.size < 4 || std::memcmp(r.d, kMagic, 4) != 0) throw ParseError("bad buffer magic", 0);
    r.pos = 4;
    ProcessorBuffer buf;
    buf.version = r.u8();
    if (buf.version != 1) throw ParseError("unsupported buffer version", 4);
    const uint8_t kind = r.u8();
    if (kind < 1 || kind > 8) throw ParseError("unknown buffer kind", 5);
    buf.kind = static_cast<BufferKind>(kind);
    const bool gh = buf.kind == BufferKind::gh_pairs_enc, hist = enc_hist_kind(buf.kind);
    if (!gh && !hist) return ref_parse(bytes);
    for (uint32_t &h : buf.header) h = r.u32();
    if (gh) {
        const hostpar::TopPadScope pad(r.size); // the limb arrays total ≈ the wire bytes
        buf.payload = parse_gh(r, buf.header[0]);
    } else {
        buf.payload = parse_hist(r, buf.header);
    }
    ++stats.parse_native;
    return buf;
}

} // namespace sfxb
