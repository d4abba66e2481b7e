// Host-side fixed-width big integers for per-key precomputation only
// (Montgomery constants, CRT constants, exponent digits).  Little-endian u32
// limbs in std::vector.  None of this runs per ciphertext; the per-element
// arithmetic is on the device (mont.cuh).
#pragma once
#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace sfxb {
namespace host {

using Big = std::vector<uint32_t>;

inline void trim(Big &a) {
    while (a.size() > 1 && a.back() == 0) a.pop_back();
    if (a.empty()) a.push_back(0);
}
inline Big from_u64(uint64_t v) {
    Big a{static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32)};
    trim(a);
    return a;
}
inline Big from_words(const uint32_t *w, size_t n) {
    Big a(w, w + n);
    trim(a);
    return a;
}
inline bool is_zero(const Big &a) {
    for (uint32_t w : a)
        if (w) return false;
    return true;
}
inline size_t bit_length(const Big &a) {
    for (size_t i = a.size(); i-- > 0;)
        if (a[i]) return i * 32 + (32 - __builtin_clz(a[i]));
    return 0;
}
inline int bit(const Big &a, size_t i) { return i / 32 < a.size() ? (a[i / 32] >> (i % 32)) & 1 : 0; }
inline int cmp(const Big &a, const Big &b) {
    size_t n = std::max(a.size(), b.size());
    for (size_t i = n; i-- > 0;) {
        uint32_t x = i < a.size() ? a[i] : 0, y = i < b.size() ? b[i] : 0;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}
inline Big add(const Big &a, const Big &b) {
    size_t n = std::max(a.size(), b.size());
    Big r(n + 1);
    uint64_t c = 0;
    for (size_t i = 0; i < n; ++i) {
        c += (uint64_t)(i < a.size() ? a[i] : 0) + (i < b.size() ? b[i] : 0);
        r[i] = (uint32_t)c;
        c >>= 32;
    }
    r[n] = (uint32_t)c;
    trim(r);
    return r;
}
// a - b, requires a >= b
inline Big sub(const Big &a, const Big &b) {
    if (cmp(a, b) < 0) throw std::logic_error("bignum sub underflow");
    Big r(a.size());
    int64_t br = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        int64_t d = (int64_t)a[i] - (i < b.size() ? b[i] : 0) - br;
        br = d < 0;
        r[i] = (uint32_t)(d + (br ? (int64_t(1) << 32) : 0));
    }
    trim(r);
    return r;
}
inline Big mul(const Big &a, const Big &b) {
    Big r(a.size() + b.size(), 0);
    for (size_t i = 0; i < a.size(); ++i) {
        uint64_t c = 0;
        for (size_t j = 0; j < b.size(); ++j) {
            c += (uint64_t)a[i] * b[j] + r[i + j];
            r[i + j] = (uint32_t)c;
            c >>= 32;
        }
        r[i + b.size()] = (uint32_t)c;
    }
    trim(r);
    return r;
}
// a mod m by binary long division (precomputation sizes only)
inline Big mod(const Big &a, const Big &m) {
    if (is_zero(m)) throw std::logic_error("bignum mod by zero");
    Big r{0};
    for (size_t i = bit_length(a); i-- > 0;) {
        // r = 2r + bit
        uint32_t c = (uint32_t)bit(a, i);
        for (size_t k = 0; k < r.size(); ++k) {
            uint32_t nc = r[k] >> 31;
            r[k] = (r[k] << 1) | c;
            c = nc;
        }
        if (c) r.push_back(c);
        if (cmp(r, m) >= 0) r = sub(r, m);
    }
    trim(r);
    return r;
}
inline Big pad(const Big &a, size_t words) {
    if (bit_length(a) > 32 * words) throw std::logic_error("bignum does not fit");
    Big r(words, 0);
    std::copy(a.begin(), a.begin() + std::min(a.size(), words), r.begin());
    return r;
}
// -m^-1 mod 2^32 (m odd)
inline uint32_t neg_inv32(uint32_t m0) {
    uint32_t x = 1;
    for (int i = 0; i < 5; ++i) x *= 2 - m0 * x; // Newton: x = m0^-1 mod 2^32
    return (uint32_t)(0u - x);
}
// low `words` limbs of a (a mod 2^(32·words)), always exactly `words` long
inline Big low(const Big &a, size_t words) {
    Big r(words, 0);
    std::copy(a.begin(), a.begin() + std::min(a.size(), words), r.begin());
    return r;
}
// m^-1 mod 2^(32·words) (m odd), Newton iteration x <- x·(2 − m·x)
inline Big inv_pow2(const Big &m, size_t words) {
    Big x = low(from_u64(0u - neg_inv32(m[0])), words); // m^-1 mod 2^32
    Big two_pow(words + 1, 0);
    two_pow[words] = 1;
    for (size_t bits = 32; bits < 32 * words; bits *= 2) {
        Big mx = low(mul(low(m, words), x), words);
        Big f = low(sub(add(two_pow, from_u64(2)), mx), words); // 2 − m·x mod 2^(32 words)
        x = low(mul(x, f), words);
    }
    return x;
}

// Montgomery context on the host (same R = 2^(32·S) as the device).
struct MontHost {
    Big m;      // modulus, S words
    size_t S;   // words
    uint32_t np;
    Big r1, r2, r3; // R, R², R³ mod m

    MontHost(const Big &mod_, size_t S_) : m(pad(mod_, S_)), S(S_) {
        if ((m[0] & 1) == 0) throw std::invalid_argument("Montgomery modulus must be odd");
        np = neg_inv32(m[0]);
        Big R(S + 1, 0);
        R[S] = 1;
        r1 = pad(mod(R, m), S);
        r2 = pad(mod(mul(r1, r1), m), S);
        r3 = pad(mod(mul(r2, r1), m), S);
    }
    // a·b·R^-1 mod m (CIOS, host reference of the device algorithm)
    Big mont_mul(const Big &a_, const Big &b_) const {
        Big a = pad(a_, S), b = pad(b_, S);
        std::vector<uint32_t> t(S + 2, 0);
        for (size_t i = 0; i < S; ++i) {
            uint64_t c = 0;
            for (size_t j = 0; j < S; ++j) {
                c += (uint64_t)a[j] * b[i] + t[j];
                t[j] = (uint32_t)c;
                c >>= 32;
            }
            c += t[S];
            t[S] = (uint32_t)c;
            t[S + 1] = (uint32_t)(c >> 32);
            uint32_t q = t[0] * np;
            c = ((uint64_t)q * m[0] + t[0]) >> 32;
            for (size_t j = 1; j < S; ++j) {
                c += (uint64_t)q * m[j] + t[j];
                t[j - 1] = (uint32_t)c;
                c >>= 32;
            }
            c += t[S];
            t[S - 1] = (uint32_t)c;
            t[S] = t[S + 1] + (uint32_t)(c >> 32);
            t[S + 1] = 0;
        }
        Big r(t.begin(), t.begin() + S + 1);
        if (cmp(r, m) >= 0) r = sub(r, m);
        return pad(r, S);
    }
    Big to_mont(const Big &x) const { return mont_mul(pad(mod(x, m), S), r2); }
    Big from_mont(const Big &x) const { return mont_mul(x, pad(from_u64(1), S)); }
    // x^e mod m (plain in/out)
    Big pow(const Big &x, const Big &e) const {
        Big acc = r1, base = to_mont(x);
        for (size_t i = bit_length(e); i-- > 0;) {
            acc = mont_mul(acc, acc);
            if (bit(e, i)) acc = mont_mul(acc, base);
        }
        return from_mont(acc);
    }
};

// x^-1 mod prime p (Fermat)
inline Big inv_mod_prime(const Big &x, const Big &p, size_t S) {
    MontHost mh(p, S);
    return mh.pow(mod(x, p), sub(p, from_u64(2)));
}

// x^-1 mod M for odd M and gcd(x, M) = 1 (binary extended Euclid, fixed-size
// in-place limb arithmetic).  Returns false when x is not invertible.
inline bool inv_mod_odd(const Big &x_, const Big &M_, Big &out) {
    const size_t W = M_.size() + 1;
    Big M = low(M_, W), u = low(mod(x_, M_), W), v = M, x1(W, 0), x2(W, 0);
    x1[0] = 1;
    auto is_one = [&](const Big &a) {
        if (a[0] != 1) return false;
        for (size_t i = 1; i < W; ++i)
            if (a[i]) return false;
        return true;
    };
    auto is_zero_w = [&](const Big &a) {
        for (size_t i = 0; i < W; ++i)
            if (a[i]) return false;
        return true;
    };
    auto shr1 = [&](Big &a) {
        for (size_t i = 0; i + 1 < W; ++i) a[i] = (a[i] >> 1) | (a[i + 1] << 31);
        a[W - 1] >>= 1;
    };
    auto add_in = [&](Big &a, const Big &b) { // a += b (no overflow: values < 2M < 2^(32W))
        uint64_t c = 0;
        for (size_t i = 0; i < W; ++i) {
            c += (uint64_t)a[i] + b[i];
            a[i] = (uint32_t)c;
            c >>= 32;
        }
    };
    auto sub_in = [&](Big &a, const Big &b) { // a -= b, requires a >= b
        int64_t br = 0;
        for (size_t i = 0; i < W; ++i) {
            int64_t d = (int64_t)a[i] - b[i] - br;
            br = d < 0;
            a[i] = (uint32_t)(d + (br ? (int64_t(1) << 32) : 0));
        }
    };
    auto geq = [&](const Big &a, const Big &b) {
        for (size_t i = W; i-- > 0;)
            if (a[i] != b[i]) return a[i] > b[i];
        return true;
    };
    auto half_mod = [&](Big &a) { // a/2 mod M
        if (a[0] & 1) add_in(a, M);
        shr1(a);
    };
    auto sub_mod = [&](Big &a, const Big &b) { // a = a − b mod M (a, b < M)
        if (!geq(a, b)) add_in(a, M);
        sub_in(a, b);
    };
    if (is_zero_w(u)) return false;
    while (!is_one(u) && !is_one(v)) {
        if (is_zero_w(u) || is_zero_w(v)) return false;
        while ((u[0] & 1) == 0) {
            shr1(u);
            half_mod(x1);
        }
        while ((v[0] & 1) == 0) {
            shr1(v);
            half_mod(x2);
        }
        if (geq(u, v)) {
            sub_in(u, v);
            sub_mod(x1, x2);
        } else {
            sub_in(v, u);
            sub_mod(x2, x1);
        }
    }
    out = is_one(u) ? x1 : x2;
    trim(out);
    out = mod(out, M_);
    return true;
}

// x^-1 mod M through libgmp's mpz_invert when libgmp.so.10 can be loaded at
// runtime (≈50 µs at 4096 bits; the reference links GMP anyway), else the
// binary extended Euclid above (≈3.5 ms).  dlopen keeps GMP an optional
// runtime dependency of libsfxb_cuda.so.
bool inv_mod_fast(const Big &x, const Big &M, Big &out);

// Fixed-window digits of e (most significant first), window w bits.
inline std::vector<uint8_t> window_digits(const Big &e, int w) {
    size_t nb = std::max<size_t>(bit_length(e), 1);
    size_t nd = (nb + w - 1) / w;
    std::vector<uint8_t> d(nd);
    for (size_t i = 0; i < nd; ++i) {
        size_t lo = (nd - 1 - i) * w;
        uint32_t v = 0;
        for (int k = 0; k < w; ++k) v |= (uint32_t)bit(e, lo + k) << k;
        d[i] = (uint8_t)v;
    }
    return d;
}

// Sliding-window program of e (e > 0), window ≤ w bits: byte pairs
// (squarings, odd digit d) — the first pair starts the accumulator at x^d,
// every later pair squares `squarings` times and then multiplies by x^d
// (d == 0: squarings only).  Uses the table of odd powers x^1, x^3, …,
// x^(2^w − 1).
inline std::vector<uint8_t> sliding_ops(const Big &e, int w) {
    std::vector<uint8_t> ops;
    long i = (long)bit_length(e) - 1;
    if (i < 0) return {0, 0};
    bool first = true;
    unsigned pend = 0; // squarings not emitted yet
    while (i >= 0) {
        if (!bit(e, (size_t)i)) {
            ++pend;
            --i;
            continue;
        }
        long lo = std::max<long>(i - w + 1, 0);
        while (!bit(e, (size_t)lo)) ++lo; // window ends in a 1
        uint32_t d = 0;
        for (long k = i; k >= lo; --k) d = (d << 1) | (uint32_t)bit(e, (size_t)k);
        const unsigned len = (unsigned)(i - lo + 1);
        if (first) {
            ops.push_back(0);
            ops.push_back((uint8_t)d);
            first = false;
        } else {
            pend += len;
            while (pend > 255) {
                ops.push_back(255);
                ops.push_back(0);
                pend -= 255;
            }
            ops.push_back((uint8_t)pend);
            ops.push_back((uint8_t)d);
        }
        pend = 0;
        i = lo - 1;
    }
    while (pend > 0) {
        const unsigned k = std::min(pend, 255u);
        ops.push_back((uint8_t)k);
        ops.push_back(0);
        pend -= k;
    }
    return ops;
}

} // namespace host
} // namespace sfxb
