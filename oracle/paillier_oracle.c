/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the vertical secure hot path.
 *
 * A plain-C restatement of the reference's algorithm (GMP C API, same
 * libgmp.so.10 the reference links), used by tests/ and by bench.py's
 * cpu_baseline leg as the *checker*.  The product path never links this.
 * Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj).
 *
 * Pinning: tests/test_oracle.py checks this file
 * against the reference's own known-answer values (tests/test_he.cpp:22-41,
 * :111-121) and against golden vectors produced by the unmodified reference
 * library (oracle/_ref, tests/golden/make_golden.py).
 *
 * Number format at this boundary = the device format: little-endian u32
 * limbs, `nw` words for values mod n, `2*nw` words for values mod n².
 */
#include <gmp.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char *orc_last_error(void) { return g_err; }
static int fail(const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return -1;
}

static void imp(mpz_t z, const uint32_t *w, size_t words) { mpz_import(z, words, -1, 4, 0, 0, w); }
static int exp_words(uint32_t *out, size_t words, const mpz_t z) {
    memset(out, 0, words * 4);
    if (mpz_sgn(z) < 0) return fail("negative value cannot be exported");
    if (mpz_sizeinbase(z, 2) > 32 * words && mpz_sgn(z) != 0) return fail("value wider than buffer");
    size_t cnt = 0;
    mpz_export(out, &cnt, -1, 4, 0, 0, z);
    return 0;
}

/* ---- keys: he.hpp:11-27, keypair_from_primes he.cpp:40-56, key_id_of he.cpp:30-38 ---- */

typedef struct {
    mpz_t n, n2, p, q, lambda, mu;
    size_t nw;
    int has_priv;
    uint64_t key_id;
} orc_key;

/* FNV-1a 64 over the lower-case hex digits of n (he.cpp:30-38). */
uint64_t orc_key_id_of(const uint32_t *n, size_t nw) {
    mpz_t z;
    mpz_init(z);
    imp(z, n, nw);
    char *hex = mpz_get_str(NULL, 16, z);
    uint64_t h = 14695981039346656037ULL;
    for (const char *c = hex; *c; ++c) {
        h ^= (unsigned char)*c;
        h *= 1099511628211ULL;
    }
    free(hex);
    mpz_clear(z);
    return h;
}

/* p, q may be NULL (public-key-only holder, federation.cpp:83-85). */
orc_key *orc_key_new(const uint32_t *n, const uint32_t *p, const uint32_t *q, size_t nw) {
    orc_key *k = calloc(1, sizeof *k);
    mpz_init(k->n);
    mpz_init(k->n2);
    mpz_init(k->p);
    mpz_init(k->q);
    mpz_init(k->lambda);
    mpz_init(k->mu);
    k->nw = nw;
    imp(k->n, n, nw);
    mpz_mul(k->n2, k->n, k->n);
    k->key_id = orc_key_id_of(n, nw);
    if (p && q) {
        k->has_priv = 1;
        /* primes are half-size: nw/2 words each (he.cpp:58-85 draws half = bits/2) */
        imp(k->p, p, nw);
        imp(k->q, q, nw);
        mpz_t pm1, qm1;
        mpz_init(pm1);
        mpz_init(qm1);
        mpz_sub_ui(pm1, k->p, 1);
        mpz_sub_ui(qm1, k->q, 1);
        mpz_lcm(k->lambda, pm1, qm1);                /* he.cpp:51-52 */
        if (!mpz_invert(k->mu, k->lambda, k->n)) {   /* he.cpp:53-54 */
            mpz_clear(pm1);
            mpz_clear(qm1);
            fail("keypair_from_primes: lambda not invertible mod n");
            return NULL;
        }
        mpz_clear(pm1);
        mpz_clear(qm1);
    }
    return k;
}

void orc_key_free(orc_key *k) {
    if (!k) return;
    mpz_clear(k->n);
    mpz_clear(k->n2);
    mpz_clear(k->p);
    mpz_clear(k->q);
    mpz_clear(k->lambda);
    mpz_clear(k->mu);
    free(k);
}

uint64_t orc_key_id(const orc_key *k) { return k->key_id; }

/* ---- HeRng: he.hpp:35-44, he.cpp:11-28 ---- */

typedef struct {
    gmp_randstate_t st;
} orc_rng;

orc_rng *orc_rng_new(uint64_t seed) {
    orc_rng *r = calloc(1, sizeof *r);
    gmp_randinit_mt(r->st); /* he.cpp:11 gmp_randinit_mt */
    mpz_t s;
    mpz_init(s);
    mpz_import(s, 1, 1, sizeof seed, 0, 0, &seed); /* he.cpp:13 */
    gmp_randseed(r->st, s);
    mpz_clear(s);
    return r;
}

void orc_rng_free(orc_rng *r) {
    if (!r) return;
    gmp_randclear(r->st);
    free(r);
}

/* unit_below(n): he.cpp:19-28 — draw mpz_urandomm, reject r <= 1 and gcd(r,n) != 1. */
static void unit_below(orc_rng *rng, const mpz_t n, mpz_t r) {
    mpz_t g;
    mpz_init(g);
    for (;;) {
        mpz_urandomm(r, rng->st, n);
        if (mpz_cmp_ui(r, 1) <= 0) continue;
        mpz_gcd(g, r, n);
        if (mpz_cmp_ui(g, 1) == 0) break;
    }
    mpz_clear(g);
}

/* `count` consecutive blinding factors (the order encrypt_gh consumes them). */
int orc_rng_draw(orc_rng *rng, const orc_key *k, size_t count, uint32_t *out) {
    mpz_t r;
    mpz_init(r);
    for (size_t i = 0; i < count; ++i) {
        unit_below(rng, k->n, r);
        if (exp_words(out + i * k->nw, k->nw, r)) return -1;
    }
    mpz_clear(r);
    return 0;
}

/* ---- fixed point: fixed_point.hpp:13-15, encode_fixed he.cpp:125-136, decode he.cpp:138-143 ---- */

int orc_encode_fixed(const orc_key *k, double x, unsigned scale, uint32_t *out_m, int64_t *out_q) {
    if (!isfinite(x)) return fail("encode_fixed: value must be finite");
    if (fabs(x) >= ldexp(1.0, (int)(62 - scale)))
        return fail("encode_fixed: value too large for the fixed-point grid");
    int64_t q = llround(ldexp(x, (int)scale)); /* fixed_encode_ll */
    mpz_t m, mag;
    mpz_init_set_si(m, (long)q);
    mpz_init(mag);
    mpz_abs(mag, m);
    mpz_mul_2exp(mag, mag, 1);
    if (mpz_cmp(mag, k->n) >= 0) {
        mpz_clear(m);
        mpz_clear(mag);
        return fail("encode_fixed: |x|·2^scale_bits must stay below n/2");
    }
    if (mpz_sgn(m) < 0) mpz_add(m, m, k->n);
    if (out_q) *out_q = q;
    int rc = out_m ? exp_words(out_m, k->nw, m) : 0;
    mpz_clear(m);
    mpz_clear(mag);
    return rc;
}

/* mpz_get_d truncates toward zero (he.cpp:142 v.get_d()). */
double orc_decode_fixed(const orc_key *k, const uint32_t *raw, unsigned scale) {
    mpz_t v, twice;
    mpz_init(v);
    mpz_init(twice);
    imp(v, raw, k->nw);
    mpz_mul_2exp(twice, v, 1);
    if (mpz_cmp(twice, k->n) > 0) mpz_sub(v, v, k->n);
    double d = ldexp(mpz_get_d(v), -(int)scale);
    mpz_clear(v);
    mpz_clear(twice);
    return d;
}

/* ---- encrypt_with_r: he.cpp:87-99 ---- */

static int encrypt_with_r(const orc_key *k, const mpz_t m, const mpz_t r, mpz_t c) {
    if (mpz_sgn(m) < 0 || mpz_cmp(m, k->n) >= 0) return fail("encrypt: plaintext out of range [0, n)");
    if (mpz_cmp_ui(r, 1) < 0 || mpz_cmp(r, k->n) >= 0) return fail("encrypt: blinding factor out of range");
    mpz_t g, rn;
    mpz_init(g);
    mpz_init(rn);
    mpz_gcd(g, r, k->n);
    if (mpz_cmp_ui(g, 1) != 0) {
        mpz_clear(g);
        mpz_clear(rn);
        return fail("encrypt: blinding factor not coprime to modulus");
    }
    mpz_mul(c, m, k->n); /* (n+1)^m = 1 + m·n (mod n²) */
    mpz_add_ui(c, c, 1);
    mpz_tdiv_r(c, c, k->n2);
    mpz_powm(rn, r, k->n, k->n2); /* he.cpp:96 */
    mpz_mul(c, c, rn);
    mpz_tdiv_r(c, c, k->n2);
    mpz_clear(g);
    mpz_clear(rn);
    return 0;
}

int orc_encrypt_with_r(const orc_key *k, const uint32_t *m, const uint32_t *r, uint32_t *out_c) {
    mpz_t zm, zr, c;
    mpz_init(zm);
    mpz_init(zr);
    mpz_init(c);
    imp(zm, m, k->nw);
    imp(zr, r, k->nw);
    int rc = encrypt_with_r(k, zm, zr, c);
    if (!rc) rc = exp_words(out_c, 2 * k->nw, c);
    mpz_clear(zm);
    mpz_clear(zr);
    mpz_clear(c);
    return rc;
}

/* PaillierPlugin::encrypt_gh: secure_processor.cpp:574-585.
 * gh = 2*count doubles interleaved (g0,h0,g1,h1,...); r drawn in that order. */
int orc_encrypt_gh(const orc_key *k, orc_rng *rng, const double *gh, size_t count, unsigned scale,
                   uint32_t *out_cts, uint64_t *encryptions) {
    mpz_t m, r, c;
    mpz_init(m);
    mpz_init(r);
    mpz_init(c);
    uint32_t *mbuf = malloc(k->nw * 4);
    int rc = 0;
    for (size_t i = 0; i < 2 * count && !rc; ++i) {
        rc = orc_encode_fixed(k, gh[i], scale, mbuf, NULL);
        if (rc) break;
        imp(m, mbuf, k->nw);
        unit_below(rng, k->n, r);
        rc = encrypt_with_r(k, m, r, c);
        if (!rc) rc = exp_words(out_cts + i * 2 * k->nw, 2 * k->nw, c);
        if (!rc && (i & 1)) *encryptions += 2;
    }
    free(mbuf);
    mpz_clear(m);
    mpz_clear(r);
    mpz_clear(c);
    return rc;
}

/* ---- accumulate_rows: secure_processor.cpp:587-620, fold_into :724-732 ----
 * cts: 2*n_samples ciphertexts (interleaved g,h), each 2*nw words.
 * bins: n_features columns of n_samples uint16 (column-major, dataset.hpp:55-57).
 * nodes: node_offsets[N+1] into rows[].
 * out: N nodes × J × K × 2 slots, slot (node, f, b, gh) at ((node*J + f)*K + b)*2 + gh. */
int orc_accumulate(const orc_key *k, const uint32_t *cts, uint32_t n_samples, const uint16_t *bins,
                   uint32_t n_features, const uint32_t *node_offsets, uint32_t n_nodes,
                   const uint32_t *rows, uint32_t n_bins, uint32_t *out, uint64_t *additions) {
    const size_t cw = 2 * k->nw;
    const size_t slots_per_node = 2ull * n_features * n_bins;
    mpz_t *acc = malloc(slots_per_node * sizeof(mpz_t));
    mpz_t x;
    mpz_init(x);
    for (size_t s = 0; s < slots_per_node; ++s) mpz_init(acc[s]);
    int rc = 0;
    for (uint32_t nd = 0; nd < n_nodes && !rc; ++nd) {
        for (size_t s = 0; s < slots_per_node; ++s) mpz_set_ui(acc[s], 1); /* trivial_zero :605 */
        for (uint32_t f = 0; f < n_features && !rc; ++f) {
            const uint16_t *col = bins + (size_t)f * n_samples;
            for (uint32_t i = node_offsets[nd]; i < node_offsets[nd + 1]; ++i) {
                uint32_t row = rows[i];
                if (row >= n_samples) {
                    rc = fail("row index out of range in accumulate");
                    break;
                }
                uint16_t b = col[row];
                if (b >= n_bins) {
                    rc = fail("bin index out of range in accumulate"); /* :610-611 */
                    break;
                }
                size_t base = 2 * ((size_t)f * n_bins + b);
                for (int gh = 0; gh < 2; ++gh) {
                    imp(x, cts + (2 * (size_t)row + gh) * cw, cw);
                    /* fold_into: rhs==1 skipped, lhs==1 assigned, else mul mod n² counted */
                    if (mpz_cmp_ui(x, 1) == 0) continue;
                    if (mpz_cmp_ui(acc[base + gh], 1) == 0) {
                        mpz_set(acc[base + gh], x);
                        continue;
                    }
                    mpz_mul(acc[base + gh], acc[base + gh], x);
                    mpz_tdiv_r(acc[base + gh], acc[base + gh], k->n2); /* he.cpp:120 */
                    *additions += 1;
                }
            }
        }
        for (size_t s = 0; s < slots_per_node && !rc; ++s)
            rc = exp_words(out + ((size_t)nd * slots_per_node + s) * cw, cw, acc[s]);
    }
    for (size_t s = 0; s < slots_per_node; ++s) mpz_clear(acc[s]);
    free(acc);
    mpz_clear(x);
    return rc;
}

/* ---- decrypt: he.cpp:105-115 (no CRT: u = c^λ mod n², ℓ = (u−1)/n, m = ℓ·μ mod n) ---- */

static int decrypt(const orc_key *k, const mpz_t c, mpz_t m) {
    if (!k->has_priv) return fail("decrypt requested without private key material");
    if (mpz_cmp_ui(c, 1) < 0 || mpz_cmp(c, k->n2) >= 0) return fail("decrypt: ciphertext out of range");
    mpz_t g, u;
    mpz_init(g);
    mpz_init(u);
    mpz_gcd(g, c, k->n);
    if (mpz_cmp_ui(g, 1) != 0) {
        mpz_clear(g);
        mpz_clear(u);
        return fail("decrypt: ciphertext not coprime to modulus");
    }
    mpz_powm(u, c, k->lambda, k->n2); /* he.cpp:112 */
    mpz_sub_ui(u, u, 1);
    mpz_tdiv_q(u, u, k->n);
    mpz_mul(m, u, k->mu);
    mpz_tdiv_r(m, m, k->n);
    mpz_clear(g);
    mpz_clear(u);
    return 0;
}

int orc_decrypt(const orc_key *k, const uint32_t *c, uint32_t *out_m) {
    mpz_t zc, m;
    mpz_init(zc);
    mpz_init(m);
    imp(zc, c, 2 * k->nw);
    int rc = decrypt(k, zc, m);
    if (!rc) rc = exp_words(out_m, k->nw, m);
    mpz_clear(zc);
    mpz_clear(m);
    return rc;
}

/* CRT decryption (the GPU algorithm, K3), restated here so the
 * tests can show it is bit-identical to the reference's non-CRT decrypt:
 *   m_p = L_p(c^(p−1) mod p²)·h_p mod p,  h_p = L_p((1+n)^(p−1) mod p²)^−1 mod p
 *   m   = m_q + q·((m_p − m_q)·q^−1 mod p)                                       */
int orc_decrypt_crt(const orc_key *k, const uint32_t *c, uint32_t *out_m) {
    if (!k->has_priv) return fail("decrypt requested without private key material");
    mpz_t zc, p2, q2, u, hp, hq, mp, mq, t, g;
    mpz_init(zc); mpz_init(p2); mpz_init(q2); mpz_init(u); mpz_init(hp); mpz_init(hq);
    mpz_init(mp); mpz_init(mq); mpz_init(t); mpz_init(g);
    imp(zc, c, 2 * k->nw);
    mpz_mul(p2, k->p, k->p);
    mpz_mul(q2, k->q, k->q);
    const mpz_srcptr prime[2] = {k->p, k->q};
    const mpz_srcptr sq[2] = {p2, q2};
    mpz_ptr h[2] = {hp, hq};
    mpz_ptr mm[2] = {mp, mq};
    for (int i = 0; i < 2; ++i) {
        mpz_sub_ui(t, prime[i], 1);
        mpz_add_ui(g, k->n, 1);
        mpz_powm(u, g, t, sq[i]);
        mpz_sub_ui(u, u, 1);
        mpz_tdiv_q(u, u, prime[i]);
        mpz_invert(h[i], u, prime[i]);
        mpz_powm(u, zc, t, sq[i]);
        mpz_sub_ui(u, u, 1);
        mpz_tdiv_q(u, u, prime[i]);
        mpz_mul(u, u, h[i]);
        mpz_mod(mm[i], u, prime[i]);
    }
    mpz_invert(t, k->q, k->p);
    mpz_sub(u, mp, mq);
    mpz_mul(u, u, t);
    mpz_mod(u, u, k->p);
    mpz_mul(u, u, k->q);
    mpz_add(u, u, mq);
    int rc = exp_words(out_m, k->nw, u);
    mpz_clear(zc); mpz_clear(p2); mpz_clear(q2); mpz_clear(u); mpz_clear(hp); mpz_clear(hq);
    mpz_clear(mp); mpz_clear(mq); mpz_clear(t); mpz_clear(g);
    return rc;
}

/* decrypt_histogram (enc_scalar) + decrypt_slot: secure_processor.cpp:679-719, :734-738.
 * Slot == 1 decodes to 0.0 and is not counted. */
int orc_decrypt_slots(const orc_key *k, const uint32_t *cts, size_t count, unsigned scale,
                      double *out, uint64_t *decryptions) {
    if (!k->has_priv) return fail("decrypt requested without private key material");
    mpz_t zc, m;
    mpz_init(zc);
    mpz_init(m);
    uint32_t *mbuf = malloc(k->nw * 4);
    int rc = 0;
    for (size_t i = 0; i < count && !rc; ++i) {
        imp(zc, cts + i * 2 * k->nw, 2 * k->nw);
        if (mpz_cmp_ui(zc, 1) == 0) {
            out[i] = 0.0;
            continue;
        }
        *decryptions += 1;
        rc = decrypt(k, zc, m);
        if (!rc) rc = exp_words(mbuf, k->nw, m);
        if (!rc) out[i] = orc_decode_fixed(k, mbuf, scale);
    }
    free(mbuf);
    mpz_clear(zc);
    mpz_clear(m);
    return rc;
}

/* ---- exact integer-sum oracle ----
 * Decrypted slot value for large configs without Paillier: Σ q_i (int64
 * fixed-point) per slot, decoded with mpz_get_d truncation semantics. */
double orc_decode_int_sum(const orc_key *k, const int64_t *terms, size_t count, unsigned scale) {
    mpz_t s, t;
    mpz_init_set_ui(s, 0);
    mpz_init(t);
    for (size_t i = 0; i < count; ++i) {
        mpz_set_si(t, (long)terms[i]);
        mpz_add(s, s, t);
    }
    mpz_mod(s, s, k->n); /* the plaintext the decryption produces */
    uint32_t *buf = malloc(k->nw * 4);
    exp_words(buf, k->nw, s);
    double d = orc_decode_fixed(k, buf, scale);
    free(buf);
    mpz_clear(s);
    mpz_clear(t);
    return d;
}

/* ---- integer-sum histograms, the checker at scale ----
 * accumulate_rows (secure_processor.cpp:587-620) followed by decrypt_histogram
 * (:679-719), expressed on plaintexts: Dec(∏ c_i) = Σ m_i mod n with m_i ≡ q_i
 * (mod n), so slot (node i, feature f, bin b, G/H) decrypts to (Σ q) mod n,
 * decoded by decode_fixed (he.cpp:138-143, orc_decode_fixed).  q: 2·n_samples
 * signed fixed-point integers (G, H interleaved); bins: n_features columns of
 * n_samples; the frontier as node offsets + rows.  Empty slots stay the
 * trivial zero (decrypt_slot → 0.0, uncounted).  out: N·J·K·2 doubles in the
 * slot layout 2(f·K+b)+{G,H} per node; *adds += Σ max(count − 1, 0) (fold_into
 * :724-732); *decs += non-empty slots.  Features run in parallel (OpenMP):
 * they write disjoint slots. */
int orc_intsum_hist(const orc_key *k, const int64_t *q, uint32_t n_samples, const uint16_t *bins, uint32_t J,
                    const uint32_t *node_offsets, uint32_t N, const uint32_t *rows, uint32_t K, unsigned scale,
                    double *out, uint64_t *adds, uint64_t *decs) {
    const size_t slots = (size_t)N * J * K * 2;
    __int128 *sum = calloc(slots ? slots : 1, sizeof(__int128));
    uint32_t *cnt = calloc(slots ? slots : 1, sizeof(uint32_t));
    if (!sum || !cnt) {
        free(sum);
        free(cnt);
        return fail("intsum_hist: out of memory");
    }
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (uint32_t f = 0; f < J; ++f) {
        const uint16_t *col = bins + (size_t)f * n_samples;
        for (uint32_t i = 0; i < N; ++i) {
            const size_t base = ((size_t)i * J + f) * K * 2;
            for (uint32_t t = node_offsets[i]; t < node_offsets[i + 1]; ++t) {
                const uint32_t row = rows[t];
                if (row >= n_samples || col[row] >= K) {
                    bad = 1;
                    continue;
                }
                const size_t s = base + 2 * (size_t)col[row];
                sum[s] += q[2 * (size_t)row];
                sum[s + 1] += q[2 * (size_t)row + 1];
                cnt[s]++;
                cnt[s + 1]++;
            }
        }
    }
    if (bad) {
        free(sum);
        free(cnt);
        return fail("bin index out of range in accumulate");
    }
    uint64_t a = 0, d = 0;
#pragma omp parallel reduction(+ : a, d)
    {
        mpz_t m;
        mpz_init(m);
        uint32_t *buf = malloc(k->nw * 4);
#pragma omp for schedule(static)
        for (size_t s = 0; s < slots; ++s) {
            if (!cnt[s]) {
                out[s] = 0.0;
                continue;
            }
            a += cnt[s] - 1;
            d += 1;
            const __int128 v = sum[s];
            const unsigned __int128 mag = v < 0 ? (unsigned __int128)(-v) : (unsigned __int128)v;
            const uint64_t w[2] = {(uint64_t)mag, (uint64_t)(mag >> 64)};
            mpz_import(m, 2, -1, 8, 0, 0, w);
            if (v < 0) mpz_neg(m, m);
            mpz_mod(m, m, k->n); /* the plaintext the decryption produces */
            exp_words(buf, k->nw, m);
            out[s] = orc_decode_fixed(k, buf, scale);
        }
        free(buf);
        mpz_clear(m);
    }
    *adds += a;
    *decs += d;
    free(sum);
    free(cnt);
    return 0;
}
