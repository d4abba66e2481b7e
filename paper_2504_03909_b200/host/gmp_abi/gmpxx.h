// Minimal `mpz_class` / `gmp_randclass` restatement of the gmpxx C++ wrapper
// (GMP 6.3.0 semantics) covering exactly what the reference uses (SURVEY.md
// §8c "Shim surface"): construction from builtin integers, + - * / % (the
// division operators truncate: mpz_tdiv_q / mpz_tdiv_r, as in gmpxx), <<=,
// >> (mpz_fdiv_q_2exp, as in gmpxx), &, comparisons, abs, get_str, get_d,
// get_mpz_t; gmp_randclass(gmp_randinit_mt) with seed / get_z_bits /
// get_z_range (mpz_urandomb / mpz_urandomm).  No expression templates: each
// operator materialises its result, which is value-identical.
//
// Used to compile the C++ adapter against the reference's headers (which
// include <gmpxx.h>) and, as test infrastructure, the read-only reference
// sources into oracle/_ref/.
#pragma once
#include <gmp.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

class mpz_class {
public:
    mpz_class() { mpz_init(mp_); }
    mpz_class(const mpz_class &o) { mpz_init_set(mp_, o.mp_); }
    mpz_class(mpz_class &&o) noexcept {
        mpz_init(mp_);
        mpz_swap(mp_, o.mp_);
    }
    explicit mpz_class(mpz_srcptr z) { mpz_init_set(mp_, z); }
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    mpz_class(T v) {
        if constexpr (std::is_signed_v<T>)
            mpz_init_set_si(mp_, static_cast<long>(v));
        else
            mpz_init_set_ui(mp_, static_cast<unsigned long>(v));
    }
    explicit mpz_class(const std::string &s, int base = 0) {
        if (mpz_init_set_str(mp_, s.c_str(), base) != 0) {
            mpz_clear(mp_);
            throw std::invalid_argument("mpz_set_str");
        }
    }
    ~mpz_class() { mpz_clear(mp_); }

    mpz_class &operator=(const mpz_class &o) {
        if (this != &o) mpz_set(mp_, o.mp_);
        return *this;
    }
    mpz_class &operator=(mpz_class &&o) noexcept {
        mpz_swap(mp_, o.mp_);
        return *this;
    }
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
    mpz_class &operator=(T v) {
        if constexpr (std::is_signed_v<T>)
            mpz_set_si(mp_, static_cast<long>(v));
        else
            mpz_set_ui(mp_, static_cast<unsigned long>(v));
        return *this;
    }

    mpz_ptr get_mpz_t() { return mp_; }
    mpz_srcptr get_mpz_t() const { return mp_; }

    double get_d() const { return mpz_get_d(mp_); }
    std::string get_str(int base = 10) const {
        char *s = mpz_get_str(nullptr, base, mp_);
        std::string out(s);
        std::free(s);
        return out;
    }

    mpz_class &operator+=(const mpz_class &o) { mpz_add(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator-=(const mpz_class &o) { mpz_sub(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator*=(const mpz_class &o) { mpz_mul(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator/=(const mpz_class &o) { mpz_tdiv_q(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator%=(const mpz_class &o) { mpz_tdiv_r(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator&=(const mpz_class &o) { mpz_and(mp_, mp_, o.mp_); return *this; }
    mpz_class &operator<<=(mp_bitcnt_t k) { mpz_mul_2exp(mp_, mp_, k); return *this; }
    mpz_class &operator>>=(mp_bitcnt_t k) { mpz_fdiv_q_2exp(mp_, mp_, k); return *this; }
    mpz_class operator-() const {
        mpz_class r;
        mpz_neg(r.mp_, mp_);
        return r;
    }

private:
    mpz_t mp_;
};

#define SFXB_SHIM_BINOP(op, fn)                                                                    \
    inline mpz_class operator op(const mpz_class &a, const mpz_class &b) {                        \
        mpz_class r;                                                                               \
        fn(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t());                                           \
        return r;                                                                                  \
    }                                                                                              \
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>                      \
    inline mpz_class operator op(const mpz_class &a, T b) {                                        \
        return a op mpz_class(b);                                                                  \
    }                                                                                              \
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>                      \
    inline mpz_class operator op(T a, const mpz_class &b) {                                        \
        return mpz_class(a) op b;                                                                  \
    }
SFXB_SHIM_BINOP(+, mpz_add)
SFXB_SHIM_BINOP(-, mpz_sub)
SFXB_SHIM_BINOP(*, mpz_mul)
SFXB_SHIM_BINOP(/, mpz_tdiv_q)
SFXB_SHIM_BINOP(%, mpz_tdiv_r)
SFXB_SHIM_BINOP(&, mpz_and)
#undef SFXB_SHIM_BINOP

inline mpz_class operator<<(const mpz_class &a, mp_bitcnt_t k) {
    mpz_class r;
    mpz_mul_2exp(r.get_mpz_t(), a.get_mpz_t(), k);
    return r;
}
inline mpz_class operator>>(const mpz_class &a, mp_bitcnt_t k) {
    mpz_class r;
    mpz_fdiv_q_2exp(r.get_mpz_t(), a.get_mpz_t(), k);
    return r;
}

inline int sfxb_shim_cmp(const mpz_class &a, const mpz_class &b) {
    return mpz_cmp(a.get_mpz_t(), b.get_mpz_t());
}
#define SFXB_SHIM_CMP(op)                                                                          \
    inline bool operator op(const mpz_class &a, const mpz_class &b) {                             \
        return sfxb_shim_cmp(a, b) op 0;                                                           \
    }                                                                                              \
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>                      \
    inline bool operator op(const mpz_class &a, T b) {                                             \
        return sfxb_shim_cmp(a, mpz_class(b)) op 0;                                                \
    }                                                                                              \
    template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>                      \
    inline bool operator op(T a, const mpz_class &b) {                                             \
        return sfxb_shim_cmp(mpz_class(a), b) op 0;                                                \
    }
SFXB_SHIM_CMP(==)
SFXB_SHIM_CMP(!=)
SFXB_SHIM_CMP(<)
SFXB_SHIM_CMP(<=)
SFXB_SHIM_CMP(>)
SFXB_SHIM_CMP(>=)
#undef SFXB_SHIM_CMP

inline mpz_class abs(const mpz_class &a) {
    mpz_class r;
    mpz_abs(r.get_mpz_t(), a.get_mpz_t());
    return r;
}

class gmp_randclass {
public:
    explicit gmp_randclass(void (*init)(gmp_randstate_t)) { init(state_); }
    gmp_randclass(const gmp_randclass &) = delete;
    gmp_randclass &operator=(const gmp_randclass &) = delete;
    ~gmp_randclass() { gmp_randclear(state_); }

    void seed(const mpz_class &s) { gmp_randseed(state_, s.get_mpz_t()); }
    void seed(unsigned long s) { gmp_randseed_ui(state_, s); }
    mpz_class get_z_bits(mp_bitcnt_t bits) {
        mpz_class r;
        mpz_urandomb(r.get_mpz_t(), state_, bits);
        return r;
    }
    mpz_class get_z_range(const mpz_class &n) {
        mpz_class r;
        mpz_urandomm(r.get_mpz_t(), state_, n.get_mpz_t());
        return r;
    }
    __gmp_randstate_struct *get_randstate_t() { return state_; }

private:
    gmp_randstate_t state_;
};
