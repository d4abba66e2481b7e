/* Minimal C declarations for the subset of GMP 6.3.0 that the host code
 * calls: the C++ adapter and wire codec (paper_2504_03909_b200/host), the
 * device library's root inversion (dlopen of the same runtime), and — as test
 * infrastructure — the reference sources compiled into oracle/_ref and the
 * oracle restatement (SURVEY.md §8c "Shim surface").  The image ships the GMP *runtime*
 * (`/usr/lib/x86_64-linux-gnu/libgmp.so.10`, GMP 6.3.0) but not its headers,
 * so this file restates the public ABI: struct layouts (`__mpz_struct`,
 * `__gmp_randstate_struct`) and the exported `__gmpz_*` / `__gmp_*` entry
 * points, with the usual `mpz_*` -> `__gmpz_*` name macros.
 */
#ifndef SFXB_ORACLE_GMP_SHIM_H
#define SFXB_ORACLE_GMP_SHIM_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long int mp_limb_t; /* 64-bit limbs on x86-64 */
typedef long int mp_limb_signed_t;
typedef unsigned long int mp_bitcnt_t;
typedef long int mp_size_t;
typedef long int mp_exp_t;

typedef struct {
    int _mp_alloc;
    int _mp_size;
    mp_limb_t *_mp_d;
} __mpz_struct;

typedef __mpz_struct mpz_t[1];
typedef __mpz_struct *mpz_ptr;
typedef const __mpz_struct *mpz_srcptr;
typedef mp_limb_t *mp_ptr;
typedef const mp_limb_t *mp_srcptr;

typedef enum { GMP_RAND_ALG_DEFAULT = 0, GMP_RAND_ALG_LC = GMP_RAND_ALG_DEFAULT } gmp_randalg_t;

typedef struct {
    mpz_t _mp_seed;
    gmp_randalg_t _mp_alg;
    union {
        void *_mp_lc;
    } _mp_algdata;
} __gmp_randstate_struct;
typedef __gmp_randstate_struct gmp_randstate_t[1];

#define mpz_init __gmpz_init
#define mpz_init2 __gmpz_init2
#define mpz_init_set __gmpz_init_set
#define mpz_init_set_si __gmpz_init_set_si
#define mpz_init_set_ui __gmpz_init_set_ui
#define mpz_init_set_str __gmpz_init_set_str
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_si __gmpz_set_si
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_str __gmpz_set_str
#define mpz_swap __gmpz_swap
#define mpz_add __gmpz_add
#define mpz_add_ui __gmpz_add_ui
#define mpz_sub __gmpz_sub
#define mpz_sub_ui __gmpz_sub_ui
#define mpz_mul __gmpz_mul
#define mpz_mul_si __gmpz_mul_si
#define mpz_mul_ui __gmpz_mul_ui
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_tdiv_qr __gmpz_tdiv_qr
#define mpz_tdiv_q_2exp __gmpz_tdiv_q_2exp
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_tdiv_r_2exp __gmpz_tdiv_r_2exp
#define mpz_mod __gmpz_mod
#define mpz_and __gmpz_and
#define mpz_cmp __gmpz_cmp
#define mpz_cmp_si __gmpz_cmp_si
#define mpz_cmp_ui __gmpz_cmp_ui
#define mpz_cmpabs __gmpz_cmpabs
#define mpz_fdiv_r_2exp __gmpz_fdiv_r_2exp
#define mpz_abs __gmpz_abs
#define mpz_neg __gmpz_neg
#define mpz_get_d __gmpz_get_d
#define mpz_get_si __gmpz_get_si
#define mpz_get_str __gmpz_get_str
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_size __gmpz_size
#define mpz_import __gmpz_import
#define mpz_export __gmpz_export
#define mpz_gcd __gmpz_gcd
#define mpz_setbit __gmpz_setbit
#define mpz_probab_prime_p __gmpz_probab_prime_p
#define mpz_powm __gmpz_powm
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_nextprime __gmpz_nextprime
#define mpz_lcm __gmpz_lcm
#define mpz_invert __gmpz_invert
#define mpz_urandomb __gmpz_urandomb
#define mpz_urandomm __gmpz_urandomm
#define mpz_limbs_read __gmpz_limbs_read
#define mpz_limbs_write __gmpz_limbs_write
#define mpz_limbs_finish __gmpz_limbs_finish
#define gmp_randinit_mt __gmp_randinit_mt
#define gmp_randinit_set __gmp_randinit_set
#define gmp_randseed __gmp_randseed
#define gmp_randseed_ui __gmp_randseed_ui
#define gmp_randclear __gmp_randclear

void mpz_init(mpz_ptr);
void mpz_init2(mpz_ptr, mp_bitcnt_t);
void mpz_init_set(mpz_ptr, mpz_srcptr);
void mpz_init_set_si(mpz_ptr, long);
void mpz_init_set_ui(mpz_ptr, unsigned long);
int mpz_init_set_str(mpz_ptr, const char *, int);
void mpz_clear(mpz_ptr);
void mpz_set(mpz_ptr, mpz_srcptr);
void mpz_set_si(mpz_ptr, long);
void mpz_set_ui(mpz_ptr, unsigned long);
int mpz_set_str(mpz_ptr, const char *, int);
void mpz_swap(mpz_ptr, mpz_ptr);
void mpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void mpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void mpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_mul_si(mpz_ptr, mpz_srcptr, long);
void mpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void mpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void mpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_tdiv_qr(mpz_ptr, mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_tdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void mpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void mpz_tdiv_r_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void mpz_mod(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_and(mpz_ptr, mpz_srcptr, mpz_srcptr);
int mpz_cmp(mpz_srcptr, mpz_srcptr);
int mpz_cmp_si(mpz_srcptr, long);
int mpz_cmp_ui(mpz_srcptr, unsigned long);
int mpz_cmpabs(mpz_srcptr, mpz_srcptr);
void mpz_fdiv_r_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void mpz_abs(mpz_ptr, mpz_srcptr);
void mpz_neg(mpz_ptr, mpz_srcptr);
double mpz_get_d(mpz_srcptr);
long mpz_get_si(mpz_srcptr);
char *mpz_get_str(char *, int, mpz_srcptr);
size_t mpz_sizeinbase(mpz_srcptr, int);
size_t mpz_size(mpz_srcptr);
void mpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void *);
void *mpz_export(void *, size_t *, int, size_t, int, size_t, mpz_srcptr);
void mpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_setbit(mpz_ptr, mp_bitcnt_t);
int mpz_probab_prime_p(mpz_srcptr, int);
void mpz_powm(mpz_ptr, mpz_srcptr, mpz_srcptr, mpz_srcptr);
void mpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
void mpz_nextprime(mpz_ptr, mpz_srcptr);
void mpz_lcm(mpz_ptr, mpz_srcptr, mpz_srcptr);
int mpz_invert(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_urandomb(mpz_ptr, gmp_randstate_t, mp_bitcnt_t);
void mpz_urandomm(mpz_ptr, gmp_randstate_t, mpz_srcptr);
mp_srcptr mpz_limbs_read(mpz_srcptr);
mp_ptr mpz_limbs_write(mpz_ptr, mp_size_t);
void mpz_limbs_finish(mpz_ptr, mp_size_t);
void gmp_randinit_mt(gmp_randstate_t);
void gmp_randinit_set(gmp_randstate_t, const __gmp_randstate_struct *);
void gmp_randseed(gmp_randstate_t, mpz_srcptr);
void gmp_randseed_ui(gmp_randstate_t, unsigned long);
void gmp_randclear(gmp_randstate_t);

#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)

#ifdef __cplusplus
}
#endif

#endif
