/* TEST INFRASTRUCTURE ONLY (oracle/_ref build). Minimal declarations of the GMP C ABI.
 *
 * This container ships the GMP runtime (/usr/lib/x86_64-linux-gnu/libgmp.so.10, GMP 6.3) but
 * not its development headers. The reference core (/root/reference/proj/core, via
 * rational.hpp:3 / highprec.hpp:3) includes <gmpxx.h>; this header and ./gmpxx.h declare just
 * the part of the public GMP ABI the reference sources and the gmpxx shim use, so the reference
 * can be compiled unmodified from its own sources and linked against the runtime library.
 *
 * The struct layouts are GMP's documented public types (mpz_t / mpq_t / mpf_t, x86-64 LP64);
 * the functions are the library's exported __gmp{z,q,f}_* entry points, reached through the
 * usual mp{z,q,f}_* names as in the real header.
 */
#ifndef PF_SHIM_GMP_H
#define PF_SHIM_GMP_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef long mp_exp_t;
typedef unsigned long mp_bitcnt_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

typedef struct {
  __mpz_struct _mp_num;
  __mpz_struct _mp_den;
} __mpq_struct;
typedef __mpq_struct mpq_t[1];
typedef __mpq_struct* mpq_ptr;
typedef const __mpq_struct* mpq_srcptr;

typedef struct {
  int _mp_prec;
  int _mp_size;
  mp_exp_t _mp_exp;
  mp_limb_t* _mp_d;
} __mpf_struct;
typedef __mpf_struct mpf_t[1];
typedef __mpf_struct* mpf_ptr;
typedef const __mpf_struct* mpf_srcptr;

#define mpq_numref(Q) (&((Q)->_mp_num))
#define mpq_denref(Q) (&((Q)->_mp_den))
#define mpz_sgn(Z) ((Z)->_mp_size < 0 ? -1 : (Z)->_mp_size > 0)
#define mpq_sgn(Q) ((Q)->_mp_num._mp_size < 0 ? -1 : (Q)->_mp_num._mp_size > 0)
#define mpf_sgn(F) ((F)->_mp_size < 0 ? -1 : (F)->_mp_size > 0)

/* ---- integers ---- */
#define mpz_init __gmpz_init
#define mpz_init_set __gmpz_init_set
#define mpz_init_set_si __gmpz_init_set_si
#define mpz_init_set_ui __gmpz_init_set_ui
#define mpz_init_set_d __gmpz_init_set_d
#define mpz_init_set_str __gmpz_init_set_str
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_si __gmpz_set_si
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_d __gmpz_set_d
#define mpz_set_str __gmpz_set_str
#define mpz_swap __gmpz_swap
#define mpz_get_si __gmpz_get_si
#define mpz_get_ui __gmpz_get_ui
#define mpz_get_d __gmpz_get_d
#define mpz_get_str __gmpz_get_str
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_mul __gmpz_mul
#define mpz_mul_si __gmpz_mul_si
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_cmp __gmpz_cmp
#define mpz_cmp_si __gmpz_cmp_si
#define mpz_cmp_d __gmpz_cmp_d
#define mpz_pow_ui __gmpz_pow_ui
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_scan1 __gmpz_scan1
#define mpz_fits_slong_p __gmpz_fits_slong_p
#define mpz_gcd __gmpz_gcd

void mpz_init(mpz_ptr);
void mpz_init_set(mpz_ptr, mpz_srcptr);
void mpz_init_set_si(mpz_ptr, long);
void mpz_init_set_ui(mpz_ptr, unsigned long);
void mpz_init_set_d(mpz_ptr, double);
int mpz_init_set_str(mpz_ptr, const char*, int);
void mpz_clear(mpz_ptr);
void mpz_set(mpz_ptr, mpz_srcptr);
void mpz_set_si(mpz_ptr, long);
void mpz_set_ui(mpz_ptr, unsigned long);
void mpz_set_d(mpz_ptr, double);
int mpz_set_str(mpz_ptr, const char*, int);
void mpz_swap(mpz_ptr, mpz_ptr);
long mpz_get_si(mpz_srcptr);
unsigned long mpz_get_ui(mpz_srcptr);
double mpz_get_d(mpz_srcptr);
char* mpz_get_str(char*, int, mpz_srcptr);
size_t mpz_sizeinbase(mpz_srcptr, int);
void mpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_mul_si(mpz_ptr, mpz_srcptr, long);
void mpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_neg(mpz_ptr, mpz_srcptr);
void mpz_abs(mpz_ptr, mpz_srcptr);
int mpz_cmp(mpz_srcptr, mpz_srcptr);
int mpz_cmp_si(mpz_srcptr, long);
int mpz_cmp_d(mpz_srcptr, double);
void mpz_pow_ui(mpz_ptr, mpz_srcptr, unsigned long);
void mpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
mp_bitcnt_t mpz_scan1(mpz_srcptr, mp_bitcnt_t);
int mpz_fits_slong_p(mpz_srcptr);
void mpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);

/* ---- rationals ---- */
#define mpq_init __gmpq_init
#define mpq_clear __gmpq_clear
#define mpq_set __gmpq_set
#define mpq_set_si __gmpq_set_si
#define mpq_set_ui __gmpq_set_ui
#define mpq_set_d __gmpq_set_d
#define mpq_set_z __gmpq_set_z
#define mpq_set_str __gmpq_set_str
#define mpq_swap __gmpq_swap
#define mpq_canonicalize __gmpq_canonicalize
#define mpq_get_d __gmpq_get_d
#define mpq_get_str __gmpq_get_str
#define mpq_add __gmpq_add
#define mpq_sub __gmpq_sub
#define mpq_mul __gmpq_mul
#define mpq_div __gmpq_div
#define mpq_neg __gmpq_neg
#define mpq_abs __gmpq_abs
#define mpq_cmp __gmpq_cmp
#define mpq_cmp_si __gmpq_cmp_si
#define mpq_equal __gmpq_equal

void mpq_init(mpq_ptr);
void mpq_clear(mpq_ptr);
void mpq_set(mpq_ptr, mpq_srcptr);
void mpq_set_si(mpq_ptr, long, unsigned long);
void mpq_set_ui(mpq_ptr, unsigned long, unsigned long);
void mpq_set_d(mpq_ptr, double);
void mpq_set_z(mpq_ptr, mpz_srcptr);
int mpq_set_str(mpq_ptr, const char*, int);
void mpq_swap(mpq_ptr, mpq_ptr);
void mpq_canonicalize(mpq_ptr);
double mpq_get_d(mpq_srcptr);
char* mpq_get_str(char*, int, mpq_srcptr);
void mpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void mpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void mpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
void mpq_div(mpq_ptr, mpq_srcptr, mpq_srcptr);
void mpq_neg(mpq_ptr, mpq_srcptr);
void mpq_abs(mpq_ptr, mpq_srcptr);
int mpq_cmp(mpq_srcptr, mpq_srcptr);
int mpq_cmp_si(mpq_srcptr, long, unsigned long);
int mpq_equal(mpq_srcptr, mpq_srcptr);

/* ---- floats ---- */
#define mpf_init2 __gmpf_init2
#define mpf_init_set __gmpf_init_set
#define mpf_clear __gmpf_clear
#define mpf_get_default_prec __gmpf_get_default_prec
#define mpf_get_prec __gmpf_get_prec
#define mpf_set_prec __gmpf_set_prec
#define mpf_set __gmpf_set
#define mpf_set_d __gmpf_set_d
#define mpf_set_si __gmpf_set_si
#define mpf_set_ui __gmpf_set_ui
#define mpf_set_q __gmpf_set_q
#define mpf_set_z __gmpf_set_z
#define mpf_set_str __gmpf_set_str
#define mpf_swap __gmpf_swap
#define mpf_get_d __gmpf_get_d
#define mpf_get_si __gmpf_get_si
#define mpf_get_str __gmpf_get_str
#define mpf_add __gmpf_add
#define mpf_sub __gmpf_sub
#define mpf_mul __gmpf_mul
#define mpf_div __gmpf_div
#define mpf_neg __gmpf_neg
#define mpf_abs __gmpf_abs
#define mpf_sqrt __gmpf_sqrt
#define mpf_pow_ui __gmpf_pow_ui
#define mpf_mul_2exp __gmpf_mul_2exp
#define mpf_div_2exp __gmpf_div_2exp
#define mpf_cmp __gmpf_cmp
#define mpf_cmp_d __gmpf_cmp_d
#define mpf_cmp_si __gmpf_cmp_si
#define mpf_floor __gmpf_floor
#define mpf_ceil __gmpf_ceil
#define mpf_trunc __gmpf_trunc

void mpf_init2(mpf_ptr, mp_bitcnt_t);
void mpf_init_set(mpf_ptr, mpf_srcptr);
void mpf_clear(mpf_ptr);
mp_bitcnt_t mpf_get_default_prec(void);
mp_bitcnt_t mpf_get_prec(mpf_srcptr);
void mpf_set_prec(mpf_ptr, mp_bitcnt_t);
void mpf_set(mpf_ptr, mpf_srcptr);
void mpf_set_d(mpf_ptr, double);
void mpf_set_si(mpf_ptr, long);
void mpf_set_ui(mpf_ptr, unsigned long);
void mpf_set_q(mpf_ptr, mpq_srcptr);
void mpf_set_z(mpf_ptr, mpz_srcptr);
int mpf_set_str(mpf_ptr, const char*, int);
void mpf_swap(mpf_ptr, mpf_ptr);
double mpf_get_d(mpf_srcptr);
long mpf_get_si(mpf_srcptr);
char* mpf_get_str(char*, mp_exp_t*, int, size_t, mpf_srcptr);
void mpf_add(mpf_ptr, mpf_srcptr, mpf_srcptr);
void mpf_sub(mpf_ptr, mpf_srcptr, mpf_srcptr);
void mpf_mul(mpf_ptr, mpf_srcptr, mpf_srcptr);
void mpf_div(mpf_ptr, mpf_srcptr, mpf_srcptr);
void mpf_neg(mpf_ptr, mpf_srcptr);
void mpf_abs(mpf_ptr, mpf_srcptr);
void mpf_sqrt(mpf_ptr, mpf_srcptr);
void mpf_pow_ui(mpf_ptr, mpf_srcptr, unsigned long);
void mpf_mul_2exp(mpf_ptr, mpf_srcptr, mp_bitcnt_t);
void mpf_div_2exp(mpf_ptr, mpf_srcptr, mp_bitcnt_t);
int mpf_cmp(mpf_srcptr, mpf_srcptr);
int mpf_cmp_d(mpf_srcptr, double);
int mpf_cmp_si(mpf_srcptr, long);
void mpf_floor(mpf_ptr, mpf_srcptr);
void mpf_ceil(mpf_ptr, mpf_srcptr);
void mpf_trunc(mpf_ptr, mpf_srcptr);

#ifdef __cplusplus
}
#endif

#endif /* PF_SHIM_GMP_H */
