// The subset of the GMP C API the host layer's exact arithmetic uses (Rational, the moment solve,
// the theta bound). The reference computes its coefficients with GMP (rational.hpp:3, mpq_class /
// mpf_class); this image ships the GMP runtime (libgmp.so.10) but not its headers, so the public
// ABI types and entry points are declared here and the library is linked by its soname.
#pragma once

#include <cstddef>

extern "C" {

typedef unsigned long mp_limb_t;
typedef long mp_exp_t;
typedef unsigned long mp_bitcnt_t;

struct pf_mpz {
  int alloc;
  int size;
  mp_limb_t* d;
};
struct pf_mpq {
  pf_mpz num, den;
};
struct pf_mpf {
  int prec;
  int size;
  mp_exp_t exp;
  mp_limb_t* d;
};

void __gmpq_init(pf_mpq*);
void __gmpq_clear(pf_mpq*);
void __gmpq_set(pf_mpq*, const pf_mpq*);
void __gmpq_set_si(pf_mpq*, long, unsigned long);
void __gmpq_set_d(pf_mpq*, double);
int __gmpq_set_str(pf_mpq*, const char*, int);
void __gmpq_canonicalize(pf_mpq*);
void __gmpq_add(pf_mpq*, const pf_mpq*, const pf_mpq*);
void __gmpq_sub(pf_mpq*, const pf_mpq*, const pf_mpq*);
void __gmpq_mul(pf_mpq*, const pf_mpq*, const pf_mpq*);
void __gmpq_div(pf_mpq*, const pf_mpq*, const pf_mpq*);
void __gmpq_neg(pf_mpq*, const pf_mpq*);
void __gmpq_abs(pf_mpq*, const pf_mpq*);
int __gmpq_cmp(const pf_mpq*, const pf_mpq*);
int __gmpq_equal(const pf_mpq*, const pf_mpq*);
double __gmpq_get_d(const pf_mpq*);
char* __gmpq_get_str(char*, int, const pf_mpq*);
size_t __gmpz_sizeinbase(const pf_mpz*, int);

void __gmpf_init2(pf_mpf*, mp_bitcnt_t);
void __gmpf_clear(pf_mpf*);
void __gmpf_set(pf_mpf*, const pf_mpf*);
void __gmpf_set_q(pf_mpf*, const pf_mpq*);
void __gmpf_set_d(pf_mpf*, double);
void __gmpf_set_ui(pf_mpf*, unsigned long);
void __gmpf_add(pf_mpf*, const pf_mpf*, const pf_mpf*);
void __gmpf_sub(pf_mpf*, const pf_mpf*, const pf_mpf*);
void __gmpf_mul(pf_mpf*, const pf_mpf*, const pf_mpf*);
void __gmpf_div(pf_mpf*, const pf_mpf*, const pf_mpf*);
void __gmpf_pow_ui(pf_mpf*, const pf_mpf*, unsigned long);
int __gmpf_cmp(const pf_mpf*, const pf_mpf*);
double __gmpf_get_d(const pf_mpf*);

}  // extern "C"
