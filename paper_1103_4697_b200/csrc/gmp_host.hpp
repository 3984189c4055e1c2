// Host-side GMP entry points (libgmp.so.10, the reference's own dependency: proj/CMakeLists.txt:12-14).
//
// Used only for the host normalisation steps the reference API requires around the GPU
// work: polynomial contents (integer gcds of coefficients), exact divisions by a content,
// and the certificate arithmetic on leading coefficients.  The image ships the shared
// library without headers, so the handful of symbols used are declared here (GMP 6 ABI).
#pragma once
#include <stddef.h>
#include <stdint.h>

extern "C" {
typedef struct {
  int _mp_alloc;
  int _mp_size;
  unsigned long* _mp_d;
} ctg_mpz_struct;
void __gmpz_init(ctg_mpz_struct*);
void __gmpz_clear(ctg_mpz_struct*);
void __gmpz_import(ctg_mpz_struct*, size_t, int, size_t, int, size_t, const void*);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, const ctg_mpz_struct*);
void __gmpz_gcd(ctg_mpz_struct*, const ctg_mpz_struct*, const ctg_mpz_struct*);
void __gmpz_divexact(ctg_mpz_struct*, const ctg_mpz_struct*, const ctg_mpz_struct*);
void __gmpz_set(ctg_mpz_struct*, const ctg_mpz_struct*);
int __gmpz_divisible_p(const ctg_mpz_struct*, const ctg_mpz_struct*);
void __gmpz_tdiv_r(ctg_mpz_struct*, const ctg_mpz_struct*, const ctg_mpz_struct*);
void __gmpz_mul(ctg_mpz_struct*, const ctg_mpz_struct*, const ctg_mpz_struct*);
size_t __gmpz_sizeinbase(const ctg_mpz_struct*, int);
// GMP 6 limb access (64-bit little-endian limbs on x86-64: the u32 words are their bytes)
unsigned long* __gmpz_limbs_write(ctg_mpz_struct*, long);
void __gmpz_limbs_finish(ctg_mpz_struct*, long);
}
