/* TEST INFRASTRUCTURE ONLY (oracle build shim).
 *
 * Minimal declarations of the GMP 6 ABI exported by the system's
 * libgmp.so.10 (6.3.0).  The image ships the shared library but not its
 * development headers, and the reference (/root/reference/proj) needs
 * <gmp.h>/<gmpxx.h> to compile (proj/CMakeLists.txt:12-14).  This header
 * declares exactly the subset the reference sources and our oracle driver
 * call; the struct layouts match GMP 6 on x86-64 (mp_limb_t = unsigned long).
 *
 * Nothing in the product (paper_1103_4697_b200/) includes this file.
 */
#ifndef CTG_ORACLE_SHIM_GMP_H
#define CTG_ORACLE_SHIM_GMP_H

#include <stddef.h>
#include <stdio.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;

typedef struct {
  int _mp_alloc;
  int _mp_size;
  mp_limb_t* _mp_d;
} __mpz_struct;

typedef struct {
  __mpz_struct _mp_num;
  __mpz_struct _mp_den;
} __mpq_struct;

typedef __mpz_struct mpz_t[1];
typedef __mpq_struct mpq_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;
typedef __mpq_struct* mpq_ptr;
typedef const __mpq_struct* mpq_srcptr;

/* ---- integers ---- */
void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
void __gmpz_init_set_d(mpz_ptr, double);
int __gmpz_init_set_str(mpz_ptr, const char*, int);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
void __gmpz_set_d(mpz_ptr, double);
int __gmpz_set_str(mpz_ptr, const char*, int);
void __gmpz_swap(mpz_ptr, mpz_ptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_addmul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_submul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_cdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_tdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_qr(mpz_ptr, mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_fdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_cdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_divexact(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mod(mpz_ptr, mpz_srcptr, mpz_srcptr);
unsigned long __gmpz_fdiv_ui(mpz_srcptr, unsigned long);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
int __gmpz_cmpabs(mpz_srcptr, mpz_srcptr);
void __gmpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_lcm(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_invert(mpz_ptr, mpz_srcptr, mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
mp_bitcnt_t __gmpz_scan1(mpz_srcptr, mp_bitcnt_t);
void __gmpz_sqrtrem(mpz_ptr, mpz_ptr, mpz_srcptr);
void __gmpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
void __gmpz_pow_ui(mpz_ptr, mpz_srcptr, unsigned long);
char* __gmpz_get_str(char*, int, mpz_srcptr);
double __gmpz_get_d(mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
unsigned long __gmpz_get_ui(mpz_srcptr);
int __gmpz_fits_slong_p(mpz_srcptr);
void __gmpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void*);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, mpz_srcptr);
size_t __gmpz_size(mpz_srcptr);
const mp_limb_t* __gmpz_limbs_read(mpz_srcptr);
mp_limb_t* __gmpz_limbs_write(mpz_ptr, mp_size_t);
void __gmpz_limbs_finish(mpz_ptr, mp_size_t);

/* ---- rationals ---- */
void __gmpq_init(mpq_ptr);
void __gmpq_clear(mpq_ptr);
void __gmpq_set(mpq_ptr, mpq_srcptr);
void __gmpq_set_z(mpq_ptr, mpz_srcptr);
void __gmpq_set_si(mpq_ptr, long, unsigned long);
void __gmpq_set_d(mpq_ptr, double);
void __gmpq_canonicalize(mpq_ptr);
void __gmpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_div(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_neg(mpq_ptr, mpq_srcptr);
void __gmpq_abs(mpq_ptr, mpq_srcptr);
void __gmpq_swap(mpq_ptr, mpq_ptr);
int __gmpq_cmp(mpq_srcptr, mpq_srcptr);
int __gmpq_equal(mpq_srcptr, mpq_srcptr);
double __gmpq_get_d(mpq_srcptr);
char* __gmpq_get_str(char*, int, mpq_srcptr);

#ifdef __cplusplus
}
#endif

/* Public names used by the reference (raw calls at elim.cpp:41, upoly.cpp:62,
 * 80, 97, numeric.cpp, bipoly.cpp, bisolve.cpp, pipeline.cpp). */
#define mpz_init __gmpz_init
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_mul __gmpz_mul
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_cmp __gmpz_cmp
#define mpz_gcd __gmpz_gcd
#define mpz_lcm __gmpz_lcm
#define mpz_invert __gmpz_invert
#define mpz_tdiv_qr __gmpz_tdiv_qr
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_fdiv_q __gmpz_fdiv_q
#define mpz_cdiv_q __gmpz_cdiv_q
#define mpz_fdiv_ui __gmpz_fdiv_ui
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_cdiv_q_2exp __gmpz_cdiv_q_2exp
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_divexact __gmpz_divexact
#define mpz_mod __gmpz_mod
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_scan1 __gmpz_scan1
#define mpz_sqrtrem __gmpz_sqrtrem
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_pow_ui __gmpz_pow_ui
#define mpz_get_str __gmpz_get_str
#define mpz_set_str __gmpz_set_str
#define mpz_get_d __gmpz_get_d
#define mpz_get_si __gmpz_get_si
#define mpz_import __gmpz_import
#define mpz_export __gmpz_export
#define mpz_size __gmpz_size
#define mpz_limbs_read __gmpz_limbs_read
#define mpz_limbs_write __gmpz_limbs_write
#define mpz_limbs_finish __gmpz_limbs_finish
#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)
#define mpq_numref(q) (&((q)->_mp_num))
#define mpq_denref(q) (&((q)->_mp_den))
#define mpq_canonicalize __gmpq_canonicalize
#define mpq_sgn(q) ((q)->_mp_num._mp_size < 0 ? -1 : (q)->_mp_num._mp_size > 0)

#endif /* CTG_ORACLE_SHIM_GMP_H */
