// Host-side number theory for plan construction: prime selection, roots of
// unity, coefficient / degree bounds and the CRT constants.  None of this is
// per-coefficient work on the hot path: it is O(P) to O(P * limbs(M)) setup,
// cached per (N, P) prime set (see api.cu).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace ctg {

using Big = std::vector<uint32_t>;  // little-endian magnitude, trimmed

bool is_prime_u32(uint32_t n);
uint32_t pow_mod_u32(uint32_t a, uint64_t e, uint32_t p);
uint32_t inv_mod_u32(uint32_t a, uint32_t p);
// Primitive root modulo the prime p.
uint32_t primitive_root(uint32_t p);

// All primes p = c*N + 1 in (lo, hi), in decreasing order, as many as
// needed so that sum(log2 p) >= need_bits.  Deterministic: the list for a
// given (N, hi, lo) is always a prefix of the same sequence.  The resultant uses
// hi = kResPrimeMax (three-product reductions), the gcd / Yun path hi = 2^31.
std::vector<uint32_t> select_primes(uint32_t N, double need_bits, uint64_t hi = (1ull << 31), uint64_t lo = (1ull << 30));

// Smallest N = r * 2^a >= D with r in {1, 3, 5, 7} (the NTT sizes the
// interpolation kernel supports).  Returns r and a through the pointers.
uint32_t choose_ntt_size(uint32_t D, uint32_t* r, uint32_t* a);

void big_trim(Big& a);
Big big_mul_u32(const Big& a, uint32_t b);
// a / b for a u32 divisor, remainder returned through rem.
Big big_div_u32(const Big& a, uint32_t b, uint32_t* rem);
uint32_t big_mod_u32(const uint32_t* limbs, int n, uint32_t p);
int big_cmp(const Big& a, const Big& b);
Big big_add(const Big& a, const Big& b);
Big big_sub(const Big& a, const Big& b);  // requires a >= b
Big big_mul_small(const uint32_t* limbs, int n, uint32_t s);

// Upper bound on log2(value) of a nonzero magnitude (within ~1e-12 bits).
double log2_upper(const uint32_t* limbs, int n);
// log2(sum 2^x_i), rounded up; -inf for an empty list.
double log2_sum_upper(const std::vector<double>& xs);

Big big_mul(const Big& a, const Big& b);
// gcd of magnitudes (binary gcd on 64-bit words).
Big big_gcd(const Big& a, const Big& b);
// a / b for an exact divisor b != 0 (throws if the remainder is nonzero).
Big big_divexact(const Big& a, const Big& b);
// g <- gcd(g, c) for u32 limbs c[0..n) (g nonzero); thread-local GMP scratch, no allocation
// unless g changes.  Returns true if it changed.
bool big_gcd_update(Big& g, const uint32_t* c, int n);
// a / c for c dividing a (not checked): writes the quotient's limbs to q (room for na - |c| + 4
// limbs) and returns their count.  Thread-local GMP scratch: no allocation per call.
size_t big_divexact_to(const uint32_t* a, int na, const Big& c, uint32_t* q);
// a mod p for a u32 modulus.
inline uint32_t big_mod(const Big& a, uint32_t p) { return big_mod_u32(a.data(), static_cast<int>(a.size()), p); }
inline bool big_is_one(const Big& a) { return a.size() == 1 && a[0] == 1; }
double big_log2(const Big& a);  // upper bound, -inf for zero

// Signed big integer (sign-magnitude) for summing repeated input terms.
struct SBig {
  int sign = 0;  // -1, 0, +1
  Big mag;
};
void sbig_add_inplace(SBig& acc, int sign, const uint32_t* limbs, int n);

}  // namespace ctg
