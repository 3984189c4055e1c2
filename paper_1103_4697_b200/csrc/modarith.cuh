// Montgomery arithmetic modulo 31-bit primes p in (2^30, 2^31), R = 2^32.
//
// Every residue on the device is kept fully reduced in [0, p).  A "two-product
// reduction" a*b + c*d (a, b, c, d < p) costs two IMAD.WIDE, one IMAD and one
// IMAD.WIDE (the reduction) plus one IADD/IMNMX pair for the final correction:
//   T = a*b + c*d < 2p^2 < 2^63,  m = lo(T) * (-p^-1) mod 2^32,
//   t = (T + m*p) / 2^32 < 2p   ->  t - p if t >= p.
// Host and device share these definitions (host code builds tables with them).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define CTG_HD __host__ __device__ __forceinline__
#else
#define CTG_HD inline
#endif

namespace ctg {

struct Mod {
  uint32_t p;     // the prime
  uint32_t pneg;  // -p^{-1} mod 2^32
  uint32_t r2;    // R^2 mod p (to enter Montgomery form)
  uint32_t one;   // R mod p (Montgomery form of 1)
};

CTG_HD uint32_t csub(uint32_t r, uint32_t p) {
  // r in [0, 2p) -> [0, p).  min(r, r - p) as unsigned: r - p wraps when r < p.
  uint32_t s = r - p;
  return s < r ? s : r;
}

CTG_HD uint32_t redc(uint64_t T, uint32_t p, uint32_t pneg) {
  uint32_t m = static_cast<uint32_t>(T) * pneg;
  uint64_t t = T + static_cast<uint64_t>(m) * p;
  return csub(static_cast<uint32_t>(t >> 32), p);
}

// a*b*R^-1 mod p
CTG_HD uint32_t mmul(uint32_t a, uint32_t b, const Mod& M) {
  return redc(static_cast<uint64_t>(a) * b, M.p, M.pneg);
}

// (a*b + c*d)*R^-1 mod p
CTG_HD uint32_t mmul2(uint32_t a, uint32_t b, uint32_t c, uint32_t d, const Mod& M) {
  return redc(static_cast<uint64_t>(a) * b + static_cast<uint64_t>(c) * d, M.p, M.pneg);
}

// (a*b + c*d + e*f)*R^-1 mod p.  Requires p < 2^30.4 (kResPrimeMax): then
// T < 3p^2 < 2^62.4, T + m p < 2^64 and the REDC output is < 1.99 p (one correction).
CTG_HD uint32_t mmul3(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f, const Mod& M) {
  return redc(static_cast<uint64_t>(a) * b + static_cast<uint64_t>(c) * d + static_cast<uint64_t>(e) * f, M.p,
              M.pneg);
}
constexpr uint32_t kResPrimeMax = 1416000000u;  // < 2^30.4 = 1,416,810,830

CTG_HD uint32_t madd(uint32_t a, uint32_t b, uint32_t p) { return csub(a + b, p); }
CTG_HD uint32_t msub(uint32_t a, uint32_t b, uint32_t p) {
  uint32_t s = a - b;
  return s > a ? s + p : s;  // borrow -> add p back
}
CTG_HD uint32_t mneg(uint32_t a, uint32_t p) { return a ? p - a : 0u; }

CTG_HD uint32_t to_mont(uint32_t a, const Mod& M) { return mmul(a, M.r2, M); }
CTG_HD uint32_t from_mont(uint32_t a, const Mod& M) { return redc(static_cast<uint64_t>(a), M.p, M.pneg); }

// a^e in Montgomery form (a in Montgomery form).
CTG_HD uint32_t mpow(uint32_t a, uint64_t e, const Mod& M) {
  uint32_t r = M.one;
  while (e) {
    if (e & 1) r = mmul(r, a, M);
    a = mmul(a, a, M);
    e >>= 1;
  }
  return r;
}

// Inverse by Fermat (a in Montgomery form, nonzero).
CTG_HD uint32_t minv(uint32_t a, const Mod& M) { return mpow(a, static_cast<uint64_t>(M.p) - 2, M); }

// Build the constants for a prime p (host or device).
CTG_HD Mod make_mod(uint32_t p) {
  Mod M;
  M.p = p;
  // Newton iteration for p^{-1} mod 2^32 (p odd).
  uint32_t inv = p;  // correct to 3 bits
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  M.pneg = 0u - inv;
  uint64_t r = (static_cast<uint64_t>(1) << 32) % p;
  M.one = static_cast<uint32_t>(r);
  M.r2 = static_cast<uint32_t>((r * r) % p);
  return M;
}

}  // namespace ctg
