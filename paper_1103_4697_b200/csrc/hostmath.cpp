#include <cstring>
#include "hostmath.hpp"

#include "gmp_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <tuple>
#include <mutex>
#include <stdexcept>

namespace ctg {

uint32_t pow_mod_u32(uint32_t a, uint64_t e, uint32_t p) {
  uint64_t r = 1 % p, b = a % p;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return static_cast<uint32_t>(r);
}

uint32_t inv_mod_u32(uint32_t a, uint32_t p) { return pow_mod_u32(a, p - 2, p); }

bool is_prime_u32(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t q : {2u, 3u, 5u, 7u, 11u, 13u, 17u, 19u, 23u, 29u, 31u, 37u}) {
    if (n % q == 0) return n == q;
  }
  uint32_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++s;
  }
  // Bases {2, 7, 61} are deterministic for n < 4,759,123,141.
  for (uint32_t a : {2u, 7u, 61u}) {
    if (a % n == 0) continue;
    uint64_t x = pow_mod_u32(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = x * x % n;
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

uint32_t primitive_root(uint32_t p) {
  std::vector<uint32_t> fac;
  uint32_t m = p - 1;
  for (uint32_t q = 2; static_cast<uint64_t>(q) * q <= m; ++q) {
    if (m % q == 0) {
      fac.push_back(q);
      while (m % q == 0) m /= q;
    }
  }
  if (m > 1) fac.push_back(m);
  for (uint32_t g = 2; g < p; ++g) {
    bool ok = true;
    for (uint32_t q : fac)
      if (pow_mod_u32(g, (p - 1) / q, p) == 1) {
        ok = false;
        break;
      }
    if (ok) return g;
  }
  throw std::runtime_error("primitive_root: none found");
}

// Cached, lazily extended sequence of the primes c*N + 1 in (lo, hi), decreasing.
static uint32_t prime_seq_at(uint32_t N, uint64_t hi, uint64_t lo, size_t i) {
  static std::mutex mu;
  // (N, hi, lo) -> (primes, next c)
  static std::map<std::tuple<uint32_t, uint64_t, uint64_t>, std::pair<std::vector<uint32_t>, uint64_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto& entry = cache[{N, hi, lo}];
  auto& list = entry.first;
  if (list.empty() && entry.second == 0) entry.second = (hi - 2) / N;
  while (i >= list.size()) {
    bool found = false;
    while (entry.second > 0) {
      uint64_t c = entry.second--;
      uint64_t p = c * N + 1;
      if (p >= hi) continue;
      if (p <= lo) {
        entry.second = 0;
        break;
      }
      if (is_prime_u32(static_cast<uint32_t>(p))) {
        list.push_back(static_cast<uint32_t>(p));
        found = true;
        break;
      }
    }
    if (!found) return 0u;
  }
  return list[i];
}

std::vector<uint32_t> select_primes(uint32_t N, double need_bits, uint64_t hi, uint64_t lo) {
  std::vector<uint32_t> out;
  double bits = 0;
  for (size_t i = 0; bits < need_bits; ++i) {
    const uint32_t p = prime_seq_at(N, hi, lo, i);
    if (!p) throw std::runtime_error("select_primes: ran out of primes p = c*N+1 in the window");
    out.push_back(p);
    bits += std::log2(static_cast<double>(p));
  }
  return out;
}

uint32_t choose_ntt_size(uint32_t D, uint32_t* r_out, uint32_t* a_out) {
  uint32_t best = 0, br = 1, ba = 0;
  for (uint32_t r : {1u, 3u, 5u, 7u}) {
    uint32_t a = 0;
    uint64_t n = r;
    while (n < D) {
      n <<= 1;
      ++a;
    }
    if (best == 0 || n < best) {
      best = static_cast<uint32_t>(n);
      br = r;
      ba = a;
    }
  }
  *r_out = br;
  *a_out = ba;
  return best;
}

void big_trim(Big& a) {
  while (!a.empty() && a.back() == 0) a.pop_back();
}

Big big_mul_u32(const Big& a, uint32_t b) {
  Big r(a.size() + 1);
  uint64_t carry = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    uint64_t t = static_cast<uint64_t>(a[i]) * b + carry;
    r[i] = static_cast<uint32_t>(t);
    carry = t >> 32;
  }
  r[a.size()] = static_cast<uint32_t>(carry);
  big_trim(r);
  return r;
}

Big big_mul_small(const uint32_t* limbs, int n, uint32_t s) {
  Big a(limbs, limbs + n);
  return big_mul_u32(a, s);
}

// Division of a 64-bit x = r 2^32 + limb (r < d) by a 32-bit d with a precomputed
// reciprocal mu = floor((2^64 - 1) / d): q = hi64(x mu) is at most 2 below floor(x / d), so
// two conditional corrections give the exact quotient (no hardware 64-bit division per limb).
namespace {
struct Div32 {
  uint64_t d, mu;
  explicit Div32(uint32_t dv) : d(dv), mu(~0ull / dv) {}
  uint64_t div(uint64_t x, uint64_t* rem) const {
    uint64_t q = static_cast<uint64_t>((static_cast<unsigned __int128>(x) * mu) >> 64);
    uint64_t r = x - q * d;
    if (r >= d) {
      r -= d;
      ++q;
    }
    if (r >= d) {
      r -= d;
      ++q;
    }
    *rem = r;
    return q;
  }
};
}  // namespace

Big big_div_u32(const Big& a, uint32_t b, uint32_t* rem) {
  Big q(a.size());
  const Div32 D(b);
  uint64_t r = 0;
  for (size_t i = a.size(); i-- > 0;) q[i] = static_cast<uint32_t>(D.div((r << 32) | a[i], &r));
  if (rem) *rem = static_cast<uint32_t>(r);
  big_trim(q);
  return q;
}

uint32_t big_mod_u32(const uint32_t* limbs, int n, uint32_t p) {
  const Div32 D(p);
  uint64_t r = 0;
  for (int i = n - 1; i >= 0; --i) D.div((r << 32) | limbs[i], &r);
  return static_cast<uint32_t>(r);
}

int big_cmp(const Big& a, const Big& b) {
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;)
    if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

Big big_add(const Big& a, const Big& b) {
  const Big& x = a.size() >= b.size() ? a : b;
  const Big& y = a.size() >= b.size() ? b : a;
  Big r(x.size() + 1);
  uint64_t c = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    uint64_t t = static_cast<uint64_t>(x[i]) + (i < y.size() ? y[i] : 0) + c;
    r[i] = static_cast<uint32_t>(t);
    c = t >> 32;
  }
  r[x.size()] = static_cast<uint32_t>(c);
  big_trim(r);
  return r;
}

Big big_sub(const Big& a, const Big& b) {
  Big r(a.size());
  int64_t br = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    int64_t t = static_cast<int64_t>(a[i]) - (i < b.size() ? b[i] : 0) - br;
    br = t < 0;
    r[i] = static_cast<uint32_t>(t + (br << 32));
  }
  big_trim(r);
  return r;
}

double log2_upper(const uint32_t* limbs, int n) {
  while (n > 0 && limbs[n - 1] == 0) --n;
  if (n == 0) return -std::numeric_limits<double>::infinity();
  // value < (top two limbs + 1) * 2^(32*(n-2))
  double top = static_cast<double>(limbs[n - 1]);
  int shift = 32 * (n - 1);
  if (n >= 2) {
    top = top * 4294967296.0 + static_cast<double>(limbs[n - 2]);
    shift = 32 * (n - 2);
  }
  top += 1.0;
  return (std::log2(top) + shift) * (1 + 1e-14) + 1e-12;
}

double log2_sum_upper(const std::vector<double>& xs) {
  double mx = -std::numeric_limits<double>::infinity();
  for (double x : xs) mx = std::max(mx, x);
  if (!std::isfinite(mx)) return mx;
  double s = 0;
  for (double x : xs)
    if (std::isfinite(x)) s += std::exp2(x - mx);
  return (mx + std::log2(s)) * (1 + 1e-14) + 1e-12;
}

// Multiplication, gcd and exact division on the host go through GMP (subquadratic; the
// reference's own dependency) -- they serve contents, primitive parts and certificates.
static_assert(sizeof(unsigned long) == 8 && __BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__,
              "64-bit little-endian GMP limbs expected");
namespace {
struct Mpz {
  ctg_mpz_struct z;
  Mpz() { __gmpz_init(&z); }
  // u32 magnitude <-> GMP limbs by copy (mpz_import / mpz_export with 4-byte words take a
  // generic ~0.5 GB/s path; a 1,000-limb content gcd spent most of its time converting)
  explicit Mpz(const Big& a) {
    __gmpz_init(&z);
    size_t n = a.size();
    while (n && a[n - 1] == 0) --n;
    if (n) {
      const size_t nl = (n + 1) / 2;
      unsigned long* d = __gmpz_limbs_write(&z, static_cast<long>(nl));
      d[nl - 1] = 0;
      std::memcpy(d, a.data(), 4 * n);
      __gmpz_limbs_finish(&z, static_cast<long>(nl));
    }
  }
  ~Mpz() { __gmpz_clear(&z); }
  Big big() const {  // magnitude
    const size_t n = static_cast<size_t>(z._mp_size < 0 ? -z._mp_size : z._mp_size);
    Big r(2 * n);
    if (n) std::memcpy(r.data(), z._mp_d, 8 * n);
    big_trim(r);
    return r;
  }
  bool is_zero() const { return z._mp_size == 0; }
};
}  // namespace

Big big_mul(const Big& a, const Big& b) {
  if (a.empty() || b.empty()) return Big();
  Mpz x(a), y(b), r;
  __gmpz_mul(&r.z, &x.z, &y.z);
  return r.big();
}

double big_log2(const Big& a) { return log2_upper(a.data(), static_cast<int>(a.size())); }

Big big_gcd(const Big& a, const Big& b) {
  Mpz x(a), y(b), r;
  __gmpz_gcd(&r.z, &x.z, &y.z);
  return r.big();
}

Big big_divexact(const Big& a, const Big& b) {
  if (b.empty()) throw std::runtime_error("big_divexact: zero divisor");
  if (a.empty()) return Big();
  Mpz x(a), y(b), r, q;
  __gmpz_tdiv_r(&r.z, &x.z, &y.z);
  if (!r.is_zero()) throw std::runtime_error("big_divexact: inexact division");
  __gmpz_divexact(&q.z, &x.z, &y.z);
  return q.big();
}

bool big_gcd_update(Big& g, const uint32_t* c, int n) {
  thread_local Mpz x, y, r;
  thread_local Big yc;
  while (n && c[n - 1] == 0) --n;
  if (!n) return false;  // gcd(g, 0) = g
  if (yc != g) {
    Mpz t(g);
    __gmpz_set(&y.z, &t.z);
    yc = g;
  }
  const size_t nl = (static_cast<size_t>(n) + 1) / 2;
  unsigned long* d = __gmpz_limbs_write(&x.z, static_cast<long>(nl));
  d[nl - 1] = 0;
  std::memcpy(d, c, 4 * static_cast<size_t>(n));
  __gmpz_limbs_finish(&x.z, static_cast<long>(nl));
  if (__gmpz_divisible_p(&x.z, &y.z)) return false;  // the common case once g is the content
  __gmpz_gcd(&r.z, &y.z, &x.z);
  if (r.z._mp_size == y.z._mp_size &&
      std::memcmp(r.z._mp_d, y.z._mp_d, 8 * static_cast<size_t>(r.z._mp_size < 0 ? -r.z._mp_size : r.z._mp_size)) == 0)
    return false;
  g = r.big();
  yc = g;
  __gmpz_set(&y.z, &r.z);
  return true;
}

size_t big_divexact_to(const uint32_t* a, int na, const Big& c, uint32_t* q) {
  // per-thread scratch (no allocation once warm): x = a, y = c (re-read only when c changes)
  thread_local Mpz x, y, r;
  thread_local Big yc;
  if (c.empty()) throw std::runtime_error("big_divexact_to: zero divisor");
  while (na && a[na - 1] == 0) --na;
  if (!na) return 0;
  if (yc != c) {
    Mpz t(c);
    __gmpz_set(&y.z, &t.z);
    yc = c;
  }
  const size_t nl = (static_cast<size_t>(na) + 1) / 2;
  unsigned long* d = __gmpz_limbs_write(&x.z, static_cast<long>(nl));
  d[nl - 1] = 0;
  std::memcpy(d, a, 4 * static_cast<size_t>(na));
  __gmpz_limbs_finish(&x.z, static_cast<long>(nl));
  __gmpz_divexact(&r.z, &x.z, &y.z);
  size_t n = 2 * static_cast<size_t>(r.z._mp_size < 0 ? -r.z._mp_size : r.z._mp_size);
  if (n) std::memcpy(q, r.z._mp_d, 4 * n);
  while (n && q[n - 1] == 0) --n;
  return n;
}

void sbig_add_inplace(SBig& acc, int sign, const uint32_t* limbs, int n) {
  Big b(limbs, limbs + n);
  big_trim(b);
  if (b.empty() || sign == 0) return;
  if (acc.sign == 0) {
    acc.sign = sign;
    acc.mag = b;
    return;
  }
  if (acc.sign == sign) {
    acc.mag = big_add(acc.mag, b);
    return;
  }
  int c = big_cmp(acc.mag, b);
  if (c == 0) {
    acc.sign = 0;
    acc.mag.clear();
  } else if (c > 0) {
    acc.mag = big_sub(acc.mag, b);
  } else {
    acc.mag = big_sub(b, acc.mag);
    acc.sign = sign;
  }
}

}  // namespace ctg
