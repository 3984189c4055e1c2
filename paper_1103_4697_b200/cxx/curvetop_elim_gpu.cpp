// Drop-in replacement for the reference's elimination TU (/root/reference/proj/src/elim.cpp).
//
// Defines every symbol elim.cpp defines, with the reference's exact signatures
// (proj/include/curvetop/elim.hpp:13-45, upoly.hpp:92), on top of the C ABI of
// libctg.so (include/ctg.h).  A curvetop build swaps elim.cpp for this file and
// links libctg.so; callers (lift.cpp, bisolve.cpp, pipeline.cpp, realroots.cpp,
// connect.cpp, bipoly.cpp and the tests) are unchanged.  See INTEGRATION.md.
//
//   resultant         -> ctg_resultant         (GPU: multi-modular, elim.cpp:95-136)
//   yun_squarefree    -> ctg_yun_squarefree    (GPU: modular Yun + certificate, elim.cpp:138-165)
//   gcd_univariate    -> ctg_gcd_univariate    (GPU: modular gcd + certificate, elim.cpp:80-93)
//   square_free_part  -> ctg_square_free_part  (GPU, elim.cpp:204-210)
//   SquareFreeFactorization::reconstruct, multiplicity_at: same semantics as elim.cpp:74-78,
//     167-176 (products / sign tests on the host, gcds on the GPU)
//   gcd_bivariate     -> ctg_gcd_bivariate     (GPU, elim.cpp:178-202: contents by modular
//     univariate gcds, a modular coprimality probe, and Brown's modular bivariate gcd with
//     an exactness certificate when the primitive parts share a factor)
//
// Status codes map to the reference's exceptions: CTG_PRECONDITION -> PreconditionError,
// anything else -> Error (there is no CPU fallback: a CUDA failure throws).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctg.h"
#include "curvetop/elim.hpp"
#include "curvetop/realroots.hpp"

namespace curvetop {
namespace {

[[noreturn]] void raise(ctg_status st, const char* what) {
  std::string msg = ctg_last_error();
  if (msg.empty()) msg = what;
  if (st == CTG_PRECONDITION) throw PreconditionError(msg);
  throw Error(msg);
}

void check(ctg_status st, const char* what) {
  if (st != CTG_OK) raise(st, what);
}

// CTG_DEVICES="0,1,2,3" shards every resultant's primes over those GPUs (ctg_opts.n_devices,
// one NCCL all-gather of the residues); unset = one device, the library default.
const ctg_opts* resultant_opts() {
  static ctg_opts opts{};
  static std::vector<int32_t> devs;
  static const ctg_opts* o = [] () -> const ctg_opts* {
    const char* e = std::getenv("CTG_DEVICES");
    if (!e || !*e) return nullptr;
    for (const char* c = e; *c;) {
      char* end = nullptr;
      const long v = std::strtol(c, &end, 10);
      if (end == c) break;
      devs.push_back(static_cast<int32_t>(v));
      c = (*end == ',') ? end + 1 : end;
    }
    if (devs.size() < 2) return nullptr;
    opts.device = devs[0];
    opts.verify = 1;
    opts.n_devices = static_cast<int32_t>(devs.size());
    opts.devices = devs.data();
    return &opts;
  }();
  return o;
}

// Little-endian u32 limbs <-> GMP's limbs.  mpz_import / mpz_export with 4-byte words take a
// generic path (~0.5 GB/s: 1.2 ms / 2 ms for R at d30, 871 coefficients of 7,813 bits); GMP 6's
// limb access is a copy (mp_limb_t is 64-bit little-endian on x86-64, so the u32 words ARE the
// limb bytes), which matters because the reference API converts R three times per curve.
static_assert(sizeof(mp_limb_t) == 8, "64-bit GMP limbs expected");
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "little-endian limb layout expected");
void append_limbs(mpz_srcptr z, std::vector<uint32_t>& out) {
  const size_t n = mpz_size(z);
  const mp_limb_t* d = mpz_limbs_read(z);
  const size_t base = out.size();
  size_t words = 2 * n;
  if (n && (d[n - 1] >> 32) == 0) --words;  // top half-limb empty
  out.resize(base + words);
  std::memcpy(out.data() + base, d, 4 * words);
}

BigInt from_limbs(int sign, const uint32_t* limbs, size_t n) {
  BigInt v;
  while (n && limbs[n - 1] == 0) --n;
  if (n) {
    const size_t nl = (n + 1) / 2;
    mp_limb_t* d = mpz_limbs_write(v.get_mpz_t(), static_cast<mp_size_t>(nl));
    d[nl - 1] = 0;
    std::memcpy(d, limbs, 4 * n);
    mpz_limbs_finish(v.get_mpz_t(), sign < 0 ? -static_cast<mp_size_t>(nl) : static_cast<mp_size_t>(nl));
  }
  return v;
}

// mpz -> sign + little-endian u32 limbs (CSR).
struct Limbs {
  std::vector<int8_t> sign;
  std::vector<uint32_t> off{0};
  std::vector<uint32_t> limbs;
  void push(const BigInt& v) {
    const int s = sgn(v);
    sign.push_back(static_cast<int8_t>(s));
    if (s != 0) append_limbs(v.get_mpz_t(), limbs);
    off.push_back(static_cast<uint32_t>(limbs.size()));
  }
};

struct BiMarshal {
  std::vector<int32_t> dx, dy;
  Limbs L;
  ctg_bipoly view{};
  explicit BiMarshal(const BivariatePolynomial& f) {
    for (const auto& [e, c] : f.terms()) {
      dx.push_back(e.first);
      dy.push_back(e.second);
      L.push(c);
    }
    view.n_terms = static_cast<int32_t>(dx.size());
    view.dx = dx.data();
    view.dy = dy.data();
    view.sign = L.sign.data();
    view.limb_off = L.off.data();
    view.limbs = L.limbs.data();
  }
};

struct UniMarshal {
  Limbs L;
  ctg_upoly view{};
  explicit UniMarshal(const UnivariatePolynomial& p) {
    size_t words = 0;
    for (const auto& c : p.coeffs()) words += 2 * mpz_size(c.get_mpz_t());
    L.limbs.reserve(words);
    L.sign.reserve(p.coeffs().size());
    L.off.reserve(p.coeffs().size() + 1);
    for (const auto& c : p.coeffs()) L.push(c);
    view.n_coeffs = static_cast<int32_t>(p.coeffs().size());
    view.sign = L.sign.data();
    view.limb_off = L.off.data();
    view.limbs = L.limbs.data();
  }
};

UnivariatePolynomial take(ctg_upoly_buf& b) {
  std::vector<BigInt> c(static_cast<size_t>(b.n_coeffs));
  for (int i = 0; i < b.n_coeffs; ++i)
    c[i] = from_limbs(b.sign[i], b.limbs + b.limb_off[i], b.limb_off[i + 1] - b.limb_off[i]);
  ctg_upoly_free(&b);
  return UnivariatePolynomial(std::move(c));
}

UnivariatePolynomial power(const UnivariatePolynomial& p, int k) {
  UnivariatePolynomial r = UnivariatePolynomial::constant(1);
  while (k-- > 0) r = r * p;
  return r;
}

}  // namespace

UnivariatePolynomial SquareFreeFactorization::reconstruct() const {
  UnivariatePolynomial r = UnivariatePolynomial::constant(unit);
  for (const auto& f : factors) r = r * power(f.poly, f.multiplicity);
  return r;
}

UnivariatePolynomial gcd_univariate(const UnivariatePolynomial& p, const UnivariatePolynomial& q) {
  UniMarshal a(p), b(q);
  ctg_upoly_buf out{};
  check(ctg_gcd_univariate(&a.view, &b.view, &out, nullptr), "gcd_univariate");
  return take(out);
}

UnivariatePolynomial resultant(const BivariatePolynomial& p, const BivariatePolynomial& q, Var eliminated) {
  BiMarshal a(p), b(q);
  ctg_upoly_buf out{};
  check(ctg_resultant(&a.view, &b.view, eliminated == Var::X ? 1 : 0, &out, resultant_opts()), "resultant");
  return take(out);
}

SquareFreeFactorization yun_squarefree(const UnivariatePolynomial& p) {
  UniMarshal a(p);
  ctg_sqf_buf out{};
  check(ctg_yun_squarefree(&a.view, &out, nullptr), "yun_squarefree");
  SquareFreeFactorization sf;
  sf.unit = from_limbs(out.unit_sign, out.unit_limbs, static_cast<size_t>(out.unit_nlimbs));
  for (int i = 0; i < out.n_factors; ++i) {
    ctg_upoly_buf& b = out.factors[i];
    std::vector<BigInt> c(static_cast<size_t>(b.n_coeffs));
    for (int j = 0; j < b.n_coeffs; ++j)
      c[j] = from_limbs(b.sign[j], b.limbs + b.limb_off[j], b.limb_off[j + 1] - b.limb_off[j]);
    sf.factors.push_back({UnivariatePolynomial(std::move(c)), out.mult[i]});
  }
  ctg_sqf_free(&out);
  return sf;
}

UnivariatePolynomial square_free_part(const UnivariatePolynomial& p) {
  UniMarshal a(p);
  ctg_upoly_buf out{};
  check(ctg_square_free_part(&a.view, &out, nullptr), "square_free_part");
  return take(out);
}

int multiplicity_at(const SquareFreeFactorization& sf, const AlgebraicNumber& a) {
  for (const auto& f : sf.factors) {
    UnivariatePolynomial g = gcd_univariate(f.poly, a.poly());
    if (g.degree() < 1) continue;
    const int slo = g.sign_at(a.interval().lo().to_rational());
    const int shi = g.sign_at(a.interval().hi().to_rational());
    if (slo * shi < 0) return f.multiplicity;
  }
  return 0;
}

BivariatePolynomial gcd_bivariate(const BivariatePolynomial& f, const BivariatePolynomial& g) {
  if (f.is_zero() && g.is_zero()) throw PreconditionError("gcd_bivariate: both inputs zero");
  if (f.is_zero()) return g;
  if (g.is_zero()) return f;
  BiMarshal mf(f), mg(g);
  ctg_bipoly_buf out{};
  check(ctg_gcd_bivariate(&mf.view, &mg.view, &out, nullptr), "gcd_bivariate");
  BivariatePolynomial::TermMap t;
  for (int i = 0; i < out.n_terms; ++i)
    t[{out.dx[i], out.dy[i]}] = from_limbs(out.sign[i], out.limbs + out.limb_off[i], out.limb_off[i + 1] - out.limb_off[i]);
  ctg_bipoly_free(&out);
  return BivariatePolynomial(std::move(t));
}

}  // namespace curvetop
