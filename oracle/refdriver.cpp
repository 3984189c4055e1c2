// TEST INFRASTRUCTURE ONLY: driver around the reference implementation
// (curvetop, /root/reference/proj) compiled unmodified into oracle/_ref/.
// It is the parity oracle for the GPU path and the CPU baseline of bench.py
// ("cpu_baseline.kind": "reference").  Never linked into the product.
//
// Commands (all big integers in hex, sign-prefixed, as GMP get_str(16)):
//   refdriver gen dense D B SEED        -> print f = dense(D, B, SEED)
//   refdriver gen sheared K SEED        -> print f = sheared(K, SEED)
//   refdriver batch < requests          -> one JSON line per request (ops below)
//   refdriver elim_cases                -> JSON lines: the reference test_elim.cpp random
//                                          inputs (seeds 21-24) with reference outputs
//   refdriver time_res KIND A B SEED REPS [yun]
//                                       -> JSON line: wall seconds of resultant(f, f_y, Y)
//                                          (+ yun_squarefree(R) when "yun" is given)
//   refdriver time_ctx KIND A B SEED REPS [q]
//                                       -> JSON line: wall seconds of the reference's own
//                                          caller CurveContext(f) (lift.cpp:59-68: R = res(f,
//                                          f_y) + Yun(R)) and, with "q", of resultant_q() +
//                                          q_factorization() (lift.cpp:76-101: gcd_bivariate,
//                                          Q, Yun(Q)).  Built twice: against the reference's
//                                          elim.cpp (refdriver) and against the GPU drop-in TU
//                                          (refdriver_gpu) -- the same caller, both libraries.
//
// Request format (text):
//   OP <resultant_y|resultant_x|resultant_fy|sylvester_y|yun|gcd|sqfp|gcd_bivariate|curve_q>
//   B <nterms>  followed by nterms lines "dx dy hexcoeff"        (bivariate operand)
//   U <ncoeffs> followed by ncoeffs lines "hexcoeff" low->high   (univariate operand)
//   END
#include <chrono>
#include <cstdio>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "curvetop/bipoly.hpp"
#include "curvetop/elim.hpp"
#include "curvetop/lift.hpp"
#include "oracles.hpp"

using namespace curvetop;

namespace {

std::string hex(const BigInt& v) { return v.get_str(16); }

BigInt from_hex(const std::string& s) {
  BigInt v;
  if (mpz_set_str(v.get_mpz_t(), s.c_str(), 16) != 0) throw std::runtime_error("bad hex: " + s);
  return v;
}

// dense(d, b, seed): SURVEY.md §8(d) -- every monomial x^i y^j, i+j <= d, in
// the order i = 0..d, j = 0..d-i; b-bit magnitude from 32-bit chunks; sign bit.
BPoly dense(int d, int b, unsigned long seed) {
  std::mt19937_64 rng(seed);
  BPoly::TermMap t;
  for (int i = 0; i <= d; ++i)
    for (int j = 0; j <= d - i; ++j) {
      BigInt v(0);
      for (int done = 0; done < b; done += 32) {
        int take = std::min(32, b - done);
        unsigned long mask = (take == 32) ? 0xffffffffUL : ((1UL << take) - 1);
        v = (v << static_cast<unsigned long>(take)) + BigInt(static_cast<unsigned long>(rng() & mask));
      }
      if (v == 0) v = 1;
      if (rng() & 1) v = -v;
      t[{i, j}] = v;
    }
  return BPoly(std::move(t));
}

// g(x, y + k x + k) by expanding (y + kx + k)^j with exact binomials.
BPoly shear(const BPoly& g, long k) {
  BPoly lin = BPoly(BPoly::TermMap{{{0, 1}, BigInt(1)}, {{1, 0}, BigInt(k)}, {{0, 0}, BigInt(k)}});
  if (k == 0) lin = BPoly(BPoly::TermMap{{{0, 1}, BigInt(1)}});
  const auto& yc = g.y_coeffs();
  BPoly out;
  BPoly pw = BPoly::constant(1);
  for (size_t j = 0; j < yc.size(); ++j) {
    out = out + BPoly::from_univariate(yc[j], Var::X) * pw;
    pw = pw * lin;
  }
  return out;
}

// sheared(K, seed): f = g * prod_{k=1}^{K-1} g(x, y + kx + k), g = dense(6, 10, seed).
BPoly sheared(int K, unsigned long seed) {
  BPoly g = dense(6, 10, seed);
  BPoly f = g;
  for (int k = 1; k < K; ++k) f = f * shear(g, k);
  return f;
}

void print_bipoly(std::ostream& os, const BPoly& f) {
  os << "B " << f.terms().size() << "\n";
  for (const auto& [e, c] : f.terms()) os << e.first << " " << e.second << " " << hex(c) << "\n";
}

std::string json_upoly(const UPoly& p) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < p.coeffs().size(); ++i) os << (i ? "," : "") << "\"" << hex(p.coeffs()[i]) << "\"";
  os << "]";
  return os.str();
}

std::string json_bipoly(const BPoly& f) {
  std::ostringstream os;
  os << "[";
  bool first = true;
  for (const auto& [e, c] : f.terms()) {
    os << (first ? "" : ",") << "[" << e.first << "," << e.second << ",\"" << hex(c) << "\"]";
    first = false;
  }
  os << "]";
  return os.str();
}

std::string json_sqf(const SquareFreeFactorization& sf) {
  std::ostringstream os;
  os << "{\"unit\":\"" << hex(sf.unit) << "\",\"factors\":[";
  for (size_t i = 0; i < sf.factors.size(); ++i)
    os << (i ? "," : "") << "{\"mult\":" << sf.factors[i].multiplicity
       << ",\"poly\":" << json_upoly(sf.factors[i].poly) << "}";
  os << "]}";
  return os.str();
}

struct Operand {
  bool bivariate = false;
  BPoly b;
  UPoly u;
};

bool read_operand(std::istream& in, const std::string& tag, Operand& out) {
  size_t n = 0;
  std::istringstream ls(tag);
  std::string kind;
  ls >> kind >> n;
  if (kind == "B") {
    BPoly::TermMap t;
    for (size_t i = 0; i < n; ++i) {
      int dx, dy;
      std::string c;
      in >> dx >> dy >> c;
      t[{dx, dy}] += from_hex(c);
    }
    out.bivariate = true;
    out.b = BPoly(std::move(t));
    return true;
  }
  if (kind == "U") {
    std::vector<BigInt> c(n);
    for (size_t i = 0; i < n; ++i) {
      std::string s;
      in >> s;
      c[i] = from_hex(s);
    }
    out.bivariate = false;
    out.u = UPoly(std::move(c));
    return true;
  }
  return false;
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int cmd_batch() {
  std::string line;
  while (std::getline(std::cin, line)) {
    if (line.rfind("OP ", 0) != 0) continue;
    std::string op = line.substr(3);
    std::vector<Operand> args;
    while (std::getline(std::cin, line)) {
      if (line == "END") break;
      if (line.empty()) continue;
      Operand o;
      if (read_operand(std::cin, line, o)) args.push_back(std::move(o));
    }
    std::ostringstream os;
    os << "{\"op\":\"" << op << "\",";
    double t0 = now();
    std::string body;
    try {
      if (op == "resultant_y" || op == "resultant_x") {
        UPoly r = resultant(args.at(0).b, args.at(1).b, op == "resultant_y" ? Var::Y : Var::X);
        body = std::string("\"result\":") + json_upoly(r);
      } else if (op == "resultant_fy") {
        UPoly r = resultant(args.at(0).b, derive(args.at(0).b, Var::Y, 1), Var::Y);
        body = std::string("\"result\":") + json_upoly(r);
      } else if (op == "sylvester_y") {  // proj/tests/oracles.cpp:82-120 (Bareiss on the Sylvester matrix)
        body = std::string("\"result\":") + json_upoly(oracles::sylvester_resultant_y(args.at(0).b, args.at(1).b));
      } else if (op == "yun") {
        body = std::string("\"result\":") + json_sqf(yun_squarefree(args.at(0).u));
      } else if (op == "gcd") {
        body = std::string("\"result\":") + json_upoly(gcd_univariate(args.at(0).u, args.at(1).u));
      } else if (op == "sqfp") {
        body = std::string("\"result\":") + json_upoly(square_free_part(args.at(0).u));
      } else if (op == "gcd_bivariate") {
        body = std::string("\"result\":") + json_bipoly(gcd_bivariate(args.at(0).b, args.at(1).b));
      } else if (op == "curve_q") {  // CurveContext::resultant_q / q_factorization (lift.cpp:76-101)
        const BPoly& f = args.at(0).b;
        BPoly h = gcd_bivariate(derive(f, Var::X, 1), derive(f, Var::Y, 1));
        CurveContext ctx(f);
        const UPoly& q = ctx.resultant_q();
        body = std::string("\"result\":") + json_upoly(q) + ",\"h\":" + json_bipoly(h) +
               ",\"qsf\":" + json_sqf(ctx.q_factorization());
      } else {
        body = "\"error\":\"unknown op\"";
      }
    } catch (const PreconditionError& e) {
      body = std::string("\"error\":\"PreconditionError\",\"msg\":\"") + e.what() + "\"";
    } catch (const Error& e) {
      body = std::string("\"error\":\"Error\",\"msg\":\"") + e.what() + "\"";
    }
    os << body << ",\"seconds\":" << (now() - t0) << "}";
    std::cout << os.str() << std::endl;
  }
  return 0;
}

// The exact random inputs of proj/tests/test_elim.cpp (same generators, seeds
// and rejection logic), together with the reference's outputs on them.
int cmd_elim_cases() {
  {  // test_elim.cpp:34-44, seed 21
    std::mt19937_64 rng(21);
    int done = 0;
    while (done < 120) {
      BPoly p = oracles::random_bipoly(rng, 4, 50);
      BPoly q = oracles::random_bipoly(rng, 4, 50);
      if (p.degree_y() < 1 || q.degree_y() < 1) continue;
      UPoly r = resultant(p, q, Var::Y);
      UPoly s = oracles::sylvester_resultant_y(p, q);
      std::cout << "{\"case\":\"sylvester_seed21\",\"p\":" << json_bipoly(p) << ",\"q\":" << json_bipoly(q)
                << ",\"result\":" << json_upoly(r) << ",\"sylvester_agrees\":" << (r == s ? "true" : "false")
                << "}\n";
      ++done;
    }
  }
  {  // test_elim.cpp:46-70, seed 22
    std::mt19937_64 rng(22);
    int done = 0;
    while (done < 40) {
      BPoly a = oracles::random_bipoly(rng, 2, 6);
      BPoly b = oracles::random_bipoly(rng, 2, 6);
      BPoly c = oracles::random_bipoly(rng, 2, 6);
      if (c.degree_y() < 1) continue;
      BPoly p = a * c, q = b * c;
      UPoly r = resultant(p, q, Var::Y);
      std::cout << "{\"case\":\"common_factor_seed22\",\"p\":" << json_bipoly(p) << ",\"q\":" << json_bipoly(q)
                << ",\"result\":" << json_upoly(r) << "}\n";
      ++done;
    }
    done = 0;
    while (done < 40) {
      BPoly p = oracles::random_bipoly(rng, 3, 10);
      BPoly q = oracles::random_bipoly(rng, 3, 10);
      if (p.degree_y() < 1 || q.degree_y() < 1) continue;
      UPoly r = resultant(p, q, Var::Y);
      std::cout << "{\"case\":\"generic_seed22\",\"p\":" << json_bipoly(p) << ",\"q\":" << json_bipoly(q)
                << ",\"result\":" << json_upoly(r) << "}\n";
      ++done;
    }
  }
  {  // test_elim.cpp:105-122, seed 23
    std::mt19937_64 rng(23);
    for (int t = 0; t < 120; ++t) {
      UPoly p = oracles::random_upoly(rng, 3, 8);
      UPoly q = oracles::random_upoly(rng, 2, 8);
      if (p.degree() < 1 || q.degree() < 1) continue;
      UPoly prod = p * q * q;
      std::cout << "{\"case\":\"yun_seed23\",\"u\":" << json_upoly(prod) << ",\"result\":"
                << json_sqf(yun_squarefree(prod)) << "}\n";
    }
  }
  {  // test_elim.cpp:124-143, seed 24
    std::mt19937_64 rng(24);
    for (int t = 0; t < 100; ++t) {
      UPoly u = oracles::random_upoly(rng, 3, 10);
      UPoly v = oracles::random_upoly(rng, 3, 10);
      UPoly w = oracles::random_upoly(rng, 2, 10);
      if (u.is_zero() || v.is_zero() || w.degree() < 1) continue;
      UPoly a = u * w, b = v * w;
      std::cout << "{\"case\":\"gcd_seed24\",\"a\":" << json_upoly(a) << ",\"b\":" << json_upoly(b)
                << ",\"result\":" << json_upoly(gcd_univariate(a, b)) << "}\n";
    }
  }
  return 0;
}

BPoly make_curve(const std::string& kind, int a, int b, unsigned long seed) {
  if (kind == "dense") return dense(a, b, seed);
  if (kind == "sheared") return sheared(a, seed);
  throw std::runtime_error("unknown curve kind " + kind);
}

int cmd_time_res(const std::string& kind, int a, int b, unsigned long seed, int reps, bool yun) {
  BPoly f = make_curve(kind, a, b, seed);
  BPoly fy = derive(f, Var::Y, 1);
  (void)f.y_coeffs();
  (void)fy.y_coeffs();
  double best = 1e300, total = 0, yun_s = -1;
  UPoly r;
  for (int i = 0; i < reps; ++i) {
    double t0 = now();
    r = resultant(f, fy, Var::Y);
    double dt = now() - t0;
    best = std::min(best, dt);
    total += dt;
  }
  std::string pattern;
  if (yun) {
    double t0 = now();
    auto sf = yun_squarefree(r);
    yun_s = now() - t0;
    for (const auto& fac : sf.factors)
      pattern += "(" + std::to_string(fac.poly.degree()) + ")^" + std::to_string(fac.multiplicity);
  }
  size_t bits = 0;
  for (const auto& c : r.coeffs()) bits = std::max(bits, mpz_sizeinbase(c.get_mpz_t(), 2));
  std::cout << "{\"kind\":\"" << kind << "\",\"a\":" << a << ",\"b\":" << b << ",\"seed\":" << seed
            << ",\"reps\":" << reps << ",\"res_seconds_best\":" << best << ",\"res_seconds_mean\":"
            << total / reps << ",\"deg_r\":" << r.degree() << ",\"bits_r\":" << bits
            << ",\"yun_seconds\":" << yun_s << ",\"yun_pattern\":\"" << pattern << "\"}" << std::endl;
  return 0;
}

int cmd_time_ctx(const std::string& kind, int a, int b, unsigned long seed, int reps, bool q) {
  BPoly f = make_curve(kind, a, b, seed);
  double best = 1e300, best_q = 1e300;
  int deg_r = -1, deg_q = -1;
  std::string pattern;
  for (int i = 0; i < reps; ++i) {
    double t0 = now();
    CurveContext ctx(f);
    const double dt = now() - t0;
    best = std::min(best, dt);
    deg_r = ctx.resultant_r().degree();
    pattern.clear();
    for (const auto& fac : ctx.r_factorization().factors)
      pattern += "(" + std::to_string(fac.poly.degree()) + ")^" + std::to_string(fac.multiplicity);
    if (q) {
      t0 = now();
      deg_q = ctx.resultant_q().degree();
      (void)ctx.q_factorization();
      best_q = std::min(best_q, now() - t0);
    }
  }
  std::cout << "{\"kind\":\"" << kind << "\",\"a\":" << a << ",\"b\":" << b << ",\"seed\":" << seed
            << ",\"reps\":" << reps << ",\"ctx_seconds_best\":" << best << ",\"deg_r\":" << deg_r
            << ",\"r_pattern\":\"" << pattern << "\"";
  if (q) std::cout << ",\"q_seconds_best\":" << best_q << ",\"deg_q\":" << deg_q;
  std::cout << "}" << std::endl;
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "gen" && argc >= 4) {
      std::string kind = argv[2];
      BPoly f = kind == "dense" ? dense(std::atoi(argv[3]), std::atoi(argv[4]), std::stoul(argv[5]))
                                : sheared(std::atoi(argv[3]), std::stoul(argv[4]));
      print_bipoly(std::cout, f);
      return 0;
    }
    if (cmd == "batch") return cmd_batch();
    if (cmd == "elim_cases") return cmd_elim_cases();
    if (cmd == "time_res" && argc >= 7)
      return cmd_time_res(argv[2], std::atoi(argv[3]), std::atoi(argv[4]), std::stoul(argv[5]),
                          std::atoi(argv[6]), argc >= 8 && std::string(argv[7]) == "yun");
    if (cmd == "time_ctx" && argc >= 7)
      return cmd_time_ctx(argv[2], std::atoi(argv[3]), std::atoi(argv[4]), std::stoul(argv[5]),
                          std::atoi(argv[6]), argc >= 8 && std::string(argv[7]) == "q");
    std::cerr << "usage: refdriver gen|batch|elim_cases|time_res|time_ctx ...\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "refdriver: " << e.what() << "\n";
    return 1;
  }
}
