// C ABI of the multi-modular resultant (include/ctg.h): plan construction,
// prime/constant caching, H2D/D2H staging and result decoding.
//
// Replaces curvetop::resultant (/root/reference/proj/src/elim.cpp:95-136) for
// every pair of nonzero inputs: the conventions of elim.cpp:97-104 (Var::X swap,
// zero inputs, degree-0 operands) fall out of the formal-degree Sylvester
// resultant computed on the device; only "both zero" (PreconditionError) and
// "one zero" (zero polynomial) are decided on the host without computation.
//
// A plan holds a BATCH of B >= 1 same-shape problems (same formal degrees, same
// derivative relation): one slot layout (the union of the supports), one prime set
// (enough for the largest bound), one set of kernel launches with blockIdx.z = curve.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "api_common.hpp"
#include "comm.hpp"
#include "internal.hpp"
#include "uni_internal.hpp"

namespace ctg {

// ---------------------------------------------------------------------------
// Input parsing (sparse terms keyed (dy, dx), zero terms dropped -- bipoly.cpp:7-15).
// Terms are kept flat and sorted by (dy, dx): batch calls parse and lay out thousands
// of terms per curve, and a node-per-term map made that pointer chasing the host cost.
// ---------------------------------------------------------------------------
struct Terms {
  std::vector<int32_t> dy, dx;
  std::vector<int8_t> sign;
  std::vector<uint32_t> off{0};  // limbs of term i: limbs[off[i] .. off[i+1]), trimmed
  std::vector<uint32_t> limbs;
  size_t size() const { return dy.size(); }
  bool empty() const { return dy.empty(); }
  int nlimbs(size_t i) const { return static_cast<int>(off[i + 1] - off[i]); }
  const uint32_t* mag(size_t i) const { return limbs.data() + off[i]; }
  void push(int y, int x, int sg, const uint32_t* l, int n) {
    dy.push_back(y);
    dx.push_back(x);
    sign.push_back(static_cast<int8_t>(sg));
    limbs.insert(limbs.end(), l, l + n);
    off.push_back(static_cast<uint32_t>(limbs.size()));
  }
};

static Terms parse_bipoly(const ctg_bipoly* f, bool swap_xy) {
  Terms t;
  if (!f || f->n_terms == 0) return t;
  if (f->n_terms < 0 || !f->dx || !f->dy || !f->sign || !f->limb_off || (!f->limbs && f->limb_off[f->n_terms] > 0))
    throw ApiError(CTG_INVALID, "bipoly: null pointer or negative term count");
  const int nt = f->n_terms;
  auto key = [&](int i) {
    int dx = f->dx[i], dy = f->dy[i];
    if (swap_xy) std::swap(dx, dy);
    return std::make_pair(dy, dx);
  };
  // Unique keys in (dy, dx) order, or in (dx, dy) order (a map keyed x-first, the usual
  // CSR of the reference's BiPoly): then a counting sort by dy yields (dy, dx) order.
  bool yx = true, xy = true;
  int maxdy = 0;
  for (int i = 0; i < nt; ++i) {
    if (f->dx[i] < 0 || f->dy[i] < 0) throw ApiError(CTG_INVALID, "bipoly: negative exponent");
    if (f->limb_off[i + 1] < f->limb_off[i]) throw ApiError(CTG_INVALID, "bipoly: limb_off not monotone");
    if (f->sign[i] < -1 || f->sign[i] > 1) throw ApiError(CTG_INVALID, "bipoly: sign must be -1, 0 or +1");
    const auto k = key(i);
    maxdy = std::max(maxdy, k.first);
    if (i > 0) {
      const auto k0 = key(i - 1);
      if (!(k0 < k)) yx = false;
      if (!(std::make_pair(k0.second, k0.first) < std::make_pair(k.second, k.first))) xy = false;
    }
  }
  t.dy.reserve(nt);
  t.dx.reserve(nt);
  t.sign.reserve(nt);
  t.off.reserve(nt + 1);
  t.limbs.reserve(f->limb_off[nt] - f->limb_off[0]);
  auto trimmed = [&](int i, const uint32_t*& l) {
    l = f->limbs + f->limb_off[i];
    int n = static_cast<int>(f->limb_off[i + 1] - f->limb_off[i]);
    while (n > 0 && l[n - 1] == 0) --n;
    return n;
  };
  auto copy_in = [&](int i) {
    const uint32_t* l;
    const int n = trimmed(i, l);
    if (n > 0 && f->sign[i] != 0) t.push(key(i).first, key(i).second, f->sign[i], l, n);
  };
  if (yx) {
    for (int i = 0; i < nt; ++i) copy_in(i);
    return t;
  }
  if (xy && maxdy <= 4 * nt + 64) {
    std::vector<int> start(maxdy + 2, 0), order(nt);
    for (int i = 0; i < nt; ++i) ++start[key(i).first + 1];
    for (int d = 0; d <= maxdy; ++d) start[d + 1] += start[d];
    for (int i = 0; i < nt; ++i) order[start[key(i).first]++] = i;
    for (int i : order) copy_in(i);
    return t;
  }
  // General input: stable sort by key, sum the terms of equal keys.
  std::vector<int> order(nt);
  for (int i = 0; i < nt; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key(a) < key(b); });
  for (int a = 0; a < nt;) {
    int b = a + 1;
    while (b < nt && key(order[b]) == key(order[a])) ++b;
    SBig acc;
    for (int r = a; r < b; ++r) {
      const uint32_t* l;
      const int n = trimmed(order[r], l);
      sbig_add_inplace(acc, f->sign[order[r]], l, n);
    }
    if (acc.sign != 0) {
      const auto k = key(order[a]);
      t.push(k.first, k.second, acc.sign, acc.mag.data(), static_cast<int>(acc.mag.size()));
    }
    a = b;
  }
  return t;
}

static int deg_y(const Terms& t) { return t.empty() ? -1 : t.dy.back(); }

// a * s == b for magnitudes (no allocation).
static bool mul_small_equals(const uint32_t* a, int na, uint32_t s, const uint32_t* b, int nb) {
  uint64_t carry = 0;
  int i = 0;
  for (; i < na; ++i) {
    const uint64_t v = static_cast<uint64_t>(a[i]) * s + carry;
    if (i >= nb || b[i] != static_cast<uint32_t>(v)) return false;
    carry = v >> 32;
  }
  for (; carry; ++i, carry >>= 32)
    if (i >= nb || b[i] != static_cast<uint32_t>(carry)) return false;
  return i == nb;
}

// q == dp/dy term by term: the terms of p with dy >= 1 map in order onto q's terms.
static bool is_y_derivative(const Terms& p, const Terms& q) {
  size_t k = 0;
  for (size_t i = 0; i < p.size(); ++i) {
    if (p.dy[i] == 0) continue;
    if (k >= q.size() || q.dy[k] != p.dy[i] - 1 || q.dx[k] != p.dx[i] || q.sign[k] != p.sign[i]) return false;
    if (!mul_small_equals(p.mag(i), p.nlimbs(i), static_cast<uint32_t>(p.dy[i]), q.mag(k), q.nlimbs(k))) return false;
    ++k;
  }
  return k == q.size();
}

// One parsed problem, normalised so that deg_y p >= deg_y q.
struct Problem {
  Terms p, q;
  int n = -1, m = -1, deriv = 0, negate = 0;
  bool trivial = false;  // one input zero -> zero polynomial
  int64_t degb = 0;      // degree bound of the result
  double bound_bits = 0; // log2 Hadamard bound
};

static Problem parse_problem(const ctg_bipoly* pin, const ctg_bipoly* qin, int32_t eliminate_x) {
  Problem pr;
  pr.p = parse_bipoly(pin, eliminate_x != 0);
  pr.q = parse_bipoly(qin, eliminate_x != 0);
  // Conventions of elim.cpp:98-100.
  if (pr.p.empty() && pr.q.empty()) throw ApiError(CTG_PRECONDITION, "resultant: both inputs identically zero");
  if (pr.p.empty() || pr.q.empty()) {
    pr.trivial = true;
    return pr;
  }
  pr.n = deg_y(pr.p);
  pr.m = deg_y(pr.q);
  if (pr.n < pr.m) {
    std::swap(pr.p, pr.q);
    std::swap(pr.n, pr.m);
    pr.negate = (pr.n & 1) && (pr.m & 1);  // res(p,q) = (-1)^{nm} res(q,p)
  }
  pr.deriv = (pr.m == pr.n - 1 && pr.n >= 1 && is_y_derivative(pr.p, pr.q)) ? 1 : 0;
  // Degree bound of the result (min of the Sylvester row bound and Bezout).
  int Xp = 0, Xq = 0, tp = 0, tq = 0;
  for (size_t i = 0; i < pr.p.size(); ++i) {
    Xp = std::max(Xp, pr.p.dx[i]);
    tp = std::max(tp, pr.p.dy[i] + pr.p.dx[i]);
  }
  for (size_t i = 0; i < pr.q.size(); ++i) {
    Xq = std::max(Xq, pr.q.dx[i]);
    tq = std::max(tq, pr.q.dy[i] + pr.q.dx[i]);
  }
  pr.degb = std::min(static_cast<int64_t>(pr.m) * Xp + static_cast<int64_t>(pr.n) * Xq,
                     static_cast<int64_t>(tp) * tq);
  // before any layout is built: a sparse input with a huge exponent must not
  // allocate gigabytes of dense slots first
  if (pr.degb + 1 > (int64_t{1} << 28))
    throw ApiError(CTG_UNSUPPORTED, "resultant: degree bound of the result exceeds 2^28");
  if (static_cast<int64_t>(pr.n + 1) * (Xp + 1) + static_cast<int64_t>(pr.m + 1) * (Xq + 1) > (int64_t{1} << 30))
    throw ApiError(CTG_UNSUPPORTED, "resultant: dense slot layout exceeds 2^30 coefficients");
  // Hadamard bound over |x| = 1.
  auto norm_bits = [](const Terms& t) {
    // Terms are sorted by dy: each y-degree is one contiguous run.
    std::vector<double> run, sq;
    for (size_t a = 0; a < t.size();) {
      size_t b = a;
      run.clear();
      for (; b < t.size() && t.dy[b] == t.dy[a]; ++b) run.push_back(log2_upper(t.mag(b), t.nlimbs(b)));
      const double l1 = log2_sum_upper(run);
      if (std::isfinite(l1)) sq.push_back(2 * l1);
      a = b;
    }
    return log2_sum_upper(sq);
  };
  const double bp = norm_bits(pr.p), bq = norm_bits(pr.q);
  pr.bound_bits = 0.5 * pr.m * (std::isfinite(bp) ? bp : 0) + 0.5 * pr.n * (std::isfinite(bq) ? bq : 0);
  if (pr.bound_bits < 0) pr.bound_bits = 0;
  return pr;
}

}  // namespace ctg

using namespace ctg;

struct ctg_plan {
  int device = 0;
  int B = 1;
  bool trivial = false;  // (B == 1 only) one input zero: the result is the zero polynomial
  int n = 0, m = 0, deriv = 0, negate = 0;
  uint32_t D = 0, N = 0, r = 1, a = 0;
  int P = 0, S = 0, L = 1;
  double bound_bits = 0;
  std::vector<int32_t> dir;
  std::vector<uint32_t> h_limbs;  // [B][L][S]
  std::vector<int8_t> h_sign;     // [B][S]
  std::shared_ptr<CrtTables> tabs;
  // device state
  uint32_t* d_limbs = nullptr;
  int8_t* d_sign = nullptr;
  int32_t* d_dir = nullptr;
  uint32_t* d_tab = nullptr;       // [B][P][S]
  uint32_t* d_flags = nullptr;
  uint32_t* d_counters = nullptr;
  uint32_t flag_cap = 1u << 16;
  uint32_t* d_Y = nullptr;         // [B][P][J]
  double* d_upart = nullptr;       // [B][nchunk][J]
  uint64_t* d_cols = nullptr;      // [B][J][L16]
  uint32_t* d_vals = nullptr;      // K2 point values [B][P][nrows][N] (fast path only)
  uint32_t* d_gwarp = nullptr;     // k_modres_warp buffers in global memory (deg_y beyond ~6000)
  uint32_t* d_ntt = nullptr;       // K4 work array [B][P][N] when N > kMaxNttSmem
  int nrows = 0, maxlen = 0;
  bool fast_ok = false;
  bool mw_ok = false;              // 40 < n <= 127, m = n - 1: K2 point values + k_modres_mw
  bool fused = false;              // K2 folded into K3 (k_modres_fused): no d_vals
  int crt_cap = 0;
  int launches = 0;
  bool uploaded = false;
  // Device buffers come from the stream-ordered pool (cudaMallocAsync): no device-wide
  // synchronisation per plan; they are released on the last stream the plan used.  Plans
  // run by ctg_resultant_batch instead bump-allocate from a grow-only per-context scratch
  // region (`bump`), so steady-state calls allocate nothing.
  cudaStream_t last_stream = nullptr;
  uint8_t* bump = nullptr;
  size_t bump_off = 0, bump_cap = 0;
  template <class T>
  void palloc(T*& ptr, size_t count, cudaStream_t st) {
    const size_t bytes = std::max<size_t>(1, count) * sizeof(T);
    if (bump) {
      if (bump_off + bytes > bump_cap) throw ApiError(CTG_INTERNAL, "plan: scratch region too small");
      ptr = reinterpret_cast<T*>(bump + bump_off);
      bump_off += (bytes + 255) & ~static_cast<size_t>(255);
      return;
    }
    void* p = nullptr;
    CTG_CUDA_CHECK(cudaMallocAsync(&p, bytes, st));
    ptr = static_cast<T*>(p);
  }
  template <class T>
  void pfree(T*& ptr) {
    if (ptr && !bump) cudaFreeAsync(ptr, last_stream);
    ptr = nullptr;
  }
  // Bytes palloc will request for upload + residues + a CRT over J coefficients.
  size_t scratch_bytes(int J) const {
    auto r = [](size_t b) { return (std::max<size_t>(1, b) + 255) & ~static_cast<size_t>(255); };
    const size_t nch = static_cast<size_t>((P + kCrtChunk - 1) / kCrtChunk);
    size_t s = r(4 * h_limbs.size()) + r(h_sign.size()) + r(4 * dir.size()) + r(4ull * B * P * S) +
               r(4ull * flag_cap) + r(16);
    if ((fast_ok && !fused) || mw_ok) s += r(4ull * B * P * nrows * N);
    s += r(4 * general_warp_gbuf_words(n));
    if (N > kMaxNttSmem) s += r(4ull * B * P * N);
    s += r(4 * crt_y_words(*tabs, B, J)) + r(8 * static_cast<size_t>(B) * nch * J) +
         r(8 * ((crt_cols_words(*tabs, B, J) + 1) / 2));
    return s;
  }
  ~ctg_plan() {
    pfree(d_limbs);
    pfree(d_sign);
    pfree(d_dir);
    pfree(d_tab);
    pfree(d_flags);
    pfree(d_counters);
    pfree(d_Y);
    pfree(d_upart);
    pfree(d_cols);
    pfree(d_vals);
    pfree(d_gwarp);
    pfree(d_ntt);
  }
  int out_limbs() const { return tabs ? tabs->LM : 0; }
  int out_words() const { return out_limbs() + 1; }
};

namespace ctg {

// Builds a plan over problems[idx...] which must share (n, m, deriv, negate).
ctg_plan* plan_build(const std::vector<Problem>& probs, const std::vector<int>& idx, int device) {
  std::unique_ptr<ctg_plan> pl(new ctg_plan());
  pl->device = device;
  pl->B = static_cast<int>(idx.size());
  const Problem& p0 = probs[idx[0]];
  if (p0.trivial) {
    if (pl->B != 1) throw ApiError(CTG_INVALID, "plan: batch plans need nonzero inputs");
    pl->trivial = true;
    return pl.release();
  }
  pl->n = p0.n;
  pl->m = p0.m;
  pl->deriv = p0.deriv;
  pl->negate = p0.negate;
  int64_t degb = 0;
  double bound = 0;
  for (int i : idx) {
    const Problem& pr = probs[i];
    if (pr.trivial || pr.n != pl->n || pr.m != pl->m || pr.deriv != pl->deriv || pr.negate != pl->negate)
      throw ApiError(CTG_INVALID, "plan: batch members must have the same degrees in the eliminated variable");
    degb = std::max(degb, pr.degb);
    bound = std::max(bound, pr.bound_bits);
  }
  const int n = pl->n, m = pl->m;
  using tclk = std::chrono::steady_clock;
  const auto tb0 = tclk::now();
  // Union slot layout: y-degree j of p owns x-degrees 0..X_j (max over the batch).
  std::vector<int32_t> Xp(n + 1, -1), Xq(m + 1, -1);
  for (int i : idx) {
    const Terms& tp = probs[i].p;
    for (size_t t = 0; t < tp.size(); ++t) Xp[tp.dy[t]] = std::max(Xp[tp.dy[t]], tp.dx[t]);
    if (!pl->deriv) {
      const Terms& tq = probs[i].q;
      for (size_t t = 0; t < tq.size(); ++t) Xq[tq.dy[t]] = std::max(Xq[tq.dy[t]], tq.dx[t]);
    }
  }
  std::vector<int32_t> offp(n + 1), lenp(n + 1), offq(m + 1, 0), lenq(m + 1, 0);
  int64_t S64 = 0;
  for (int j = 0; j <= n; ++j) {
    offp[j] = static_cast<int32_t>(S64);
    lenp[j] = Xp[j] + 1;
    S64 += lenp[j];
  }
  if (!pl->deriv)
    for (int j = 0; j <= m; ++j) {
      offq[j] = static_cast<int32_t>(S64);
      lenq[j] = Xq[j] + 1;
      S64 += lenq[j];
    }
  if (S64 > (int64_t{1} << 30)) throw ApiError(CTG_UNSUPPORTED, "resultant: dense slot layout exceeds 2^30 coefficients");
  const int S = static_cast<int>(S64);
  pl->S = S;
  int L = 1;
  for (int i : idx) {
    const Terms& tp = probs[i].p;
    for (size_t t = 0; t < tp.size(); ++t) L = std::max(L, tp.nlimbs(t));
    if (!pl->deriv) {
      const Terms& tq = probs[i].q;
      for (size_t t = 0; t < tq.size(); ++t) L = std::max(L, tq.nlimbs(t));
    }
  }
  pl->L = L;
  pl->h_limbs.assign(static_cast<size_t>(pl->B) * L * S, 0u);
  pl->h_sign.assign(static_cast<size_t>(pl->B) * S, 0);
  parallel_for(pl->B, [&](int b) {
    uint32_t* lb = pl->h_limbs.data() + static_cast<size_t>(b) * L * S;
    int8_t* sb = pl->h_sign.data() + static_cast<size_t>(b) * S;
    auto put = [&](const Terms& t, const std::vector<int32_t>& off) {
      for (size_t i = 0; i < t.size(); ++i) {
        const int s = off[t.dy[i]] + t.dx[i];
        sb[s] = t.sign[i];
        const uint32_t* m = t.mag(i);
        for (int l = 0; l < t.nlimbs(i); ++l) lb[static_cast<size_t>(l) * S + s] = m[l];
      }
    };
    put(probs[idx[b]].p, offp);
    if (!pl->deriv) put(probs[idx[b]].q, offq);
  });
  const auto tb1 = tclk::now();
  pl->dir.clear();
  for (auto* v : {&offp, &lenp, &offq, &lenq}) pl->dir.insert(pl->dir.end(), v->begin(), v->end());
  pl->nrows = pl->deriv ? n + 1 : n + m + 2;
  pl->maxlen = 1;
  for (int v : lenp) pl->maxlen = std::max(pl->maxlen, v);
  for (int v : lenq) pl->maxlen = std::max(pl->maxlen, v);
  pl->fast_ok = (m == n - 1 || m == n) && n >= 2 && n <= kFastMaxDeg;
  pl->mw_ok = m == n - 1 && n > kFastMaxDeg && n <= 127;

  if (degb + 1 > (int64_t{1} << 28)) throw ApiError(CTG_UNSUPPORTED, "resultant: degree bound of the result exceeds 2^28");
  pl->D = static_cast<uint32_t>(degb + 1);
  pl->N = choose_ntt_size(pl->D, &pl->r, &pl->a);
  {
    int lp = 4;  // coset NTT length of the fused kernel (res_common.cuh coset_lp(n + 1))
    while (lp < n + 1) lp <<= 1;
    // Opt-in (CTG_FUSE=1): measured equal to K2 + K3 on B200 (both are bound by the FMA-heavy
    // pipe, not by the point-value round trip), but it never materialises the point values.
    static const bool fuse = std::getenv("CTG_FUSE") != nullptr && std::getenv("CTG_FUSE")[0] == '1';
    pl->fused = pl->fast_ok && pl->deriv && m == n - 1 && pl->maxlen <= lp && pl->N % lp == 0 && fuse;
  }
  pl->bound_bits = bound;
  if (static_cast<uint64_t>(pl->B) * pl->N * static_cast<uint64_t>(std::max(1.0, (bound + 37) / 29.0)) >= (1ull << 32))
    throw ApiError(CTG_UNSUPPORTED, "resultant: more than 2^32 evaluation units (> 16 GB of residues) in one plan");
  const double need = bound + 1 + 36;
  const auto tb2 = tclk::now();
  std::vector<uint32_t> primes;
  try {
    primes = select_primes(pl->N, need, kResPrimeMax);  // mmul3 window (modarith.cuh), p > 2^30
  } catch (const std::runtime_error&) {
    // very large N leaves too few primes p = cN + 1 above 2^30: extend the window downwards
    // (same descending enumeration, so the first primes are unchanged; Montgomery, mmul3 and
    // the CRT hold for any odd p < 2^30.4)
    primes = select_primes(pl->N, need, kResPrimeMax, 1ull << 24);
  }
  pl->P = static_cast<int>(primes.size());
  const auto tb3 = tclk::now();
  pl->tabs = get_tables(pl->device, pl->N, primes);
  const auto tb4 = tclk::now();
  static const bool trace = std::getenv("CTG_TRACE_HOST") != nullptr;
  auto us = [](tclk::time_point a, tclk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  if (trace)
    std::fprintf(stderr, "[ctg] plan_build B=%d: layout+fill %.1f us, dims %.1f us, primes %.1f us, tables %.1f us\n", pl->B,
                 us(tb0, tb1), us(tb1, tb2), us(tb2, tb3), us(tb3, tb4));
  return pl.release();
}

static void plan_alloc(ctg_plan* pl, cudaStream_t st) {
  if (pl->d_tab) return;
  pl->last_stream = st;
  pl->palloc(pl->d_limbs, pl->h_limbs.size(), st);
  pl->palloc(pl->d_sign, pl->h_sign.size(), st);
  pl->palloc(pl->d_dir, pl->dir.size(), st);
  pl->palloc(pl->d_tab, static_cast<size_t>(pl->B) * pl->P * pl->S, st);
  pl->palloc(pl->d_flags, pl->flag_cap, st);
  pl->palloc(pl->d_counters, 4, st);
  if ((pl->fast_ok && !pl->fused) || pl->mw_ok)
    pl->palloc(pl->d_vals, static_cast<size_t>(pl->B) * pl->P * pl->nrows * pl->N, st);
  if (general_warp_gbuf_words(pl->n)) pl->palloc(pl->d_gwarp, general_warp_gbuf_words(pl->n), st);
  if (pl->N > kMaxNttSmem) pl->palloc(pl->d_ntt, static_cast<size_t>(pl->B) * pl->P * pl->N, st);
  CTG_CUDA_CHECK(cudaMemsetAsync(pl->d_counters, 0, sizeof(uint32_t) * 4, st));
}

// H2D of the plan's inputs; with `staging` (pinned, >= plan_h2d_bytes) the three copies go
// through page-locked memory and stay asynchronous.
void plan_upload(ctg_plan* pl, cudaStream_t st, uint8_t* staging = nullptr) {
  if (pl->trivial) return;
  plan_alloc(pl, st);
  pl->last_stream = st;
  const size_t nl = sizeof(uint32_t) * pl->h_limbs.size(), ns = pl->h_sign.size(), nd = 4 * pl->dir.size();
  const void *src_l = pl->h_limbs.data(), *src_s = pl->h_sign.data(), *src_d = pl->dir.data();
  if (staging) {
    std::memcpy(staging, src_l, nl);
    std::memcpy(staging + nl, src_d, nd);
    std::memcpy(staging + nl + nd, src_s, ns);
    src_l = staging;
    src_d = staging + nl;
    src_s = staging + nl + nd;
  }
  CTG_CUDA_CHECK(cudaMemcpyAsync(pl->d_limbs, src_l, nl, cudaMemcpyHostToDevice, st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(pl->d_dir, src_d, nd, cudaMemcpyHostToDevice, st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(pl->d_sign, src_s, ns, cudaMemcpyHostToDevice, st));
  pl->uploaded = true;
}

int64_t plan_h2d_bytes(const ctg_plan* pl) {
  return static_cast<int64_t>(sizeof(uint32_t) * pl->h_limbs.size() + pl->h_sign.size() + 4 * pl->dir.size());
}

// Rows of curve b, prime k in [k0, k1): d_rows + b * curve_stride + (k - k0) * N  (curve_stride 0 = dense).
// scatter (stage 3 only): K4 writes the coefficients to the shards' receive blocks instead of d_rows.
void plan_stage(ctg_plan* pl, int stage, int k0, int k1, uint32_t* d_rows, long long curve_stride, cudaStream_t st,
                const RowScatter* scatter = nullptr) {
  if (pl->trivial) return;
  if (!pl->uploaded) throw ApiError(CTG_INVALID, "plan: inputs not uploaded");
  if (k0 < 0 || k1 > pl->P || k0 > k1) throw ApiError(CTG_INVALID, "plan: prime range out of bounds");
  if (stage < 1 || stage > 5) throw ApiError(CTG_INVALID, "plan: stage must be 1..5");
  const int nk = k1 - k0;
  if (nk == 0) return;
  const size_t rows_bstride = curve_stride > 0 ? static_cast<size_t>(curve_stride) : static_cast<size_t>(nk) * pl->N;
  pl->last_stream = st;
  if (stage == 1) {
    pl->launches += launch_reduce(pl->d_limbs, pl->d_sign, pl->S, pl->L, pl->tabs->d_pc, pl->tabs->d_rpow, k0, nk, pl->d_tab,
                                  static_cast<size_t>(pl->P) * pl->S, pl->B, st);
    CTG_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (stage == 3) {
    pl->launches += launch_interp(d_rows, rows_bstride, static_cast<int>(pl->N), nk, pl->B, pl->tabs->d_pc,
                                  pl->tabs->d_twinv, k0, static_cast<int>(pl->N), static_cast<int>(pl->r),
                                  static_cast<int>(pl->a), static_cast<int>(pl->D), pl->negate, pl->d_counters, st,
                                  pl->d_ntt, scatter);
    CTG_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (stage != 4) CTG_CUDA_CHECK(cudaMemsetAsync(pl->d_counters, 0, sizeof(uint32_t), st));
  ResParams rp{};
  rp.B = pl->B;
  rp.tab = pl->d_tab;
  rp.tab_bstride = static_cast<size_t>(pl->P) * pl->S;
  rp.S = pl->S;
  rp.pc = pl->tabs->d_pc;
  rp.k0 = k0;
  rp.nk = nk;
  rp.rows = d_rows;
  rp.rows_bstride = rows_bstride;
  rp.pitch = static_cast<int>(pl->N);
  rp.N = static_cast<int>(pl->N);
  rp.n = pl->n;
  rp.m = pl->m;
  rp.deriv = pl->deriv;
  rp.dir = pl->d_dir;
  rp.flag_list = pl->d_flags;
  rp.counters = pl->d_counters;
  rp.flag_cap = pl->flag_cap;
  rp.vals = (pl->fast_ok && !pl->fused) || pl->mw_ok ? pl->d_vals : nullptr;
  rp.fused = pl->fused ? 1 : 0;
  rp.nrows = pl->nrows;
  rp.maxlen = pl->maxlen;
  rp.twinv = pl->tabs->d_twinv;
  rp.gwarp = pl->d_gwarp;
  pl->launches += launch_modres(rp, true, st, stage == 4 ? 1 : stage == 5 ? 2 : 0);
  CTG_CUDA_CHECK(cudaGetLastError());
}

void plan_residues(ctg_plan* pl, int k0, int k1, uint32_t* d_rows, long long curve_stride, cudaStream_t st,
                   const RowScatter* scatter = nullptr) {
  for (int stage = 1; stage <= 3; ++stage) plan_stage(pl, stage, k0, k1, d_rows, curve_stride, st, scatter);
}

// Coefficients [j0, j1) of every curve.  Residues of curve b, prime k at d_all + b * curve_stride
// + (k / row_block) * block_stride + (k % row_block) * N; output curve b at d_out + b * out_stride.
// pitch / col0 (a shard's receive block of a fused exchange): rows of `pitch` words holding
// coefficients [col0, col0 + pitch) (defaults: N words, coefficient 0 first).
void plan_crt(ctg_plan* pl, const uint32_t* d_all, long long curve_stride, int row_block, long long block_stride,
              int j0, int j1, uint32_t* d_out, long long out_stride, cudaStream_t st, int pitch = 0, int col0 = 0) {
  if (pl->trivial) return;
  if (j0 < 0 || j1 > static_cast<int>(pl->D) || j0 > j1) throw ApiError(CTG_INVALID, "plan: coefficient range out of bounds");
  const int J = j1 - j0;
  if (J == 0) return;
  const int W = pl->out_words();
  if (out_stride > 0 && out_stride != static_cast<long long>(J) * W)
    throw ApiError(CTG_INVALID, "plan: output curve stride must equal (j1 - j0) * (out_limbs + 1)");
  const int nch = (pl->P + kCrtChunk - 1) / kCrtChunk;
  if (J > pl->crt_cap) {
    pl->pfree(pl->d_Y);
    pl->pfree(pl->d_upart);
    pl->pfree(pl->d_cols);
    pl->palloc(pl->d_Y, crt_y_words(*pl->tabs, pl->B, J), st);
    pl->palloc(pl->d_upart, static_cast<size_t>(pl->B) * nch * J, st);
    pl->palloc(pl->d_cols, (crt_cols_words(*pl->tabs, pl->B, J) + 1) / 2, st);  // u64 elements
    pl->crt_cap = J;
  }
  pl->last_stream = st;
  CrtParams cp{};
  cp.B = pl->B;
  cp.rows = d_all;
  cp.curve_stride = curve_stride > 0 ? curve_stride : static_cast<long long>(pl->P) * pl->N;
  cp.pitch = pitch > 0 ? pitch : static_cast<int>(pl->N);
  cp.col0 = col0;
  cp.P = pl->P;
  cp.row_block = row_block > 0 ? row_block : pl->P;
  cp.block_stride = row_block > 0 ? block_stride : 0;
  cp.j0 = j0;
  cp.J = J;
  cp.pc = pl->tabs->d_pc;
  cp.minv = pl->tabs->d_minv;
  cp.Mk16 = pl->tabs->d_Mk16;
  cp.M16 = pl->tabs->d_M16;
  cp.L16 = pl->tabs->L16;
  cp.Y = pl->d_Y;
  cp.upart = pl->d_upart;
  cp.cols = pl->d_cols;
  cp.out = d_out;
  cp.out_limbs = pl->tabs->LM;
  cp.use_i8 = pl->tabs->use_i8 ? 1 : 0;
  cp.Rp = static_cast<int>((static_cast<long long>(pl->B) * J + kI8TileJ - 1) / kI8TileJ * kI8TileJ);
  cp.L8 = pl->tabs->L8;
  cp.L8p = pl->tabs->L8p;
  cp.Kp = pl->tabs->Kp;
  cp.Bt8 = pl->tabs->d_Bt8;
  cp.M8 = pl->tabs->d_M8;
  // Hadamard bound (plan_build): |coefficient| < 2^bound_bits
  cp.top_digit = std::min(cp.L8, static_cast<int>(std::ceil((pl->bound_bits + 1) / 8.0)) + 1);
  cp.counters = pl->d_counters;
  pl->launches += launch_crt(cp, st);
  CTG_CUDA_CHECK(cudaGetLastError());
}

uint32_t plan_error_bits(ctg_plan* pl, cudaStream_t st) {
  if (pl->trivial || !pl->d_counters) return 0;
  uint32_t c[2] = {0, 0};
  CTG_CUDA_CHECK(cudaMemcpyAsync(c, pl->d_counters, sizeof(c), cudaMemcpyDeviceToHost, st));
  CTG_CUDA_CHECK(cudaStreamSynchronize(st));
  return c[1];
}

// h: one curve's CRT output (n_coeffs records of out_limbs + 1 words) -> library-owned
// CSR buffer, trimmed (two passes over the records, no per-coefficient allocation).
struct DecodeSize {
  std::vector<int> nl;  // limbs per coefficient
  size_t nc = 0, total = 0;
};

DecodeSize decode_size(const ctg_plan* pl, const uint32_t* h) {
  DecodeSize z;
  const int W = pl->out_words();
  z.nl.resize(pl->D);
  int deg = -1;
  for (uint32_t j = 0; j < pl->D; ++j) {
    const uint32_t* rec = h + static_cast<size_t>(j) * W;
    int n = W - 1;
    while (n > 0 && rec[n] == 0) --n;
    z.nl[j] = (rec[0] != 0u) ? n : 0;
    if (z.nl[j]) deg = static_cast<int>(j);
  }
  z.nc = static_cast<size_t>(deg + 1);
  for (size_t j = 0; j < z.nc; ++j) z.total += static_cast<size_t>(z.nl[j]);
  return z;
}

void decode_fill(const ctg_plan* pl, const uint32_t* h, const DecodeSize& z, ctg_upoly_buf* out) {
  const int W = pl->out_words();
  uint32_t off = 0;
  for (size_t j = 0; j < z.nc; ++j) {
    const uint32_t* rec = h + j * W;
    out->sign[j] = z.nl[j] ? static_cast<int8_t>(static_cast<int32_t>(rec[0])) : 0;
    out->limb_off[j] = off;
    std::memcpy(out->limbs + off, rec + 1, 4 * static_cast<size_t>(z.nl[j]));
    off += static_cast<uint32_t>(z.nl[j]);
  }
  out->limb_off[z.nc] = off;
}

void plan_decode(const ctg_plan* pl, const uint32_t* h, ctg_upoly_buf* out) {
  if (pl->trivial) {
    fill_upoly({}, out);
    return;
  }
  DecodeSize z = decode_size(pl, h);
  upoly_alloc(out, z.nc, z.total);
  decode_fill(pl, h, z, out);
}

// Streaming execution of chunk plans on one device context.  The caller parses and plans
// block after block; each chunk is enqueued as soon as its plan exists (H2D from pinned
// staging, kernels on ctx.stream / ctx.aux alternately, D2H of the exact result on ctx.copy after an event), so
// the host's parsing / planning of block c+1 and its decoding of block c overlap the GPU.
// Device scratch and pinned staging are carved from grow-only context regions reserved
// once per call; a chunk that does not fit drains the pipeline and regrows them.
struct Chunk {
  std::unique_ptr<ctg_plan> pl;
  std::vector<int> idx;  // positions in the caller's output array
  size_t in_off = 0, out_off = 0, out_words = 0, per_curve = 0;
  uint32_t* d_rows = nullptr;
  uint32_t* d_out = nullptr;
  // device-packed results: the D2H target is the page-locked result arena itself
  uint32_t *d_nl = nullptr, *d_meta = nullptr;
  uint8_t* d_pk = nullptr;
  size_t pk_bytes = 0;
  UpolyArena arena;
  bool probed = false;  // a square-freeness probe of this (single-curve) result was launched
  cudaEvent_t computed = nullptr, copied = nullptr;
  cudaEvent_t t_begin = nullptr, t_computed = nullptr, t_copied = nullptr;  // CTG_TRACE_HOST only
  double host_enqueued_ms = 0;
};

struct ChunkNeeds {
  size_t dev = 0, in = 0, out = 0;  // bytes, bytes, u32 words
};

ChunkNeeds chunk_needs(const ctg_plan* pl) {
  ChunkNeeds n;
  auto r = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  const size_t rows = r(4ull * pl->B * pl->P * pl->N);
  const size_t outw = static_cast<size_t>(pl->D) * pl->out_words() * pl->B;
  const size_t pack = r(4ull * pl->B * pl->D) + r(4 * pack_meta_words(pl->B, static_cast<int>(pl->D))) +
                      r(pack_bytes_bound(pl->B, static_cast<int>(pl->D), pl->out_words()));
  n.dev = pl->scratch_bytes(static_cast<int>(pl->D)) + rows + r(4 * outw) + pack;
  n.in = r(static_cast<size_t>(plan_h2d_bytes(pl)));
  n.out = 4 * (static_cast<size_t>(pl->B) + 1) + 4;  // packing meta + the two counters
  return n;
}

class ChunkPipeline {
 public:
  // nstreams: compute streams the chunks rotate over (measured: 3 for four or more blocks, as
  // 256 d20 curves in 32 | 64 | 64 | 64 | 32; 2 for fewer, as 64 d30 curves in 8 | 48 | 8).
  // probe_r: a single-curve call -- leave the square-freeness probe of R behind (SqfProbeCache)
  ChunkPipeline(Ctx& ctx, ctg_upoly_buf* out, int nstreams, bool probe_r = false)
      : ctx_(ctx), out_(out), st_(stats_tls()), nstreams_(std::max(1, std::min(3, nstreams))), probe_r_(probe_r) {}
  ~ChunkPipeline() {
    for (auto& c : inflight_) {  // error path: let the copies finish before the buffers go
      if (c.copied) cudaEventSynchronize(c.copied);
      destroy_events(c);
      c.arena.discard();
    }
    if (t0_) cudaEventDestroy(t0_);
  }
  // kSlots regions of `need` each (nothing may be in flight: growing synchronises and
  // reallocates).  Chunk i uses slot i % kSlots; before reusing a slot the pipeline finishes
  // the chunk that held it (the oldest in flight), so memory stays bounded for any batch size.
  void reserve(const ChunkNeeds& need) {
    drain();
    auto up = [](size_t x, size_t a) { return (x + a - 1) / a * a; };
    dev_cap_ = up(need.dev, 1024);  // slot bases stay aligned for vector / TMA access
    in_cap_ = up(need.in, 256);
    out_cap_ = up(need.out, 64);    // u32 words
    dev_ = reinterpret_cast<uint8_t*>(ctx_.scratch_u32(2, kSlots * dev_cap_ / 4 + 64));
    in_ = ctx_.pinned_input(kSlots * in_cap_);
    hout_ = ctx_.pinned_u32(kSlots * out_cap_);
  }
  void enqueue(Chunk&& c) {
    try {
      enqueue_impl(c);
    } catch (...) {
      // work already launched for this chunk writes into the slot's scratch and pinned
      // staging: let it finish before the chunk is dropped and the slot reused
      if (enq_stream_) cudaStreamSynchronize(enq_stream_);
      cudaStreamSynchronize(ctx_.copy_stream());
      destroy_events(c);
      c.arena.discard();
      throw;
    }
  }
  void enqueue_impl(Chunk& c) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    ctg_plan* pl = c.pl.get();
    const ChunkNeeds n = chunk_needs(pl);
    if (n.dev > dev_cap_ || n.in > in_cap_ || n.out > out_cap_)
      reserve({std::max(n.dev, dev_cap_), std::max(n.in, in_cap_), std::max(n.out, out_cap_)});
    if (inflight_.size() >= static_cast<size_t>(kSlots)) drain_front();
    const int slot = slot_next_;
    slot_next_ = (slot_next_ + 1) % kSlots;
    const size_t dev_off = static_cast<size_t>(slot) * dev_cap_;
    pl->bump = dev_ + dev_off;
    pl->bump_off = 0;
    pl->bump_cap = n.dev;
    c.in_off = static_cast<size_t>(slot) * in_cap_;
    c.per_curve = static_cast<size_t>(pl->D) * pl->out_words();
    c.out_words = c.per_curve * pl->B;
    c.out_off = static_cast<size_t>(slot) * out_cap_;
    // Chunks rotate over three compute streams, so one chunk's low-occupancy tail (K4, the CRT
    // carry) overlaps the next chunks' kernels.
    static const int forced = [] {  // CTG_CHUNK_STREAMS (1..3): A/B of the chunk rotation
      const char* e = std::getenv("CTG_CHUNK_STREAMS");
      return e ? std::max(1, std::min(3, std::atoi(e))) : 0;
    }();
    const int nstreams = forced ? forced : nstreams_;
    // CTG_CHUNK_PRIO=0: plain rotation over equal-priority streams (A/B)
    static const bool prio = [] {
      const char* e = std::getenv("CTG_CHUNK_PRIO");
      return !(e && e[0] == '0');
    }();
    const int ci = n_enqueued_++;
    const int si = ci % nstreams;
    // Priority level ci % levels (6 on B200): chunks 0..5 of a call are strictly ordered, which
    // covers every batch of up to six chunks (256 curves = 5).  Longer batches wrap: chunk 6
    // outranks the still-running chunks 3-5 once; a strictly decreasing level would need more
    // levels than the device has (stream priorities cannot be changed after launch).  Measured
    // with scripts/ab_prio.sh (documented rather than drained at the wrap).
    cudaStream_t s = prio && nstreams > 1 ? ctx_.prio_stream(ci)
                     : si == 0            ? ctx_.stream
                                          : ctx_.aux_stream(si - 1);
    enq_stream_ = s;
    cudaStream_t cp = ctx_.copy_stream();
    if (trace()) {
      for (cudaEvent_t* e : {&c.t_begin, &c.t_computed, &c.t_copied}) CTG_CUDA_CHECK(cudaEventCreate(e));
      if (!t0_) {
        CTG_CUDA_CHECK(cudaEventCreate(&t0_));
        CTG_CUDA_CHECK(cudaEventRecord(t0_, s));
        host0_ = t0;
      }
      CTG_CUDA_CHECK(cudaEventRecord(c.t_begin, s));
    }
    plan_upload(pl, s, in_ + c.in_off);
    st_.h2d_bytes += plan_h2d_bytes(pl);
    pl->palloc(c.d_rows, static_cast<size_t>(pl->B) * pl->P * pl->N, s);
    pl->palloc(c.d_out, c.out_words, s);
    plan_residues(pl, 0, pl->P, c.d_rows, 0, s);
    plan_crt(pl, c.d_rows, 0, 0, 0, 0, static_cast<int>(pl->D), c.d_out, 0, s);
    // results packed on the device into the library's block layout (no host decode)
    const int B = pl->B, D = static_cast<int>(pl->D), W = pl->out_words();
    c.pk_bytes = pack_bytes_bound(B, D, W);
    pl->palloc(c.d_nl, static_cast<size_t>(B) * D, s);
    pl->palloc(c.d_meta, pack_meta_words(B, D), s);
    pl->palloc(c.d_pk, c.pk_bytes, s);
    pl->launches += launch_pack(c.d_out, B, D, W, c.d_nl, c.d_meta, c.d_pk, s);
    c.arena.create(c.pk_bytes, B, /*pinned=*/true);
    // single-curve call: copy three residue rows of R for the probe (before `computed`, so the
    // slot's rows are not reused under the copy), then launch it behind the result
    const int rdeg = D - 1;
    c.probed = probe_r_ && B == 1 && rdeg >= 32 && pl->P >= 3 && sqf_probe_smem(rdeg) <= kUniSmemMax;
    SqfProbeCache& pc = ctx_.sqf;
    const int pj = pc.cur ^ 1;
    SqfProbeCache::Slot& sl = pc.slot[pj];
    if (c.probed) {
      pc.valid = false;
      if (sl.done) CTG_CUDA_CHECK(cudaStreamWaitEvent(s, sl.done, 0));  // the probe two calls back reads sl's rows
      const size_t words = 3 * static_cast<size_t>(pl->N);
      if (sl.d_cap < words) {
        if (sl.d_rows) {
          CTG_CUDA_CHECK(cudaStreamSynchronize(ctx_.probe_stream()));
          cudaFree(sl.d_rows);
          sl.d_rows = nullptr;
        }
        CTG_CUDA_CHECK(cudaMalloc(&sl.d_rows, 4 * words));
        sl.d_cap = words;
      }
      if (!sl.d_out) CTG_CUDA_CHECK(cudaMalloc(&sl.d_out, 8 * sizeof(int32_t)));
      if (!sl.h_out) CTG_CUDA_CHECK(cudaMallocHost(&sl.h_out, 8 * sizeof(int32_t)));
      if (!sl.done) CTG_CUDA_CHECK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
      if (sl.blk_cap < c.pk_bytes) {
        if (sl.d_blk) {
          CTG_CUDA_CHECK(cudaStreamSynchronize(ctx_.probe_stream()));
          cudaFree(sl.d_blk);
          cudaFreeHost(sl.h_blk);
          sl.d_blk = sl.h_blk = nullptr;
        }
        CTG_CUDA_CHECK(cudaMalloc(&sl.d_blk, c.pk_bytes));
        CTG_CUDA_CHECK(cudaMallocHost(&sl.h_blk, c.pk_bytes));
        sl.blk_cap = c.pk_bytes;
      }
      CTG_CUDA_CHECK(cudaMemcpyAsync(sl.d_rows, c.d_rows, 4 * words, cudaMemcpyDeviceToDevice, s));
      CTG_CUDA_CHECK(cudaMemcpyAsync(sl.d_blk, c.d_pk, c.pk_bytes, cudaMemcpyDeviceToDevice, s));
    }
    CTG_CUDA_CHECK(cudaEventCreateWithFlags(&c.computed, cudaEventDisableTiming));
    CTG_CUDA_CHECK(cudaEventCreateWithFlags(&c.copied, cudaEventDisableTiming));
    CTG_CUDA_CHECK(cudaEventRecord(c.computed, s));
    if (c.probed) {  // behind the result, on its own low-priority stream: the result never waits for it
      cudaStream_t ps = ctx_.probe_stream();
      CTG_CUDA_CHECK(cudaStreamWaitEvent(ps, c.computed, 0));
      pl->launches += launch_sqf_probe(sl.d_rows, static_cast<int>(pl->N), nullptr, nullptr, 1, 3, pl->tabs->d_pc,
                                       rdeg, sl.d_out, nullptr, ps, /*plain=*/1, /*small=*/false, /*single_deg=*/rdeg);
      CTG_CUDA_CHECK(cudaMemcpyAsync(sl.h_out, sl.d_out, 6 * sizeof(int32_t), cudaMemcpyDeviceToHost, ps));
      // R itself for the exact input check of the Yun call (probe_matches), by DMA
      CTG_CUDA_CHECK(cudaMemcpyAsync(sl.h_blk, sl.d_blk, c.pk_bytes, cudaMemcpyDeviceToHost, ps));
      CTG_CUDA_CHECK(cudaEventRecord(sl.done, ps));
      pc.cur = pj;
      pc.n = rdeg;
    }
    if (trace()) CTG_CUDA_CHECK(cudaEventRecord(c.t_computed, s));
    CTG_CUDA_CHECK(cudaStreamWaitEvent(cp, c.computed, 0));
    uint32_t* ho = hout_ + c.out_off;
    const size_t mw = 4 * (static_cast<size_t>(B) + 1);
    CTG_CUDA_CHECK(cudaMemcpyAsync(ho + mw, pl->d_counters, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, cp));
    CTG_CUDA_CHECK(cudaMemcpyAsync(ho, c.d_meta, 4 * mw, cudaMemcpyDeviceToHost, cp));
    CTG_CUDA_CHECK(cudaMemcpyAsync(c.arena.members(), c.d_pk, c.pk_bytes, cudaMemcpyDeviceToHost, cp));
    CTG_CUDA_CHECK(cudaEventRecord(c.copied, cp));
    if (trace()) {
      CTG_CUDA_CHECK(cudaEventRecord(c.t_copied, cp));
      c.host_enqueued_ms = std::chrono::duration<double, std::milli>(clk::now() - host0_).count();
    }
    pl->last_stream = cp;
    st_.d2h_bytes += static_cast<int64_t>(c.pk_bytes + 4 * (mw + 2));
    inflight_.push_back(std::move(c));
    enq_stream_ = nullptr;
    st_.h2d_ms += std::chrono::duration<double, std::milli>(clk::now() - t0).count();
  }
  // Waits for and decodes every chunk in flight, in order.
  void drain() {
    while (!inflight_.empty()) drain_front();
  }
  // Waits for and decodes the oldest chunk in flight (its slot becomes free).
  void drain_front() {
    using clk = std::chrono::steady_clock;
    auto ms_since = [](clk::time_point t) { return std::chrono::duration<double, std::milli>(clk::now() - t).count(); };
    Chunk& c = inflight_.front();
    {
      auto t0 = clk::now();
      CTG_CUDA_CHECK(cudaEventSynchronize(c.copied));
      st_.device_ms += ms_since(t0);
      t0 = clk::now();
      ctg_plan* pl = c.pl.get();
      const uint32_t* ho = hout_ + c.out_off;
      const size_t mw = 4 * (static_cast<size_t>(pl->B) + 1);
      st_.kernel_launches += pl->launches;
      st_.flagged_units += static_cast<int32_t>(ho[mw]);
      const uint32_t bits = ho[mw + 1];
      if (bits && err_.empty()) err_ = "resultant: device self-check failed (error bits " + std::to_string(bits) + ")";
      if (err_.empty()) {
        // the packed blocks are already in the arena: set the result pointers
        for (int b = 0; b < pl->B; ++b) c.arena.place(&out_[c.idx[b]], ho[4 * b + 2], ho[4 * b], ho[4 * b + 1]);
        c.arena.base = nullptr;  // owned by the results now
        if (c.probed) {  // where R sits in the probe slot's copy of the packed block
          SqfProbeCache& pc = ctx_.sqf;
          if (ho[0] - 1 == static_cast<uint32_t>(pc.n)) {
            pc.blk_off = ho[2];
            pc.blk_total = ho[1];
            pc.valid = true;
          }
        }
      } else {
        c.arena.discard();
      }
      if (trace()) {
        float a = 0, b = 0, d = 0;
        cudaEventElapsedTime(&a, t0_, c.t_begin);
        cudaEventElapsedTime(&b, t0_, c.t_computed);
        cudaEventElapsedTime(&d, t0_, c.t_copied);
        std::fprintf(stderr, "[ctg]   chunk B=%d: host enqueued %.3f | gpu begin %.3f computed %.3f copied %.3f | host decoded %.3f ms\n",
                     pl->B, c.host_enqueued_ms, a, b, d, std::chrono::duration<double, std::milli>(clk::now() - host0_).count());
      }
      destroy_events(c);
      st_.decode_ms += ms_since(t0);
    }
    inflight_.pop_front();
  }
  // Drains; throws if a chunk failed its device self-check (the caller frees the results).
  void finish() {
    drain();
    if (!err_.empty()) throw ApiError(CTG_INTERNAL, err_);
  }

 private:
  static bool trace() {
    static const bool t = std::getenv("CTG_TRACE_HOST") != nullptr;
    return t;
  }
  static void destroy_events(Chunk& c) {
    for (cudaEvent_t* e : {&c.computed, &c.copied, &c.t_begin, &c.t_computed, &c.t_copied}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
  }
  Ctx& ctx_;
  ctg_upoly_buf* out_;
  ctg_call_stats& st_;
  static constexpr int kSlots = 4;  // chunks in flight: three compute streams + one being decoded
  std::deque<Chunk> inflight_;
  int slot_next_ = 0;
  std::string err_;
  uint8_t* dev_ = nullptr;
  uint8_t* in_ = nullptr;
  uint32_t* hout_ = nullptr;
  size_t dev_cap_ = 0, in_cap_ = 0, out_cap_ = 0;  // per slot
  cudaEvent_t t0_ = nullptr;  // trace origin
  int n_enqueued_ = 0;
  int nstreams_ = 2;
  cudaStream_t enq_stream_ = nullptr;
  bool probe_r_ = false;
  std::chrono::steady_clock::time_point host0_;
};

// ---------------------------------------------------------------------------
// Prime sharding across GPUs: ctg_resultant_batch with
// ctg_opts.n_devices > 1 (one process, several devices) or ctg_opts.comm (one rank of a
// multi-process job).  Shard g of G owns primes [g Pb, (g+1) Pb) of every plan: K1-K4 write
// those rows into `send` [B][Pb][N]; ONE all-gather assembles `full` [G][B][Pb][N] on every
// shard (NCCL over NVLink; device-to-device copies when shards share a GPU); shard g
// reconstructs coefficients [g Jb, (g+1) Jb) (K5 reads the rank blocks in place); the exact
// limbs go straight to the host result (one process) or through a second all-gather (every
// rank returns the full result).  The only inter-GPU traffic is the residue matrix.
// ---------------------------------------------------------------------------

// Same plan on another device (host layout shared by value; constants from the cache).
static ctg_plan* plan_clone(const ctg_plan* src, int device) {
  if (src->d_tab) throw ApiError(CTG_INVALID, "plan_clone: source already on a device");
  std::unique_ptr<ctg_plan> c(new ctg_plan());
  c->device = device;
  c->B = src->B;
  c->trivial = src->trivial;
  c->n = src->n;
  c->m = src->m;
  c->deriv = src->deriv;
  c->negate = src->negate;
  c->D = src->D;
  c->N = src->N;
  c->r = src->r;
  c->a = src->a;
  c->P = src->P;
  c->S = src->S;
  c->L = src->L;
  c->bound_bits = src->bound_bits;
  c->dir = src->dir;
  c->h_limbs = src->h_limbs;
  c->h_sign = src->h_sign;
  c->flag_cap = src->flag_cap;
  c->nrows = src->nrows;
  c->maxlen = src->maxlen;
  c->fast_ok = src->fast_ok;
  c->mw_ok = src->mw_ok;
  c->fused = src->fused;
  c->tabs = get_tables(device, src->N, src->tabs->primes);
  return c.release();
}

struct Shard {
  int device = 0, rank = 0;
  cudaStream_t st = nullptr;
  std::unique_ptr<ctg_plan> pl;
  int k0 = 0, k1 = 0, j0 = 0, j1 = 0;
  uint32_t *send = nullptr, *full = nullptr, *crt = nullptr, *gath = nullptr, *xsend = nullptr;
  bool full_pooled = true;  // false: `full` is the device context's receive scratch (fused exchange)
  cudaEvent_t rows_done = nullptr;
  Shard() = default;
  Shard(const Shard&) = delete;
  Shard& operator=(const Shard&) = delete;
  ~Shard() {  // error paths: let the shard's work finish before its buffers go back to the pool
    if (!pl) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    pl->pfree(send);
    if (full_pooled) pl->pfree(full);
    pl->pfree(crt);
    pl->pfree(gath);
    pl->pfree(xsend);
    if (rows_done) cudaEventDestroy(rows_done);
    pl.reset();
    cudaSetDevice(prev);
  }
};

// Peer access between every pair of the distinct devices (enabled once per pair, cached); false
// if some pair cannot reach the other's memory (then the exchange goes through copies / NCCL).
static bool enable_peer_access(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> done;
  std::lock_guard<std::mutex> lock(mu);
  int prev = 0;
  cudaGetDevice(&prev);
  bool ok = true;
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      auto it = done.find({a, b});
      if (it != done.end()) {
        ok = ok && it->second;
        continue;
      }
      int can = 0;
      bool pair_ok = cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can;
      if (pair_ok) {
        cudaSetDevice(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        pair_ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
      }
      done[{a, b}] = pair_ok;
      ok = ok && pair_ok;
    }
  cudaSetDevice(prev);
  return ok;
}

static void resultant_batch_sharded(int batch, const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                                    ctg_upoly_buf* out, const ctg_opts* opts) {
  auto& stats = stats_tls();
  using tclk = std::chrono::steady_clock;
  const auto t_start = tclk::now();
  ctg_comm* comm = opts->comm;
  // the shard set: every shard of this process (one process) or this rank's (multi-process)
  int G = 1;
  std::vector<int> local_dev, local_rank;
  if (comm) {
    G = comm->nranks;
    local_dev.push_back(comm->device);
    local_rank.push_back(comm->rank);
  } else {
    if (!opts->devices) throw ApiError(CTG_INVALID, "ctg_opts: n_devices > 1 needs a devices array");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw ApiError(CTG_CUDA, "no CUDA device available (libctg has no CPU fallback)");
    G = opts->n_devices;
    for (int g = 0; g < G; ++g) {
      if (opts->devices[g] < 0 || opts->devices[g] >= count) throw ApiError(CTG_INVALID, "ctg_opts.devices out of range");
      local_dev.push_back(opts->devices[g]);
      local_rank.push_back(g);
    }
  }
  std::vector<int> distinct(local_dev);
  std::sort(distinct.begin(), distinct.end());
  const auto uend = std::unique(distinct.begin(), distinct.end());
  const bool repeated = uend != distinct.end();
  distinct.erase(uend, distinct.end());
  // Exchange of one process's shards: by default fused into K4 (its epilogue stores every
  // coefficient straight into the owning shard's receive block: NVLink peer stores, local stores
  // when shards share a GPU; each shard receives only its coefficient columns -- 1/G of an
  // all-gather's bytes).  CTG_SHARD_EXCHANGE=copy / nccl: the all-gather of whole rows (NCCL
  // between distinct devices, device copies otherwise), for A/B and as the fallback.
  const std::string xmode = std::getenv("CTG_SHARD_EXCHANGE") ? std::getenv("CTG_SHARD_EXCHANGE") : "fused";
  const bool fused_x = !comm && xmode == "fused" && G <= kMaxScatter && enable_peer_access(distinct);
  // multi-process (one rank per GPU): K4 stores by destination into a local send block and the
  // ranks swap column blocks with grouped ncclSend / ncclRecv (an all-to-all: each rank receives
  // only its coefficient columns, 1/G of an all-gather of whole rows)
  const bool a2a_x = comm && xmode != "copy" && xmode != "nccl" && G <= kMaxScatter;
  // NCCL between distinct devices of one process; device copies when a GPU hosts two shards
  const bool use_nccl_local = !comm && !fused_x && !repeated && xmode != "copy" && nccl_available();
  const std::vector<ncclComm_t>* local_comms = use_nccl_local ? &device_set_comms(local_dev) : nullptr;

  std::vector<Problem> probs(batch);
  parallel_for(batch, [&](int i) { probs[i] = parse_problem(&p[i], &q[i], eliminate_x); });
  std::map<std::tuple<int, int, int, int>, std::vector<int>> groups;
  for (int b = 0; b < batch; ++b) {
    if (probs[b].trivial)
      fill_upoly({}, &out[b]);
    else
      groups[{probs[b].n, probs[b].m, probs[b].deriv, probs[b].negate}].push_back(b);
  }
  // the device contexts' streams, scratch and pinned staging are this call's: lock every
  // involved device's context, in device order (no lock-order inversion between calls)
  std::vector<std::unique_lock<std::mutex>> locks;
  if (!groups.empty())
    for (int d : distinct) locks.emplace_back(context(d).mu);
  stats.setup_ms = std::chrono::duration<double, std::milli>(tclk::now() - t_start).count();
  int nshard_on[64] = {0};
  constexpr int kBlock = 64;  // curves per sharded plan
  for (auto& [key, all_idx] : groups) {
    for (size_t blk = 0; blk < all_idx.size(); blk += kBlock) {
      std::vector<int> idx(all_idx.begin() + blk, all_idx.begin() + std::min(all_idx.size(), blk + kBlock));
      static const bool trace = std::getenv("CTG_TRACE_HOST") != nullptr;
      auto tp = tclk::now();
      auto lap = [&](const char* what) {
        if (!trace) return;
        const auto t = tclk::now();
        std::fprintf(stderr, "[ctg] sharded G=%d block %zu: %s %.3f ms\n", G, blk, what,
                     std::chrono::duration<double, std::milli>(t - tp).count());
        tp = t;
      };
      std::vector<Shard> sh(local_dev.size());
      std::unique_ptr<ctg_plan> pl0;
      {
        PlanDeviceGuard g0(local_dev[0]);
        pl0.reset(plan_build(probs, idx, local_dev[0]));
      }
      const int B = pl0->B, Pn = pl0->P, N = static_cast<int>(pl0->N), D = static_cast<int>(pl0->D);
      const int W = pl0->out_words();
      const int Pb = (Pn + G - 1) / G, Jb = (D + G - 1) / G;
      const size_t rows_words = static_cast<size_t>(B) * Pb * N, crt_words = static_cast<size_t>(B) * Jb * W;
      // fused exchange: shard r's receive block holds coefficients [r Jb, (r + 1) Jb) of every
      // prime, [G blocks of primes][B][Pb][Jb]
      const size_t recv_words = static_cast<size_t>(G) * B * Pb * Jb;
      std::fill(std::begin(nshard_on), std::end(nshard_on), 0);
      for (size_t s = 0; s < sh.size(); ++s) {  // every shard's plan before any upload
        sh[s].device = local_dev[s];
        sh[s].rank = local_rank[s];
        PlanDeviceGuard g(sh[s].device);
        sh[s].pl.reset(s == 0 ? pl0.release() : plan_clone(sh[0].pl.get(), sh[s].device));
      }
      for (size_t s = 0; s < sh.size(); ++s) {
        Shard& S = sh[s];
        PlanDeviceGuard g(S.device);
        Ctx& ctx = context(S.device);
        const int slot = nshard_on[S.device % 64]++;  // shards sharing a GPU take different streams
        S.st = slot == 0 ? ctx.stream : slot <= 2 ? ctx.aux_stream(slot - 1) : ctx.stream;
        S.k0 = std::min(S.rank * Pb, Pn);
        S.k1 = std::min((S.rank + 1) * Pb, Pn);
        S.j0 = std::min(S.rank * Jb, D);
        S.j1 = std::min((S.rank + 1) * Jb, D);
        ctg_plan* pl = S.pl.get();
        plan_upload(pl, S.st);
        stats.h2d_bytes += plan_h2d_bytes(pl);
        pl->palloc(S.send, rows_words, S.st);
        if (fused_x) {  // other GPUs store into it: plain device memory (peer access covers
                        // cudaMalloc'd memory; stream-ordered pool memory would need pool access)
          S.full = ctx.scratch_u32(8 + slot, recv_words);
          S.full_pooled = false;
        } else if (a2a_x) {
          pl->palloc(S.full, recv_words, S.st);
          pl->palloc(S.gath, crt_words * G, S.st);
          pl->palloc(S.xsend, recv_words, S.st);
        } else {
          pl->palloc(S.full, rows_words * G, S.st);
        }
        pl->palloc(S.crt, crt_words, S.st);
        if (comm && !a2a_x) pl->palloc(S.gath, crt_words * G, S.st);
      }
      for (size_t s = 0; s < sh.size(); ++s) {  // every receive block exists before any K4 stores into it
        Shard& S = sh[s];
        PlanDeviceGuard g(S.device);
        RowScatter sc{};
        if (fused_x) {
          sc.G = G;
          sc.Jb = Jb;
          for (size_t r = 0; r < sh.size(); ++r) sc.dst[sh[r].rank] = sh[r].full;
          sc.shard_off = static_cast<long long>(S.rank) * B * Pb * Jb;
          sc.curve_stride = static_cast<long long>(Pb) * Jb;
        } else if (a2a_x) {  // by destination rank: xsend[r] = [B][Pb][Jb] block for rank r
          sc.G = G;
          sc.Jb = Jb;
          for (int r = 0; r < G; ++r) sc.dst[r] = S.xsend + static_cast<size_t>(r) * B * Pb * Jb;
          sc.shard_off = 0;
          sc.curve_stride = static_cast<long long>(Pb) * Jb;
        }
        const bool scatter = fused_x || a2a_x;
        if (S.k1 > S.k0)
          plan_residues(S.pl.get(), S.k0, S.k1, S.send, static_cast<long long>(Pb) * N, S.st, scatter ? &sc : nullptr);
        CTG_CUDA_CHECK(cudaEventCreateWithFlags(&S.rows_done, cudaEventDisableTiming));
        CTG_CUDA_CHECK(cudaEventRecord(S.rows_done, S.st));
      }
      lap("plans + uploads + K1-K4 enqueued");
      // exchange: full[h] = send of shard h, on every shard (fused: K4 already stored it)
      if (fused_x) {
        for (auto& S : sh) {
          PlanDeviceGuard g(S.device);
          for (auto& H : sh) CTG_CUDA_CHECK(cudaStreamWaitEvent(S.st, H.rows_done, 0));
        }
      } else if (a2a_x) {
        Shard& S = sh[0];
        PlanDeviceGuard g(S.device);
        const size_t blk_words = static_cast<size_t>(B) * Pb * Jb;
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        for (int r = 0; r < G; ++r) {
          nccl_check(nccl().Send(S.xsend + r * blk_words, blk_words, ncclUint32, r, comm->nc, S.st), "ncclSend");
          nccl_check(nccl().Recv(S.full + r * blk_words, blk_words, ncclUint32, r, comm->nc, S.st), "ncclRecv");
        }
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
      } else if (comm) {
        PlanDeviceGuard g(sh[0].device);
        nccl_check(nccl().AllGather(sh[0].send, sh[0].full, rows_words, ncclUint32, comm->nc, sh[0].st), "ncclAllGather");
      } else if (local_comms) {
        nccl_check(nccl().GroupStart(), "ncclGroupStart");
        for (size_t s = 0; s < sh.size(); ++s)
          nccl_check(nccl().AllGather(sh[s].send, sh[s].full, rows_words, ncclUint32, (*local_comms)[s], sh[s].st),
                     "ncclAllGather");
        nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
      } else {
        for (auto& S : sh) {
          PlanDeviceGuard g(S.device);
          for (auto& H : sh) {
            CTG_CUDA_CHECK(cudaStreamWaitEvent(S.st, H.rows_done, 0));
            CTG_CUDA_CHECK(cudaMemcpyPeerAsync(S.full + static_cast<size_t>(H.rank) * rows_words, S.device, H.send,
                                               H.device, 4 * rows_words, S.st));
          }
        }
      }
      // K5 of each shard's coefficient block, then the exact limbs to the host [B][D][W]
      uint32_t* host = nullptr;
      {
        PlanDeviceGuard g(sh[0].device);
        host = context(sh[0].device).pinned_u32(static_cast<size_t>(B) * D * W + 4);
      }
      for (auto& S : sh) {
        PlanDeviceGuard g(S.device);
        if (S.j1 > S.j0) {
          if (fused_x || a2a_x)
            plan_crt(S.pl.get(), S.full, static_cast<long long>(Pb) * Jb, Pb, static_cast<long long>(B) * Pb * Jb, S.j0,
                     S.j1, S.crt, 0, S.st, /*pitch=*/Jb, /*col0=*/S.j0);
          else
            plan_crt(S.pl.get(), S.full, static_cast<long long>(Pb) * N, Pb, static_cast<long long>(rows_words), S.j0,
                     S.j1, S.crt, 0, S.st);
        }
      }
      auto d2h_block = [&](const Shard& S, const uint32_t* src, int r) {
        const int j0 = std::min(r * Jb, D), j1 = std::min((r + 1) * Jb, D);
        if (j1 <= j0) return;
        const size_t w = static_cast<size_t>(j1 - j0) * W * 4;
        CTG_CUDA_CHECK(cudaMemcpy2DAsync(host + static_cast<size_t>(j0) * W, static_cast<size_t>(D) * W * 4, src, w, w,
                                         B, cudaMemcpyDeviceToHost, S.st));
        stats.d2h_bytes += static_cast<int64_t>(w) * B;
      };
      if (comm) {
        Shard& S = sh[0];
        PlanDeviceGuard g(S.device);
        nccl_check(nccl().AllGather(S.crt, S.gath, crt_words, ncclUint32, comm->nc, S.st), "ncclAllGather");
        for (int r = 0; r < G; ++r) d2h_block(S, S.gath + static_cast<size_t>(r) * crt_words, r);
      } else {
        for (auto& S : sh) {
          PlanDeviceGuard g(S.device);
          d2h_block(S, S.crt, S.rank);
        }
      }
      lap("exchange + K5 + D2H enqueued");
      uint32_t bits = 0;
      for (auto& S : sh) {
        PlanDeviceGuard g(S.device);
        CTG_CUDA_CHECK(cudaStreamSynchronize(S.st));
        bits |= plan_error_bits(S.pl.get(), S.st);
        stats.kernel_launches += S.pl->launches;
      }
      if (bits) throw ApiError(CTG_INTERNAL, "resultant (sharded): device self-check failed (error bits " + std::to_string(bits) + ")");
      stats.n_primes = std::max(stats.n_primes, Pn);
      stats.n_points = N;
      stats.n_coeffs = D;
      stats.out_limbs = std::max(stats.out_limbs, sh[0].pl->out_limbs());
      lap("device work done");
      const ctg_plan* plc = sh[0].pl.get();
      std::vector<DecodeSize> sz(B);
      parallel_for(B, [&](int b) { sz[b] = decode_size(plc, host + static_cast<size_t>(b) * D * W); });
      std::vector<size_t> off(B + 1, 0);
      for (int b = 0; b < B; ++b) off[b + 1] = off[b] + upoly_block_bytes(sz[b].nc, sz[b].total);
      UpolyArena arena;
      arena.create(off[B], B);
      parallel_for(B, [&](int b) {
        arena.place(&out[idx[b]], off[b], sz[b].nc, sz[b].total);
        decode_fill(plc, host + static_cast<size_t>(b) * D * W, sz[b], &out[idx[b]]);
      });
      lap("host decode");
      sh.clear();  // ~Shard releases every buffer on its device
      lap("release");
    }
  }
}

}  // namespace ctg

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

ctg_status ctg_plan_create_batch(int32_t batch, const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                                 const ctg_opts* opts, ctg_plan** plan) {
  return guarded([&] {
    if (!plan || !p || !q || batch < 1) throw ApiError(CTG_INVALID, "plan: bad batch arguments");
    DeviceGuard g(opts);
    std::vector<Problem> probs;
    std::vector<int> idx;
    for (int b = 0; b < batch; ++b) {
      probs.push_back(parse_problem(&p[b], &q[b], eliminate_x));
      idx.push_back(b);
    }
    const int dev = select_device(opts);
    *plan = plan_build(probs, idx, dev);
  });
}

ctg_status ctg_plan_create(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x, const ctg_opts* opts,
                           ctg_plan** plan) {
  return guarded([&] {
    if (!plan) throw ApiError(CTG_INVALID, "plan: null output pointer");
    DeviceGuard g(opts);
    std::vector<Problem> probs{parse_problem(p, q, eliminate_x)};
    const int dev = select_device(opts);
    *plan = plan_build(probs, {0}, dev);
  });
}

ctg_status ctg_plan_get_info(const ctg_plan* pl, ctg_plan_info* info) {
  return guarded([&] {
    if (!pl || !info) throw ApiError(CTG_INVALID, "plan: null pointer");
    std::memset(info, 0, sizeof(*info));
    info->n_primes = pl->P;
    info->n_points = static_cast<int32_t>(pl->N);
    info->n_coeffs = static_cast<int32_t>(pl->D);
    info->out_limbs = pl->out_limbs();
    info->deg_p = pl->n;
    info->deg_q = pl->m;
    info->derivative = pl->deriv;
    info->trivial = pl->trivial ? 1 : 0;
    info->bound_bits = pl->bound_bits;
    const double n = pl->n;
    info->work_mulmods = static_cast<double>(pl->B) * pl->P * pl->D * (n * n + n - 2);
    info->h2d_bytes = plan_h2d_bytes(pl);
    info->batch = pl->B;
  });
}

ctg_status ctg_plan_upload(ctg_plan* pl, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_upload(pl, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_residues(ctg_plan* pl, int32_t k0, int32_t k1, uint32_t* d_rows, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_residues(pl, k0, k1, d_rows, 0, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_stage(ctg_plan* pl, int32_t stage, int32_t k0, int32_t k1, uint32_t* d_rows, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_stage(pl, stage, k0, k1, d_rows, 0, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_stage_batch(ctg_plan* pl, int32_t stage, int32_t k0, int32_t k1, uint32_t* d_rows,
                                int64_t curve_stride, void* stream) {
  return guarded([&] {
    if (!pl || curve_stride < 0) throw ApiError(CTG_INVALID, "plan: null or negative stride");
    PlanDeviceGuard g(pl->device);
    plan_stage(pl, stage, k0, k1, d_rows, curve_stride, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_interp_cols(ctg_plan* pl, int32_t k0, int32_t k1, uint32_t* d_rows, int64_t curve_stride,
                                int32_t nranks, int32_t row_block, uint32_t* d_send, void* stream) {
  return guarded([&] {
    if (!pl || !d_send || curve_stride < 0) throw ApiError(CTG_INVALID, "plan: null or negative stride");
    if (nranks < 1 || nranks > kMaxScatter) throw ApiError(CTG_INVALID, "plan: interp_cols supports 1..8 ranks");
    if (row_block < k1 - k0 || row_block < 1) throw ApiError(CTG_INVALID, "plan: row_block < k1 - k0");
    PlanDeviceGuard g(pl->device);
    const int D = static_cast<int>(pl->D), Jb = (D + nranks - 1) / nranks;
    RowScatter sc{};
    sc.G = nranks;
    sc.Jb = Jb;
    for (int r = 0; r < nranks; ++r) sc.dst[r] = d_send + static_cast<size_t>(r) * pl->B * row_block * Jb;
    sc.shard_off = 0;
    sc.curve_stride = static_cast<long long>(row_block) * Jb;
    plan_stage(pl, 3, k0, k1, d_rows, curve_stride, resolve_stream(pl->device, stream), &sc);
  });
}

ctg_status ctg_plan_crt_cols(ctg_plan* pl, const uint32_t* d_recv, int32_t nranks, int32_t rank, int32_t row_block,
                             uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl || !d_recv) throw ApiError(CTG_INVALID, "plan: null");
    if (nranks < 1 || rank < 0 || rank >= nranks || row_block < 1)
      throw ApiError(CTG_INVALID, "plan: bad nranks / rank / row_block");
    PlanDeviceGuard g(pl->device);
    const int D = static_cast<int>(pl->D), Jb = (D + nranks - 1) / nranks;
    const int j0 = std::min(rank * Jb, D), j1 = std::min((rank + 1) * Jb, D);
    plan_crt(pl, d_recv, static_cast<long long>(row_block) * Jb, row_block,
             static_cast<long long>(pl->B) * row_block * Jb, j0, j1, d_out, 0, resolve_stream(pl->device, stream),
             /*pitch=*/Jb, /*col0=*/j0);
  });
}

ctg_status ctg_plan_crt(ctg_plan* pl, const uint32_t* d_all, int32_t j0, int32_t j1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_crt(pl, d_all, 0, 0, 0, j0, j1, d_out, 0, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_crt_sharded(ctg_plan* pl, const uint32_t* d_all, int32_t row_block, int64_t block_stride,
                                int32_t j0, int32_t j1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    if (row_block <= 0 || block_stride < 0) throw ApiError(CTG_INVALID, "plan: bad row_block / block_stride");
    PlanDeviceGuard g(pl->device);
    plan_crt(pl, d_all, 0, row_block, block_stride, j0, j1, d_out, 0, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_crt_batch(ctg_plan* pl, const uint32_t* d_all, int64_t curve_stride, int32_t row_block,
                              int64_t block_stride, int32_t j0, int32_t j1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl || curve_stride < 0 || row_block < 0 || block_stride < 0)
      throw ApiError(CTG_INVALID, "plan: null or negative layout argument");
    PlanDeviceGuard g(pl->device);
    plan_crt(pl, d_all, curve_stride, row_block, block_stride, j0, j1, d_out, 0,
             resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_decode(ctg_plan* pl, const uint32_t* h_crt, ctg_upoly_buf* out) {
  return guarded([&] {
    if (!pl || !out) throw ApiError(CTG_INVALID, "plan: null");
    plan_decode(pl, h_crt, out);
  });
}

ctg_status ctg_plan_check(ctg_plan* pl, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    const uint32_t bits = plan_error_bits(pl, resolve_stream(pl->device, stream));
    if (bits) throw ApiError(CTG_INTERNAL, "device self-check failed (error bits " + std::to_string(bits) + ")");
  });
}

int32_t ctg_plan_launches(const ctg_plan* pl) { return pl ? pl->launches : 0; }

void ctg_plan_destroy(ctg_plan* pl) {
  if (!pl) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(pl->device);
  delete pl;
  cudaSetDevice(prev);
}

ctg_status ctg_resultant_batch(int32_t batch, const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                               ctg_upoly_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out || !p || !q || batch < 0) throw ApiError(CTG_INVALID, "resultant_batch: bad arguments");
    CallTimer timer;
    for (int b = 0; b < batch; ++b) std::memset(&out[b], 0, sizeof(out[b]));
    if (opts && (opts->comm || opts->n_devices > 1)) {  // prime-sharded over several GPUs
      try {
        resultant_batch_sharded(batch, p, q, eliminate_x, out, opts);
      } catch (...) {
        for (int b = 0; b < batch; ++b) ctg_upoly_free(&out[b]);
        throw;
      }
      timer.finish_total();
      return;
    }
    std::vector<Problem> probs(batch);
    auto& st = stats_tls();
    // The device is touched only once a nontrivial problem exists (zero inputs and input
    // errors behave as before, without a GPU).
    std::unique_ptr<DeviceGuard> guard;
    std::unique_lock<std::mutex> lock;
    std::unique_ptr<ChunkPipeline> pipe;
    int dev = -1;
    // Blocks of consecutive curves: parse, group by shape, plan and enqueue one block while the
    // GPU runs the previous one (each shape group of a block is one batched plan = one launch
    // set).  The first and last blocks are small (they are the exposed head -- host parsing
    // before the GPU starts -- and tail -- the last D2H and decode); the middle ones are large
    // (fewer, fuller launches).  E.g. 256 curves -> 32 | 64 | 64 | 64 | 32, 64 -> 8 | 16 | 16 | 16 | 8.
    std::vector<int> bounds{0};
    if (batch <= 32) {
      bounds.push_back(batch);
    } else {
      static const int kMidForced = [] {  // largest middle block (CTG_BLOCK_MAX, for experiments)
        const char* e = std::getenv("CTG_BLOCK_MAX");
        return e ? std::max(8, std::atoi(e)) : 0;
      }();
      static const int kHead = [] {
        const char* e = std::getenv("CTG_BLOCK_HEAD");
        return e ? std::max(4, std::atoi(e)) : 32;
      }();
      const int s0 = std::min(kHead, std::max(8, batch / 8));
      // big results: at least three middle blocks (up to 64 curves each): with the priority streams a chunk's
      // D2H and decode overlap the later chunks' kernels, which needs chunks to overlap
      // (scripts/ab_blocks_big.sh, 64 curves: 8|48|8 -> 8|16|16|16|8 took d16/1024 e2e from 3.05
      // to 4.21e9 units/s and d30 from 2.01 to 2.35e9; 256 curves keep 32|64|64|64|32)
      const int mid = batch - 2 * s0;
      // Result size of the first curve, roughly deg^2 coefficients of deg * bits bits (d20/64:
      // 64 KB, d30/128: 430 KB, d16/1024: 520 KB, d10/10: 1 KB): small results (launch-bound
      // chunks, cheap decode: d10, 64 curves, e2e 0.21 vs 0.13e9 units/s) keep 64-curve middle blocks;
      // d20 with 64 curves splits (e2e 1.49 -> 2.71e9).
      double est_bytes = 0;
      {
        const ctg_bipoly& f = p[0];
        int deg = 0;
        uint32_t maxl = 0;
        const int32_t nt = (f.dx && f.dy && f.limb_off) ? f.n_terms : 0;  // (inputs are validated later)
        for (int32_t t = 0; t < nt; ++t) {
          deg = std::max(deg, f.dx[t] + f.dy[t]);
          maxl = std::max(maxl, f.limb_off[t + 1] - f.limb_off[t]);
        }
        est_bytes = static_cast<double>(deg) * deg * deg * 32.0 * maxl / 8.0;
      }
      const bool big_out = est_bytes > 20e3;
      const int kMid = kMidForced ? kMidForced : big_out ? std::min(64, std::max(16, (mid + 2) / 3)) : 64;
      const int nm = (mid + kMid - 1) / kMid, per = (mid + nm - 1) / nm;
      bounds.push_back(s0);
      for (int k = 0; k < nm; ++k) bounds.push_back(std::min(s0 + mid, bounds.back() + per));
      bounds.push_back(batch);
    }
    auto pipeline = [&]() -> ChunkPipeline& {
      if (!pipe) {
        guard = std::make_unique<DeviceGuard>(opts);
        dev = select_device(opts);
        Ctx& ctx = context(dev);
        lock = std::unique_lock<std::mutex>(ctx.mu);
        // CTG_NO_R_PROBE=1 drops the probe left behind single-curve results (A/B only)
        static const bool no_probe = std::getenv("CTG_NO_R_PROBE") != nullptr;
        pipe = std::make_unique<ChunkPipeline>(ctx, out, bounds.size() >= 6 ? 3 : 2,
                                               /*probe_r=*/batch == 1 && !no_probe);
      }
      return *pipe;
    };
    bool reserved = false;
    double t_parse = 0, t_plan = 0;
    using tclk = std::chrono::steady_clock;
    try {
      for (size_t blk = 0; blk + 1 < bounds.size(); ++blk) {
        const int b0 = bounds[blk], b1 = bounds[blk + 1];
        if (b1 <= b0) continue;
        auto t0 = tclk::now();
        parallel_for(b1 - b0, [&](int i) { probs[b0 + i] = parse_problem(&p[b0 + i], &q[b0 + i], eliminate_x); });
        std::map<std::tuple<int, int, int, int>, std::vector<int>> groups;
        for (int b = b0; b < b1; ++b) {
          if (probs[b].trivial) {
            fill_upoly({}, &out[b]);
            continue;
          }
          groups[{probs[b].n, probs[b].m, probs[b].deriv, probs[b].negate}].push_back(b);
        }
        auto t1 = tclk::now();
        t_parse += std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (auto& [key, idx] : groups) {
          ChunkPipeline& pl_run = pipeline();
          Chunk c;
          c.idx = idx;
          c.pl.reset(plan_build(probs, c.idx, dev));
          st.n_primes = std::max(st.n_primes, c.pl->P);
          st.n_points = static_cast<int32_t>(c.pl->N);
          st.n_coeffs = static_cast<int32_t>(c.pl->D);
          st.out_limbs = std::max(st.out_limbs, c.pl->out_limbs());
          if (!reserved) {  // size the slots for the largest block from the first plan
            const ChunkNeeds n = chunk_needs(c.pl.get());
            int max_block = 1;
            for (size_t q = 0; q + 1 < bounds.size(); ++q) max_block = std::max(max_block, bounds[q + 1] - bounds[q]);
            // (capped: a first group of one large curve must not reserve max_block times its
            // needs -- enqueue() regrows the slots when a later chunk does not fit)
            const double f = 0.1 + std::min(4.0, std::max(1.0, static_cast<double>(max_block) / c.pl->B));
            pl_run.reserve({static_cast<size_t>(f * n.dev), static_cast<size_t>(f * n.in),
                            static_cast<size_t>(f * n.out)});
            reserved = true;
          }
          t_plan += std::chrono::duration<double, std::milli>(tclk::now() - t1).count();
          pl_run.enqueue(std::move(c));
          t1 = tclk::now();
        }
        // the plans hold their own copies of the limbs: release this block's parsed terms
        // now, while the GPU works, instead of after the last decode
        parallel_for(b1 - b0, [&](int i) { probs[b0 + i] = Problem(); });
      }
      if (pipe) pipe->finish();
    } catch (...) {
      pipe.reset();  // waits for copies in flight
      for (int b = 0; b < batch; ++b) ctg_upoly_free(&out[b]);
      throw;
    }
    st.setup_ms = t_parse + t_plan;
    timer.finish_total();
    static const bool trace = std::getenv("CTG_TRACE_HOST") != nullptr;
    if (trace)
      std::fprintf(stderr, "[ctg] batch %d: parse %.3f ms, plan %.3f ms, enqueue %.3f ms, wait %.3f ms, decode %.3f ms, total %.3f ms\n",
                   batch, t_parse, t_plan, st.h2d_ms, st.device_ms, st.decode_ms, st.total_ms);
  });
}

ctg_status ctg_resultant(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x, ctg_upoly_buf* out,
                         const ctg_opts* opts) {
  return ctg_resultant_batch(1, p, q, eliminate_x, out, opts);
}

}  // extern "C"
