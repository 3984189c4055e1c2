// C ABI of the multi-modular resultant (include/ctg.h): plan construction,
// prime/constant caching, H2D/D2H staging and result decoding.
//
// Replaces curvetop::resultant (/root/reference/proj/src/elim.cpp:95-136) for
// every pair of nonzero inputs: the conventions of elim.cpp:97-104 (Var::X swap,
// zero inputs, degree-0 operands) fall out of the formal-degree Sylvester
// resultant computed on the device; only "both zero" (PreconditionError) and
// "one zero" (zero polynomial) are decided on the host without computation.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "api_common.hpp"
#include "internal.hpp"

namespace ctg {

// Cached per-(device, N, P) prime tables for the resultant path.
static std::shared_ptr<CrtTables> get_tables(int device, uint32_t N, int P, const std::vector<uint32_t>& primes) {
  static std::mutex mu;
  static std::map<std::tuple<int, uint32_t, int>, std::shared_ptr<CrtTables>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(device, N, P);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto T = build_tables(device, primes, N);
  cache[key] = T;
  return T;
}

// ---------------------------------------------------------------------------
// Input parsing (sparse map keyed (dy, dx), zero terms dropped -- bipoly.cpp:7-15)
// ---------------------------------------------------------------------------
using TermMap = std::map<std::pair<int, int>, SBig>;  // (dy, dx) -> coefficient

static TermMap parse_bipoly(const ctg_bipoly* f, bool swap_xy) {
  TermMap t;
  if (!f || f->n_terms == 0) return t;
  if (f->n_terms < 0 || !f->dx || !f->dy || !f->sign || !f->limb_off || (!f->limbs && f->limb_off[f->n_terms] > 0))
    throw ApiError(CTG_INVALID, "bipoly: null pointer or negative term count");
  for (int i = 0; i < f->n_terms; ++i) {
    int dx = f->dx[i], dy = f->dy[i];
    if (dx < 0 || dy < 0) throw ApiError(CTG_INVALID, "bipoly: negative exponent");
    if (swap_xy) std::swap(dx, dy);
    const uint32_t b = f->limb_off[i], e = f->limb_off[i + 1];
    if (e < b) throw ApiError(CTG_INVALID, "bipoly: limb_off not monotone");
    int s = f->sign[i];
    if (s < -1 || s > 1) throw ApiError(CTG_INVALID, "bipoly: sign must be -1, 0 or +1");
    sbig_add_inplace(t[{dy, dx}], s, f->limbs + b, static_cast<int>(e - b));
  }
  for (auto it = t.begin(); it != t.end();) it = (it->second.sign == 0) ? t.erase(it) : std::next(it);
  return t;
}

static int deg_y(const TermMap& t) { return t.empty() ? -1 : t.rbegin()->first.first; }

static bool is_y_derivative(const TermMap& p, const TermMap& q) {
  size_t cnt = 0;
  for (const auto& [e, c] : p) {
    if (e.first == 0) continue;
    ++cnt;
    auto it = q.find({e.first - 1, e.second});
    if (it == q.end() || it->second.sign != c.sign) return false;
    Big want = big_mul_small(c.mag.data(), static_cast<int>(c.mag.size()), static_cast<uint32_t>(e.first));
    if (big_cmp(want, it->second.mag) != 0) return false;
  }
  return cnt == q.size();
}

}  // namespace ctg

using namespace ctg;

struct ctg_plan {
  int device = 0;
  bool trivial = false;
  int trivial_kind = 0;  // 0: zero polynomial
  int n = 0, m = 0, deriv = 0, negate = 0;
  uint32_t D = 0, N = 0, r = 1, a = 0;
  int P = 0, S = 0, L = 1;
  double bound_bits = 0;
  std::vector<int32_t> dir;
  std::vector<uint32_t> h_limbs;  // [L][S]
  std::vector<int8_t> h_sign;     // [S]
  std::shared_ptr<CrtTables> tabs;
  // device state
  uint32_t* d_limbs = nullptr;
  int8_t* d_sign = nullptr;
  int32_t* d_dir = nullptr;
  uint32_t* d_tab = nullptr;
  uint32_t* d_flags = nullptr;
  uint32_t* d_counters = nullptr;
  uint32_t flag_cap = 1u << 16;
  uint32_t* d_Y = nullptr;
  int64_t* d_tq = nullptr;
  uint64_t* d_cols = nullptr;
  int crt_cap = 0;
  int launches = 0;
  bool uploaded = false;
  ~ctg_plan() {
    cudaFree(d_limbs);
    cudaFree(d_sign);
    cudaFree(d_dir);
    cudaFree(d_tab);
    cudaFree(d_flags);
    cudaFree(d_counters);
    cudaFree(d_Y);
    cudaFree(d_tq);
    cudaFree(d_cols);
  }
  int out_limbs() const { return tabs ? tabs->LM : 0; }
};

namespace ctg {

static void build_slots(const TermMap& t, int deg, int& S, std::vector<int32_t>& off, std::vector<int32_t>& len,
                        std::vector<std::pair<int, const SBig*>>& slot_vals) {
  off.assign(deg + 1, 0);
  len.assign(deg + 1, 0);
  std::vector<int> X(deg + 1, -1);
  for (const auto& [e, c] : t) X[e.first] = std::max(X[e.first], e.second);
  for (int j = 0; j <= deg; ++j) {
    off[j] = S;
    len[j] = X[j] + 1;
    S += len[j];
  }
  slot_vals.resize(S, {0, nullptr});
  for (const auto& [e, c] : t) slot_vals[off[e.first] + e.second] = {1, &c};
}

ctg_plan* plan_build(const ctg_bipoly* pin, const ctg_bipoly* qin, int32_t eliminate_x, const ctg_opts* opts) {
  std::unique_ptr<ctg_plan> pl(new ctg_plan());
  TermMap p = parse_bipoly(pin, eliminate_x != 0), q = parse_bipoly(qin, eliminate_x != 0);
  // Conventions of elim.cpp:98-100.
  if (p.empty() && q.empty()) throw ApiError(CTG_PRECONDITION, "resultant: both inputs identically zero");
  pl->device = select_device(opts);
  if (p.empty() || q.empty()) {
    pl->trivial = true;
    pl->trivial_kind = 0;
    return pl.release();
  }
  int n = deg_y(p), m = deg_y(q);
  if (n < m) {
    std::swap(p, q);
    std::swap(n, m);
    pl->negate = (n & 1) && (m & 1);  // res(p,q) = (-1)^{nm} res(q,p)
  }
  pl->n = n;
  pl->m = m;
  if (n > kGeneralMaxDeg) throw ApiError(CTG_UNSUPPORTED, "resultant: degree in the eliminated variable exceeds 128");
  pl->deriv = (m == n - 1 && n >= 1 && is_y_derivative(p, q)) ? 1 : 0;

  // Slots and limbs.
  std::vector<int32_t> offp, lenp, offq, lenq;
  std::vector<std::pair<int, const SBig*>> vals;
  int S = 0;
  build_slots(p, n, S, offp, lenp, vals);
  if (!pl->deriv) {
    build_slots(q, m, S, offq, lenq, vals);
  } else {
    offq.assign(m + 1, 0);
    lenq.assign(m + 1, 0);
  }
  pl->S = S;
  int L = 1;
  for (auto& v : vals)
    if (v.second) L = std::max<int>(L, static_cast<int>(v.second->mag.size()));
  pl->L = L;
  pl->h_limbs.assign(static_cast<size_t>(L) * S, 0u);
  pl->h_sign.assign(S, 0);
  for (int s = 0; s < S; ++s) {
    if (!vals[s].second) continue;
    const SBig& c = *vals[s].second;
    pl->h_sign[s] = static_cast<int8_t>(c.sign);
    for (size_t l = 0; l < c.mag.size(); ++l) pl->h_limbs[l * S + s] = c.mag[l];
  }
  pl->dir.clear();
  pl->dir.insert(pl->dir.end(), offp.begin(), offp.end());
  pl->dir.insert(pl->dir.end(), lenp.begin(), lenp.end());
  pl->dir.insert(pl->dir.end(), offq.begin(), offq.end());
  pl->dir.insert(pl->dir.end(), lenq.begin(), lenq.end());

  // Degree bound of the result (min of the Sylvester row bound and Bezout).
  int Xp = 0, Xq = 0, tp = 0, tq = 0;
  for (const auto& [e, c] : p) {
    Xp = std::max(Xp, e.second);
    tp = std::max(tp, e.first + e.second);
  }
  for (const auto& [e, c] : q) {
    Xq = std::max(Xq, e.second);
    tq = std::max(tq, e.first + e.second);
  }
  const int64_t row_bound = static_cast<int64_t>(m) * Xp + static_cast<int64_t>(n) * Xq;
  const int64_t bez = static_cast<int64_t>(tp) * tq;
  const int64_t degb = std::min(row_bound, bez);
  if (degb + 1 > kMaxNtt) throw ApiError(CTG_UNSUPPORTED, "resultant: degree bound of the result exceeds 16383");
  pl->D = static_cast<uint32_t>(degb + 1);
  pl->N = choose_ntt_size(pl->D, &pl->r, &pl->a);

  // Hadamard bound over |x| = 1.
  auto norm_bits = [](const TermMap& t, int deg) {
    std::vector<std::vector<double>> per(deg + 1);
    for (const auto& [e, c] : t) per[e.first].push_back(log2_upper(c.mag.data(), static_cast<int>(c.mag.size())));
    std::vector<double> sq;
    for (auto& v : per) {
      double l1 = log2_sum_upper(v);
      if (std::isfinite(l1)) sq.push_back(2 * l1);
    }
    return log2_sum_upper(sq);
  };
  const double bp = norm_bits(p, n), bq = norm_bits(q, m);
  pl->bound_bits = 0.5 * m * (std::isfinite(bp) ? bp : 0) + 0.5 * n * (std::isfinite(bq) ? bq : 0);
  if (pl->bound_bits < 0) pl->bound_bits = 0;
  const double need = pl->bound_bits + 1 + 36;
  std::vector<uint32_t> primes = select_primes(pl->N, need);
  pl->P = static_cast<int>(primes.size());
  pl->tabs = get_tables(pl->device, pl->N, pl->P, primes);
  return pl.release();
}

static void plan_alloc(ctg_plan* pl) {
  if (pl->d_tab) return;
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_limbs, sizeof(uint32_t) * std::max<size_t>(1, pl->h_limbs.size())));
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_sign, std::max<size_t>(1, pl->h_sign.size())));
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_dir, sizeof(int32_t) * pl->dir.size()));
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_tab, sizeof(uint32_t) * std::max<size_t>(1, static_cast<size_t>(pl->P) * pl->S)));
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_flags, sizeof(uint32_t) * pl->flag_cap));
  CTG_CUDA_CHECK(cudaMalloc(&pl->d_counters, sizeof(uint32_t) * 4));
  CTG_CUDA_CHECK(cudaMemset(pl->d_counters, 0, sizeof(uint32_t) * 4));
}

void plan_upload(ctg_plan* pl, cudaStream_t st) {
  if (pl->trivial) return;
  plan_alloc(pl);
  CTG_CUDA_CHECK(cudaMemcpyAsync(pl->d_limbs, pl->h_limbs.data(), sizeof(uint32_t) * pl->h_limbs.size(),
                                 cudaMemcpyHostToDevice, st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(pl->d_sign, pl->h_sign.data(), pl->h_sign.size(), cudaMemcpyHostToDevice, st));
  CTG_CUDA_CHECK(
      cudaMemcpyAsync(pl->d_dir, pl->dir.data(), sizeof(int32_t) * pl->dir.size(), cudaMemcpyHostToDevice, st));
  pl->uploaded = true;
}

int64_t plan_h2d_bytes(const ctg_plan* pl) {
  return static_cast<int64_t>(sizeof(uint32_t) * pl->h_limbs.size() + pl->h_sign.size() + 4 * pl->dir.size());
}

void plan_stage(ctg_plan* pl, int stage, int k0, int k1, uint32_t* d_rows, cudaStream_t st) {
  if (pl->trivial) return;
  if (!pl->uploaded) throw ApiError(CTG_INVALID, "plan: inputs not uploaded");
  if (k0 < 0 || k1 > pl->P || k0 > k1) throw ApiError(CTG_INVALID, "plan: prime range out of bounds");
  if (stage < 1 || stage > 3) throw ApiError(CTG_INVALID, "plan: stage must be 1, 2 or 3");
  const int nk = k1 - k0;
  if (nk == 0) return;
  if (stage == 1) {
    pl->launches += launch_reduce(pl->d_limbs, pl->d_sign, pl->S, pl->L, pl->tabs->d_pc, k0, nk, pl->d_tab, st);
    CTG_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (stage == 3) {
    pl->launches += launch_interp(d_rows, static_cast<int>(pl->N), nk, pl->tabs->d_pc, k0, static_cast<int>(pl->N),
                                  static_cast<int>(pl->r), static_cast<int>(pl->a), static_cast<int>(pl->D),
                                  pl->negate, pl->d_counters, st);
    CTG_CUDA_CHECK(cudaGetLastError());
    return;
  }
  CTG_CUDA_CHECK(cudaMemsetAsync(pl->d_counters, 0, sizeof(uint32_t), st));
  ResParams rp{};
  rp.tab = pl->d_tab;
  rp.S = pl->S;
  rp.pc = pl->tabs->d_pc;
  rp.k0 = k0;
  rp.rows = d_rows;
  rp.pitch = static_cast<int>(pl->N);
  rp.N = static_cast<int>(pl->N);
  rp.n = pl->n;
  rp.m = pl->m;
  rp.deriv = pl->deriv;
  rp.dir = pl->d_dir;
  rp.flag_list = pl->d_flags;
  rp.counters = pl->d_counters;
  rp.flag_cap = pl->flag_cap;
  pl->launches += launch_modres(rp, nk, true, st);
  CTG_CUDA_CHECK(cudaGetLastError());
}

void plan_residues(ctg_plan* pl, int k0, int k1, uint32_t* d_rows, cudaStream_t st) {
  for (int stage = 1; stage <= 3; ++stage) plan_stage(pl, stage, k0, k1, d_rows, st);
}

void plan_crt(ctg_plan* pl, const uint32_t* d_all, int j0, int j1, uint32_t* d_out, cudaStream_t st,
              int row_block = 0, long long block_stride = 0) {
  if (pl->trivial) return;
  if (j0 < 0 || j1 > static_cast<int>(pl->D) || j0 > j1) throw ApiError(CTG_INVALID, "plan: coefficient range out of bounds");
  const int J = j1 - j0;
  if (J == 0) return;
  if (J > pl->crt_cap) {
    cudaFree(pl->d_Y);
    cudaFree(pl->d_tq);
    cudaFree(pl->d_cols);
    CTG_CUDA_CHECK(cudaMalloc(&pl->d_Y, sizeof(uint32_t) * static_cast<size_t>(pl->P) * J));
    CTG_CUDA_CHECK(cudaMalloc(&pl->d_tq, sizeof(int64_t) * J));
    CTG_CUDA_CHECK(cudaMalloc(&pl->d_cols, sizeof(uint64_t) * static_cast<size_t>(pl->tabs->L16) * J));
    pl->crt_cap = J;
  }
  CrtParams cp{};
  cp.rows = d_all;
  cp.pitch = static_cast<int>(pl->N);
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
  cp.tq = pl->d_tq;
  cp.cols = pl->d_cols;
  cp.out = d_out;
  cp.out_limbs = pl->tabs->LM;
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

void plan_decode(const ctg_plan* pl, const uint32_t* h, ctg_upoly_buf* out) {
  std::vector<UCoeff> coeffs;
  if (!pl->trivial) {
    const int W = pl->out_limbs() + 1;
    coeffs.resize(pl->D);
    for (uint32_t j = 0; j < pl->D; ++j) {
      const uint32_t* rec = h + static_cast<size_t>(j) * W;
      UCoeff& c = coeffs[j];
      c.sign = static_cast<int8_t>(static_cast<int32_t>(rec[0]));
      int n = W - 1;
      while (n > 0 && rec[n] == 0) --n;
      c.limbs.assign(rec + 1, rec + 1 + n);
      if (c.limbs.empty()) c.sign = 0;
    }
  }
  fill_upoly(coeffs, out);
}

}  // namespace ctg

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

ctg_status ctg_plan_create(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x, const ctg_opts* opts,
                           ctg_plan** plan) {
  return guarded([&] {
    if (!plan) throw ApiError(CTG_INVALID, "plan: null output pointer");
    DeviceGuard g(opts);
    *plan = plan_build(p, q, eliminate_x, opts);
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
    info->work_mulmods = static_cast<double>(pl->P) * pl->D * (n * n + n - 2);
    info->h2d_bytes = plan_h2d_bytes(pl);
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
    plan_residues(pl, k0, k1, d_rows, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_stage(ctg_plan* pl, int32_t stage, int32_t k0, int32_t k1, uint32_t* d_rows, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_stage(pl, stage, k0, k1, d_rows, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_crt(ctg_plan* pl, const uint32_t* d_all, int32_t j0, int32_t j1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    PlanDeviceGuard g(pl->device);
    plan_crt(pl, d_all, j0, j1, d_out, resolve_stream(pl->device, stream));
  });
}

ctg_status ctg_plan_crt_sharded(ctg_plan* pl, const uint32_t* d_all, int32_t row_block, int64_t block_stride,
                                int32_t j0, int32_t j1, uint32_t* d_out, void* stream) {
  return guarded([&] {
    if (!pl) throw ApiError(CTG_INVALID, "plan: null");
    if (row_block <= 0 || block_stride < 0) throw ApiError(CTG_INVALID, "plan: bad row_block / block_stride");
    PlanDeviceGuard g(pl->device);
    plan_crt(pl, d_all, j0, j1, d_out, resolve_stream(pl->device, stream), row_block, block_stride);
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

ctg_status ctg_resultant(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x, ctg_upoly_buf* out,
                         const ctg_opts* opts) {
  return guarded([&] {
    if (!out) throw ApiError(CTG_INVALID, "resultant: null output");
    CallTimer timer;
    DeviceGuard g(opts);
    std::unique_ptr<ctg_plan> pl(plan_build(p, q, eliminate_x, opts));
    timer.mark_setup();
    auto& st = stats_tls();
    st.n_primes = pl->P;
    st.n_points = static_cast<int32_t>(pl->N);
    st.n_coeffs = static_cast<int32_t>(pl->D);
    st.out_limbs = pl->out_limbs();
    if (pl->trivial) {
      plan_decode(pl.get(), nullptr, out);
      timer.finish();
      return;
    }
    Ctx& ctx = context(pl->device);
    std::lock_guard<std::mutex> lock(ctx.mu);
    cudaStream_t s = ctx.stream;
    plan_upload(pl.get(), s);
    st.h2d_bytes = plan_h2d_bytes(pl.get());
    const size_t rows_words = static_cast<size_t>(pl->P) * pl->N;
    const size_t out_words = static_cast<size_t>(pl->D) * (pl->out_limbs() + 1);
    uint32_t* d_rows = ctx.scratch_u32(0, rows_words);
    uint32_t* d_out = ctx.scratch_u32(1, out_words);
    timer.mark_h2d();
    plan_residues(pl.get(), 0, pl->P, d_rows, s);
    plan_crt(pl.get(), d_rows, 0, static_cast<int>(pl->D), d_out, s);
    uint32_t* h_out = ctx.pinned_u32(out_words + 4);
    CTG_CUDA_CHECK(cudaMemcpyAsync(h_out, d_out, sizeof(uint32_t) * out_words, cudaMemcpyDeviceToHost, s));
    CTG_CUDA_CHECK(cudaMemcpyAsync(h_out + out_words, pl->d_counters, sizeof(uint32_t) * 2, cudaMemcpyDeviceToHost, s));
    CTG_CUDA_CHECK(cudaStreamSynchronize(s));
    timer.mark_device();
    st.d2h_bytes = static_cast<int64_t>(sizeof(uint32_t) * (out_words + 2));
    st.kernel_launches = pl->launches;
    st.flagged_units = static_cast<int32_t>(h_out[out_words]);
    const uint32_t bits = h_out[out_words + 1];
    if (bits) throw ApiError(CTG_INTERNAL, "resultant: device self-check failed (error bits " + std::to_string(bits) + ")");
    plan_decode(pl.get(), h_out, out);
    timer.finish();
  });
}

}  // extern "C"
