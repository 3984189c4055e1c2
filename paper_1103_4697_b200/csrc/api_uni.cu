// C ABI of the modular univariate path: gcd_univariate, yun_squarefree, square_free_part.
//
//   ctg_gcd_univariate    replaces curvetop::gcd_univariate  (/root/reference/proj/src/elim.cpp:80-93)
//   ctg_yun_squarefree    replaces curvetop::yun_squarefree  (elim.cpp:138-165)
//   ctg_square_free_part  replaces curvetop::square_free_part (elim.cpp:204-210)
//
// Method: images modulo many 31-bit primes on the GPU
// (K1 reduce, K6 per-prime gcd / Yun), lucky-prime selection by degree pattern,
// CRT of leading-coefficient-scaled images (K5), then an exactness certificate:
//   gcd:  g U = e A and g W = e B hold modulo every CRT prime by construction; the
//         norm bounds ||g||_1 ||U||_1 < M/2 and |e| ||A||_inf < M/2 make them exact
//         over Z, so g | A, g | B, and deg g = min mod-p degree >= deg gcd(A, B).
//   Yun:  P = prod r_m^m modulo every CRT prime iff prod lc(r_m)^m = lc(P) (checked
//         exactly); with sum_m m log||r_m||_1 < log(M/2) the identity is exact.  The r_m
//         are square-free and pairwise coprime modulo a prime not dividing their leading
//         coefficients, hence over Q, so this is THE primitive square-free decomposition
//         the reference returns (it is unique).
// Host work is limited to marshaling, contents (integer gcds of coefficients) and
// the certificate arithmetic on leading coefficients; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "api_common.hpp"
#include "internal.hpp"
#include "uni_internal.hpp"

namespace ctg {
namespace {

using ZPoly = std::vector<SBig>;  // low -> high, trimmed

// One coefficient to reduce: sign and trimmed little-endian u32 magnitude (not owned).
struct Slot {
  int8_t sign;
  const uint32_t* mag;
  int n;
};


// Primes of the univariate path: (2^30, 2^30.4), the window where the fused two-elimination
// pass of blk_gcd (a three-product sum, mmul3) needs one Montgomery reduction.
std::vector<uint32_t> select_uni_primes(double need_bits) { return select_primes(1, need_bits, kResPrimeMax); }

// Square-freeness probe primes: the three largest primes below 2^15 above max(n, 2^14) (a prime
// p not dividing lc(P) with deg gcd(P, P') = 0 mod p certifies P square-free; p > n keeps the
// derivative's degree).  Small primes run the probe in 32-bit arithmetic (lehmer::SmallA).
std::vector<uint32_t> select_probe_primes(int n) {
  std::vector<uint32_t> out;
  const uint32_t lo = std::max<uint32_t>(static_cast<uint32_t>(std::max(n, 0)), 1u << 14);
  for (uint32_t p = (1u << 15) - 1; p > lo && out.size() < 3; p -= 2)
    if (is_prime_u32(p)) out.push_back(p);
  if (out.size() < 3) out.clear();
  return out;
}
constexpr int kProbeMinDeg = 32;  // Yun inputs from this degree get the early square-freeness probe

ZPoly parse_upoly(const ctg_upoly* p) {
  ZPoly out;
  if (!p || p->n_coeffs == 0) return out;
  if (p->n_coeffs < 0 || !p->sign || !p->limb_off || (!p->limbs && p->limb_off[p->n_coeffs] > 0))
    throw ApiError(CTG_INVALID, "upoly: null pointer or negative coefficient count");
  out.resize(p->n_coeffs);
  for (int i = 0; i < p->n_coeffs; ++i) {
    const uint32_t b = p->limb_off[i], e = p->limb_off[i + 1];
    if (e < b) throw ApiError(CTG_INVALID, "upoly: limb_off not monotone");
    const int s = p->sign[i];
    if (s < -1 || s > 1) throw ApiError(CTG_INVALID, "upoly: sign must be -1, 0 or +1");
    uint32_t n = e - b;  // one coefficient per slot: take the limbs as they are (trimmed)
    while (n > 0 && p->limbs[b + n - 1] == 0u) --n;
    if (s == 0 || n == 0) continue;
    out[i].sign = s;
    out[i].mag.assign(p->limbs + b, p->limbs + b + n);
  }
  while (!out.empty() && out.back().sign == 0) out.pop_back();
  return out;
}

int zdeg(const ZPoly& p) { return static_cast<int>(p.size()) - 1; }
// The input equals the polynomial the resultant's probe ran on (signs and limbs, exactly),
// compared with the slot's pinned copy of R's block (the caller has synchronised on its event).
bool probe_matches(const SqfProbeCache& pc, const std::vector<Slot>& slots) {
  const SqfProbeCache::Slot& sl = pc.slot[pc.cur];
  const size_t n = static_cast<size_t>(pc.n) + 1;
  if (!pc.valid || slots.size() != n || !sl.h_blk) return false;
  const uint8_t* block = sl.h_blk + pc.blk_off;
  const uint32_t* off = reinterpret_cast<const uint32_t*>(block + 16);  // after the 16-byte block header
  const uint32_t* limbs = off + (n + 1);
  const int8_t* sign = reinterpret_cast<const int8_t*>(limbs + pc.blk_total);
  if (off[n] != pc.blk_total) return false;
  for (size_t i = 0; i < n; ++i) {
    const Slot& c = slots[i];
    const uint32_t len = off[i + 1] - off[i];
    if (c.sign != sign[i] || static_cast<uint32_t>(c.n) != len) return false;
    if (len && std::memcmp(c.mag, limbs + off[i], 4 * static_cast<size_t>(len)) != 0) return false;
  }
  return true;
}

// The caller's CSR polynomial as trimmed slots (pointers into its limbs; validated like
// parse_upoly; trailing zero coefficients dropped).
std::vector<Slot> view_upoly(const ctg_upoly* p) {
  std::vector<Slot> out;
  if (!p || p->n_coeffs == 0) return out;
  if (p->n_coeffs < 0 || !p->sign || !p->limb_off || (!p->limbs && p->limb_off[p->n_coeffs] > 0))
    throw ApiError(CTG_INVALID, "upoly: null pointer or negative coefficient count");
  out.resize(p->n_coeffs);
  for (int i = 0; i < p->n_coeffs; ++i) {
    const uint32_t b = p->limb_off[i], e = p->limb_off[i + 1];
    if (e < b) throw ApiError(CTG_INVALID, "upoly: limb_off not monotone");
    const int sg = p->sign[i];
    if (sg < -1 || sg > 1) throw ApiError(CTG_INVALID, "upoly: sign must be -1, 0 or +1");
    uint32_t n = e - b;
    while (n > 0 && p->limbs[b + n - 1] == 0u) --n;
    out[i] = (sg == 0 || n == 0) ? Slot{0, nullptr, 0} : Slot{static_cast<int8_t>(sg), p->limbs + b, static_cast<int>(n)};
  }
  while (!out.empty() && out.back().n == 0) out.pop_back();
  return out;
}


// Positive gcd of all coefficients, stopping at 1 (upoly.cpp:59-66).  The coefficients are
// visited shortest first, so the one full-size gcd is between the two smallest and every
// later step is a cheap gcd of a big number with an already small content.
Big zcontent(const ZPoly& p) {
  std::vector<const SBig*> order;
  for (const auto& c : p)
    if (c.sign != 0) order.push_back(&c);
  std::stable_sort(order.begin(), order.end(),
                   [](const SBig* a, const SBig* b) { return a->mag.size() < b->mag.size(); });
  // gcd(g, c) for a one-limb g: c mod g, then a word gcd (no big-integer allocation).
  auto small_gcd = [](uint32_t g, const Big& c) {
    uint32_t r = big_mod_u32(c.data(), static_cast<int>(c.size()), g);
    while (r) {
      const uint32_t t = g % r;
      g = r;
      r = t;
    }
    return g;
  };
  auto step = [&](const Big& g, const Big& c) {
    return g.size() == 1 ? Big{small_gcd(g[0], c)} : big_gcd(g, c);
  };
  auto chain = [&](size_t i0, size_t i1) {
    Big g;
    for (size_t i = i0; i < i1; ++i) {
      g = g.empty() ? order[i]->mag : step(g, order[i]->mag);
      if (big_is_one(g)) break;
    }
    return g;
  };
  if (order.size() <= 32) return chain(0, order.size());
  // Parallel tree: the two smallest coefficients first (usually enough), then groups.
  Big g = chain(0, 2);
  if (big_is_one(g)) return g;
  const int groups = 16;
  std::vector<Big> part(groups);
  const size_t rest = order.size() - 2, per = (rest + groups - 1) / groups;
  parallel_for(groups, [&](int t) {
    const size_t i0 = 2 + t * per, i1 = std::min(order.size(), i0 + per);
    Big h = g;
    for (size_t i = i0; i < i1 && !big_is_one(h); ++i) h = step(h, order[i]->mag);
    part[t] = h;
  });
  for (const Big& h : part) g = big_gcd(g, h);
  return g;
}

// zcontent over slots (the same visiting order and early exit).
Big slots_content(const std::vector<Slot>& p) {
  std::vector<const Slot*> order;
  for (const auto& c : p)
    if (c.n) order.push_back(&c);
  std::stable_sort(order.begin(), order.end(), [](const Slot* a, const Slot* b) { return a->n < b->n; });
  auto big = [](const Slot* c) { return Big(c->mag, c->mag + c->n); };
  auto small_gcd = [](uint32_t g, const Slot* c) {
    uint32_t r = big_mod_u32(c->mag, c->n, g);
    while (r) {
      const uint32_t t = g % r;
      g = r;
      r = t;
    }
    return g;
  };
  // g <- gcd(g, c): a word gcd after c mod g for a one-limb g, else GMP on thread-local scratch
  auto step = [&](Big& g, const Slot* c) {
    if (g.size() == 1)
      g = Big{small_gcd(g[0], c)};
    else
      big_gcd_update(g, c->mag, c->n);
  };
  if (order.empty()) return Big();
  Big g = big(order[0]);
  if (order.size() > 1) g = big_gcd(g, big(order[1]));
  if (big_is_one(g) || order.size() <= 2) return g;
  const int groups = 16;
  std::vector<Big> part(groups);
  const size_t rest = order.size() - 2, per = (rest + groups - 1) / groups;
  parallel_for(groups, [&](int t) {
    const size_t i0 = 2 + t * per, i1 = std::min(order.size(), i0 + per);
    Big h = g;
    for (size_t i = i0; i < i1 && !big_is_one(h); ++i) step(h, order[i]);
    part[t] = h;
  });
  for (const Big& h : part) g = big_gcd(g, h);
  return g;
}

// p / (s * c) for the content c (computed unless given) and s = sign(lc p): primitive with
// positive leading coefficient.
ZPoly divide_content(const ZPoly& p, Big c, Big* content, int* lcsign);

ZPoly zprimitive_positive(const ZPoly& p, Big* content = nullptr, int* lcsign = nullptr) {
  if (p.empty()) return p;
  return divide_content(p, zcontent(p), content, lcsign);
}

// The same, consuming p: a primitive input (content 1, the common case) is returned in place.
ZPoly zprimitive_positive(ZPoly&& p, Big* content = nullptr, int* lcsign = nullptr) {
  if (p.empty()) return std::move(p);
  Big c = zcontent(p);
  if (!big_is_one(c)) return divide_content(p, std::move(c), content, lcsign);
  const int s = p.back().sign;
  if (content) *content = c;
  if (lcsign) *lcsign = s;
  if (s < 0)
    for (auto& x : p) x.sign = -x.sign;
  return std::move(p);
}

ZPoly divide_content(const ZPoly& p, Big c, Big* content, int* lcsign) {
  const int s = p.back().sign;
  if (content) *content = c;
  if (lcsign) *lcsign = s;
  ZPoly q(p.size());
  const bool unit = big_is_one(c);
  parallel_for(static_cast<int>(p.size() + 15) / 16, [&](int blk) {
    const size_t i0 = static_cast<size_t>(blk) * 16, i1 = std::min(p.size(), i0 + 16);
    for (size_t i = i0; i < i1; ++i) {
      if (p[i].sign == 0) continue;
      q[i].sign = p[i].sign * s;
      if (unit) {
        q[i].mag = p[i].mag;
      } else if (c.size() == 1) {
        uint32_t rem = 0;
        q[i].mag = big_div_u32(p[i].mag, c[0], &rem);  // exact: c divides every coefficient
      } else {
        q[i].mag = big_divexact(p[i].mag, c);
      }
    }
  });
  return q;
}

double zlog2_l2(const ZPoly& p) {
  std::vector<double> sq;
  for (const auto& c : p)
    if (c.sign) sq.push_back(2 * big_log2(c.mag));
  return 0.5 * log2_sum_upper(sq);
}
double zlog2_l1(const ZPoly& p) {
  std::vector<double> v;
  for (const auto& c : p)
    if (c.sign) v.push_back(big_log2(c.mag));
  return log2_sum_upper(v);
}
double zlog2_linf(const ZPoly& p) {
  double m = -INFINITY;
  for (const auto& c : p)
    if (c.sign) m = std::max(m, big_log2(c.mag));
  return m;
}

// Device scratch owned by one call.  Small requests are bump-allocated from a per-thread,
// per-device slab (tiny gcds -- realroots.cpp:119,136,196 -- are latency-bound and paid ~1-2 us
// per cudaMallocAsync / cudaFreeAsync pair); arenas nest LIFO and every call of a thread runs
// on its device's context stream, so a region released here is reused only by work that
// stream-orders after the work that used it.  Larger requests use the stream-ordered pool.
struct Slab {
  uint8_t* base = nullptr;
  size_t top = 0, cap = 0;
};
Slab& tls_slab(int device) {
  thread_local std::map<int, Slab> slabs;  // process lifetime (one small region per thread and device)
  Slab& sl = slabs[device];
  if (!sl.base) {
    constexpr size_t kSlabBytes = size_t{8} << 20;
    void* p = nullptr;
    CTG_CUDA_CHECK(cudaMalloc(&p, kSlabBytes));
    sl.base = static_cast<uint8_t*>(p);
    sl.cap = kSlabBytes;
  }
  return sl;
}
struct DevArena {
  cudaStream_t st;
  std::vector<void*> ptrs;
  Slab* slab = nullptr;
  size_t mark = 0;
  explicit DevArena(cudaStream_t s) : st(s) {
    int dev = 0;
    CTG_CUDA_CHECK(cudaGetDevice(&dev));
    slab = &tls_slab(dev);
    mark = slab->top;
  }
  DevArena(const DevArena&) = delete;
  DevArena& operator=(const DevArena&) = delete;
  template <class T>
  T* alloc(size_t n) {
    const size_t bytes = (std::max<size_t>(1, n) * sizeof(T) + 255) & ~static_cast<size_t>(255);
    if (slab->top + bytes <= slab->cap) {
      T* p = reinterpret_cast<T*>(slab->base + slab->top);
      slab->top += bytes;
      return p;
    }
    void* p = nullptr;
    CTG_CUDA_CHECK(cudaMallocAsync(&p, bytes, st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~DevArena() {
    slab->top = mark;
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

struct Launches {
  int n = 0;
};
// Launcher result -> launch count (a negative result means a missing global scratch buffer).
inline int launched(int r) {
  if (r < 0) throw ApiError(CTG_INTERNAL, "K6 launch: global scratch buffer missing");
  return r;
}

// Residues of a primitive polynomial modulo every prime of `tabs` (K1): [P][n+1] Montgomery.
// Per-thread pinned staging for the H2D of reduce_poly (a pageable copy of R's ~1 MB of limbs
// at d30 is staged by the driver at a fraction of the pinned rate).  Reuse waits for the
// previous copy; never freed (process lifetime, no teardown-order hazards).
struct PinnedStage {
  uint8_t* buf = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  int device = -1;
  bool pending = false;
  uint8_t* get(size_t bytes) {
    if (pending) CTG_CUDA_CHECK(cudaEventSynchronize(done));
    pending = false;
    if (bytes > cap) {
      if (buf) cudaFreeHost(buf);
      buf = nullptr;
      cap = 0;
      CTG_CUDA_CHECK(cudaMallocHost(&buf, bytes));
      cap = bytes;
    }
    return buf;
  }
  void mark(cudaStream_t st) {
    int dev = 0;
    CTG_CUDA_CHECK(cudaGetDevice(&dev));
    if (done && dev != device) {
      cudaEventDestroy(done);
      done = nullptr;
    }
    if (!done) CTG_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    device = dev;
    CTG_CUDA_CHECK(cudaEventRecord(done, st));
    pending = true;
  }
};
thread_local PinnedStage tls_stage;

// Coefficients reduced modulo every prime of `tabs` (K1) in ONE staging copy and ONE launch:
// row k of the result holds the slots in order (pitch = slots.size()), Montgomery form.
uint32_t* reduce_slots(DevArena& ar, const std::vector<Slot>& slot, const CrtTables& tabs, Launches& L) {
  const int S = static_cast<int>(slot.size());
  int Lw = 1;
  for (const Slot& c : slot) Lw = std::max(Lw, c.n);
  const size_t nl = static_cast<size_t>(Lw) * S;
  uint8_t* stage = tls_stage.get(4 * nl + S);
  uint32_t* limbs = reinterpret_cast<uint32_t*>(stage);
  int8_t* sign = reinterpret_cast<int8_t*>(stage + 4 * nl);
  // coefficient-major [S][Lw]: one contiguous copy per coefficient (K1 reads either layout),
  // filled in parallel over blocks of 64 slots (a batch stages tens of MB)
  parallel_for((S + 63) / 64, [&](int blk) {
    for (int s = blk * 64; s < std::min(S, blk * 64 + 64); ++s) {
      const Slot& c = slot[s];
      sign[s] = c.sign;
      uint32_t* row = limbs + static_cast<size_t>(s) * Lw;
      if (c.n) std::memcpy(row, c.mag, 4 * static_cast<size_t>(c.n));
      if (c.n < Lw) std::memset(row + c.n, 0, 4 * static_cast<size_t>(Lw - c.n));
    }
  });
  uint32_t* d_limbs = ar.alloc<uint32_t>(nl);
  int8_t* d_sign = ar.alloc<int8_t>(S);
  uint32_t* d_tab = ar.alloc<uint32_t>(static_cast<size_t>(tabs.P) * S);
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_limbs, limbs, 4 * nl, cudaMemcpyHostToDevice, ar.st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_sign, sign, S, cudaMemcpyHostToDevice, ar.st));
  tls_stage.mark(ar.st);
  L.n += launch_reduce(d_limbs, d_sign, S, Lw, tabs.d_pc, tabs.d_rpow, 0, tabs.P, d_tab, static_cast<size_t>(tabs.P) * S, 1,
                       ar.st, 1);
  auto& st = stats_tls();
  st.h2d_bytes += static_cast<int64_t>(4 * nl + S);
  return d_tab;
}

// The staging half of reduce_slots without the K1 launch (kernels that reduce their own inputs):
// coefficient-major limbs [S][Lw] followed by the S signs, ONE H2D copy.
struct StagedSlots {
  const uint32_t* limbs = nullptr;
  const int8_t* sign = nullptr;
  int Lw = 0;
};
template <class List>
StagedSlots stage_polys(DevArena& ar, const List& ps) {
  int S = 0, Lw = 1;
  for (const ZPoly* p : ps)
    for (const auto& c : *p) {
      ++S;
      Lw = std::max(Lw, static_cast<int>(c.mag.size()));
    }
  const size_t nl = static_cast<size_t>(Lw) * S, bytes = 4 * nl + S;
  uint8_t* stage = tls_stage.get(bytes);
  uint32_t* limbs = reinterpret_cast<uint32_t*>(stage);
  int8_t* sign = reinterpret_cast<int8_t*>(stage + 4 * nl);
  int s = 0;
  for (const ZPoly* p : ps)
    for (const auto& c : *p) {
      sign[s] = static_cast<int8_t>(c.sign);
      uint32_t* row = limbs + static_cast<size_t>(s) * Lw;
      const int n = static_cast<int>(c.mag.size());
      if (n) std::memcpy(row, c.mag.data(), 4 * static_cast<size_t>(n));
      if (n < Lw) std::memset(row + n, 0, 4 * static_cast<size_t>(Lw - n));
      ++s;
    }
  uint8_t* d = ar.alloc<uint8_t>(bytes);
  CTG_CUDA_CHECK(cudaMemcpyAsync(d, stage, bytes, cudaMemcpyHostToDevice, ar.st));
  tls_stage.mark(ar.st);
  stats_tls().h2d_bytes += static_cast<int64_t>(bytes);
  return StagedSlots{reinterpret_cast<const uint32_t*>(d), reinterpret_cast<const int8_t*>(d + 4 * nl), Lw};
}

// Several polynomials as consecutive slots of one table (row k = p_0 | p_1 | ...).
template <class List>
uint32_t* reduce_polys(DevArena& ar, const List& ps, const CrtTables& tabs, Launches& L) {
  std::vector<Slot> slot;
  for (const ZPoly* p : ps)
    for (const auto& c : *p) slot.push_back({static_cast<int8_t>(c.sign), c.mag.data(), static_cast<int>(c.mag.size())});
  return reduce_slots(ar, slot, tabs, L);
}

uint32_t* reduce_poly(DevArena& ar, const ZPoly& p, const CrtTables& tabs, Launches& L) {
  return reduce_polys(ar, std::initializer_list<const ZPoly*>{&p}, tabs, L);
}

// Gather rows `lucky` of d_src (plain residues, pitch src_pitch), scale segment s of row r
// by scale[r][s] (plain), CRT the first `cols` columns over the lucky primes.
ZPoly crt_rows(DevArena& ar, const uint32_t* d_src, int src_pitch, const std::vector<int>& lucky,
               const std::vector<uint32_t>& primes, int cols, const std::vector<int32_t>& seg_end,
               const std::vector<uint32_t>& scale_plain, int device, double* log2M, Launches& L) {
  std::vector<uint32_t> lp;
  for (int k : lucky) lp.push_back(primes[k]);
  auto T = get_tables(device, 1, lp);
  const int R = static_cast<int>(lp.size());
  const int nseg = static_cast<int>(seg_end.size());
  std::vector<uint32_t> scale_m(static_cast<size_t>(R) * nseg);
  for (int r = 0; r < R; ++r)
    for (int s = 0; s < nseg; ++s)
      scale_m[static_cast<size_t>(r) * nseg + s] =
          static_cast<uint32_t>((static_cast<uint64_t>(scale_plain[static_cast<size_t>(r) * nseg + s] % lp[r]) << 32) %
                                lp[r]);
  int32_t* d_idx = ar.alloc<int32_t>(R);
  int32_t* d_seg = ar.alloc<int32_t>(nseg);
  uint32_t* d_scale = ar.alloc<uint32_t>(scale_m.size());
  uint32_t* d_rows = ar.alloc<uint32_t>(static_cast<size_t>(R) * cols);
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_idx, lucky.data(), 4 * R, cudaMemcpyHostToDevice, ar.st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_seg, seg_end.data(), 4 * nseg, cudaMemcpyHostToDevice, ar.st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_scale, scale_m.data(), 4 * scale_m.size(), cudaMemcpyHostToDevice, ar.st));
  L.n += launch_gather_scale(d_src, src_pitch, d_idx, R, cols, d_seg, nseg, d_scale, T->d_pc, d_rows, ar.st);
  const int W = T->LM + 1;
  uint32_t* d_out = ar.alloc<uint32_t>(static_cast<size_t>(cols) * W);
  uint32_t* d_Y = ar.alloc<uint32_t>(crt_y_words(*T, 1, cols));
  double* d_upart = ar.alloc<double>(static_cast<size_t>((R + kCrtChunk - 1) / kCrtChunk) * cols);
  uint64_t* d_cols = ar.alloc<uint64_t>((crt_cols_words(*T, 1, cols) + 1) / 2);
  uint32_t* d_cnt = ar.alloc<uint32_t>(4);
  CTG_CUDA_CHECK(cudaMemsetAsync(d_cnt, 0, 16, ar.st));
  CrtParams cp{};
  cp.B = 1;
  cp.rows = d_rows;
  cp.curve_stride = static_cast<long long>(R) * cols;
  cp.pitch = cols;
  cp.P = R;
  cp.row_block = R;
  cp.block_stride = 0;
  cp.j0 = 0;
  cp.J = cols;
  cp.pc = T->d_pc;
  cp.minv = T->d_minv;
  cp.Mk16 = T->d_Mk16;
  cp.M16 = T->d_M16;
  cp.L16 = T->L16;
  cp.Y = d_Y;
  cp.upart = d_upart;
  cp.cols = d_cols;
  cp.out = d_out;
  cp.out_limbs = T->LM;
  cp.use_i8 = T->use_i8 ? 1 : 0;
  cp.Rp = (cols + kI8TileJ - 1) / kI8TileJ * kI8TileJ;
  cp.L8 = T->L8;
  cp.L8p = T->L8p;
  cp.Kp = T->Kp;
  cp.Bt8 = T->d_Bt8;
  cp.M8 = T->d_M8;
  cp.top_digit = cp.L8;
  cp.counters = d_cnt;
  L.n += launch_crt(cp, ar.st);
  CTG_CUDA_CHECK(cudaGetLastError());
  std::vector<uint32_t> h(static_cast<size_t>(cols) * W + 4);
  CTG_CUDA_CHECK(cudaMemcpyAsync(h.data(), d_out, 4 * static_cast<size_t>(cols) * W, cudaMemcpyDeviceToHost, ar.st));
  CTG_CUDA_CHECK(cudaMemcpyAsync(h.data() + static_cast<size_t>(cols) * W, d_cnt, 16, cudaMemcpyDeviceToHost, ar.st));
  CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
  stats_tls().d2h_bytes += static_cast<int64_t>(4 * h.size());
  if (h[static_cast<size_t>(cols) * W + 1]) throw ApiError(CTG_INTERNAL, "CRT self-check failed (bound exceeded)");
  ZPoly out(cols);
  for (int j = 0; j < cols; ++j) {
    const uint32_t* rec = h.data() + static_cast<size_t>(j) * W;
    int n = W - 1;
    while (n > 0 && rec[n] == 0) --n;
    out[j].sign = static_cast<int32_t>(rec[0]);
    out[j].mag.assign(rec + 1, rec + 1 + n);
    if (out[j].mag.empty()) out[j].sign = 0;
  }
  *log2M = T->log2M;
  return out;
}

ZPoly slice(const ZPoly& p, int a, int b) {
  ZPoly r(p.begin() + a, p.begin() + b);
  while (!r.empty() && r.back().sign == 0) r.pop_back();
  return r;
}

// ---------------------------------------------------------------------------
// Yun over Z via per-prime Yun (K6) + CRT (K5) + certificate.
// ---------------------------------------------------------------------------
struct YunResult {
  bool squarefree = false;  // certified square-free: the factorization is (P, 1) and sqfp = P (not copied)
  std::vector<std::pair<ZPoly, int>> factors;
  ZPoly sqfp;
};

struct YunImages {
  std::vector<uint32_t> primes;
  std::vector<int32_t> deg;  // [P][n+1]
  int32_t* d_deg = nullptr;
  uint32_t* d_fac = nullptr;
  uint32_t* d_sqf = nullptr;
};

YunImages run_modyun(DevArena& ar, const ZPoly& P, const std::vector<uint32_t>& primes, int device, Launches& L) {
  using tclk = std::chrono::steady_clock;
  static const bool trace = std::getenv("CTG_TRACE_HOST") != nullptr;
  const auto t0 = tclk::now();
  const int n = zdeg(P);
  auto T = get_tables(device, 1, primes);
  const auto t1 = tclk::now();
  uint32_t* d_tab = reduce_poly(ar, P, *T, L);
  const auto t2 = tclk::now();
  const int nk = static_cast<int>(primes.size());
  YunImages im;
  im.primes = primes;
  int32_t* d_deg = ar.alloc<int32_t>(static_cast<size_t>(nk) * (n + 1));
  im.d_fac = ar.alloc<uint32_t>(static_cast<size_t>(nk) * (2 * n + 2));
  im.d_sqf = ar.alloc<uint32_t>(static_cast<size_t>(nk) * (n + 1));
  const size_t gb = uni_gbuf_bytes(modyun_smem(n), nk);
  uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
  L.n += launched(launch_modyun(d_tab, n, T->d_pc, nk, d_deg, im.d_fac, im.d_sqf, gbuf, ar.st));
  CTG_CUDA_CHECK(cudaGetLastError());
  // First only columns 0..1 of every prime's pattern (status, degree of the multiplicity-1
  // factor): enough to certify a square-free input; fetch_patterns() copies the rest.
  im.deg.assign(static_cast<size_t>(nk) * (n + 1), 0);
  im.d_deg = d_deg;
  CTG_CUDA_CHECK(cudaMemcpy2DAsync(im.deg.data(), 4 * static_cast<size_t>(n + 1), d_deg, 4 * static_cast<size_t>(n + 1),
                                   8, nk, cudaMemcpyDeviceToHost, ar.st));
  const auto t3 = tclk::now();
  CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
  if (trace) {
    auto us = [](tclk::time_point a, tclk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "[ctg] run_modyun n=%d P=%zu: tables %.1f us, reduce(stage+h2d+K1) %.1f us, launch %.1f us, sync %.1f us\n",
                 n, primes.size(), us(t0, t1), us(t1, t2), us(t2, t3), us(t3, tclk::now()));
  }
  stats_tls().d2h_bytes += static_cast<int64_t>(8) * nk;
  return im;
}

// The full degree patterns of a run_modyun result.
void fetch_patterns(DevArena& ar, YunImages& im) {
  CTG_CUDA_CHECK(cudaMemcpyAsync(im.deg.data(), im.d_deg, 4 * im.deg.size(), cudaMemcpyDeviceToHost, ar.st));
  CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
  stats_tls().d2h_bytes += static_cast<int64_t>(4 * im.deg.size());
}

// A prime with p !| lc(P) and deg gcd(P, P') = 0 mod p certifies a square-free P.
bool certifies_squarefree(const YunImages& im, int n) {
  for (size_t k = 0; k < im.primes.size(); ++k) {
    const int32_t* d = im.deg.data() + k * (n + 1);
    if (d[0] == 0 && d[1] == n) return true;
  }
  return false;
}

// Square-freeness probe launched BEFORE the host computes the content (elim.cpp:141-144), so
// the content gcd (one full-size integer gcd: ~1 ms at d16/1024) overlaps the GPU: for a
// prime p not dividing lc(R), deg gcd(R mod p, R' mod p) is the same for R and pp(R) = R / c
// (p | c implies p | lc(R), and such primes report status 1 and certify nothing).
struct YunProbe {
  std::unique_ptr<DevArena> ar;
  std::vector<uint32_t> primes;
  int n = -1;
  int32_t* h = nullptr;  // pinned: (status, deg of the multiplicity-1 part) per prime
  cudaEvent_t done = nullptr;
  ~YunProbe() {
    if (done) cudaEventDestroy(done);
  }
};
int32_t* probe_pinned() {
  thread_local int32_t* buf = nullptr;
  if (!buf) CTG_CUDA_CHECK(cudaMallocHost(&buf, 64 * sizeof(int32_t)));
  return buf;
}

// Launches the probe on the coefficient slots of R (deg n): K1 modulo 3 primes and one
// k_sqf_probe CTA per prime (gcd(R, R') mod p only -- the rest of Yun runs only if needed).
void probe_start(YunProbe& pb, const std::vector<Slot>& slots, int n, int device, cudaStream_t st, Launches& L) {
  pb.n = n;
  pb.primes = select_probe_primes(n);
  const bool small = !pb.primes.empty();
  if (!small) pb.primes = select_uni_primes(3 * 30.0);
  pb.ar = std::make_unique<DevArena>(st);
  DevArena& ar = *pb.ar;
  const int nk = static_cast<int>(pb.primes.size());
  auto T = get_tables(device, 1, pb.primes);
  uint32_t* d_tab = reduce_slots(ar, slots, *T, L);
  const int32_t meta_h[2] = {0, n};
  int32_t* d_meta = ar.alloc<int32_t>(2);
  int32_t* d_out = ar.alloc<int32_t>(2 * static_cast<size_t>(nk));
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_meta, meta_h, sizeof(meta_h), cudaMemcpyHostToDevice, ar.st));
  const size_t gb = uni_gbuf_bytes(sqf_probe_smem(n), nk);
  uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
  L.n += launched(launch_sqf_probe(d_tab, static_cast<int>(slots.size()), d_meta, d_meta + 1, 1, nk, T->d_pc, n, d_out,
                                   gbuf, ar.st, 0, small));
  CTG_CUDA_CHECK(cudaGetLastError());
  pb.h = probe_pinned();
  CTG_CUDA_CHECK(cudaMemcpyAsync(pb.h, d_out, 8 * static_cast<size_t>(nk), cudaMemcpyDeviceToHost, ar.st));
  CTG_CUDA_CHECK(cudaEventCreateWithFlags(&pb.done, cudaEventDisableTiming));
  CTG_CUDA_CHECK(cudaEventRecord(pb.done, ar.st));
  stats_tls().d2h_bytes += static_cast<int64_t>(8) * nk;
}

// True if some probe prime certifies the input square-free.
bool probe_finish(YunProbe& pb) {
  CTG_CUDA_CHECK(cudaEventSynchronize(pb.done));
  for (size_t k = 0; k < pb.primes.size(); ++k)
    if (pb.h[2 * k] == 0 && pb.h[2 * k + 1] == 0) return true;  // lc != 0 mod p, deg gcd(R, R') = 0
  return false;
}

YunResult yun_modular(const ZPoly& P, bool want_sqfp, int device, cudaStream_t st, Launches& L, bool probed = false) {
  const int n = zdeg(P);
  DevArena ar(st);
  YunResult res;
  // A prime with p !| lc(P) and deg gcd(P, P') = 0 certifies a square-free P at once (no CRT).
  // When the full prime set fits one wave of CTAs, it is run directly (every prime's Yun runs
  // in parallel: the latency of one prime, and a non-square-free P reuses the same images);
  // beyond that a 3-prime probe first spares square-free inputs (every dense config) the K1
  // and Yun work of hundreds of primes.
  const Big& lcP = P.back().mag;
  const double need = big_log2(lcP) + n + zlog2_l2(P) + 2 + 40;
  if (!probed && select_uni_primes(need + 62).size() > 148) {
    YunImages im = run_modyun(ar, P, select_uni_primes(3 * 30.0), device, L);
    if (certifies_squarefree(im, n)) {
      res.squarefree = true;
      return res;
    }
  }
  double extra = 62;
  for (int attempt = 0; attempt < 4; ++attempt, extra *= 4) {
    std::vector<uint32_t> primes = select_uni_primes(need + extra);
    const int nk = static_cast<int>(primes.size());
    YunImages im = run_modyun(ar, P, primes, device, L);
    if (certifies_squarefree(im, n)) {
      res.squarefree = true;
      return res;
    }
    fetch_patterns(ar, im);
    // lucky pattern: maximal square-free-part degree, then the most frequent pattern
    std::map<std::vector<int32_t>, std::vector<int>> by_pattern;
    int best_sd = -1;
    for (int k = 0; k < nk; ++k) {
      const int32_t* d = im.deg.data() + static_cast<size_t>(k) * (n + 1);
      if (d[0] != 0) continue;
      int sd = 0;
      for (int m = 1; m <= n; ++m) sd += d[m];
      if (sd > best_sd) {
        best_sd = sd;
        by_pattern.clear();
      }
      if (sd == best_sd) by_pattern[std::vector<int32_t>(d + 1, d + n + 1)].push_back(k);
    }
    if (by_pattern.empty()) continue;
    auto best = by_pattern.begin();
    for (auto it = by_pattern.begin(); it != by_pattern.end(); ++it)
      if (it->second.size() > best->second.size()) best = it;
    const std::vector<int32_t>& pat = best->first;
    const std::vector<int>& lucky = best->second;
    double bits = 0;
    for (int k : lucky) bits += std::log2(static_cast<double>(primes[k]));
    if (bits < need) continue;
    // CRT of lc(P) * monic factor images, concatenated in increasing multiplicity.
    std::vector<std::pair<int, int>> fm;  // (multiplicity, degree)
    int cols = 0;
    for (int m = 1; m <= n; ++m)
      if (pat[m - 1] > 0) {
        fm.push_back({m, pat[m - 1]});
        cols += pat[m - 1] + 1;
      }
    std::vector<uint32_t> scale;
    for (int k : lucky) scale.push_back(big_mod(lcP, primes[k]));
    double log2M = 0;
    ZPoly H = crt_rows(ar, im.d_fac, 2 * n + 2, lucky, primes, cols, {cols}, scale, device, &log2M, L);
    // r_m = pp(H_m); certificate
    int off = 0, degsum = 0;
    Big lcprod{1u};
    double normsum = 0;
    for (auto [m, dm] : fm) {
      ZPoly Hm = slice(H, off, off + dm + 1);
      off += dm + 1;
      if (zdeg(Hm) != dm) throw ApiError(CTG_INTERNAL, "yun: factor degree mismatch after CRT");
      ZPoly rm = zprimitive_positive(Hm);
      degsum += m * dm;
      for (int e = 0; e < m; ++e) lcprod = big_mul(lcprod, rm.back().mag);
      normsum += m * zlog2_l1(rm);
      res.factors.push_back({std::move(rm), m});
    }
    const bool ok = degsum == n && big_cmp(lcprod, lcP) == 0 && normsum + 1 < log2M - 1 &&
                    zlog2_linf(P) + 1 < log2M - 1;
    if (!ok) throw ApiError(CTG_INTERNAL, "yun: exactness certificate failed");
    if (want_sqfp) {
      // sqfp = prod r_m: CRT of L * v_p with L = prod lc(r_m) (v_p = monic square-free part mod p).
      Big Lc{1u};
      double l1 = 0;
      int ds = 0;
      for (auto& f : res.factors) {
        Lc = big_mul(Lc, f.first.back().mag);
        l1 += zlog2_l1(f.first);
        ds += zdeg(f.first);
      }
      std::vector<uint32_t> sc;
      for (int k : lucky) sc.push_back(big_mod(Lc, primes[k]));
      double log2M2 = 0;
      ZPoly S = crt_rows(ar, im.d_sqf, n + 1, lucky, primes, ds + 1, {ds + 1}, sc, device, &log2M2, L);
      if (zdeg(S) != ds || big_cmp(S.back().mag, Lc) != 0 || S.back().sign != 1 || !(l1 + 1 < log2M2 - 1))
        throw ApiError(CTG_INTERNAL, "square_free_part: exactness certificate failed");
      res.sqfp = std::move(S);
    }
    return res;
  }
  throw ApiError(CTG_INTERNAL, "yun: could not find enough lucky primes");
}

// ---------------------------------------------------------------------------
// gcd over Z via per-prime gcd + cofactors (K6) + CRT (K5) + certificate.
// ---------------------------------------------------------------------------
ZPoly gcd_modular(const ZPoly& A, const ZPoly& B, int device, cudaStream_t st, Launches& L) {
  const int na = zdeg(A), nb = zdeg(B);
  DevArena ar(st);
  const Big gamma = big_gcd(A.back().mag, B.back().mag);
  const double lg = big_log2(gamma), la = zlog2_l2(A), lb = zlog2_l2(B);
  const double need = std::max({lg + std::min(na, nb) + std::min(la, lb), lg + na + la, lg + nb + lb}) + 2 + 40;
  double extra = 62;
  for (int attempt = 0; attempt < 4; ++attempt, extra *= 4) {
    std::vector<uint32_t> primes = select_uni_primes(need + extra);
    const int nk = static_cast<int>(primes.size());
    auto T = get_tables(device, 1, primes);
    const int pitch = na + nb + 3;
    int32_t* d_deg = ar.alloc<int32_t>(nk);
    uint32_t* d_out = ar.alloc<uint32_t>(static_cast<size_t>(nk) * pitch);
    const size_t gb = uni_gbuf_bytes(modgcd_smem(na, nb), nk);
    uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
    int maxl = 1;
    for (const ZPoly* p : {&A, &B})
      for (const auto& c : *p) maxl = std::max(maxl, static_cast<int>(c.mag.size()));
    if (maxl <= kRedL && na + nb + 2 <= 4096) {
      // small inputs (the realroots / multiplicity_at calls): one staging copy and ONE launch --
      // the gcd kernel reduces the coefficients itself (a GPU round trip is the whole cost)
      const StagedSlots sg = stage_polys(ar, std::initializer_list<const ZPoly*>{&A, &B});
      L.n += launched(launch_modgcd(nullptr, na, nullptr, nb, 0, T->d_pc, nk, d_deg, d_out, pitch, gbuf, ar.st,
                                    sg.limbs, sg.sign, sg.Lw, T->d_rpow));
    } else {
      // one staging copy, one K1 launch for both operands
      const int pitch_ab = na + nb + 2;
      uint32_t* tA = reduce_polys(ar, std::initializer_list<const ZPoly*>{&A, &B}, *T, L);
      uint32_t* tB = tA + (na + 1);
      L.n += launched(launch_modgcd(tA, na, tB, nb, pitch_ab, T->d_pc, nk, d_deg, d_out, pitch, gbuf, ar.st));
    }
    CTG_CUDA_CHECK(cudaGetLastError());
    std::vector<int32_t> deg(nk);
    CTG_CUDA_CHECK(cudaMemcpyAsync(deg.data(), d_deg, 4 * nk, cudaMemcpyDeviceToHost, ar.st));
    CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
    int dmin = INT32_MAX;
    for (int d : deg)
      if (d >= 0) dmin = std::min(dmin, d);
    if (dmin == INT32_MAX) continue;
    if (dmin == 0) return ZPoly{SBig{1, Big{1u}}};  // coprime modulo a prime not dividing lc(A) lc(B)
    std::vector<int> lucky;
    double bits = 0;
    for (int k = 0; k < nk; ++k)
      if (deg[k] == dmin) {
        lucky.push_back(k);
        bits += std::log2(static_cast<double>(primes[k]));
      }
    if (bits < need) continue;
    const int cg = dmin + 1, cu = na - dmin + 1, cw = nb - dmin + 1;
    std::vector<uint32_t> scale;
    for (int k : lucky) {
      scale.push_back(big_mod(gamma, primes[k]));
      scale.push_back(1u);
    }
    double log2M = 0;
    ZPoly all = crt_rows(ar, d_out, pitch, lucky, primes, cg + cu + cw, {cg, cg + cu + cw}, scale, device, &log2M, L);
    ZPoly G = slice(all, 0, cg), U = slice(all, cg, cg + cu), Wc = slice(all, cg + cu, cg + cu + cw);
    if (zdeg(G) != dmin) throw ApiError(CTG_INTERNAL, "gcd: degree mismatch after CRT");
    Big c;
    int s = 0;
    ZPoly g = zprimitive_positive(G, &c, &s);
    // e = gamma / (s c) must be an integer; then g U = e A and g W = e B modulo M.
    Big e;
    try {
      e = big_divexact(gamma, c);
    } catch (const std::exception&) {
      throw ApiError(CTG_INTERNAL, "gcd: exactness certificate failed (content)");
    }
    const double lg1 = zlog2_l1(g);
    const bool ok = lg1 + zlog2_l1(U) + 1 < log2M - 1 && lg1 + zlog2_l1(Wc) + 1 < log2M - 1 &&
                    big_log2(e) + zlog2_linf(A) + 1 < log2M - 1 && big_log2(e) + zlog2_linf(B) + 1 < log2M - 1;
    if (!ok) throw ApiError(CTG_INTERNAL, "gcd: exactness certificate failed (norm bound)");
    return g;
  }
  throw ApiError(CTG_INTERNAL, "gcd: could not find enough lucky primes");
}


// ---------------------------------------------------------------------------
// gcd_bivariate (elim.cpp:178-202) for coprime primitive parts.
// ---------------------------------------------------------------------------
using YPoly = std::vector<ZPoly>;  // y-degree -> coefficient in Z[x] (trimmed), bipoly.hpp y_coeffs

YPoly parse_bipoly_y(const ctg_bipoly* f) {
  YPoly out;
  if (!f || f->n_terms == 0) return out;
  if (f->n_terms < 0 || !f->dx || !f->dy || !f->sign || !f->limb_off || (!f->limbs && f->limb_off[f->n_terms] > 0))
    throw ApiError(CTG_INVALID, "bipoly: null pointer or negative term count");
  for (int i = 0; i < f->n_terms; ++i) {
    const int dx = f->dx[i], dy = f->dy[i];
    if (dx < 0 || dy < 0) throw ApiError(CTG_INVALID, "bipoly: negative exponent");
    const uint32_t b = f->limb_off[i], e = f->limb_off[i + 1];
    if (e < b) throw ApiError(CTG_INVALID, "bipoly: limb_off not monotone");
    const int sg = f->sign[i];
    if (sg < -1 || sg > 1) throw ApiError(CTG_INVALID, "bipoly: sign must be -1, 0 or +1");
    if (static_cast<int>(out.size()) <= dy) out.resize(dy + 1);
    if (static_cast<int>(out[dy].size()) <= dx) out[dy].resize(dx + 1);
    sbig_add_inplace(out[dy][dx], sg, f->limbs + b, static_cast<int>(e - b));
  }
  for (auto& c : out)
    while (!c.empty() && c.back().sign == 0) c.pop_back();
  while (!out.empty() && out.back().empty()) out.pop_back();
  return out;
}

// curvetop::gcd_univariate semantics (elim.cpp:80-93) on the GPU path.
ZPoly gcd_uni(const ZPoly& a, const ZPoly& b, int dev, cudaStream_t st, Launches& L) {
  if (a.empty() && b.empty()) throw ApiError(CTG_PRECONDITION, "gcd_univariate: both inputs zero");
  if (a.empty() || b.empty()) return zprimitive_positive(a.empty() ? b : a);
  ZPoly A = zprimitive_positive(a), B = zprimitive_positive(b);
  if (zdeg(A) == 0 || zdeg(B) == 0) return ZPoly{SBig{1, Big{1u}}};
  return gcd_modular(A, B, dev, st, L);
}

bool zis_one(const ZPoly& g) { return g.size() == 1 && g[0].sign == 1 && big_is_one(g[0].mag); }

// content_y (bipoly.cpp:192-201): gcd chain over the nonzero y-coefficients (stopping at 1),
// returned with positive leading coefficient and its full integer content.
ZPoly content_y(const YPoly& f, int dev, cudaStream_t st, Launches& L) {
  ZPoly g;
  for (const auto& fi : f) {
    if (fi.empty()) continue;
    g = g.empty() ? fi : gcd_uni(g, fi, dev, st, L);
    if (zis_one(g)) break;
  }
  if (!g.empty() && g.back().sign < 0)
    for (auto& c : g) c.sign = -c.sign;
  return g;
}

// deg_y gcd(f/cf, g/cg) == 0, certified by one (p, a) image of degree 0 whose formal leading
// y-coefficient survives: the image of the primitive gcd H then has degree deg_y H.
bool primitive_parts_coprime(const YPoly& f, const YPoly& g, int dev, cudaStream_t st, Launches& L) {
  const int nf = static_cast<int>(f.size()) - 1, ng = static_cast<int>(g.size()) - 1;
  ZPoly slots;
  std::vector<int32_t> dir;
  std::vector<int32_t> off, len;
  for (const YPoly* h : {&f, &g}) {
    std::vector<int32_t> o, l;
    for (const auto& row : *h) {
      o.push_back(static_cast<int32_t>(slots.size()));
      l.push_back(static_cast<int32_t>(row.size()));
      slots.insert(slots.end(), row.begin(), row.end());
    }
    dir.insert(dir.end(), o.begin(), o.end());
    dir.insert(dir.end(), l.begin(), l.end());
  }
  if (slots.empty()) return false;
  DevArena ar(st);
  const std::vector<uint32_t> primes = select_uni_primes(4 * 30.0);
  auto T = get_tables(dev, 1, primes);
  uint32_t* tab = reduce_poly(ar, slots, *T, L);
  int32_t* d_dir = ar.alloc<int32_t>(dir.size());
  CTG_CUDA_CHECK(cudaMemcpyAsync(d_dir, dir.data(), 4 * dir.size(), cudaMemcpyHostToDevice, ar.st));
  constexpr int kPoints = 8;
  const int units = T->P * kPoints;
  int32_t* d_deg = ar.alloc<int32_t>(units);
  const size_t gb = uni_gbuf_bytes(bigcd_probe_smem(nf, ng), static_cast<size_t>(units));
  uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
  L.n += launched(launch_bigcd_probe(tab, static_cast<int>(slots.size()), d_dir, nf, ng, T->d_pc, T->P, kPoints, d_deg, gbuf,
                            ar.st));
  CTG_CUDA_CHECK(cudaGetLastError());
  std::vector<int32_t> deg(units);
  CTG_CUDA_CHECK(cudaMemcpyAsync(deg.data(), d_deg, 4 * units, cudaMemcpyDeviceToHost, ar.st));
  CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
  for (int d : deg)
    if (d == 0) return true;
  return false;
}

// ---- small signed Z[x] helpers for the Brown gcd's normalisation (degrees ~ tens) ----
SBig sb_mul(const SBig& a, const SBig& b) {
  if (a.sign == 0 || b.sign == 0) return SBig{};
  return SBig{a.sign * b.sign, big_mul(a.mag, b.mag)};
}

ZPoly zmul(const ZPoly& a, const ZPoly& b) {
  if (a.empty() || b.empty()) return ZPoly{};
  ZPoly r(a.size() + b.size() - 1);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) {
      const SBig t = sb_mul(a[i], b[j]);
      if (t.sign) sbig_add_inplace(r[i + j], t.sign, t.mag.data(), static_cast<int>(t.mag.size()));
    }
  while (!r.empty() && r.back().sign == 0) r.pop_back();
  return r;
}

// a / c in Z[x] for an exact divisor c (throws CTG_INTERNAL otherwise).
ZPoly zdivexact(ZPoly a, const ZPoly& c) {
  const int dc = zdeg(c);
  if (dc < 0) throw ApiError(CTG_INTERNAL, "zdivexact: zero divisor");
  if (zdeg(a) < dc) {
    if (!a.empty()) throw ApiError(CTG_INTERNAL, "zdivexact: inexact division");
    return a;
  }
  ZPoly q(a.size() - dc);
  for (int t = zdeg(a) - dc; t >= 0; --t) {
    SBig& top = a[t + dc];
    if (top.sign == 0) continue;
    SBig qt{top.sign * c[dc].sign, big_divexact(top.mag, c[dc].mag)};
    for (int i = 0; i <= dc; ++i) {
      const SBig m = sb_mul(qt, c[i]);
      if (m.sign) sbig_add_inplace(a[t + i], -m.sign, m.mag.data(), static_cast<int>(m.mag.size()));
    }
    q[t] = std::move(qt);
  }
  for (const auto& r : a)
    if (r.sign != 0) throw ApiError(CTG_INTERNAL, "zdivexact: inexact division");
  while (!q.empty() && q.back().sign == 0) q.pop_back();
  return q;
}

double ylog2_l1(const YPoly& f) {
  std::vector<double> v;
  for (const auto& r : f)
    for (const auto& c : r)
      if (c.sign) v.push_back(big_log2(c.mag));
  return log2_sum_upper(v);
}
double ylog2_linf(const YPoly& f) {
  double m = -INFINITY;
  for (const auto& r : f) m = std::max(m, zlog2_linf(r));
  return m;
}
int ydeg_x(const YPoly& f) {
  int d = -1;
  for (const auto& r : f) d = std::max(d, zdeg(r));
  return d;
}

uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Brown's modular gcd of f, g in Z[x][y] (replaces the PRS of
// elim.cpp:184-190 when the primitive parts share a factor).  Returns H = pp_{Z[x]} gcd(f, g)
// with lc_x(lc_y H) > 0.
//   gamma = gcd_{Z[x]}(lc_y f, lc_y g) (GPU univariate gcd times the integer gcd of contents)
//   is a multiple of lc_y gcd(f, g); for every prime p and point a with gamma(a) != 0 the GPU
//   computes h = gamma(a) * monic gcd(f(a, y), g(a, y)) and the cofactors u = f(a, y) / g,
//   w = g(a, y) / g (k_bigcd_images); primes whose N points all reach the minimal degree are
//   interpolated in x (k_newton_interp) and CRT'd (K5) to Ht, U, W in Z[x][y].
//   Certificate: deg_x Ht <= bH, deg_x U <= deg_x f, deg_x W <= deg_x g with N > bH + max
//   makes Ht U = gamma f and Ht W = gamma g hold mod every CRT prime as polynomials, and the
//   norm bounds ||Ht||_1 ||U||_1 < M/2, ||gamma||_1 ||f||_inf < M/2 (same for g) make them exact
//   over Z; then pp(Ht) divides f and g and has y-degree = the minimal modular degree >=
//   deg_y gcd(f, g), so it IS the primitive gcd (up to sign).
YPoly bigcd_modular(const YPoly& f, const YPoly& g, int dev, cudaStream_t st, Launches& L) {
  const int nf = static_cast<int>(f.size()) - 1, ng = static_cast<int>(g.size()) - 1;
  const ZPoly& lf = f.back();
  const ZPoly& lg = g.back();
  // gamma = gcd(cont lf, cont lg) * gcd_uni(lf, lg)
  ZPoly gamma = gcd_uni(lf, lg, dev, st, L);
  {
    const Big ci = big_gcd(zcontent(lf), zcontent(lg));
    for (auto& c : gamma) c.mag = big_mul(c.mag, ci);
  }
  const int dxf = ydeg_x(f), dxg = ydeg_x(g), dgam = zdeg(gamma);
  const int bH = dgam + std::min(dxf, dxg);
  const int N = bH + std::max(dxf, dxg) + 1;
  // slot table: rows of f, rows of g, gamma
  ZPoly slots;
  std::vector<int32_t> dir;
  for (const YPoly* h : {&f, &g}) {
    std::vector<int32_t> o, l;
    for (const auto& row : *h) {
      o.push_back(static_cast<int32_t>(slots.size()));
      l.push_back(static_cast<int32_t>(row.size()));
      slots.insert(slots.end(), row.begin(), row.end());
    }
    dir.insert(dir.end(), o.begin(), o.end());
    dir.insert(dir.end(), l.begin(), l.end());
  }
  const int gam_off = static_cast<int>(slots.size()), gam_len = static_cast<int>(gamma.size());
  slots.insert(slots.end(), gamma.begin(), gamma.end());
  const double lgam = zlog2_l1(gamma);
  const double need = 2 * lgam + ylog2_l1(f) + ylog2_l1(g) + (dxf + nf + dxg + ng) + 2 + 40;
  double extra = 62;
  for (int attempt = 0; attempt < 4; ++attempt, extra *= 4) {
    DevArena ar(st);
    const std::vector<uint32_t> primes = select_uni_primes(need + extra);
    const int nk = static_cast<int>(primes.size());
    auto T = get_tables(dev, 1, primes);
    uint32_t* tab = reduce_poly(ar, slots, *T, L);
    std::vector<uint32_t> offs(nk);
    for (int k = 0; k < nk; ++k)
      offs[k] = 1u + static_cast<uint32_t>(mix64((static_cast<uint64_t>(primes[k]) << 8) ^ attempt) %
                                            (primes[k] - static_cast<uint32_t>(N) - 2u));
    int32_t* d_dir = ar.alloc<int32_t>(dir.size());
    uint32_t* d_offs = ar.alloc<uint32_t>(nk);
    CTG_CUDA_CHECK(cudaMemcpyAsync(d_dir, dir.data(), 4 * dir.size(), cudaMemcpyHostToDevice, ar.st));
    CTG_CUDA_CHECK(cudaMemcpyAsync(d_offs, offs.data(), 4 * nk, cudaMemcpyHostToDevice, ar.st));
    const int pitch = nf + ng + 3;
    int32_t* d_deg = ar.alloc<int32_t>(static_cast<size_t>(nk) * N);
    uint32_t* d_img = ar.alloc<uint32_t>(static_cast<size_t>(nk) * N * pitch);
    const size_t gbi = uni_gbuf_bytes(modgcd_smem(nf, ng), static_cast<size_t>(nk) * N);
    uint32_t* gbuf = gbi ? ar.alloc<uint32_t>(gbi / 4) : nullptr;
    L.n += launched(launch_bigcd_images(tab, static_cast<int>(slots.size()), d_dir, nf, ng, gam_off, gam_len, T->d_pc, d_offs,
                               nk, N, d_deg, d_img, pitch, gbuf, ar.st));
    CTG_CUDA_CHECK(cudaGetLastError());
    std::vector<int32_t> deg(static_cast<size_t>(nk) * N);
    CTG_CUDA_CHECK(cudaMemcpyAsync(deg.data(), d_deg, 4 * deg.size(), cudaMemcpyDeviceToHost, ar.st));
    CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
    stats_tls().d2h_bytes += static_cast<int64_t>(4 * deg.size());
    int dmin = INT32_MAX;
    for (int d : deg)
      if (d >= 0) dmin = std::min(dmin, d);
    if (dmin == INT32_MAX) continue;
    if (dmin == 0) return YPoly{ZPoly{SBig{1, Big{1u}}}};
    std::vector<int> lucky;
    double bits = 0;
    for (int k = 0; k < nk; ++k) {
      bool ok = true;
      for (int j = 0; j < N && ok; ++j) ok = deg[static_cast<size_t>(k) * N + j] == dmin;
      if (ok) {
        lucky.push_back(k);
        bits += std::log2(static_cast<double>(primes[k]));
      }
    }
    if (bits < need) continue;
    const int cols = nf + ng - dmin + 3;
    int32_t* d_idx = ar.alloc<int32_t>(lucky.size());
    CTG_CUDA_CHECK(cudaMemcpyAsync(d_idx, lucky.data(), 4 * lucky.size(), cudaMemcpyHostToDevice, ar.st));
    uint32_t* d_coef = ar.alloc<uint32_t>(static_cast<size_t>(nk) * N * cols);
    // Newton beyond the shared-memory budget: global slices for up to ~256 MB of CTAs at a time
    const size_t per_row = newton_smem(N) * ((cols + kNewtonColsPerCta - 1) / kNewtonColsPerCta);
    const int nrows_l = static_cast<int>(lucky.size());
    const int grows = uni_gbuf_bytes(newton_smem(N), 1)
                          ? std::max(1, std::min(nrows_l, static_cast<int>((size_t{256} << 20) / per_row)))
                          : 0;
    uint32_t* gnew = grows ? ar.alloc<uint32_t>(per_row * grows / 4) : nullptr;
    L.n += launched(launch_newton_interp(d_img, pitch, d_idx, nrows_l, T->d_pc, d_offs, N, cols, d_coef, gnew, grows, ar.st));
    CTG_CUDA_CHECK(cudaGetLastError());
    double log2M = 0;
    const int total = N * cols;
    ZPoly all = crt_rows(ar, d_coef, total, lucky, primes, total, {total}, std::vector<uint32_t>(lucky.size(), 1u), dev,
                         &log2M, L);
    // unpack: column c = y-row of Ht (c <= dmin), U, W; coefficient t = x-degree
    auto unpack = [&](int c0, int rows, int bound, YPoly* out) {
      out->assign(rows, ZPoly{});
      for (int r = 0; r < rows; ++r) {
        ZPoly& z = (*out)[r];
        z.resize(N);
        for (int t = 0; t < N; ++t) z[t] = std::move(all[static_cast<size_t>(t) * cols + c0 + r]);
        while (!z.empty() && z.back().sign == 0) z.pop_back();
        if (zdeg(z) > bound) return false;
      }
      while (!out->empty() && out->back().empty()) out->pop_back();
      return true;
    };
    YPoly Ht, U, W;
    if (!unpack(0, dmin + 1, bH, &Ht) || !unpack(dmin + 1, nf - dmin + 1, dxf, &U) ||
        !unpack(nf + 2, ng - dmin + 1, dxg, &W))
      continue;  // an undetected unlucky prime: retry with a fresh prime set
    if (static_cast<int>(Ht.size()) != dmin + 1) throw ApiError(CTG_INTERNAL, "gcd_bivariate: degree mismatch after CRT");
    const double lH = ylog2_l1(Ht);
    const bool ok = lH + ylog2_l1(U) + 1 < log2M - 1 && lH + ylog2_l1(W) + 1 < log2M - 1 &&
                    lgam + ylog2_linf(f) + 1 < log2M - 1 && lgam + ylog2_linf(g) + 1 < log2M - 1;
    if (!ok) continue;  // bound too small for these coefficients: more primes
    // H = pp_{Z[x]}(Ht): integer content, then the primitive gcd of the rows (GPU chain)
    Big ci;
    for (const auto& r : Ht)
      if (!r.empty()) {
        const Big c = zcontent(r);
        ci = ci.empty() ? c : big_gcd(ci, c);
      }
    ZPoly cx;
    for (const auto& r : Ht) {
      if (r.empty()) continue;
      cx = cx.empty() ? zprimitive_positive(r) : gcd_uni(cx, r, dev, st, L);
      if (zdeg(cx) == 0) break;
    }
    YPoly H(Ht.size());
    const bool unit_ci = big_is_one(ci);
    for (size_t r = 0; r < Ht.size(); ++r) {
      ZPoly row = Ht[r];
      if (!unit_ci)
        for (auto& c : row)
          if (c.sign) c.mag = big_divexact(c.mag, ci);
      H[r] = zdeg(cx) > 0 ? zdivexact(std::move(row), cx) : std::move(row);
    }
    if (H.back().back().sign < 0)
      for (auto& r : H)
        for (auto& c : r) c.sign = -c.sign;
    return H;
  }
  throw ApiError(CTG_INTERNAL, "gcd_bivariate: could not certify the modular gcd");
}

void fill_bipoly_x(const ZPoly& c, ctg_bipoly_buf* out) {
  std::vector<int> idx;
  size_t total = 0;
  for (size_t i = 0; i < c.size(); ++i)
    if (c[i].sign != 0) {
      idx.push_back(static_cast<int>(i));
      total += c[i].mag.size();
    }
  const size_t n = idx.size();
  const size_t bytes = 8 * n + 4 * (n + 1) + 4 * total + n + 16;
  auto* base = static_cast<uint8_t*>(std::malloc(bytes));
  if (!base) throw std::bad_alloc();
  out->n_terms = static_cast<int32_t>(n);
  out->dx = reinterpret_cast<int32_t*>(base);
  out->dy = out->dx + n;
  out->limb_off = reinterpret_cast<uint32_t*>(out->dy + n);
  out->limbs = out->limb_off + n + 1;
  out->sign = reinterpret_cast<int8_t*>(out->limbs + total);
  uint32_t pos = 0;
  for (size_t t = 0; t < n; ++t) {
    const SBig& v = c[idx[t]];
    out->dx[t] = idx[t];
    out->dy[t] = 0;
    out->sign[t] = static_cast<int8_t>(v.sign);
    out->limb_off[t] = pos;
    std::memcpy(out->limbs + pos, v.mag.data(), 4 * v.mag.size());
    pos += static_cast<uint32_t>(v.mag.size());
  }
  out->limb_off[n] = pos;
}

// Copy of a parsed operand, terms sorted by (dx, dy) (the reference returns it as is).
void fill_bipoly(const YPoly& f, ctg_bipoly_buf* out) {
  struct T {
    int dx, dy;
    const SBig* c;
  };
  std::vector<T> terms;
  size_t total = 0;
  for (size_t y = 0; y < f.size(); ++y)
    for (size_t x = 0; x < f[y].size(); ++x)
      if (f[y][x].sign != 0) {
        terms.push_back({static_cast<int>(x), static_cast<int>(y), &f[y][x]});
        total += f[y][x].mag.size();
      }
  std::sort(terms.begin(), terms.end(), [](const T& a, const T& b) { return a.dx != b.dx ? a.dx < b.dx : a.dy < b.dy; });
  const size_t n = terms.size();
  auto* base = static_cast<uint8_t*>(std::malloc(8 * n + 4 * (n + 1) + 4 * total + n + 16));
  if (!base) throw std::bad_alloc();
  out->n_terms = static_cast<int32_t>(n);
  out->dx = reinterpret_cast<int32_t*>(base);
  out->dy = out->dx + n;
  out->limb_off = reinterpret_cast<uint32_t*>(out->dy + n);
  out->limbs = out->limb_off + n + 1;
  out->sign = reinterpret_cast<int8_t*>(out->limbs + total);
  uint32_t pos = 0;
  for (size_t t = 0; t < n; ++t) {
    out->dx[t] = terms[t].dx;
    out->dy[t] = terms[t].dy;
    out->sign[t] = static_cast<int8_t>(terms[t].c->sign);
    out->limb_off[t] = pos;
    std::memcpy(out->limbs + pos, terms[t].c->mag.data(), 4 * terms[t].c->mag.size());
    pos += static_cast<uint32_t>(terms[t].c->mag.size());
  }
  out->limb_off[n] = pos;
}

// A ZPoly straight into a library buffer (one pass, no per-coefficient staging vectors).
void fill_upoly_z(const ZPoly& p, ctg_upoly_buf* out) {
  size_t n = p.size();
  while (n > 0 && p[n - 1].sign == 0) --n;
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) total += p[i].mag.size();
  upoly_alloc(out, n, total);
  uint32_t off = 0;
  for (size_t i = 0; i < n; ++i) {
    out->sign[i] = static_cast<int8_t>(p[i].sign);
    out->limb_off[i] = off;
    if (!p[i].mag.empty()) std::memcpy(out->limbs + off, p[i].mag.data(), 4 * p[i].mag.size());
    off += static_cast<uint32_t>(p[i].mag.size());
  }
  out->limb_off[n] = off;
}

// A primitive polynomial given as slots, divided by sgn(lc), into a library buffer.
void fill_upoly_slots(const std::vector<Slot>& p, int lcsign, ctg_upoly_buf* out) {
  const size_t n = p.size();
  size_t total = 0;
  for (const Slot& c : p) total += static_cast<size_t>(c.n);
  upoly_alloc(out, n, total);
  uint32_t off = 0;
  for (size_t i = 0; i < n; ++i) {
    out->sign[i] = static_cast<int8_t>(p[i].sign * lcsign);
    out->limb_off[i] = off;
    if (p[i].n) std::memcpy(out->limbs + off, p[i].mag, 4 * static_cast<size_t>(p[i].n));
    off += static_cast<uint32_t>(p[i].n);
  }
  out->limb_off[n] = off;
}

// pp(R) straight from the caller's limbs: R / content / sgn(lc R) (content != 1 divides every
// coefficient).  Quotients go to a scratch region at upper-bound offsets (parallel, GMP exact
// division on thread-local scratch: no allocation per coefficient), then packed into out.
// CurveContext at d30 (R of degree 870, 7,800-bit coefficients, 123-bit content): replaces a
// parse of R into per-coefficient vectors, a checked division and a second copy (~0.27 ms).
void fill_upoly_slots_divided(const std::vector<Slot>& p, const Big& content, int lcsign, ctg_upoly_buf* out) {
  const size_t n = p.size();
  const int nc = static_cast<int>(content.size());
  std::vector<size_t> cap_off(n + 1, 0);
  for (size_t i = 0; i < n; ++i)
    cap_off[i + 1] = cap_off[i] + (p[i].n ? static_cast<size_t>(std::max(2, p[i].n - nc + 4)) : 0);  // GMP writes whole 64-bit limbs
  thread_local std::vector<uint32_t> scratch;  // the caller's thread (workers get the pointer)
  if (scratch.size() < cap_off[n]) scratch.resize(cap_off[n]);
  uint32_t* const sp = scratch.data();
  std::vector<uint32_t> len(n, 0);
  const int blk = 16;
  parallel_for(static_cast<int>((n + blk - 1) / blk), [&](int b) {
    for (size_t i = static_cast<size_t>(b) * blk; i < std::min(n, static_cast<size_t>(b + 1) * blk); ++i)
      if (p[i].n) len[i] = static_cast<uint32_t>(big_divexact_to(p[i].mag, p[i].n, content, sp + cap_off[i]));
  });
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) total += len[i];
  upoly_alloc(out, n, total);
  uint32_t off = 0;
  for (size_t i = 0; i < n; ++i) {
    out->sign[i] = static_cast<int8_t>(len[i] ? p[i].sign * lcsign : 0);
    out->limb_off[i] = off;
    off += len[i];
  }
  out->limb_off[n] = off;
  parallel_for(static_cast<int>((n + blk - 1) / blk), [&](int b) {
    for (size_t i = static_cast<size_t>(b) * blk; i < std::min(n, static_cast<size_t>(b + 1) * blk); ++i)
      if (len[i]) std::memcpy(out->limbs + out->limb_off[i], sp + cap_off[i], 4 * static_cast<size_t>(len[i]));
  });
}

void fill_sqf(const Big& unit, int unit_sign, const std::vector<std::pair<ZPoly, int>>& factors, ctg_sqf_buf* out,
              const ZPoly* single = nullptr, const std::vector<Slot>* single_slots = nullptr,
              const Big* single_divisor = nullptr) {
  std::memset(out, 0, sizeof(*out));
  out->unit_sign = static_cast<int8_t>(unit.empty() ? 0 : unit_sign);
  out->unit_nlimbs = static_cast<int32_t>(unit.size());
  out->unit_limbs = static_cast<uint32_t*>(std::malloc(4 * std::max<size_t>(1, unit.size())));
  std::memcpy(out->unit_limbs, unit.data(), 4 * unit.size());
  const size_t nf = (single || single_slots) ? 1 : factors.size();
  out->n_factors = static_cast<int32_t>(nf);
  out->mult = static_cast<int32_t*>(std::malloc(4 * std::max<size_t>(1, nf)));
  out->factors = static_cast<ctg_upoly_buf*>(std::calloc(std::max<size_t>(1, nf), sizeof(ctg_upoly_buf)));
  if (!out->unit_limbs || !out->mult || !out->factors) throw std::bad_alloc();
  if (single) {  // square-free input: the one factor (multiplicity 1) is the primitive input itself
    out->mult[0] = 1;
    fill_upoly_z(*single, &out->factors[0]);
    return;
  }
  if (single_slots) {  // the same from the caller's limbs: R / content / sgn(lc R)
    out->mult[0] = 1;
    if (single_divisor)
      fill_upoly_slots_divided(*single_slots, *single_divisor, unit_sign, &out->factors[0]);
    else
      fill_upoly_slots(*single_slots, unit_sign, &out->factors[0]);
    return;
  }
  for (size_t i = 0; i < factors.size(); ++i) {
    out->mult[i] = factors[i].second;
    fill_upoly_z(factors[i].first, &out->factors[i]);
  }
}

}  // namespace
}  // namespace ctg

using namespace ctg;

extern "C" {

ctg_status ctg_yun_squarefree(const ctg_upoly* p, ctg_sqf_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out) throw ApiError(CTG_INVALID, "yun_squarefree: null output");
    CallTimer timer;
    // The input as slots over the caller's CSR (no copies): the common case -- a primitive,
    // square-free R (every dense config) -- is answered from them directly.
    std::vector<Slot> slots = view_upoly(p);
    if (slots.empty()) throw ApiError(CTG_PRECONDITION, "yun_squarefree: zero polynomial");  // elim.cpp:139
    const int n = static_cast<int>(slots.size()) - 1;
    Launches L;
    std::unique_ptr<DeviceGuard> g;
    std::unique_lock<std::mutex> lock;
    int dev = -1;
    Ctx* ctx = nullptr;
    auto device = [&] {
      if (ctx) return;
      g = std::make_unique<DeviceGuard>(opts);
      dev = select_device(opts);
      ctx = &context(dev);
      lock = std::unique_lock<std::mutex>(ctx->mu);
    };
    YunProbe probe;
    // R straight from a single-curve ctg_resultant (CurveContext, lift.cpp:64-67): its probe ran
    // on the GPU behind the resultant -- use it when the input is exactly that R
    int cached = -1;  // -1 no, 0 probed and not certified, 1 certified square-free
    bool candidate = false;  // the latest resultant's R has this degree: compare after the content
    if (n >= kProbeMinDeg) {
      device();
      const SqfProbeCache& pc = ctx->sqf;
      candidate = pc.valid && pc.n == n;
    }
    // square-freeness probe on the GPU while the host takes the content -- only where
    // yun_modular would probe too (its full prime set exceeds one wave of CTAs), so a
    // non-square-free input never pays for it twice
    bool probe_first = false;
    if (n >= kProbeMinDeg) {
      std::vector<double> sq;
      for (const Slot& c : slots)
        if (c.n) sq.push_back(2 * log2_upper(c.mag, c.n));
      const double need = log2_upper(slots.back().mag, slots.back().n) + n + 0.5 * log2_sum_upper(sq) + 2 + 40;
      probe_first = select_uni_primes(need + 62).size() > 148;
    }
    if (probe_first && !candidate) {
      device();
      probe_start(probe, slots, n, dev, ctx->stream, L);
    }
    const int s = slots.back().sign;
    Big content = slots_content(slots);  // elim.cpp:141-144: unit = sign(lc) * content
    timer.mark_setup();
    if (n == 0) {  // elim.cpp:145
      fill_sqf(content, s, {}, out);
      timer.finish();
      return;
    }
    if (candidate) {  // the resultant's probe has had the content computation to finish
      const SqfProbeCache& pc = ctx->sqf;
      const SqfProbeCache::Slot& sl = pc.slot[pc.cur];
      CTG_CUDA_CHECK(cudaEventSynchronize(sl.done));
      if (probe_matches(pc, slots)) {
        cached = 0;
        for (int k = 0; k < 3; ++k)
          if (sl.h_out[2 * k] == 0 && sl.h_out[2 * k + 1] == 0) cached = 1;
      }
    }
    const bool certified = cached >= 0 ? cached == 1 : (probe.done && probe_finish(probe));
    if (certified) {  // (R / (sgn(lc) content), 1): straight from the caller's limbs
      timer.mark_device();
      stats_tls().kernel_launches = L.n;
      fill_sqf(content, s, {}, out, nullptr, &slots, big_is_one(content) ? nullptr : &content);
      timer.finish();
      return;
    }
    ZPoly P = divide_content(parse_upoly(p), content, nullptr, nullptr);
    device();
    YunResult r = yun_modular(P, false, dev, ctx->stream, L, (probe_first && !candidate) || cached >= 0);
    timer.mark_device();
    stats_tls().kernel_launches = L.n;
    fill_sqf(content, s, r.factors, out, r.squarefree ? &P : nullptr);
    timer.finish();
  });
}

// Throughput form of yun_squarefree (CurveContext over many curves): ONE K1 launch reduces every
// input modulo the 3 probe primes, ONE k_sqf_probe launch runs gcd(P, P') mod p for every
// (input, prime) pair in parallel, and the host takes the contents meanwhile (parallel_for).
// Inputs certified square-free return (sgn * content, [(pp, 1)]); the rest go through the
// single-input path.  Results are identical to calling ctg_yun_squarefree on each input.
ctg_status ctg_yun_squarefree_batch(int32_t batch, const ctg_upoly* p, ctg_sqf_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out || !p || batch < 0) throw ApiError(CTG_INVALID, "yun_squarefree_batch: bad arguments");
    CallTimer timer;
    for (int b = 0; b < batch; ++b) std::memset(&out[b], 0, sizeof(out[b]));
    // every input as slots over the caller's CSR (no copies, as ctg_yun_squarefree)
    std::vector<std::vector<Slot>> sl(batch);
    for (int b = 0; b < batch; ++b) {
      sl[b] = view_upoly(&p[b]);
      if (sl[b].empty())
        throw ApiError(CTG_PRECONDITION, "yun_squarefree: zero polynomial (batch entry " + std::to_string(b) + ")");
    }
    DeviceGuard g(opts);
    const int dev = select_device(opts);
    Ctx& ctx = context(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    Launches L;
    // probe every input of degree >= 2 (one K1 over all their slots, one launch)
    std::vector<int> idx;
    std::vector<int32_t> off, degs;
    std::vector<Slot> all;
    int maxd = 0;
    for (int b = 0; b < batch; ++b) {
      const int d = static_cast<int>(sl[b].size()) - 1;
      if (d >= 2) {
        idx.push_back(b);
        off.push_back(static_cast<int32_t>(all.size()));
        degs.push_back(d);
        all.insert(all.end(), sl[b].begin(), sl[b].end());
        maxd = std::max(maxd, d);
      }
    }
    const int np = static_cast<int>(idx.size());
    const int S = static_cast<int>(all.size());
    static const bool trace = std::getenv("CTG_TRACE_HOST") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto tms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t_a = tnow();
    std::vector<uint32_t> primes = select_probe_primes(maxd);
    const bool small = !primes.empty();
    if (!small) primes = select_uni_primes(3 * 30.0);
    const int nk = static_cast<int>(primes.size());
    DevArena ar(ctx.stream);
    thread_local int32_t* h_out = nullptr;
    thread_local size_t h_cap = 0;
    cudaEvent_t done = nullptr;
    if (np) {
      auto T = get_tables(dev, 1, primes);
      uint32_t* d_tab = reduce_slots(ar, all, *T, L);
      int32_t* d_meta = ar.alloc<int32_t>(2 * static_cast<size_t>(np));
      int32_t* d_out = ar.alloc<int32_t>(2 * static_cast<size_t>(np) * nk);
      std::vector<int32_t> meta(off);
      meta.insert(meta.end(), degs.begin(), degs.end());
      CTG_CUDA_CHECK(cudaMemcpyAsync(d_meta, meta.data(), 4 * meta.size(), cudaMemcpyHostToDevice, ar.st));
      const size_t gb = uni_gbuf_bytes(sqf_probe_smem(maxd), static_cast<size_t>(np) * nk);
      uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
      L.n += launched(launch_sqf_probe(d_tab, S, d_meta, d_meta + np, np, nk, T->d_pc, maxd, d_out, gbuf, ar.st, 0,
                                       small));
      CTG_CUDA_CHECK(cudaGetLastError());
      const size_t need = 2 * static_cast<size_t>(np) * nk;
      if (h_cap < need) {
        if (h_out) cudaFreeHost(h_out);
        h_out = nullptr;
        CTG_CUDA_CHECK(cudaMallocHost(&h_out, 4 * need));
        h_cap = need;
      }
      CTG_CUDA_CHECK(cudaMemcpyAsync(h_out, d_out, 4 * need, cudaMemcpyDeviceToHost, ar.st));
      CTG_CUDA_CHECK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
      CTG_CUDA_CHECK(cudaEventRecord(done, ar.st));
      stats_tls().d2h_bytes += static_cast<int64_t>(4 * need);
    }
    // contents on the host while the GPU probes (elim.cpp:141-144)
    const auto t_b = tnow();
    std::vector<Big> content(batch);
    std::vector<int> sgn(batch, 0);
    parallel_for(batch, [&](int b) {
      content[b] = slots_content(sl[b]);
      sgn[b] = sl[b].back().sign;
    });
    if (trace) std::fprintf(stderr, "[ctg] yun batch %d: probe enqueue (K1 staging) %.3f ms, contents %.3f ms\n", batch,
                            tms(t_a, t_b), tms(t_b, tnow()));
    timer.mark_setup();
    std::vector<char> sqfree(batch, 0);
    if (done) {
      CTG_CUDA_CHECK(cudaEventSynchronize(done));
      cudaEventDestroy(done);
      for (int q = 0; q < np; ++q)
        for (int k = 0; k < nk; ++k) {
          const int32_t* o = h_out + 2 * (static_cast<size_t>(q) * nk + k);
          if (o[0] == 0 && o[1] == 0) sqfree[idx[q]] = 1;
        }
    }
    timer.mark_device();
    try {
      // constants and certified square-free inputs: (R / (sgn content), 1) straight from the
      // caller's limbs, in parallel; the rest through the full modular Yun one by one
      parallel_for(batch, [&](int b) {
        if (sl[b].size() == 1)  // elim.cpp:145
          fill_sqf(content[b], sgn[b], {}, &out[b]);
        else if (sqfree[b])
          fill_sqf(content[b], sgn[b], {}, &out[b], nullptr, &sl[b], big_is_one(content[b]) ? nullptr : &content[b]);
      });
      for (int b = 0; b < batch; ++b) {
        if (sl[b].size() == 1 || sqfree[b]) continue;
        ZPoly Pb = divide_content(parse_upoly(&p[b]), content[b], nullptr, nullptr);
        YunResult r = yun_modular(Pb, false, dev, ctx.stream, L);
        fill_sqf(content[b], sgn[b], r.factors, &out[b], r.squarefree ? &Pb : nullptr);
      }
    } catch (...) {
      for (int b = 0; b < batch; ++b) ctg_sqf_free(&out[b]);
      throw;
    }
    stats_tls().kernel_launches = L.n;
    timer.finish();
  });
}

ctg_status ctg_square_free_part(const ctg_upoly* p, ctg_upoly_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out) throw ApiError(CTG_INVALID, "square_free_part: null output");
    CallTimer timer;
    ZPoly a = parse_upoly(p);
    if (a.empty()) throw ApiError(CTG_PRECONDITION, "square_free_part: zero polynomial");  // elim.cpp:205
    ZPoly P = zprimitive_positive(std::move(a));
    timer.mark_setup();
    if (zdeg(P) == 0) {  // elim.cpp:207
      fill_upoly_z(P, out);
      timer.finish();
      return;
    }
    DeviceGuard g(opts);
    const int dev = select_device(opts);
    Ctx& ctx = context(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    Launches L;
    YunResult r = yun_modular(P, true, dev, ctx.stream, L);
    timer.mark_device();
    stats_tls().kernel_launches = L.n;
    fill_upoly_z(r.squarefree ? P : r.sqfp, out);
    timer.finish();
  });
}

ctg_status ctg_gcd_univariate(const ctg_upoly* p, const ctg_upoly* q, ctg_upoly_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out) throw ApiError(CTG_INVALID, "gcd_univariate: null output");
    CallTimer timer;
    ZPoly a = parse_upoly(p), b = parse_upoly(q);
    // elim.cpp:81-85
    if (a.empty() && b.empty()) throw ApiError(CTG_PRECONDITION, "gcd_univariate: both inputs zero");
    if (a.empty() || b.empty()) {
      fill_upoly_z(zprimitive_positive(a.empty() ? b : a), out);
      timer.finish();
      return;
    }
    ZPoly A = zprimitive_positive(std::move(a)), B = zprimitive_positive(std::move(b));
    timer.mark_setup();
    if (zdeg(A) == 0 || zdeg(B) == 0) {
      fill_upoly_z(ZPoly{SBig{1, Big{1u}}}, out);
      timer.finish();
      return;
    }
    DeviceGuard g(opts);
    const int dev = select_device(opts);
    Ctx& ctx = context(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    Launches L;
    ZPoly r = gcd_modular(A, B, dev, ctx.stream, L);
    timer.mark_device();
    stats_tls().kernel_launches = L.n;
    fill_upoly_z(r, out);
    timer.finish();
  });
}

ctg_status ctg_gcd_bivariate(const ctg_bipoly* f, const ctg_bipoly* g, ctg_bipoly_buf* out, const ctg_opts* opts) {
  return guarded([&] {
    if (!out) throw ApiError(CTG_INVALID, "gcd_bivariate: null output");
    CallTimer timer;
    YPoly a = parse_bipoly_y(f), b = parse_bipoly_y(g);
    // elim.cpp:179-181
    if (a.empty() && b.empty()) throw ApiError(CTG_PRECONDITION, "gcd_bivariate: both inputs zero");
    if (a.empty() || b.empty()) {
      fill_bipoly(a.empty() ? b : a, out);
      timer.finish();
      return;
    }
    timer.mark_setup();
    DeviceGuard guard(opts);
    const int dev = select_device(opts);
    Ctx& ctx = context(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    Launches L;
    const ZPoly cf = content_y(a, dev, ctx.stream, L), cg = content_y(b, dev, ctx.stream, L);
    // elim.cpp:193-201: result = pp(gcd) * gcd_univariate(cf, cg), leading (y, then x)
    // coefficient positive (gcd_univariate's leading coefficient is positive).
    const ZPoly c = gcd_uni(cf, cg, dev, ctx.stream, L);
    if (primitive_parts_coprime(a, b, dev, ctx.stream, L)) {  // pp = +-1
      timer.mark_device();
      stats_tls().kernel_launches = L.n;
      fill_bipoly_x(c, out);
      timer.finish();
      return;
    }
    YPoly H = bigcd_modular(a, b, dev, ctx.stream, L);
    timer.mark_device();
    stats_tls().kernel_launches = L.n;
    if (!(c.size() == 1 && big_is_one(c[0].mag)))
      for (auto& r : H) r = zmul(r, c);
    fill_bipoly(H, out);
    timer.finish();
  });
}

void ctg_bipoly_free(ctg_bipoly_buf* buf) {
  if (!buf) return;
  std::free(buf->dx);
  std::memset(buf, 0, sizeof(*buf));
}

}  // extern "C"

ctg_status ctg_modp_gcd_degree(const uint32_t* a, int32_t na, const uint32_t* b, int32_t nb, int32_t prime_index,
                               int32_t method, int32_t* deg, uint32_t* prime, float* ms, const ctg_opts* opts) {
  using namespace ctg;
  return guarded([&] {
    if (!a || !b || !deg || na < 0 || nb < 0 || prime_index < 0 || prime_index > 15 || method < 0 || method > 2 ||
        (method == 2 && prime_index > 2))
      throw ApiError(CTG_INVALID, "modp_gcd_degree: bad arguments");
    DeviceGuard g(opts);
    const int dev = select_device(opts);
    Ctx& ctx = context(dev);
    std::lock_guard<std::mutex> lock(ctx.mu);
    const std::vector<uint32_t> all = method == 2 ? select_probe_primes(0) : select_uni_primes(30.0 * (prime_index + 1));
    if (static_cast<int>(all.size()) <= prime_index) throw ApiError(CTG_INTERNAL, "modp_gcd_degree: prime table");
    const std::vector<uint32_t> one{all[prime_index]};
    for (int32_t i = 0; i <= na; ++i)
      if (a[i] >= one[0]) throw ApiError(CTG_INVALID, "modp_gcd_degree: residue >= p");
    for (int32_t i = 0; i <= nb; ++i)
      if (b[i] >= one[0]) throw ApiError(CTG_INVALID, "modp_gcd_degree: residue >= p");
    auto T = get_tables(dev, 1, one);
    DevArena ar(ctx.stream);
    uint32_t* d_a = ar.alloc<uint32_t>(na + 1);
    uint32_t* d_b = ar.alloc<uint32_t>(nb + 1);
    int32_t* d_out = ar.alloc<int32_t>(1);
    CTG_CUDA_CHECK(cudaMemcpyAsync(d_a, a, 4 * static_cast<size_t>(na + 1), cudaMemcpyHostToDevice, ar.st));
    CTG_CUDA_CHECK(cudaMemcpyAsync(d_b, b, 4 * static_cast<size_t>(nb + 1), cudaMemcpyHostToDevice, ar.st));
    const size_t gb = uni_gbuf_bytes(gcd_degree_smem(na, nb), 1);
    uint32_t* gbuf = gb ? ar.alloc<uint32_t>(gb / 4) : nullptr;
    cudaEvent_t e0, e1;
    CTG_CUDA_CHECK(cudaEventCreate(&e0));
    CTG_CUDA_CHECK(cudaEventCreate(&e1));
    CTG_CUDA_CHECK(cudaEventRecord(e0, ar.st));
    // CTG_LEHMER_PROF=1: phase cycles of the blocked kernel (printed to stderr; A/B only)
    static const bool prof_on = std::getenv("CTG_LEHMER_PROF") != nullptr;
    unsigned long long* d_prof = nullptr;
    if (prof_on) {
      d_prof = ar.alloc<unsigned long long>(8);
      CTG_CUDA_CHECK(cudaMemsetAsync(d_prof, 0, 64, ar.st));
    }
    const int rc = launch_gcd_degree(d_a, na, d_b, nb, T->d_pc, method, d_out, gbuf, ar.st, d_prof);
    CTG_CUDA_CHECK(cudaEventRecord(e1, ar.st));
    CTG_CUDA_CHECK(cudaGetLastError());
    int32_t h = 0;
    CTG_CUDA_CHECK(cudaMemcpyAsync(&h, d_out, 4, cudaMemcpyDeviceToHost, ar.st));
    CTG_CUDA_CHECK(cudaStreamSynchronize(ar.st));
    float t = 0.f;
    CTG_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc < 0) throw ApiError(CTG_INTERNAL, "modp_gcd_degree: no scratch");
    if (d_prof) {
      unsigned long long hp[8];
      CTG_CUDA_CHECK(cudaMemcpy(hp, d_prof, 64, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "lehmer prof n=%d: leaf %llu, bottom %llu, top %llu cycles; blocks %llu, gap passes %llu\n",
                   na, hp[0], hp[1], hp[2], hp[3], hp[4]);
    }
    *deg = h;
    if (prime) *prime = one[0];
    if (ms) *ms = t;
    stats_tls().kernel_launches = 1;
  });
}
