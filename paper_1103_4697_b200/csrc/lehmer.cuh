// K6 blocked remainder sequence (Lehmer-style): deg gcd(X, Y) over F_p with one CTA barrier per
// ~31 Euclid steps instead of one per step.
//
// blk_gcd (kernels_uni.cu) runs the division-free Euclid of the reference's gcd
// (/root/reference/proj/src/elim.cpp:80-93, over F_p) one pass per step: at deg 870 (the d30
// square-freeness probe, elim.cpp:138-165 via lift.cpp:64-67) that is 870 CTA passes of a few
// products per thread, each ~600 cycles of latency (load, scalars, update, barrier, trim).
// Here one warp (the "leaf") holds the top T = 62 coefficients of X and Y in registers (two per
// lane, lane 31 a zero sentinel) and runs every step those coefficients determine -- about 30 --
// with warp shuffles only, accumulating the 2x2 matrix of polynomials M (one coefficient per
// lane, degree <= 30) with (X_cur, Y_cur) = M (X_0, Y_0).  The CTA then applies M to the full
// polynomials: the top 62 coefficients of each first (all warps, so the leaf can start its next
// block), the rest by the warps on the other three SM sub-partitions while the leaf runs
// (lazily reduced dot products).  Exactness: every window tracks the lowest coefficient index it
// knows exactly (lo); a step runs only when its scalars and the new remainder's leading
// coefficient are exact.  A degree gap beyond M's reach (> 30) takes a direct elimination pass;
// a remainder whose exact window is all zero ends the block and the CTA finds its degree after
// the full product.  The algorithm is modelled step for step (and checked against a plain
// Euclid) in tests/test_lehmer_model.py.
//
// Measured (B200, n = 870 square-free, scripts/lehmer_ab.py): 275 us one pass per step, 192 us
// blocked with the 31-bit primes, 157 us blocked modulo a probe prime < 2^15.  The leaf is bound
// by its single warp's issue (about 86 instructions per Euclid step, IMAD / IMAD.WIDE pipe
// occupancy and fixed-latency waits: ~250 cycles per step), the top rows by latency.
#pragma once
#include <cstdint>

#include "modarith.cuh"

namespace ctg {
namespace lehmer {

constexpr int kT = 62;            // window coefficients (2 per lane, lanes 0..30)
constexpr int kMD = 30;           // max degree of M's entries (1 coefficient per lane, lanes 1..31)
constexpr int kAll = -(1 << 20);  // lo of a window that holds its whole polynomial
enum : int { kOk = 0, kDone = 1, kConst = 2, kUnknown = 3 };

// Two arithmetics, one algorithm.  MontA: Montgomery residues modulo the 31-bit K6 primes
// (p < 2^30.4, three-product reductions: modarith.cuh); a product is IMAD.WIDE (~6 issue cycles
// per warp on B200: 22 results/clk/SM) plus the reduction.  SmallA: plain residues modulo primes
// p < 2^15 (the square-freeness probe: any prime not dividing lc certifies), where three
// products fit 32 bits and a product is one IMAD (2 cycles) plus a shared Barrett reduction --
// half the pipe time and a shorter dependency chain per Euclid step.
struct MontA {
  Mod M;
  using Acc = uint64_t;
  static constexpr int kFoldA = 2;  // apply_bottom: fold every 2 a (4 products per accumulator)
  static constexpr int kFoldQ = 4;  // dot_half: fold every 4 q (4 products per accumulator)
  __device__ __forceinline__ uint32_t one() const { return M.one; }
  // -a mod p as a value in [1, p] (p stands for 0; three products of operands <= p still < 2^62.4)
  __device__ __forceinline__ uint32_t neg(uint32_t a) const { return M.p - a; }
  __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return mmul(a, b, M); }
  __device__ __forceinline__ uint32_t mul2(uint32_t a, uint32_t b, uint32_t c, uint32_t d) const {
    return mmul2(a, b, c, d, M);
  }
  __device__ __forceinline__ uint32_t mul3(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                           uint32_t f) const {
    return mmul3(a, b, c, d, e, f, M);
  }
  __device__ __forceinline__ Acc mac(Acc t, uint32_t a, uint32_t b) const { return t + static_cast<uint64_t>(a) * b; }
  // t mod p up to a multiple of p: hi * (2^32 mod p) + lo  (< 2^61.7 for t < 2^64, p < 2^30.4)
  __device__ __forceinline__ Acc fold(Acc t) const {
    return static_cast<uint64_t>(static_cast<uint32_t>(t >> 32)) * M.one + static_cast<uint32_t>(t);
  }
  __device__ __forceinline__ uint32_t finish(Acc t) const { return redc(fold(t), M.p, M.pneg); }
  __device__ __forceinline__ uint32_t inv(uint32_t a) const { return minv(a, M); }
  __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const { return msub(a, b, M.p); }
};
struct SmallA {
  uint32_t p, m, np;  // m = floor(2^32 / p), np = 2^32 - p (opaque: see make_small)
  using Acc = uint32_t;
  static constexpr int kFoldA = 1;  // 2 products per accumulator between reductions (< p + 2^31)
  static constexpr int kFoldQ = 2;
  __device__ __forceinline__ uint32_t red(uint32_t x) const {  // x mod p, any x < 2^32
    const uint32_t q = __umulhi(x, m);
    return csub(x + q * np, p);  // one IMAD (q np + x): np must not be folded back into -p
  }
  __device__ __forceinline__ uint32_t one() const { return 1u; }
  // -a mod p as a value in [1, p] (p itself stands for 0: operands up to p keep every bound)
  __device__ __forceinline__ uint32_t neg(uint32_t a) const { return p - a; }
  __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return red(a * b); }
  __device__ __forceinline__ uint32_t mul2(uint32_t a, uint32_t b, uint32_t c, uint32_t d) const {
    return red(a * b + c * d);
  }
  __device__ __forceinline__ uint32_t mul3(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e,
                                           uint32_t f) const {
    return red(a * b + c * d + e * f);
  }
  __device__ __forceinline__ Acc mac(Acc t, uint32_t a, uint32_t b) const { return t + a * b; }
  __device__ __forceinline__ Acc fold(Acc t) const { return red(t); }
  __device__ __forceinline__ uint32_t finish(Acc t) const { return red(t); }
  __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const { return a >= b ? a - b : a + p - b; }
  __device__ __forceinline__ uint32_t inv(uint32_t a) const {  // a^(p-2)
    uint32_t r = 1u, b = a;
    for (uint32_t e = p - 2; e; e >>= 1) {
      if (e & 1u) r = mul(r, b);
      b = mul(b, b);
    }
    return r;
  }
};
__device__ __forceinline__ SmallA make_small(uint32_t p) {
  uint32_t np;
  asm("mov.b32 %0, %1;" : "=r"(np) : "r"(0u - p));  // keeps ptxas from rewriting q*np + x as -(q)*p + x
  return SmallA{p, 0xffffffffu / p, np};
}

// Shift a blocked window (entry 2l in w0, 2l+1 in w1 of lane l) left by z: entry j <- j + z.
__device__ __forceinline__ void win_shift(uint32_t& w0, uint32_t& w1, int z, int lane) {
  const int h = z >> 1;
  if ((z & 1) == 0) {
    const uint32_t a = __shfl_down_sync(0xffffffffu, w0, h), b = __shfl_down_sync(0xffffffffu, w1, h);
    const bool in = lane + h < 32;
    w0 = in ? a : 0u;
    w1 = in ? b : 0u;
  } else {
    const uint32_t a = __shfl_down_sync(0xffffffffu, w1, h), b = __shfl_down_sync(0xffffffffu, w0, (h + 1) & 31);
    w0 = lane + h < 32 ? a : 0u;
    w1 = lane + h + 1 < 32 ? b : 0u;
  }
}

// First exact nonzero entry of a window whose entry j is coefficient dtop - j (exact iff
// dtop - j >= max(lo, 0)); -1 if none.
__device__ __forceinline__ int win_first(uint32_t w0, uint32_t w1, int dtop, int lo, int lane) {
  const int jmax = dtop - (lo > 0 ? lo : 0);
  const unsigned m0 = __ballot_sync(0xffffffffu, w0 != 0u && 2 * lane <= jmax);
  const unsigned m1 = __ballot_sync(0xffffffffu, w1 != 0u && 2 * lane + 1 <= jmax);
  const unsigned m = m0 | m1;
  if (!m) return -1;
  const int L = __ffs(m) - 1;
  return 2 * L + (((m0 >> L) & 1u) ? 0 : 1);
}

struct LeafResult {
  int dx, dy, status;
};

// One normal step on named registers (the roles of the X / Y register sets alternate between
// calls, so the fast loop needs no register moves).  In: X window (P0, P1), Y window (Q0, Q1),
// M rows (MX0, MX1) / (MY0, MY1), warp-uniform tops X[0..3] = (xa, xb, xc, xd), Y[0..3] =
// (ya..yd).  Out: the remainder r in (P0, P1), r's M row in (MX0, MX1), r's tops in (xa..xd);
// so afterwards the (P, MX, x) sets hold the new Y and the (Q, MY, y) sets the new X.
//   r = b^2 X - (b a y + X1) Y,  X1 = b x1 - a y1   (blk_gcd's normal step, top-aligned).
// The critical path is warp-uniform: the scalars and r's two leading entries are computed by
// every lane from the replicated tops (no shuffle waits); r's entries 2 and 3 arrive from lane
// 1 one step ahead of their use.  Lane 31 of the windows and lane 0 of M are zero sentinels, so
// the neighbour shuffles need no masking.
#define CTG_LEHMER_STEP(P0, P1, Q0, Q1, MX0, MX1, MY0, MY1, xa, xb, xc, xd, ya, yb, yc, yd)          \
  do {                                                                                              \
    const uint32_t na_ = A.neg(xa), nxb_ = A.neg(xb);                                               \
    const uint32_t c1_ = A.mul(ya, ya), c2_ = A.mul(ya, na_);                                       \
    const uint32_t c3_ = A.mul2(xa, yb, nxb_, ya); /* -(b x1 - a y1) */                             \
    const uint32_t xn0_ = __shfl_down_sync(0xffffffffu, P0, 1), xn1_ = __shfl_down_sync(0xffffffffu, P1, 1); \
    const uint32_t yn0_ = __shfl_down_sync(0xffffffffu, Q0, 1), yn1_ = __shfl_down_sync(0xffffffffu, Q1, 1); \
    const uint32_t u0_ = __shfl_up_sync(0xffffffffu, MY0, 1), u1_ = __shfl_up_sync(0xffffffffu, MY1, 1);     \
    const uint32_t r0u_ = A.mul3(c1_, xc, c2_, yc, c3_, yb), r1u_ = A.mul3(c1_, xd, c2_, yd, c3_, yc);       \
    P0 = A.mul3(c1_, xn0_, c2_, yn0_, c3_, Q1);                                                     \
    P1 = A.mul3(c1_, xn1_, c2_, yn1_, c3_, yn0_);                                                   \
    MX0 = A.mul3(c1_, MX0, c2_, u0_, c3_, MY0);                                                     \
    MX1 = A.mul3(c1_, MX1, c2_, u1_, c3_, MY1);                                                     \
    xc = __shfl_sync(0xffffffffu, P0, 1);                                                           \
    xd = __shfl_sync(0xffffffffu, P1, 1);                                                           \
    xa = r0u_;                                                                                      \
    xb = r1u_;                                                                                      \
  } while (0)

// The leaf: warp-uniform call by one warp.  Windows come from X (degree dx) and Y (degree dy),
// dx >= dy >= 1, dx - dy <= kMD; M goes to Mo[4 a + e] (e = m00, m01, m10, m11).
// Layout: window entry j (coefficient d - j) in lane j / 2, register j % 2, lanes 0..30 (kT = 62
// entries; lane 31 stays zero); M's coefficient a in lane a + 1 (lane 0 stays zero).
template <class Ar>
__device__ __forceinline__ LeafResult leaf_run(const uint32_t* X, int dx, const uint32_t* Y, int dy, const Ar& A,
                                               uint32_t* Mo) {
  const int lane = threadIdx.x & 31;
  const bool dl = lane < 31;
  uint32_t wx0 = dl && dx - 2 * lane >= 0 ? X[dx - 2 * lane] : 0u;
  uint32_t wx1 = dl && dx - 2 * lane - 1 >= 0 ? X[dx - 2 * lane - 1] : 0u;
  uint32_t wy0 = dl && dy - 2 * lane >= 0 ? Y[dy - 2 * lane] : 0u;
  uint32_t wy1 = dl && dy - 2 * lane - 1 >= 0 ? Y[dy - 2 * lane - 1] : 0u;
  int lox = dx >= kT ? dx - kT + 1 : kAll, loy = dy >= kT ? dy - kT + 1 : kAll;
  uint32_t m00 = lane == 1 ? A.one() : 0u, m01 = 0u, m10 = 0u, m11 = m00;
  int dmx = 0, dmy = 0, status = kOk;
  // warp-uniform copies of the windows' entries 0..3 (lanes 0 and 1)
  uint32_t xa = __shfl_sync(0xffffffffu, wx0, 0), xb = __shfl_sync(0xffffffffu, wx1, 0);
  uint32_t xc = __shfl_sync(0xffffffffu, wx0, 1), xd = __shfl_sync(0xffffffffu, wx1, 1);
  uint32_t ya = __shfl_sync(0xffffffffu, wy0, 0), yb = __shfl_sync(0xffffffffu, wy1, 0);
  uint32_t yc = __shfl_sync(0xffffffffu, wy0, 1), yd = __shfl_sync(0xffffffffu, wy1, 1);
  for (;;) {
    if (dy == 0) {
      status = kConst;
      break;
    }
    if (dx == dy + 1) {
      if (dx - 1 < lox || dy - 1 < loy || dmy + 1 > kMD) break;
      // Fast loop: normal steps, two per iteration.  Each step: X' = Y, Y' = r with
      // deg r = dy - 1 (checked: r's leading entry exact and nonzero), lo_r = max(lox, loy + 1).
      int lr, dt;
      bool drop = false;
      for (;;) {
        CTG_LEHMER_STEP(wx0, wx1, wy0, wy1, m00, m01, m10, m11, xa, xb, xc, xd, ya, yb, yc, yd);
        // now: X = (wy, m1*, y*), Y = r = (wx, m0*, x*)
        lr = lox > loy + 1 ? lox : loy + 1;
        dt = dy - 1;
        {
          const int dm = dmx > dmy + 1 ? dmx : dmy + 1;
          dmx = dmy;
          dmy = dm;
        }
        lox = loy;
        dx = dy;
        if (xa == 0u || dt < (lr > 0 ? lr : 0)) {
          drop = true;
        } else {
          loy = lr;
          dy = dt;
          if (!(dx - 1 < lox || dy - 1 < loy || dmy + 1 > kMD)) {
            CTG_LEHMER_STEP(wy0, wy1, wx0, wx1, m10, m11, m00, m01, ya, yb, yc, yd, xa, xb, xc, xd);
            // canonical again: X = (wx, m0*, x*), Y = r = (wy, m1*, y*)
            lr = lox > loy + 1 ? lox : loy + 1;
            dt = dy - 1;
            const int dm = dmx > dmy + 1 ? dmx : dmy + 1;
            dmx = dmy;
            dmy = dm;
            lox = loy;
            dx = dy;
            if (ya == 0u || dt < (lr > 0 ? lr : 0)) {
              drop = true;
              break;
            }
            loy = lr;
            dy = dt;
            if (dx - 1 < lox || dy - 1 < loy || dmy + 1 > kMD) break;
            continue;
          }
        }
        // odd exit: swap the register sets back to canonical (X in wx / m0* / x*)
        uint32_t s;
        s = wx0, wx0 = wy0, wy0 = s;
        s = wx1, wx1 = wy1, wy1 = s;
        s = m00, m00 = m10, m10 = s;
        s = m01, m01 = m11, m11 = s;
        s = xa, xa = ya, ya = s;
        s = xb, xb = yb, yb = s;
        s = xc, xc = yc, yc = s;
        s = xd, xd = yd, yd = s;
        break;
      }
      if (!drop) {
        if (dx - 1 < lox || dy - 1 < loy || dmy + 1 > kMD) break;  // block ends with exact degrees
        continue;
      }
      // r (in wy) has no exact nonzero leading entry at dt: find its degree
      const int z = win_first(wy0, wy1, dt, lr, lane);
      if (z < 0) {
        status = lr <= 0 ? kDone : kUnknown;
        dy = lr <= 0 ? -1 : dt;
        break;
      }
      win_shift(wy0, wy1, z, lane);
      loy = lr;
      dy = dt - z;
      ya = __shfl_sync(0xffffffffu, wy0, 0);
      yb = __shfl_sync(0xffffffffu, wy1, 0);
      yc = __shfl_sync(0xffffffffu, wy0, 1);
      yd = __shfl_sync(0xffffffffu, wy1, 1);
    } else {
      const int sh = dx - dy;
      if (dx < lox || dy < loy || dmy + sh > kMD) break;
      // X <- b X - a y^sh Y  (the top coefficient cancels)
      const uint32_t t = A.neg(xa);
      uint32_t n0 = A.mul2(ya, wx0, t, wy0), n1 = A.mul2(ya, wx1, t, wy1);
      uint32_t u10 = __shfl_up_sync(0xffffffffu, m10, sh), u11 = __shfl_up_sync(0xffffffffu, m11, sh);
      if (lane < sh) u10 = u11 = 0u;
      m00 = A.mul2(ya, m00, t, u10);
      m01 = A.mul2(ya, m01, t, u11);
      dmx = dmx > dmy + sh ? dmx : dmy + sh;
      const int ln = lox > loy + sh ? lox : loy + sh;
      const int z = win_first(n0, n1, dx, ln, lane);
      if (z < 0) {
        // X is zero (gcd = Y) or of unknown degree: hand back (Y, X) so that X is exact
        uint32_t s = m00;
        m00 = m10;
        m10 = s;
        s = m01;
        m01 = m11;
        m11 = s;
        status = ln <= 0 ? kDone : kUnknown;
        const int ody = ln <= 0 ? -1 : dx - 1;
        dx = dy;
        dy = ody;
        break;
      }
      win_shift(n0, n1, z, lane);
      wx0 = n0;
      wx1 = n1;
      lox = ln;
      dx -= z;
      xa = __shfl_sync(0xffffffffu, wx0, 0);
      xb = __shfl_sync(0xffffffffu, wx1, 0);
      xc = __shfl_sync(0xffffffffu, wx0, 1);
      xd = __shfl_sync(0xffffffffu, wx1, 1);
      if (dx < dy) {
        uint32_t s;
        s = wx0, wx0 = wy0, wy0 = s;
        s = wx1, wx1 = wy1, wy1 = s;
        s = m00, m00 = m10, m10 = s;
        s = m01, m01 = m11, m11 = s;
        s = xa, xa = ya, ya = s;
        s = xb, xb = yb, yb = s;
        s = xc, xc = yc, yc = s;
        s = xd, xd = yd, yd = s;
        int q;
        q = lox, lox = loy, loy = q;
        q = dx, dx = dy, dy = q;
        q = dmx, dmx = dmy, dmy = q;
      }
    }
  }
  // coefficient a of M lives in lane a + 1; lane 0 writes the (zero) coefficient 31
  reinterpret_cast<uint4*>(Mo)[lane == 0 ? 31 : lane - 1] =
      lane == 0 ? make_uint4(0u, 0u, 0u, 0u) : make_uint4(m00, m01, m10, m11);
  return LeafResult{dx, dy, status};
}
#undef CTG_LEHMER_STEP

// One output coefficient: sum over a = a0, a0 + 2, ..., a0 + 30 of e0[a] X[i - a] + e1[a] Y[i - a]
// (two threads split the a range; fully unrolled, two accumulator chains).  Returns a folded
// accumulator congruent to the sum.
template <class Ar>
__device__ __forceinline__ typename Ar::Acc dot_half(const uint32_t* Ms, int e, const uint32_t* X, int dx,
                                                     const uint32_t* Y, int dy, int i, int a0, const Ar& A) {
  typename Ar::Acc acc0 = 0, acc1 = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int a = a0 + 2 * q, j = i - a;
    const uint2 m = *reinterpret_cast<const uint2*>(Ms + 4 * a + e);
    const uint32_t xv = (j >= 0 && j <= dx) ? X[j] : 0u, yv = (j >= 0 && j <= dy) ? Y[j] : 0u;
    if (q & 1)
      acc1 = A.mac(A.mac(acc1, m.x, xv), m.y, yv);
    else
      acc0 = A.mac(A.mac(acc0, m.x, xv), m.y, yv);
    if ((q % Ar::kFoldQ) == Ar::kFoldQ - 1) {
      acc0 = A.fold(acc0);
      acc1 = A.fold(acc1);
    }
  }
  return A.fold(A.fold(acc0) + A.fold(acc1));
}

// X2[i] (i in [lo_x, hi_x]) and Y2[i] (i in [lo_y, hi_y]) = M (X, Y): two threads per output,
// thread t of `nthr` (consecutive, nthr even).
template <class Ar>
__device__ __forceinline__ void apply_top(const uint32_t* Ms, const uint32_t* X, int dx, const uint32_t* Y, int dy,
                                          uint32_t* X2, int lo_x, int hi_x, uint32_t* Y2, int lo_y, int hi_y,
                                          int t, int nthr, const Ar& A) {
  const int nx = hi_x - lo_x + 1, ny = hi_y >= lo_y ? hi_y - lo_y + 1 : 0;
  for (int ob = 0; ob < nx + ny; ob += nthr >> 1) {  // warp-uniform trip count (shuffles below)
    const int o = ob + (t >> 1);
    const bool valid = o < nx + ny, isx = o < nx;
    const int i = isx ? hi_x - o : hi_y - (o - nx);
    typename Ar::Acc acc = valid ? dot_half(Ms, isx ? 0 : 2, X, dx, Y, dy, i, t & 1, A) : 0u;
    const typename Ar::Acc other = __shfl_xor_sync(0xffffffffu, acc, 1);
    if (valid && !(t & 1)) (isx ? X2 : Y2)[i] = A.finish(acc + other);
  }
}

// Bottom rows: X2[i] for i in [0, hx], Y2[i] for i in [0, hy], 4 consecutive outputs of both per
// thread with a sliding register window over X and Y (thread t of nthr).
template <class Ar>
__device__ __forceinline__ void apply_bottom(const uint32_t* Ms, const uint32_t* X, int dx, const uint32_t* Y, int dy,
                                             uint32_t* X2, int hx, uint32_t* Y2, int hy, int t, int nthr,
                                             const Ar& A) {
  const int hi = hx > hy ? hx : hy;
  for (int i0 = 4 * t; i0 <= hi; i0 += 4 * nthr) {
    typename Ar::Acc ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0};
    uint32_t xs[4], ys[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xs[k] = i0 + k <= dx ? X[i0 + k] : 0u;
      ys[k] = i0 + k <= dy ? Y[i0 + k] : 0u;
    }
#pragma unroll 2
    for (int a = 0; a <= kMD; ++a) {
      if (a) {
#pragma unroll
        for (int k = 3; k > 0; --k) {
          xs[k] = xs[k - 1];
          ys[k] = ys[k - 1];
        }
        const int j = i0 - a;
        xs[0] = j >= 0 && j <= dx ? X[j] : 0u;
        ys[0] = j >= 0 && j <= dy ? Y[j] : 0u;
      }
      const uint4 m = reinterpret_cast<const uint4*>(Ms)[a];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ax[k] = A.mac(A.mac(ax[k], m.x, xs[k]), m.y, ys[k]);
        ay[k] = A.mac(A.mac(ay[k], m.z, xs[k]), m.w, ys[k]);
      }
      if (a % Ar::kFoldA == Ar::kFoldA - 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          ax[k] = A.fold(ax[k]);
          ay[k] = A.fold(ay[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + k;
      if (i <= hx) X2[i] = A.finish(ax[k]);
      if (i <= hy) Y2[i] = A.finish(ay[k]);
    }
  }
}

// Scale X[0..d] to monic in place (lc nonzero); every thread calls it.
template <class Ar>
__device__ __forceinline__ void blk_make_monic(uint32_t* X, int d, const Ar& A) {
  const uint32_t inv = A.inv(X[d]);
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) X[i] = A.mul(X[i], inv);
  if (threadIdx.x == 0) X[d] = A.one();
  __syncthreads();
}

// gcd(X, Y) over F_p by the blocked remainder sequence.  X, Y: exact degrees dx, dy, written and
// synchronised by the caller; X2, Y2: two more buffers of the same capacity.  The four buffer
// pointers are permuted (the caller's set of four stays the same; all are clobbered).
// FULL = false: returns deg gcd (-1 if both vanish).  FULL = true: also leaves the monic gcd in
// X (its degree returned).  Ms: 2 x 128 words of shared memory, ctl: 4 ints of shared memory.
// Every thread of the CTA calls it (blockDim.x a multiple of 128); returns on every thread.
// prof (A/B hook only, null otherwise): cycles of [0] leaf, [1] bottom rows (warp 1), [2] top rows +
// barriers (thread 0), [3] blocks, [4] gap passes.
template <bool FULL, class Ar>
__device__ int blk_gcd_core(uint32_t*& X, int dx, uint32_t*& Y, int dy, uint32_t*& X2, uint32_t*& Y2, uint32_t* Ms,
                            int* ctl, const Ar& A, unsigned long long* prof = nullptr) {
  const int tid = threadIdx.x, bs = blockDim.x, warp = tid >> 5;
  // warps off the leaf's sub-partition (warp % 4 != 0) apply the bottom rows during the leaf
  const int napp = (bs >> 5) - ((bs >> 5) + 3) / 4;
  const bool app = (warp & 3) != 0;
  bool pend = false;
  const uint32_t *Xp = nullptr, *Yp = nullptr, *Mp = nullptr;
  int pdx = 0, pdy = 0, cur = 0;
  auto constant_gcd = [&]() {  // gcd is a nonzero constant: monic 1
    if constexpr (FULL) {
      if (tid == 0) X[0] = A.one();
      __syncthreads();
    }
    return 0;
  };
  for (;;) {
    if (dx < dy) {  // (never with a pending bottom: the leaf hands back dx >= dy when it is exact)
      uint32_t* s = X;
      X = Y;
      Y = s;
      s = X2;
      X2 = Y2;
      Y2 = s;
      const int q = dx;
      dx = dy;
      dy = q;
    }
    if (dy < 0) {  // (X is complete here: no pending bottom)
      if constexpr (FULL) {
        if (dx >= 0) blk_make_monic(X, dx, A);
      }
      return dx;
    }
    if (dy == 0) return constant_gcd();
    if (dx - dy > kMD) {
      // gap beyond M: complete the full polynomials, then one direct elimination pass
      if (pend) {
        apply_bottom(Mp, Xp, pdx, Yp, pdy, X, dx - kT, Y, dy - kT, tid, bs, A);
        pend = false;
        __syncthreads();
      }
      if (prof && tid == 0) atomicAdd(prof + 4, 1ull);
      const uint32_t c = Y[dy], t = A.neg(X[dx]);
      const int sh = dx - dy;
      for (int i = tid; i < dx; i += bs) X[i] = i >= sh ? A.mul2(c, X[i], t, Y[i - sh]) : A.mul(c, X[i]);
      __syncthreads();
      int d = dx - 1;
      while (d >= 0 && X[d] == 0u) --d;
      dx = d;
      continue;
    }
    uint32_t* Mc = Ms + 128 * cur;
    long long c0 = prof ? clock64() : 0;
    if (warp == 0) {
      const LeafResult r = leaf_run(X, dx, Y, dy, A, Mc);
      if (prof && tid == 0) {
        atomicAdd(prof, static_cast<unsigned long long>(clock64() - c0));
        atomicAdd(prof + 3, 1ull);
      }
      if (tid == 0) {
        ctl[0] = r.dx;
        ctl[1] = r.dy;
        ctl[2] = r.status;
      }
    } else if (pend && app) {
      apply_bottom(Mp, Xp, pdx, Yp, pdy, X, dx - kT, Y, dy - kT, (warp - 1 - (warp >> 2)) * 32 + (tid & 31),
                   napp * 32, A);
      if (prof && tid == 32) atomicAdd(prof + 1, static_cast<unsigned long long>(clock64() - c0));
    }
    __syncthreads();
    c0 = prof ? clock64() : 0;
    const int ndx = ctl[0], st = ctl[2];
    int ndy = ctl[1];
    pend = false;
    if (st == kConst) {
      __syncthreads();  // everyone has read ctl
      return constant_gcd();
    }
    if (st == kDone) {
      if constexpr (FULL) {  // the gcd is the new X: its full product, then monic
        apply_bottom(Mc, X, dx, Y, dy, X2, ndx, Y2, -1, tid, bs, A);
        __syncthreads();
        uint32_t* s = X;
        X = X2;
        X2 = s;
        blk_make_monic(X, ndx, A);
      }
      return ndx;
    }
    if (st == kUnknown) {
      // full product, then the degree of Y2 from its upper bound
      apply_bottom(Mc, X, dx, Y, dy, X2, ndx, Y2, ndy, tid, bs, A);
      if (tid == 0) ctl[3] = -1;
      __syncthreads();
      for (int i = tid; i <= ndy; i += bs)
        if (Y2[i] != 0u) atomicMax(ctl + 3, i);
      __syncthreads();
      ndy = ctl[3];
      __syncthreads();  // ctl is rewritten by the next leaf
    } else {
      apply_top(Mc, X, dx, Y, dy, X2, ndx - kT + 1 > 0 ? ndx - kT + 1 : 0, ndx, Y2, ndy - kT + 1 > 0 ? ndy - kT + 1 : 0,
                ndy, tid, bs, A);
      __syncthreads();
      if (prof && tid == 0) atomicAdd(prof + 2, static_cast<unsigned long long>(clock64() - c0));
      pend = true;
      Xp = X;
      Yp = Y;
      Mp = Mc;
      pdx = dx;
      pdy = dy;
      cur ^= 1;
    }
    uint32_t* s = X;
    X = X2;
    X2 = s;
    s = Y;
    Y = Y2;
    Y2 = s;
    dx = ndx;
    dy = ndy;
  }
}

// deg gcd(X, Y) over F_p (-1 if both vanish); the four buffers are clobbered.
template <class Ar>
__device__ int blk_gcd_degree(uint32_t* X, int dx, uint32_t* Y, int dy, uint32_t* X2, uint32_t* Y2, uint32_t* Ms,
                              int* ctl, const Ar& A, unsigned long long* prof = nullptr) {
  return blk_gcd_core<false>(X, dx, Y, dy, X2, Y2, Ms, ctl, A, prof);
}

// Exact division by a monic divisor, blocked the same way: Q = X / D (deg dq = dx - dd; X
// destroyed).  Per block of 32 quotient coefficients one warp runs the long division on the top
// 32 coefficients of X in registers (one broadcast + one product per coefficient and step: the
// chain is a shuffle and a multiply, not a CTA pass), then the CTA subtracts the block's
// Q_blk * D from the coefficients below (dot products of length <= 32) and synchronises once.
// One CTA pass per 32 quotient coefficients instead of one per coefficient (blk_divexact_monic).
template <class Ar>
__device__ int blk_divexact_blocked(uint32_t* X, int dx, const uint32_t* D, int dd, uint32_t* Q, const Ar& A) {
  const int tid = threadIdx.x, bs = blockDim.x, lane = tid & 31;
  if (dd == 0) {
    for (int i = tid; i <= dx; i += bs) Q[i] = X[i];
    __syncthreads();
    return dx;
  }
  const int dq = dx - dd;
  for (int top = dq; top >= 0; top -= 32) {  // quotient coefficients top .. top - K + 1
    const int K = top + 1 < 32 ? top + 1 : 32;
    if (tid < 32) {
      uint32_t w = lane < K ? X[dd + top - lane] : 0u;  // X's window, top coefficient in lane 0
      uint32_t sd = lane <= dd ? D[dd - lane] : 0u;     // at step t: lane l holds D[dd - (l - t)]
      for (int t = 0; t < K; ++t) {
        const uint32_t q = __shfl_sync(0xffffffffu, w, t);
        if (lane == t) Q[top - t] = q;
        if (lane > t) w = A.sub(w, A.mul(q, sd));
        sd = __shfl_up_sync(0xffffffffu, sd, 1);
        if (lane == 0) sd = 0u;
      }
    }
    __syncthreads();
    // the coefficients below the window: X[i] -= sum_t q_t D[i - (top - t)]
    const int lo = top - K + 1, hi = dd + top - K;
    for (int i = lo + tid; i <= hi; i += bs) {
      typename Ar::Acc acc = 0;
      int n = 0;
      for (int t = 0; t < K; ++t) {
        const int j = i - top + t;
        if (j < 0) continue;
        if (j > dd) break;
        acc = A.mac(acc, Q[top - t], D[j]);
        if (++n == 2 * Ar::kFoldA) {
          acc = A.fold(acc);
          n = 0;
        }
      }
      X[i] = A.sub(X[i], A.finish(acc));
    }
    __syncthreads();
  }
  return dq;
}

}  // namespace lehmer
}  // namespace ctg
