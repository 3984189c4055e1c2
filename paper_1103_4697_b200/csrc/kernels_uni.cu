// K6: per-prime univariate gcd / Yun square-free decomposition (one CTA per prime,
// polynomials staged in shared memory), and the gather/scale kernel that builds
// the CRT residue matrix of the lucky primes (K7 then reuses the K5 CRT kernels).
//
// Replaces the reference's primitive PRS gcd (/root/reference/proj/src/elim.cpp:80-93)
// and Yun's loop (elim.cpp:138-165): over F_p there is no coefficient growth, so
// the Euclidean remainder sequence runs division-free in place; each pass is one
// vector update of the remainder (threads stride the coefficients) and one barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>

#include "internal.hpp"
#include "uni_internal.hpp"
#include "lehmer.cuh"

namespace ctg {
namespace {

__device__ __forceinline__ Mod load_mod_u(const PrimeConst& c) { return Mod{c.p, c.pneg, c.r2, c.one}; }

__device__ __forceinline__ int blk_trim(const uint32_t* X, int d) {
  while (d >= 0 && X[d] == 0u) --d;
  return d;
}

__device__ __forceinline__ void swp(uint32_t*& a, uint32_t*& b) {
  uint32_t* t = a;
  a = b;
  b = t;
}

// Polynomial buffers of a CTA: shared memory, or (degrees beyond the shared-memory budget)
// this CTA's slice of a global scratch region -- the kernels use generic pointers, so the
// same code runs on either (global buffers stay L2-resident: 8 x (n + 2) words per CTA).
// (Two instantiations of each kernel, GB = false / true: derived from the extern __shared__
// array the pointers stay in the shared window and compile to LDS / STS; a run-time select
// between the two would make every access a generic LD / ST -- measured 1.6x slower K6.)
template <bool GB>
__device__ __forceinline__ uint32_t* cta_buffers(uint32_t* sm, uint32_t* gbuf, size_t words_per_cta) {
  if constexpr (GB) return gbuf + static_cast<size_t>(blockIdx.x) * words_per_cta;
  return sm;
}

// Primes p < kResPrimeMax (2^30.4): the fused pass uses mmul3 (modarith.cuh).
// Monic gcd of X (degree dx) and Y (degree dy), destroying both; the result ends
// up in X (pointers are swapped as the remainder sequence proceeds).  Degrees are
// exact (top coefficient nonzero) or -1.  Returns the gcd's degree (-1 if both zero).
// Caller must have synchronised after writing X and Y.
__device__ int blk_gcd(uint32_t*& X, int dx, uint32_t*& Y, int dy, const Mod& M) {
  const int tid = threadIdx.x, bs = blockDim.x;
  if (dx < dy) {
    swp(X, Y);
    const int t = dx;
    dx = dy;
    dy = t;
  }
  while (dy >= 0) {
    while (dx >= dy) {
      if (dx == dy + 1 && dy >= 1) {
        // Two eliminations in one pass (the normal remainder step, as K3):
        //   X1 = b X - a_{k+1} y Y,  r = b X1 - X1_k Y = b^2 (X mod Y)   (k = dy, b = lc Y)
        //   r_i = b^2 x_i - b a_{k+1} y_{i-1} - X1_k y_i: three products, one reduction (mmul3).
        const uint32_t b = Y[dy], na = mneg(X[dx], M.p);
        const uint32_t c1 = mmul(b, b, M), c2 = mmul(b, na, M);
        const uint32_t c3 = mneg(mmul2(b, X[dy], na, Y[dy - 1], M), M.p);
        for (int i = tid; i < dy; i += bs)
          X[i] = i ? mmul3(c1, X[i], c2, Y[i - 1], c3, Y[i], M) : mmul2(c1, X[0], c3, Y[0], M);
        __syncthreads();
        dx = blk_trim(X, dy - 1);
        continue;
      }
      // X <- c X - t y^(dx-dy) Y   (c = lc Y, t = lc X): the top coefficient cancels.
      const uint32_t c = Y[dy], t = mneg(X[dx], M.p);
      const int sh = dx - dy;
      for (int i = tid; i < dx; i += bs) {
        const uint32_t v = X[i];
        X[i] = (i >= sh) ? mmul2(c, v, t, Y[i - sh], M) : mmul(c, v, M);
      }
      __syncthreads();
      dx = blk_trim(X, dx - 1);
    }
    swp(X, Y);
    const int t = dx;
    dx = dy;
    dy = t;
  }
  if (dx >= 0) {
    const uint32_t inv = minv(X[dx], M);
    __syncthreads();
    for (int i = tid; i < dx; i += bs) X[i] = mmul(X[i], inv, M);
    if (tid == 0) X[dx] = M.one;
    __syncthreads();
  }
  return dx;
}

// Q = X / D for a monic divisor D (degree dd <= dx); X is destroyed.  Returns deg Q.
__device__ int blk_divexact_monic(uint32_t* X, int dx, const uint32_t* D, int dd, uint32_t* Q, const Mod& M) {
  const int tid = threadIdx.x, bs = blockDim.x;
  if (dd == 0) {
    for (int i = tid; i <= dx; i += bs) Q[i] = X[i];
    __syncthreads();
    return dx;
  }
  for (int i = dx; i >= dd; --i) {
    const uint32_t q = X[i];
    const uint32_t nq = mneg(q, M.p);
    for (int j = tid; j < dd; j += bs) X[i - dd + j] = mmul2(M.one, X[i - dd + j], nq, D[j], M);
    if (tid == 0) Q[i - dd] = q;
    __syncthreads();
  }
  return dx - dd;
}

__device__ void blk_copy(uint32_t* dst, const uint32_t* src, int d) {
  for (int i = threadIdx.x; i <= d; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
}

// Z = d/dx V  (degree dv - 1), Montgomery form.
__device__ void blk_derivative(uint32_t* Z, const uint32_t* V, int dv, const Mod& M) {
  for (int i = threadIdx.x; i < dv; i += blockDim.x)
    Z[i] = mmul(V[i + 1], mmul(static_cast<uint32_t>(i + 1), M.r2, M), M);
  __syncthreads();
}

// Scale to monic in place (lc nonzero).
__device__ void blk_monic(uint32_t* X, int d, const Mod& M) {
  const uint32_t inv = minv(X[d], M);
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) X[i] = mmul(X[i], inv, M);
  if (threadIdx.x == 0) X[d] = M.one;
  __syncthreads();
}

__device__ void blk_store_plain(uint32_t* dst, const uint32_t* X, int d, const Mod& M) {
  for (int i = threadIdx.x; i <= d; i += blockDim.x) dst[i] = from_mont(X[i], M);
}

// ---------------------------------------------------------------------------
// Yun modulo p (elim.cpp:138-165 over F_p, p > deg P):
//   g = gcd(P, P'), v = P/g, w = P'/g;  repeat: z = w - v', h = gcd(v, z),
//   emit h (multiplicity k), v = v/h, w = z/h, k++  until deg v = 0.
// Outputs (plain residues): deg[k][m] = degree of the multiplicity-m factor (m >= 1),
// deg[k][0] = status (0 ok, 1 lc(P) = 0 mod p); the monic factors concatenated in
// increasing m (deg + 1 words each) at fac[k][...]; the monic square-free part at sqf[k][...].
// ---------------------------------------------------------------------------
template <bool GB>
__global__ void __launch_bounds__(512) k_modyun(const uint32_t* __restrict__ tab, int n, const PrimeConst* __restrict__ pc,
                                                int32_t* deg, uint32_t* fac, uint32_t* sqf, uint32_t* gbuf) {
  extern __shared__ uint32_t sm[];
  __shared__ __align__(16) uint32_t Ms[2 * 128];  // lehmer::blk_gcd_core's matrices and control
  __shared__ int ctl[4];
  const int kl = blockIdx.x;
  const Mod M = load_mod_u(pc[kl]);
  const lehmer::MontA MA{M};
  const int cap = n + 2;
  uint32_t* base = cta_buffers<GB>(sm, gbuf, 8 * cap);
  uint32_t* buf[8];
  for (int b = 0; b < 8; ++b) buf[b] = base + b * cap;
  int32_t* dk = deg + static_cast<size_t>(kl) * (n + 1);
  uint32_t* fk = fac + static_cast<size_t>(kl) * (2 * n + 2);
  uint32_t* sk = sqf + static_cast<size_t>(kl) * (n + 1);
  const uint32_t* row = tab + static_cast<size_t>(kl) * (n + 1);
  for (int i = threadIdx.x; i <= n; i += blockDim.x) {
    buf[0][i] = row[i];
    dk[i] = 0;
  }
  __syncthreads();
  if (buf[0][n] == 0u) {
    if (threadIdx.x == 0) dk[0] = 1;
    return;
  }
  uint32_t *A0 = buf[0], *A1 = buf[1], *X = buf[2], *Y = buf[3], *V = buf[4], *W = buf[5], *F1 = buf[6],
           *F2 = buf[7];
  blk_derivative(A1, A0, n, M);  // deg n-1 exactly (p > n, lc != 0)
  blk_copy(X, A0, n);
  blk_copy(Y, A1, n - 1);
  const int dg = lehmer::blk_gcd_core<true>(X, n, Y, n - 1, V, W, Ms, ctl, MA);  // monic gcd in X (V, W: scratch)
  if (dg == 0) {
    blk_monic(A0, n, M);
    blk_store_plain(fk, A0, n, M);
    blk_store_plain(sk, A0, n, M);
    if (threadIdx.x == 0) dk[1] = n;
    return;
  }
  int dv = lehmer::blk_divexact_blocked(A0, n, X, dg, V, MA);      // v = P / g
  int dw = lehmer::blk_divexact_blocked(A1, n - 1, X, dg, W, MA);  // w = P' / g
  {
    blk_copy(F1, V, dv);
    blk_monic(F1, dv, M);
    blk_store_plain(sk, F1, dv, M);
  }
  int off = 0;
  for (int k = 1; dv > 0 && k <= n; ++k) {
    // z = w - v'   (in place in W)
    for (int i = threadIdx.x; i <= dw || i < dv; i += blockDim.x) {
      const uint32_t wi = (i <= dw) ? W[i] : 0u;
      const uint32_t di = (i < dv) ? mmul(V[i + 1], mmul(static_cast<uint32_t>(i + 1), M.r2, M), M) : 0u;
      W[i] = msub(wi, di, M.p);
    }
    __syncthreads();
    const int dz = blk_trim(W, dw > dv - 1 ? dw : dv - 1);
    int dh;
    uint32_t* H;
    if (dz < 0) {
      blk_copy(X, V, dv);
      blk_monic(X, dv, M);
      H = X;
      dh = dv;
    } else {
      blk_copy(X, V, dv);
      blk_copy(Y, W, dz);
      dh = lehmer::blk_gcd_core<true>(X, dv, Y, dz, A0, A1, Ms, ctl, MA);  // A0, A1 are free by now
      H = X;
    }
    if (dh > 0) {
      blk_store_plain(fk + off, H, dh, M);
      off += dh + 1;
      if (threadIdx.x == 0) dk[k] = dh;
    }
    dv = lehmer::blk_divexact_blocked(V, dv, H, dh, F1, MA);
    swp(V, F1);
    if (dz >= 0) {
      dw = lehmer::blk_divexact_blocked(W, dz, H, dh, F2, MA);
      swp(W, F2);
    } else {
      dw = -1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Batched square-freeness probe (ctg_yun_squarefree_batch): CTA per (problem i, prime k);
// problem i's residues mod p_k are slots [off[i], off[i] + n_i] of row k (pitch S) of one K1
// table.  out[2 (i nk + k)] = status (0 ok, 1 lc(P) = 0 mod p), out[+1] = deg gcd(P, P') mod p.
// Four polynomial buffers of cap words (the largest degree + 2): lehmer::blk_gcd_degree.
// ---------------------------------------------------------------------------
template <bool GB, bool SMALL>
__global__ void __launch_bounds__(256) k_sqf_probe(const uint32_t* __restrict__ tab, int S, const int32_t* __restrict__ off,
                                                   const int32_t* __restrict__ degs, int nk,
                                                   const PrimeConst* __restrict__ pc, int cap, int32_t* out,
                                                   uint32_t* gbuf, int plain, int single_deg) {
  extern __shared__ uint32_t sm[];
  __shared__ __align__(16) uint32_t Ms[2 * 128];
  __shared__ int ctl[4];
  const int i = blockIdx.x / nk, k = blockIdx.x % nk;
  const int n = degs ? degs[i] : single_deg;  // one problem at offset 0 when degs is null
  const Mod M = load_mod_u(pc[k]);
  uint32_t* X = cta_buffers<GB>(sm, gbuf, 4 * static_cast<size_t>(cap));
  uint32_t *Y = X + cap, *X2 = X + 2 * cap, *Y2 = X + 3 * cap;
  const uint32_t* row = tab + static_cast<size_t>(k) * S + (off ? off[i] : 0);
  // SMALL: K1 residues (Montgomery form, i.e. 2^32 R mod p: a constant multiple of R, the same
  // gcd degree) read as plain residues modulo a prime < 2^15.
  for (int t = threadIdx.x; t <= n; t += blockDim.x) X[t] = (plain && !SMALL) ? mmul(row[t], M.r2, M) : row[t];
  __syncthreads();
  int32_t* o = out + 2 * (static_cast<size_t>(i) * nk + k);
  if (X[n] == 0u) {
    if (threadIdx.x == 0) {
      o[0] = 1;
      o[1] = -1;
    }
    return;
  }
  int dg;
  if constexpr (SMALL) {
    const lehmer::SmallA A = lehmer::make_small(M.p);
    for (int t = threadIdx.x; t < n; t += blockDim.x) Y[t] = A.mul(static_cast<uint32_t>(t + 1) % M.p, X[t + 1]);
    __syncthreads();
    dg = lehmer::blk_gcd_degree(X, n, Y, n - 1, X2, Y2, Ms, ctl, A);
  } else {
    blk_derivative(Y, X, n, M);  // deg n - 1 exactly (p > n, lc != 0)
    dg = lehmer::blk_gcd_degree(X, n, Y, n - 1, X2, Y2, Ms, ctl, lehmer::MontA{M});
  }
  if (threadIdx.x == 0) {
    o[0] = 0;
    o[1] = dg;
  }
}

// ---------------------------------------------------------------------------
// Test / A-B hook (ctg_modp_gcd_degree): deg gcd(a, b) mod one prime, plain residues in,
// by the blocked kernel (method 0: lehmer::blk_gcd_degree) or one pass per step (1: blk_gcd).
// ---------------------------------------------------------------------------
template <bool GB>
__global__ void __launch_bounds__(256) k_gcd_degree(const uint32_t* __restrict__ a, int na, const uint32_t* __restrict__ b,
                                                    int nb, const PrimeConst* __restrict__ pc, int cap, int method,
                                                    int32_t* out, uint32_t* gbuf, unsigned long long* prof) {
  extern __shared__ uint32_t sm[];
  __shared__ __align__(16) uint32_t Ms[2 * 128];
  __shared__ int ctl[4];
  const Mod M = load_mod_u(pc[0]);
  uint32_t* X = cta_buffers<GB>(sm, gbuf, 4 * static_cast<size_t>(cap));
  uint32_t *Y = X + cap, *X2 = X + 2 * cap, *Y2 = X + 3 * cap;
  for (int t = threadIdx.x; t < cap; t += blockDim.x) {  // method 2: plain residues mod a small prime
    X[t] = t <= na ? (method == 2 ? a[t] : mmul(a[t], M.r2, M)) : 0u;
    Y[t] = t <= nb ? (method == 2 ? b[t] : mmul(b[t], M.r2, M)) : 0u;
  }
  __syncthreads();
  const int dx = blk_trim(X, na), dy = blk_trim(Y, nb);
  int dg;
  if (method == 0) {
    dg = lehmer::blk_gcd_degree(X, dx, Y, dy, X2, Y2, Ms, ctl, lehmer::MontA{M}, prof);
  } else if (method == 2) {
    dg = lehmer::blk_gcd_degree(X, dx, Y, dy, X2, Y2, Ms, ctl, lehmer::make_small(M.p), prof);
  } else {
    dg = blk_gcd(X, dx, Y, dy, M);
  }
  if (threadIdx.x == 0) out[0] = dg;
}

// ---------------------------------------------------------------------------
// gcd modulo p with cofactors: g = monic gcd(A, B), u = A / g, w = B / g.
// Row layout (plain residues): g (dg+1) | u (na-dg+1) | w (nb-dg+1).  deg[k] = dg,
// or -2 if lc(A) or lc(B) vanishes mod p.
// ---------------------------------------------------------------------------
// Inputs either as K1 residue rows (tabA / tabB) or, for small gcds (one launch instead of two),
// as the staged coefficients themselves: `limbs` [na + nb + 2][Lw] (coefficient-major, A then B)
// and `sign`, reduced here with the K1 weights rpow (Lw <= kRedL).
struct GcdStaged {
  const uint32_t* limbs = nullptr;
  const int8_t* sign = nullptr;
  int Lw = 0;
  const uint32_t* rpow = nullptr;
};

template <bool GB>
__global__ void __launch_bounds__(512) k_modgcd(const uint32_t* __restrict__ tabA, int na,
                                                const uint32_t* __restrict__ tabB, int nb, int tab_pitch,
                                                const PrimeConst* __restrict__ pc, int32_t* deg, uint32_t* out,
                                                int pitch, uint32_t* gbuf, GcdStaged sg) {
  extern __shared__ uint32_t sm[];
  __shared__ __align__(16) uint32_t Ms[2 * 128];  // lehmer::blk_gcd_core's matrices and control
  __shared__ int ctl[4];
  const int kl = blockIdx.x;
  const Mod M = load_mod_u(pc[kl]);
  const int cap = (na > nb ? na : nb) + 2;
  uint32_t* base = cta_buffers<GB>(sm, gbuf, 6 * static_cast<size_t>(cap));
  uint32_t *A = base, *B = base + cap, *X = base + 2 * cap, *Y = base + 3 * cap, *Q = base + 4 * cap,
           *Z = base + 5 * cap;
  if (sg.limbs) {  // fused K1: coefficient s of A (s <= na) or B (s - na - 1), Montgomery form
    const uint32_t* w = sg.rpow + static_cast<size_t>(kl) * kRedL;
    for (int s = threadIdx.x; s <= na + nb + 1; s += blockDim.x) {
      const uint32_t* lb = sg.limbs + static_cast<size_t>(s) * sg.Lw;
      uint32_t acc = 0;
      for (int l = 0; l < sg.Lw; ++l) acc = madd(acc, mmul(lb[l], __ldg(&w[l]), M), M.p);
      if (sg.sign[s] < 0) acc = mneg(acc, M.p);
      if (s <= na)
        A[s] = X[s] = acc;
      else
        B[s - na - 1] = Y[s - na - 1] = acc;
    }
  } else {
    const uint32_t* ra = tabA + static_cast<size_t>(kl) * (tab_pitch ? tab_pitch : na + 1);
    const uint32_t* rb = tabB + static_cast<size_t>(kl) * (tab_pitch ? tab_pitch : nb + 1);
    for (int i = threadIdx.x; i <= na; i += blockDim.x) A[i] = X[i] = ra[i];
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) B[i] = Y[i] = rb[i];
  }
  __syncthreads();
  if (A[na] == 0u || B[nb] == 0u) {
    if (threadIdx.x == 0) deg[kl] = -2;
    return;
  }
  const lehmer::MontA MA{M};
  const int dg = lehmer::blk_gcd_core<true>(X, na, Y, nb, Q, Z, Ms, ctl, MA);  // monic gcd in X
  uint32_t* o = out + static_cast<size_t>(kl) * pitch;
  blk_store_plain(o, X, dg, M);
  const int du = lehmer::blk_divexact_blocked(A, na, X, dg, Q, MA);
  blk_store_plain(o + dg + 1, Q, du, M);
  __syncthreads();
  const int dw = lehmer::blk_divexact_blocked(B, nb, X, dg, Q, MA);
  blk_store_plain(o + dg + 1 + du + 1, Q, dw, M);
  if (threadIdx.x == 0) deg[kl] = dg;
}

// dst[r][c] = src[idx[r]][c] * scale[r][seg(c)]  (plain residues; scale in Montgomery form),
// seg(c) = number of segment boundaries <= c.
__global__ void k_gather_scale(const uint32_t* __restrict__ src, int src_pitch, const int32_t* __restrict__ idx,
                               int rows, int cols, const int32_t* __restrict__ seg_end, int nseg,
                               const uint32_t* __restrict__ scale, const PrimeConst* __restrict__ pc_dst,
                               uint32_t* __restrict__ dst) {
  const int r = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows || c >= cols) return;
  int s = 0;
  while (s + 1 < nseg && c >= seg_end[s]) ++s;
  const Mod M = load_mod_u(pc_dst[r]);
  const uint32_t v = src[static_cast<size_t>(idx[r]) * src_pitch + c];
  dst[static_cast<size_t>(r) * cols + c] = mmul(v, scale[static_cast<size_t>(r) * nseg + s], M);
}


// Bivariate gcd probe (ctg_gcd_bivariate): CTA per unit (prime k, point j).  The y-rows of
// f and g (slot runs of the reduced coefficient table, x-degree ascending) are evaluated at
// a_j by Horner, then gcd(f(a_j, y), g(a_j, y)) mod p_k runs in shared memory.  deg[unit] is
// the gcd degree, or -1 when the unit proves nothing (both formal leading y-coefficients
// vanish at a_j, or an image is identically zero).
template <bool GB>
__global__ void k_bigcd_probe(const uint32_t* __restrict__ tab, int S, const int32_t* __restrict__ dir, int nf,
                              int ng, const PrimeConst* __restrict__ pc, int npts, int32_t* __restrict__ deg,
                              uint32_t* gbuf) {
  extern __shared__ uint32_t sm[];
  const int unit = blockIdx.x, k = unit / npts, j = unit - k * npts;
  const Mod M = load_mod_u(pc[k]);
  const int w = (nf > ng ? nf : ng) + 2;
  uint32_t* X = cta_buffers<GB>(sm, gbuf, 2 * static_cast<size_t>(w));
  uint32_t* Y = X + w;
  const int32_t *offf = dir, *lenf = dir + nf + 1, *offg = dir + 2 * (nf + 1), *leng = offg + ng + 1;
  // a_j: distinct small integers 2, 3, ... in Montgomery form
  const uint32_t a = mmul(static_cast<uint32_t>(j + 2), M.r2, M);
  const uint32_t* t = tab + static_cast<size_t>(k) * S;
  for (int r = threadIdx.x; r <= nf + ng + 1; r += blockDim.x) {
    const bool isf = r <= nf;
    const int row = isf ? r : r - nf - 1;
    const int off = isf ? offf[row] : offg[row], len = isf ? lenf[row] : leng[row];
    uint32_t acc = 0u;
    for (int i = len - 1; i >= 0; --i) acc = madd(mmul(acc, a, M), t[off + i], M.p);
    (isf ? X : Y)[row] = acc;
  }
  __syncthreads();
  const bool lc_ok = X[nf] != 0u || Y[ng] != 0u;
  const int dx = blk_trim(X, nf), dy = blk_trim(Y, ng);
  int d = -1;
  if (dx >= 0 && dy >= 0) d = blk_gcd(X, dx, Y, dy, M);
  if (threadIdx.x == 0) deg[unit] = lc_ok ? d : -1;
}

// ---------------------------------------------------------------------------
// Modular bivariate gcd (Brown), ctg_gcd_bivariate when the primitive parts share a factor.
// CTA per unit (prime k, point a = off_k + j): the y-rows of A, B and gamma (gcd of the
// leading y-coefficients, slot run `gam`) are evaluated at a by Horner; then
//   g = monic gcd(A(a, y), B(a, y)),  h = gamma(a) g,  u = A(a, y) / g,  w = B(a, y) / g
// are stored (plain) as h (dg+1) | u (na-dg+1) | w (nb-dg+1) at out[k][j][...], pitch words.
// deg[k][j] = dg, or -2 when gamma(a) = 0 mod p (then A(a, y) or B(a, y) may drop degree).
// ---------------------------------------------------------------------------
template <bool GB>
__global__ void __launch_bounds__(128) k_bigcd_images(const uint32_t* __restrict__ tab, int S,
                                                      const int32_t* __restrict__ dir, int na, int nb, int gam_off,
                                                      int gam_len, const PrimeConst* __restrict__ pc,
                                                      const uint32_t* __restrict__ offs, int npts,
                                                      int32_t* __restrict__ deg, uint32_t* __restrict__ out,
                                                      int pitch, uint32_t* gbuf) {
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t s_gam;
  const int unit = blockIdx.x, k = unit / npts, j = unit - k * npts;
  const Mod M = load_mod_u(pc[k]);
  const int cap = (na > nb ? na : nb) + 2;
  uint32_t* base = cta_buffers<GB>(sm, gbuf, 5 * static_cast<size_t>(cap));
  uint32_t *A = base, *Bv = base + cap, *X = base + 2 * cap, *Y = base + 3 * cap, *Q = base + 4 * cap;
  const int32_t *offa = dir, *lena = dir + na + 1, *offb = dir + 2 * (na + 1), *lenb = offb + nb + 1;
  uint32_t av = offs[k] + static_cast<uint32_t>(j);
  if (av >= M.p) av -= M.p;
  const uint32_t a = mmul(av, M.r2, M);
  const uint32_t* t = tab + static_cast<size_t>(k) * S;
  for (int r = threadIdx.x; r <= na + nb + 2; r += blockDim.x) {
    const int which = r <= na ? 0 : (r <= na + nb + 1 ? 1 : 2);
    const int row = which == 0 ? r : r - na - 1;
    const int off = which == 0 ? offa[row] : (which == 1 ? offb[row] : gam_off);
    const int len = which == 0 ? lena[row] : (which == 1 ? lenb[row] : gam_len);
    uint32_t acc = 0u;
    for (int i = len - 1; i >= 0; --i) acc = madd(mmul(acc, a, M), t[off + i], M.p);
    if (which == 0) {
      A[row] = X[row] = acc;
    } else if (which == 1) {
      Bv[row] = Y[row] = acc;
    } else {
      s_gam = acc;
    }
  }
  __syncthreads();
  int32_t* dk = deg + static_cast<size_t>(k) * npts + j;
  if (s_gam == 0u || A[na] == 0u || Bv[nb] == 0u) {
    if (threadIdx.x == 0) *dk = -2;
    return;
  }
  const uint32_t gam = s_gam;
  const int dg = blk_gcd(X, na, Y, nb, M);
  uint32_t* o = out + (static_cast<size_t>(k) * npts + j) * pitch;
  for (int i = threadIdx.x; i <= dg; i += blockDim.x) o[i] = from_mont(mmul(X[i], gam, M), M);
  const int du = blk_divexact_monic(A, na, X, dg, Q, M);
  blk_store_plain(o + dg + 1, Q, du, M);
  __syncthreads();
  const int dw = blk_divexact_monic(Bv, nb, X, dg, Q, M);
  blk_store_plain(o + dg + 1 + du + 1, Q, dw, M);
  if (threadIdx.x == 0) *dk = dg;
}

// Newton interpolation in x on the consecutive points a_j = off_k + j (j < N): for row r
// (prime idx[r]) and column c, the values src[idx[r]][j][c] (plain, pitch src_pitch) become
// the monomial coefficients dst[idx[r]][t][c] (t < N, plain).  CTA = (32 columns, one row);
// column c of the CTA lives in shared memory v[j * 32 + lane]: divided differences with
// spacing j - i (inverses 1..N-1 from a per-CTA table), then Horner with (x - a_i) in place,
// the growing coefficient array stored reversed in the slots the consumed values free up.
constexpr int kNewtonCols = 32;
template <bool GB>
__global__ void __launch_bounds__(kNewtonCols) k_newton_interp(const uint32_t* __restrict__ src, int src_pitch,
                                                               const int32_t* __restrict__ idx,
                                                               const PrimeConst* __restrict__ pc,
                                                               const uint32_t* __restrict__ offs, int N, int cols,
                                                               uint32_t* __restrict__ dst, uint32_t* gbuf) {
  extern __shared__ uint32_t smem_[];
  // shared memory, or this CTA's slice of the global scratch (N x 33 words beyond ~227 KB)
  uint32_t* sm = smem_;
  if constexpr (GB) sm = gbuf + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * N * (kNewtonCols + 1);
  const int k = idx[blockIdx.y];
  const Mod M = load_mod_u(pc[k]);
  const int lane = threadIdx.x, c = blockIdx.x * kNewtonCols + lane;
  uint32_t* inv = sm;              // inv[i] = 1 / i (Montgomery), i < N
  uint32_t* v = sm + N;            // [N][32]
  for (int i = lane + 1; i < N; i += kNewtonCols) inv[i] = minv(mmul(static_cast<uint32_t>(i), M.r2, M), M);
  const uint32_t* s = src + static_cast<size_t>(k) * N * src_pitch;
  for (int j = 0; j < N; ++j) v[j * kNewtonCols + lane] = c < cols ? mmul(s[static_cast<size_t>(j) * src_pitch + c], M.r2, M) : 0u;
  __syncthreads();
  // divided differences: v[i] <- (v[i] - v[i-1]) / (a_i - a_{i-d}) = ... / d
  for (int d = 1; d < N; ++d) {
    const uint32_t id = inv[d];
    for (int i = N - 1; i >= d; --i) {
      const uint32_t x1 = v[i * kNewtonCols + lane], x0 = v[(i - 1) * kNewtonCols + lane];
      v[i * kNewtonCols + lane] = mmul(msub(x1, x0, M.p), id, M);
    }
  }
  // Horner: cf(x) = v_{N-1}; cf <- cf (x - a_i) + v_i for i = N-2..0.  cf[t] at slot N-1-t.
  uint32_t ob = offs[k];
  for (int i = N - 2; i >= 0; --i) {
    uint32_t ai = ob + static_cast<uint32_t>(i);
    if (ai >= M.p) ai -= M.p;
    const uint32_t nai = mneg(mmul(ai, M.r2, M), M.p);
    const uint32_t vi = v[i * kNewtonCols + lane];
    const int dgn = N - 1 - i;  // new degree
    // newcf[t] = cf[t-1] - a_i cf[t]  (cf[dgn] = 0), t = dgn..1;  newcf[0] = v_i - a_i cf[0]
    uint32_t hi = 0u;  // cf[t] for the t being written (cf[dgn] = 0)
    for (int t = dgn; t >= 1; --t) {
      const uint32_t lo = v[(N - 1 - (t - 1)) * kNewtonCols + lane];  // cf[t-1]
      v[(N - 1 - t) * kNewtonCols + lane] = mmul2(hi, nai, lo, M.one, M);
      hi = lo;
    }
    v[(N - 1) * kNewtonCols + lane] = madd(mmul(hi, nai, M), vi, M.p);
  }
  if (c < cols) {
    uint32_t* o = dst + static_cast<size_t>(k) * N * cols;
    for (int t = 0; t < N; ++t) o[static_cast<size_t>(t) * cols + c] = from_mont(v[(N - 1 - t) * kNewtonCols + lane], M);
  }
}

}  // namespace

size_t modyun_smem(int n) { return static_cast<size_t>(8) * (n + 2) * 4; }
size_t modgcd_smem(int na, int nb) { return static_cast<size_t>(6) * ((na > nb ? na : nb) + 2) * 4; }
size_t gcd_degree_smem(int na, int nb) { return static_cast<size_t>(4) * ((na > nb ? na : nb) + 2) * 4; }
size_t sqf_probe_smem(int max_deg) { return static_cast<size_t>(4) * (max_deg + 2) * 4; }
size_t bigcd_probe_smem(int nf, int ng) { return static_cast<size_t>(2) * ((nf > ng ? nf : ng) + 2) * 4; }
size_t newton_smem(int N) { return static_cast<size_t>(N) * (kNewtonCols + 1) * 4; }

namespace {
// Launch with `smem` bytes of shared memory, or with none and the buffers in gbuf when it
// exceeds the per-CTA budget (the caller allocated gbuf from uni_gbuf_bytes).
template <class K>
size_t smem_or_global(K kern, size_t smem, uint32_t* gbuf) {
  if (smem > kUniSmemMax) {
    if (!gbuf) return SIZE_MAX;
    return 0;
  }
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return smem;
}
}  // namespace

// CTA size of the per-prime kernels (CTG_UNI_THREADS overrides, for A/B).  k_modyun at n = 870
// (3 probe primes): 256 threads 277 us, 512 threads 285 us.
int uni_threads(int n) {
  static const int forced = std::getenv("CTG_UNI_THREADS") ? std::atoi(std::getenv("CTG_UNI_THREADS")) : 0;
  if (forced == 128 || forced == 256 || forced == 512) return forced;
  return 256;  // 512 measured slower at n = 870 (285 vs 277 us)
}

int launch_sqf_probe(const uint32_t* tab, int S, const int32_t* off, const int32_t* degs, int nprob, int nk,
                     const PrimeConst* pc, int max_deg, int32_t* out, uint32_t* gbuf, cudaStream_t st, int plain,
                     bool small, int single_deg) {
  if (nprob == 0) return 0;
  const int cap = max_deg + 2;
  const size_t smem = smem_or_global(small ? k_sqf_probe<false, true> : k_sqf_probe<false, false>,
                                     sqf_probe_smem(max_deg), gbuf);
  if (smem == SIZE_MAX) return -1;
  const int g = nprob * nk;
  if (smem) {
    if (small)
      k_sqf_probe<false, true><<<g, 256, smem, st>>>(tab, S, off, degs, nk, pc, cap, out, nullptr, plain, single_deg);
    else
      k_sqf_probe<false, false><<<g, 256, smem, st>>>(tab, S, off, degs, nk, pc, cap, out, nullptr, plain, single_deg);
  } else {
    if (small)
      k_sqf_probe<true, true><<<g, 256, 0, st>>>(tab, S, off, degs, nk, pc, cap, out, gbuf, plain, single_deg);
    else
      k_sqf_probe<true, false><<<g, 256, 0, st>>>(tab, S, off, degs, nk, pc, cap, out, gbuf, plain, single_deg);
  }
  return 1;
}

int launch_gcd_degree(const uint32_t* a, int na, const uint32_t* b, int nb, const PrimeConst* pc, int method,
                      int32_t* out, uint32_t* gbuf, cudaStream_t st, unsigned long long* prof) {
  const int cap = (na > nb ? na : nb) + 2;
  const size_t smem = smem_or_global(k_gcd_degree<false>, gcd_degree_smem(na, nb), gbuf);
  if (smem == SIZE_MAX) return -1;
  if (smem)
    k_gcd_degree<false><<<1, 256, smem, st>>>(a, na, b, nb, pc, cap, method, out, nullptr, prof);
  else
    k_gcd_degree<true><<<1, 256, 0, st>>>(a, na, b, nb, pc, cap, method, out, gbuf, prof);
  return 1;
}

size_t uni_gbuf_bytes(size_t smem, size_t ctas) { return smem > kUniSmemMax ? smem * ctas : 0; }

int launch_modyun(const uint32_t* tab, int n, const PrimeConst* pc, int nk, int32_t* deg, uint32_t* fac,
                  uint32_t* sqf, uint32_t* gbuf, cudaStream_t st) {
  const size_t smem = smem_or_global(k_modyun<false>, modyun_smem(n), gbuf);
  if (smem == SIZE_MAX) return -1;
  if (smem)
    k_modyun<false><<<nk, uni_threads(n), smem, st>>>(tab, n, pc, deg, fac, sqf, nullptr);
  else
    k_modyun<true><<<nk, uni_threads(n), 0, st>>>(tab, n, pc, deg, fac, sqf, gbuf);
  return 1;
}

int launch_modgcd(const uint32_t* tabA, int na, const uint32_t* tabB, int nb, int tab_pitch, const PrimeConst* pc,
                  int nk, int32_t* deg, uint32_t* out, int pitch, uint32_t* gbuf, cudaStream_t st,
                  const uint32_t* staged_limbs, const int8_t* staged_sign, int Lw, const uint32_t* rpow) {
  const size_t smem = smem_or_global(k_modgcd<false>, modgcd_smem(na, nb), gbuf);
  if (smem == SIZE_MAX) return -1;
  GcdStaged sg;
  if (staged_limbs) {
    if (Lw < 1 || Lw > kRedL || !staged_sign || !rpow) return -1;
    sg.limbs = staged_limbs;
    sg.sign = staged_sign;
    sg.Lw = Lw;
    sg.rpow = rpow;
  }
  if (smem)
    k_modgcd<false><<<nk, uni_threads(std::max(na, nb)), smem, st>>>(tabA, na, tabB, nb, tab_pitch, pc, deg, out, pitch,
                                                                     nullptr, sg);
  else
    k_modgcd<true><<<nk, uni_threads(std::max(na, nb)), 0, st>>>(tabA, na, tabB, nb, tab_pitch, pc, deg, out, pitch, gbuf,
                                                                 sg);
  return 1;
}

int launch_bigcd_probe(const uint32_t* tab, int S, const int32_t* dir, int nf, int ng, const PrimeConst* pc,
                       int nk, int npts, int32_t* deg, uint32_t* gbuf, cudaStream_t st) {
  const size_t smem = smem_or_global(k_bigcd_probe<false>, bigcd_probe_smem(nf, ng), gbuf);
  if (smem == SIZE_MAX) return -1;
  if (smem)
    k_bigcd_probe<false><<<nk * npts, 128, smem, st>>>(tab, S, dir, nf, ng, pc, npts, deg, nullptr);
  else
    k_bigcd_probe<true><<<nk * npts, 128, 0, st>>>(tab, S, dir, nf, ng, pc, npts, deg, gbuf);
  return 1;
}

int launch_bigcd_images(const uint32_t* tab, int S, const int32_t* dir, int na, int nb, int gam_off, int gam_len,
                        const PrimeConst* pc, const uint32_t* offs, int nk, int npts, int32_t* deg, uint32_t* out,
                        int pitch, uint32_t* gbuf, cudaStream_t st) {
  const size_t smem = smem_or_global(k_bigcd_images<false>, modgcd_smem(na, nb), gbuf);
  if (smem == SIZE_MAX) return -1;
  if (smem)
    k_bigcd_images<false><<<nk * npts, 128, smem, st>>>(tab, S, dir, na, nb, gam_off, gam_len, pc, offs, npts, deg,
                                                        out, pitch, nullptr);
  else
    k_bigcd_images<true><<<nk * npts, 128, 0, st>>>(tab, S, dir, na, nb, gam_off, gam_len, pc, offs, npts, deg, out,
                                                       pitch, gbuf);
  return 1;
}

int launch_newton_interp(const uint32_t* src, int src_pitch, const int32_t* idx, int rows, const PrimeConst* pc,
                         const uint32_t* offs, int N, int cols, uint32_t* dst, uint32_t* gbuf, int gbuf_rows,
                         cudaStream_t st) {
  if (rows == 0 || cols == 0) return 0;
  const size_t smem = smem_or_global(k_newton_interp<false>, newton_smem(N), gbuf);
  if (smem == SIZE_MAX || (!smem && gbuf_rows < 1)) return -1;
  const int step = smem ? rows : gbuf_rows;  // global scratch: row chunks reuse the same slices
  int launches = 0;
  for (int r0 = 0; r0 < rows; r0 += step) {
    dim3 grid((cols + kNewtonCols - 1) / kNewtonCols, std::min(step, rows - r0));
    if (smem)
      k_newton_interp<false><<<grid, kNewtonCols, smem, st>>>(src, src_pitch, idx + r0, pc, offs, N, cols, dst, nullptr);
    else
      k_newton_interp<true><<<grid, kNewtonCols, 0, st>>>(src, src_pitch, idx + r0, pc, offs, N, cols, dst, gbuf);
    ++launches;
  }
  return launches;
}

int launch_gather_scale(const uint32_t* src, int src_pitch, const int32_t* idx, int rows, int cols,
                        const int32_t* seg_end, int nseg, const uint32_t* scale, const PrimeConst* pc_dst,
                        uint32_t* dst, cudaStream_t st) {
  if (rows == 0 || cols == 0) return 0;
  dim3 grid((cols + 127) / 128, rows);
  k_gather_scale<<<grid, 128, 0, st>>>(src, src_pitch, idx, rows, cols, seg_end, nseg, scale, pc_dst, dst);
  return 1;
}

}  // namespace ctg
