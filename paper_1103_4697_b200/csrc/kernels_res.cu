// sm_100a kernels of the multi-modular resultant (SURVEY.md §2 kernel table).  Every
// kernel processes a batch of B same-shape curves (blockIdx.z = curve).
//
//   K1 k_reduce          multiprecision coefficients -> residues mod each prime (Montgomery)
//   K2 k_eval_ntt<LP>    y-coefficient rows evaluated at x = omega^i, i < N: coset
//                        decomposition into LP-point NTTs in registers (k_eval_horner otherwise)
//   K3 k_modres_fast<n>  (modres_fast.cuh) division-free Euclid per (prime, point) in registers
//   K3' k_modres_general exact formal-degree resultant (degree drops, zero pivots, any shape)
//                        for the units the fast path flags, or for shapes without a template
//   K4 k_interp          inverse mixed-radix NTT (N = r 2^a) per prime: values -> coefficients
//   K5 k_crt_prep / k_crt_gemm / k_crt_carry   fixed-point CRT  c = sum_k y_k (M/p_k) - t M
//
// The reference computes the same R = res_y(p, q) by a subresultant PRS over Z[x]
// (/root/reference/proj/src/elim.cpp:95-136); R is unique, so the modular images of the
// Sylvester determinant at every (prime, point) determine it bit-exactly.
#include <cuda_runtime.h>

#include <stdexcept>

#include <cudaTypedefs.h>

#include <type_traits>

#include "crt_gemm_tma.cuh"

#include <algorithm>
#include <cstdlib>

#include "internal.hpp"
#include "res_common.cuh"

namespace ctg {

namespace {

// ---------------------------------------------------------------------------
// K1: reduce multiprecision slots modulo the primes.  Limbs are limb-major per curve
// ([B][L][S]) so consecutive threads (slots) read consecutive words.
// ---------------------------------------------------------------------------
// K1: every coefficient (L little-endian 32-bit limbs, sign) modulo every prime, Montgomery
// form.  One thread per (prime, slot) over a flat index (no idle lanes when S is small):
//   value R = sum_l limb_l 2^(32 l) R = sum_l mmul(limb_l, R^(l+2))
// with the weights from a per-prime table: independent products (no Horner chain), each
// REDC exact for any 32-bit limb (limb * w < 2^32 p), summed with a conditional subtract.
template <bool CM>
__global__ void __launch_bounds__(128) k_reduce(const uint32_t* __restrict__ limbs, const int8_t* __restrict__ sign,
                                                int S, int L, const PrimeConst* __restrict__ pc,
                                                const uint32_t* __restrict__ rpow, int k0, int nk,
                                                uint32_t* __restrict__ tab, size_t tab_bstride) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (idx >= static_cast<long long>(nk) * S) return;
  const int kl = static_cast<int>(idx / S), s = static_cast<int>(idx - static_cast<long long>(kl) * S);
  const int k = k0 + kl;
  const Mod M = load_mod(pc[k]);
  // limb l of slot s: limb-major [B][L][S] (plans, CM = false) or coefficient-major [B][S][L]
  // (univariate, CM = true)
  const size_t ls = CM ? 1 : static_cast<size_t>(S);
  const uint32_t* lb = limbs + static_cast<size_t>(b) * L * S + (CM ? static_cast<size_t>(s) * L : s);
  const uint32_t* w = rpow + static_cast<size_t>(k) * kRedL;
  uint32_t acc = 0;
  const int Lt = L < kRedL ? L : kRedL;
#pragma unroll 4
  for (int l = 0; l < Lt; ++l) acc = madd(acc, mmul(lb[l * ls], __ldg(&w[l]), M), M.p);
  if (L > kRedL) {  // very long coefficients: extend the weights by R per limb
    uint32_t wl = __ldg(&w[kRedL - 1]);
    for (int l = kRedL; l < L; ++l) {
      wl = mmul(wl, M.r2, M);
      acc = madd(acc, mmul(lb[l * ls], wl, M), M.p);
    }
  }
  if (sign[static_cast<size_t>(b) * S + s] < 0) acc = mneg(acc, M.p);
  tab[b * tab_bstride + static_cast<size_t>(k) * S + s] = acc;
}

// K1 for few (prime, slot) pairs with long coefficients (the Yun / gcd probes on 3 primes, a
// single big-coefficient curve): a WARP per pair, lane l summing the limbs l, l + 32, ... (the
// weight of limb l + 32 is the weight of limb l times R^32: rpow[31] = R^33 in the table's
// convention), then a shuffle reduction -- 32 short chains instead of one long one.
__global__ void __launch_bounds__(128) k_reduce_warp(const uint32_t* __restrict__ limbs,
                                                     const int8_t* __restrict__ sign, int S, int L,
                                                     const PrimeConst* __restrict__ pc,
                                                     const uint32_t* __restrict__ rpow, int k0, int nk,
                                                     uint32_t* __restrict__ tab, size_t tab_bstride, int coef_major) {
  const long long pair = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, b = blockIdx.y;
  if (pair >= static_cast<long long>(nk) * S) return;  // whole warps
  const int kl = static_cast<int>(pair / S), s_ = static_cast<int>(pair - static_cast<long long>(kl) * S);
  const int k = k0 + kl;
  const Mod M = load_mod(pc[k]);
  const size_t ls = coef_major ? 1 : static_cast<size_t>(S);  // coefficient-major: lanes read 128 B
  const uint32_t* lb = limbs + static_cast<size_t>(b) * L * S + (coef_major ? static_cast<size_t>(s_) * L : s_);
  const uint32_t* w = rpow + static_cast<size_t>(k) * kRedL;
  const uint32_t r33 = __ldg(&w[31]);
  uint32_t acc = 0, wl = __ldg(&w[lane]);
  for (int l = lane; l < L; l += 32) {
    if (l >= 32) wl = l < kRedL ? __ldg(&w[l]) : mmul(wl, r33, M);
    acc = madd(acc, mmul(lb[l * ls], wl, M), M.p);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc = madd(acc, __shfl_xor_sync(0xffffffffu, acc, off), M.p);
  if (lane == 0) {
    if (sign[static_cast<size_t>(b) * S + s_] < 0) acc = mneg(acc, M.p);
    tab[b * tab_bstride + static_cast<size_t>(k) * S + s_] = acc;
  }
}

// ---------------------------------------------------------------------------
// K2: evaluate every y-coefficient row at all N points omega^i (Montgomery form).
// Row r < n+1 is p_r(x); rows n+1.. are q_r(x) when q is not dp/dy.
//
// Coset decomposition: with LP = 2^b >= row length, LP | N and K = N / LP,
//   V[u + K v] = sum_t (c_t omega^{t u}) (omega^K)^{t v} = NTT_LP(c_t omega^{t u})[v],
// so each thread (prime, row, u) twists <= LP coefficients and runs one LP-point NTT
// in registers: N (1 + log2(LP)/2) mulmods per row instead of N * len for Horner.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void row_slots(const ResParams& P, int r, int& off, int& len) {
  const int nq = P.n + 1;
  if (r < nq) {
    off = P.dir[r];
    len = P.dir[nq + r];
  } else {
    const int j = r - nq, base = 2 * nq;
    off = P.dir[base + j];
    len = P.dir[base + P.m + 1 + j];
  }
}

__device__ __forceinline__ uint32_t* vals_row(const ResParams& P, int b, int kl, int r) {
  return P.vals + ((static_cast<size_t>(b) * P.nk + kl) * P.nrows + r) * P.N;
}

template <int LP, int LG>
__global__ void __launch_bounds__(128) k_eval_ntt(ResParams P, int K) {
  __shared__ uint32_t tw[LP / 2];
  const int kl = blockIdx.y, b = blockIdx.z;
  const int k = P.k0 + kl;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const PrimeConst pcv = P.pc[k];
  const Mod M = load_mod(pcv);
  const uint32_t* twr = P.twinv + static_cast<size_t>(k) * P.N;
  load_coset_twiddles<LP>(tw, twr, P.N, K, M);
  __syncthreads();
  if (idx >= P.nrows * K) return;
  const int r = idx / K, u = idx - r * K;
  int off, len;
  row_slots(P, r, off, len);
  const uint32_t* tab = P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S + off;
  uint32_t a[LP];
  coset_ntt<LP, LG>(tab, len, u ? __ldg(&twr[P.N - u]) : M.one, tw, M, a);
  uint32_t* out = vals_row(P, b, kl, r) + u;
#pragma unroll
  for (int j = 0; j < LP; ++j) out[static_cast<size_t>(K) * bitrev_c(j, LG)] = a[j];
}

// Fallback K2 (any row length / N): thread per (prime, row, point), Horner.
__global__ void __launch_bounds__(128) k_eval_horner(ResParams P) {
  const int r = blockIdx.y % P.nrows, kl = blockIdx.y / P.nrows, b = blockIdx.z;
  const int k = P.k0 + kl;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.N) return;
  const PrimeConst pcv = P.pc[k];
  const Mod M = load_mod(pcv);
  int off, len;
  row_slots(P, r, off, len);
  const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
  vals_row(P, b, kl, r)[i] = horner(P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S, off, len, x, M);
}

template <int LP, int LG>
void launch_eval_ntt(const ResParams& rp, cudaStream_t st) {
  const int K = rp.N / LP;
  dim3 grid((rp.nrows * K + 127) / 128, rp.nk, rp.B);
  k_eval_ntt<LP, LG><<<grid, 128, 0, st>>>(rp, K);
}

int launch_eval(const ResParams& rp, cudaStream_t st) {
  int lp = 4, lg = 2;
  while (lp < rp.maxlen) {
    lp <<= 1;
    ++lg;
  }
  if ((rp.N % lp) == 0 && lp <= 64) {
    switch (lp) {
      case 4: launch_eval_ntt<4, 2>(rp, st); return 1;
      case 8: launch_eval_ntt<8, 3>(rp, st); return 1;
      case 16: launch_eval_ntt<16, 4>(rp, st); return 1;
      case 32: launch_eval_ntt<32, 5>(rp, st); return 1;
      case 64: launch_eval_ntt<64, 6>(rp, st); return 1;
      default: break;
    }
  }
  dim3 grid((rp.N + 127) / 128, rp.nrows * rp.nk, rp.B);
  k_eval_horner<<<grid, 128, 0, st>>>(rp);
  return 1;
}

// Exact resultant of univariate images with FORMAL degrees na, nb (Montgomery
// form).  Handles leading coefficients that vanish mod p, zero polynomials and
// constant operands with the Sylvester-determinant conventions:
//   res_{n,0}(A, c) = c^n, res_{0,m}(c, B) = c^m, res_{0,0} = 1;
//   A's degree drops n -> n':  res = (-1)^{(n-n')m} lc(B)^{n-n'} res_{n',m}
//   B's degree drops m -> m':  res = lc(A)^{m-m'} res_{n,m'}
//   both drop / a zero operand (n, m >= 1): 0
//   A = Q B + R:  res_{n,m}(A,B) = (-1)^{nm} lc(B)^{n-m+1} res_{m,m-1}(B, R)
__device__ uint32_t res_general(uint32_t* A, int na, uint32_t* B, int nb, const Mod& M) {
  uint32_t acc = M.one;
  while (true) {
    if (na == 0) return mmul(acc, mpow(A[0], static_cast<uint64_t>(nb), M), M);
    if (nb == 0) return mmul(acc, mpow(B[0], static_cast<uint64_t>(na), M), M);
    int da = na;
    while (da >= 0 && A[da] == 0u) --da;
    int db = nb;
    while (db >= 0 && B[db] == 0u) --db;
    if (da < 0 || db < 0) return 0u;
    if (da < na && db < nb) return 0u;
    if (da < na) {
      const int e = na - da;
      acc = mmul(acc, mpow(B[nb], static_cast<uint64_t>(e), M), M);
      if ((e & 1) && (nb & 1)) acc = mneg(acc, M.p);
      na = da;
      continue;
    }
    if (db < nb) {
      acc = mmul(acc, mpow(A[na], static_cast<uint64_t>(nb - db), M), M);
      nb = db;
      continue;
    }
    if (na < nb) {
      uint32_t* t = A;
      A = B;
      B = t;
      const int tn = na;
      na = nb;
      nb = tn;
      if ((na & 1) && (nb & 1)) acc = mneg(acc, M.p);
    }
    const uint32_t inv = minv(B[nb], M);
    for (int i = na; i >= nb; --i) {
      const uint32_t q = mmul(A[i], inv, M);
      if (q)
        for (int j = 0; j < nb; ++j) A[i - nb + j] = msub(A[i - nb + j], mmul(q, B[j], M), M.p);
      A[i] = 0u;
    }
    acc = mmul(acc, mpow(B[nb], static_cast<uint64_t>(na - nb + 1), M), M);
    if ((na & 1) && (nb & 1)) acc = mneg(acc, M.p);
    uint32_t* t = A;
    A = B;
    B = t;
    na = nb;
    nb = nb - 1;
  }
}

// General path: one thread per unit, either all units (use_list = 0) or the
// degenerate units listed by the fast path.  Unit id = (b * nk + kl) * N + i.
// When the fast path flagged more units than the list holds (curves whose remainder sequence
// drops degree at every point, e.g. y^n + g(x), n >= 3), the list is abandoned and every unit
// of the launch is scanned: the ones the fast kernel left at kSentinel are recomputed.
__global__ void __launch_bounds__(128) k_modres_general(ResParams P, int use_list, uint32_t total_units) {
  const uint32_t flagged = use_list ? P.counters[0] : 0u;
  const bool scan = use_list && flagged > P.flag_cap;
  const uint32_t all = static_cast<uint32_t>(P.B) * static_cast<uint32_t>(P.nk) * static_cast<uint32_t>(P.N);
  const uint32_t count = scan ? all : (use_list ? flagged : total_units);
  const int nq = P.n + 1;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < count; u += gridDim.x * blockDim.x) {
    const uint32_t unit = (use_list && !scan) ? P.flag_list[u] : u;
    const uint32_t bk = unit / P.N;
    const int i = static_cast<int>(unit % P.N);
    const int kl = static_cast<int>(bk % P.nk), b = static_cast<int>(bk / P.nk);
    if (scan && P.rows[b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch + i] != kSentinel) continue;
    const int k = P.k0 + kl;
    const PrimeConst pcv = P.pc[k];
    const Mod M = load_mod(pcv);
    const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
    const uint32_t* tab = P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S;
    uint32_t bufA[kThreadGeneralMax + 1], bufB[kThreadGeneralMax + 1];
    for (int j = 0; j <= P.n; ++j) bufA[j] = horner(tab, P.dir[j], P.dir[nq + j], x, M);
    if (P.deriv) {
      uint32_t c = M.one;
      for (int j = 0; j <= P.m; ++j) {
        bufB[j] = mmul(bufA[j + 1], c, M);
        c = madd(c, M.one, M.p);
      }
    } else {
      const int base = 2 * nq;
      for (int j = 0; j <= P.m; ++j) bufB[j] = horner(tab, P.dir[base + j], P.dir[base + P.m + 1 + j], x, M);
    }
    P.rows[b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch + i] = res_general(bufA, P.n, bufB, P.m, M);
  }
}

// ---------------------------------------------------------------------------
// K3'' k_modres_warp: the same formal-degree resultant (res_general's conventions) with one
// WARP per unit, for deg_y > kThreadGeneralMax (any size: no per-thread arrays).  A and B live
// in shared memory (kWarpsGeneral warps per CTA, 2 (n + 1) words each) or, beyond the
// shared-memory budget, in this warp's slice of the global scratch P.gwarp.  Every scalar
// (degrees, leading coefficients, quotients) is computed lane-uniformly; coefficient updates
// are spread over the lanes, with __syncwarp between dependent passes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int warp_trim(const uint32_t* X, int d, int lane) {
  for (int base = d; base >= 0; base -= 32) {
    const int idx = base - lane;
    const unsigned nz = __ballot_sync(0xffffffffu, idx >= 0 && X[idx] != 0u);
    if (nz) return base - (__ffs(nz) - 1);
  }
  return -1;
}

__device__ uint32_t warp_res_general(uint32_t* A, int na, uint32_t* B, int nb, const Mod& M, int lane) {
  uint32_t acc = M.one;
  while (true) {
    __syncwarp();
    if (na == 0) return mmul(acc, mpow(A[0], static_cast<uint64_t>(nb), M), M);
    if (nb == 0) return mmul(acc, mpow(B[0], static_cast<uint64_t>(na), M), M);
    const int da = warp_trim(A, na, lane), db = warp_trim(B, nb, lane);
    if (da < 0 || db < 0) return 0u;
    if (da < na && db < nb) return 0u;
    if (da < na) {
      const int e = na - da;
      acc = mmul(acc, mpow(B[nb], static_cast<uint64_t>(e), M), M);
      if ((e & 1) && (nb & 1)) acc = mneg(acc, M.p);
      na = da;
      continue;
    }
    if (db < nb) {
      acc = mmul(acc, mpow(A[na], static_cast<uint64_t>(nb - db), M), M);
      nb = db;
      continue;
    }
    if (na < nb) {
      uint32_t* t = A;
      A = B;
      B = t;
      const int tn = na;
      na = nb;
      nb = tn;
      if ((na & 1) && (nb & 1)) acc = mneg(acc, M.p);
    }
    const uint32_t inv = minv(B[nb], M);
    for (int i = na; i >= nb; --i) {
      const uint32_t q = mmul(A[i], inv, M);
      if (q) {
        const uint32_t nq = mneg(q, M.p);
        for (int j = lane; j < nb; j += 32) A[i - nb + j] = mmul2(M.one, A[i - nb + j], nq, B[j], M);
      }
      __syncwarp();
      if (lane == 0) A[i] = 0u;
      __syncwarp();
    }
    acc = mmul(acc, mpow(B[nb], static_cast<uint64_t>(na - nb + 1), M), M);
    if ((na & 1) && (nb & 1)) acc = mneg(acc, M.p);
    uint32_t* t = A;
    A = B;
    B = t;
    na = nb;
    nb = nb - 1;
  }
}

// K3's fused division-free Euclid (fast_euclid, modres_fast.cuh) with the coefficients spread
// over the lanes of a warp (A, B in shared memory): r'_i = b_k^2 a_i - b_k a_{k+1} b_{i-1} - A1_k b_i,
// one three-product reduction per coefficient per step, no inversion until the end
// (res = r'_0 / (prod b_k^{k-1})^2).  A (deg n) and B (deg n - 1) are consumed.  flag != 0: a
// leading coefficient vanished (degree drop) -- the caller recomputes with warp_res_general.
__device__ uint32_t warp_fast_euclid(uint32_t* A, uint32_t* B, int n, const Mod& M, int lane, uint32_t& flag) {
  __syncwarp();
  flag = (A[n] == 0u) | (B[n - 1] == 0u);
  uint32_t U = M.one, E = M.one;
  for (int kk = n - 1; kk >= 1 && !flag; --kk) {
    const uint32_t bk = B[kk];
    const uint32_t na = mneg(A[kk + 1], M.p);
    const uint32_t c1 = mmul(bk, bk, M);
    const uint32_t c2 = mmul(bk, na, M);
    const uint32_t c3 = mneg(mmul2(bk, A[kk], na, B[kk - 1], M), M.p);
    __syncwarp();  // every lane has read the step's leading coefficients
    for (int t = lane; t < kk; t += 32) A[t] = t ? mmul3(c1, A[t], c2, B[t - 1], c3, B[t], M) : mmul2(c1, A[0], c3, B[0], M);
    __syncwarp();
    flag |= (A[kk - 1] == 0u);
    U = mmul(U, bk, M);
    if (kk >= 2) E = mmul(E, U, M);
    uint32_t* t = A;  // (A, B) <- (B, r')
    A = B;
    B = t;
  }
  if (flag) return 0u;
  return mmul(B[0], minv(mmul(E, E, M), M), M);
}

// ---------------------------------------------------------------------------
// K3 for 40 < deg_y <= 127 with the derivative / n, n-1 shape: FOUR units per warp, 8 lanes per
// unit, each lane holding C consecutive coefficients of A and B in registers (n + 1 <= 8 C).
// Same fused division-free step as fast_euclid; the two new leading remainder coefficients of
// a step come from their owner lanes by shuffle (the other two step inputs carry over from the
// previous step), y_{i-1} across a lane boundary by shfl_up.  A unit whose leading coefficient
// vanishes mod p (degree drop) is marked kSentinel and recomputed by k_modres_warp's exact
// path.  (k_modres_warp alone -- one unit per warp, coefficients in shared memory -- ran deg_y
// 41 / 50 / 64 at 1.0e8 / 8.7e7 / 6.9e7 units/s.)
// ---------------------------------------------------------------------------
template <int C>
__global__ void __launch_bounds__(128) k_modres_mw(ResParams P, uint32_t total_units) {
  constexpr int G = 8;  // lanes per unit
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gbase = lane & ~(G - 1);
  const int nq = P.n + 1, n = P.n;
  const uint32_t units_per_block = (blockDim.x / G);
  for (uint32_t u0 = blockIdx.x * units_per_block; u0 < total_units; u0 += gridDim.x * units_per_block) {
    const uint32_t unit = u0 + threadIdx.x / G;
    const bool live = unit < total_units;
    const uint32_t uu = live ? unit : total_units - 1;
    const uint32_t bk_ = uu / P.N;
    const int i = static_cast<int>(uu % P.N);
    const int kl = static_cast<int>(bk_ % P.nk), b = static_cast<int>(bk_ / P.nk);
    const int k = P.k0 + kl;
    const PrimeConst pcv = P.pc[k];
    const Mod M = load_mod(pcv);
    const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
    const uint32_t* tab = P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S;
    uint32_t A[C], B[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {  // K2's point values when present, else Horner
      const int j = gl * C + c;
      A[c] = j > n ? 0u : (P.vals ? vals_row(P, b, kl, j)[i] : horner(tab, P.dir[j], P.dir[nq + j], x, M));
    }
    // B = A' (deriv) or the second operand's rows
    {
      const uint32_t up = __shfl_down_sync(0xffffffffu, A[0], 1);  // A[j + 1] across the lane boundary
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int j = gl * C + c;
        if (P.deriv) {
          const uint32_t an = c + 1 < C ? A[c + 1 < C ? c + 1 : c] : (gl + 1 < G ? up : 0u);
          B[c] = j <= n - 1 ? mmul(an, mmul(static_cast<uint32_t>(j + 1), M.r2, M), M) : 0u;
        } else {
          B[c] = j > n - 1 ? 0u
                           : (P.vals ? vals_row(P, b, kl, nq + j)[i]
                                     : horner(tab, P.dir[2 * nq + j], P.dir[2 * nq + n + j], x, M));
        }
      }
    }
    // owner lane of coefficient j within the group, and the value there
    auto fetch = [&](const uint32_t (&V)[C], int j) -> uint32_t {
      uint32_t v = 0u;
      const int oc = j % C;
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (c == oc) v = V[c];
      return __shfl_sync(0xffffffffu, v, gbase + j / C);
    };
    uint32_t a1 = fetch(A, n), a0 = fetch(A, n - 1), b1 = fetch(B, n - 1), b0 = fetch(B, n - 2);
    uint32_t flag = (a1 == 0u) | (b1 == 0u);
    uint32_t U = M.one, E = M.one;
    for (int kk = n - 1; kk >= 1; --kk) {
      // step on (A deg kk + 1, B deg kk): a1 = A[kk+1], a0 = A[kk], b1 = B[kk], b0 = B[kk-1]
      const uint32_t na = mneg(a1, M.p);
      const uint32_t c1 = mmul(b1, b1, M), c2 = mmul(b1, na, M);
      const uint32_t c3 = mneg(mmul2(b1, a0, na, b0, M), M.p);
      const uint32_t bprev = __shfl_up_sync(0xffffffffu, B[C - 1], 1);  // B[gl C - 1]
      uint32_t R[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int j = gl * C + c;
        const uint32_t bm1 = c ? B[c ? c - 1 : 0] : (gl ? bprev : 0u);
        R[c] = j < kk ? mmul3(c1, A[c], c2, bm1, c3, B[c], M) : 0u;
      }
      U = mmul(U, b1, M);
      if (kk >= 2) E = mmul(E, U, M);
      // (A, B) <- (B, R): the next step's a1, a0 are this step's b1, b0
      const uint32_t r1 = fetch(R, kk - 1), r0 = kk >= 2 ? fetch(R, kk - 2) : 0u;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        A[c] = B[c];
        B[c] = R[c];
      }
      a1 = b1;
      a0 = b0;
      b1 = r1;
      b0 = r0;
      flag |= (r1 == 0u);
    }
    // after the last step B[0] is the numerator (fast_euclid: num = B[0])
    const uint32_t num = __shfl_sync(0xffffffffu, B[0], gbase);
    if (live && gl == 0) {
      uint32_t* out = P.rows + b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch + i;
      *out = flag ? kSentinel : mmul(num, minv(mmul(E, E, M), M), M);
    }
  }
}

__global__ void __launch_bounds__(32 * kWarpsGeneral) k_modres_warp(ResParams P, int use_list, uint32_t total_units) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // use_list: 0 every unit, 1 the flag list (or a scan when it overflowed), 2 scan for kSentinel
  const uint32_t flagged = use_list == 1 ? P.counters[0] : 0u;
  const bool scan = use_list == 2 || (use_list == 1 && flagged > P.flag_cap);
  const uint32_t all = static_cast<uint32_t>(P.B) * static_cast<uint32_t>(P.nk) * static_cast<uint32_t>(P.N);
  const uint32_t count = scan ? all : (use_list ? flagged : total_units);
  const int nq = P.n + 1, cap = P.n + 1;
  const size_t wid = static_cast<size_t>(blockIdx.x) * kWarpsGeneral + wib;
  uint32_t* bufA = P.gwarp ? P.gwarp + wid * 2 * cap : sm + static_cast<size_t>(wib) * 2 * cap;
  uint32_t* bufB = bufA + cap;
  for (uint32_t u = blockIdx.x * kWarpsGeneral + wib; u < count; u += gridDim.x * kWarpsGeneral) {
    const uint32_t unit = (use_list && !scan) ? P.flag_list[u] : u;
    const uint32_t bk = unit / P.N;
    const int i = static_cast<int>(unit % P.N);
    const int kl = static_cast<int>(bk % P.nk), b = static_cast<int>(bk / P.nk);
    uint32_t* out = P.rows + b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch + i;
    if (scan && *out != kSentinel) continue;
    const int k = P.k0 + kl;
    const PrimeConst pcv = P.pc[k];
    const Mod M = load_mod(pcv);
    const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
    const uint32_t* tab = P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S;
    __syncwarp();
    for (int j = lane; j <= P.n; j += 32) bufA[j] = horner(tab, P.dir[j], P.dir[nq + j], x, M);
    __syncwarp();
    if (P.deriv) {
      for (int j = lane; j <= P.m; j += 32) bufB[j] = mmul(bufA[j + 1], mmul(static_cast<uint32_t>(j + 1), M.r2, M), M);
    } else {
      const int base = 2 * nq;
      for (int j = lane; j <= P.m; j += 32) bufB[j] = horner(tab, P.dir[base + j], P.dir[base + P.m + 1 + j], x, M);
    }
    uint32_t r;
    uint32_t flag = 1u;
    if (P.m == P.n - 1) r = warp_fast_euclid(bufA, bufB, P.n, M, lane, flag);
    if (flag) {  // not the normal shape, or a degree drop mod p: the exact formal-degree path
      __syncwarp();
      for (int j = lane; j <= P.n; j += 32) bufA[j] = horner(tab, P.dir[j], P.dir[nq + j], x, M);
      __syncwarp();
      if (P.deriv) {
        for (int j = lane; j <= P.m; j += 32) bufB[j] = mmul(bufA[j + 1], mmul(static_cast<uint32_t>(j + 1), M.r2, M), M);
      } else {
        const int base = 2 * nq;
        for (int j = lane; j <= P.m; j += 32) bufB[j] = horner(tab, P.dir[base + j], P.dir[base + P.m + 1 + j], x, M);
      }
      r = warp_res_general(bufA, P.n, bufB, P.m, M, lane);
    }
    if (lane == 0) *out = r;
  }
}

// ---------------------------------------------------------------------------
// K4: per prime, inverse DFT of size N = r * 2^a over the values R(omega^i):
//   c_j = s * sum_{i1 < r} omega^{-i1 j} u[i1][j mod 2^a],
//   u[i1] = radix-2 inverse NTT (root omega^{-r}) of v[r*i2 + i1],
// with s = +-N^{-1}.  Coefficients j >= D must vanish (degree bound check).
// ---------------------------------------------------------------------------
__global__ void k_twiddles(const PrimeConst* __restrict__ pc, int P, int N, uint32_t* twinv) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<size_t>(P) * N) return;
  const int k = static_cast<int>(idx / N), i = static_cast<int>(idx % N);
  const PrimeConst pcv = pc[k];
  twinv[idx] = mpow(pcv.omega_inv, static_cast<uint64_t>(i), load_mod(pcv));
}

template <int R, bool SCATTER>
__global__ void __launch_bounds__(256) k_interp(uint32_t* rows, size_t rows_bstride, int pitch,
                                                const PrimeConst* __restrict__ pc,
                                                const uint32_t* __restrict__ twinv, int k0, int N, int a,
                                                int D, int negate, uint32_t* counters, RowScatter sc) {
  extern __shared__ uint32_t sm[];
  uint32_t* tw = sm;      // omega^{-i}, i < N
  uint32_t* w = sm + N;   // work array
  const int kl = blockIdx.x, b = blockIdx.y;
  const PrimeConst pcv = pc[k0 + kl];
  const Mod M = load_mod(pcv);
  uint32_t* row = rows + b * rows_bstride + static_cast<size_t>(kl) * pitch;
  const uint32_t* twk = twinv + static_cast<size_t>(k0 + kl) * N;
  const int Mlen = 1 << a;
  const int tid = threadIdx.x, bs = blockDim.x;
  bool bad = false;
  for (int i = tid; i < N; i += bs) {
    tw[i] = twk[i];
    const uint32_t val = row[i];
    bad |= (val == kSentinel);
    const int i1 = i % R, i2 = i / R;  // R is a compile-time 1, 3, 5 or 7
    const int br = a ? static_cast<int>(__brev(static_cast<uint32_t>(i2)) >> (32 - a)) : 0;
    w[i1 * Mlen + br] = val;
  }
  if (bad) atomicOr(&counters[1], kErrSentinel);
  __syncthreads();
  // R inverse NTTs of length Mlen, DIT on the bit-reversed input: stages (lg, lg + 1) fused
  // into radix-4 passes (4 elements per thread: the same 4 twiddle products as two radix-2
  // stages, half the shared-memory traffic, index math and barriers), then a last radix-2
  // stage when log2(Mlen) is odd.  Index math by shifts (every length is a power of 2).
  int lg = 1;
  for (; lg + 1 <= a; lg += 2) {
    const int h = 1 << (lg - 1), l4 = a - 2;  // items per NTT: Mlen / 4 = 2^l4
    const int s1 = a - lg, s2 = a - lg - 1;   // twiddle strides of the two stages
    for (int bb = tid; bb < (R << l4); bb += bs) {
      const int rw = bb >> l4, q = bb & ((1 << l4) - 1);
      const int g = q >> (lg - 1), t = q & (h - 1);
      uint32_t* base = w + rw * Mlen + (g << (lg + 1));
      const uint32_t x0 = base[t], x1 = base[t + h], x2 = base[t + 2 * h], x3 = base[t + 3 * h];
      const uint32_t w1 = tw[(R * t) << s1];
      const uint32_t v1 = mmul(x1, w1, M), v3 = mmul(x3, w1, M);
      const uint32_t y0 = madd(x0, v1, M.p), y1 = msub(x0, v1, M.p);
      const uint32_t y2 = madd(x2, v3, M.p), y3 = msub(x2, v3, M.p);
      const uint32_t u2 = mmul(y2, tw[(R * t) << s2], M), u3 = mmul(y3, tw[(R * (t + h)) << s2], M);
      base[t] = madd(y0, u2, M.p);
      base[t + 2 * h] = msub(y0, u2, M.p);
      base[t + h] = madd(y1, u3, M.p);
      base[t + 3 * h] = msub(y1, u3, M.p);
    }
    __syncthreads();
  }
  if (lg == a) {  // odd log2(Mlen): one radix-2 stage
    const int half = 1 << (lg - 1), lgh = a - 1;
    for (int bb = tid; bb < (R << lgh); bb += bs) {
      const int rw = bb >> lgh, q = bb & ((1 << lgh) - 1);
      const int g = q >> (lg - 1), t = q & (half - 1);
      uint32_t* base = w + rw * Mlen + (g << lg);
      const uint32_t u = base[t];
      const uint32_t v = mmul(base[t + half], tw[R * t], M);
      base[t] = madd(u, v, M.p);
      base[t + half] = msub(u, v, M.p);
    }
    __syncthreads();
  }
  bool tail = false;
  for (int j = tid; j < N; j += bs) {
    const int j1 = j & (Mlen - 1);
    uint32_t acc;
    if (R == 1) {
      acc = w[j1];
    } else {
      acc = 0;
      int e = 0;  // i1 * j mod N, stepped (j < N)
#pragma unroll
      for (int i1 = 0; i1 < R; ++i1) {
        acc = madd(acc, mmul(w[i1 * Mlen + j1], tw[e], M), M.p);
        e += j;
        if (e >= N) e -= N;
      }
    }
    uint32_t c = mmul(acc, pcv.scale, M);  // Montgomery x plain -> plain
    if (negate) c = mneg(c, M.p);
    if (j < D) {
      if constexpr (SCATTER) {  // straight into the owning shard's receive block (peer store over NVLink)
        const int r = j / sc.Jb;
        sc.dst[r][sc.shard_off + b * sc.curve_stride + static_cast<long long>(kl) * sc.Jb + (j - r * sc.Jb)] = c;
      } else {
        row[j] = c;
      }
    } else {
      tail |= (c != 0u);
    }
  }
  if (tail) atomicOr(&counters[1], kErrNttTail);
}

// K4 for sizes beyond shared memory (N > kMaxNttSmem): the same inverse DFT on a global
// work array, one launch per pass -- the permutation into [R][2^a] bit-reversed rows, a
// radix-2 DIT stages (butterfly per thread, twiddles from the [P][N] table), then the
// r-point twiddled DFT, scaling, negation and degree-bound check of k_interp.
__global__ void k_interp_big_permute(const uint32_t* __restrict__ rows, size_t rows_bstride, int pitch, int nk,
                                     int N, int R, int a, uint32_t* __restrict__ w) {
  const int kl = blockIdx.y, b = blockIdx.z;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const uint32_t* row = rows + b * rows_bstride + static_cast<size_t>(kl) * pitch;
  uint32_t* wk = w + (static_cast<size_t>(b) * nk + kl) * N;
  const int i1 = i % R, i2 = i / R;
  const int br = a ? static_cast<int>(__brev(static_cast<uint32_t>(i2)) >> (32 - a)) : 0;
  wk[(i1 << a) + br] = row[i];
}

__global__ void k_interp_big_stage(uint32_t* __restrict__ w, int nk, int N, int R, int a, int lg,
                                   const PrimeConst* __restrict__ pc, const uint32_t* __restrict__ twinv, int k0) {
  const int kl = blockIdx.y, b = blockIdx.z;
  const int bb = blockIdx.x * blockDim.x + threadIdx.x;  // butterfly: R * 2^(a-1) per (curve, prime)
  if (bb >= (R << (a - 1))) return;
  const Mod M = load_mod(pc[k0 + kl]);
  const uint32_t* tw = twinv + static_cast<size_t>(k0 + kl) * N;
  uint32_t* wk = w + (static_cast<size_t>(b) * nk + kl) * N;
  const int half = 1 << (lg - 1), lgh = a - 1;
  const int rw = bb >> lgh, q = bb & ((1 << lgh) - 1);
  const int g = q >> (lg - 1), t = q & (half - 1);
  uint32_t* base = wk + (rw << a) + (g << lg);
  const uint32_t u = base[t];
  const uint32_t v = mmul(base[t + half], __ldg(&tw[(R * t) << (a - lg)]), M);
  base[t] = madd(u, v, M.p);
  base[t + half] = msub(u, v, M.p);
}

template <bool SCATTER>
__global__ void k_interp_big_final(const uint32_t* __restrict__ w, uint32_t* rows, size_t rows_bstride, int pitch,
                                   int nk, int N, int R, int a, int D, int negate, const PrimeConst* __restrict__ pc,
                                   const uint32_t* __restrict__ twinv, int k0, uint32_t* counters, RowScatter sc) {
  const int kl = blockIdx.y, b = blockIdx.z;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  const PrimeConst pcv = pc[k0 + kl];
  const Mod M = load_mod(pcv);
  const uint32_t* tw = twinv + static_cast<size_t>(k0 + kl) * N;
  const uint32_t* wk = w + (static_cast<size_t>(b) * nk + kl) * N;
  const int j1 = j & ((1 << a) - 1);
  uint32_t acc = 0;
  long long e = 0;
  for (int i1 = 0; i1 < R; ++i1) {
    acc = madd(acc, mmul(wk[(i1 << a) + j1], __ldg(&tw[e]), M), M.p);
    e += j;
    if (e >= N) e -= N;
  }
  uint32_t c = mmul(acc, pcv.scale, M);
  if (negate) c = mneg(c, M.p);
  if (j < D) {
    if constexpr (SCATTER) {
      const int r = j / sc.Jb;
      sc.dst[r][sc.shard_off + b * sc.curve_stride + static_cast<long long>(kl) * sc.Jb + (j - r * sc.Jb)] = c;
    } else {
      rows[b * rows_bstride + static_cast<size_t>(kl) * pitch + j] = c;
    }
  } else if (c != 0u) {
    atomicOr(&counters[1], kErrNttTail);
  }
}

// ---------------------------------------------------------------------------
// K5: fixed-point CRT.  For coefficient j with residues v_k:
//   y_k = v_k (M/p_k)^{-1} mod p_k,   u = sum_k y_k / p_k,   t = round(u),
//   c = sum_k y_k (M/p_k) - t M      (|c| < M / 2^35 by the choice of primes, so
//   u is within 2^-34 of an integer and the double sum rounds exactly).
// ---------------------------------------------------------------------------
__device__ __forceinline__ const uint32_t* crt_row(const CrtParams& C, int b, int k) {
  return C.rows + b * C.curve_stride + static_cast<long long>(k / C.row_block) * C.block_stride +
         static_cast<long long>(k % C.row_block) * C.pitch;
}

// grid (ceil(J/32), ceil(P/kCrtChunk), B), block (32, 8): y_k for 32 coefficients x 64 primes,
// plus the partial sum of y_k / p_k over the chunk.
__global__ void __launch_bounds__(256) k_crt_prep(CrtParams C) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int jl = blockIdx.x * 32 + tx;
  const int chunk = blockIdx.y, b = blockIdx.z;
  const int kbeg = chunk * kCrtChunk, kend = min(kbeg + kCrtChunk, C.P);
  double u = 0;
  if (jl < C.J) {
    for (int k = kbeg + ty; k < kend; k += 8) {
      const PrimeConst& pcv = C.pc[k];
      const Mod M = load_mod(pcv);
      const uint32_t v = crt_row(C, b, k)[C.j0 - C.col0 + jl];
      const uint32_t y = mmul(v, pcv.crt_c, M);
      C.Y[(static_cast<size_t>(b) * C.P + k) * C.J + jl] = y;
      u += static_cast<double>(y) * C.minv[k];
    }
  }
  red[ty][tx] = u;
  __syncthreads();
  if (ty == 0 && jl < C.J) {
    double s = 0;
    for (int q = 0; q < 8; ++q) s += red[q][tx];
    const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
    C.upart[(static_cast<size_t>(b) * nch + chunk) * C.J + jl] = s;
  }
}

// cols[j][l] = sum_k Y[k][j] * Mk16[k][l]  (31-bit x 16-bit products, exact u64 sums:
// one IMAD.WIDE.U32 with 64-bit accumulate per MAC).  Tile 32 j x 64 l, 128 threads,
// 4 x 4 accumulators per thread, k staged through shared memory 16 primes at a time.
__global__ void __launch_bounds__(128) k_crt_gemm(CrtParams C) {
  __shared__ __align__(16) uint32_t Ys[16][32];
  __shared__ __align__(16) uint32_t Ms[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // ty < 8
  const int jb = blockIdx.y * 32, lb = blockIdx.x * 64, b = blockIdx.z;
  const uint32_t* Yb = C.Y + static_cast<size_t>(b) * C.P * C.J;
  uint64_t acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = 0;
  for (int k0 = 0; k0 < C.P; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 32; e += 128) {
      const int kk = e >> 5, c = e & 31;
      const int k = k0 + kk;
      Ys[kk][c] = (k < C.P && jb + c < C.J) ? Yb[static_cast<size_t>(k) * C.J + jb + c] : 0u;
    }
    for (int e = threadIdx.x; e < 16 * 64; e += 128) {
      const int kk = e >> 6, c = e & 63;
      const int k = k0 + kk;
      Ms[kk][c] = (k < C.P && lb + c < C.L16) ? C.Mk16[static_cast<size_t>(k) * C.L16 + lb + c] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      const uint4 yv = *reinterpret_cast<const uint4*>(&Ys[kk][ty * 4]);
      const uint4 mv = *reinterpret_cast<const uint4*>(&Ms[kk][tx * 4]);
      const uint32_t ya[4] = {yv.x, yv.y, yv.z, yv.w};
      const uint32_t ma[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] += static_cast<uint64_t>(ya[a]) * ma[q];
    }
    __syncthreads();
  }
  uint64_t* cols = C.cols + static_cast<size_t>(b) * C.J * C.L16;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int j = jb + ty * 4 + a;
    if (j >= C.J) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = lb + tx * 4 + q;
      if (l < C.L16) cols[static_cast<size_t>(j) * C.L16 + l] = acc[a][q];
    }
  }
}

// Carry propagation of sum_l cols[l] 2^(16 l) - t M, one warp per coefficient.
// t = round(sum of the partial sums of y_k / p_k).  Lane i owns `chunk` 16-bit digits
// (chunk even, >= 4, so a lane's value spans >= 64 bits): (1) local propagation with
// carry-in 0 gives the lane's digits V_i and carry-out c_i; (2) the carry-ins follow
// sequentially, C_{i+1} = c_i + floor((V_i + C_i) / 2^W), where |C_i| < 2^45 << 2^W makes
// the floor -1, 0 or +1 -- decided from V_i's low 64 bits and whether its higher digits
// are all ones / all zeros; (3) each lane adds its C_i; (4) a negative total is negated
// in two's complement (sign-magnitude output).
__global__ void __launch_bounds__(128) k_crt_carry(CrtParams C) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= C.J * C.B) return;
  const int b = gw / C.J, jl = gw - b * C.J;
  const int L16 = C.L16, OL = C.out_limbs;
  // rounding estimate t
  const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
  double s = 0;
  for (int q = lane; q < nch; q += 32) s += C.upart[(static_cast<size_t>(b) * nch + q) * C.J + jl];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  const double tr = rint(s);
  if (lane == 0 && fabs(s - tr) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
  const int64_t t = static_cast<int64_t>(tr);

  int chunk = 2 * ((L16 + 63) / 64);
  if (chunk < 4) chunk = 4;
  const int d0 = lane * chunk;
  const uint64_t* col = C.cols + (static_cast<size_t>(b) * C.J + jl) * L16;
  uint32_t* out = C.out + (static_cast<size_t>(b) * C.J + jl) * (OL + 1);
  // (1) local propagation
  int64_t carry = 0;
  uint64_t low = 0;
  bool ones = true, zeros = true;
  for (int k = 0; k < chunk; k += 2) {
    uint32_t limb = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l = d0 + k + h;
      int64_t v = carry;
      if (l < L16) v += static_cast<int64_t>(col[l]) - t * static_cast<int64_t>(C.M16[l]);
      limb |= static_cast<uint32_t>(v & 0xffff) << (16 * h);
      carry = v >> 16;
    }
    const int w = (d0 + k) >> 1;
    if (w < OL) out[1 + w] = limb;
    if (k < 4) {
      low |= static_cast<uint64_t>(limb) << (16 * k);
    } else {
      ones &= (limb == 0xffffffffu);
      zeros &= (limb == 0u);
    }
  }
  // (2) sequential carry-in scan over the lanes
  int64_t cin = 0, my_cin = 0;
  const uint32_t flags = (ones ? 1u : 0u) | (zeros ? 2u : 0u);
  for (int i = 0; i < 32; ++i) {
    const int64_t ci = __shfl_sync(0xffffffffu, carry, i);
    const uint64_t lo = __shfl_sync(0xffffffffu, low, i);
    const uint32_t fl = __shfl_sync(0xffffffffu, flags, i);
    if (lane == i) my_cin = cin;
    int64_t adj = 0;
    if (cin > 0) {
      adj = ((fl & 1u) && lo + static_cast<uint64_t>(cin) < lo) ? 1 : 0;
    } else if (cin < 0) {
      adj = ((fl & 2u) && lo < static_cast<uint64_t>(-cin)) ? -1 : 0;
    }
    cin = ci + adj;
  }
  const int64_t total_carry = cin;
  // (3) add the carry-in to this lane's limbs
  int64_t c = my_cin;
  for (int k = 0; k < chunk && c != 0; k += 2) {
    const int w = (d0 + k) >> 1;
    if (w >= OL) break;
    const int64_t v = static_cast<int64_t>(out[1 + w]) + c;
    out[1 + w] = static_cast<uint32_t>(v);
    c = v >> 32;
  }
  __syncwarp();
  // (4) sign and magnitude
  int lowest = OL;
  for (int k = 0; k < chunk; k += 2) {
    const int w = (d0 + k) >> 1;
    if (w < OL && out[1 + w] != 0u) {
      lowest = w;
      break;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lowest = min(lowest, __shfl_xor_sync(0xffffffffu, lowest, off));
  if (total_carry < 0) {
    for (int k = 0; k < chunk; k += 2) {
      const int w = (d0 + k) >> 1;
      if (w >= OL || w < lowest) continue;
      out[1 + w] = (w == lowest) ? (0u - out[1 + w]) : ~out[1 + w];
    }
  }
  if (lane == 0) out[0] = static_cast<uint32_t>(lowest >= OL ? 0 : (total_carry < 0 ? -1 : 1));
}

// ---------------------------------------------------------------------------
// K5 on the tensor cores.  With Yt[j][k] = y_k (u32, k contiguous) read as bytes,
//   A[j][4k+a] = byte a of y_k,   Bt8[l][4k+a] = byte (l-a) of M/p_k,
//   C[j][l] = sum_{k,a} A[j][4k+a] Bt8[l][4k+a]  = the coefficient of 2^(8l) in sum_k y_k M/p_k
// (u8 x u8 -> s32, exact while 4P * 255^2 < 2^31).  One mma.sync.m16n8k32 per 16x8x32.
// ---------------------------------------------------------------------------

// grid (ceil(J/32), ceil(P/64), B), block (32, 8): y_k for 32 coefficients x 64 primes,
// transposed through shared memory into Yt (k contiguous), plus the partial sums of y_k/p_k.
__global__ void __launch_bounds__(256) k_crt_prep_t(CrtParams C) {
  __shared__ uint32_t tile[kCrtChunk][33];
  __shared__ double red[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int jb = blockIdx.x * 32, jl = jb + tx;
  const int chunk = blockIdx.y, b = blockIdx.z;
  const int kbeg = chunk * kCrtChunk, kend = min(kbeg + kCrtChunk, C.P);
  double u = 0;
  for (int k = kbeg + ty; k < kbeg + kCrtChunk; k += 8) {
    uint32_t y = 0;
    if (k < kend && jl < C.J) {
      const PrimeConst& pcv = C.pc[k];
      const Mod M = load_mod(pcv);
      y = mmul(crt_row(C, b, k)[C.j0 - C.col0 + jl], pcv.crt_c, M);
      u += static_cast<double>(y) * C.minv[k];
    }
    tile[k - kbeg][tx] = y;
  }
  red[ty][tx] = u;
  __syncthreads();
  if (ty == 0 && jl < C.J) {
    double s = 0;
    for (int q = 0; q < 8; ++q) s += red[q][tx];
    const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
    C.upart[(static_cast<size_t>(b) * nch + chunk) * C.J + jl] = s;
  }
  const int ppad = C.Kp / 4;
  const int t = ty * 32 + tx;
  for (int e = t; e < 32 * kCrtChunk; e += 256) {
    const int jj = e / kCrtChunk, kk = e % kCrtChunk;
    if (jb + jj < C.J && kbeg + kk < ppad)  // row b * J + j (the padding rows past B * J are never read back)
      C.Y[(static_cast<size_t>(b) * C.J + jb + jj) * ppad + kbeg + kk] = tile[kk][jj];
  }
}

__device__ __forceinline__ void mma_u8(int32_t (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* smem) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}

// grid (L8p / 128, Rp / 128), 256 threads = 8 warps (2 along j x 4 along l), warp tile
// 64 j x 32 l (4 x 4 mma tiles).  K is staged 64 bytes per step through a 2-deep cp.async
// pipeline; fragments come from ldmatrix (row pitch 80 B: conflict-free).
__global__ void __launch_bounds__(256) k_crt_gemm_i8(CrtParams C) {
  constexpr int kBK = 64, kPitch = 80;
  __shared__ __align__(128) uint8_t As[2][kI8TileJ * kPitch];
  __shared__ __align__(128) uint8_t Bs[2][kI8TileL * kPitch];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  const int jb = blockIdx.y * kI8TileJ, lb = blockIdx.x * kI8TileL;  // jb: first flattened row
  const uint8_t* Ab = reinterpret_cast<const uint8_t*>(C.Y) + static_cast<size_t>(jb) * C.Kp;
  const uint8_t* Bb = C.Bt8 + static_cast<size_t>(lb) * C.Kp;
  const int nst = C.Kp / kBK;
  auto load = [&](int stage, int buf) {
    const int k0 = stage * kBK;
#pragma unroll
    for (int e = tid; e < 1024; e += 256) {
      const bool isB = e >= 512;
      const int ee = e & 511, row = ee >> 2, ch = ee & 3;
      const uint8_t* src = (isB ? Bb : Ab) + static_cast<size_t>(row) * C.Kp + k0 + ch * 16;
      uint8_t* dst = (isB ? Bs[buf] : As[buf]) + row * kPitch + ch * 16;
      cp_async16(dst, src);
    }
    cp_async_commit();
  };
  int32_t acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0;
  load(0, 0);
  for (int s = 0; s < nst; ++s) {
    if (s + 1 < nst) {
      load(s + 1, (s + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint8_t* as = As[s & 1];
    const uint8_t* bs = Bs[s & 1];
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 32) {
      uint32_t af[4][4], bf[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        ldmatrix_x4(af[mi], as + (wm * 64 + mi * 16 + (lane & 15)) * kPitch + kk + (lane >> 4) * 16);
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        uint32_t t[4];
        ldmatrix_x4(t, bs + (wn * 32 + nj * 16 + ((lane >> 4) << 3) + (lane & 7)) * kPitch + kk + ((lane >> 3) & 1) * 16);
        bf[2 * nj][0] = t[0];
        bf[2 * nj][1] = t[1];
        bf[2 * nj + 1][0] = t[2];
        bf[2 * nj + 1][1] = t[3];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma_u8(acc[mi][ni], af[mi], bf[ni][0], bf[ni][1]);
    }
    __syncthreads();
  }
  // C layout [row tile of 128][digit group l / 4][row in tile][4] (see the carry kernel).
  int32_t* Cb = reinterpret_cast<int32_t*>(C.cols) + static_cast<size_t>(jb) * C.L8p;  // tile jb / 128
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int r = jb + wm * 64 + mi * 16 + g;
      const int c = lb + wn * 32 + ni * 8 + tig * 2;
      int32_t* at = Cb + (static_cast<size_t>(c >> 2) * kI8TileJ + (r - jb)) * 4 + (c & 3);
      *reinterpret_cast<int2*>(at) = make_int2(acc[mi][ni][0], acc[mi][ni][1]);
      *reinterpret_cast<int2*>(at + 32) = make_int2(acc[mi][ni][2], acc[mi][ni][3]);  // row r + 8
    }
}



// Carry propagation of V = sum_l C[l] 2^(8 l) - t M (K5 epilogue), one THREAD per coefficient:
// a sequential walk over the L8 byte digits (4 per limb step: one int4 of the GEMM output,
// whose [digit group][coefficient] layout makes every warp load 512 contiguous bytes; 8 loads
// in flight per thread, M8 broadcast from L1), then, for V < 0, a two's-
// complement pass over the limbs the same thread just wrote.  Each coefficient is a few
// hundred to a few thousand digits; thousands of independent walks hide the carry-chain
// latency.  (Measured on B200 against a warp-per-coefficient lookahead scan, SEG threads per
// coefficient with a segment scan, shared-memory row tiles, and a variant that settles the
// sign first to avoid the second pass: this is the fastest at d20 / d30 / d16.)
// WIDE: 64-bit carry arithmetic (needed when 4P * 255^2 + 2^25 >= 2^31).
template <bool WIDE>
__global__ void __launch_bounds__(128) k_crt_carry_seq(CrtParams C) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= C.J * C.B) return;
  const int b = g / C.J, jl = g - b * C.J;
  const int OL = C.out_limbs;
  const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
  double s = 0;
  for (int q = 0; q < nch; ++q) s += C.upart[(static_cast<size_t>(b) * nch + q) * C.J + jl];
  const double tr = rint(s);
  if (fabs(s - tr) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
  const int32_t t = static_cast<int32_t>(tr);
  // GEMM output [row tile of 128][digit group][row in tile] of int4, row = b * J + jl = g:
  // limb w of this coefficient is col[w * 128]; a warp's loads of one limb are consecutive
  // rows of one tile (coalesced), and a thread's walk strides 2 KB through its tile's slab.
  const int4* col = reinterpret_cast<const int4*>(C.cols) + static_cast<size_t>(g >> 7) * (C.L8p / 4) * 128 + (g & 127);
  const uint4* m8 = reinterpret_cast<const uint4*>(C.M8);
  uint32_t* out = C.out + (static_cast<size_t>(b) * C.J + jl) * (OL + 1) + 1;
  using acc_t = typename std::conditional<WIDE, long long, int>::type;
  acc_t carry = 0;
  uint32_t any = 0;
  constexpr int kBatch = 8;
  for (int w0 = 0; w0 < OL; w0 += kBatch) {
    int4 cb[kBatch];
    uint4 mb[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      if (w0 + i < OL) {
        cb[i] = col[static_cast<size_t>(w0 + i) * 128];
        mb[i] = __ldg(&m8[w0 + i]);
      }
    }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
      if (w0 + i >= OL) break;
      const int4 c = cb[i];
      const uint4 m = mb[i];
      uint32_t limb;
      acc_t v = carry + c.x - static_cast<acc_t>(t) * static_cast<int>(m.x);
      limb = static_cast<uint32_t>(v) & 0xffu;
      v = (v >> 8) + c.y - static_cast<acc_t>(t) * static_cast<int>(m.y);
      limb |= (static_cast<uint32_t>(v) & 0xffu) << 8;
      v = (v >> 8) + c.z - static_cast<acc_t>(t) * static_cast<int>(m.z);
      limb |= (static_cast<uint32_t>(v) & 0xffu) << 16;
      v = (v >> 8) + c.w - static_cast<acc_t>(t) * static_cast<int>(m.w);
      limb |= static_cast<uint32_t>(v) << 24;
      carry = v >> 8;
      out[w0 + i] = limb;
      any |= limb;
    }
  }
  // |V| < M / 2 < 2^(32 OL - 1): the final carry is 0 (V >= 0) or -1 (V < 0); -V = ~V + 1.
  int sign = any ? 1 : 0;
  if (carry < 0) {
    sign = -1;
    uint32_t cin = 1;
    for (int w = 0; w < OL; ++w) {
      const uint32_t x = ~out[w] + cin;
      cin = (cin && x == 0u) ? 1u : 0u;
      out[w] = x;
    }
  }
  out[-1] = static_cast<uint32_t>(sign);
}


// The same walk with coalesced output: a warp's 32 coefficients are consecutive rows, each lane
// walks its own row's digits (as k_crt_carry_seq), the limbs go through a 32 x 33 shared-memory
// tile per warp, and every 32 limbs the warp stores them row by row (128 contiguous bytes per
// store instead of 32 scattered words); negative values are then negated -- rows of <= 128
// limbs by the whole warp, one row at a time (two's complement: the +1 ripples to the lowest
// nonzero limb, found by a ballot), longer rows by their own lane (a warp-serial pass over
// 1,000-limb rows costs more than it saves).  CTA = 4 warps = one 128-row tile of the output.
template <bool WIDE, int kBatch>
__global__ void __launch_bounds__(128) k_crt_carry_tile(CrtParams C) {
  __shared__ uint32_t stage[4][32 * 33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int ncoef = C.J * C.B;
  const bool live = g < ncoef;
  const int gc = live ? g : ncoef - 1;  // idle lanes shadow the last row (never stored)
  const int b = gc / C.J, jl = gc - b * C.J;
  const int OL = C.out_limbs;
  const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
  double s = 0;
  for (int q = 0; q < nch; ++q) s += C.upart[(static_cast<size_t>(b) * nch + q) * C.J + jl];
  const double tr = rint(s);
  if (live && fabs(s - tr) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
  const int32_t t = static_cast<int32_t>(tr);
  const int4* col = reinterpret_cast<const int4*>(C.cols) + static_cast<size_t>(gc >> 7) * (C.L8p / 4) * 128 + (gc & 127);
  const uint4* m8 = reinterpret_cast<const uint4*>(C.M8);
  const int row0 = blockIdx.x * blockDim.x + warp * 32;  // first row of this warp
  uint32_t* st = stage[warp];
  using acc_t = typename std::conditional<WIDE, long long, int>::type;
  acc_t carry = 0;
  uint32_t any = 0;
  for (int w0 = 0; w0 < OL; w0 += 32) {
#pragma unroll
    for (int wb = 0; wb < 32; wb += kBatch) {
      int4 cb[kBatch];
      uint4 mb[kBatch];
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int w = w0 + wb + i;
        if (w < OL) {
          cb[i] = col[static_cast<size_t>(w) * 128];
          mb[i] = __ldg(&m8[w]);
        }
      }
#pragma unroll
      for (int i = 0; i < kBatch; ++i) {
        const int w = w0 + wb + i;
        if (w >= OL) break;
        const int4 c = cb[i];
        const uint4 m = mb[i];
        acc_t v = carry + c.x - static_cast<acc_t>(t) * static_cast<int>(m.x);
        uint32_t limb = static_cast<uint32_t>(v) & 0xffu;
        v = (v >> 8) + c.y - static_cast<acc_t>(t) * static_cast<int>(m.y);
        limb |= (static_cast<uint32_t>(v) & 0xffu) << 8;
        v = (v >> 8) + c.z - static_cast<acc_t>(t) * static_cast<int>(m.z);
        limb |= (static_cast<uint32_t>(v) & 0xffu) << 16;
        v = (v >> 8) + c.w - static_cast<acc_t>(t) * static_cast<int>(m.w);
        limb |= static_cast<uint32_t>(v) << 24;
        carry = v >> 8;
        any |= limb;
        st[(wb + i) * 33 + lane] = limb;
      }
    }
    __syncwarp();
    // flush limbs [w0, w0 + 32) of the warp's rows: lane l stores limb w0 + l of row c
    const int nw = min(32, OL - w0);
    for (int c = 0; c < 32; ++c) {
      const int r = row0 + c;
      if (r < ncoef && lane < nw)
        C.out[static_cast<size_t>(r) * (OL + 1) + 1 + w0 + lane] = st[lane * 33 + c];
    }
    __syncwarp();
  }
  // |V| < M / 2 < 2^(32 OL - 1): the final carry is 0 (V >= 0) or -1 (V < 0); -V = ~V + 1.
  const bool neg = live && carry < 0;
  if (live) C.out[static_cast<size_t>(g) * (OL + 1)] = static_cast<uint32_t>(neg ? -1 : (any ? 1 : 0));
  __syncwarp();  // this warp's limb stores are visible to all its lanes
  if (OL > 128) {  // long rows: every negative lane negates its own row (rows in parallel)
    if (neg) {
      uint32_t* rowp = C.out + static_cast<size_t>(g) * (OL + 1) + 1;
      uint32_t cin = 1;
      for (int w = 0; w < OL; ++w) {
        const uint32_t x = ~rowp[w] + cin;
        cin = (cin && x == 0u) ? 1u : 0u;
        rowp[w] = x;
      }
    }
    return;
  }
  unsigned todo = __ballot_sync(0xffffffffu, neg);
  while (todo) {
    const int c = __ffs(todo) - 1;
    todo &= todo - 1;
    uint32_t* rowp = C.out + static_cast<size_t>(row0 + c) * (OL + 1) + 1;
    bool seen = false;  // warp-uniform: the lowest nonzero limb has been passed
    for (int w0 = 0; w0 < OL; w0 += 32) {
      const int w = w0 + lane;
      const uint32_t x = w < OL ? rowp[w] : 0u;
      uint32_t y = ~x;
      if (!seen) {
        const unsigned nz = __ballot_sync(0xffffffffu, x != 0u);
        if (nz) {
          const int z = __ffs(nz) - 1;
          y = lane < z ? 0u : (lane == z ? 0u - x : ~x);
          seen = true;
        } else {
          y = 0u;
        }
      }
      if (w < OL) rowp[w] = y;
    }
  }
}

// Same carry propagation with a WARP per coefficient, for calls with few coefficients (single
// curves: 871 coefficients at d30 or 241 at d16/1024 leave the thread-per-coefficient walk
// with 7 or 2 CTAs walking 1,000-4,000 digits each).  Lane l walks limbs [l S, (l+1) S) with
// a local carry starting at 0 and keeps, for its segment L_l: the low 64 bits, whether the
// limbs above them are all ones / all zeros, and its carry-out c_l (|c_l| < 2^42).  Adding a
// carry-in to L_l can only overflow (+1) or underflow (-1) through those flags, so a 32-step
// shuffle recurrence gives every lane its carry-in; each lane then adds it to its own limbs
// (the ripple normally stops after two limbs) and, for V < 0, negates its limbs in parallel
// (two's complement: zeros below the lowest nonzero limb, -limb there, ~limb above).
template <bool WIDE>
__global__ void __launch_bounds__(128) k_crt_carry_warp(CrtParams C) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= C.J * C.B) return;  // whole warps exit together
  const int b = gw / C.J, jl = gw - b * C.J;
  const int OL = C.out_limbs;
  const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
  double sp = 0;
  for (int q = lane; q < nch; q += 32) sp += C.upart[(static_cast<size_t>(b) * nch + q) * C.J + jl];
#pragma unroll
  for (int off = 16; off; off >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, off);
  const double tr = rint(sp);
  if (lane == 0 && fabs(sp - tr) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
  const int32_t t = static_cast<int32_t>(tr);
  const int4* col = reinterpret_cast<const int4*>(C.cols) + static_cast<size_t>(gw >> 7) * (C.L8p / 4) * 128 +
                    (gw & 127);  // row b * J + jl, layout as k_crt_carry_seq
  const uint4* m8 = reinterpret_cast<const uint4*>(C.M8);
  uint32_t* out = C.out + (static_cast<size_t>(b) * C.J + jl) * (OL + 1) + 1;
  const int S = (OL + 31) / 32, w0 = lane * S, w1 = min(OL, w0 + S);
  using acc_t = typename std::conditional<WIDE, long long, int>::type;
  acc_t carry = 0;
  uint32_t lo0 = 0, lo1 = 0;
  bool ones = true, zeros = true;  // limbs w0+2 .. w1-1
  constexpr int kBatch = 8;  // loads in flight per lane
  for (int wb = w0; wb < w1; wb += kBatch) {
    int4 cb[kBatch];
    uint4 mb[kBatch];
#pragma unroll
    for (int i = 0; i < kBatch; ++i)
      if (wb + i < w1) {
        cb[i] = col[static_cast<size_t>(wb + i) * 128];
        mb[i] = __ldg(&m8[wb + i]);
      }
#pragma unroll
    for (int i = 0; i < kBatch; ++i) {
    const int w = wb + i;
    if (w >= w1) break;
    const int4 c = cb[i];
    const uint4 m = mb[i];
    acc_t v = carry + c.x - static_cast<acc_t>(t) * static_cast<int>(m.x);
    uint32_t limb = static_cast<uint32_t>(v) & 0xffu;
    v = (v >> 8) + c.y - static_cast<acc_t>(t) * static_cast<int>(m.y);
    limb |= (static_cast<uint32_t>(v) & 0xffu) << 8;
    v = (v >> 8) + c.z - static_cast<acc_t>(t) * static_cast<int>(m.z);
    limb |= (static_cast<uint32_t>(v) & 0xffu) << 16;
    v = (v >> 8) + c.w - static_cast<acc_t>(t) * static_cast<int>(m.w);
    limb |= static_cast<uint32_t>(v) << 24;
    carry = v >> 8;
    out[w] = limb;
    if (w == w0) lo0 = limb;
    else if (w == w0 + 1) lo1 = limb;
    else {
      ones &= (limb == 0xffffffffu);
      zeros &= (limb == 0u);
    }
    }
  }
  const int nseg = w1 > w0 ? w1 - w0 : 0;  // limbs in my segment (0 for idle lanes)
  const uint64_t lo = static_cast<uint64_t>(lo0) | (static_cast<uint64_t>(lo1) << 32);
  const long long co = static_cast<long long>(carry);
  // carry-in of every lane: ci_0 = 0, ci_{l+1} = c_l + ovf_l(ci_l)
  long long c = 0, my_ci = 0;
  for (int l = 0; l < 32; ++l) {
    const uint64_t llo = __shfl_sync(0xffffffffu, lo, l);
    const long long lco = __shfl_sync(0xffffffffu, co, l);
    const int lns = __shfl_sync(0xffffffffu, nseg, l);
    const unsigned lflags = __ballot_sync(0xffffffffu, ones) >> l & 1u;
    const unsigned lzero = __ballot_sync(0xffffffffu, zeros) >> l & 1u;
    if (lane == l) my_ci = c;
    if (lns == 0) continue;  // idle lane: carries pass through
    // ovf of L + c over the segment's 32 * lns bits (|c| < 2^42)
    long long ovf = 0;
    if (lns <= 2) {  // the whole segment is in llo (lns = 1: one limb)
      const int bits = 32 * lns;
      const unsigned __int128 full = static_cast<unsigned __int128>(llo);
      const __int128 sum = static_cast<__int128>(full) + c;
      const __int128 modv = static_cast<__int128>(1) << bits;
      ovf = sum >= modv ? 1 : (sum < 0 ? -1 : 0);
    } else {
      const uint64_t nlo = llo + static_cast<uint64_t>(c);
      if (c > 0 && nlo < llo && lflags) ovf = 1;
      if (c < 0 && nlo > llo && lzero) ovf = -1;
    }
    c = lco + ovf;
  }
  // c is the carry out of the top limb: 0 (V >= 0) or -1 (V < 0); apply my carry-in
  if (my_ci != 0 && nseg > 0) {
    long long cc = my_ci;
    for (int w = w0; w < w1 && cc != 0; ++w) {
      const long long x = static_cast<long long>(out[w]) + cc;
      out[w] = static_cast<uint32_t>(x);
      cc = x >> 32;  // arithmetic: borrow -1, carry +1, or the carry's high part
    }
  }
  __syncwarp();
  const int sign_neg = c < 0;
  uint32_t any = 0;
  for (int w = w0; w < w1; ++w) any |= out[w];
  const unsigned nz = __ballot_sync(0xffffffffu, any != 0u);
  if (sign_neg) {
    const int zl = __ffs(nz) - 1;  // first lane holding a nonzero limb
    bool seen = lane > zl;
    for (int w = w0; w < w1; ++w) {
      const uint32_t x = out[w];
      if (seen) {
        out[w] = ~x;
      } else if (x != 0u) {
        out[w] = 0u - x;
        seen = true;
      }
    }
  }
  if (lane == 0) out[-1] = static_cast<uint32_t>(sign_neg ? -1 : (nz ? 1 : 0));
}
}  // namespace

size_t crt_y_words(const CrtTables& T, int B, int J) {
  if (T.use_i8) {
    const size_t Rp = (static_cast<size_t>(B) * J + kI8TileJ - 1) / kI8TileJ * kI8TileJ;
    return Rp * (T.Kp / 4);
  }
  return static_cast<size_t>(B) * T.P * J;
}

size_t crt_cols_words(const CrtTables& T, int B, int J) {
  if (T.use_i8) {
    const size_t Rp = (static_cast<size_t>(B) * J + kI8TileJ - 1) / kI8TileJ * kI8TileJ;
    return Rp * T.L8p;
  }
  return static_cast<size_t>(B) * J * T.L16 * 2;
}

int launch_reduce(const uint32_t* d_limbs, const int8_t* d_sign, int S, int L, const PrimeConst* d_pc,
                  const uint32_t* d_rpow, int k0, int nk, uint32_t* d_tab, size_t tab_bstride, int B, cudaStream_t st,
                  int coef_major) {
  if (S == 0 || nk == 0 || B == 0) return 0;
  const long long n = static_cast<long long>(nk) * S;
  if (L >= 32 && n * B < 148LL * 256) {  // few pairs, long coefficients: a warp per pair
    dim3 grid(static_cast<unsigned>((n * 32 + 127) / 128), B);
    k_reduce_warp<<<grid, 128, 0, st>>>(d_limbs, d_sign, S, L, d_pc, d_rpow, k0, nk, d_tab, tab_bstride, coef_major);
    return 1;
  }
  dim3 grid(static_cast<unsigned>((n + 127) / 128), B);
  if (coef_major)
    k_reduce<true><<<grid, 128, 0, st>>>(d_limbs, d_sign, S, L, d_pc, d_rpow, k0, nk, d_tab, tab_bstride);
  else
    k_reduce<false><<<grid, 128, 0, st>>>(d_limbs, d_sign, S, L, d_pc, d_rpow, k0, nk, d_tab, tab_bstride);
  return 1;
}

// Enough blocks for the scan mode of k_modres_general (blocks beyond a short list exit at once).
constexpr int kGeneralListBlocks = 148 * 4;

// k_modres_warp over the units a previous kernel left at kSentinel (scan mode).
static int launch_sentinel_scan(const ResParams& rp, size_t smem, cudaStream_t st) {
  const int blocks = rp.gwarp ? static_cast<int>(kGeneralWarpGlobalBlocks) : 148 * 16;
  k_modres_warp<<<blocks, 32 * kWarpsGeneral, smem, st>>>(rp, 2, 0u);
  return 1;
}

int launch_modres(const ResParams& rp, bool fast, cudaStream_t st, int part) {
  if (rp.nk == 0 || rp.B == 0) return 0;
  if (fast && rp.fused) {  // K2 folded into K3: the point values never leave shared memory
    if (part == 1) return 0;
    if (dispatch_fused_any(rp.n, rp, st)) {
      k_modres_general<<<kGeneralListBlocks, 128, 0, st>>>(rp, 1, 0u);
      return 2;
    }
  }
  if (fast && rp.vals && (rp.m == rp.n - 1 || (rp.m == rp.n && !rp.deriv)) && rp.n >= 2 && rp.n <= kFastMaxDeg) {
    const int launches = part == 2 ? 0 : launch_eval(rp, st);  // K2
    if (part == 1) return launches;
    if (dispatch_fast_any(rp.n, rp, st)) {                      // K3
      k_modres_general<<<kGeneralListBlocks, 128, 0, st>>>(rp, 1, 0u);          // degenerate units, exact
      return launches + 2;
    }
  }
  const uint32_t total = static_cast<uint32_t>(rp.B) * rp.nk * static_cast<uint32_t>(rp.N);
  if (rp.n > kThreadGeneralMax && rp.n <= 127 && rp.m == rp.n - 1) {
    // K2 (point values by coset NTT, when the plan holds the buffer), then four units per warp in
    // registers, then the exact path for the units it marked
    const int ev = rp.vals && part != 2 ? launch_eval(rp, st) : 0;
    if (part == 1) return ev;
    const uint32_t blocks_mw = std::min<uint32_t>((total + 15) / 16, 148u * 32u);
    const int C = (rp.n + 1 + 7) / 8;
    if (C <= 6)
      k_modres_mw<6><<<blocks_mw, 128, 0, st>>>(rp, total);
    else if (C <= 8)
      k_modres_mw<8><<<blocks_mw, 128, 0, st>>>(rp, total);
    else if (C <= 12)
      k_modres_mw<12><<<blocks_mw, 128, 0, st>>>(rp, total);
    else
      k_modres_mw<16><<<blocks_mw, 128, 0, st>>>(rp, total);
    const size_t smem = rp.gwarp ? 0 : general_warp_smem(rp.n);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_modres_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    return ev + 1 + launch_sentinel_scan(rp, smem, st);
  }
  if (part == 1) return 0;
  if (rp.n > kThreadGeneralMax) {  // warp per unit (any degree)
    const size_t smem = rp.gwarp ? 0 : general_warp_smem(rp.n);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_modres_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const uint32_t want = (total + kWarpsGeneral - 1) / kWarpsGeneral;
    const int blocks = static_cast<int>(std::min<uint32_t>(want, rp.gwarp ? kGeneralWarpGlobalBlocks : 148u * 16u));
    k_modres_warp<<<blocks, 32 * kWarpsGeneral, smem, st>>>(rp, 0, total);
    return 1;
  }
  const int blocks = static_cast<int>(std::min<uint32_t>((total + 127) / 128, 148u * 16u));
  k_modres_general<<<blocks, 128, 0, st>>>(rp, 0, total);
  return 1;
}

size_t general_warp_smem(int n) { return static_cast<size_t>(kWarpsGeneral) * 2 * (n + 1) * 4; }
size_t general_warp_gbuf_words(int n) {
  return general_warp_smem(n) > kGeneralWarpSmemMax
             ? static_cast<size_t>(kGeneralWarpGlobalBlocks) * kWarpsGeneral * 2 * (n + 1)
             : 0;
}

int launch_interp(uint32_t* rows, size_t rows_bstride, int pitch, int nk, int B, const PrimeConst* d_pc,
                  const uint32_t* d_twinv, int k0, int N, int r, int a, int D, int negate, uint32_t* counters,
                  cudaStream_t st, uint32_t* d_work, const RowScatter* scatter) {
  if (nk == 0 || B == 0) return 0;
  RowScatter sc{};
  if (scatter) sc = *scatter;
  if (static_cast<uint32_t>(N) > kMaxNttSmem) {  // global-memory passes (d_work: B * nk * N words)
    if (!d_work) throw std::runtime_error("launch_interp: work array missing for N > kMaxNttSmem");
    const dim3 gp((N + 255) / 256, nk, B);
    k_interp_big_permute<<<gp, 256, 0, st>>>(rows, rows_bstride, pitch, nk, N, r, a, d_work);
    const dim3 gs(((r << (a - 1)) + 255) / 256, nk, B);
    for (int lg = 1; lg <= a; ++lg)
      k_interp_big_stage<<<gs, 256, 0, st>>>(d_work, nk, N, r, a, lg, d_pc, d_twinv, k0);
    if (sc.G)
      k_interp_big_final<true><<<gp, 256, 0, st>>>(d_work, rows, rows_bstride, pitch, nk, N, r, a, D, negate, d_pc,
                                                   d_twinv, k0, counters, sc);
    else
      k_interp_big_final<false><<<gp, 256, 0, st>>>(d_work, rows, rows_bstride, pitch, nk, N, r, a, D, negate, d_pc,
                                                    d_twinv, k0, counters, sc);
    return a + 2;
  }
  const size_t smem = static_cast<size_t>(2) * N * 4;
  // one radix-2 butterfly per thread per stage where possible (r * 2^(a-1) of them)
  int threads = (r << a) / 2;
  threads = threads < 32 ? 32 : (threads > 256 ? 256 : (threads + 31) / 32 * 32);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<dim3(nk, B), threads, smem, st>>>(rows, rows_bstride, pitch, d_pc, d_twinv, k0, N, a, D, negate, counters, sc);
  };
  if (sc.G) {
    switch (r) {
      case 1: go(k_interp<1, true>); break;
      case 3: go(k_interp<3, true>); break;
      case 5: go(k_interp<5, true>); break;
      default: go(k_interp<7, true>); break;
    }
  } else {
    switch (r) {
      case 1: go(k_interp<1, false>); break;
      case 3: go(k_interp<3, false>); break;
      case 5: go(k_interp<5, false>); break;
      default: go(k_interp<7, false>); break;
    }
  }
  return 1;
}

void launch_twiddles(const PrimeConst* d_pc, int P, int N, uint32_t* d_twinv) {
  const size_t total = static_cast<size_t>(P) * N;
  k_twiddles<<<static_cast<unsigned>((total + 255) / 256), 256>>>(d_pc, P, N, d_twinv);
}

// ---------------------------------------------------------------------------
// K5 with the carry walk fused into the tcgen05 GEMM epilogue.
//
// The unfused CRT wrote one s32 per 8-bit digit (4x the bytes of the result limbs) from the
// GEMM and read it back in the carry walk.  Here each epilogue thread owns one coefficient
// (its TMEM lane) and the tile's BN digit columns: it subtracts t M (t = round(sum y_k / p_k),
// M's byte digits), propagates the carries through its BN digits, and stores BN / 4 finished
// u32 limbs (transposed through the freed pipeline stages: coalesced row stores straight
// into the output records) plus a 16-byte summary of its segment: the low 64 bits, whether
// the limbs above them are all ones / all zeros, and the signed carry out.  k_crt_fixup then
// chains the segments of a coefficient (a carry in changes a segment only through those
// summaries: +1 ripples through all-ones limbs, -1 through all-zeros ones), applies the rare
// ripples, negates negative coefficients (two's complement, warp-parallel) and writes the
// sign word.  HBM traffic of the stage: residues in, limbs out (+ the limbs of negative
// coefficients once more), no digit matrix.
// ---------------------------------------------------------------------------
constexpr int kCrtMaxTiles = 64;  // segments per coefficient the fixup chains (L8p <= 64 * BN)

template <int BN, int ST>
__global__ void __launch_bounds__(128)
    k_gemm_u8_carry(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, CrtParams C) {
  using namespace tma;
  extern __shared__ uint8_t smraw[];
  using SM = Smem<BN, ST>;
  SM& sm = *reinterpret_cast<SM*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~static_cast<uintptr_t>(1023));
  static_assert(sizeof(sm.a) + sizeof(sm.b) >= 128 * (BN / 4 + 1) * 4, "epilogue staging must fit the stages");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN, ti = blockIdx.x, nt = gridDim.x;
  const uint32_t tmem = gemm_mainloop<BN, ST>(sm, ta, tb, m0, n0, C.Kp);

  const int nrows = C.B * C.J, OL = C.out_limbs;
  const int r = m0 + tid;  // this thread's coefficient (TMEM lane = row of the tile)
  const bool live = r < nrows;
  const int rc = live ? r : nrows - 1;
  const int b = rc / C.J, jl = rc - b * C.J;
  const int nch = (C.P + kCrtChunk - 1) / kCrtChunk;
  double s = 0;
  for (int q = 0; q < nch; ++q) s += C.upart[(static_cast<size_t>(b) * nch + q) * C.J + jl];
  const double tr = rint(s);
  if (live && ti == 0 && fabs(s - tr) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
  const int t32 = static_cast<int>(tr);  // t < P
  constexpr int LW = BN / 4, PITCH = LW + 1;  // limbs per segment, staging pitch (conflict-free)
  uint32_t* stg = reinterpret_cast<uint32_t*>(sm.a);  // the pipeline stages (a then b, contiguous) are free now
  const uint4* m8 = reinterpret_cast<const uint4*>(C.M8) + n0 / 4;
  long long carry = 0;
  uint64_t low = 0;
  bool ones = true, zero = true;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0), v);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint4 m = __ldg(&m8[c0 / 4 + q]);
      // the 4-digit group's value sum_e (C_e - t M_e) 256^e (|C_e| < 2^31: < 2^57) first, off the
      // carry chain; then ONE dependent 64-bit add and shift per limb
      // C_e - t M_e in int32 (C_e < 4 P 255^2 < 2^31, t M_e < P 255), then widened
      const long long g = static_cast<long long>(static_cast<int>(v[4 * q]) - t32 * static_cast<int>(m.x)) +
                          (static_cast<long long>(static_cast<int>(v[4 * q + 1]) - t32 * static_cast<int>(m.y)) << 8) +
                          (static_cast<long long>(static_cast<int>(v[4 * q + 2]) - t32 * static_cast<int>(m.z)) << 16) +
                          (static_cast<long long>(static_cast<int>(v[4 * q + 3]) - t32 * static_cast<int>(m.w)) << 24);
      const long long x = carry + g;
      const uint32_t limb = static_cast<uint32_t>(x);
      carry = x >> 32;
      const int li = c0 / 4 + q;
      stg[tid * PITCH + li] = limb;
      if (li < 2) {
        low |= static_cast<uint64_t>(limb) << (32 * li);
      } else {
        ones = ones && limb == 0xffffffffu;
        zero = zero && limb == 0u;
      }
    }
  }
  if (live) {
    uint4* meta = reinterpret_cast<uint4*>(C.cols);
    meta[static_cast<size_t>(r) * nt + ti] =
        make_uint4(static_cast<uint32_t>(low), static_cast<uint32_t>(low >> 32), static_cast<uint32_t>(static_cast<int>(carry)),
                   (ones ? 1u : 0u) | (zero ? 2u : 0u));
  }
  __syncthreads();
  // coalesced stores: warp w writes rows 32w..32w+31 of the tile, lanes along the limbs
  const int lim0 = n0 / 4;
  for (int rr = warp * 32; rr < warp * 32 + 32; ++rr) {
    const int row = m0 + rr;
    if (row >= nrows) break;
    uint32_t* dst = C.out + static_cast<size_t>(row) * (OL + 1) + 1 + lim0;
    for (int li = lane; li < LW && lim0 + li < OL; li += 32) dst[li] = stg[rr * PITCH + li];
  }
  gemm_teardown<BN, ST>(sm, tmem);
}

// Warp per coefficient: chain the segment summaries, apply ripples, negate, sign word.  Lane i
// loads segment i's summary; every lane walks the chain redundantly (values by shuffle), and
// lane i keeps the fix-up of segment i.
__global__ void __launch_bounds__(128) k_crt_fixup(CrtParams C, int nt, int LW) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= C.B * C.J) return;  // whole warps
  const int OL = C.out_limbs;
  const uint4* meta = reinterpret_cast<const uint4*>(C.cols) + static_cast<size_t>(row) * nt;
  uint32_t* rowp = C.out + static_cast<size_t>(row) * (OL + 1) + 1;
  // every lane walks the chain (the summaries are broadcast loads: one LDG per segment, no
  // shuffles) and the warp applies a segment's fix-up as soon as it is known
  long long cin = 0;
  int nonzero = 0;
  for (int i = 0; i < nt; ++i) {
    const uint4 mm = meta[i];
    uint64_t low = (static_cast<uint64_t>(mm.y) << 32) | mm.x;
    long long co = static_cast<int>(mm.z);
    bool ones = mm.w & 1u, zero = (mm.w & 2u) != 0;
    if (cin != 0) {
      const uint64_t nl = low + static_cast<uint64_t>(cin);
      int hi = 0;  // carry out of the low 64 bits: cin > 0 overflows, cin < 0 borrows
      if (cin > 0 && nl < low) hi = 1;
      if (cin < 0 && nl > low) hi = -1;
      low = nl;
      const int base = i * LW;
      if (lane < 2 && base + lane < OL) rowp[base + lane] = static_cast<uint32_t>(lane ? low >> 32 : low);
      if (hi != 0) {
        const bool flip = hi == 1 ? ones : zero;  // every upper limb ripples: all ones -> zeros / zeros -> ones
        if (flip) {
          for (int li = 2 + lane; li < LW && base + li < OL; li += 32) rowp[base + li] = hi == 1 ? 0u : 0xffffffffu;
          co += hi;
          ones = hi == -1;
          zero = hi == 1;
        } else {
          // +1: the lowest upper limb != all-ones gets +1, the ones below it become 0 (-1: mirrored)
          const uint32_t stop = hi == 1 ? 0xffffffffu : 0u;
          for (int l0 = 2; l0 < LW; l0 += 32) {
            const int li = l0 + lane;
            const bool in = li < LW && base + li < OL;
            const uint32_t x = in ? rowp[base + li] : stop;
            const unsigned hit = __ballot_sync(0xffffffffu, in && x != stop);
            const int z = hit ? __ffs(hit) - 1 : 32;
            if (in && lane <= z) rowp[base + li] = lane == z ? (hi == 1 ? x + 1u : x - 1u) : ~stop;
            if (hit) break;
          }
          if (hi == 1)
            zero = false;
          else
            ones = false;
        }
      }
    }
    // limbs >= OL are part of the two's complement chain but not of the record
    nonzero |= (low != 0 || !zero) ? 1 : 0;
    cin = co;
  }
  const int neg = cin < 0 ? 1 : 0;  // |V| < M / 2 fits the record: the final carry is 0 or -1
  __syncwarp();
  if (neg) {  // two's complement: zeros below the lowest nonzero limb, -limb there, ~limb above
    bool seen = false;
    for (int w0 = 0; w0 < OL; w0 += 32) {
      const int w = w0 + lane;
      const uint32_t x = w < OL ? rowp[w] : 0u;
      uint32_t y = ~x;
      if (!seen) {
        const unsigned nz = __ballot_sync(0xffffffffu, x != 0u);
        if (nz) {
          const int z = __ffs(nz) - 1;
          y = lane < z ? 0u : (lane == z ? 0u - x : ~x);
          seen = true;
        } else {
          y = 0u;
        }
      }
      if (w < OL) rowp[w] = y;
    }
  }
  if (lane == 0) rowp[-1] = static_cast<uint32_t>(neg ? -1 : (nonzero ? 1 : 0));
}

// ---------------------------------------------------------------------------
// Result packing on the device (ctg_resultant_batch): the CRT records [B][D][W] (sign word +
// LM limbs per coefficient) become the library's result blocks exactly as the host would build
// them (api_common: [16-byte header][limb_off n+1][limbs total][sign n], padded to 16 bytes,
// blocks of consecutive curves back to back), so the D2H lands straight in the page-locked
// result arena and the host only sets pointers.  meta[b] = (n_coeffs, total limbs, byte offset).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_block_bytes(uint32_t n, uint32_t total) {
  return (16u + 4u * (n + 1u) + 4u * total + n + 15u) & ~15u;
}

// (1) limb counts: CTA (256 coefficients, curve); partial (max nonzero index + 1, limb sum)
__global__ void __launch_bounds__(256) k_pack_size(const uint32_t* __restrict__ out, int D, int W,
                                                   uint32_t* __restrict__ nl, uint32_t* __restrict__ part) {
  __shared__ int s_max[8];
  __shared__ unsigned long long s_sum[8];
  const int b = blockIdx.y, tid = threadIdx.x;
  const int j = blockIdx.x * blockDim.x + tid;
  int jmax = -1;
  unsigned long long sum = 0;
  if (j < D) {
    const uint32_t* rec = out + (static_cast<size_t>(b) * D + j) * W;
    int n = W - 1;
    while (n > 0 && rec[n] == 0u) --n;
    const int v = rec[0] != 0u ? n : 0;
    nl[static_cast<size_t>(b) * D + j] = static_cast<uint32_t>(v);
    if (v) jmax = j;
    sum = static_cast<unsigned long long>(v);
  }
  for (int o = 16; o; o >>= 1) {
    jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((tid & 31) == 0) {
    s_max[tid >> 5] = jmax;
    s_sum[tid >> 5] = sum;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) {
      jmax = max(jmax, s_max[w]);
      sum += s_sum[w];
    }
    uint32_t* pp = part + 2 * (static_cast<size_t>(b) * gridDim.x + blockIdx.x);
    pp[0] = static_cast<uint32_t>(jmax + 1);
    pp[1] = static_cast<uint32_t>(sum);
  }
}

// (2) per curve: n_coeffs, total limbs (limbs beyond the last nonzero coefficient are 0) and the
//     block's byte offset (blocks back to back in curve order)
__global__ void k_pack_offsets(int B, int nblk, const uint32_t* __restrict__ part, uint32_t* __restrict__ meta) {
  uint32_t off = 0;
  for (int b = 0; b < B; ++b) {
    uint32_t n = 0, total = 0;
    for (int q = 0; q < nblk; ++q) {
      n = max(n, part[2 * (b * nblk + q)]);
      total += part[2 * (b * nblk + q) + 1];
    }
    meta[4 * b] = n;
    meta[4 * b + 1] = total;
    meta[4 * b + 2] = off;
    off += pack_block_bytes(n, total);
  }
  meta[4 * B] = off;
}

// (3) per curve: header, limb_off (exclusive scan of the counts) and the sign bytes
__global__ void __launch_bounds__(256) k_pack_index(const uint32_t* __restrict__ out, int D, int W,
                                                    const uint32_t* __restrict__ nl, const uint32_t* __restrict__ meta,
                                                    uint8_t* __restrict__ pk) {
  __shared__ uint32_t s_wsum[8];
  __shared__ uint32_t s_carry;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = meta[4 * b], total = meta[4 * b + 1];
  uint8_t* base = pk + meta[4 * b + 2];
  uint32_t* loff = reinterpret_cast<uint32_t*>(base + 16);
  int8_t* sg = reinterpret_cast<int8_t*>(loff + n + 1 + total);
  const uint32_t* nlb = nl + static_cast<size_t>(b) * D;
  if (tid < 4) reinterpret_cast<uint32_t*>(base)[tid] = 0u;
  if (tid == 0) s_carry = 0u;
  __syncthreads();
  for (uint32_t j0 = 0; j0 < n; j0 += blockDim.x) {
    const uint32_t j = j0 + tid;
    const uint32_t v = j < n ? nlb[j] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t before = s_carry;
    for (int w = 0; w < warp; ++w) before += s_wsum[w];
    if (j < n) {
      loff[j] = before + x - v;
      sg[j] = v ? static_cast<int8_t>(static_cast<int32_t>(out[(static_cast<size_t>(b) * D + j) * W])) : static_cast<int8_t>(0);
    }
    __syncthreads();
    if (tid == blockDim.x - 1) s_carry = before + x;
    __syncthreads();
  }
  if (tid == 0) loff[n] = total;
}

// (4) limbs: a warp per coefficient over the whole grid, lanes along the limbs (coalesced)
__global__ void __launch_bounds__(256) k_pack_copy(const uint32_t* __restrict__ out, int D, int W,
                                                   const uint32_t* __restrict__ nl, const uint32_t* __restrict__ meta,
                                                   uint8_t* __restrict__ pk) {
  const int b = blockIdx.y, lane = threadIdx.x & 31;
  const uint32_t j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const uint32_t n = meta[4 * b];
  if (j >= n) return;
  const uint32_t* loff = reinterpret_cast<const uint32_t*>(pk + meta[4 * b + 2] + 16);
  uint32_t* limbs = reinterpret_cast<uint32_t*>(pk + meta[4 * b + 2] + 16) + n + 1;
  const uint32_t o = loff[j], c = nl[static_cast<size_t>(b) * D + j];
  const uint32_t* rec = out + (static_cast<size_t>(b) * D + j) * W + 1;
  for (uint32_t l = lane; l < c; l += 32) limbs[o + l] = rec[l];
}

// (1-3) in one CTA for a single curve (the latency path: one launch instead of three small
// ones): limb counts, n_coeffs / total / offset, header, limb_off (block scan) and sign bytes.
__global__ void __launch_bounds__(1024) k_pack_one(const uint32_t* __restrict__ out, int D, int W,
                                                   uint32_t* __restrict__ nl, uint32_t* __restrict__ meta,
                                                   uint8_t* __restrict__ pk) {
  __shared__ uint32_t s_w[32];
  __shared__ int s_max[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // pass 1: counts and the last nonzero coefficient
  int jmax = -1;
  for (int j = tid; j < D; j += blockDim.x) {
    const uint32_t* rec = out + static_cast<size_t>(j) * W;
    int n = W - 1;
    while (n > 0 && rec[n] == 0u) --n;
    const int v = rec[0] != 0u ? n : 0;
    nl[j] = static_cast<uint32_t>(v);
    if (v) jmax = j;
  }
  for (int o = 16; o; o >>= 1) jmax = max(jmax, __shfl_xor_sync(0xffffffffu, jmax, o));
  if (lane == 0) s_max[warp] = jmax;
  if (tid == 0) s_carry = 0u;
  __syncthreads();
  if (tid == 0)
    for (int w = 1; w < nw; ++w) s_max[0] = max(s_max[0], s_max[w]);
  __syncthreads();
  const uint32_t n = static_cast<uint32_t>(s_max[0] + 1);
  uint32_t* loff = reinterpret_cast<uint32_t*>(pk + 16);
  if (tid < 4) reinterpret_cast<uint32_t*>(pk)[tid] = 0u;
  // pass 2: exclusive scan of the counts -> limb_off; the sign bytes go after the limbs, so
  // they are written once the total is known (pass 3)
  for (uint32_t j0 = 0; j0 < n; j0 += blockDim.x) {
    const uint32_t j = j0 + tid;
    const uint32_t v = j < n ? nl[j] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t before = s_carry;
    for (int w = 0; w < warp; ++w) before += s_w[w];
    if (j < n) loff[j] = before + x - v;
    __syncthreads();
    if (tid == blockDim.x - 1) s_carry = before + x;
    __syncthreads();
  }
  const uint32_t total = s_carry;
  if (tid == 0) {
    loff[n] = total;
    meta[0] = n;
    meta[1] = total;
    meta[2] = 0u;
    meta[4] = pack_block_bytes(n, total);
  }
  int8_t* sg = reinterpret_cast<int8_t*>(loff + n + 1 + total);
  for (uint32_t j = tid; j < n; j += blockDim.x)
    sg[j] = nl[j] ? static_cast<int8_t>(static_cast<int32_t>(out[static_cast<size_t>(j) * W])) : static_cast<int8_t>(0);
}

int launch_pack(const uint32_t* d_out, int B, int D, int W, uint32_t* d_nl, uint32_t* d_meta, uint8_t* d_pk,
                cudaStream_t st) {
  if (B == 0) return 0;
  if (B == 1) {  // single curve: counts, offsets and index in one CTA, then the copy
    k_pack_one<<<1, 1024, 0, st>>>(d_out, D, W, d_nl, d_meta, d_pk);
    k_pack_copy<<<dim3((D + 7) / 8, 1), 256, 0, st>>>(d_out, D, W, d_nl, d_meta, d_pk);
    return 2;
  }
  const int nblk = (D + 255) / 256;
  uint32_t* part = d_meta + 4 * (static_cast<size_t>(B) + 1);  // [B][nblk][2] after the meta
  k_pack_size<<<dim3(nblk, B), 256, 0, st>>>(d_out, D, W, d_nl, part);
  k_pack_offsets<<<1, 1, 0, st>>>(B, nblk, part, d_meta);
  k_pack_index<<<B, 256, 0, st>>>(d_out, D, W, d_nl, d_meta, d_pk);
  k_pack_copy<<<dim3((D + 7) / 8, B), 256, 0, st>>>(d_out, D, W, d_nl, d_meta, d_pk);
  return 4;
}

size_t pack_meta_words(int B, int D) { return 4 * (static_cast<size_t>(B) + 1) + 2 * static_cast<size_t>(B) * ((D + 255) / 256); }

size_t pack_bytes_bound(int B, int D, int W) {
  return static_cast<size_t>(B) * ((16u + 4u * (static_cast<size_t>(D) + 1) + 4u * static_cast<size_t>(D) * (W - 1) + D + 15u) & ~static_cast<size_t>(15));
}

// 2D u8 tensor map (K-major rows of `kbytes` bytes), SWIZZLE_128B boxes of 128 B x box_rows.
static bool make_u8_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t kbytes, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&f), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return f;
  }();
  if (!fn) return false;
  cuuint64_t dims[2] = {kbytes, rows};
  cuuint64_t strides[1] = {kbytes};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(tma::kBK), box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The CRT product as ONE TMA-fed tcgen05 GEMM over every curve of the batch:
// cols[Rp/128][L8p/4][128] (int4) = Yt[Rp][Kp] x Bt8[L8p][Kp]^T.
template <int BN>
static bool launch_gemm_tma(const CrtParams& cp, cudaStream_t st) {
  CUtensorMap ta, tb;
  const uint64_t rows = static_cast<uint64_t>(cp.Rp);
  if (!make_u8_map(&ta, cp.Y, rows, cp.Kp, tma::kBM) || !make_u8_map(&tb, cp.Bt8, cp.L8p, cp.Kp, BN)) return false;
  static const bool attr = [] {
    return cudaFuncSetAttribute(tma::k_gemm_u8_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(tma::smem_bytes<BN>())) == cudaSuccess;
  }();
  if (!attr) return false;
  tma::k_gemm_u8_tma<BN><<<dim3(cp.L8p / BN, static_cast<unsigned>(rows / tma::kBM)), 128, tma::smem_bytes<BN>(), st>>>(
      ta, tb, reinterpret_cast<int4*>(cp.cols), cp.Rp, cp.Kp);
  return true;
}

// prep_t -> tcgen05 GEMM with the carry in its epilogue -> k_crt_fixup (false: not applicable).
// Two pipeline stages (96 / 64 KB of shared memory: 2 / 3 CTAs per SM, so one CTA's serial
// carry epilogue overlaps another's TMA + MMA) unless CTG_CRT_STAGES=4.
template <int BN, int ST>
static bool launch_crt_fused_st(const CrtParams& cp, cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb,
                                int nt) {
  static const bool attr = [] {
    return cudaFuncSetAttribute(k_gemm_u8_carry<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(tma::smem_bytes<BN, ST>())) == cudaSuccess;
  }();
  if (!attr) return false;
  k_gemm_u8_carry<BN, ST><<<dim3(nt, static_cast<unsigned>(cp.Rp / tma::kBM)), 128, tma::smem_bytes<BN, ST>(), st>>>(
      ta, tb, cp);
  return true;
}

template <int BN>
static bool launch_crt_fused(const CrtParams& cp, cudaStream_t st) {
  const int nt = cp.L8p / BN;
  if (cp.L8p % BN || nt > kCrtMaxTiles) return false;
  CUtensorMap ta, tb;
  const uint64_t rows = static_cast<uint64_t>(cp.Rp);
  if (!make_u8_map(&ta, cp.Y, rows, cp.Kp, tma::kBM) || !make_u8_map(&tb, cp.Bt8, cp.L8p, cp.Kp, BN)) return false;
  static const int stages = std::getenv("CTG_CRT_STAGES") ? std::atoi(std::getenv("CTG_CRT_STAGES")) : 2;
  const bool ok = stages == 4 ? launch_crt_fused_st<BN, 4>(cp, st, ta, tb, nt) : launch_crt_fused_st<BN, 2>(cp, st, ta, tb, nt);
  if (!ok) return false;
  const long long coeffs = static_cast<long long>(cp.J) * cp.B;
  k_crt_fixup<<<static_cast<unsigned>((coeffs * 32 + 127) / 128), 128, 0, st>>>(cp, nt, BN / 4);
  return true;
}

int launch_crt(const CrtParams& cp, cudaStream_t st) {
  if (cp.J == 0 || cp.B == 0) return 0;
  const int nch = (cp.P + kCrtChunk - 1) / kCrtChunk;
  if (cp.use_i8) {
    k_crt_prep_t<<<dim3((cp.J + 31) / 32, nch, cp.B), dim3(32, 8), 0, st>>>(cp);
    // Default: the carry fused into the tcgen05 GEMM's epilogue (any K).  CTG_CRT_UNFUSED=1:
    // the r1 path (digit matrix to HBM, then the carry walk) for A/B.
    static const bool unfused_forced = std::getenv("CTG_CRT_UNFUSED") && std::getenv("CTG_CRT_UNFUSED")[0] == '1';
    // Few coefficients (single-curve calls: 871 at d30): the fused GEMM has only ~30 CTAs for
    // its serial epilogues, where the unfused GEMM + warp-per-coefficient carry is faster
    // (d30, one curve: 38 vs 30 us); batches take the fused path.
    static const long long fused_min = [] {
      const char* e = std::getenv("CTG_CRT_FUSED_MIN");
      return e ? std::atoll(e) : 4737LL;
    }();
    const bool unfused = unfused_forced || static_cast<long long>(cp.J) * cp.B < fused_min;
    static const int bn_forced = std::getenv("CTG_CRT_BN") ? std::atoi(std::getenv("CTG_CRT_BN")) : 0;  // A/B
    const bool bn256 = bn_forced ? bn_forced == 256 && cp.L8p % 256 == 0 : (cp.L8p % 256 == 0 && cp.L8p / 256 >= 2);
    if (!unfused && (bn256 ? launch_crt_fused<256>(cp, st) : launch_crt_fused<128>(cp, st)))
      return 3;
    // Long K (>= 8 stages): TMA + tcgen05; short K: the mma.sync kernel has less fixed cost.
    bool done = false;
    if (cp.Kp >= 1024) done = (cp.L8p % 256 == 0) ? launch_gemm_tma<256>(cp, st) : launch_gemm_tma<128>(cp, st);
    if (!done) k_crt_gemm_i8<<<dim3(cp.L8p / kI8TileL, cp.Rp / kI8TileJ, 1), 256, 0, st>>>(cp);
    // 4P * 255^2 + 2^25 < 2^31: the per-digit sum fits int32
    const bool wide = static_cast<double>(cp.P) * 4 * 255 * 255 + 33554432.0 >= 2147483648.0;
    const long long coeffs = static_cast<long long>(cp.J) * cp.B;
    static const long long warp_max = [] {  // CTG_CARRY_WARP_MAX: A/B switch
      const char* e = std::getenv("CTG_CARRY_WARP_MAX");
      return e ? std::atoll(e) : 4736LL;
    }();
    if (coeffs <= warp_max) {  // few coefficients: a warp per coefficient
      const unsigned blocks = static_cast<unsigned>((coeffs * 32 + 127) / 128);
      if (wide)
        k_crt_carry_warp<true><<<blocks, 128, 0, st>>>(cp);
      else
        k_crt_carry_warp<false><<<blocks, 128, 0, st>>>(cp);
      return 3;
    }
    const unsigned blocks = static_cast<unsigned>((coeffs + 127) / 128);
    // Coalesced-store tile walk (CRT stage vs the scattered-store walk: d20 / 256 curves 0.246 ->
    // 0.204 ms, d30 / 64 0.326 -> 0.267 ms, d16/1024 / 64 0.486 -> 0.497 ms).
    static const bool seq_forced = std::getenv("CTG_CARRY_SEQ") != nullptr;  // A/B switch
    if (seq_forced) {
      if (wide)
        k_crt_carry_seq<true><<<blocks, 128, 0, st>>>(cp);
      else
        k_crt_carry_seq<false><<<blocks, 128, 0, st>>>(cp);
    } else {
      // limbs loaded per batch (memory-level parallelism of the walk; CTG_CARRY_KB=8 for A/B):
      // 16 vs 8 measured d16/1024 CRT 0.498 -> 0.461 ms, d30 0.268 -> 0.262 ms, d20 equal; 32
      // (255 registers) slower everywhere (scripts/ab_carry_kb.sh)
      static const bool kb8 = [] {
        const char* e = std::getenv("CTG_CARRY_KB");
        return e && std::atoi(e) == 8;
      }();
      if (kb8) {
        if (wide)
          k_crt_carry_tile<true, 8><<<blocks, 128, 0, st>>>(cp);
        else
          k_crt_carry_tile<false, 8><<<blocks, 128, 0, st>>>(cp);
      } else if (wide) {
        k_crt_carry_tile<true, 16><<<blocks, 128, 0, st>>>(cp);
      } else {
        k_crt_carry_tile<false, 16><<<blocks, 128, 0, st>>>(cp);
      }
    }
    return 3;
  }
  k_crt_prep<<<dim3((cp.J + 31) / 32, nch, cp.B), dim3(32, 8), 0, st>>>(cp);
  k_crt_gemm<<<dim3((cp.L16 + 63) / 64, (cp.J + 31) / 32, cp.B), 128, 0, st>>>(cp);
  k_crt_carry<<<(cp.J * cp.B + 3) / 4, 128, 0, st>>>(cp);
  return 3;
}

}  // namespace ctg
