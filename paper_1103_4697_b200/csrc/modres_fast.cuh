// Fast mod-p resultant kernel template (see kernels_res.cu for the pipeline).
// Included by fast_g*.cu, each of which instantiates the degrees of one group.
#pragma once
#include <cstdlib>

#include "res_common.cuh"

namespace ctg {
namespace {

// ---------------------------------------------------------------------------
// K2+K3 fast path: deg_y p = NN, deg_y q = NN - 1 (the res(f, f_y) shape).
//
// Division-free Euclid on A (deg k+1), B (deg k):
//   A1 = b_k A - a_{k+1} y B,   r' = b_k A1 - A1_k B = b_k^2 (A mod B)
//   res(A, B) = res(B, r') / b_k^(2k-2)
// so res = r'_0 / E^2 with E = prod_{k=2}^{NN-1} b_k^(k-1), accumulated as
// U <- U b_k, E <- E U.  Both half-steps are fused into ONE pass over the coefficients,
//   r'_i = (b_k^2) a_i + (-b_k a_{k+1}) b_{i-1} + (-A1_k) b_i,
// a three-product sum with a single Montgomery reduction (mmul3: valid for p < 2^30.4,
// the resultant's prime window): 3 IMAD.WIDE + IMAD + IMAD.HI per coefficient instead of
// two two-product reductions.  Any vanishing leading coefficient (a degree drop mod p,
// or a formal leading coefficient vanishing at the point) flags the unit for the exact
// general kernel.  All arrays live in registers (fully unrolled).
// ---------------------------------------------------------------------------
// Resident blocks per SM requested from ptxas (caps registers at 65536 / (128 * minB)).
constexpr int fast_min_blocks(int n) { return n <= 12 ? 8 : n <= 20 ? 6 : n <= 26 ? 5 : n <= 32 ? 4 : 3; }

// Montgomery's batch inversion across the CTA (blockDim = 128, all threads call it): returns
// 1/d for every thread's d (nonzero; threads with nothing to invert pass M.one).  In-warp
// prefix / suffix products by shuffles, one Fermat inversion of the CTA product by thread 0,
// then 1/d_i = 1/T * (product of all others): ~13 multiplications per unit instead of the
// ~45 of a Fermat inversion per unit (the SIMT lanes would each run their own).
__device__ __forceinline__ uint32_t cta_batch_inverse(uint32_t d, const Mod& M) {
  constexpr int kWarps = 4;
  __shared__ uint32_t s_w[kWarps], s_c[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t pf = d, sf = d;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, pf, off);
    const uint32_t c = __shfl_down_sync(0xffffffffu, sf, off);
    if (lane >= off) pf = mmul(pf, a, M);
    if (lane + off < 32) sf = mmul(sf, c, M);
  }
  if (lane == 31) s_w[warp] = pf;
  uint32_t pe = __shfl_up_sync(0xffffffffu, pf, 1), se = __shfl_down_sync(0xffffffffu, sf, 1);
  if (lane == 0) pe = M.one;
  if (lane == 31) se = M.one;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t T = M.one;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) T = mmul(T, s_w[w], M);
    const uint32_t inv = minv(T, M);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      uint32_t c = inv;
#pragma unroll
      for (int v = 0; v < kWarps; ++v)
        if (v != w) c = mmul(c, s_w[v], M);
      s_c[w] = c;
    }
  }
  __syncthreads();
  return mmul(mmul(s_c[warp], pe, M), se, M);
}

// The fused division-free Euclid on A (deg NN), B (deg NN - 1) in registers; returns the
// numerator of res(A, B) and its (nonzero unless flagged) denominator through den_out (EQ:
// the caller's pre-elimination folded in via bn).  flag != 0 marks a degree drop (the unit
// goes to the exact general kernel).
template <int NN, bool EQ>
__device__ __forceinline__ uint32_t fast_euclid(uint32_t (&A)[NN + 1], uint32_t (&B)[NN + 1], uint32_t bn,
                                                uint32_t& flag, const Mod& M, uint32_t& den_out) {
  flag |= (A[NN] == 0u) | (B[NN - 1] == 0u);
  uint32_t U = M.one, E = M.one;
#pragma unroll
  for (int kk = NN - 1; kk >= 1; --kk) {
    const uint32_t bk = B[kk];
    const uint32_t na = mneg(A[kk + 1], M.p);
    const uint32_t c1 = mmul(bk, bk, M);                                          // b_k^2
    const uint32_t c2 = mmul(bk, na, M);                                          // -b_k a_{k+1}
    const uint32_t c3 = mneg(mmul2(bk, A[kk], na, kk >= 1 ? B[kk - 1] : 0u, M), M.p);  // -A1_k
    A[0] = mmul2(c1, A[0], c3, B[0], M);
#pragma unroll
    for (int t = 1; t < kk; ++t) A[t] = mmul3(c1, A[t], c2, B[t - 1], c3, B[t], M);
    flag |= (A[kk - 1] == 0u);
    U = mmul(U, bk, M);
    if (kk >= 2) E = mmul(E, U, M);
#pragma unroll
    for (int t = 0; t <= kk; ++t) {
      const uint32_t tmp = A[t];
      A[t] = B[t];
      B[t] = tmp;
    }
  }
  uint32_t den = mmul(E, E, M);
  if constexpr (EQ) den = mmul(den, mpow(bn, NN - 1, M), M);
  den_out = den;
  uint32_t num = B[0];
  if constexpr (EQ && (NN & 1)) num = mneg(num, M.p);
  return num;
}

// ---------------------------------------------------------------------------
// Hybrid arithmetic for the Euclid's coefficient updates (K3, NN <= kHybMaxDeg).
// Values are PLAIN residues kept as signed int32 in [-0.51 p, 0.51 p] together with their
// double copies.  r = x1 y1 + x2 y2 + x3 y3 mod p:
//   u = x1 (y1/p) + x2 (y2/p) + x3 (y3/p) + (1.5*2^44 + 1/2)      3 DFMA (FP64 pipe)
//   q = floor(S/p + 1/2) = bits [8, 40) of u                        1 SHF (ALU)
//   r = x1 y1 + x2 y2 + x3 y3 - q p  in wrapping int32               4 IMAD (plain, full rate)
// The y_i/p are per-step scalars (one DMUL each).  u carries 2^-8 granularity, so three
// roundings move it by < 0.006 and |r| <= 0.51 p < 2^31 for p < 2^30.4 (the resultant's prime
// window): the representation is closed under the update.  Plain IMAD co-issues with DFMA,
// whereas the Montgomery form's IMAD.WIDE / IMAD.HI occupy the same wide multiplier as FP64:
// measured on B200 (scripts/pipes_bench.cu, fully unrolled rows) 8.4 vs 6.5 three-product
// updates per clock per SM.  r == 0 iff r = 0 mod p (|r| < p), so the degree-drop flags are
// unchanged.  (u never leaves [2^44, 2^45): |S/p| < 0.8 p < 2^43.)
// ---------------------------------------------------------------------------
constexpr int kHybMaxDeg = 32;          // 6 (NN + 1) registers of coefficients: <= 200 at NN = 32
constexpr double kHybMagic = 26388279066624.5;  // 1.5 * 2^44 + 1/2
struct HMod {
  int32_t negp;
  double pinv;
};
__device__ __forceinline__ int32_t hyb_q(double u) {
  return static_cast<int32_t>(__funnelshift_r(static_cast<uint32_t>(__double2loint(u)),
                                              static_cast<uint32_t>(__double2hiint(u)), 8));
}
// exact int32 -> double: 2^52 + 2^31 + r has r + 2^31 as its low mantissa word
__device__ __forceinline__ double hyb_d(int32_t r) {
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int32_t>(static_cast<uint32_t>(r) ^ 0x80000000u)),
                   4503601774854144.0);
}
__device__ __forceinline__ int32_t hmul1(int32_t x, double xd, int32_t y, double ty, const HMod& H) {
  return x * y + hyb_q(__fma_rn(xd, ty, kHybMagic)) * H.negp;
}
__device__ __forceinline__ int32_t hmul2(int32_t x1, double x1d, int32_t y1, double t1, int32_t x2, double x2d,
                                         int32_t y2, double t2, const HMod& H) {
  const double u = __fma_rn(x2d, t2, __fma_rn(x1d, t1, kHybMagic));
  return x1 * y1 + x2 * y2 + hyb_q(u) * H.negp;
}
__device__ __forceinline__ int32_t hmul3(int32_t x1, double x1d, int32_t y1, double t1, int32_t x2, double x2d,
                                         int32_t y2, double t2, int32_t x3, double x3d, int32_t y3, double t3,
                                         const HMod& H) {
  const double u = __fma_rn(x3d, t3, __fma_rn(x2d, t2, __fma_rn(x1d, t1, kHybMagic)));
  return x1 * y1 + x2 * y2 + x3 * y3 + hyb_q(u) * H.negp;
}
// Montgomery [0, p) -> plain symmetric, and back
__device__ __forceinline__ int32_t hyb_from_mont(uint32_t x, const Mod& M) {
  const uint32_t v = from_mont(x, M);
  return v > (M.p >> 1) ? static_cast<int32_t>(v - M.p) : static_cast<int32_t>(v);
}
__device__ __forceinline__ uint32_t hyb_to_mont(int32_t x, const Mod& M) {
  const uint32_t v = x < 0 ? static_cast<uint32_t>(x + static_cast<int32_t>(M.p)) : static_cast<uint32_t>(x);
  return to_mont(v, M);
}

// fast_euclid in the hybrid arithmetic: same recurrence, same flags, same outputs (Montgomery
// numerator and denominator) from the same Montgomery inputs.
template <int NN, bool EQ>
__device__ __forceinline__ uint32_t fast_euclid_h(const uint32_t (&Am)[NN + 1], const uint32_t (&Bm)[NN + 1],
                                                  uint32_t bn, uint32_t& flag, const Mod& M, uint32_t& den_out) {
  const HMod H{-static_cast<int32_t>(M.p), 1.0 / static_cast<double>(M.p)};
  int32_t A[NN + 1], B[NN + 1];
  double Ad[NN + 1], Bd[NN + 1];
#pragma unroll
  for (int j = 0; j <= NN; ++j) {
    A[j] = hyb_from_mont(Am[j], M);
    Ad[j] = hyb_d(A[j]);
  }
#pragma unroll
  for (int j = 0; j < NN; ++j) {
    B[j] = hyb_from_mont(Bm[j], M);
    Bd[j] = hyb_d(B[j]);
  }
  B[NN] = 0;
  Bd[NN] = 0.0;
  flag |= (A[NN] == 0) | (B[NN - 1] == 0);
  // Step scalars on the integer pipe (Montgomery), coefficient updates in the hybrid form.
  // mmul of plain residues carries R^-1: the scalars are c_i R^-1, so each step's new
  // remainder is R^-1 r' and res(B, r') = R^kk res(B, R^-1 r'): the result picks up
  // R^(NN (NN - 1) / 2), folded into the numerator at the end.  U, E are in Montgomery form
  // of the true products (b_k enters through mmul(b_k, R^2) = b_k R).
  uint32_t U = M.one, E = M.one;
  auto u32 = [&](int32_t x) { return x < 0 ? static_cast<uint32_t>(x + static_cast<int32_t>(M.p)) : static_cast<uint32_t>(x); };
#pragma unroll
  for (int kk = NN - 1; kk >= 1; --kk) {
    const uint32_t ub = u32(B[kk]), una = u32(-A[kk + 1]);
    const uint32_t c1 = mmul(ub, ub, M);                                             // b_k^2 R^-1
    const uint32_t c2 = mmul(ub, una, M);                                            // -b_k a_{k+1} R^-1
    const uint32_t c3 = mneg(mmul2(ub, u32(A[kk]), una, u32(B[kk - 1]), M), M.p);    // -A1_k R^-1
    const int32_t i1 = static_cast<int32_t>(c1), i2 = static_cast<int32_t>(c2), i3 = static_cast<int32_t>(c3);
    const double t1 = hyb_d(i1) * H.pinv, t2 = hyb_d(i2) * H.pinv, t3 = hyb_d(i3) * H.pinv;
    A[0] = hmul2(A[0], Ad[0], i1, t1, B[0], Bd[0], i3, t3, H);
    Ad[0] = hyb_d(A[0]);
#pragma unroll
    for (int t = 1; t < kk; ++t) {
      A[t] = hmul3(A[t], Ad[t], i1, t1, B[t - 1], Bd[t - 1], i2, t2, B[t], Bd[t], i3, t3, H);
      Ad[t] = hyb_d(A[t]);
    }
    flag |= (A[kk - 1] == 0);
    U = mmul(U, mmul(ub, M.r2, M), M);
    if (kk >= 2) E = mmul(E, U, M);
#pragma unroll
    for (int t = 0; t <= kk; ++t) {
      const int32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
      const double y = Ad[t];
      Ad[t] = Bd[t];
      Bd[t] = y;
    }
  }
  uint32_t den = mmul(E, E, M);
  if constexpr (EQ) den = mmul(den, mpow(bn, NN - 1, M), M);
  den_out = den;
  // R^(NN (NN - 1) / 2) in Montgomery form: r2 is the Montgomery form of R
  uint32_t num = mmul(hyb_to_mont(B[0], M), mpow(M.r2, NN * (NN - 1) / 2, M), M);
  if constexpr (EQ && (NN & 1)) num = mneg(num, M.p);
  return num;
}

//
// EQ = true: deg_y p = deg_y q = NN (e.g. Q = res(f_x, f_y) of a curve whose y^n
// coefficient is constant).  One extra elimination A' = b_n A - a_n B (deg NN - 1) reduces
// it to the shape above:  res(A, B) = (-1)^NN b_n^-(NN-1) res(B, A')  (A = (a_n/b_n) B + A'/b_n).
template <int NN, bool EQ, bool HYB>
__global__ void __launch_bounds__(128) k_modres_fast(ResParams P) {
  const int kl = blockIdx.y, b = blockIdx.z;
  const int k = P.k0 + kl;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // Threads past the last point (N < 128 or not a multiple of it) redo point N - 1 and stay
  // in the CTA for the batch inversion; they store nothing.
  const bool active = i < P.N;
  const int ic = active ? i : P.N - 1;
  const PrimeConst pcv = P.pc[k];
  const Mod M = load_mod(pcv);

  // Point values p_j(omega^i) (and q_j) from the K2 evaluation kernel: row j of this
  // prime's block, column i -- consecutive threads read consecutive words.
  const uint32_t* vals = P.vals + (static_cast<size_t>(b) * P.nk + kl) * P.nrows * P.N + ic;
  uint32_t A[NN + 1], B[NN + 1];
  uint32_t flag = 0u, bn = 0u;
  if constexpr (EQ) {
#pragma unroll
    for (int j = 0; j <= NN; ++j) B[j] = vals[static_cast<size_t>(j) * P.N];            // p
#pragma unroll
    for (int j = 0; j <= NN; ++j) A[j] = vals[static_cast<size_t>(NN + 1 + j) * P.N];   // q
    // (A, B) <- (q, b_n p - a_n q) with a_n = lc p, b_n = lc q
    const uint32_t an = B[NN];
    bn = A[NN];
    flag = (an == 0u) | (bn == 0u);
    const uint32_t nan = mneg(an, M.p);
#pragma unroll
    for (int j = 0; j < NN; ++j) B[j] = mmul2(bn, B[j], nan, A[j], M);
  } else {
#pragma unroll
    for (int j = 0; j <= NN; ++j) A[j] = vals[static_cast<size_t>(j) * P.N];
    if (P.deriv) {
      uint32_t c = M.one;
#pragma unroll
      for (int j = 0; j < NN; ++j) {
        B[j] = mmul(A[j + 1], c, M);
        c = madd(c, M.one, M.p);
      }
    } else {
#pragma unroll
      for (int j = 0; j < NN; ++j) B[j] = vals[static_cast<size_t>(NN + 1 + j) * P.N];
    }
  }

  uint32_t den, num;
  if constexpr (HYB)
    num = fast_euclid_h<NN, EQ>(A, B, bn, flag, M, den);
  else
    num = fast_euclid<NN, EQ>(A, B, bn, flag, M, den);
  const uint32_t inv = cta_batch_inverse(flag ? M.one : den, M);
  if (!active) return;
  uint32_t* out = P.rows + b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch;
  if (flag) {
    out[i] = kSentinel;
    push_flag(P, (static_cast<uint32_t>(b) * P.nk + kl) * P.N + i);
  } else {
    out[i] = mmul(num, inv, M);
  }
}

// ---------------------------------------------------------------------------
// Fused K2+K3 for res(f, f_y) (deg_y q = NN - 1, q = dp/dy, rows of <= LP slots).
// CTA = (tile of TU = 128 / LP cosets, prime, curve): 128 points {u + K v : u in tile, v < LP}.
//   phase 1: thread (row r, coset u) evaluates row r at the tile's LP points of coset u by
//            one LP-point NTT in registers (coset_ntt, as K2) and stores them to shared
//            memory sv[r][v * TU + (u - u0)] (row stride 128 + TU: conflict-free stores);
//   phase 2: thread i runs the Euclid of K3 on its point's NN + 1 values sv[.][i].
// The [B][P][NN+1][N] point-value array of the two-kernel path (K2 store + K3 load, 8 (NN+1)
// bytes of HBM traffic per unit) is never materialised.
// ---------------------------------------------------------------------------
constexpr int fused_min_blocks(int n) { return n <= 24 ? 8 : n <= 32 ? 6 : 4; }
template <int NN>
__global__ void __launch_bounds__(128, fused_min_blocks(NN)) k_modres_fused(ResParams P, int K) {
  constexpr int LP = coset_lp(NN + 1), LG = ilog2_c(LP), TU = 128 / LP, RS = 128 + TU;
  __shared__ uint32_t sv[(NN + 1) * RS];
  __shared__ uint32_t tw[LP / 2];
  const int kl = blockIdx.y, b = blockIdx.z;
  const int k = P.k0 + kl;
  const int u0 = blockIdx.x * TU;
  const PrimeConst pcv = P.pc[k];
  const Mod M = load_mod(pcv);
  const uint32_t* tab = P.tab + b * P.tab_bstride + static_cast<size_t>(k) * P.S;
  const uint32_t* twr = P.twinv + static_cast<size_t>(k) * P.N;
  load_coset_twiddles<LP>(tw, twr, P.N, K, M);
  __syncthreads();
  {
    const int r = threadIdx.x / TU, uu = threadIdx.x - r * TU, u = u0 + uu;
    if (r <= NN && u < K) {
      uint32_t a[LP];
      coset_ntt<LP, LG>(tab + P.dir[r], P.dir[NN + 1 + r], u ? __ldg(&twr[P.N - u]) : M.one, tw, M, a);
#pragma unroll
      for (int j = 0; j < LP; ++j) sv[r * RS + bitrev_c(j, LG) * TU + uu] = a[j];
    }
  }
  __syncthreads();
  const int uu = threadIdx.x % TU, v = threadIdx.x / TU, u = u0 + uu;
  const bool active = u < K;  // inactive threads redo the tile's first coset (batch inversion)
  const int i = u + K * v;    // the point omega^i of this thread
  uint32_t A[NN + 1], B[NN + 1];
  const int col = active ? threadIdx.x : v * TU;
#pragma unroll
  for (int j = 0; j <= NN; ++j) A[j] = sv[j * RS + col];
  {
    uint32_t c = M.one;
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      B[j] = mmul(A[j + 1], c, M);
      c = madd(c, M.one, M.p);
    }
  }
  uint32_t flag = 0u, den;
  const uint32_t num = fast_euclid<NN, false>(A, B, 0u, flag, M, den);
  const uint32_t inv = cta_batch_inverse(flag ? M.one : den, M);
  if (!active) return;
  uint32_t* out = P.rows + b * P.rows_bstride + static_cast<size_t>(kl) * P.pitch;
  if (flag) {
    out[i] = kSentinel;
    push_flag(P, (static_cast<uint32_t>(b) * P.nk + kl) * P.N + i);
  } else {
    out[i] = mmul(num, inv, M);
  }
}

template <int NN>
void launch_fused_n(const ResParams& rp, cudaStream_t st) {
  constexpr int LP = coset_lp(NN + 1), TU = 128 / LP;
  const int K = rp.N / LP;
  dim3 grid((K + TU - 1) / TU, rp.nk, rp.B);
  k_modres_fused<NN><<<grid, 128, 0, st>>>(rp, K);
}

template <int G, int NN>
bool dispatch_fused(int n, const ResParams& rp, cudaStream_t st) {
  if constexpr (NN > kFastMaxDeg) {
    return false;
  } else {
    if constexpr (fast_group_of(NN) == G) {
      if (n == NN) {
        launch_fused_n<NN>(rp, st);
        return true;
      }
    }
    return dispatch_fused<G, NN + 1>(n, rp, st);
  }
}

// K3 runs the all-Montgomery Euclid; CTG_K3_HYB=1 selects the hybrid FP64/IMAD Euclid
// (fast_euclid_h: parity-tested in tests/test_resultant_gpu.py::test_k3_hybrid_euclid, measured slower).
inline bool k3_montgomery_only() {
  static const bool v = [] {
    const char* e = std::getenv("CTG_K3_HYB");
    return !(e && e[0] == '1');
  }();
  return v;
}

template <int NN>
void launch_fast_n(const ResParams& rp, cudaStream_t st) {
  dim3 grid((rp.N + 127) / 128, rp.nk, rp.B);
  if constexpr (NN <= kHybMaxDeg) {
    if (!k3_montgomery_only()) {
      if (rp.m == rp.n)
        k_modres_fast<NN, true, true><<<grid, 128, 0, st>>>(rp);
      else
        k_modres_fast<NN, false, true><<<grid, 128, 0, st>>>(rp);
      return;
    }
  }
  if (rp.m == rp.n)
    k_modres_fast<NN, true, false><<<grid, 128, 0, st>>>(rp);
  else
    k_modres_fast<NN, false, false><<<grid, 128, 0, st>>>(rp);
}

template <int G, int NN>
bool dispatch_group(int n, const ResParams& rp, cudaStream_t st) {
  if constexpr (NN > kFastMaxDeg) {
    return false;
  } else {
    if constexpr (fast_group_of(NN) == G) {
      if (n == NN) {
        launch_fast_n<NN>(rp, st);
        return true;
      }
    }
    return dispatch_group<G, NN + 1>(n, rp, st);
  }
}

}  // namespace
}  // namespace ctg

#define CTG_DEFINE_FAST_GROUP(G)                                                                 \
  namespace ctg {                                                                                \
  bool dispatch_fast_group_##G(int n, const ResParams& rp, cudaStream_t st) {                    \
    return dispatch_group<G, 2>(n, rp, st);                                                      \
  }                                                                                              \
  bool dispatch_fused_group_##G(int n, const ResParams& rp, cudaStream_t st) {                   \
    return dispatch_fused<G, 2>(n, rp, st);                                                      \
  }                                                                                              \
  }
