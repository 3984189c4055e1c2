// sm_100a kernels of the multi-modular resultant (SURVEY.md §2 kernel table):
//
//   K1 k_reduce        multiprecision coefficients -> residues mod each prime (Montgomery form)
//   K2+K3 k_modres_fast<n>  per (prime, point): evaluate p, q at x = omega^i (Horner over the
//                      residue table staged in shared memory) and run a division-free
//                      Euclid on the two univariate images entirely in registers
//   K3' k_modres_general  exact formal-degree resultant (degree drops, zero pivots, any shape)
//                      for the units the fast path flags, or for shapes without a fast template
//   K4 k_interp        inverse mixed-radix NTT (N = r * 2^a) per prime: values -> coefficients
//   K5 k_crt_prep / k_crt_gemm / k_crt_carry  fixed-point CRT:  c = sum_k y_k (M/p_k) - t M
//
// The reference computes the same R = res_y(p, q) by a subresultant PRS over Z[x]
// (/root/reference/proj/src/elim.cpp:95-136); R is unique, so the modular image of
// the Sylvester determinant at every (prime, point) determines it bit-exactly.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.hpp"
#include "res_common.cuh"

namespace ctg {

namespace {

// ---------------------------------------------------------------------------
// K1: reduce multiprecision slots modulo the primes.  limbs are stored limb-major
// ([L][S]) so consecutive threads (slots) read consecutive words.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_reduce(const uint32_t* __restrict__ limbs, const int8_t* __restrict__ sign,
                                                int S, int L, const PrimeConst* __restrict__ pc, int k0,
                                                uint32_t* __restrict__ tab) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = k0 + blockIdx.y;
  if (s >= S) return;
  const Mod M = load_mod(pc[k]);
  uint32_t acc = 0;
  // Horner over limbs from the top: acc <- acc * 2^32 + limb  (in Montgomery form:
  // mmul(acc, R^2) = acc*2^32, mmul(limb, R^2) = limb in Montgomery form).
  for (int l = L - 1; l >= 0; --l) {
    uint32_t v = limbs[static_cast<size_t>(l) * S + s];
    v = v >= 2u * M.p ? v - 2u * M.p : v;  // p > 2^30: v < 4p
    v = csub(v, M.p);
    acc = mmul2(acc, M.r2, v, M.r2, M);
  }
  if (sign[s] < 0) acc = mneg(acc, M.p);
  tab[static_cast<size_t>(k) * S + s] = acc;
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
// degenerate units listed by the fast path.
__global__ void __launch_bounds__(128) k_modres_general(ResParams P, int use_list, uint32_t total_units) {
  const uint32_t count = use_list ? min(P.counters[0], P.flag_cap) : total_units;
  const int nq = P.n + 1;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < count; u += gridDim.x * blockDim.x) {
    const uint32_t unit = use_list ? P.flag_list[u] : u;
    const int kl = static_cast<int>(unit / P.N), i = static_cast<int>(unit % P.N);
    const int k = P.k0 + kl;
    const PrimeConst pcv = P.pc[k];
    const Mod M = load_mod(pcv);
    const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
    const uint32_t* tab = P.tab + static_cast<size_t>(k) * P.S;
    uint32_t bufA[kGeneralMaxDeg + 1], bufB[kGeneralMaxDeg + 1];
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
    P.rows[static_cast<size_t>(kl) * P.pitch + i] = res_general(bufA, P.n, bufB, P.m, M);
  }
}

// ---------------------------------------------------------------------------
// K4: per prime, inverse DFT of size N = r * 2^a over the values R(omega^i):
//   c_j = s * sum_{i1 < r} omega^{-i1 j} u[i1][j mod 2^a],
//   u[i1] = radix-2 inverse NTT (root omega^{-r}) of v[r*i2 + i1],
// with s = +-N^{-1}.  Coefficients j >= D must vanish (degree bound check).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_interp(uint32_t* rows, int pitch, const PrimeConst* __restrict__ pc, int k0,
                                                int N, int r, int a, int D, int negate, uint32_t* counters) {
  extern __shared__ uint32_t sm[];
  uint32_t* tw = sm;      // omega^{-i}, i < N
  uint32_t* w = sm + N;   // work array
  const int kl = blockIdx.x;
  const PrimeConst pcv = pc[k0 + kl];
  const Mod M = load_mod(pcv);
  uint32_t* row = rows + static_cast<size_t>(kl) * pitch;
  const int Mlen = 1 << a;
  const int tid = threadIdx.x, bs = blockDim.x;
  bool bad = false;
  for (int i = tid; i < N; i += bs) {
    tw[i] = mpow(pcv.omega_inv, static_cast<uint64_t>(i), M);
    const uint32_t val = row[i];
    bad |= (val == kSentinel);
    const int i1 = i % r, i2 = i / r;
    const int br = a ? static_cast<int>(__brev(static_cast<uint32_t>(i2)) >> (32 - a)) : 0;
    w[i1 * Mlen + br] = val;
  }
  if (bad) atomicOr(&counters[1], kErrSentinel);
  __syncthreads();
  const int halfM = Mlen >> 1;
  for (int len = 2; len <= Mlen; len <<= 1) {
    const int half = len >> 1, step = Mlen / len;
    for (int b = tid; b < r * halfM; b += bs) {
      const int rw = b / halfM, bb = b % halfM;
      const int g = bb / half, t = bb % half;
      uint32_t* base = w + rw * Mlen + g * len;
      const uint32_t u = base[t];
      const uint32_t v = mmul(base[t + half], tw[r * t * step], M);
      base[t] = madd(u, v, M.p);
      base[t + half] = msub(u, v, M.p);
    }
    __syncthreads();
  }
  bool tail = false;
  for (int j = tid; j < N; j += bs) {
    const int j1 = j & (Mlen - 1);
    uint32_t acc = 0;
    for (int i1 = 0; i1 < r; ++i1) {
      const uint32_t e = static_cast<uint32_t>((static_cast<uint64_t>(i1) * j) % N);
      acc = madd(acc, mmul(w[i1 * Mlen + j1], tw[e], M), M.p);
    }
    uint32_t c = mmul(acc, pcv.scale, M);  // Montgomery x plain -> plain
    if (negate) c = mneg(c, M.p);
    if (j < D)
      row[j] = c;
    else
      tail |= (c != 0u);
  }
  if (tail) atomicOr(&counters[1], kErrNttTail);
}

// ---------------------------------------------------------------------------
// K5: fixed-point CRT.  For coefficient j with residues v_k:
//   y_k = v_k (M/p_k)^{-1} mod p_k,   u = sum_k y_k / p_k,   t = round(u),
//   c = sum_k y_k (M/p_k) - t M      (|c| < M / 2^35 by the choice of primes, so
//   u is within 2^-34 of an integer and the double sum rounds exactly).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_crt_prep(CrtParams C) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int jl = blockIdx.x * 32 + tx;
  double u = 0;
  if (jl < C.J) {
    for (int k = ty; k < C.P; k += 8) {
      const PrimeConst& pcv = C.pc[k];
      const Mod M = load_mod(pcv);
      const uint32_t v = C.rows[static_cast<long long>(k / C.row_block) * C.block_stride +
                                static_cast<long long>(k % C.row_block) * C.pitch + C.j0 + jl];
      const uint32_t y = mmul(v, pcv.crt_c, M);
      C.Y[static_cast<size_t>(k) * C.J + jl] = y;
      u += static_cast<double>(y) * C.minv[k];
    }
  }
  red[ty][tx] = u;
  __syncthreads();
  if (ty == 0 && jl < C.J) {
    double s = 0;
    for (int q = 0; q < 8; ++q) s += red[q][tx];
    const double t = rint(s);
    if (fabs(s - t) > 1e-6) atomicOr(&C.counters[1], kErrCrtRound);
    C.tq[jl] = static_cast<int64_t>(t);
  }
}

// cols[j][l] = sum_k Y[k][j] * Mk16[k][l]  (31-bit x 16-bit products, exact u64 sums)
__global__ void __launch_bounds__(256) k_crt_gemm(CrtParams C) {
  __shared__ __align__(16) uint32_t Ys[16][64];
  __shared__ __align__(16) uint32_t Ms[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int jb = blockIdx.y * 64, lb = blockIdx.x * 64;
  uint64_t acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0;
  for (int k0 = 0; k0 < C.P; k0 += 16) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int kk = e >> 6, c = e & 63;
      const int k = k0 + kk;
      Ys[kk][c] = (k < C.P && jb + c < C.J) ? C.Y[static_cast<size_t>(k) * C.J + jb + c] : 0u;
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
        for (int b = 0; b < 4; ++b) acc[a][b] += static_cast<uint64_t>(ya[a]) * ma[b];
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int j = jb + ty * 4 + a;
    if (j >= C.J) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int l = lb + tx * 4 + b;
      if (l < C.L16) C.cols[static_cast<size_t>(j) * C.L16 + l] = acc[a][b];
    }
  }
}

// Carry propagation (16-bit digits), subtraction of t*M, sign-magnitude output.
__global__ void __launch_bounds__(128) k_crt_carry(CrtParams C) {
  const int jl = blockIdx.x * blockDim.x + threadIdx.x;
  if (jl >= C.J) return;
  const uint64_t* col = C.cols + static_cast<size_t>(jl) * C.L16;
  const int64_t t = C.tq[jl];
  uint32_t* out = C.out + static_cast<size_t>(jl) * (C.out_limbs + 1);
  int64_t carry = 0;
  uint32_t any = 0;
  for (int w = 0; w < C.out_limbs; ++w) {
    uint32_t limb = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int l = 2 * w + h;
      int64_t v = carry;
      if (l < C.L16) v += static_cast<int64_t>(col[l]) - t * static_cast<int64_t>(C.M16[l]);
      limb |= static_cast<uint32_t>(v & 0xffff) << (16 * h);
      carry = v >> 16;
    }
    out[1 + w] = limb;
    any |= limb;
  }
  int sign = any ? 1 : 0;
  if (carry < 0) {
    uint32_t c = 1;
    for (int w = 0; w < C.out_limbs; ++w) {
      const uint64_t s = static_cast<uint64_t>(~out[1 + w]) + c;
      out[1 + w] = static_cast<uint32_t>(s);
      c = static_cast<uint32_t>(s >> 32);
    }
    sign = -1;
  }
  out[0] = static_cast<uint32_t>(sign);
}

}  // namespace

int launch_reduce(const uint32_t* d_limbs, const int8_t* d_sign, int S, int L, const PrimeConst* d_pc, int k0, int nk,
                  uint32_t* d_tab, cudaStream_t st) {
  if (S == 0 || nk == 0) return 0;
  dim3 grid((S + 127) / 128, nk);
  k_reduce<<<grid, 128, 0, st>>>(d_limbs, d_sign, S, L, d_pc, k0, d_tab);
  return 1;
}

int launch_modres(const ResParams& rp, int nk, bool fast, cudaStream_t st) {
  if (nk == 0) return 0;
  if (fast && rp.m == rp.n - 1 && dispatch_fast_any(rp.n, rp, nk, st)) {
    k_modres_general<<<64, 128, 0, st>>>(rp, 1, 0u);
    return 2;
  }
  const uint32_t total = static_cast<uint32_t>(nk) * static_cast<uint32_t>(rp.N);
  const int blocks = static_cast<int>(std::min<uint32_t>((total + 127) / 128, 148u * 16u));
  k_modres_general<<<blocks, 128, 0, st>>>(rp, 0, total);
  return 1;
}

int launch_interp(uint32_t* rows, int pitch, int nk, const PrimeConst* d_pc, int k0, int N, int r, int a, int D,
                  int negate, uint32_t* counters, cudaStream_t st) {
  if (nk == 0) return 0;
  const size_t smem = static_cast<size_t>(2) * N * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_interp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_interp<<<nk, 256, smem, st>>>(rows, pitch, d_pc, k0, N, r, a, D, negate, counters);
  return 1;
}

int launch_crt(const CrtParams& cp, cudaStream_t st) {
  if (cp.J == 0) return 0;
  k_crt_prep<<<(cp.J + 31) / 32, dim3(32, 8), 0, st>>>(cp);
  dim3 g2((cp.L16 + 63) / 64, (cp.J + 63) / 64);
  k_crt_gemm<<<g2, 256, 0, st>>>(cp);
  k_crt_carry<<<(cp.J + 127) / 128, 128, 0, st>>>(cp);
  return 3;
}

}  // namespace ctg
