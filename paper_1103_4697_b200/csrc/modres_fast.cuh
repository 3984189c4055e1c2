// Fast mod-p resultant kernel template (see kernels_res.cu for the pipeline).
// Included by fast_g*.cu, each of which instantiates the degrees of one group.
#pragma once
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
// U <- U b_k, E <- E U.  Any vanishing leading coefficient (a degree drop mod p,
// or a formal leading coefficient vanishing at the point) flags the unit for
// the exact general kernel.  All arrays live in registers (fully unrolled).
// ---------------------------------------------------------------------------
template <int NN>
__global__ void __launch_bounds__(128) k_modres_fast(ResParams P) {
  extern __shared__ uint32_t sm[];
  const int kl = blockIdx.y;
  const int k = P.k0 + kl;
  const PrimeConst pcv = P.pc[k];
  const Mod M = load_mod(pcv);
  uint32_t* s_tab = sm;
  int32_t* s_dir = reinterpret_cast<int32_t*>(sm + P.S);
  constexpr int kDir = 2 * (NN + 1) + 2 * NN;
  for (int s = threadIdx.x; s < P.S; s += blockDim.x) s_tab[s] = P.tab[static_cast<size_t>(k) * P.S + s];
  for (int s = threadIdx.x; s < kDir; s += blockDim.x) s_dir[s] = P.dir[s];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.N) return;

  const uint32_t x = mpow(pcv.omega, static_cast<uint64_t>(i), M);
  uint32_t A[NN + 1], B[NN];
#pragma unroll
  for (int j = 0; j <= NN; ++j) A[j] = horner(s_tab, s_dir[j], s_dir[NN + 1 + j], x, M);
  if (P.deriv) {
    uint32_t c = M.one;
#pragma unroll
    for (int j = 0; j < NN; ++j) {
      B[j] = mmul(A[j + 1], c, M);
      c = madd(c, M.one, M.p);
    }
  } else {
#pragma unroll
    for (int j = 0; j < NN; ++j) B[j] = horner(s_tab, s_dir[2 * (NN + 1) + j], s_dir[2 * (NN + 1) + NN + j], x, M);
  }

  uint32_t flag = (A[NN] == 0u) | (B[NN - 1] == 0u);
  uint32_t U = M.one, E = M.one;
#pragma unroll
  for (int kk = NN - 1; kk >= 1; --kk) {
    const uint32_t bk = B[kk];
    const uint32_t na = mneg(A[kk + 1], M.p);
    A[0] = mmul(bk, A[0], M);
#pragma unroll
    for (int t = 1; t <= kk; ++t) A[t] = mmul2(bk, A[t], na, B[t - 1], M);
    const uint32_t nt = mneg(A[kk], M.p);
#pragma unroll
    for (int t = 0; t < kk; ++t) A[t] = mmul2(bk, A[t], nt, B[t], M);
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
  const uint32_t Ei = minv(E, M);
  const uint32_t res = mmul(B[0], mmul(Ei, Ei, M), M);
  uint32_t* out = P.rows + static_cast<size_t>(kl) * P.pitch;
  if (flag) {
    out[i] = kSentinel;
    push_flag(P, static_cast<uint32_t>(kl) * P.N + i);
  } else {
    out[i] = res;
  }
}

template <int NN>
void launch_fast_n(const ResParams& rp, int nk, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(rp.S) * 4 + static_cast<size_t>(2 * (NN + 1) + 2 * NN) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_modres_fast<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  dim3 grid((rp.N + 127) / 128, nk);
  k_modres_fast<NN><<<grid, 128, smem, st>>>(rp);
}

template <int G, int NN>
bool dispatch_group(int n, const ResParams& rp, int nk, cudaStream_t st) {
  if constexpr (NN > kFastMaxDeg) {
    return false;
  } else {
    if constexpr (fast_group_of(NN) == G) {
      if (n == NN) {
        launch_fast_n<NN>(rp, nk, st);
        return true;
      }
    }
    return dispatch_group<G, NN + 1>(n, rp, nk, st);
  }
}

}  // namespace
}  // namespace ctg

#define CTG_DEFINE_FAST_GROUP(G)                                                                 \
  namespace ctg {                                                                                \
  bool dispatch_fast_group_##G(int n, const ResParams& rp, int nk, cudaStream_t st) {            \
    return dispatch_group<G, 2>(n, rp, nk, st);                                                  \
  }                                                                                              \
  }
