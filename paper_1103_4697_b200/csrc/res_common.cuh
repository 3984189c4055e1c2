// Device helpers shared by the resultant kernels.
#pragma once
#include "internal.hpp"

namespace ctg {

static __device__ __forceinline__ Mod load_mod(const PrimeConst& c) { return Mod{c.p, c.pneg, c.r2, c.one}; }

// Horner over slots [off, off+len) (slot off+t = coefficient of x^t), Montgomery form.
static __device__ __forceinline__ uint32_t horner(const uint32_t* tab, int off, int len, uint32_t x, const Mod& M) {
  if (len <= 0) return 0u;
  uint32_t acc = tab[off + len - 1];
  for (int t = len - 2; t >= 0; --t) acc = madd(mmul(acc, x, M), tab[off + t], M.p);
  return acc;
}

constexpr int bitrev_c(int t, int lg) {
  int r = 0;
  for (int i = 0; i < lg; ++i) r |= ((t >> i) & 1) << (lg - 1 - i);
  return r;
}

// Coset evaluation of one y-coefficient row (slots c_0..c_{len-1}, len <= LP) at the LP points
// omega^{u + K v}, v < LP (N = K LP):  NTT_LP(c_t omega^{t u})[v]  (Montgomery form).
// Decimation in frequency: natural-order input, output in bit-reversed order, i.e.
// a[j] = value at v = bitrev(j) -- callers fold the permutation into their store addresses,
// so every register-array index stays a compile-time constant (no local-memory arrays).
// x = omega^u; tw = w^e (e < LP/2, w = omega^K of order LP) in shared memory (a broadcast
// read per butterfly, no registers held).  Shared by K2 and the fused K2+K3 kernel.
template <int LP, int LG>
static __device__ __forceinline__ void coset_ntt(const uint32_t* __restrict__ c, int len, uint32_t x,
                                                 const uint32_t* tw, const Mod& M, uint32_t (&a)[LP]) {
  uint32_t xp = M.one;
#pragma unroll
  for (int t = 0; t < LP; ++t) {  // c_t x^t (slots past the row length are zero)
    uint32_t v = 0u;
    if (t < len) {
      v = mmul(c[t], xp, M);
      xp = mmul(xp, x, M);
    }
    a[t] = v;
  }
#pragma unroll
  for (int len2 = LP; len2 >= 2; len2 >>= 1) {
    const int half = len2 >> 1, step = LP / len2;
#pragma unroll
    for (int g = 0; g < LP; g += len2) {
#pragma unroll
      for (int t = 0; t < half; ++t) {
        const uint32_t x0 = a[g + t], x1 = a[g + t + half];
        a[g + t] = madd(x0, x1, M.p);
        a[g + t + half] = t == 0 ? msub(x0, x1, M.p) : mmul(msub(x0, x1, M.p), tw[t * step], M);
      }
    }
  }
}

// Stage the coset twiddles w^e = omega^{K e} (e < LP/2) of one prime in shared memory
// (twr = the prime's omega^{-i} table: omega^j = omega^{-(N - j)}).  Caller syncs.
template <int LP>
static __device__ __forceinline__ void load_coset_twiddles(uint32_t* tw, const uint32_t* __restrict__ twr, int N,
                                                           int K, const Mod& M) {
  for (int e = threadIdx.x; e < LP / 2; e += blockDim.x) tw[e] = e ? __ldg(&twr[N - K * e]) : M.one;
}

// Smallest power of two >= len (>= 4): the coset NTT length for rows of `len` slots.
constexpr int coset_lp(int len) {
  int lp = 4;
  while (lp < len) lp <<= 1;
  return lp;
}
constexpr int ilog2_c(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

static __device__ __forceinline__ void push_flag(const ResParams& P, uint32_t unit) {
  uint32_t idx = atomicAdd(&P.counters[0], 1u);
  if (idx < P.flag_cap) P.flag_list[idx] = unit;  // beyond the cap: k_modres_general scans for kSentinel
}


// Fast-path dispatch: the templates k_modres_fast<n> are split over fast_g*.cu
// (compiled in parallel); each group launches the n it owns.
constexpr int kFastGroups = 8;
constexpr int fast_group_of(int n) {
  const int idx = kFastMaxDeg - n, round = idx / kFastGroups, pos = idx % kFastGroups;
  return (round % 2 == 0) ? pos : kFastGroups - 1 - pos;
}
bool dispatch_fast_group(int group, int n, const ResParams& rp, cudaStream_t st);
inline bool dispatch_fast_any(int n, const ResParams& rp, cudaStream_t st) {
  if (n < 2 || n > kFastMaxDeg) return false;
  return dispatch_fast_group(fast_group_of(n), n, rp, st);
}
// Fused K2+K3 (derivative shape, rows of <= coset_lp(n + 1) slots): rp.vals unused.
bool dispatch_fused_group(int group, int n, const ResParams& rp, cudaStream_t st);
inline bool dispatch_fused_any(int n, const ResParams& rp, cudaStream_t st) {
  if (n < 2 || n > kFastMaxDeg) return false;
  return dispatch_fused_group(fast_group_of(n), n, rp, st);
}

}  // namespace ctg
