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

static __device__ __forceinline__ void push_flag(const ResParams& P, uint32_t unit) {
  uint32_t idx = atomicAdd(&P.counters[0], 1u);
  if (idx < P.flag_cap)
    P.flag_list[idx] = unit;
  else
    atomicOr(&P.counters[1], kErrFlagOverflow);
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

}  // namespace ctg
