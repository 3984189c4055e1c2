// Launchers of the univariate (gcd / Yun) kernels, kernels_uni.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.hpp"

namespace ctg {

constexpr int kMaxUniDeg = 6000;  // 8 shared-memory polynomial buffers per CTA

size_t modyun_smem(int n);
size_t modgcd_smem(int na, int nb);
int launch_modyun(const uint32_t* tab, int n, const PrimeConst* pc, int nk, int32_t* deg, uint32_t* fac,
                  uint32_t* sqf, cudaStream_t st);
int launch_modgcd(const uint32_t* tabA, int na, const uint32_t* tabB, int nb, const PrimeConst* pc, int nk,
                  int32_t* deg, uint32_t* out, int pitch, cudaStream_t st);
// Bivariate gcd probe: deg[k * npts + j] = deg gcd(f(a_j, y), g(a_j, y)) mod p_k, or -1.
// dir = offf[nf+1], lenf[nf+1], offg[ng+1], leng[ng+1] (slot runs in tab, x ascending).
int launch_bigcd_probe(const uint32_t* tab, int S, const int32_t* dir, int nf, int ng, const PrimeConst* pc,
                       int nk, int npts, int32_t* deg, cudaStream_t st);
int launch_gather_scale(const uint32_t* src, int src_pitch, const int32_t* idx, int rows, int cols,
                        const int32_t* seg_end, int nseg, const uint32_t* scale, const PrimeConst* pc_dst,
                        uint32_t* dst, cudaStream_t st);

}  // namespace ctg
