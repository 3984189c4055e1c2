// Launchers of the univariate (gcd / Yun) kernels, kernels_uni.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "internal.hpp"

namespace ctg {

// Per-CTA shared-memory budget of the K6 kernels.  Beyond it (degrees above ~7,000 for Yun)
// the polynomial buffers live in a global scratch region instead: every launcher takes
// `gbuf` (uni_gbuf_bytes(smem bytes, CTAs) bytes, or null when that is 0) and returns -1 if
// it needed one and got none.  No degree limit remains.
constexpr size_t kUniSmemMax = 200 * 1024;
size_t uni_gbuf_bytes(size_t smem, size_t ctas);

size_t modyun_smem(int n);
size_t modgcd_smem(int na, int nb);
size_t bigcd_probe_smem(int nf, int ng);
size_t sqf_probe_smem(int max_deg);
// Batched square-freeness probe: CTA per (problem, prime); out[2 (i nk + k)] = (status, deg gcd(P, P')).
// plain = 1: the table holds plain residues (e.g. a resultant's interpolated rows), else Montgomery.
// small: the primes are probe primes < 2^15 (api_uni.cu select_probe_primes; K1 residues), run with the
// 32-bit Barrett arithmetic of lehmer::SmallA.
int launch_sqf_probe(const uint32_t* tab, int S, const int32_t* off, const int32_t* degs, int nprob, int nk,
                     const PrimeConst* pc, int max_deg, int32_t* out, uint32_t* gbuf, cudaStream_t st, int plain = 0,
                     bool small = false, int single_deg = 0);  // off = degs = null: one problem at 0

// deg gcd(a, b) mod pc[0] (plain residues; method 0 blocked Lehmer, 1 one pass per step) -> out[0].
size_t gcd_degree_smem(int na, int nb);
int launch_gcd_degree(const uint32_t* a, int na, const uint32_t* b, int nb, const PrimeConst* pc, int method,
                      int32_t* out, uint32_t* gbuf, cudaStream_t st, unsigned long long* prof = nullptr);
int launch_modyun(const uint32_t* tab, int n, const PrimeConst* pc, int nk, int32_t* deg, uint32_t* fac,
                  uint32_t* sqf, uint32_t* gbuf, cudaStream_t st);
// tab_pitch: words between the rows of consecutive primes for both operands (0: na + 1 / nb + 1)
// staged_limbs / staged_sign / Lw / rpow: the inputs as staged coefficients ([na + nb + 2][Lw],
// A then B, Lw <= kRedL) reduced inside the kernel (no K1 launch); tabA / tabB are then unused.
int launch_modgcd(const uint32_t* tabA, int na, const uint32_t* tabB, int nb, int tab_pitch, const PrimeConst* pc,
                  int nk, int32_t* deg, uint32_t* out, int pitch, uint32_t* gbuf, cudaStream_t st,
                  const uint32_t* staged_limbs = nullptr, const int8_t* staged_sign = nullptr, int Lw = 0,
                  const uint32_t* rpow = nullptr);
// Bivariate gcd probe: deg[k * npts + j] = deg gcd(f(a_j, y), g(a_j, y)) mod p_k, or -1.
// dir = offf[nf+1], lenf[nf+1], offg[ng+1], leng[ng+1] (slot runs in tab, x ascending).
int launch_bigcd_probe(const uint32_t* tab, int S, const int32_t* dir, int nf, int ng, const PrimeConst* pc,
                       int nk, int npts, int32_t* deg, uint32_t* gbuf, cudaStream_t st);
// Brown images: per (prime k, point off[k] + j): gamma(a) * monic gcd | A/g | B/g (plain, pitch
// words at out[k][j]); deg[k][j] = gcd degree or -2 (gamma(a) = 0).  dir as for the probe;
// gamma is the slot run [gam_off, gam_off + gam_len) of tab.
int launch_bigcd_images(const uint32_t* tab, int S, const int32_t* dir, int na, int nb, int gam_off, int gam_len,
                        const PrimeConst* pc, const uint32_t* offs, int nk, int npts, int32_t* deg, uint32_t* out,
                        int pitch, uint32_t* gbuf, cudaStream_t st);
// Newton interpolation on the points off[k] + j, j < N: src[k][j][c] (pitch src_pitch) ->
// dst[k][t][c] (t < N, row pitch cols) for the rows k = idx[0..rows).
size_t newton_smem(int N);
int launch_newton_interp(const uint32_t* src, int src_pitch, const int32_t* idx, int rows, const PrimeConst* pc,
                         const uint32_t* offs, int N, int cols, uint32_t* dst, uint32_t* gbuf, int gbuf_rows,
                         cudaStream_t st);
constexpr int kNewtonColsPerCta = 32;
int launch_gather_scale(const uint32_t* src, int src_pitch, const int32_t* idx, int rows, int cols,
                        const int32_t* seg_end, int nseg, const uint32_t* scale, const PrimeConst* pc_dst,
                        uint32_t* dst, cudaStream_t st);

}  // namespace ctg
