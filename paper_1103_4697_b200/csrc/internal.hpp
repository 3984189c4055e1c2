// Internal declarations shared by the host API (api_*.cu) and the kernels.
//
// Every resultant kernel processes a BATCH of B same-shape problems (curves): the
// batch index is blockIdx.z and each per-curve array has a batch stride.  A single
// ctg_resultant call is a batch of one.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/ctg.h"
#include "hostmath.hpp"
#include "modarith.cuh"

namespace ctg {

// Per-prime constants, one 32-byte record per row of the residue matrix.
struct PrimeConst {
  uint32_t p, pneg, r2, one;  // Montgomery constants (modarith.cuh)
  uint32_t omega;             // primitive N-th root of unity, Montgomery form
  uint32_t omega_inv;         // its inverse, Montgomery form
  uint32_t scale;             // N^{-1} mod p, PLAIN (mmul(x_mont, scale) -> plain x*scale)
  uint32_t crt_c;             // ((M / p)^{-1} mod p) in Montgomery form
};

constexpr int kFastMaxDeg = 40;     // fast mod-p resultant templates: deg_y p in [2, kFastMaxDeg], deg_y q = deg_y p - 1
constexpr int kThreadGeneralMax = kFastMaxDeg;  // thread-per-unit formal-degree kernel up to this deg_y;
                                                // above it k_modres_warp (warp per unit, any degree)
constexpr int kWarpsGeneral = 4;                // warps per CTA of k_modres_warp
constexpr size_t kGeneralWarpSmemMax = 200 * 1024;  // beyond: per-warp slices of global scratch
constexpr uint32_t kGeneralWarpGlobalBlocks = 296;
constexpr uint32_t kMaxNttSmem = 1u << 14;  // K4 in shared memory up to this size; beyond, global passes
constexpr uint32_t kSentinel = 0xffffffffu;
constexpr int kCrtChunk = 64;       // primes per partial sum of the CRT rounding estimate
constexpr int kI8TileJ = 128;       // tensor-core CRT GEMM block tile: coefficients
constexpr int kI8TileL = 128;       //                                   byte digits of the output
constexpr int kI8MaxPrimes = 8192;  // s32 exactness: 4P * 255^2 < 2^31
constexpr int kRedL = 64;           // limb powers tabulated per prime for K1 (longer inputs extend on the fly)

// Device error bits (plan counters[1]).
enum : uint32_t {
  kErrFlagOverflow = 1u,   // more degenerate units than the fallback list holds
  kErrNttTail = 2u,        // interpolated coefficient beyond the degree bound is nonzero
  kErrCrtRound = 4u,       // fixed-point CRT estimate not near an integer (bound violated)
  kErrSentinel = 8u,       // an evaluation unit was never resolved
};

struct CrtTables {
  int device = -1;
  uint32_t N = 0;
  int P = 0;
  int LM = 0, L16 = 0;
  std::vector<uint32_t> primes;
  PrimeConst* d_pc = nullptr;
  double* d_minv = nullptr;
  uint32_t* d_Mk16 = nullptr;
  uint32_t* d_M16 = nullptr;
  // tensor-core CRT operands (tables.cu): Bt8 [L8p][Kp] bytes, M8 [L8] byte digits of M
  bool use_i8 = false;
  int L8 = 0, L8p = 0, Kp = 0;
  uint8_t* d_Bt8 = nullptr;
  uint32_t* d_M8 = nullptr;
  uint32_t* d_twinv = nullptr;  // [P][N] omega_k^{-i} (Montgomery), N > 1 only
  uint32_t* d_rpow = nullptr;   // [P][kRedL] R^(l+2) mod p_k (plain): mmul(limb_l, .) = limb_l 2^(32 l) R
  std::vector<PrimeConst> h_pc;
  double log2M = 0;
  ~CrtTables();
};
// Builds the tables for `primes` (in order) on `device`; N = NTT size (1 if unused).
std::shared_ptr<CrtTables> build_tables(int device, const std::vector<uint32_t>& primes, uint32_t N);
// Cached build_tables (per device, N, prime list; least recently used entries beyond 64 are
// dropped).  Building costs device allocations and synchronous copies, so every caller --
// resultant plans, the gcd / Yun images, their CRTs -- goes through the cache.
std::shared_ptr<CrtTables> get_tables(int device, uint32_t N, const std::vector<uint32_t>& primes);

struct ResParams {
  int B;                    // curves in the batch (blockIdx.z)
  const uint32_t* tab;      // [B][P][S] Montgomery residues of the slots (global prime index)
  size_t tab_bstride;       // = P * S
  int S;
  const PrimeConst* pc;     // [P]
  int k0, nk;               // this launch covers primes [k0, k0 + nk)
  uint32_t* rows;           // curve b, prime k: rows + b * rows_bstride + (k - k0) * pitch
  size_t rows_bstride;
  int pitch;
  int N;                    // evaluation points per prime
  int n, m;                 // formal degrees in y (n >= m)
  int deriv;                // q == dp/dy: q_j(x) = (j+1) p_{j+1}(x)
  const int32_t* dir;       // slot directory: off_p[n+1], len_p[n+1], off_q[m+1], len_q[m+1]
  uint32_t* flag_list;      // degenerate units (fast path) -> general kernel
  uint32_t* counters;       // [0] flagged count, [1] error bits
  uint32_t flag_cap;
  uint32_t* vals;           // K2 output: [B][nk][nrows][N] point values (Montgomery); null = no fast path
  int nrows;                // n + 1 (derivative mode) or n + m + 2
  int maxlen;               // longest slot run (max x-degree + 1) over the rows
  const uint32_t* twinv;    // [P][N] omega_k^{-i} (Montgomery; global prime index k)
  int fused;                // K2 folded into the K3 launch (k_modres_fused); vals unused
  uint32_t* gwarp;          // k_modres_warp buffers in global memory (huge deg_y), else null
};
size_t general_warp_smem(int n);
size_t general_warp_gbuf_words(int n);  // 0 when the buffers fit in shared memory

struct CrtParams {
  int B;
  const uint32_t* rows;  // plain residues; curve b, prime k at rows + b * curve_stride
                         //   + (k / row_block) * block_stride + (k % row_block) * pitch
  long long curve_stride;
  int pitch, P;
  int row_block;
  long long block_stride;
  int j0, J;             // coefficient range
  int col0;              // column of coefficient col0 is 0 in each row (a shard's receive block), else 0
  const PrimeConst* pc;
  const double* minv;    // 1/p_k
  const uint32_t* Mk16;  // [P][L16] 16-bit digits of M / p_k
  const uint32_t* M16;   // [L16] 16-bit digits of M
  int L16;
  uint32_t* Y;           // scratch: IMAD path [B][P][J]; tensor path Yt [Rp][Kp/4] (k contiguous)
  double* upart;         // scratch [B][ceil(P / kCrtChunk)][J]: partial sums of y_k / p_k
  uint64_t* cols;        // scratch: IMAD path [B][J][L16] u64; tensor path [Rp/128][L8p/4][128] int4
  uint32_t* out;         // [B][J][out_limbs + 1]
  int out_limbs;
  uint32_t* counters;
  // tensor-core path (use_i8): the GEMM rows are the coefficients of all curves flattened,
  // row (b, j) = b * J + j, padded to Rp = a multiple of kI8TileJ (no per-curve padding: a
  // rank's small coefficient block of a sharded CRT fills its tiles)
  int use_i8;
  int Rp, L8, L8p, Kp;
  const uint8_t* Bt8;
  const uint32_t* M8;
  int top_digit;         // |value| < 2^(8 top_digit) (coefficient bound; L8 when unknown)
};

// Scratch words the CRT needs for J coefficients of B curves (Y and cols).
size_t crt_y_words(const CrtTables& T, int B, int J);
size_t crt_cols_words(const CrtTables& T, int B, int J);  // in 32-bit words

// Kernel launchers (kernels_res.cu).  Each returns the number of launches issued.
// Limbs limb-major [B][L][S] (coef_major = 0) or coefficient-major [B][S][L] (coef_major = 1).
int launch_reduce(const uint32_t* d_limbs, const int8_t* d_sign, int S, int L, const PrimeConst* d_pc,
                  const uint32_t* d_rpow, int k0, int nk, uint32_t* d_tab, size_t tab_bstride, int B, cudaStream_t st,
                  int coef_major = 0);
// part: 0 = K2 + K3 (+ general), 1 = K2 only, 2 = K3 (+ general) only.
int launch_modres(const ResParams& rp, bool fast, cudaStream_t st, int part = 0);
// K4's epilogue as the prime-sharded exchange: coefficient j of curve b, local
// prime kl goes straight to shard r = j / Jb's receive buffer,
//   dst[r][shard_off + b * curve_stride + kl * Jb + (j - r * Jb)],
// by (NVLink peer) stores from the kernel -- no all-gather of whole rows.  G = 0: in place.
constexpr int kMaxScatter = 8;
struct RowScatter {
  uint32_t* dst[kMaxScatter];
  int G, Jb;
  long long shard_off, curve_stride;
};
int launch_interp(uint32_t* rows, size_t rows_bstride, int pitch, int nk, int B, const PrimeConst* d_pc,
                  const uint32_t* d_twinv, int k0, int N, int r, int a, int D, int negate, uint32_t* counters,
                  cudaStream_t st, uint32_t* d_work = nullptr,  // d_work: B * nk * N words when N > kMaxNttSmem
                  const RowScatter* scatter = nullptr);
// Fills twinv[k][i] = omega_k^{-i} for all primes of a table (one launch, at table build).
void launch_twiddles(const PrimeConst* d_pc, int P, int N, uint32_t* d_twinv);
int launch_crt(const CrtParams& cp, cudaStream_t st);
// Device packing of B CRT outputs [B][D][W] into result blocks (api_common layout, back to back):
// meta [B + 1][4] u32 = (n_coeffs, total limbs, byte offset, -) per curve, meta[4 B] = bytes;
// nl scratch [B][D].  pack_bytes_bound = the image size for any result of the plan.
int launch_pack(const uint32_t* d_out, int B, int D, int W, uint32_t* d_nl, uint32_t* d_meta, uint8_t* d_pk,
                cudaStream_t st);
size_t pack_bytes_bound(int B, int D, int W);
size_t pack_meta_words(int B, int D);  // meta + the per-block partial sums (device words)

}  // namespace ctg
