/* ctg.h -- C ABI of the B200 multi-modular elimination library (libctg.so).
 *
 * This is the drop-in boundary for the reference's elimination hot path
 * (namespace curvetop, /root/reference/proj):
 *
 *   ctg_resultant         replaces  curvetop::resultant(p, q, Var)
 *                                   proj/include/curvetop/elim.hpp:30-31, proj/src/elim.cpp:95-136
 *   ctg_yun_squarefree    replaces  curvetop::yun_squarefree(p)
 *                                   elim.hpp:34, elim.cpp:138-165
 *   ctg_gcd_univariate    replaces  curvetop::gcd_univariate(p, q)
 *                                   upoly.hpp:92, elim.cpp:80-93
 *   ctg_square_free_part  replaces  curvetop::square_free_part(p)
 *                                   elim.hpp:45, elim.cpp:204-210
 *   ctg_gcd_bivariate     replaces  curvetop::gcd_bivariate(f, g)
 *                                   elim.hpp:42, elim.cpp:178-202 (callers lift.cpp:85,
 *                                   pipeline.cpp:321)
 *
 * The C++ TU paper_1103_4697_b200/cxx/curvetop_elim_gpu.cpp defines those
 * curvetop:: symbols with the reference's exact signatures on top of this ABI
 * (see INTEGRATION.md), mapping status codes to the reference's exceptions:
 * CTG_PRECONDITION -> curvetop::PreconditionError, everything else -> curvetop::Error.
 *
 * Big integers cross the ABI in sign-magnitude form: one int8 sign (-1, 0, +1)
 * per coefficient and little-endian uint32 magnitude limbs in CSR layout
 * (limb_off has n+1 entries; coefficient i owns limbs[limb_off[i] .. limb_off[i+1])).
 * All input pointers are caller-owned host memory; outputs are library-allocated
 * host buffers released with the matching ctg_*_free.  There is no CPU fallback:
 * when no usable CUDA device is present, every compute entry point returns CTG_CUDA.
 */
#ifndef CTG_H
#define CTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTG_ABI_VERSION 2

typedef enum {
  CTG_OK = 0,
  CTG_PRECONDITION = 1, /* reference PreconditionError (e.g. both inputs zero)        */
  CTG_INVALID = 2,      /* malformed arguments (null pointers, bad CSR, bad range)     */
  CTG_UNSUPPORTED = 3,  /* size beyond the library's limits (message says which)       */
  CTG_INTERNAL = 4,     /* a self-check failed (bound exceeded, certificate failed)    */
  CTG_CUDA = 5,         /* CUDA runtime error or no device                             */
} ctg_status;

/* Sparse bivariate polynomial sum c_t x^dx[t] y^dy[t] (exponents >= 0; repeated
 * exponent pairs are summed, zero terms ignored -- bipoly.cpp:7-15). */
typedef struct {
  int32_t n_terms;
  const int32_t* dx;
  const int32_t* dy;
  const int8_t* sign;
  const uint32_t* limb_off; /* n_terms + 1 */
  const uint32_t* limbs;
} ctg_bipoly;

/* Dense univariate polynomial, coefficients low -> high; n_coeffs = 0 is the zero polynomial.
 * Trailing zero coefficients are allowed on input (they are trimmed, upoly.hpp:83-85). */
typedef struct {
  int32_t n_coeffs;
  const int8_t* sign;
  const uint32_t* limb_off; /* n_coeffs + 1 */
  const uint32_t* limbs;
} ctg_upoly;

/* Library-allocated univariate result (trimmed: the last coefficient is nonzero). */
typedef struct {
  int32_t n_coeffs;
  int8_t* sign;
  uint32_t* limb_off;
  uint32_t* limbs;
} ctg_upoly_buf;

/* Square-free factorization: value = unit * prod factors[i]^mult[i] (elim.hpp:13-22). */
typedef struct {
  int8_t unit_sign;
  int32_t unit_nlimbs;
  uint32_t* unit_limbs;
  int32_t n_factors;
  int32_t* mult;          /* strictly increasing */
  ctg_upoly_buf* factors; /* primitive, positive leading coefficient, square-free */
} ctg_sqf_buf;

/* Library-allocated bivariate result, terms sorted by (dx, dy), no zero terms. */
typedef struct {
  int32_t n_terms;
  int32_t* dx;
  int32_t* dy;
  int8_t* sign;
  uint32_t* limb_off; /* n_terms + 1 */
  uint32_t* limbs;
} ctg_bipoly_buf;

/* Multi-process communicator (one process per GPU, e.g. under torchrun): ctg_comm_init_rank. */
typedef struct ctg_comm ctg_comm;

typedef struct {
  int32_t device;   /* CUDA device ordinal; -1 = current device */
  int32_t verify;   /* 1 (default) = run the on-device self-checks; 0 = skip the optional ones */
  /* Prime sharding of ctg_resultant / ctg_resultant_batch:
   *  - n_devices > 1: this process drives devices[0..n_devices); shard g owns a contiguous
   *    block of the primes, computes those rows of the residue matrix (K1-K4), the rows are
   *    all-gathered over NCCL (distinct devices) or device copies (a device listed twice:
   *    shards share it), shard g reconstructs a block of coefficients (K5) and copies it
   *    straight into the host result.  Results are bit-identical to one device.
   *  - comm != NULL: multi-process; every rank calls with the same inputs, computes its prime
   *    block, NCCL all-gathers residues and CRT'd coefficient blocks; every rank returns the
   *    full result. */
  int32_t n_devices;
  int32_t reserved0;
  const int32_t* devices;
  ctg_comm* comm;
} ctg_opts;

/* Timings of the last call on this thread (milliseconds; host wall clock around each phase). */
typedef struct {
  double total_ms, setup_ms, h2d_ms, device_ms, d2h_ms, decode_ms;
  int64_t h2d_bytes, d2h_bytes;
  int32_t n_primes, n_points, n_coeffs, out_limbs, kernel_launches, flagged_units;
} ctg_call_stats;

/* ---- entry points (the drop-in surface) ---- */
ctg_status ctg_resultant(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                         ctg_upoly_buf* out, const ctg_opts* opts);
ctg_status ctg_yun_squarefree(const ctg_upoly* p, ctg_sqf_buf* out, const ctg_opts* opts);
ctg_status ctg_gcd_univariate(const ctg_upoly* p, const ctg_upoly* q, ctg_upoly_buf* out,
                              const ctg_opts* opts);
/* yun_squarefree over a batch (CurveContext over many curves, lift.cpp:67): one K1 launch and
 * one square-freeness probe launch for all inputs, contents on the host meanwhile; inputs the
 * probe does not certify go through ctg_yun_squarefree's path.  out[b] = Yun(p[b]) exactly. */
ctg_status ctg_yun_squarefree_batch(int32_t batch, const ctg_upoly* p, ctg_sqf_buf* out, const ctg_opts* opts);
ctg_status ctg_square_free_part(const ctg_upoly* p, ctg_upoly_buf* out, const ctg_opts* opts);
/* gcd_bivariate (elim.cpp:178-202): y-contents by GPU univariate gcds, then a GPU probe of
 * gcd(f(a, y), g(a, y)) mod p at several (p, a) with lc_y(f)(a) or lc_y(g)(a) nonzero mod p.
 * A degree-0 image certifies that the primitive parts are coprime; the result is then
 * gcd_univariate(content_y f, content_y g).  Otherwise Brown's modular gcd runs on the GPU
 * (images gamma(a) * gcd(f(a, y), g(a, y)) mod p with cofactors, Newton interpolation in x,
 * CRT) and an exactness certificate proves the result; output terms sorted by (dx, dy).
 * No size limit: beyond the shared-memory budget the kernels' buffers move to global memory. */
ctg_status ctg_gcd_bivariate(const ctg_bipoly* f, const ctg_bipoly* g, ctg_bipoly_buf* out,
                             const ctg_opts* opts);

void ctg_upoly_free(ctg_upoly_buf* buf);
void ctg_bipoly_free(ctg_bipoly_buf* buf);
void ctg_upoly_free_batch(ctg_upoly_buf* bufs, int32_t n); /* = ctg_upoly_free on each */
void ctg_sqf_free(ctg_sqf_buf* buf);
const char* ctg_last_error(void); /* thread-local message of the last failing call */
int32_t ctg_abi_version(void);
int32_t ctg_device_count(void);
void ctg_last_call_stats(ctg_call_stats* out);

/* ---- staged resultant (prime sharding across GPUs; device-resident benchmarking) ----
 * A plan fixes the primes, the evaluation points and the CRT constants for one
 * resultant on the device that is current when it is created.  Prime k of the
 * plan owns row k of the residue matrix (pitch = n_points words, values R mod p_k
 * coefficients 0..n_coeffs-1 after ctg_plan_residues).  Any subset of rows can be
 * computed on any GPU (one plan per GPU), exchanged (e.g. NCCL all-gather), and
 * ctg_plan_crt reconstructs any coefficient range from the full matrix. */
typedef struct ctg_plan ctg_plan;

typedef struct {
  int32_t n_primes;    /* rows of the residue matrix                              */
  int32_t n_points;    /* evaluation points per prime (= row pitch, NTT size)      */
  int32_t n_coeffs;    /* degree bound + 1 of the result                           */
  int32_t out_limbs;   /* uint32 limbs per reconstructed coefficient               */
  int32_t deg_p, deg_q;/* formal degrees in the eliminated variable                */
  int32_t derivative;  /* 1 if q == dp/dy was detected (shared evaluation)         */
  int32_t trivial;     /* 1 if the result is fixed by a convention (no GPU work)    */
  double bound_bits;   /* log2 of the Hadamard coefficient bound                    */
  double work_mulmods; /* algorithmic mulmods of the mod-p resultant stage */
  int64_t h2d_bytes;   /* bytes ctg_plan_upload copies host -> device                */
  int32_t batch;       /* number of problems (curves) in the plan                     */
} ctg_plan_info;

ctg_status ctg_plan_create(const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                           const ctg_opts* opts, ctg_plan** plan);
ctg_status ctg_plan_get_info(const ctg_plan* plan, ctg_plan_info* info);
/* Upload the inputs (H2D) -- part of an end-to-end call, separate for device-only timing. */
ctg_status ctg_plan_upload(ctg_plan* plan, void* stream);
/* Rows [k0, k1) of the residue matrix into d_rows (device, (k1-k0) x n_points words). */
ctg_status ctg_plan_residues(ctg_plan* plan, int32_t k0, int32_t k1, uint32_t* d_rows, void* stream);
/* One stage of ctg_plan_residues (for per-kernel timing): 1 = reduce (K1),
 * 2 = evaluate + mod-p resultant (K2/K3 + the exact fallback), 3 = interpolate (K4);
 * stage 2 split in two: 4 = evaluate only (K2; nothing without the fast path),
 * 5 = mod-p resultant only (K3 + the exact fallback; needs stage 4 first). */
ctg_status ctg_plan_stage(ctg_plan* plan, int32_t stage, int32_t k0, int32_t k1, uint32_t* d_rows, void* stream);
/* Coefficients [j0, j1) from the full residue matrix d_all (device, n_primes x n_points):
 * d_out gets (j1-j0) x (out_limbs + 1) words: word 0 = sign (as int32), then magnitude limbs. */
ctg_status ctg_plan_crt(ctg_plan* plan, const uint32_t* d_all, int32_t j0, int32_t j1, uint32_t* d_out,
                        void* stream);
/* Same, with the residue matrix spread over rank blocks (e.g. the output of an NCCL
 * all-gather): row k lives at d_all + (k / row_block) * block_stride + (k % row_block) * n_points. */
ctg_status ctg_plan_crt_sharded(ctg_plan* plan, const uint32_t* d_all, int32_t row_block, int64_t block_stride,
                                int32_t j0, int32_t j1, uint32_t* d_out, void* stream);
/* Decode a host copy of the full CRT output (n_coeffs x (out_limbs + 1) words) into a result. */
ctg_status ctg_plan_decode(ctg_plan* plan, const uint32_t* h_crt, ctg_upoly_buf* out);
/* Device error flags accumulated by the plan's kernels (0 = clean); synchronizes the stream. */
ctg_status ctg_plan_check(ctg_plan* plan, void* stream);
/* Number of kernel launches issued by the plan since creation. */
int32_t ctg_plan_launches(const ctg_plan* plan);
void ctg_plan_destroy(ctg_plan* plan);

/* ---- batches: B same-shape problems per plan / call (one set of kernel launches) ----
 * ctg_resultant_batch takes arrays p[0..batch), q[0..batch) and fills out[0..batch); inputs
 * of different shapes are grouped internally.  A batch plan requires every member to have
 * the same degrees in the eliminated variable (and the same q == dp/dy relation); its
 * primes cover the largest coefficient bound of the batch.  Device layouts: residue rows of
 * curve b at d_rows + b * curve_stride (curve_stride = 0: dense, (k1-k0) * n_points); CRT
 * output of curve b at d_out + b * (j1-j0) * (out_limbs + 1). */
ctg_status ctg_resultant_batch(int32_t batch, const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                               ctg_upoly_buf* out, const ctg_opts* opts);
ctg_status ctg_plan_create_batch(int32_t batch, const ctg_bipoly* p, const ctg_bipoly* q, int32_t eliminate_x,
                                 const ctg_opts* opts, ctg_plan** plan);
ctg_status ctg_plan_stage_batch(ctg_plan* plan, int32_t stage, int32_t k0, int32_t k1, uint32_t* d_rows,
                                int64_t curve_stride, void* stream);
/* Residues of curve b, prime k at d_all + b * curve_stride + (k / row_block) * block_stride
 * + (k % row_block) * n_points (curve_stride 0: n_primes * n_points; row_block 0: n_primes). */
ctg_status ctg_plan_crt_batch(ctg_plan* plan, const uint32_t* d_all, int64_t curve_stride, int32_t row_block,
                              int64_t block_stride, int32_t j0, int32_t j1, uint32_t* d_out, void* stream);

/* ---- multi-process communicators (NCCL, loaded at run time) ----
 * Rank 0 creates an id with ctg_comm_unique_id, shares the bytes with the other ranks
 * (any host channel), and every rank calls ctg_comm_init_rank with its own device.
 * ctg_comm_all_gather: words u32 per rank, d_recv = nranks x words (device buffers). */
#define CTG_COMM_ID_BYTES 128
ctg_status ctg_comm_unique_id(uint8_t* id /* CTG_COMM_ID_BYTES */);
ctg_status ctg_comm_init_rank(int32_t nranks, int32_t rank, const uint8_t* id, int32_t device, ctg_comm** comm);
void ctg_comm_destroy(ctg_comm* comm);
ctg_status ctg_comm_all_gather(ctg_comm* comm, const void* d_send, void* d_recv, size_t words, void* stream);
/* All-to-all (grouped ncclSend / ncclRecv): block r of d_send (words u32 each) goes to rank r,
 * block s of d_recv arrives from rank s. */
ctg_status ctg_comm_all_to_all(ctg_comm* comm, const void* d_send, void* d_recv, size_t words, void* stream);

/* Column-block exchange of a prime-sharded plan: instead of all-gathering whole
 * residue rows, the interpolation (stage 3) of primes [k0, k1) writes each coefficient j straight
 * into the block of the rank that reconstructs it, r = j / Jb with Jb = ceil(D / nranks):
 * d_send = [nranks][B][row_block][Jb] (prime k at row k - k0; row_block >= k1 - k0), point values
 * read from d_rows as for ctg_plan_stage_batch(stage 3).  After ctg_comm_all_to_all (or any
 * exchange giving rank r the blocks [s][B][row_block][Jb] of every rank s), ctg_plan_crt_cols
 * reconstructs coefficients [r Jb, min(D, (r + 1) Jb)) of every curve from d_recv (prime k in
 * block k / row_block) into d_out [B][J][out_limbs + 1].  Each rank then receives 1/nranks of
 * the bytes of a row all-gather. */
ctg_status ctg_plan_interp_cols(ctg_plan* plan, int32_t k0, int32_t k1, uint32_t* d_rows, int64_t curve_stride,
                                int32_t nranks, int32_t row_block, uint32_t* d_send, void* stream);
ctg_status ctg_plan_crt_cols(ctg_plan* plan, const uint32_t* d_recv, int32_t nranks, int32_t rank, int32_t row_block,
                             uint32_t* d_out, void* stream);

/* Integer-pipe peak microbenchmarks on `device` (-1 = current): 32-bit IMAD
 * (a*b+c) and IMAD.WIDE (u32*u32+u64) results per second over all SMs, and
 * Montgomery two-product reductions (modarith.cuh mmul2) per second. */
ctg_status ctg_microbench_int(int32_t device, double* imad_per_s, double* imad_wide_per_s, double* mmul2_per_s);

/* Test and A/B hook of K6's remainder-sequence kernels (no reference counterpart): deg gcd(a, b)
 * over F_p for p = the prime_index-th (0..15) univariate prime, a[0..na] and b[0..nb] plain
 * residues < p; method 0 = the blocked (Lehmer-style) kernel the square-freeness probe runs,
 * 1 = one CTA pass per Euclid step.  *deg = -1 when both vanish; *prime = p, *ms = kernel time
 * (either may be NULL). */
ctg_status ctg_modp_gcd_degree(const uint32_t* a, int32_t na, const uint32_t* b, int32_t nb, int32_t prime_index,
                               int32_t method, int32_t* deg, uint32_t* prime, float* ms, const ctg_opts* opts);

#ifdef __cplusplus
}
#endif

#endif /* CTG_H */
