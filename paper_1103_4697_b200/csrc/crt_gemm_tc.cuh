// K5 CRT product on the 5th-generation tensor cores (tcgen05, sm_100a):
//
//   C[m][n] = sum_k A[m][k] * B[n][k]      u8 x u8 -> s32, exact (4P * 255^2 < 2^31)
//
// A = Yt (byte slices of the CRT digits y_k, one row per coefficient), B = Bt8 (shift-expanded
// byte slices of M / p_k, one row per output byte digit), both K-major in global memory.
//
// One CTA (128 threads) computes a 128 x BN tile.  Operands are staged by cp.async into
// shared memory in the canonical no-swizzle K-major UMMA layout (8-row x 16-byte core
// matrices: LBO = 128 B between the two K halves of one instruction, SBO = 512 B between
// 8-row groups), STAGES deep.  One elected thread issues tcgen05.mma.cta_group::1.kind::i8
// (M = 128, N = BN, K = 32 per instruction) into a TMEM accumulator (128 lanes x BN columns)
// and tcgen05.commit signals an mbarrier per stage, which gates the reuse of that stage's
// smem.  The epilogue reads TMEM with tcgen05.ld.32x32b (warp w owns lanes 32w..32w+31 =
// rows) and stores rows of C with 16-byte stores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ctg {
namespace tc {

constexpr int kBM = 128;      // rows per CTA (= UMMA M, one TMEM lane per row)
constexpr int kBK = 64;       // bytes of K per stage (2 UMMA instructions of K = 32)
constexpr int kStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

// Shared-memory matrix descriptor, no swizzle, K-major (start, LBO, SBO in bytes).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;  // descriptor version 1 (sm_100)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}

// Instruction descriptor: kind::i8, unsigned A and B, s32 accumulate, K-major A and B.
__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4)                                  // c_format = S32
         | (0u << 7) | (0u << 10)                   // a/b format = unsigned 8-bit
         | (static_cast<uint32_t>(N >> 3) << 17)    // n_dim
         | (static_cast<uint32_t>(M >> 4) << 24);   // m_dim
}

template <int BN, int MT = 1>
struct GemmSmem {
  uint8_t a[kStages][MT * kBM * kBK];
  uint8_t b[kStages][BN * kBK];
  uint64_t mma_done[kStages];
  uint64_t final_done;
  uint32_t tmem_base;
};

// Canonical K-major no-swizzle offset of 16-byte chunk c (0..3) of row r in a stage tile.
__device__ __forceinline__ uint32_t tile_off(int r, int c) { return (r >> 3) * 512 + c * 128 + (r & 7) * 16; }

// C tile [m0, m0 + MT * 128) x [n0, n0 + BN), rows of A / B at stride lda / ldb bytes, K bytes
// (multiple of kBK), C at stride ldc int32.  MT = 2 runs two M = 128 accumulators (TMEM
// columns [0, BN) and [BN, 2 BN)) against the same B stage, halving B's L2 traffic.
template <int BN, int MT = 1>
__device__ __forceinline__ void gemm_u8_tile(const uint8_t* __restrict__ A, size_t lda, const uint8_t* __restrict__ Bm,
                                             size_t ldb, int32_t* __restrict__ Cm, size_t ldc, int K,
                                             GemmSmem<BN, MT>& sm) {
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(MT * BN <= 512 && (MT * BN & (MT * BN - 1)) == 0, "TMEM columns");
  constexpr int kCols = MT * BN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&sm.tmem_base)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) mbar_init(&sm.mma_done[s], 1);
    mbar_init(&sm.final_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = sm.tmem_base;

  const int nk = K / kBK;
  auto load_stage = [&](int kb, int s) {
    const int k0 = kb * kBK;
    const uint32_t sa = smem_u32(sm.a[s]), sb = smem_u32(sm.b[s]);
#pragma unroll
    for (int i = tid; i < MT * kBM * 4; i += 128) {
      const int r = i >> 2, c = i & 3;
      cp_async16(sa + tile_off(r, c), A + r * lda + k0 + c * 16);
    }
#pragma unroll
    for (int i = tid; i < BN * 4; i += 128) {
      const int r = i >> 2, c = i & 3;
      cp_async16(sb + tile_off(r, c), Bm + r * ldb + k0 + c * 16);
    }
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }
  constexpr uint32_t idesc = umma_idesc_u8(kBM, BN);
  for (int kb = 0; kb < nk; ++kb) {
    const int s = kb % kStages;
    // Refill the stage that k-block kb - 1 used, once its MMAs have drained it.
    const int kn = kb + kStages - 1;
    if (kn < nk) {
      const int sn = kn % kStages;
      if (kb >= 1) mbar_wait(&sm.mma_done[sn], static_cast<uint32_t>(((kb - 1) / kStages) & 1));
      load_stage(kn, sn);
    }
    cp_commit();
    cp_wait<kStages - 1>();  // k-block kb has landed (this thread's copies)
    asm volatile("fence.proxy.async.shared::cta;\n" ::);  // generic-proxy writes -> tensor-core reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t sa = smem_u32(sm.a[s]), sb = smem_u32(sm.b[s]);
#pragma unroll
      for (int h = 0; h < kBK / 32; ++h) {
        const uint64_t db = umma_desc(sb + h * 256, 128, 512);
        const uint32_t acc = (kb > 0 || h > 0) ? 1u : 0u;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint64_t da = umma_desc(sa + mt * (kBM / 8) * 512 + h * 256, 128, 512);
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + mt * BN),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&sm.mma_done[s])));
      if (kb == nk - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&sm.final_done)));
    }
  }
  mbar_wait(&sm.final_done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);

  // Epilogue: warp w reads TMEM lanes 32w..32w+31 (rows), 32 columns per load.
#pragma unroll 1
  for (int cc = 0; cc < kCols; cc += 32) {
    const int mt = cc / BN, c0 = cc - mt * BN;
    int32_t* crow = Cm + static_cast<size_t>(mt * kBM + warp * 32 + lane) * ldc;
    uint32_t v[32];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cc);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<int4*>(crow + c0)[q] =
          make_int4(static_cast<int>(v[4 * q]), static_cast<int>(v[4 * q + 1]), static_cast<int>(v[4 * q + 2]),
                    static_cast<int>(v[4 * q + 3]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kCols));
}

}  // namespace tc
}  // namespace ctg
