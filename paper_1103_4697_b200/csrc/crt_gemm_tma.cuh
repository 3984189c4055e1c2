// K5 CRT product on the 5th-generation tensor cores, TMA-fed (sm_100a):
//
//   C[m][n] = sum_k A[m][k] * B[n][k]      u8 x u8 -> s32, exact (4P * 255^2 < 2^31)
//
// A = Yt (byte slices of the CRT digits y_k of every coefficient of every curve, [rows][K]),
// B = Bt8 (shift-expanded byte slices of M / p_k, [L8p][K]); both K-major.
//
// CTA = 128 threads, tile 128 x BN, K in stages of 128 bytes (one 128-byte swizzle atom):
//   warp 0 / lane 0  TMA producer: cp.async.bulk.tensor (SWIZZLE_128B boxes 128 x 128 B and
//                    BN x 128 B) into stage s, completion counted on full[s] (expect_tx)
//   warp 1 / lane 0  MMA issuer: waits full[s], issues 4 x tcgen05.mma.cta_group::1.kind::i8
//                    (M 128, N BN, K 32) into the TMEM accumulator, tcgen05.commit -> empty[s]
//   all warps        epilogue: tcgen05.ld.32x32b (warp w owns TMEM lanes / rows 32w..32w+31)
//                    -> coalesced 16-byte stores, C laid out [row tile][digit group][row in tile].
// Shared-memory descriptors: K-major SWIZZLE_128B, SBO = 1024 B (8 rows x 128 B), the K step
// of one instruction advances the start address by 32 B inside the 1024-B-aligned atom.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ctg {
namespace tma {

constexpr int kBM = 128;
constexpr int kBK = 128;  // bytes of K per stage
constexpr int kStages = 4;

template <int BN, int ST = kStages>
struct alignas(1024) Smem {
  uint8_t a[ST][kBM * kBK];
  uint8_t b[ST][BN * kBK];
  uint64_t full[ST], empty[ST], final_done;
  uint32_t tmem_base;
};
template <int BN, int ST = kStages>
constexpr size_t smem_bytes() {
  return sizeof(Smem<BN, ST>) + 1024;  // + alignment slack of the dynamic smem base
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(su32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

// K-major SWIZZLE_128B shared-memory descriptor.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fffu);
  d |= static_cast<uint64_t>(1u) << 16;           // LBO (unused for swizzled K-major) = 1
  d |= static_cast<uint64_t>(1024u >> 4) << 32;   // SBO = 1024 B between 8-row groups
  d |= static_cast<uint64_t>(1u) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;           // layout: SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// The GEMM main loop shared by both epilogues: TMEM allocation, barrier setup, TMA producer
// (warp 0), MMA issuer (warp 1); returns the TMEM accumulator base once every MMA retired.
template <int BN, int ST = kStages>
__device__ __forceinline__ uint32_t gemm_mainloop(Smem<BN, ST>& sm, const CUtensorMap& ta, const CUtensorMap& tb, int m0,
                                                  int n0, int K) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&sm.tmem_base)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 32) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    mbar_init(&sm.final_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = sm.tmem_base;
  const int nk = K / kBK;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % ST;
        if (kb >= ST) mbar_wait(&sm.empty[s], static_cast<uint32_t>(((kb / ST) - 1) & 1));
        mbar_expect_tx(&sm.full[s], static_cast<uint32_t>((kBM + BN) * kBK));
        tma_load_2d(sm.a[s], &ta, &sm.full[s], kb * kBK, m0);
        tma_load_2d(sm.b[s], &tb, &sm.full[s], kb * kBK, n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = idesc_u8(kBM, BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % ST;
        mbar_wait(&sm.full[s], static_cast<uint32_t>((kb / ST) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t sa = su32(sm.a[s]), sb = su32(sm.b[s]);
#pragma unroll
        for (int kk = 0; kk < kBK / 32; ++kk) {
          const uint64_t da = desc_sw128(sa + kk * 32), db = desc_sw128(sb + kk * 32);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            su32(&sm.empty[s])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          su32(&sm.final_done)));
    }
    __syncwarp();
  }
  mbar_wait(&sm.final_done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  return tmem;
}

// 32 consecutive accumulator columns of this thread's TMEM lane (row).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
}

template <int BN, int ST = kStages>
__device__ __forceinline__ void gemm_teardown(Smem<BN, ST>& sm, uint32_t tmem) {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(BN));
}

// C rows [blockIdx.y * 128, +128) x cols [blockIdx.x * BN, +BN); K multiple of kBK.
template <int BN>
__global__ void __launch_bounds__(128, 1)
    k_gemm_u8_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int4* __restrict__ C,
                  int Rp, int K) {
  extern __shared__ uint8_t smraw[];
  Smem<BN>& sm = *reinterpret_cast<Smem<BN>*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
  const uint32_t tmem = gemm_mainloop<BN>(sm, ta, tb, m0, n0, K);
  // C layout [row tile of 128][digit group l / 4][row in tile] of int4 (4 digits), rows = the
  // flattened coefficients of all curves: each warp's stores of one digit group are 32
  // consecutive int4 (512 contiguous bytes), and the carry kernel's per-coefficient walk over
  // the digit groups reads them back coalesced with a 2 KB stride (one tile's slab).
  const long long slab = static_cast<long long>(gridDim.x) * BN / 4;  // digit groups per row (L8p / 4)
  int4* cbase = C + (static_cast<long long>(m0 / kBM) * slab + n0 / 4) * kBM + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0), v);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      cbase[static_cast<long long>(c0 / 4 + q) * kBM] =
          make_int4(static_cast<int>(v[4 * q]), static_cast<int>(v[4 * q + 1]), static_cast<int>(v[4 * q + 2]),
                    static_cast<int>(v[4 * q + 3]));
  }
  gemm_teardown<BN>(sm, tmem);
}

}  // namespace tma
}  // namespace ctg
