// Scratch check of the TMA + tcgen05 u8 GEMM (paper_1103_4697_b200/csrc/crt_gemm_tma.cuh)
// against a plain CUDA-core reference on random bytes, plus timing at the CRT shapes.
// (A cp.async-fed variant of the same tcgen05 kernel measured 600 TOPS at the d16 shape;
// the TMA/SWIZZLE_128B/warp-specialised one 1.9 POPS; the mma.sync kernel ~610 TOPS.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc_gemm_test tc_gemm_test.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1103_4697_b200/csrc/crt_gemm_tma.cuh"
#include <cudaTypedefs.h>

using namespace ctg;

__global__ void k_ref(const uint8_t* A, const uint8_t* B, int32_t* C, int M, int N, int K) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N) return;
  int32_t s = 0;
  for (int k = 0; k < K; ++k) s += static_cast<int32_t>(A[static_cast<size_t>(m) * K + k]) * B[static_cast<size_t>(n) * K + k];
  C[static_cast<size_t>(m) * N + n] = s;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q);
  }
  return fn;
}
static CUtensorMap make_map(const void* base, uint64_t rows, uint64_t kbytes, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {kbytes, rows};
  cuuint64_t strides[1] = {kbytes};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("cuTensorMapEncodeTiled failed %d\n", static_cast<int>(r));
  return m;
}

template <int BN>
int run_tma(int M, int N, int K, unsigned seed) {
  std::vector<uint8_t> hA(static_cast<size_t>(M) * K), hB(static_cast<size_t>(N) * K);
  srand(seed);
  for (auto& x : hA) x = rand() & 0xff;
  for (auto& x : hB) x = rand() & 0xff;
  uint8_t *A, *B;
  int32_t *C, *R;
  cudaMalloc(&A, hA.size());
  cudaMalloc(&B, hB.size());
  cudaMalloc(&C, 4ull * M * N);
  cudaMalloc(&R, 4ull * M * N);
  cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  cudaMemset(C, 0xff, 4ull * M * N);
  CUtensorMap ta = make_map(A, M, K, tma::kBM), tb = make_map(B, N, K, BN);
  const size_t smem = tma::smem_bytes<BN>();
  cudaFuncSetAttribute(tma::k_gemm_u8_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  dim3 grid(N / BN, M / tma::kBM);
  tma::k_gemm_u8_tma<BN><<<grid, 128, smem>>>(ta, tb, reinterpret_cast<int4*>(C), M, K);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("tma kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  k_ref<<<dim3((N + 127) / 128, M), 128>>>(A, B, R, M, N, K);
  cudaDeviceSynchronize();
  std::vector<int32_t> hC(static_cast<size_t>(M) * N), hR(hC.size());
  cudaMemcpy(hC.data(), C, 4 * hC.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(hR.data(), R, 4 * hR.size(), cudaMemcpyDeviceToHost);
  size_t bad = 0, first = 0;
  // C is laid out [m / 128][n / 4][m % 128][n % 4]; R is row-major [m][n].
  for (size_t i = 0; i < hR.size(); ++i) {
    const size_t m = i / N, n = i % N;
    if (hC[(((m / 128) * (N / 4) + n / 4) * 128 + m % 128) * 4 + n % 4] != hR[i]) {
      if (!bad) first = i;
      ++bad;
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) tma::k_gemm_u8_tma<BN><<<grid, 128, smem>>>(ta, tb, reinterpret_cast<int4*>(C), M, K);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  const double tops = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("TMA BN=%d M=%d N=%d K=%d: mismatches %zu", BN, M, N, K, bad);
  if (bad) printf(" (first at m=%zu n=%zu: want %d)", first / N, first % N, hR[first]);
  printf("  time %.3f ms  %.1f TOPS\n", ms, tops);
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  cudaFree(R);
  return bad ? 1 : 0;
}

int main() {
  int rc = 0;
  rc |= run_tma<128>(128, 128, 128, 1);
  rc |= run_tma<128>(256, 256, 512, 2);
  rc |= run_tma<256>(256, 512, 4224, 3);
  rc |= run_tma<256>(64 * 256, 4352, 4224, 4);  // d16/1024 CRT shape, batch 64
  rc |= run_tma<128>(64 * 384, 384, 384, 5);    // d20/64 CRT shape, batch 64
  printf("%s\n", rc ? "FAIL" : "OK");
  return rc;
}
