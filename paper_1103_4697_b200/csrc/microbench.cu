// Integer-pipe peak microbenchmarks: the denominators of the K3 roofline.
// MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks; the mod-p
// resultant is bound by the FMA pipe's integer multiplies (IMAD / IMAD.WIDE),
// so bench.py measures those peaks live on the same GPU with these kernels.
#include <cuda_runtime.h>

#include "api_common.hpp"
#include "modarith.cuh"

namespace ctg {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

// 8 independent IMAD chains per thread: a_i = a_i * b + c.
__global__ void __launch_bounds__(256) k_imad(uint32_t b, uint32_t c, uint32_t* sink) {
  uint32_t a[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x + i;
#pragma unroll 16
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = a[i] * b + c;
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= a[i];
  if (s == 0x12345678u) sink[0] = s;
}

// 8 independent IMAD.WIDE chains: acc_i = x_i * b + acc_i (u32 x u32 + u64).
__global__ void __launch_bounds__(256) k_imad_wide(uint32_t b, uint32_t* sink) {
  uint64_t acc[kChains];
  uint32_t x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = threadIdx.x + i;
    x[i] = threadIdx.x * 7 + i;
  }
#pragma unroll 16
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      acc[i] = static_cast<uint64_t>(x[i]) * b + acc[i];
      x[i] ^= static_cast<uint32_t>(acc[i]);
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= acc[i];
  if (s == 0x123456789ull) sink[0] = static_cast<uint32_t>(s);
}

// 8 independent chains of Montgomery two-product reductions (the K3 inner op).
__global__ void __launch_bounds__(256) k_mmul2(uint32_t p, uint32_t* sink) {
  const Mod M = make_mod(p);
  uint32_t a[kChains], b[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    a[i] = (threadIdx.x * 131u + i) % p;
    b[i] = (threadIdx.x * 17u + 3u * i + 1u) % p;
  }
  const uint32_t u = 12345u % p, v = 67891u % p;
#pragma unroll 8
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = mmul2(u, a[i], v, b[i], M);
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= a[i];
  if (s == 0x12345678u) sink[0] = s;
}

}  // namespace
}  // namespace ctg

extern "C" ctg_status ctg_microbench_int(int32_t device, double* imad_per_s, double* imad_wide_per_s,
                                         double* mmul2_per_s) {
  using namespace ctg;
  return guarded([&] {
    ctg_opts o{};
    o.device = device;
    DeviceGuard g(&o);
    int dev = select_device(&o);
    int sms = 0;
    CTG_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    uint32_t* sink = nullptr;
    CTG_CUDA_CHECK(cudaMalloc(&sink, 4));
    cudaEvent_t e0, e1;
    CTG_CUDA_CHECK(cudaEventCreate(&e0));
    CTG_CUDA_CHECK(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256;
    const double lanes = static_cast<double>(blocks) * threads * kChains;
    auto time_ms = [&](auto launch) {
      launch();  // warm-up
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      return static_cast<double>(best);
    };
    const double t1 = time_ms([&] { k_imad<<<blocks, threads>>>(0x9e3779b9u, 7u, sink); });
    const double t2 = time_ms([&] { k_imad_wide<<<blocks, threads>>>(0x9e3779b9u, sink); });
    const double t3 = time_ms([&] { k_mmul2<<<blocks, threads>>>(2147483647u - 18u * 16u, sink); });
    CTG_CUDA_CHECK(cudaGetLastError());
    if (imad_per_s) *imad_per_s = lanes * kIters / (t1 * 1e-3);
    if (imad_wide_per_s) *imad_wide_per_s = lanes * kIters / (t2 * 1e-3);
    if (mmul2_per_s) *mmul2_per_s = lanes * (kIters / 4) / (t3 * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
  });
}
