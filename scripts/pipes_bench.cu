// Scratch microbenchmark (not part of the library): per-SM throughput of the integer and
// FP64 multiply forms the mod-p Euclid step can be written in, and of two candidate inner
// ops (Montgomery 3-product vs Shoup 3-product with lazy [0, 2^32) residues).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes_bench pipes_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kC = 8;
constexpr int kIt = 2048;

__global__ void k_imad(uint32_t b, uint32_t c, uint32_t* sink) {
  uint32_t a[kC];
  for (int i = 0; i < kC; ++i) a[i] = threadIdx.x + i;
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) a[i] = a[i] * b + c;
  uint32_t s = 0;
  for (int i = 0; i < kC; ++i) s ^= a[i];
  if (s == 0x12345678u) sink[0] = s;
}

__global__ void k_imad_hi(uint32_t b, uint32_t* sink) {
  uint32_t a[kC];
  for (int i = 0; i < kC; ++i) a[i] = threadIdx.x * 77u + i * 12345u + 99999u;
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) a[i] = __umulhi(a[i], b) + a[i];
  uint32_t s = 0;
  for (int i = 0; i < kC; ++i) s ^= a[i];
  if (s == 0x12345678u) sink[0] = s;
}

__global__ void k_imad_wide(uint32_t b, uint32_t* sink) {
  uint64_t acc[kC];
  for (int i = 0; i < kC; ++i) acc[i] = threadIdx.x + i;
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) acc[i] = static_cast<uint64_t>(static_cast<uint32_t>(acc[i] >> 7)) * b + acc[i];
  uint64_t s = 0;
  for (int i = 0; i < kC; ++i) s ^= acc[i];
  if (s == 0x12345678u) sink[0] = static_cast<uint32_t>(s);
}

__global__ void k_dfma(double b, double c, uint32_t* sink) {
  double a[kC];
  for (int i = 0; i < kC; ++i) a[i] = threadIdx.x + i;
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < kC; ++i) s += a[i];
  if (s == 1.2345) sink[0] = 1;
}

// IMAD chains and DFMA chains interleaved in one thread (same counts as the two above).
__global__ void k_mixed(uint32_t b, uint32_t c, double bd, double cd, uint32_t* sink) {
  uint32_t a[kC];
  double d[kC];
  for (int i = 0; i < kC; ++i) {
    a[i] = threadIdx.x + i;
    d[i] = threadIdx.x + i;
  }
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      a[i] = a[i] * b + c;
      d[i] = fma(d[i], bd, cd);
    }
  uint32_t s = 0;
  double t = 0;
  for (int i = 0; i < kC; ++i) {
    s ^= a[i];
    t += d[i];
  }
  if (s == 0x12345678u || t == 1.2345) sink[0] = s;
}

struct Mod {
  uint32_t p, pneg;
};
__device__ __forceinline__ uint32_t csub(uint32_t r, uint32_t p) {
  uint32_t s = r - p;
  return s < r ? s : r;
}
__device__ __forceinline__ uint32_t mmul3(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t e, uint32_t f,
                                          Mod M) {
  uint64_t T = static_cast<uint64_t>(a) * b + static_cast<uint64_t>(c) * d + static_cast<uint64_t>(e) * f;
  uint32_t m = static_cast<uint32_t>(T) * M.pneg;
  uint64_t t = T + static_cast<uint64_t>(m) * M.p;
  return csub(static_cast<uint32_t>(t >> 32), M.p);
}
// x1 c1 + x2 c2 + x3 c3 mod p in [0, 6p) for any x < 2^32 (c < p, c' = floor(c 2^32 / p), 6p < 2^32).
__device__ __forceinline__ uint32_t shoup3(uint32_t x1, uint32_t c1, uint32_t s1, uint32_t x2, uint32_t c2,
                                           uint32_t s2, uint32_t x3, uint32_t c3, uint32_t s3, uint32_t negp) {
  const uint32_t q = __umulhi(x1, s1) + __umulhi(x2, s2) + __umulhi(x3, s3);
  return x1 * c1 + x2 * c2 + x3 * c3 + q * negp;
}

// Euclid-like recurrence over a register row: A[t] = op(c1, A[t], c2, B[t-1], c3, B[t]).
constexpr int kRow = 16;
__global__ void k_row_mont(uint32_t p, uint32_t pneg, uint32_t* sink) {
  Mod M{p, pneg};
  uint32_t A[kRow], B[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = (threadIdx.x * 131u + i) % p;
    B[i] = (threadIdx.x * 17u + 3u * i + 1u) % p;
  }
  uint32_t c1 = 12345u, c2 = 678u, c3 = 91011u;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) A[t] = mmul3(c1, A[t], c2, B[t - 1], c3, B[t], M);
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      uint32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
    }
    c1 ^= A[3];
    c1 = csub(c1, p);
  }
  uint32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i];
  if (s == 0x12345678u) sink[0] = s;
}
__global__ void k_row_shoup(uint32_t p, uint32_t* sink) {
  const uint32_t negp = 0u - p;
  uint32_t A[kRow], B[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = (threadIdx.x * 131u + i) % p;
    B[i] = (threadIdx.x * 17u + 3u * i + 1u) % p;
  }
  uint32_t c1 = 12345u, c2 = 678u, c3 = 91011u;
  uint32_t s1 = 0x1234567u, s2 = 0x2345678u, s3 = 0x3456789u;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) A[t] = shoup3(A[t], c1, s1, B[t - 1], c2, s2, B[t], c3, s3, negp);
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      uint32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
    }
    s1 ^= A[3];
  }
  uint32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i];
  if (s == 0x12345678u) sink[0] = s;
}


__global__ void k_mixed_wide(uint32_t b, double bd, double cd, uint32_t* sink) {
  uint64_t acc[kC];
  double d[kC];
  for (int i = 0; i < kC; ++i) {
    acc[i] = threadIdx.x + i;
    d[i] = threadIdx.x + i;
  }
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      acc[i] = static_cast<uint64_t>(static_cast<uint32_t>(acc[i] >> 7)) * b + acc[i];
      d[i] = fma(d[i], bd, cd);
    }
  uint64_t s = 0;
  double t = 0;
  for (int i = 0; i < kC; ++i) {
    s ^= acc[i];
    t += d[i];
  }
  if (s == 0x12345678u || t == 1.2345) sink[0] = 1;
}

__global__ void k_mixed_hi(uint32_t b, double bd, double cd, uint32_t* sink) {
  uint32_t a[kC];
  double d[kC];
  for (int i = 0; i < kC; ++i) {
    a[i] = threadIdx.x * 77u + i * 12345u + 99999u;
    d[i] = threadIdx.x + i;
  }
#pragma unroll 16
  for (int it = 0; it < kIt; ++it)
#pragma unroll
    for (int i = 0; i < kC; ++i) {
      a[i] = __umulhi(a[i], b) + a[i];
      d[i] = fma(d[i], bd, cd);
    }
  uint32_t s = 0;
  double t = 0;
  for (int i = 0; i < kC; ++i) {
    s ^= a[i];
    t += d[i];
  }
  if (s == 0x12345678u || t == 1.2345) sink[0] = 1;
}

constexpr double kMagic = 6755399441055744.0;
__device__ __forceinline__ double fred(double T, double p, double pinv) {
  const double q = __dsub_rn(__fma_rn(T, pinv, kMagic), kMagic);
  return __fma_rn(-q, p, T);
}
__global__ void k_row_fp(uint32_t pp, uint32_t* sink) {
  const double p = pp, pinv = 1.0 / p;
  double A[kRow], B[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = static_cast<double>((threadIdx.x * 131u + i) % pp) - 0.5 * p;
    B[i] = static_cast<double>((threadIdx.x * 17u + 3u * i + 1u) % pp) - 0.5 * p;
  }
  double c1 = 12345, c2 = 678, c3 = 91011;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) A[t] = fred(__fma_rn(c1, A[t], __fma_rn(c2, B[t - 1], __dmul_rn(c3, B[t]))), p, pinv);
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      double x = A[t];
      A[t] = B[t];
      B[t] = x;
    }
    c1 = fred(c1 * A[3], p, pinv);
  }
  double s = 0;
  for (int i = 0; i < kRow; ++i) s += A[i];
  if (s == 1.2345) sink[0] = 1;
}
// One integer row and one FP64 row per thread, interleaved.
__global__ void k_row_both(uint32_t p, uint32_t pneg, uint32_t pf, uint32_t* sink) {
  Mod M{p, pneg};
  const double fp = pf, fpinv = 1.0 / fp;
  uint32_t A[kRow], B[kRow];
  double X[kRow], Y[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = (threadIdx.x * 131u + i) % p;
    B[i] = (threadIdx.x * 17u + 3u * i + 1u) % p;
    X[i] = static_cast<double>((threadIdx.x * 131u + i) % pf) - 0.5 * fp;
    Y[i] = static_cast<double>((threadIdx.x * 17u + 3u * i + 1u) % pf) - 0.5 * fp;
  }
  uint32_t c1 = 12345u, c2 = 678u, c3 = 91011u;
  double d1 = 12345, d2 = 678, d3 = 91011;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) {
      A[t] = mmul3(c1, A[t], c2, B[t - 1], c3, B[t], M);
      X[t] = fred(__fma_rn(d1, X[t], __fma_rn(d2, Y[t - 1], __dmul_rn(d3, Y[t]))), fp, fpinv);
    }
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      uint32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
      double y = X[t];
      X[t] = Y[t];
      Y[t] = y;
    }
    c1 ^= A[3];
    c1 = csub(c1, p);
    d1 = fred(d1 * X[3], fp, fpinv);
  }
  uint32_t s = 0;
  double z = 0;
  for (int i = 0; i < kRow; ++i) {
    s ^= A[i];
    z += X[i];
  }
  if (s == 0x12345678u || z == 1.2345) sink[0] = s;
}

// Hybrid: exact low word by IMAD (lo), quotient estimate by FP64; values kept as int32
// (symmetric) + double copies.  CONV = 0: I2F.F64, 1: magic-constant DADD.
template <int CONV>
__device__ __forceinline__ double i2d(int32_t r) {
  if (CONV == 0) return static_cast<double>(r);
  const double x = __hiloint2double(0x43300000, static_cast<int32_t>(static_cast<uint32_t>(r) ^ 0x80000000u));
  return __dsub_rn(x, 4503601774854144.0);  // 2^52 + 2^31
}
template <int CONV>
__global__ void k_row_hyb(uint32_t pp, uint32_t* sink) {
  const double pd = pp, pinv = 1.0 / pd;
  const int32_t negp = -static_cast<int32_t>(pp);
  int32_t A[kRow], B[kRow];
  double Ad[kRow], Bd[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = static_cast<int32_t>((threadIdx.x * 131u + i) % pp) - static_cast<int32_t>(pp / 2);
    B[i] = static_cast<int32_t>((threadIdx.x * 17u + 3u * i + 1u) % pp) - static_cast<int32_t>(pp / 2);
    Ad[i] = A[i];
    Bd[i] = B[i];
  }
  int32_t c1 = 12345, c2 = 678, c3 = 91011;
  double d1 = 12345, d2 = 678, d3 = 91011;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) {
      const double T = __fma_rn(d1, Ad[t], __fma_rn(d2, Bd[t - 1], __dmul_rn(d3, Bd[t])));
      const int32_t q = __double2loint(__fma_rn(T, pinv, kMagic));
      const int32_t r = c1 * A[t] + c2 * B[t - 1] + c3 * B[t] + q * negp;
      A[t] = r;
      Ad[t] = i2d<CONV>(r);
    }
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      int32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
      double y = Ad[t];
      Ad[t] = Bd[t];
      Bd[t] = y;
    }
    c1 ^= A[3] & 0xffff;
    d1 = i2d<CONV>(c1);
  }
  int32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i];
  if (s == 0x12345678) sink[0] = 1;
}

// Hybrid 2: scalars pre-divided by p (t_i = c_i / p, one DMUL per scalar per step) and the
// rounding constant folded into the first FMA at 2^-8 granularity (magic 1.5*2^44 + 0.5):
// u = a t1 + b t2 + c t3 + magic in 3 DFMA, q = floor(S/p + 1/2) = bits [8, 40) of u (SHF),
// r = S - q p exactly in wrapping int32 (4 IMAD), |r| <= 0.51 p.  4 FP64 ops per update.
constexpr double kMagic8 = 26388279066624.5;  // 1.5 * 2^44 + 0.5
__device__ __forceinline__ int32_t hyb_q(double u) {
  return static_cast<int32_t>(__funnelshift_r(static_cast<uint32_t>(__double2loint(u)),
                                              static_cast<uint32_t>(__double2hiint(u)), 8));
}
template <int CONV>
__global__ void k_row_hyb2(uint32_t pp, uint32_t* sink) {
  const double pd = pp, pinv = 1.0 / pd;
  const int32_t negp = -static_cast<int32_t>(pp);
  int32_t A[kRow], B[kRow];
  double Ad[kRow], Bd[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = static_cast<int32_t>((threadIdx.x * 131u + i) % pp) - static_cast<int32_t>(pp / 2);
    B[i] = static_cast<int32_t>((threadIdx.x * 17u + 3u * i + 1u) % pp) - static_cast<int32_t>(pp / 2);
    Ad[i] = A[i];
    Bd[i] = B[i];
  }
  int32_t c1 = 12345, c2 = 678, c3 = 91011;
  double t1 = c1 * pinv, t2 = c2 * pinv, t3 = c3 * pinv;
#pragma unroll 1
  for (int it = 0; it < kIt / 8; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) {
      const double u = __fma_rn(t3, Bd[t], __fma_rn(t2, Bd[t - 1], __fma_rn(t1, Ad[t], kMagic8)));
      const int32_t r = c1 * A[t] + c2 * B[t - 1] + c3 * B[t] + hyb_q(u) * negp;
      A[t] = r;
      Ad[t] = i2d<CONV>(r);
    }
#pragma unroll
    for (int t = 0; t < kRow; ++t) {
      int32_t x = A[t];
      A[t] = B[t];
      B[t] = x;
      double y = Ad[t];
      Ad[t] = Bd[t];
      Bd[t] = y;
    }
    c1 ^= A[3] & 0xffff;
    t1 = i2d<CONV>(c1) * pinv;
  }
  int32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i];
  if (s == 0x12345678) sink[0] = 1;
}

// Exactness of the hybrid update on random symmetric inputs: out[i] = r, host checks
// r == S mod p (as integers) and |r| <= 0.51 p.
__global__ void k_hyb_check(uint32_t pp, const int32_t* in, int32_t* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double pinv = 1.0 / static_cast<double>(pp);
  const int32_t negp = -static_cast<int32_t>(pp);
  const int32_t* x = in + 6 * i;  // c1 a c2 b c3 c
  const double u = __fma_rn(x[4] * pinv, static_cast<double>(x[5]),
                            __fma_rn(x[2] * pinv, static_cast<double>(x[3]),
                                     __fma_rn(x[0] * pinv, static_cast<double>(x[1]), kMagic8)));
  out[i] = x[0] * x[1] + x[2] * x[3] + x[4] * x[5] + hyb_q(u) * negp;
}

// Swap-free rows (the real K3 is fully unrolled, so the A/B role swap costs nothing there):
// two half-iterations per loop trip, the second updating B from A.
__global__ void k_row_mont_ns(uint32_t p, uint32_t pneg, uint32_t* sink) {
  Mod M{p, pneg};
  uint32_t A[kRow], B[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = (threadIdx.x * 131u + i) % p;
    B[i] = (threadIdx.x * 17u + 3u * i + 1u) % p;
  }
  uint32_t c1 = 12345u, c2 = 678u, c3 = 91011u;
#pragma unroll 1
  for (int it = 0; it < kIt / 16; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) A[t] = mmul3(c1, A[t], c2, B[t - 1], c3, B[t], M);
    c1 = csub(c1 ^ A[3], p);
#pragma unroll
    for (int t = 1; t < kRow; ++t) B[t] = mmul3(c1, B[t], c2, A[t - 1], c3, A[t], M);
    c1 = csub(c1 ^ B[3], p);
  }
  uint32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i] ^ B[i];
  if (s == 0x12345678u) sink[0] = s;
}
template <int CONV>
__global__ void k_row_hyb2_ns(uint32_t pp, uint32_t* sink) {
  const double pd = pp, pinv = 1.0 / pd;
  const int32_t negp = -static_cast<int32_t>(pp);
  int32_t A[kRow], B[kRow];
  double Ad[kRow], Bd[kRow];
  for (int i = 0; i < kRow; ++i) {
    A[i] = static_cast<int32_t>((threadIdx.x * 131u + i) % pp) - static_cast<int32_t>(pp / 2);
    B[i] = static_cast<int32_t>((threadIdx.x * 17u + 3u * i + 1u) % pp) - static_cast<int32_t>(pp / 2);
    Ad[i] = A[i];
    Bd[i] = B[i];
  }
  int32_t c1 = 12345, c2 = 678, c3 = 91011;
  double t1 = c1 * pinv, t2 = c2 * pinv, t3 = c3 * pinv;
#pragma unroll 1
  for (int it = 0; it < kIt / 16; ++it) {
#pragma unroll
    for (int t = 1; t < kRow; ++t) {
      const double u = __fma_rn(t3, Bd[t], __fma_rn(t2, Bd[t - 1], __fma_rn(t1, Ad[t], kMagic8)));
      const int32_t r = c1 * A[t] + c2 * B[t - 1] + c3 * B[t] + hyb_q(u) * negp;
      A[t] = r;
      Ad[t] = i2d<CONV>(r);
    }
    c1 ^= A[3] & 0xffff;
    t1 = i2d<CONV>(c1) * pinv;
#pragma unroll
    for (int t = 1; t < kRow; ++t) {
      const double u = __fma_rn(t3, Ad[t], __fma_rn(t2, Ad[t - 1], __fma_rn(t1, Bd[t], kMagic8)));
      const int32_t r = c1 * B[t] + c2 * A[t - 1] + c3 * A[t] + hyb_q(u) * negp;
      B[t] = r;
      Bd[t] = i2d<CONV>(r);
    }
    c1 ^= B[3] & 0xffff;
    t1 = i2d<CONV>(c1) * pinv;
  }
  int32_t s = 0;
  for (int i = 0; i < kRow; ++i) s ^= A[i] ^ B[i];
  if (s == 0x12345678) sink[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto tm = [&](const char* name, double ops_per_thread, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double threads = static_cast<double>(sms) * 8 * 256;
    const double rate = threads * ops_per_thread / (best * 1e-3);
    printf("%-12s %8.3f ms  %10.3f T/s  %7.2f per SM per clk@1.965GHz\n", name, best, rate * 1e-12,
           rate / sms / 1.965e9);
  };
  const int G = sms * 8, T = 256;
  tm("imad", 1.0 * kC * kIt, [&] { k_imad<<<G, T>>>(0x9e3779b9u, 7u, sink); });
  tm("imad_hi", 1.0 * kC * kIt, [&] { k_imad_hi<<<G, T>>>(0x9e3779b9u, sink); });
  tm("imad_wide", 1.0 * kC * kIt, [&] { k_imad_wide<<<G, T>>>(0x9e3779b9u, sink); });
  tm("dfma", 1.0 * kC * kIt, [&] { k_dfma<<<G, T>>>(1.0000001, 1e-9, sink); });
  tm("mixed(pairs)", 1.0 * kC * kIt, [&] { k_mixed<<<G, T>>>(0x9e3779b9u, 7u, 1.0000001, 1e-9, sink); });
  const uint32_t p = 715827881u;  // < 2^32 / 6 (value irrelevant for timing)
  uint32_t inv = p;
  for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
  tm("row_mont", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_mont<<<G, T>>>(p, 0u - inv, sink); });
  tm("row_shoup", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_shoup<<<G, T>>>(p, sink); });
  tm("mixed_wide", 1.0 * kC * kIt, [&] { k_mixed_wide<<<G, T>>>(0x9e3779b9u, 1.0000001, 1e-9, sink); });
  tm("mixed_hi", 1.0 * kC * kIt, [&] { k_mixed_hi<<<G, T>>>(0x9e3779b9u, 1.0000001, 1e-9, sink); });
  tm("row_fp", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_fp<<<G, T>>>(109000001u, sink); });
  tm("row_both(x2)", 2.0 * (kRow - 1) * (kIt / 8), [&] { k_row_both<<<G, T>>>(p, 0u - inv, 109000001u, sink); });
  tm("row_hyb_i2f", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb<0><<<G, T>>>(1073741789u, sink); });
  tm("row_hyb_magic", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb<1><<<G, T>>>(1073741789u, sink); });
  tm("row_hyb2_i2f", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb2<0><<<G, T>>>(1073741789u, sink); });
  tm("row_hyb2_magic", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb2<1><<<G, T>>>(1073741789u, sink); });
  tm("row_mont_ns", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_mont_ns<<<G, T>>>(p, 0u - inv, sink); });
  tm("row_hyb2_ns_i2f", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb2_ns<0><<<G, T>>>(1073741789u, sink); });
  tm("row_hyb2_ns_mag", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_hyb2_ns<1><<<G, T>>>(1073741789u, sink); });
  tm("row_mont2", 1.0 * (kRow - 1) * (kIt / 8), [&] { k_row_mont<<<G, T>>>(p, 0u - inv, sink); });
  {
    const int n = 1 << 22;
    const uint32_t pc = 1415999977u;  // near the top of the prime window (odd; primality irrelevant here)
    int32_t *din, *dout;
    cudaMalloc(&din, 6ull * n * 4);
    cudaMalloc(&dout, 1ull * n * 4);
    int32_t* hin = new int32_t[6ull * n];
    int32_t* hout = new int32_t[n];
    uint64_t s = 88172645463325252ull;
    auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    const int64_t lim = static_cast<int64_t>(0.51 * pc);
    for (int64_t i = 0; i < 6ll * n; ++i) {
      int64_t v = static_cast<int64_t>(rnd() % (2 * lim + 1)) - lim;
      if (i % 97 == 0) v = (i & 1) ? lim : -lim;  // extremes
      hin[i] = static_cast<int32_t>(v);
    }
    cudaMemcpy(din, hin, 6ull * n * 4, cudaMemcpyHostToDevice);
    k_hyb_check<<<(n + 255) / 256, 256>>>(pc, din, dout, n);
    cudaMemcpy(hout, dout, 4ull * n, cudaMemcpyDeviceToHost);
    long bad = 0, wide = 0;
    for (int i = 0; i < n; ++i) {
      const int32_t* x = hin + 6ll * i;
      __int128 S = (__int128)x[0] * x[1] + (__int128)x[2] * x[3] + (__int128)x[4] * x[5];
      __int128 d = S - hout[i];
      if (d % pc != 0) ++bad;
      if (hout[i] > lim || hout[i] < -lim) ++wide;
    }
    printf("hyb_check n=%d wrong=%ld out_of_range=%ld\n", n, bad, wide);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
