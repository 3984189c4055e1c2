#include <algorithm>
// Prime tables: Montgomery constants, roots of unity (for the NTT size N) and the
// fixed-point CRT constants: (M/p_k)^{-1} mod p_k, 1/p_k and the digits of M/p_k in two
// layouts -- 16-bit digits for the IMAD GEMM, and the byte-sliced, shift-expanded
// operand of the tensor-core GEMM:
//   Bt8[l][4k + a] = byte (l - a) of M/p_k,
// so that  sum_k y_k (M/p_k) = sum_l 2^(8 l) sum_{k,a} byte_a(y_k) Bt8[l][4k+a]
// is ONE u8 x u8 -> s32 matrix product (exact: 4P * 255^2 < 2^31 for P < 8250).
#include <cuda_runtime.h>

#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "api_common.hpp"
#include "internal.hpp"

namespace ctg {

CrtTables::~CrtTables() {
  cudaFree(d_pc);
  cudaFree(d_minv);
  cudaFree(d_Mk16);
  cudaFree(d_M16);
  cudaFree(d_Bt8);
  cudaFree(d_M8);
  cudaFree(d_twinv);
  cudaFree(d_rpow);
}

std::shared_ptr<CrtTables> build_tables(int device, const std::vector<uint32_t>& primes, uint32_t N) {
  const int P = static_cast<int>(primes.size());
  auto T = std::make_shared<CrtTables>();
  T->device = device;
  T->N = N;
  T->P = P;
  T->primes = primes;
  // M = prod p_k
  Big Mb{1u};
  for (uint32_t p : primes) Mb = big_mul_u32(Mb, p);
  T->LM = static_cast<int>(Mb.size());
  T->L16 = 2 * T->LM;
  T->L8 = 4 * T->LM;
  T->L8p = (T->L8 + kI8TileL - 1) / kI8TileL * kI8TileL;
  T->Kp = (4 * P + 127) / 128 * 128;  // 128-byte K stages (TMA / tcgen05 GEMM; 2 mma.sync stages)
  T->use_i8 = P <= kI8MaxPrimes;
  std::vector<PrimeConst> pc(P);
  std::vector<double> minv(P);
  std::vector<uint32_t> Mk16(static_cast<size_t>(P) * T->L16, 0u), M16(T->L16, 0u),
      M8(std::max(T->L8, T->L8p), 0u);  // zero-padded to L8p: the fused CRT epilogue reads whole tiles
  std::vector<uint8_t> Bt8;
  if (T->use_i8) Bt8.assign(static_cast<size_t>(T->L8p) * T->Kp, 0u);
  for (int l = 0; l < T->LM; ++l) {
    M16[2 * l] = Mb[l] & 0xffffu;
    M16[2 * l + 1] = Mb[l] >> 16;
    for (int a = 0; a < 4; ++a) M8[4 * l + a] = (Mb[l] >> (8 * a)) & 0xffu;
  }
  for (int k = 0; k < P; ++k) {
    const uint32_t p = primes[k];
    Mod M = make_mod(p);
    PrimeConst& c = pc[k];
    c.p = M.p;
    c.pneg = M.pneg;
    c.r2 = M.r2;
    c.one = M.one;
    const uint32_t g = N > 1 ? primitive_root(p) : 1u;
    const uint32_t w = N > 1 ? pow_mod_u32(g, (p - 1) / N, p) : 1u;
    const uint32_t wi = inv_mod_u32(w, p);
    c.omega = static_cast<uint32_t>((static_cast<uint64_t>(w) << 32) % p);
    c.omega_inv = static_cast<uint32_t>((static_cast<uint64_t>(wi) << 32) % p);
    c.scale = inv_mod_u32(N % p, p);
    uint32_t rem = 0;
    Big Mk = big_div_u32(Mb, p, &rem);
    const uint32_t mk_mod = big_mod_u32(Mk.data(), static_cast<int>(Mk.size()), p);
    const uint32_t ck = inv_mod_u32(mk_mod, p);
    c.crt_c = static_cast<uint32_t>((static_cast<uint64_t>(ck) << 32) % p);
    minv[k] = 1.0 / static_cast<double>(p);
    for (size_t l = 0; l < Mk.size(); ++l) {
      Mk16[static_cast<size_t>(k) * T->L16 + 2 * l] = Mk[l] & 0xffffu;
      Mk16[static_cast<size_t>(k) * T->L16 + 2 * l + 1] = Mk[l] >> 16;
    }
    if (T->use_i8) {
      const int nbytes = 4 * static_cast<int>(Mk.size());
      for (int i = 0; i < nbytes; ++i) {
        const uint8_t byte = static_cast<uint8_t>(Mk[i / 4] >> (8 * (i % 4)));
        if (!byte) continue;
        for (int a = 0; a < 4; ++a) {
          const int l = i + a;
          if (l < T->L8) Bt8[static_cast<size_t>(l) * T->Kp + 4 * k + a] = byte;
        }
      }
    }
  }
  // K1 limb weights: R^(l+2) mod p, so that mmul(limb, w_l) = limb * 2^(32 l) in Montgomery form.
  std::vector<uint32_t> rpow(static_cast<size_t>(P) * kRedL);
  for (int k = 0; k < P; ++k) {
    const uint64_t p = primes[k], r = (static_cast<uint64_t>(1) << 32) % p;
    uint64_t x = (r * r) % p;
    for (int l = 0; l < kRedL; ++l) {
      rpow[static_cast<size_t>(k) * kRedL + l] = static_cast<uint32_t>(x);
      x = (x * r) % p;
    }
  }
  CTG_CUDA_CHECK(cudaMalloc(&T->d_rpow, sizeof(uint32_t) * rpow.size()));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_rpow, rpow.data(), sizeof(uint32_t) * rpow.size(), cudaMemcpyHostToDevice));
  T->h_pc = pc;
  T->log2M = 0;
  for (uint32_t p : primes) T->log2M += std::log2(static_cast<double>(p));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_pc, sizeof(PrimeConst) * P));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_minv, sizeof(double) * P));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_Mk16, sizeof(uint32_t) * Mk16.size()));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_M16, sizeof(uint32_t) * M16.size()));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_M8, sizeof(uint32_t) * M8.size()));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_pc, pc.data(), sizeof(PrimeConst) * P, cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_minv, minv.data(), sizeof(double) * P, cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_Mk16, Mk16.data(), sizeof(uint32_t) * Mk16.size(), cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_M16, M16.data(), sizeof(uint32_t) * M16.size(), cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_M8, M8.data(), sizeof(uint32_t) * M8.size(), cudaMemcpyHostToDevice));
  if (T->use_i8) {
    CTG_CUDA_CHECK(cudaMalloc(&T->d_Bt8, Bt8.size()));
    CTG_CUDA_CHECK(cudaMemcpy(T->d_Bt8, Bt8.data(), Bt8.size(), cudaMemcpyHostToDevice));
  }
  if (N >= 1 && P > 0) {
    CTG_CUDA_CHECK(cudaMalloc(&T->d_twinv, sizeof(uint32_t) * static_cast<size_t>(P) * N));
    launch_twiddles(T->d_pc, P, static_cast<int>(N), T->d_twinv);
    CTG_CUDA_CHECK(cudaGetLastError());
    CTG_CUDA_CHECK(cudaDeviceSynchronize());
  }
  return T;
}

std::shared_ptr<CrtTables> get_tables(int device, uint32_t N, const std::vector<uint32_t>& primes) {
  using Key = std::tuple<int, uint32_t, std::vector<uint32_t>>;
  static std::mutex mu;
  static std::map<Key, std::pair<std::shared_ptr<CrtTables>, uint64_t>> cache;
  static uint64_t tick = 0;
  constexpr size_t kCap = 64;
  std::lock_guard<std::mutex> lock(mu);
  Key key = std::make_tuple(device, N, primes);
  auto it = cache.find(key);
  if (it != cache.end()) {
    it->second.second = ++tick;
    return it->second.first;
  }
  auto T = build_tables(device, primes, N);
  if (cache.size() >= kCap) {
    auto lru = cache.begin();
    for (auto j = cache.begin(); j != cache.end(); ++j)
      if (j->second.second < lru->second.second) lru = j;
    cache.erase(lru);  // in-flight users hold their own reference
  }
  cache.emplace(std::move(key), std::make_pair(T, ++tick));
  return T;
}

}  // namespace ctg
