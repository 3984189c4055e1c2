// Prime tables: Montgomery constants, roots of unity (for the NTT size N) and the
// fixed-point CRT constants M/p_k (16-bit digits), (M/p_k)^{-1} mod p_k, 1/p_k.
#include <cuda_runtime.h>

#include <cmath>

#include "api_common.hpp"
#include "internal.hpp"

namespace ctg {

CrtTables::~CrtTables() {
  cudaFree(d_pc);
  cudaFree(d_minv);
  cudaFree(d_Mk16);
  cudaFree(d_M16);
}

// ---------------------------------------------------------------------------
// Per-prime constants and fixed-point CRT tables for an ordered prime set.
// ---------------------------------------------------------------------------

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
  std::vector<PrimeConst> pc(P);
  std::vector<double> minv(P);
  std::vector<uint32_t> Mk16(static_cast<size_t>(P) * T->L16, 0u), M16(T->L16, 0u);
  for (int l = 0; l < T->LM; ++l) {
    M16[2 * l] = Mb[l] & 0xffffu;
    M16[2 * l + 1] = Mb[l] >> 16;
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
  }
  T->h_pc = pc;
  T->log2M = 0;
  for (uint32_t p : primes) T->log2M += std::log2(static_cast<double>(p));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_pc, sizeof(PrimeConst) * P));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_minv, sizeof(double) * P));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_Mk16, sizeof(uint32_t) * Mk16.size()));
  CTG_CUDA_CHECK(cudaMalloc(&T->d_M16, sizeof(uint32_t) * M16.size()));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_pc, pc.data(), sizeof(PrimeConst) * P, cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_minv, minv.data(), sizeof(double) * P, cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_Mk16, Mk16.data(), sizeof(uint32_t) * Mk16.size(), cudaMemcpyHostToDevice));
  CTG_CUDA_CHECK(cudaMemcpy(T->d_M16, M16.data(), sizeof(uint32_t) * M16.size(), cudaMemcpyHostToDevice));
  return T;
}

}  // namespace ctg
