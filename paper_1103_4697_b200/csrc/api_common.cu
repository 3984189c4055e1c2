#include "api_common.hpp"

#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>

namespace ctg {

static thread_local std::string g_last_error;
static thread_local ctg_call_stats g_stats;

void set_last_error(const std::string& msg) { g_last_error = msg; }
ctg_call_stats& stats_tls() { return g_stats; }

int select_device(const ctg_opts* opts) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw ApiError(CTG_CUDA, "no CUDA device available (libctg has no CPU fallback)");
  int dev = 0;
  if (opts && opts->device >= 0) {
    if (opts->device >= count) throw ApiError(CTG_INVALID, "ctg_opts.device out of range");
    dev = opts->device;
  } else {
    CTG_CUDA_CHECK(cudaGetDevice(&dev));
  }
  return dev;
}

DeviceGuard::DeviceGuard(const ctg_opts* opts) {
  if (opts && opts->device >= 0) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw ApiError(CTG_CUDA, "no CUDA device available (libctg has no CPU fallback)");
    if (opts->device >= count) throw ApiError(CTG_INVALID, "ctg_opts.device out of range");
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(opts->device));
  }
}
DeviceGuard::~DeviceGuard() {
  if (prev >= 0) cudaSetDevice(prev);
}
PlanDeviceGuard::PlanDeviceGuard(int device) {
  cudaGetDevice(&prev);
  if (prev == device) {
    prev = -1;
    return;
  }
  CTG_CUDA_CHECK(cudaSetDevice(device));
}
PlanDeviceGuard::~PlanDeviceGuard() {
  if (prev >= 0) cudaSetDevice(prev);
}

uint32_t* Ctx::scratch_u32(int slot, size_t words) {
  if (scratch.size() <= static_cast<size_t>(slot)) {
    scratch.resize(slot + 1, nullptr);
    scratch_bytes.resize(slot + 1, 0);
  }
  const size_t bytes = std::max<size_t>(4, words * 4);
  if (scratch_bytes[slot] < bytes) {
    CTG_CUDA_CHECK(cudaStreamSynchronize(stream));
    cudaFree(scratch[slot]);
    scratch[slot] = nullptr;
    CTG_CUDA_CHECK(cudaMalloc(&scratch[slot], bytes));
    scratch_bytes[slot] = bytes;
  }
  return static_cast<uint32_t*>(scratch[slot]);
}

uint32_t* Ctx::pinned_u32(size_t words) {
  const size_t bytes = std::max<size_t>(4, words * 4);
  if (pinned_bytes < bytes) {
    CTG_CUDA_CHECK(cudaStreamSynchronize(stream));
    cudaFreeHost(pinned);
    pinned = nullptr;
    CTG_CUDA_CHECK(cudaMallocHost(&pinned, bytes));
    pinned_bytes = bytes;
  }
  return static_cast<uint32_t*>(pinned);
}

Ctx& context(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Ctx>> ctxs;
  std::lock_guard<std::mutex> lock(mu);
  auto& c = ctxs[device];
  if (!c) {
    c.reset(new Ctx());
    c->device = device;
    int prev = 0;
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(device));
    CTG_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    // Keep stream-ordered allocations cached in the pool between calls.
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaSetDevice(prev);
  }
  return *c;
}

cudaStream_t resolve_stream(int device, void* stream) {
  if (stream) return static_cast<cudaStream_t>(stream);
  return context(device).stream;
}

CallTimer::CallTimer() {
  t0 = t_last = clk::now();
  std::memset(&g_stats, 0, sizeof(g_stats));
}
double CallTimer::lap() {
  auto t = clk::now();
  double ms = std::chrono::duration<double, std::milli>(t - t_last).count();
  t_last = t;
  return ms;
}
void CallTimer::mark_setup() { g_stats.setup_ms = lap(); }
void CallTimer::mark_h2d() { g_stats.h2d_ms = lap(); }
void CallTimer::mark_device() { g_stats.device_ms = lap(); }
void CallTimer::finish() {
  g_stats.decode_ms = lap();
  g_stats.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

void fill_upoly(const std::vector<UCoeff>& coeffs, ctg_upoly_buf* out) {
  size_t n = coeffs.size();
  while (n > 0 && coeffs[n - 1].sign == 0) --n;
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) total += coeffs[i].limbs.size();
  out->n_coeffs = static_cast<int32_t>(n);
  out->sign = static_cast<int8_t*>(std::malloc(std::max<size_t>(1, n)));
  out->limb_off = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (n + 1)));
  out->limbs = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * std::max<size_t>(1, total)));
  if (!out->sign || !out->limb_off || !out->limbs) throw std::bad_alloc();
  uint32_t off = 0;
  for (size_t i = 0; i < n; ++i) {
    out->sign[i] = coeffs[i].sign;
    out->limb_off[i] = off;
    std::memcpy(out->limbs + off, coeffs[i].limbs.data(), 4 * coeffs[i].limbs.size());
    off += static_cast<uint32_t>(coeffs[i].limbs.size());
  }
  out->limb_off[n] = off;
}

}  // namespace ctg

extern "C" {

void ctg_upoly_free(ctg_upoly_buf* buf) {
  if (!buf) return;
  std::free(buf->sign);
  std::free(buf->limb_off);
  std::free(buf->limbs);
  std::memset(buf, 0, sizeof(*buf));
}

void ctg_sqf_free(ctg_sqf_buf* buf) {
  if (!buf) return;
  std::free(buf->unit_limbs);
  for (int i = 0; i < buf->n_factors; ++i) ctg_upoly_free(&buf->factors[i]);
  std::free(buf->factors);
  std::free(buf->mult);
  std::memset(buf, 0, sizeof(*buf));
}

const char* ctg_last_error(void) { return ctg::g_last_error.c_str(); }
int32_t ctg_abi_version(void) { return CTG_ABI_VERSION; }
int32_t ctg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
void ctg_last_call_stats(ctg_call_stats* out) {
  if (out) *out = ctg::g_stats;
}

}  // extern "C"
