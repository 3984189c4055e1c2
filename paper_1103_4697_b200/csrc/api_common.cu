#include "api_common.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <thread>

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

cudaStream_t Ctx::copy_stream() {
  if (!copy) {
    int prev = 0;
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(device));
    CTG_CUDA_CHECK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    cudaSetDevice(prev);
  }
  return copy;
}

cudaStream_t Ctx::aux_stream(int i) {
  if (!aux[i]) {
    int prev = 0;
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(device));
    CTG_CUDA_CHECK(cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking));
    cudaSetDevice(prev);
  }
  return aux[i];
}

int Ctx::prio_levels() {
  if (!nprio) {
    int least = 0, greatest = 0;
    CTG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    nprio = std::max(1, std::min(8, least - greatest + 1));
  }
  return nprio;
}

cudaStream_t Ctx::prio_stream(int level) {
  level %= prio_levels();
  if (!prio[level]) {
    int prev = 0;
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(device));
    int least = 0, greatest = 0;
    CTG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CTG_CUDA_CHECK(cudaStreamCreateWithPriority(&prio[level], cudaStreamNonBlocking, greatest + level));
    cudaSetDevice(prev);
  }
  return prio[level];
}

cudaStream_t Ctx::probe_stream() {
  if (!probe) {
    int prev = 0;
    cudaGetDevice(&prev);
    CTG_CUDA_CHECK(cudaSetDevice(device));
    int least = 0, greatest = 0;
    CTG_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CTG_CUDA_CHECK(cudaStreamCreateWithPriority(&probe, cudaStreamNonBlocking, least));
    cudaSetDevice(prev);
  }
  return probe;
}

uint8_t* Ctx::pinned_input(size_t bytes) {
  bytes = std::max<size_t>(16, bytes);
  if (pinned_in_bytes < bytes) {
    CTG_CUDA_CHECK(cudaStreamSynchronize(stream));
    cudaFreeHost(pinned_in);
    pinned_in = nullptr;
    CTG_CUDA_CHECK(cudaMallocHost(&pinned_in, bytes));
    pinned_in_bytes = bytes;
  }
  return static_cast<uint8_t*>(pinned_in);
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
void CallTimer::finish_total() {
  g_stats.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}
void CallTimer::finish() {
  g_stats.decode_ms = lap();
  g_stats.total_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

namespace {
// Persistent pool for per-curve host work.  A call publishes a Job; workers claim indices
// with an atomic counter (no lock per item) and, after a job, spin ~200 us for the next one
// before sleeping, so the back-to-back parallel_for calls of one batch do not pay a
// futex wake-up each.  `active_` guards the stack-allocated Job: the caller unpublishes it
// and waits until no worker still holds it.
class Pool {
 public:
  Pool() {
    unsigned hc = std::thread::hardware_concurrency();
    nthreads_ = static_cast<int>(std::min(16u, std::max(1u, hc)));
    for (int t = 1; t < nthreads_; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> call(call_mu_);  // one parallel_for at a time
    Job job{&fn, n};
    job_.store(&job);
    {
      std::lock_guard<std::mutex> l(mu_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    work(&job);
    while (job.done.load(std::memory_order_acquire) < n) std::this_thread::yield();
    job_.store(nullptr);
    while (active_.load() != 0) std::this_thread::yield();
  }

 private:
  struct Job {
    const std::function<void(int)>* fn;
    int n;
    std::atomic<int> next{0}, done{0};
  };
  static void work(Job* j) {
    for (int i = j->next.fetch_add(1); i < j->n; i = j->next.fetch_add(1)) {
      (*j->fn)(i);
      j->done.fetch_add(1, std::memory_order_release);
    }
  }
  void loop() {
    using clk = std::chrono::steady_clock;
    uint64_t seen = gen_.load();
    while (true) {
      const auto t_end = clk::now() + std::chrono::microseconds(200);
      while (gen_.load(std::memory_order_acquire) == seen && !stop_.load() && clk::now() < t_end)
        std::this_thread::yield();
      if (gen_.load() == seen && !stop_.load()) {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_.load() || gen_.load() != seen; });
      }
      if (stop_.load()) return;
      seen = gen_.load();
      active_.fetch_add(1);
      if (Job* j = job_.load()) work(j);
      active_.fetch_sub(1);
    }
  }
  int nthreads_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_;
  std::atomic<Job*> job_{nullptr};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> active_{0};
  std::atomic<bool> stop_{false};
};
}  // namespace

// Set while a thread runs items of a parallel_for: a nested parallel_for (e.g. a content gcd
// inside a batch's per-input work) runs inline instead of re-entering the pool (whose one-job-
// at-a-time lock would deadlock).
static thread_local bool tls_in_parallel_for = false;

void parallel_for(int n, const std::function<void(int)>& fn) {
  if (n <= 1 || tls_in_parallel_for) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  static Pool pool;
  // Exceptions are captured per index and the first one rethrown on the caller's thread.
  std::vector<std::exception_ptr> errs(n);
  pool.run(n, [&](int i) {
    const bool outer = tls_in_parallel_for;
    tls_in_parallel_for = true;
    try {
      fn(i);
    } catch (...) {
      errs[i] = std::current_exception();
    }
    tls_in_parallel_for = outer;
  });
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

namespace {
constexpr uint64_t kSingleMagic = 0x31666675625f6774ull;  // "tg_buff1"
constexpr uint64_t kMemberMagic = 0x32666675625f6774ull;  // "tg_buff2"
constexpr uint64_t kArenaMagic = 0x33666675625f6774ull;   // "tg_buff3"
struct BufHdr {
  uint64_t magic;
  uint64_t aux;  // member: byte offset back to the arena header; arena: live members
};
size_t pad16(size_t x) { return (x + 15) & ~static_cast<size_t>(15); }

// Arena blocks: [ArenaHdr | members...].  Released arenas are kept in a small cache and
// handed to the next batch call, so steady-state batches write into pages that are already
// mapped (a fresh multi-MB malloc is an mmap whose first-touch faults cost more than the
// decode itself).
struct ArenaHdr {
  BufHdr h;         // magic, live members
  uint64_t cap;     // usable bytes after the header
  uint64_t pinned;  // 1: page-locked (cudaMallocHost), the D2H target of device-packed results
};
class ArenaCache {
 public:
  explicit ArenaCache(bool pinned) : pinned_(pinned) {}
  uint8_t* take(size_t bytes) {
    {
      std::lock_guard<std::mutex> l(mu_);
      size_t best = blocks_.size();
      for (size_t i = 0; i < blocks_.size(); ++i) {
        const uint64_t cap = reinterpret_cast<ArenaHdr*>(blocks_[i])->cap;
        if (cap >= bytes && cap <= 4 * bytes + (1u << 20) &&
            (best == blocks_.size() || cap < reinterpret_cast<ArenaHdr*>(blocks_[best])->cap))
          best = i;
      }
      if (best < blocks_.size()) {
        uint8_t* b = blocks_[best];
        held_ -= reinterpret_cast<ArenaHdr*>(b)->cap;
        blocks_.erase(blocks_.begin() + static_cast<std::ptrdiff_t>(best));
        return b;
      }
    }
    const size_t cap = (bytes + 65535) & ~static_cast<size_t>(65535);
    uint8_t* b = nullptr;
    if (pinned_) {
      void* p = nullptr;
      if (cudaMallocHost(&p, sizeof(ArenaHdr) + cap) != cudaSuccess) throw std::bad_alloc();
      b = static_cast<uint8_t*>(p);
    } else {
      b = static_cast<uint8_t*>(std::malloc(sizeof(ArenaHdr) + cap));
    }
    if (!b) throw std::bad_alloc();
    reinterpret_cast<ArenaHdr*>(b)->cap = cap;
    reinterpret_cast<ArenaHdr*>(b)->pinned = pinned_ ? 1u : 0u;
    return b;
  }
  void give(uint8_t* b) {
    const uint64_t cap = reinterpret_cast<ArenaHdr*>(b)->cap;
    {
      std::lock_guard<std::mutex> l(mu_);
      if (blocks_.size() < kMaxBlocks && held_ + cap <= kMaxHeld) {
        blocks_.push_back(b);
        held_ += cap;
        return;
      }
    }
    release(b);
  }
  ~ArenaCache() {
    for (uint8_t* b : blocks_) release(b);
  }

 private:
  void release(uint8_t* b) const {
    if (pinned_)
      cudaFreeHost(b);
    else
      std::free(b);
  }
  bool pinned_;
  static constexpr size_t kMaxBlocks = 32;
  static constexpr uint64_t kMaxHeld = 1ull << 30;
  std::mutex mu_;
  std::vector<uint8_t*> blocks_;
  uint64_t held_ = 0;
};
ArenaCache& arena_cache(bool pinned = false) {
  static ArenaCache* c = new ArenaCache(false);  // never destroyed: results may be freed at exit
  static ArenaCache* cp = new ArenaCache(true);
  return pinned ? *cp : *c;
}

void place_block(uint8_t* block, uint64_t magic, uint64_t aux, ctg_upoly_buf* out, size_t n, size_t total) {
  auto* h = reinterpret_cast<BufHdr*>(block);
  h->magic = magic;
  h->aux = aux;
  out->n_coeffs = static_cast<int32_t>(n);
  out->limb_off = reinterpret_cast<uint32_t*>(block + sizeof(BufHdr));
  out->limbs = out->limb_off + (n + 1);
  out->sign = reinterpret_cast<int8_t*>(out->limbs + total);
}
}  // namespace

size_t upoly_block_bytes(size_t n, size_t total) { return pad16(sizeof(BufHdr) + 4 * (n + 1) + 4 * total + n); }

void upoly_alloc(ctg_upoly_buf* out, size_t n, size_t total) {
  auto* block = static_cast<uint8_t*>(std::malloc(upoly_block_bytes(n, total)));
  if (!block) throw std::bad_alloc();
  place_block(block, kSingleMagic, 0, out, n, total);
}

void UpolyArena::create(size_t bytes, int64_t members, bool pinned) {
  base = arena_cache(pinned).take(bytes);
  auto* h = reinterpret_cast<BufHdr*>(base);
  h->magic = kArenaMagic;
  h->aux = static_cast<uint64_t>(members);
}

uint8_t* UpolyArena::members() const { return base + sizeof(ArenaHdr); }

void UpolyArena::discard() {
  if (!base) return;
  reinterpret_cast<BufHdr*>(base)->magic = 0;
  arena_cache(reinterpret_cast<ArenaHdr*>(base)->pinned != 0).give(base);
  base = nullptr;
}

void UpolyArena::place(ctg_upoly_buf* out, size_t off, size_t n, size_t total) const {
  uint8_t* block = base + sizeof(ArenaHdr) + off;
  place_block(block, kMemberMagic, static_cast<uint64_t>(block - base), out, n, total);
}

void fill_upoly(const std::vector<UCoeff>& coeffs, ctg_upoly_buf* out) {
  size_t n = coeffs.size();
  while (n > 0 && coeffs[n - 1].sign == 0) --n;
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) total += coeffs[i].limbs.size();
  upoly_alloc(out, n, total);
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
  using namespace ctg;
  if (!buf) return;
  if (buf->limb_off) {
    uint8_t* block = reinterpret_cast<uint8_t*>(buf->limb_off) - sizeof(BufHdr);
    auto* h = reinterpret_cast<BufHdr*>(block);
    if (h->magic == kSingleMagic) {
      h->magic = 0;
      std::free(block);
    } else if (h->magic == kMemberMagic) {
      h->magic = 0;
      uint8_t* base = block - h->aux;
      auto* ah = reinterpret_cast<BufHdr*>(base);
      if (__atomic_sub_fetch(&ah->aux, 1, __ATOMIC_ACQ_REL) == 0) {
        ah->magic = 0;
        arena_cache(reinterpret_cast<ArenaHdr*>(base)->pinned != 0).give(base);
      }
    }
  }
  std::memset(buf, 0, sizeof(*buf));
}

void ctg_upoly_free_batch(ctg_upoly_buf* bufs, int32_t n) {
  if (!bufs) return;
  for (int32_t i = 0; i < n; ++i) ctg_upoly_free(&bufs[i]);
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
