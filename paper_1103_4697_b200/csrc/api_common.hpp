// Shared host plumbing of the C ABI: error mapping, device contexts (stream,
// scratch, pinned staging), call statistics and result buffers.
#pragma once
#include <cuda_runtime.h>

#include <chrono>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ctg.h"

namespace ctg {

struct ApiError {
  ctg_status code;
  std::string msg;
  ApiError(ctg_status c, std::string m) : code(c), msg(std::move(m)) {}
};

#define CTG_CUDA_CHECK(expr)                                                                        \
  do {                                                                                              \
    cudaError_t ctg_err_ = (expr);                                                                  \
    if (ctg_err_ != cudaSuccess)                                                                    \
      throw ::ctg::ApiError(CTG_CUDA, std::string("CUDA error: ") + cudaGetErrorString(ctg_err_) + \
                                          " at " + __FILE__ + ":" + std::to_string(__LINE__));      \
  } while (0)

void set_last_error(const std::string& msg);
ctg_call_stats& stats_tls();

template <class F>
ctg_status guarded(F&& f) {
  try {
    f();
    set_last_error("");
    return CTG_OK;
  } catch (const ApiError& e) {
    set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return CTG_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return CTG_INTERNAL;
  }
}

// Resolves opts->device (or the current device); throws CTG_CUDA without a device.
int select_device(const ctg_opts* opts);

// Sets the requested device for the scope of a call and restores the previous one.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const ctg_opts* opts);
  ~DeviceGuard();
};
struct PlanDeviceGuard {
  int prev = -1;
  explicit PlanDeviceGuard(int device);
  ~PlanDeviceGuard();
};

// The square-freeness probe a single-curve ctg_resultant leaves behind (lift.cpp:64-67 calls
// yun_squarefree(R) right after resultant): gcd(R, R') modulo three of the resultant's own
// primes, run on its interpolated residues while the host decodes R.  ctg_yun_squarefree
// uses it when its input equals R exactly (compared limb by limb with the copy kept here).
struct SqfProbeCache {
  bool valid = false;
  int n = -1;                        // deg R
  // Two slots, alternating per call, so a probe still running never holds up the next result
  // (its inputs are copied on the compute stream; the probe runs on a low-priority stream).
  struct Slot {
    uint32_t* d_rows = nullptr;      // 3 rows of plain residues
    size_t d_cap = 0;                // words
    int32_t* d_out = nullptr;        // [2 * 3] results
    int32_t* h_out = nullptr;        // pinned copy of the results
    uint8_t* d_blk = nullptr;        // R in the library's block layout (device copy of the packed result)
    uint8_t* h_blk = nullptr;        // ... and its pinned host copy (DMA behind the probe: no host time)
    size_t blk_cap = 0;
    cudaEvent_t done = nullptr;      // probe results and h_blk are ready
  };
  Slot slot[2];
  int cur = 0;                       // slot of the latest probe
  size_t blk_off = 0, blk_total = 0; // R's block in h_blk: byte offset, limbs (n + 1 coefficients)
};
// Per-device context: one non-blocking stream, grow-only device scratch and pinned staging.
struct Ctx {
  std::mutex mu;
  SqfProbeCache sqf;
  int device = -1;
  cudaStream_t stream = nullptr;
  std::vector<void*> scratch;
  std::vector<size_t> scratch_bytes;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* pinned_in = nullptr;
  size_t pinned_in_bytes = 0;
  cudaStream_t copy = nullptr;            // D2H stream (overlaps the next chunk's kernels)
  cudaStream_t copy_stream();
  cudaStream_t aux[2] = {nullptr, nullptr};  // extra compute streams (batch chunks rotate)
  cudaStream_t aux_stream(int i = 0);
  // Compute streams of decreasing priority (level 0 = the device's greatest priority): batch
  // chunk i runs at level i % prio_levels(), so the oldest chunk in flight wins the block
  // scheduler and chunks complete in order while younger ones fill the idle SMs.
  cudaStream_t prio[8] = {};
  int nprio = 0;
  int prio_levels();
  cudaStream_t prio_stream(int level);
  cudaStream_t probe = nullptr;           // lowest priority: the square-freeness probe left behind results
  cudaStream_t probe_stream();
  uint32_t* scratch_u32(int slot, size_t words);
  uint32_t* pinned_u32(size_t words);     // D2H staging
  uint8_t* pinned_input(size_t bytes);    // H2D staging
};
Ctx& context(int device);
cudaStream_t resolve_stream(int device, void* stream);

struct CallTimer {
  using clk = std::chrono::steady_clock;
  clk::time_point t0, t_last;
  CallTimer();
  double lap();
  void mark_setup();
  void mark_h2d();
  void mark_device();
  void finish();
  void finish_total();  // total only (phases were accumulated by the callee)
};

// Runs fn(i) for i in [0, n) on a persistent host thread pool (inline when n <= 1).
// Used for per-curve marshaling of batches (parsing, result decoding).
void parallel_for(int n, const std::function<void(int)>& fn);

// Decoded coefficient (sign-magnitude), used to fill library-owned result buffers.
struct UCoeff {
  int8_t sign = 0;
  std::vector<uint32_t> limbs;
};
// Trims trailing zero coefficients and allocates/fills a ctg_upoly_buf.
void fill_upoly(const std::vector<UCoeff>& coeffs, ctg_upoly_buf* out);

// Result-buffer storage.  Every ctg_upoly_buf owns one block: a 16-byte header right
// before limb_off, then limb_off[n+1], limbs[total], sign[n].  Blocks are either single
// mallocs or members of a refcounted arena shared by one batch call (one allocation and
// one release for the whole batch); ctg_upoly_free handles both.
size_t upoly_block_bytes(size_t n_coeffs, size_t total_limbs);
void upoly_alloc(ctg_upoly_buf* out, size_t n_coeffs, size_t total_limbs);  // single block
struct UpolyArena {
  uint8_t* base = nullptr;
  UpolyArena() = default;
  UpolyArena(const UpolyArena&) = delete;
  UpolyArena& operator=(const UpolyArena&) = delete;
  UpolyArena(UpolyArena&& o) noexcept : base(o.base) { o.base = nullptr; }
  UpolyArena& operator=(UpolyArena&& o) noexcept {
    base = o.base;
    o.base = nullptr;
    return *this;
  }
  // Creates an arena for `members` blocks totalling `bytes` (sum of upoly_block_bytes);
  // pinned: page-locked host memory (a D2H target), from its own recycled cache.
  void create(size_t bytes, int64_t members, bool pinned = false);
  // First byte of the member area (block offsets are relative to it).
  uint8_t* members() const;
  // Places a block at byte offset `off` (from the first block) into out.
  void place(ctg_upoly_buf* out, size_t off, size_t n_coeffs, size_t total_limbs) const;
  // Returns an arena that never got its members (error paths) to its cache.
  void discard();
};

}  // namespace ctg
