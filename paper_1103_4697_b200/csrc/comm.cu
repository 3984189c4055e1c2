// NCCL binding (dlopen) and the ctg_comm C ABI.  See comm.hpp.
#include <dlfcn.h>

#include <cstring>
#include <map>
#include <type_traits>
#include <mutex>

#include "api_common.hpp"
#include "comm.hpp"

namespace ctg {

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // RTLD_NOLOAD first: a copy the process already holds (torch's) is the one to share.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    a.ok = sym(a.GetUniqueId, "ncclGetUniqueId") && sym(a.CommInitRank, "ncclCommInitRank") &&
           sym(a.CommInitAll, "ncclCommInitAll") && sym(a.CommDestroy, "ncclCommDestroy") &&
           sym(a.AllGather, "ncclAllGather") && sym(a.Send, "ncclSend") && sym(a.Recv, "ncclRecv") &&
           sym(a.GroupStart, "ncclGroupStart") &&
           sym(a.GroupEnd, "ncclGroupEnd") && sym(a.GetErrorString, "ncclGetErrorString");
    if (!a.ok) a.why = "libnccl.so.2 lacks an expected entry point";
    return a;
  }();
  if (!api.ok) throw ApiError(CTG_CUDA, "NCCL unavailable: " + api.why);
  return api;
}

bool nccl_available() {
  try {
    nccl();
    return true;
  } catch (const ApiError&) {
    return false;
  }
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw ApiError(CTG_CUDA, std::string(what) + ": NCCL error: " + nccl().GetErrorString(r));
}

const std::vector<ncclComm_t>& device_set_comms(const std::vector<int>& devices) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;  // process lifetime
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(devices);
  if (it != cache.end()) return it->second;
  std::vector<ncclComm_t> comms(devices.size());
  int prev = 0;
  cudaGetDevice(&prev);
  const ncclResult_t r = nccl().CommInitAll(comms.data(), static_cast<int>(devices.size()), devices.data());
  cudaSetDevice(prev);
  nccl_check(r, "ncclCommInitAll");
  return cache.emplace(devices, std::move(comms)).first->second;
}

}  // namespace ctg

using namespace ctg;

extern "C" {

ctg_status ctg_comm_unique_id(uint8_t* id) {
  return guarded([&] {
    if (!id) throw ApiError(CTG_INVALID, "comm: null id");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == CTG_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, &u, sizeof(u));
  });
}

ctg_status ctg_comm_init_rank(int32_t nranks, int32_t rank, const uint8_t* id, int32_t device, ctg_comm** comm) {
  return guarded([&] {
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks) throw ApiError(CTG_INVALID, "comm: bad arguments");
    ctg_opts o{};
    o.device = device;
    DeviceGuard g(&o);
    auto c = std::make_unique<ctg_comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = select_device(&o);
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    nccl_check(nccl().CommInitRank(&c->nc, nranks, u, rank), "ncclCommInitRank");
    *comm = c.release();
  });
}

void ctg_comm_destroy(ctg_comm* comm) {
  if (!comm) return;
  if (comm->nc && nccl_available()) nccl().CommDestroy(comm->nc);
  delete comm;
}

ctg_status ctg_comm_all_gather(ctg_comm* comm, const void* d_send, void* d_recv, size_t words, void* stream) {
  return guarded([&] {
    if (!comm || !comm->nc) throw ApiError(CTG_INVALID, "comm: null communicator");
    PlanDeviceGuard g(comm->device);
    nccl_check(nccl().AllGather(d_send, d_recv, words, ncclUint32, comm->nc,
                                resolve_stream(comm->device, stream)),
               "ncclAllGather");
  });
}

ctg_status ctg_comm_all_to_all(ctg_comm* comm, const void* d_send, void* d_recv, size_t words, void* stream) {
  return guarded([&] {
    if (!comm || !comm->nc) throw ApiError(CTG_INVALID, "comm: null communicator");
    PlanDeviceGuard g(comm->device);
    const cudaStream_t st = resolve_stream(comm->device, stream);
    const auto* s = static_cast<const uint32_t*>(d_send);
    auto* r = static_cast<uint32_t*>(d_recv);
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int q = 0; q < comm->nranks; ++q) {
      nccl_check(nccl().Send(s + q * words, words, ncclUint32, q, comm->nc, st), "ncclSend");
      nccl_check(nccl().Recv(r + q * words, words, ncclUint32, q, comm->nc, st), "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  });
}

}  // extern "C"
