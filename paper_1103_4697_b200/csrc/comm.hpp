// Prime sharding across GPUs: NCCL, loaded at run time, and the
// communicators the sharded resultant (api_res.cu) exchanges residues over.
//
// libctg does not link NCCL: the single-GPU path never touches it, and a process that
// already loaded one (e.g. torch's bundled libnccl.so.2) must not get a second copy.  The
// first multi-GPU call dlopen()s "libnccl.so.2" (the already-loaded one if any) and binds
// the handful of entry points below.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/ctg.h"

namespace ctg {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;  // load failure
};
// Loaded once per process; throws CTG_CUDA-class ApiError when NCCL is unavailable.
const NcclApi& nccl();
bool nccl_available();
void nccl_check(ncclResult_t r, const char* what);

// Communicators over a set of DISTINCT local devices (ncclCommInitAll), cached per set.
const std::vector<ncclComm_t>& device_set_comms(const std::vector<int>& devices);

}  // namespace ctg

// Multi-process communicator: this process is rank `rank` of `nranks` (one GPU each).
struct ctg_comm {
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t nc = nullptr;
};
