// lms_nccl.cuh -- NCCL, loaded at run time (dlopen of libnccl.so.2), for the
// sharded band search's two small exchanges (seed records, final records)
// over NVLink / NVSwitch.  The library links without NCCL; entry points that
// need it report LMS_ERR_INVALID when it cannot be loaded.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace lmsb {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

// The process-wide NCCL binding (loaded once; .ok false when unavailable).
const NcclApi& nccl();

}  // namespace lmsb
