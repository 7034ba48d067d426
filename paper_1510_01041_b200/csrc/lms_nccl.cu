// lms_nccl.cu -- run-time binding of NCCL (see lms_nccl.cuh).
#include "lms_nccl.cuh"

#include <dlfcn.h>

#include <mutex>

namespace lmsb {

namespace {

template <typename F>
bool bind(void* h, const char* name, F* fn) {
  *fn = reinterpret_cast<F>(dlsym(h, name));
  return *fn != nullptr;
}

NcclApi load() {
  NcclApi api;
  void* h = nullptr;
  for (const char* lib : {"libnccl.so.2", "libnccl.so"}) {
    h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) return api;
  api.ok = bind(h, "ncclGetUniqueId", &api.GetUniqueId) &&
           bind(h, "ncclCommInitRank", &api.CommInitRank) &&
           bind(h, "ncclCommInitAll", &api.CommInitAll) &&
           bind(h, "ncclCommDestroy", &api.CommDestroy) &&
           bind(h, "ncclAllGather", &api.AllGather) && bind(h, "ncclGroupStart", &api.GroupStart) &&
           bind(h, "ncclGroupEnd", &api.GroupEnd) &&
           bind(h, "ncclGetErrorString", &api.GetErrorString) &&
           bind(h, "ncclGetVersion", &api.GetVersion);
  return api;
}

}  // namespace

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  std::call_once(once, [] { api = load(); });
  return api;
}

}  // namespace lmsb
