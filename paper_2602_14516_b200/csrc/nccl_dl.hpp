// nccl_dl.hpp — NCCL, resolved at first use with dlopen (host only).
//
// The plan search has exactly one collective: the
// per-candidate SLO counts (int64 sum) and invalid/pruned flags (max) of every
// GPU's shard, all-reduced over NVLink before the argmax. The library does
// not link libnccl at build time: a Python process has usually loaded
// PyTorch's bundled libnccl.so.2 already, and a second, different NCCL under
// the same soname would clash. dlopen("libnccl.so.2") returns the copy that is
// already resident, or loads the system one. Types and enum values come from
// the NCCL header; only the symbols are resolved at run time.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace pdg {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;  // non-empty: NCCL unavailable
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      const char* e = dlerror();
      api.error = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto get = [&](const char* name, auto* fn) {
      *reinterpret_cast<void**>(fn) = dlsym(h, name);
      if (!*reinterpret_cast<void**>(fn) && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
    };
    get("ncclGetUniqueId", &api.GetUniqueId);
    get("ncclCommInitRank", &api.CommInitRank);
    get("ncclCommInitAll", &api.CommInitAll);
    get("ncclCommDestroy", &api.CommDestroy);
    get("ncclAllReduce", &api.AllReduce);
    get("ncclGroupStart", &api.GroupStart);
    get("ncclGroupEnd", &api.GroupEnd);
    get("ncclGetErrorString", &api.GetErrorString);
  });
  return api;
}

inline std::string nccl_error(ncclResult_t r) {
  const NcclApi& n = nccl();
  return n.GetErrorString ? n.GetErrorString(r) : ("nccl error " + std::to_string(static_cast<int>(r)));
}

}  // namespace pdg
