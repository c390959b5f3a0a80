// okg_nccl.h -- the NCCL entry points the one-process-per-GPU slab transport
// uses, resolved at run time (dlopen of libnccl.so.2: torch's copy when torch
// is already loaded in the process, else the system one), so libokg.so has no
// link-time NCCL dependency and single-process contexts never touch NCCL.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace okg {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// nullptr + message when NCCL cannot be loaded
inline const NcclApi* nccl_api(std::string* why) {
  static NcclApi api;
  static std::string err;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      err = std::string("dlopen(libnccl.so.2): ") + (e ? e : "not found");
    } else {
      bool all = true;
      auto sym = [&](auto& fp, const char* name) {
        fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
        if (!fp) {
          all = false;
          err = std::string("libnccl.so.2 lacks ") + name;
        }
      };
      sym(api.GetUniqueId, "ncclGetUniqueId");
      sym(api.CommInitRank, "ncclCommInitRank");
      sym(api.CommDestroy, "ncclCommDestroy");
      sym(api.AllReduce, "ncclAllReduce");
      sym(api.Send, "ncclSend");
      sym(api.Recv, "ncclRecv");
      sym(api.GroupStart, "ncclGroupStart");
      sym(api.GroupEnd, "ncclGroupEnd");
      sym(api.GetErrorString, "ncclGetErrorString");
      api.ok = all;
    }
  }
  if (!api.ok && why) *why = err;
  return api.ok ? &api : nullptr;
}

}  // namespace okg
