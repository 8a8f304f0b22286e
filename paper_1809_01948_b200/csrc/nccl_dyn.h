// nccl_dyn.h -- NCCL entry points resolved at run time (dlopen "libnccl.so.2").
//
// The library does not link NCCL: a process that already loaded NCCL (torch
// does) reuses that copy, a single-GPU process never needs it, and the .so
// loads on machines without NCCL.  Types come from the system nccl.h.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <string>

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  // optional (NCCL >= 2.14): communicator limits (maxCTAs of the reduction comm)
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) {
    const char* e = dlerror();
    api.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return api;
  }
#define NCCL_SYM(field, name)                                      \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(lib, name)); \
  if (!api.field) {                                                \
    api.err = std::string("missing NCCL symbol ") + name;          \
    return api;                                                    \
  }
  NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
  NCCL_SYM(CommInitRank, "ncclCommInitRank");
  NCCL_SYM(CommDestroy, "ncclCommDestroy");
  NCCL_SYM(AllReduce, "ncclAllReduce");
  NCCL_SYM(AllGather, "ncclAllGather");
  NCCL_SYM(Send, "ncclSend");
  NCCL_SYM(Recv, "ncclRecv");
  NCCL_SYM(GroupStart, "ncclGroupStart");
  NCCL_SYM(GroupEnd, "ncclGroupEnd");
  NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef NCCL_SYM
  api.CommInitRankConfig = reinterpret_cast<decltype(api.CommInitRankConfig)>(
      dlsym(lib, "ncclCommInitRankConfig"));
  api.ok = true;
  return api;
}
