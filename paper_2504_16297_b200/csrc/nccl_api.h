// nccl_api.h -- NCCL loaded at run time (dlopen), for state sharding.
//
// libptsbe.so does not link NCCL: a process that already loaded one (torch's
// bundled libnccl.so.2) shares it through the soname, and hosts without NCCL can
// still load the library for single-GPU work.  Only the calls sharding needs.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace ptsbe {
namespace nccl {

struct Api {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

inline Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);   // already in the process?
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) { a.why = "libnccl.so.2 not found"; return; }
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(lib, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(lib, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(lib, "ncclCommDestroy");
    a.group_start = (decltype(a.group_start))dlsym(lib, "ncclGroupStart");
    a.group_end = (decltype(a.group_end))dlsym(lib, "ncclGroupEnd");
    a.send = (decltype(a.send))dlsym(lib, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(lib, "ncclRecv");
    a.all_reduce = (decltype(a.all_reduce))dlsym(lib, "ncclAllReduce");
    a.error_string = (decltype(a.error_string))dlsym(lib, "ncclGetErrorString");
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.group_start || !a.group_end || !a.send ||
        !a.recv || !a.all_reduce || !a.error_string) {
      a.why = "NCCL symbols missing";
      return;
    }
    a.ok = true;
  });
  return a;
}

}  // namespace nccl
}  // namespace ptsbe
