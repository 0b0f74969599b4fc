// NCCL resolved at run time (the libnccl torch already loaded, else the
// system one), so libirismpc_gpu.so has no link-time NCCL dependency.  Used by
// party mode (party.cu: send/recv between the three parties) and the
// DB-sharded query (api.cu: query broadcast + partial all-gather).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace irisgpu {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommSplit) comm_split = nullptr;  // optional (streaming sharded queries)
  bool ok = false;
};

inline const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
    a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
    a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    a.broadcast = (decltype(a.broadcast))dlsym(h, "ncclBroadcast");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
    a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
    a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
    a.comm_split = (decltype(a.comm_split))dlsym(h, "ncclCommSplit");
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.send && a.recv && a.broadcast &&
           a.all_gather && a.group_start && a.group_end && a.error_string;
    return a;
  }();
  return api;
}

}  // namespace irisgpu
