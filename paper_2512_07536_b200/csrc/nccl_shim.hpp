// NCCL entry points of the sharded projection, resolved at first use. The
// library does not link libnccl: torch ships its own (newer) libnccl.so.2,
// and a load-time dependency would bind the process to whichever copy came
// first. An already loaded copy is preferred (RTLD_NOLOAD), else the system's.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"

namespace tpb {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
};

inline const NcclApi& nccl() {
    static const NcclApi api = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        NcclApi a;
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
        return a;
    }();
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.group_start || !api.group_end)
        throw Error(kCuda, "NCCL (libnccl.so.2) not found: the sharded projection needs it");
    return api;
}

}  // namespace tpb
