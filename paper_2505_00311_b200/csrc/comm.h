// comm.h — NCCL, loaded at run time (dlopen) so that single-GPU use of
// libpdcs.so has no NCCL dependency.  In a process that already imported
// torch, libnccl.so.2 is resident and RTLD_NOLOAD returns that copy.
//
// Row-sharded PDCS: K~ is split by rows; the
// primal side is replicated, so the only exchanges are all-reduces of
//   * the local K~^T y partial sums (n doubles per accepted step),
//   * the line-search sums ||dy||^2 and <dy, K dx> (2 doubles per trial),
//   * the row-side Eq. 9 maxima / sums (5 doubles per candidate per check),
//   * the Ruiz / Pock-Chambolle column norms and eta0 / omega0 scalars (setup).
// NCCL returns bitwise-identical results on every rank, so every rank takes
// the same decisions.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <string>

namespace pdcs {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (h) break;
    }
    if (!h)
      for (const char* nm : names) {
        h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
      }
    if (!h) { err = "cannot load libnccl.so.2"; return false; }
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllReduce || !CommDestroy || !GetErrorString) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};

inline NcclApi& nccl() {
  static NcclApi api;
  return api;
}

}  // namespace pdcs
