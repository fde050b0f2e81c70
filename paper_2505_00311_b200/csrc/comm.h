// comm.h — the exchange layer of the row-sharded path.
//
// K~ is split by rows; the primal side is replicated, so the only exchanges are
// all-reduces of
//   * the local K~^T y partial sums (n doubles per accepted step),
//   * the line-search sums ||dy||^2 and <dy, K dx> (2 doubles per trial),
//   * the row-side Eq. 9 maxima / sums (5 doubles per candidate per check),
//   * a stop flag per check (time limit decided collectively),
//   * the Ruiz / Pock-Chambolle column norms, ||h||_inf and eta0 / omega0 (setup).
// Every backend returns bitwise-identical results on every rank, so every
// rank takes the same decisions (asserted by tests/test_dist.py).
//
// Backends:
//   NcclComm      NCCL over NVLink / NVSwitch, loaded at run time (dlopen) so
//                 that single-GPU use of libpdcs.so has no NCCL dependency.  In a
//                 process that already imported torch, libnccl.so.2 is resident
//                 and RTLD_NOLOAD returns that copy; PDCS_NCCL_LIB names another.
//   LoopbackComm  N ranks as N contexts of ONE process on one device, driven
//                 from N host threads (tests: gpurun gives one GPU and NCCL
//                 refuses two ranks on one device).  Each call is a host
//                 rendezvous: every rank publishes its device buffer, then each
//                 rank sums the N buffers in rank order into scratch on its own
//                 stream (identical kernel, identical order -> identical bits),
//                 a second rendezvous, then the copy back.  Not graph-capturable.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

namespace pdcs {

enum class RedOp { Sum, Max };

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // In-place all-reduce of count doubles on stream st.  Returns "" or an error.
  virtual std::string allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) = 0;
  // May the calls be recorded into a CUDA graph (stream capture)?
  virtual bool capturable() const = 0;
  virtual const char* name() const = 0;
  // This rank failed a call and will not join further collectives.
  virtual void on_error(const std::string&) {}
};

// ---------------------------------------------------------------- NCCL
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
    std::vector<const char*> names;
    if (const char* e = std::getenv("PDCS_NCCL_LIB")) names.push_back(e);
    names.push_back("libnccl.so.2");
    names.push_back("libnccl.so");
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (h) break;
    }
    if (!h)
      for (const char* nm : names) {
        h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
      }
    if (!h) { err = "cannot load libnccl.so.2 (import torch first, or set PDCS_NCCL_LIB)"; return false; }
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

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  std::string init(const void* unique_id, int rank_, int world_) {
    std::string e;
    if (!nccl().load(e)) return e;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    const ncclResult_t r = nccl().CommInitRank(&comm, world_, id, rank_);
    if (r != ncclSuccess) return std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
    rank = rank_;
    world = world_;
    return "";
  }
  std::string allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) override {
    if (count == 0) return "";
    const ncclResult_t r =
        nccl().AllReduce(buf, buf, count, ncclFloat64, op == RedOp::Sum ? ncclSum : ncclMax, comm, st);
    return r == ncclSuccess ? "" : std::string("ncclAllReduce: ") + nccl().GetErrorString(r);
  }
  bool capturable() const override { return true; }
  const char* name() const override { return "nccl"; }
};

// ---------------------------------------------------------------- loopback
constexpr int kLoopMaxRanks = 16;

struct LoopPtrs {
  const double* p[kLoopMaxRanks];
};

// out[i] = buf_0[i] (+|max) buf_1[i] ... in rank order (deterministic, the
// same bits on every rank).
__global__ void k_loop_reduce(LoopPtrs in, int world, size_t count, int op, double* out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    double s = in.p[0][i];
    for (int r = 1; r < world; ++r) {
      const double v = in.p[r][i];
      s = op == 0 ? s + v : fmax(s, v);
    }
    out[i] = s;
  }
}

// One in-process group of `world` ranks (pdcs_loopback in include/pdcs.h).
struct LoopbackGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  std::string abort_msg;
  double timeout_s = 600.0;
  std::vector<double*> bufs;
  std::vector<size_t> counts;
  std::vector<int> ops;

  explicit LoopbackGroup(int w) : world(w), bufs(w, nullptr), counts(w, 0), ops(w, 0) {
    if (const char* e = std::getenv("PDCS_LOOPBACK_TIMEOUT_S")) timeout_s = std::atof(e);
  }
  // Rendezvous of all ranks; "" or an error (abort by a peer, timeout).
  std::string barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return "loopback group aborted: " + abort_msg;
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return "";
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return gen != g || aborted; });
    if (aborted) return "loopback group aborted: " + abort_msg;
    if (!ok) {
      aborted = true;
      abort_msg = "rendezvous timeout (a rank stopped calling collectives)";
      cv.notify_all();
      return "loopback " + abort_msg;
    }
    return "";
  }
  void abort(const std::string& why) {
    std::lock_guard<std::mutex> lk(mu);
    if (!aborted) { aborted = true; abort_msg = why; }
    cv.notify_all();
  }
};

struct LoopbackComm : Comm {
  LoopbackGroup* g = nullptr;
  double* scratch = nullptr;
  size_t cap = 0;
  ~LoopbackComm() override {
    if (scratch) cudaFree(scratch);
  }
  std::string allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) override {
    if (count == 0) return "";
    if (count > cap) {
      if (scratch) cudaFree(scratch);
      scratch = nullptr;
      if (cudaMalloc(&scratch, count * sizeof(double)) != cudaSuccess) return "loopback: cudaMalloc failed";
      cap = count;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return "loopback: stream sync failed";
    g->bufs[rank] = buf;
    g->counts[rank] = count;
    g->ops[rank] = op == RedOp::Sum ? 0 : 1;
    std::string e = g->barrier();                       // every rank's input is ready
    if (!e.empty()) return e;
    for (int r = 0; r < world; ++r)
      if (g->counts[r] != count || g->ops[r] != g->ops[rank]) {
        g->abort("mismatched collective across ranks");
        return "loopback: mismatched collective across ranks";
      }
    LoopPtrs P{};
    for (int r = 0; r < world; ++r) P.p[r] = g->bufs[r];
    const int blocks = (int)std::min<size_t>((count + 255) / 256, 4096);
    k_loop_reduce<<<blocks, 256, 0, st>>>(P, world, count, g->ops[rank], scratch);
    if (cudaStreamSynchronize(st) != cudaSuccess) return "loopback: reduce kernel failed";
    e = g->barrier();                                   // every rank has read every input
    if (!e.empty()) return e;
    if (cudaMemcpyAsync(buf, scratch, count * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return "loopback: copy failed";
    return "";
  }
  bool capturable() const override { return false; }
  const char* name() const override { return "loopback"; }
  void on_error(const std::string& msg) override { g->abort("rank " + std::to_string(rank) + ": " + msg); }
};

}  // namespace pdcs
