// pdcs.cu — libpdcs.so: C ABI (include/pdcs.h) and the host state machine of
// Alg. 1.  Every step of the method runs in the kernels of
// ops.cuh / kernels.cuh / spmv.cuh / cones.cuh; the host only validates input,
// lays data out in HBM, enqueues kernels on the caller's stream and reads
// back the few control flags the next launch depends on.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pdcs.h"
#include "ops.cuh"
#include "tiled.cuh"
#include "panels.cuh"
#include "comm.h"

using namespace pdcs;

namespace {

thread_local std::string g_create_error;

struct CudaErr {
  cudaError_t e;
  const char* what;
  int line;
};

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t _e = (call);                                            \
    if (_e != cudaSuccess) throw CudaErr{_e, #call, __LINE__};          \
  } while (0)

struct StatusErr {
  pdcs_status st;
  std::string msg;
};
[[noreturn]] void fail(pdcs_status st, const std::string& msg) { throw StatusErr{st, msg}; }

// Device memory of every context (include/pdcs.h, pdcs_set_allocator): the
// caller's allocator when one is set, else cudaMalloc / cudaFree.
std::atomic<pdcs_alloc_fn> g_alloc{nullptr};
std::atomic<pdcs_free_fn> g_free{nullptr};
std::atomic<void*> g_alloc_user{nullptr};
// Default: a library-owned stream-ordered pool per device that keeps freed
// memory (release threshold = max), used synchronously: an allocation is
// complete when dev_alloc returns, and dev_free waits for the device as
// cudaFree does.  Multi-GB cudaMalloc / cudaFree calls had cost 0.1-2 s each,
// run to run, in setup and destroy (the driver maps and unmaps the pages);
// the pool maps a context's peak once per process.  PDCS_POOL=0: cudaMalloc.
struct DevPool {
  cudaMemPool_t pool = nullptr;
  cudaStream_t st = nullptr;
};
std::mutex g_pool_mu;
DevPool g_pool[64];
DevPool* dev_pool() {
  static const bool off = std::getenv("PDCS_POOL") && std::atoi(std::getenv("PDCS_POOL")) == 0;
  if (off) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  DevPool& P = g_pool[dev];
  if (!P.pool) {
    cudaMemPoolProps pr{};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    if (cudaMemPoolCreate(&P.pool, &pr) != cudaSuccess) { P.pool = nullptr; return nullptr; }
    uint64_t keep = ~(uint64_t)0;
    cudaMemPoolSetAttribute(P.pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (cudaStreamCreateWithFlags(&P.st, cudaStreamNonBlocking) != cudaSuccess) {
      cudaMemPoolDestroy(P.pool);
      P.pool = nullptr;
      return nullptr;
    }
  }
  return &P;
}
void* dev_alloc(size_t bytes) {
  if (pdcs_alloc_fn f = g_alloc.load()) {
    void* p = f(bytes, g_alloc_user.load());
    if (!p) fail(PDCS_ERR_CUDA, "caller allocator returned NULL for " + std::to_string(bytes) + " bytes");
    return p;
  }
  void* p = nullptr;
  // PDCS_DEBUG_POISON=1: every new buffer starts as 0xff bytes (NaN doubles, -1
  // ids), so a read of memory no kernel wrote shows up (tests, diagnostics)
  static const bool poison = std::getenv("PDCS_DEBUG_POISON") && std::atoi(std::getenv("PDCS_DEBUG_POISON"));
  if (DevPool* P = dev_pool()) {
    CK(cudaMallocFromPoolAsync(&p, bytes, P->pool, P->st));
    if (poison) CK(cudaMemsetAsync(p, 0xff, bytes, P->st));
    CK(cudaStreamSynchronize(P->st));
    return p;
  }
  CK(cudaMalloc(&p, bytes));
  if (poison) CK(cudaMemset(p, 0xff, bytes));
  return p;
}
void dev_free(void* p) {
  if (pdcs_free_fn f = g_free.load()) { f(p, g_alloc_user.load()); return; }
  if (DevPool* P = dev_pool()) {
    cudaDeviceSynchronize();                     // as cudaFree: no kernel may still use p
    cudaFreeAsync(p, P->st);
    cudaStreamSynchronize(P->st);
    return;
  }
  cudaFree(p);
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    free_();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void free_() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free_(); }
};

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
  d.alloc(h.size());
  if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

template <class T>
void take(DBuf<T>& to, DBuf<T>& from) {
  to.free_();
  std::swap(to.p, from.p);
  std::swap(to.n, from.n);
}

// Bank balancing of nb warp blocks (tiled.cuh k_tile_balance_w, one warp each).
void launch_tile_balance(const TDefer* dseg, const std::vector<TDefer>&, const int2* dblk, int64_t nb, int elem,
                         const int32_t* rowptr, const uint16_t* pcol, const int32_t* pperm, uint16_t* bcol,
                         int32_t* bperm, uint16_t* ncol, int32_t* nperm, cudaStream_t st) {
  if (nb <= 0) return;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>((nb + kBalWarps - 1) / kBalWarps, (int64_t)sms * 16));
  k_tile_balance_w<<<(unsigned)g, 32 * kBalWarps, 0, st>>>(dseg, dblk, nb, elem, rowptr, pcol, pperm, bcol, bperm,
                                                          ncol, nperm);
}

// staged share of the entries above which the tiled copy is built
constexpr double kTiledMinFrac = 0.3;

int grid_for(int64_t n, int sms, int per_sm = 8) {
  int64_t g = (n + kThreads - 1) / kThreads;
  g = std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * per_sm));
  return (int)g;
}

// PDCS_SETUP_TRACE=1: wall ms of the setup phases on stderr (diagnostics).
struct SetupTrace {
  bool on = std::getenv("PDCS_SETUP_TRACE") && std::atoi(std::getenv("PDCS_SETUP_TRACE"));
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, cudaStream_t st = nullptr, bool sync = true) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pdcs setup] %-28s %9.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// ---------------------------------------------------------------- tiled format builder
// Host construction of the column-tiled format of tiled.cuh from a CSR
// structure.  perm_* give the CSR position of every entry so that the (scaled)
// values are gathered on the device afterwards.
struct TiledHost {
  std::vector<TBatch> batch;
  std::vector<TWork> work;
  std::vector<TChunk> chunk;
  std::vector<TSeg> seg;
  std::vector<int32_t> rowptr;
  std::vector<uint16_t> srow;      // per segment position: chunk-local row (rows sorted by length)
  std::vector<uint16_t> col_s;
  std::vector<int32_t> col_d;
  std::vector<int32_t> perm_s, perm_d;
  std::vector<int32_t> blkb;       // sliced staged segments: segment-relative first quad of each warp block
  int64_t scratch = 0, staged = 0, nnz = 0;
  int32_t T = 0, elem = 1;
  bool sliced = false, tma = false;   // layout / kernel decided once per build (environment read here)
  double build_ms = 0.0, ranges_ms = 0.0;
  // Parts mode (the solver's builds): the per-entry arrays stay in the
  // per-thread parts and are uploaded slice by slice at these offsets
  // (no host concatenation; tot_* are the concatenated sizes incl. padding).
  std::vector<TiledHost> parts;
  std::vector<size_t> o_s, o_d, o_rp, o_bb;
  size_t tot_s = 0, tot_d = 0, tot_rp = 0, tot_bb = 0;
  // Deferred build (device bank balancing + slicing): col_s /
  // perm_s hold the unbalanced row-major quads ("pre"); fin_s is the size of
  // the final sliced layout; dseg the staged segments, dblk their warp blocks
  // (dseg index, block).  Parts mode: o_pre offsets of the pre arrays.
  bool defer = false;
  bool devbuilt = false;           // built on the device (build_tiled_device)
  int64_t fin_s = 0;
  std::vector<TDefer> dseg;
  std::vector<int2> dblk;
  std::vector<size_t> o_pre;
  size_t tot_pre = 0;
  size_t n_s() const { return parts.empty() ? col_s.size() : tot_s; }
  size_t n_d() const { return parts.empty() ? col_d.size() : tot_d; }
};

// shared-memory tile size in bytes (PDCS_TILE_KB overrides; default 32 KB)
int tiled_tile_bytes() {
  return std::getenv("PDCS_TILE_KB") ? 1024 * std::atoi(std::getenv("PDCS_TILE_KB")) : 32768;
}

// TMA-pipelined partial kernel (opt-in, PDCS_TMA=1): it streams row-major
// segments, so the sliced layout is off with it.
bool tiled_tma_env() { return std::getenv("PDCS_TMA") && std::atoi(std::getenv("PDCS_TMA")) != 0; }
// sliced (warp-interleaved) staged segments, tiled.cuh seg_row_dot_sliced;
// PDCS_TILE_SLICED=0 keeps the row-major quad layout
bool tiled_sliced() {
  return !tiled_tma_env() && !(std::getenv("PDCS_TILE_SLICED") && std::atoi(std::getenv("PDCS_TILE_SLICED")) == 0);
}

// lanes per row for a segment with `avg` quads (staged) or entries (direct) per
// row: at least 2*lpe units per lane so that the unrolled loop body is used.
// Measured on B200 (profiles/r1_sweep_lpe.txt): lpe 4 for the pair gather,
// 2 for the single gather (PDCS_TILE_LPE overrides both).
int pick_v(double avg, int elem) {
  static const double env = std::getenv("PDCS_TILE_LPE") ? std::atof(std::getenv("PDCS_TILE_LPE")) : 0.0;
  const double lpe = env > 0 ? env : elem == 2 ? 4.0 : 2.0;
  int v = 1;
  while (v < 32 && avg >= 2.0 * v * lpe) v *= 2;
  return v;
}

// Gather schedule of k_tiled_partial (seg_rows) over one staged segment: warp
// block `blk` is the 32/V consecutive positions i0 = blk * 32/V ...; lane
// a*V + l reads quads l, l + V, ... of position i0 + a, one per time step.
// lanes[lane] lists (local row, quad) in time order; rows[] maps local rows to
// segment positions.
int tiled_blocks(int32_t nr, int V) { return (nr + 32 / V - 1) / (32 / V); }
void tiled_block_schedule(const int32_t* rp, int32_t nr, int V, int blk, std::vector<int32_t>& rows,
                          std::vector<std::vector<std::pair<int32_t, int32_t>>>& lanes) {
  rows.clear();
  lanes.assign(32, {});
  const int rpw = 32 / V;
  const int32_t i0 = blk * rpw;
  for (int a = 0; a < rpw && i0 + a < nr; ++a) {
    rows.push_back(i0 + a);
    const int32_t nq = rp[i0 + a + 1] - rp[i0 + a];
    for (int l = 0; l < V; ++l)
      for (int32_t q = l; q < nq; q += V) lanes[a * V + l].push_back({a, q});
  }
}

// Physical quad (segment-relative) of logical quad j of segment position pos:
// row-major, or sliced (warp block base + (pos in block) * V + j % V + 32 (j / V)).
int64_t quad_slot(const std::vector<int32_t>& blkb, const TSeg& S, const int32_t* rp, int32_t pos, int32_t j) {
  if (S.bb < 0) return (int64_t)rp[pos] + j;
  const int rpw = 32 / S.V;
  return (int64_t)blkb[S.bb + pos / rpw] + (pos % rpw) * S.V + j % S.V + 32 * (int64_t)(j / S.V);
}

// Re-lay the staged segments among [s0, s1) of the chunk just built (all at
// the end of H.col_s, in order) in the sliced layout of seg_row_dot_sliced.
// The bank balancing is preserved: every (warp block, time step, lane) reads
// the same quad as before.  Segments start on 16-quad boundaries (512 B of
// values, 128 B of column ids), so a warp's loads cover whole lines.
void slice_segments(TiledHost& H, int32_t s0, int32_t s1, int32_t nr) {
  int64_t base = -1;
  for (int32_t si = s0; si < s1; ++si)
    if (H.seg[si].tile >= 0) { base = H.seg[si].nz; break; }
  if (base < 0) return;
  std::vector<uint16_t> nc;
  std::vector<int32_t> np;
  for (int32_t si = s0; si < s1; ++si) {
    TSeg& S = H.seg[si];
    if (S.tile < 0) continue;
    const int32_t* rp = H.rowptr.data() + S.rp;
    const int64_t off = (int64_t)((base + (int64_t)nc.size() + 63) & ~(int64_t)63) - base;
    const int rpw = 32 / S.V;
    const int nblk = tiled_blocks(nr, S.V);
    S.bb = (int64_t)H.blkb.size();
    int64_t cur = 0;
    for (int blk = 0; blk < nblk; ++blk) {
      H.blkb.push_back((int32_t)cur);
      int32_t tmax = 0;
      for (int a = 0; a < rpw && blk * rpw + a < nr; ++a) {
        const int32_t nq = rp[blk * rpw + a + 1] - rp[blk * rpw + a];
        tmax = std::max(tmax, (nq + S.V - 1) / S.V);
      }
      cur += 32 * (int64_t)tmax;
    }
    nc.resize(off + 4 * cur, 0);
    np.resize(off + 4 * cur, -1);
    for (int32_t pos = 0; pos < nr; ++pos)
      for (int32_t j = 0; j < rp[pos + 1] - rp[pos]; ++j) {
        const int64_t from = S.nz + 4 * ((int64_t)rp[pos] + j), to = off + 4 * quad_slot(H.blkb, S, rp, pos, j);
        for (int k = 0; k < 4; ++k) { nc[to + k] = H.col_s[from + k]; np[to + k] = H.perm_s[from + k]; }
      }
    S.nz = base + off;
  }
  H.col_s.resize(base);
  H.perm_s.resize(base);
  H.col_s.insert(H.col_s.end(), nc.begin(), nc.end());
  H.perm_s.insert(H.perm_s.end(), np.begin(), np.end());
}

// The deferred build's counterpart of slice_segments: the final (sliced)
// offsets, warp-block bases and the device work list of the staged segments
// among [s0, s1), with the same sizes and alignment as slice_segments; no data
// moves (k_tile_balance_w / k_tile_slice do that on the device).
void slice_plan(TiledHost& H, int32_t s0, int32_t s1, int32_t nr) {
  bool any = false;
  for (int32_t si = s0; si < s1; ++si) any |= H.seg[si].tile >= 0;
  if (!any) return;
  const int64_t base = (H.fin_s + 7) & ~(int64_t)7;     // the first staged segment's start when built in place
  int64_t cur = 0;
  for (int32_t si = s0; si < s1; ++si) {
    TSeg& S = H.seg[si];
    if (S.tile < 0) continue;
    const int32_t* rp = H.rowptr.data() + S.rp;
    const int64_t off = ((base + cur + 63) & ~(int64_t)63) - base;
    const int rpw = 32 / S.V;
    const int nblk = tiled_blocks(nr, S.V);
    S.bb = (int64_t)H.blkb.size();
    const int32_t di = (int32_t)H.dseg.size();
    int64_t q = 0;
    for (int blk = 0; blk < nblk; ++blk) {
      H.blkb.push_back((int32_t)q);
      int32_t tmax = 0;
      for (int a = 0; a < rpw && blk * rpw + a < nr; ++a) {
        const int32_t nq = rp[blk * rpw + a + 1] - rp[blk * rpw + a];
        tmax = std::max(tmax, (nq + S.V - 1) / S.V);
      }
      q += 32 * (int64_t)tmax;
      H.dblk.push_back(make_int2(di, blk));
    }
    H.dseg.push_back(TDefer{S.nz, base + off, S.rp, S.bb, nr, S.V});
    cur = off + 4 * q;
    S.nz = base + off;
  }
  H.fin_s = base + cur;
}

// Shared-memory bank balancing of one staged segment (in place).  At every
// time step each lane of a warp reads one quad (tiled_block_schedule), and
// position k of those quads is one warp-wide ld.shared: v2.f64 for the pair
// tile, served in 4 phases of 8 lanes, f64 otherwise, 2 phases of 16 lanes
// (measured: tools/lds_probe.cu).  A phase costs as many wavefronts as the
// largest number of distinct addresses in one bank group (16-B groups: col % 8
// for pairs; 8-B groups: col % 16).  Within a row the entry order is free (its
// partial dot product is one sum), so each row's entries are redistributed over
// its own quads.  Per slot, lanes with the fewest choices go first and take the
// free bank group with the most entries left in the block (a phase needs at
// least as many wavefronts as its most loaded group has entries, so those are
// drained first); a lane that would conflict uses one of its row's pads if it
// has one, reading an address another lane already reads (a broadcast).
void balance_banks(uint16_t* cols, int32_t* perm, const int32_t* rp, int32_t nr, int V, int elem) {
  const int G = elem == 2 ? 8 : 16;                           // bank groups = lanes per phase
  const int rpw = 32 / V;
  // flat per-(row, group) buckets, filled in entry order and consumed from the
  // back; the schedule of tiled_block_schedule is computed inline (lane a*V+l
  // reads quad l + t V of block row a at step t); scratch reused across calls
  thread_local std::vector<uint16_t> ncol, bcol;
  thread_local std::vector<int32_t> nperm, bperm, bstart, bleft, left, slots;
  thread_local std::vector<uint32_t> mask;
  const int64_t nslot = 4 * (int64_t)rp[nr];
  ncol.assign(nslot, 0);
  nperm.assign(nslot, -1);
  const int nblk = tiled_blocks(nr, V);
  for (int blk = 0; blk < nblk; ++blk) {
    const int32_t i0 = blk * rpw;
    const int R = std::min<int32_t>(rpw, nr - i0);
    bstart.assign((size_t)R * G + 1, 0);
    left.assign(R, 0);
    slots.assign(R, 0);
    mask.assign(R, 0);
    int rem[16] = {0};
    int32_t tmax = 0;
    for (int a = 0; a < R; ++a) {
      const int32_t q0 = rp[i0 + a], q1 = rp[i0 + a + 1];
      tmax = std::max(tmax, (q1 - q0 + V - 1) / V);
      slots[a] = 4 * (q1 - q0);
      for (int64_t e = 4 * (int64_t)q0; e < 4 * (int64_t)q1; ++e)
        if (perm[e] >= 0) {
          const int g = cols[e] % G;
          ++bstart[(size_t)a * G + g + 1];
          mask[a] |= 1u << g;
          ++rem[g];
          ++left[a];
        }
    }
    for (size_t z = 1; z < bstart.size(); ++z) bstart[z] += bstart[z - 1];
    bleft.assign(bstart.begin(), bstart.end() - 1);            // fill cursor, then top (exclusive)
    bcol.resize(bstart.back());
    bperm.resize(bstart.back());
    for (int a = 0; a < R; ++a)
      for (int64_t e = 4 * (int64_t)rp[i0 + a]; e < 4 * (int64_t)rp[i0 + a + 1]; ++e)
        if (perm[e] >= 0) {
          const int32_t z = bleft[(size_t)a * G + cols[e] % G]++;
          bcol[z] = cols[e];
          bperm[z] = perm[e];
        }
    int unit_a[16];
    int64_t unit_slot[16];
    for (int32_t t = 0; t < tmax; ++t)
      for (int k = 0; k < 4; ++k)
        for (int ph = 0; ph < 32 / G; ++ph) {
          int nu = 0;
          for (int lane = ph * G; lane < ph * G + G; ++lane) {
            const int a = lane / V, l = lane % V;
            if (a >= R) continue;
            const int32_t q = l + t * V;
            if (q >= rp[i0 + a + 1] - rp[i0 + a]) continue;
            unit_a[nu] = a;
            unit_slot[nu] = 4 * (int64_t)(rp[i0 + a] + q) + k;
            ++nu;
          }
          // fewest choices first (stable insertion sort on the popcount of the row's groups)
          if (nu > 1) {                                             // (as a counting sort)
            int pc[16], cnt[18] = {0}, sa[16];
            int64_t ss[16];
            for (int x = 0; x < nu; ++x) { pc[x] = __builtin_popcount(mask[unit_a[x]]); ++cnt[pc[x] + 1]; }
            for (int z = 1; z < 18; ++z) cnt[z] += cnt[z - 1];
            for (int x = 0; x < nu; ++x) { const int z = cnt[pc[x]]++; sa[z] = unit_a[x]; ss[z] = unit_slot[x]; }
            for (int x = 0; x < nu; ++x) { unit_a[x] = sa[x]; unit_slot[x] = ss[x]; }
          }
          uint32_t used = 0;
          int any_col = -1;
          for (int x = 0; x < nu; ++x) {
            const int a = unit_a[x];
            const int64_t slot = unit_slot[x];
            const uint32_t avail = mask[a] & ~used;
            int g = -1;
            if (avail || (left[a] > 0 && slots[a] == left[a])) {
              uint32_t from = avail ? avail : mask[a];              // forced: a conflict
              for (; from; from &= from - 1) {                      // lowest group wins ties
                const int h = __builtin_ctz(from);
                if (g < 0 || rem[h] > rem[g]) g = h;
              }
            }
            if (g >= 0) {
              const size_t bi = (size_t)a * G + g;
              const int32_t z = --bleft[bi];
              ncol[slot] = bcol[z];
              nperm[slot] = bperm[z];
              if (bleft[bi] == bstart[bi]) mask[a] &= ~(1u << g);
              --rem[g];
              --left[a];
              used |= 1u << g;
              if (any_col < 0) any_col = ncol[slot];
            } else {                                                // pad: re-read an address
              ncol[slot] = (uint16_t)(any_col >= 0 ? any_col : 0);
              nperm[slot] = -1;
              if (any_col < 0) any_col = 0;
            }
            --slots[a];
          }
        }
  }
  std::copy(ncol.begin(), ncol.end(), cols);
  std::copy(nperm.begin(), nperm.end(), perm);
}

// Chunks [row_a, row_b) (row_a a multiple of kTRows) into H, offsets local to H.
void build_tiled_range(const int64_t* ptr, const int32_t* col, int64_t row_a, int64_t row_b, int64_t nvec,
                       int elem, int64_t group_nz, TiledHost& H) {
  const int tile_bytes = H.T * 8 * elem;
  const int32_t T = H.T;
  const int64_t stage_min = tile_bytes / 16;           // staging must save >= 2x the gather sectors
  const int64_t ntiles = (nvec + T - 1) / T;
  H.elem = elem;
  H.perm_s.reserve(ptr[row_b] - ptr[row_a]);
  H.col_s.reserve(ptr[row_b] - ptr[row_a]);
  std::vector<int64_t> cnt(ntiles, 0);
  std::vector<int32_t> segof(ntiles, -1);
  std::vector<int64_t> touched;
  const int64_t rows = row_b;
  for (int64_t r0 = row_a; r0 < rows; r0 += kTRows) {
    const int32_t nr = (int32_t)std::min<int64_t>(kTRows, rows - r0);
    touched.clear();
    for (int64_t p = ptr[r0]; p < ptr[r0 + nr]; ++p) {
      const int64_t t = col[p] / T;
      if (cnt[t]++ == 0) touched.push_back(t);
    }
    std::sort(touched.begin(), touched.end());
    // segments: direct first (if any), then staged tiles in order
    std::vector<int64_t> staged_tiles;
    int64_t direct_nz = 0;
    (void)0;
    for (int64_t t : touched) {
      if (cnt[t] >= stage_min) staged_tiles.push_back(t); else direct_nz += cnt[t];
    }
    const int32_t s_begin = (int32_t)H.seg.size();
    std::vector<int64_t> seg_nz;
    if (direct_nz) { H.seg.push_back(TSeg{-1, 1, 0, 0, -1}); seg_nz.push_back(direct_nz); }
    for (int64_t t : staged_tiles) {
      segof[t] = (int32_t)(H.seg.size() - s_begin);
      H.seg.push_back(TSeg{(int32_t)t, 1, 0, 0, -1});
      seg_nz.push_back(cnt[t]);
    }
    const int nseg = (int)seg_nz.size();
    // per-segment per-row counts (staged segments are padded to quads of 4)
    auto seg_k = [&](int64_t t) { return cnt[t] >= stage_min ? segof[t] : 0; };   // direct is index 0
    std::vector<int32_t> rc((size_t)nseg * nr, 0);
    for (int32_t i = 0; i < nr; ++i)
      for (int64_t p = ptr[r0 + i]; p < ptr[r0 + i + 1]; ++p) rc[(size_t)seg_k(col[p] / T) * nr + i]++;
    std::vector<int64_t> rpbase(nseg);
    // staged segments hold their rows longest first (stable), so that the
    // lanes of a warp run rows of about equal length; pos_of maps row -> position
    std::vector<int32_t> pos_of((size_t)nseg * nr), order(nr);
    for (int k = 0; k < nseg; ++k) {
      TSeg& S = H.seg[s_begin + k];
      const bool stg = S.tile >= 0;
      const int32_t* rck = rc.data() + (size_t)k * nr;
      for (int32_t i = 0; i < nr; ++i) order[i] = i;
      if (stg) std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return rck[a] > rck[b]; });
      rpbase[k] = (int64_t)H.rowptr.size();
      S.rp = rpbase[k];
      H.rowptr.resize(H.rowptr.size() + nr + 1, 0);
      H.srow.resize(H.rowptr.size(), 0);
      int64_t units = 0;                                  // quads (staged) or entries (direct)
      for (int32_t pos = 0; pos < nr; ++pos) {
        const int32_t i = order[pos];
        const int32_t u = stg ? (rck[i] + 3) / 4 : rck[i];
        H.rowptr[rpbase[k] + pos + 1] = H.rowptr[rpbase[k] + pos] + u;
        H.srow[rpbase[k] + pos] = (uint16_t)i;
        pos_of[(size_t)k * nr + i] = pos;
        units += u;
      }
      S.V = pick_v(stg ? (double)units / nr : (double)seg_nz[k] / nr, elem);
      if (stg) {
        // segments start on an even quad: 16-B aligned TMA sources for the column ids
        H.col_s.resize((H.col_s.size() + 7) & ~(size_t)7, 0);
        H.perm_s.resize(H.col_s.size(), -1);
        S.nz = (int64_t)H.col_s.size();
        H.col_s.resize(H.col_s.size() + 4 * units, 0);
        H.perm_s.resize(H.col_s.size(), -1);
      } else {
        S.nz = (int64_t)H.col_d.size();
        H.col_d.resize(H.col_d.size() + units);
        H.perm_d.resize(H.col_d.size());
      }
    }
    std::vector<int32_t> fill((size_t)nseg * nr, 0);
    for (int32_t i = 0; i < nr; ++i)
      for (int64_t p = ptr[r0 + i]; p < ptr[r0 + i + 1]; ++p) {
        const int64_t t = col[p] / T;
        const int k = seg_k(t);
        const TSeg& S = H.seg[s_begin + k];
        const int32_t f = fill[(size_t)k * nr + i]++;
        const int32_t pos = pos_of[(size_t)k * nr + i];
        if (S.tile >= 0) {
          const int64_t q = S.nz + 4 * (int64_t)H.rowptr[rpbase[k] + pos] + f;
          H.col_s[q] = (uint16_t)(col[p] - t * T);
          H.perm_s[q] = (int32_t)p;
          H.staged++;
        } else {
          const int64_t q = S.nz + H.rowptr[rpbase[k] + pos] + f;
          H.col_d[q] = col[p];
          H.perm_d[q] = (int32_t)p;
        }
      }
    const bool balance = !std::getenv("PDCS_TILE_BALANCE") || std::atoi(std::getenv("PDCS_TILE_BALANCE"));
    if (balance && !H.defer)
      for (int k = 0; k < nseg; ++k) {
        const TSeg& S = H.seg[s_begin + k];
        if (S.tile < 0 || S.V > 32) continue;
        balance_banks(H.col_s.data() + S.nz, H.perm_s.data() + S.nz, H.rowptr.data() + rpbase[k], nr, S.V, elem);
      }
    if (H.defer) slice_plan(H, s_begin, s_begin + nseg, nr);
    else if (H.sliced) slice_segments(H, s_begin, s_begin + nseg, nr);
    // work items: consecutive segments up to group_nz nonzeros; the staged
    // segments of an item are cut into TMA batches of <= kBQ quads (row-major
    // layout only, PDCS_TMA=1)
    auto emit_item = [&](int32_t gg, int32_t sa, int32_t sb) {
      const int32_t b0 = (int32_t)H.batch.size();
      int32_t ord = -1;
      for (int32_t si = sa; si < sb; ++si) {
        const TSeg& S = H.seg[si];
        if (S.tile < 0) continue;
        ++ord;
        const int32_t* rp = H.rowptr.data() + S.rp;
        int first = 1;
        int32_t ra = 0, qa = rp[0];
        auto emit = [&](int32_t r_a, int32_t r_b, int32_t q_a, int32_t q_b) {
          if (q_b > q_a) { H.batch.push_back(TBatch{si, r_a, r_b, q_a, q_b, first, ord, 0}); first = 0; }
        };
        for (int32_t r = 0; r < nr; ++r) {
          const int32_t rq0 = rp[r], rq1 = rp[r + 1];
          while (rq1 - qa > kBQ) {
            if (rq0 > qa) { emit(ra, r, qa, rq0); qa = rq0; ra = r; }
            else { emit(r, r + 1, qa, qa + kBQ); qa += kBQ; ra = r; }
          }
        }
        emit(ra, nr, qa, rp[nr]);
      }
      H.work.push_back(TWork{(int32_t)H.chunk.size(), gg, sa, sb, b0, (int32_t)H.batch.size()});
    };
    int32_t g = 0;
    int64_t acc = 0;
    int32_t ws = s_begin;
    for (int k = 0; k < nseg; ++k) {
      acc += seg_nz[k];
      if (acc >= group_nz || k == nseg - 1) {
        emit_item(g++, ws, s_begin + k + 1);
        ws = s_begin + k + 1;
        acc = 0;
      }
    }
    if (nseg == 0) emit_item(g++, s_begin, s_begin);
    H.chunk.push_back(TChunk{r0, nr, g, H.scratch});
    H.scratch += (int64_t)g * nr * elem;
    for (int64_t t : touched) { cnt[t] = 0; segof[t] = -1; }
  }
}

// Tiled format of a whole CSR: contiguous chunk ranges of about equal nnz are
// built on host threads (build_tiled_range) and concatenated in order with
// their offsets rebased, so the result does not depend on the thread count.
void build_tiled(const int64_t* ptr, const int32_t* col, int64_t rows, int64_t nvec, int elem,
                 TiledHost& H, bool keep_parts = false, bool defer = false) {
  const auto t_start = std::chrono::steady_clock::now();
  // work-item size: enough items to fill the GPU several times over, no more
  // partial groups per chunk than needed (PDCS_TILE_GROUP overrides)
  const int64_t group_nz = std::getenv("PDCS_TILE_GROUP") ? std::atol(std::getenv("PDCS_TILE_GROUP"))
                                                          : std::max<int64_t>(32768, ptr[rows] / 3000);
  const int64_t nchunk = (rows + kTRows - 1) / kTRows;
  int nth = (int)std::min<int64_t>({(int64_t)std::max(1u, std::thread::hardware_concurrency()), 32,
                                    std::max<int64_t>(1, nchunk / 4)});
  if (const char* e = std::getenv("PDCS_BUILD_THREADS")) nth = std::max(1, std::atoi(e));
  // chunk-aligned range starts at equal shares of nnz
  std::vector<int64_t> cut(nth + 1, rows);
  cut[0] = 0;
  for (int w = 1; w < nth; ++w) {
    const int64_t target = ptr[rows] / nth * w;
    const int64_t r = std::lower_bound(ptr, ptr + rows + 1, target) - ptr;
    cut[w] = std::max(cut[w - 1], std::min(rows, r / kTRows * kTRows));
  }
  H.T = tiled_tile_bytes() / (8 * elem);
  H.elem = elem;
  H.tma = tiled_tma_env();
  H.sliced = tiled_sliced();
  // the deferred build needs the parts mode (the device assembles) and the
  // sliced, bank-balanced layout; PDCS_TILE_DEVICE=0 keeps the host build
  const bool bal_env = !std::getenv("PDCS_TILE_BALANCE") || std::atoi(std::getenv("PDCS_TILE_BALANCE"));
  H.defer = defer && keep_parts && H.sliced && bal_env &&
            !(std::getenv("PDCS_TILE_DEVICE") && std::atoi(std::getenv("PDCS_TILE_DEVICE")) == 0);
  std::vector<TiledHost> part(nth);
  for (auto& P : part) { P.T = H.T; P.sliced = H.sliced; P.tma = H.tma; P.defer = H.defer; }
  std::vector<std::thread> th;
  for (int w = 0; w < nth; ++w)
    th.emplace_back([&, w] { build_tiled_range(ptr, col, cut[w], cut[w + 1], nvec, elem, group_nz, part[w]); });
  for (auto& t : th) t.join();
  H.ranges_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  H.nnz = ptr[rows];
  // Concatenate the parts in order.  The small per-segment / per-item arrays
  // are rebased serially; the per-entry arrays (column ids, value permutation,
  // row pointers, block bases) are copied verbatim, one thread per part, into
  // vectors sized once (the serial inserts had taken ~25% of the build).
  const int np = (int)part.size();
  std::vector<size_t> o_s(np), o_d(np), o_rp(np), o_bb(np), o_pre(np);
  size_t ns = 0, nd = 0, nrp = 0, nbb = 0, npre = 0;
  for (int w = 0; w < np; ++w) {
    const TiledHost& P = part[w];
    ns = (ns + 63) & ~(size_t)63;              // keep segment starts 512-B aligned (values)
    o_s[w] = ns; o_d[w] = nd; o_rp[w] = nrp; o_bb[w] = nbb; o_pre[w] = npre;
    ns += H.defer ? (size_t)P.fin_s : P.col_s.size();
    nd += P.col_d.size(); nrp += P.rowptr.size(); nbb += P.blkb.size();
    npre += H.defer ? P.col_s.size() : 0;
  }
  for (int w = 0; w < np; ++w) {
    TiledHost& P = part[w];
    const int64_t sbase = (int64_t)H.seg.size(), bbase = (int64_t)H.batch.size(), cbase = (int64_t)H.chunk.size();
    for (TSeg S : P.seg) {
      S.rp += (int64_t)o_rp[w];
      S.nz += S.tile >= 0 ? (int64_t)o_s[w] : (int64_t)o_d[w];
      if (S.bb >= 0) S.bb += (int64_t)o_bb[w];
      H.seg.push_back(S);
    }
    for (TBatch B : P.batch) { B.seg += (int32_t)sbase; H.batch.push_back(B); }
    for (TWork W : P.work) {
      W.chunk += (int32_t)cbase; W.s0 += (int32_t)sbase; W.s1 += (int32_t)sbase;
      W.b0 += (int32_t)bbase; W.b1 += (int32_t)bbase;
      H.work.push_back(W);
    }
    for (TChunk C : P.chunk) { C.scratch += H.scratch; H.chunk.push_back(C); }
    H.scratch += P.scratch;
    H.staged += P.staged;
    const int32_t dbase = (int32_t)H.dseg.size();
    for (TDefer D : P.dseg) {
      D.src += (int64_t)o_pre[w]; D.dst += (int64_t)o_s[w]; D.rp += (int64_t)o_rp[w]; D.bb += (int64_t)o_bb[w];
      H.dseg.push_back(D);
    }
    for (int2 b : P.dblk) H.dblk.push_back(make_int2(b.x + dbase, b.y));
  }
  if (keep_parts) {
    H.o_s = std::move(o_s); H.o_d = std::move(o_d); H.o_rp = std::move(o_rp); H.o_bb = std::move(o_bb);
    H.tot_s = ns + 8;          // TMA column-id copies may read one quad past the end
    H.tot_d = nd;
    H.tot_rp = nrp + 8;        // TMA row-pointer slices are rounded up to 16 B
    H.tot_bb = nbb + 1;        // never empty (device upload)
    H.o_pre = std::move(o_pre);
    H.tot_pre = npre;
    for (auto& P : part) {
      P.seg.clear(); P.batch.clear(); P.work.clear(); P.chunk.clear(); P.dseg.clear(); P.dblk.clear();
    }
    H.parts = std::move(part);
    H.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    return;
  }
  H.col_s.assign(ns, 0); H.perm_s.assign(ns, -1);
  H.col_d.resize(nd); H.perm_d.resize(nd);
  H.rowptr.resize(nrp); H.srow.resize(nrp); H.blkb.resize(nbb);
  {
    std::vector<std::thread> cp;
    for (int w = 0; w < np; ++w)
      cp.emplace_back([&, w] {
        TiledHost& P = part[w];
        std::copy(P.col_s.begin(), P.col_s.end(), H.col_s.begin() + o_s[w]);
        std::copy(P.perm_s.begin(), P.perm_s.end(), H.perm_s.begin() + o_s[w]);
        std::copy(P.col_d.begin(), P.col_d.end(), H.col_d.begin() + o_d[w]);
        std::copy(P.perm_d.begin(), P.perm_d.end(), H.perm_d.begin() + o_d[w]);
        std::copy(P.rowptr.begin(), P.rowptr.end(), H.rowptr.begin() + o_rp[w]);
        std::copy(P.srow.begin(), P.srow.end(), H.srow.begin() + o_rp[w]);
        std::copy(P.blkb.begin(), P.blkb.end(), H.blkb.begin() + o_bb[w]);
        P = TiledHost();
      });
    for (auto& t : cp) t.join();
  }
  H.col_s.resize(H.col_s.size() + 8, 0);      // TMA column-id copies may read one quad past the end
  H.blkb.push_back(0);                        // never empty (device upload)
  H.rowptr.resize(H.rowptr.size() + 8, 0);    // TMA row-pointer slices are rounded up to 16 B
  H.srow.resize(H.rowptr.size(), 0);
  H.perm_s.resize(H.col_s.size(), -1);
  H.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

// ---------------------------------------------------------------- device structure build
// The tiled format of a DEVICE CSR (tiled.cuh: k_tile_hist / k_tile_rowcnt /
// k_tile_fill, then k_tile_balance_w / k_tile_slice): the entries never pass
// through the host.  The host sees the (chunk, tile) counts and the per-row
// segment counts only, and runs build_tiled_range's decisions on them (staged
// tiles, segment order, rows longest first, lanes per row, quad padding, the
// sliced plan, work items and batches) in the same order, so the layout is
// the one build_tiled + the deferred device finish produce
// (pdcs_tiled_devbuild_check compares them entry by entry).
struct TiledDevArrays {
  DBuf<int32_t> rowptr, col_d, blkb, perm_s, perm_d;
  DBuf<uint16_t> srow, col_s;
};

template <class F>
void parallel_chunks(int64_t n, const F& f, int64_t grain_max = -1) {
  int nth = (int)std::min<int64_t>({(int64_t)std::max(1u, std::thread::hardware_concurrency()), 32,
                                    std::max<int64_t>(1, n / 8)});
  if (const char* e = std::getenv("PDCS_BUILD_THREADS")) nth = std::max(1, std::atoi(e));
  if (nth <= 1) { f((int64_t)0, n); return; }
  // dynamic: chunks differ widely in work (Lasso K^T: 20 of ~1000 hold half the entries)
  std::atomic<int64_t> next{0};
  int64_t grain = std::max<int64_t>(1, n / (nth * 16));
  if (grain_max > 0) grain = std::min(grain, grain_max);
  std::vector<std::thread> th;
  for (int w = 0; w < nth; ++w)
    th.emplace_back([&] {
      for (int64_t a; (a = next.fetch_add(grain)) < n;) f(a, std::min(n, a + grain));
    });
  for (auto& t : th) t.join();
}

// Whether the solver's builds take this path: the sliced, bank-balanced layout
// (the default); PDCS_TILE_DEVBUILD=0 keeps the host build.
bool tiled_devbuild_env() {
  const bool bal = !std::getenv("PDCS_TILE_BALANCE") || std::atoi(std::getenv("PDCS_TILE_BALANCE"));
  const bool dev = !(std::getenv("PDCS_TILE_DEVICE") && std::atoi(std::getenv("PDCS_TILE_DEVICE")) == 0);
  const bool db = !(std::getenv("PDCS_TILE_DEVBUILD") && std::atoi(std::getenv("PDCS_TILE_DEVBUILD")) == 0);
  return tiled_sliced() && bal && dev && db;
}

// dptr / dcol: the device CSR (int32 row pointers); hptr: its row pointers on
// the host.  Fills H's descriptors (seg, work, chunk, batch, scratch, staged,
// sizes) and the device arrays of A; A.perm_s / perm_d are the CSR positions
// the values are gathered from.  H.devbuilt stays false (nothing built) when
// the staged share is below min_frac: the caller keeps the CSR kernel then.
void build_tiled_device(const int32_t* dptr, const int32_t* dcol, const int64_t* hptr, int64_t rows, int64_t nvec,
                        int elem, double min_frac, TiledHost& H, TiledDevArrays& A, cudaStream_t st, int sms) {
  const auto t_start = std::chrono::steady_clock::now();
  SetupTrace tr;
  H = TiledHost();
  H.T = tiled_tile_bytes() / (8 * elem);
  H.elem = elem;
  H.tma = false;
  H.sliced = true;
  H.defer = true;
  H.nnz = hptr[rows];
  const int32_t T = H.T;
  const int64_t stage_min = (int64_t)T * 8 * elem / 16;
  const int64_t ntiles = (nvec + T - 1) / T;
  const int64_t nchunk = (rows + kTRows - 1) / kTRows;
  const int64_t group_nz = std::getenv("PDCS_TILE_GROUP") ? std::atol(std::getenv("PDCS_TILE_GROUP"))
                                                          : std::max<int64_t>(32768, H.nnz / 3000);
  if (H.nnz == 0 || rows == 0) return;
  // ---- (chunk, tile) counts -> staged tiles per chunk
  std::vector<std::vector<int32_t>> stiles(nchunk);
  std::vector<std::vector<int64_t>> scnt(nchunk);
  std::vector<int64_t> dnz(nchunk, 0);
  {
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(nchunk, ((int64_t)16 << 20) / std::max<int64_t>(ntiles, 1)));
    DBuf<int32_t> dc;
    dc.alloc((size_t)per * ntiles);
    std::vector<int32_t> hc((size_t)per * ntiles);
    const bool smem = ntiles <= 12288;
    std::vector<THistItem> items;
    DBuf<THistItem> ditems;
    for (int64_t c0 = 0; c0 < nchunk; c0 += per) {
      const int64_t nc = std::min(per, nchunk - c0);
      items.clear();
      for (int64_t c = c0; c < c0 + nc; ++c) {
        const int64_t pa = hptr[c * kTRows], pb = hptr[std::min(rows, (c + 1) * kTRows)];
        for (int64_t q = pa; q < pb; q += 65536) items.push_back(THistItem{c, q, std::min(pb, q + 65536)});
      }
      CK(cudaMemsetAsync(dc.p, 0, (size_t)nc * ntiles * sizeof(int32_t), st));
      if (!items.empty()) {
        upload(ditems, items, st);
        k_tile_hist<<<(unsigned)items.size(), 256, smem ? ntiles * sizeof(int32_t) : 0, st>>>(
            dcol, ditems.p, T, ntiles, c0, dc.p, smem ? 1 : 0);
      }
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(hc.data(), dc.p, (size_t)nc * ntiles * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      parallel_chunks(nc, [&](int64_t a, int64_t b) {
        for (int64_t c = a; c < b; ++c) {
          const int32_t* h = hc.data() + (size_t)c * ntiles;
          for (int64_t t = 0; t < ntiles; ++t) {
            if (!h[t]) continue;
            if (h[t] >= stage_min) { stiles[c0 + c].push_back((int32_t)t); scnt[c0 + c].push_back(h[t]); }
            else dnz[c0 + c] += h[t];
          }
        }
      });
    }
  }
  tr.mark("    devbuild: tile counts", st);
  std::vector<TBChunk> cb(nchunk);
  std::vector<int32_t> stl;
  int64_t nseg = 0;
  for (int64_t c = 0; c < nchunk; ++c) {
    cb[c].sbase = nseg;
    cb[c].soff = (int32_t)stl.size();
    cb[c].nst = (int32_t)stiles[c].size();
    cb[c].direct = dnz[c] ? 1 : 0;
    cb[c].pad = 0;
    stl.insert(stl.end(), stiles[c].begin(), stiles[c].end());
    nseg += cb[c].direct + cb[c].nst;
    for (int64_t v : scnt[c]) H.staged += v;
  }
  const double frac = (double)H.staged / (double)H.nnz;
  const char* env = std::getenv("PDCS_TILED");
  if (!(env ? std::atoi(env) != 0 : frac >= min_frac)) return;
  // ---- per-row segment counts
  DBuf<TBChunk> dcb;
  DBuf<int32_t> dstl, drc;
  upload(dcb, cb, st);
  dstl.alloc(std::max<size_t>(stl.size(), 1));
  if (!stl.empty()) CK(cudaMemcpyAsync(dstl.p, stl.data(), stl.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  drc.alloc((size_t)nseg * kTRows);
  CK(cudaMemsetAsync(drc.p, 0, (size_t)nseg * kTRows * sizeof(int32_t), st));
  const int gw = (int)std::min<int64_t>((rows + 7) / 8, (int64_t)sms * 16);
  k_tile_rowcnt<<<gw, 256, 0, st>>>(dptr, dcol, rows, T, dcb.p, dstl.p, drc.p);
  CK(cudaGetLastError());
  std::vector<int32_t> rc((size_t)nseg * kTRows);
  CK(cudaMemcpyAsync(rc.data(), drc.p, rc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  drc.free_();
  tr.mark("    devbuild: row counts", st);
  // ---- per chunk: build_tiled_range's layout decisions on the counts
  struct CL {
    std::vector<TSeg> seg;                 // rp relative to the chunk; bb: first block slot (chunk-local)
    std::vector<int64_t> pre;              // staged: pre offset (chunk-local entries); direct: col_d offset
    std::vector<int32_t> rowptr;
    std::vector<uint16_t> srow;
    std::vector<int32_t> blkq;             // block quad bases of the staged segments
    std::vector<int64_t> fin;              // staged: sliced size (entries, 4 * quads); direct: 0
    std::vector<TBatch> batch;             // seg: chunk-local
    std::vector<TWork> work;               // s0/s1/b0/b1 chunk-local
    int32_t ngroups = 0, nr = 0;
    int64_t npre = 0, nd = 0;
  };
  std::vector<CL> cl(nchunk);
  parallel_chunks(nchunk, [&](int64_t ca, int64_t cbnd) {
    std::vector<int32_t> order, bucket;
    for (int64_t c = ca; c < cbnd; ++c) {
      CL& L = cl[c];
      const int32_t nr = (int32_t)std::min<int64_t>(kTRows, rows - c * kTRows);
      L.nr = nr;
      const TBChunk& C = cb[c];
      const int ns = C.direct + C.nst;
      std::vector<int64_t> seg_nz;
      if (C.direct) { L.seg.push_back(TSeg{-1, 1, 0, 0, -1}); seg_nz.push_back(dnz[c]); }
      for (int k = 0; k < C.nst; ++k) { L.seg.push_back(TSeg{stiles[c][k], 1, 0, 0, -1}); seg_nz.push_back(scnt[c][k]); }
      order.resize(nr);
      for (int k = 0; k < ns; ++k) {
        TSeg& S = L.seg[k];
        const bool stg = S.tile >= 0;
        const int32_t* rck = rc.data() + (size_t)(C.sbase + k) * kTRows;
        for (int32_t i = 0; i < nr; ++i) order[i] = i;
        if (stg) {
          // rows longest first, stable: a counting sort on the count when the
          // counts are small (the permutation std::stable_sort gives)
          int32_t mx = 0;
          for (int32_t i = 0; i < nr; ++i) mx = std::max(mx, rck[i]);
          if (mx <= 4 * nr) {
            bucket.assign((size_t)mx + 2, 0);
            for (int32_t i = 0; i < nr; ++i) ++bucket[(size_t)(mx - rck[i]) + 1];
            for (size_t z = 1; z < bucket.size(); ++z) bucket[z] += bucket[z - 1];
            for (int32_t i = 0; i < nr; ++i) order[bucket[(size_t)(mx - rck[i])]++] = i;
          } else {
            std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return rck[a] > rck[b]; });
          }
        }
        S.rp = (int64_t)L.rowptr.size();
        L.rowptr.resize(L.rowptr.size() + nr + 1, 0);
        L.srow.resize(L.rowptr.size(), 0);
        int64_t units = 0;
        for (int32_t pos = 0; pos < nr; ++pos) {
          const int32_t i = order[pos];
          const int32_t u = stg ? (rck[i] + 3) / 4 : rck[i];
          L.rowptr[S.rp + pos + 1] = L.rowptr[S.rp + pos] + u;
          L.srow[S.rp + pos] = (uint16_t)i;
          units += u;
        }
        S.V = pick_v(stg ? (double)units / nr : (double)seg_nz[k] / nr, elem);
        if (stg) {
          L.npre = (L.npre + 7) & ~(int64_t)7;
          L.pre.push_back(L.npre);
          L.npre += 4 * units;
          // slice_plan: warp-block quad bases
          const int rpw = 32 / S.V;
          const int nblk = tiled_blocks(nr, S.V);
          const int32_t* rp = L.rowptr.data() + S.rp;
          S.bb = (int64_t)L.blkq.size();
          int64_t q = 0;
          for (int blk = 0; blk < nblk; ++blk) {
            L.blkq.push_back((int32_t)q);
            int32_t tmax = 0;
            for (int a = 0; a < rpw && blk * rpw + a < nr; ++a) {
              const int32_t nq = rp[blk * rpw + a + 1] - rp[blk * rpw + a];
              tmax = std::max(tmax, (nq + S.V - 1) / S.V);
            }
            q += 32 * (int64_t)tmax;
          }
          L.fin.push_back(4 * q);
        } else {
          L.pre.push_back(L.nd);
          L.nd += units;
          L.fin.push_back(0);
        }
      }
      // work items and batches (build_tiled_range's emit_item)
      auto emit_item = [&](int32_t gg, int32_t sa, int32_t sb) {
        const int32_t b0 = (int32_t)L.batch.size();
        int32_t ord = -1;
        for (int32_t si = sa; si < sb; ++si) {
          const TSeg& S = L.seg[si];
          if (S.tile < 0) continue;
          ++ord;
          const int32_t* rp = L.rowptr.data() + S.rp;
          int first = 1;
          int32_t ra = 0, qa = rp[0];
          auto emit = [&](int32_t r_a, int32_t r_b, int32_t q_a, int32_t q_b) {
            if (q_b > q_a) { L.batch.push_back(TBatch{si, r_a, r_b, q_a, q_b, first, ord, 0}); first = 0; }
          };
          for (int32_t r = 0; r < nr; ++r) {
            const int32_t rq0 = rp[r], rq1 = rp[r + 1];
            while (rq1 - qa > kBQ) {
              if (rq0 > qa) { emit(ra, r, qa, rq0); qa = rq0; ra = r; }
              else { emit(r, r + 1, qa, qa + kBQ); qa += kBQ; ra = r; }
            }
          }
          emit(ra, nr, qa, rp[nr]);
        }
        L.work.push_back(TWork{0, gg, sa, sb, b0, (int32_t)L.batch.size()});
      };
      int32_t g = 0, ws = 0;
      int64_t acc = 0;
      for (int k = 0; k < ns; ++k) {
        acc += seg_nz[k];
        if (acc >= group_nz || k == ns - 1) { emit_item(g++, ws, k + 1); ws = k + 1; acc = 0; }
      }
      if (ns == 0) emit_item(g++, 0, 0);
      L.ngroups = g;
    }
  });
  tr.mark("    devbuild: host layout", nullptr, false);
  // ---- global offsets, in chunk order (the concatenation of build_tiled)
  std::vector<int64_t> o_rp(nchunk), o_bb(nchunk);
  std::vector<TFillSeg> fsv;
  fsv.reserve(nseg);
  int64_t nrp = 0, nbb = 0, npre = 0, nd = 0, fin = 0;
  for (int64_t c = 0; c < nchunk; ++c) {
    CL& L = cl[c];
    o_rp[c] = nrp;
    o_bb[c] = nbb;
    npre = (npre + 7) & ~(int64_t)7;
    const int32_t sbase = (int32_t)H.seg.size(), bbase = (int32_t)H.batch.size();
    for (size_t k = 0; k < L.seg.size(); ++k) {
      TSeg S = L.seg[k];
      S.rp += nrp;
      TFillSeg F{0, S.rp, S.tile, L.nr};
      if (S.tile >= 0) {
        const int64_t src = npre + L.pre[k];
        fin = (fin + 63) & ~(int64_t)63;
        S.bb += nbb;
        H.dseg.push_back(TDefer{src, fin, S.rp, S.bb, L.nr, S.V});
        const int32_t di = (int32_t)H.dseg.size() - 1;
        for (int blk = 0; blk < tiled_blocks(L.nr, S.V); ++blk) H.dblk.push_back(make_int2(di, blk));
        S.nz = fin;
        fin += L.fin[k];
        F.off = src;
      } else {
        S.nz = nd + L.pre[k];
        F.off = S.nz;
      }
      H.seg.push_back(S);
      fsv.push_back(F);
    }
    for (TBatch B : L.batch) { B.seg += sbase; H.batch.push_back(B); }
    for (TWork W : L.work) {
      W.chunk = (int32_t)c; W.s0 += sbase; W.s1 += sbase; W.b0 += bbase; W.b1 += bbase;
      H.work.push_back(W);
    }
    H.chunk.push_back(TChunk{c * kTRows, L.nr, L.ngroups, H.scratch});
    H.scratch += (int64_t)L.ngroups * L.nr * elem;
    nrp += (int64_t)L.rowptr.size();
    nbb += (int64_t)L.blkq.size();
    npre += L.npre;
    nd += L.nd;
  }
  H.tot_rp = nrp + 8;
  H.tot_bb = nbb + 1;
  H.tot_s = fin + 8;
  H.tot_d = nd;
  H.tot_pre = npre;
  H.fin_s = fin;
  // ---- host structure arrays to the device; the inverse row order on the device
  A.rowptr.alloc(H.tot_rp); A.srow.alloc(H.tot_rp); A.blkb.alloc(H.tot_bb);
  DBuf<uint16_t> dposof;
  dposof.alloc(H.tot_rp);
  {
    // uninitialised host buffers: every element is copied below, only the
    // pads are zeroed (zero-filling ~60 MB first had cost ~10 ms on Lasso)
    std::unique_ptr<int32_t[]> hrp(new int32_t[H.tot_rp]), hbb(new int32_t[H.tot_bb]);
    std::unique_ptr<uint16_t[]> hsr(new uint16_t[H.tot_rp]);
    parallel_chunks(nchunk, [&](int64_t a, int64_t b) {
      for (int64_t c = a; c < b; ++c) {
        const CL& L = cl[c];
        std::copy(L.rowptr.begin(), L.rowptr.end(), hrp.get() + o_rp[c]);
        std::copy(L.srow.begin(), L.srow.end(), hsr.get() + o_rp[c]);
        std::copy(L.blkq.begin(), L.blkq.end(), hbb.get() + o_bb[c]);
      }
    });
    for (int64_t i = nrp; i < H.tot_rp; ++i) { hrp[i] = 0; hsr[i] = 0; }
    for (int64_t i = nbb; i < H.tot_bb; ++i) hbb[i] = 0;
    CK(cudaMemcpyAsync(A.rowptr.p, hrp.get(), H.tot_rp * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(A.blkb.p, hbb.get(), H.tot_bb * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(A.srow.p, hsr.get(), H.tot_rp * 2, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  cl = std::vector<CL>();
  tr.mark("    devbuild: offsets + uploads", st);
  // ---- fill: entries to their pre / direct slots
  DBuf<TFillSeg> dfs;
  upload(dfs, fsv, st);
  DBuf<uint16_t> pcol;
  DBuf<int32_t> pperm;
  const int64_t npre1 = std::max<int64_t>(npre, 1);
  pcol.alloc(npre1);
  pperm.alloc(npre1);
  CK(cudaMemsetAsync(pcol.p, 0, npre1 * sizeof(uint16_t), st));
  CK(cudaMemsetAsync(pperm.p, 0xff, npre1 * sizeof(int32_t), st));
  A.col_d.alloc(std::max<int64_t>(nd, 1));
  A.perm_d.alloc(std::max<int64_t>(nd, 1));
  k_tile_posof<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(nseg, (int64_t)sms * 32)), 256, 0, st>>>(
      dfs.p, nseg, A.srow.p, dposof.p);
  k_tile_fill<<<gw, 256, 0, st>>>(dptr, dcol, rows, T, dcb.p, dstl.p, dfs.p, A.rowptr.p, dposof.p, pcol.p, pperm.p,
                                  A.col_d.p, A.perm_d.p);
  CK(cudaGetLastError());
  tr.mark("    devbuild: fill", st);
  // ---- bank balancing + sliced re-layout (the deferred build's kernels)
  A.col_s.alloc(H.tot_s);
  A.perm_s.alloc(H.tot_s);
  CK(cudaMemsetAsync(A.col_s.p, 0, H.tot_s * sizeof(uint16_t), st));
  CK(cudaMemsetAsync(A.perm_s.p, 0xff, H.tot_s * sizeof(int32_t), st));
  const int64_t nb = (int64_t)H.dblk.size();
  if (nb) {
    DBuf<TDefer> dseg;
    DBuf<int2> dblk;
    upload(dseg, H.dseg, st);
    upload(dblk, H.dblk, st);
    DBuf<uint16_t> bcol, ncol;
    DBuf<int32_t> bperm, nperm;
    bcol.alloc(npre1); ncol.alloc(npre1); bperm.alloc(npre1); nperm.alloc(npre1);
    const int tb = 128;
    launch_tile_balance(dseg.p, H.dseg, dblk.p, nb, elem, A.rowptr.p, pcol.p, pperm.p, bcol.p, bperm.p, ncol.p, nperm.p,
                        st);
    tr.mark("    devbuild: balance", st);
    k_tile_slice<<<(int)((nb + tb - 1) / tb), tb, 0, st>>>(dseg.p, dblk.p, nb, A.rowptr.p, A.blkb.p, ncol.p,
                                                           nperm.p, A.col_s.p, A.perm_s.p);
    CK(cudaGetLastError());
    tr.mark("    devbuild: slice", st);
    bcol.free_(); ncol.free_(); bperm.free_(); nperm.free_();
    tr.mark("    devbuild: frees (balance scratch)", nullptr, false);
  }
  CK(cudaStreamSynchronize(st));
  pcol.free_(); pperm.free_(); dfs.free_(); dposof.free_(); dcb.free_(); dstl.free_();
  tr.mark("    devbuild: frees", nullptr, false);
  H.devbuilt = true;
  H.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

// Input checks of the CSR on host threads: column ids in
// range and strictly increasing per row, finite values.  Reports the first
// offending row (and, within it, the first offending entry's check).
void validate_csr(const int64_t* ptr, const int32_t* col, const double* val, int64_t m, int64_t n) {
  const int nth = (int)std::max<int64_t>(1, std::min<int64_t>(16, ptr[m] / 4000000 + 1));
  std::vector<int64_t> bad(nth, INT64_MAX);
  std::vector<std::thread> th;
  for (int w = 0; w < nth; ++w)
    th.emplace_back([&, w] {
      const int64_t a = m * w / nth, b = m * (w + 1) / nth;
      for (int64_t i = a; i < b; ++i)
        for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
          int why = 0;
          if (col[q] < 0 || col[q] >= n) why = 1;
          else if (q > ptr[i] && col[q] <= col[q - 1]) why = 2;
          else if (!std::isfinite(val[q])) why = 3;
          if (why) { bad[w] = i * 4 + why; return; }
        }
    });
  for (auto& t : th) t.join();
  const int64_t b = *std::min_element(bad.begin(), bad.end());
  if (b == INT64_MAX) return;
  const std::string row = std::to_string(b / 4);
  if (b % 4 == 1) fail(PDCS_ERR_DIM, "column index out of range in row " + row);
  if (b % 4 == 2) fail(PDCS_ERR_DIM, "column indices not strictly increasing in row " + row);
  fail(PDCS_ERR_NONFINITE, "non-finite matrix entry in row " + row);
}

// Column order of the box coordinates for gather locality.
// The SpMV sweeps gather 16-byte (x^_j, x_j) pairs, two per 32-byte sector.  A
// long row (>= kPermLongRow entries, served by one CTA, so no other row reuses
// its sectors) whose columns are strided pays a whole sector per entry; this is
// Fisher's supply rows, sum_i X_ij = b_j, over a buyer-major X.  Box columns are
// elementwise (their projection is a clip), so they may be stored in any order:
// they are stably sorted by the longest row that holds them (ties: the lower
// row), which puts each long row's box columns next to each other.  The order
// is used when it cuts the sectors the long rows touch by >= 20%; cone columns
// keep their places.  Returns false (identity) otherwise.
constexpr int64_t kPermLongRow = 1024;

int64_t long_row_sectors(const int64_t* ptr, const int32_t* col, int64_t m, int64_t n, const int32_t* u2i) {
  // distinct 2-column sectors per long row, by marking (no sort: Fisher's 1000
  // rows of 1e4 mapped ids had taken ~0.2 s sorted)
  int64_t total = 0;
  std::vector<uint8_t> mark((size_t)(n >> 1) + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t a = ptr[i], b = ptr[i + 1];
    if (b - a < kPermLongRow) continue;
    for (int64_t q = a; q < b; ++q) {
      const int64_t sct = (u2i ? u2i[col[q]] : col[q]) >> 1;
      if (!mark[sct]) { mark[sct] = 1; ++total; }
    }
    for (int64_t q = a; q < b; ++q) mark[(u2i ? u2i[col[q]] : col[q]) >> 1] = 0;
  }
  return total;
}

bool plan_colperm(const int64_t* ptr, const int32_t* col, int64_t m, int64_t n, int64_t n1, int sms,
                  std::vector<int32_t>& u2i, std::vector<int32_t>& i2u) {
  if (n1 < 2) return false;
  // only the few-long-rows case (the CSR plan's one-CTA-per-row class, < 16
  // per SM): many long rows run side by side and share sectors anyway, and
  // checking them would cost O(nnz log) host time (Lasso 4e5 x 7e6: 1400 per row)
  int64_t nlong = 0;
  for (int64_t i = 0; i < m; ++i) nlong += ptr[i + 1] - ptr[i] >= kPermLongRow;
  if (nlong == 0 || nlong >= 16 * (int64_t)sms) return false;
  const int64_t before = long_row_sectors(ptr, col, m, n, nullptr);
  if (before == 0) return false;
  // best[j]: the longest row holding box column j (the first such row on
  // ties).  Host threads own column ranges and each scans all rows in order
  // (same result as one pass; the random writes stay in a thread's range)
  std::vector<int64_t> best(n1, -1), blen(n1, -1);
  {
    int nth = (int)std::min<int64_t>({(int64_t)std::max(1u, std::thread::hardware_concurrency()), 16,
                                      std::max<int64_t>(1, n1 / 65536)});
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
      th.emplace_back([&, w] {
        const int64_t j0 = n1 * w / nth, j1 = n1 * (w + 1) / nth;
        for (int64_t i = 0; i < m; ++i) {
          const int64_t len = ptr[i + 1] - ptr[i];
          for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
            const int64_t j = col[q];
            if (j >= j0 && j < j1 && len > blen[j]) { blen[j] = len; best[j] = i; }
          }
        }
      });
    for (auto& t : th) t.join();
  }
  // stable order by the holding row: a counting sort over best in [-1, m)
  // (std::stable_sort of Fisher's 1e7 box columns had taken ~1 s)
  std::vector<int32_t> order(n1);
  {
    std::vector<int64_t> start((size_t)m + 2, 0);
    for (int64_t j = 0; j < n1; ++j) ++start[(size_t)(best[j] + 1) + 1];
    for (size_t z = 1; z < start.size(); ++z) start[z] += start[z - 1];
    for (int64_t j = 0; j < n1; ++j) order[start[(size_t)(best[j] + 1)]++] = (int32_t)j;
  }
  i2u.resize(n);
  u2i.resize(n);
  for (int64_t k = 0; k < n; ++k) i2u[k] = k < n1 ? order[k] : (int32_t)k;
  for (int64_t k = 0; k < n; ++k) u2i[i2u[k]] = (int32_t)k;
  const int64_t after = long_row_sectors(ptr, col, m, n, u2i.data());
  if ((double)after > 0.8 * (double)before) { u2i.clear(); i2u.clear(); return false; }
  return true;
}

// The CSR with column ids mapped through u2i, each row re-sorted (host threads).
void permute_csr(const int64_t* ptr, const int32_t* col, const double* val, int64_t m,
                 const std::vector<int32_t>& u2i, std::vector<int32_t>& pcol, std::vector<double>& pval) {
  const int64_t nnz = ptr[m];
  pcol.resize(nnz);
  pval.resize(nnz);
  // rows handed out dynamically: Fisher's 1000 long supply rows (1e7 of its
  // 1.2e7 entries) are its first rows and had all fallen to one thread (~0.9 s)
  parallel_chunks(m, [&](int64_t ra, int64_t rb) {
    std::vector<std::pair<int32_t, double>> buf;
    for (int64_t i = ra; i < rb; ++i) {
      const int64_t a = ptr[i], b = ptr[i + 1];
      buf.resize(b - a);
      for (int64_t q = a; q < b; ++q) buf[q - a] = {u2i[col[q]], val[q]};
      std::sort(buf.begin(), buf.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (int64_t q = a; q < b; ++q) { pcol[q] = buf[q - a].first; pval[q] = buf[q - a].second; }
    }
  }, 8);
  (void)nnz;
}

// Size class of each cone block: 0 thread, 1 warp, 2 CTA,
// 3 cluster, 4 grid.  Exp blocks and SOC/RSOC of dim <= 32 take one thread.
// The warp class covers dims up to 512, or up to 16384 when it then holds
// enough blocks to give every SM 32 warps; the CTA class up to 4096, or up to
// 262144 when it holds >= 2 blocks per SM; the cluster class the rest up to
// 131072; the grid team beyond.  (Measured: profiles/r1_proj_v2.json, the
// unit-scaling sweep of PAPER.md:719-742 Fig. 3 with every team forced.)
struct ClassPolicy {
  int64_t t_warp = 512, t_cta = 4096;
  int of(const Block& b) const {
    if (b.kind == C_EXP || b.kind == C_DEXP || b.dim <= 32) return 0;
    if (b.dim <= t_warp) return 1;
    if (b.dim <= t_cta) return 2;
    return b.dim <= 131072 ? 3 : 4;
  }
};
ClassPolicy class_policy(const std::vector<Block>& v, int sms) {
  ClassPolicy P;
  int64_t n_warp = 0;
  for (const Block& b : v)
    if ((b.kind == C_SOC || b.kind == C_RSOC) && b.dim > 32 && b.dim <= 16384) ++n_warp;
  if (n_warp >= 32 * (int64_t)sms) P.t_warp = 16384;
  int64_t n_cta = 0;
  for (const Block& b : v)
    if ((b.kind == C_SOC || b.kind == C_RSOC) && b.dim > P.t_warp && b.dim <= 262144) ++n_cta;
  if (n_cta >= 2 * (int64_t)sms) P.t_cta = std::max<int64_t>(P.t_warp, 262144);
  else P.t_cta = std::max<int64_t>(P.t_warp, 4096);
  return P;
}

}  // namespace

// ============================================================================

struct pdcs_ctx {
  // problem (host copies of what the setup needs)
  int64_t m = 0, n = 0, n1 = 0, mg = 0, row_begin = 0;
  pdcs_params prm{};
  int device = 0, sms = 148;
  cudaStream_t st = nullptr;
  int mem_kind = PDCS_MEM_HOST;
  int rank = 0, world = 1;
  bool cones_set = false;
  std::string err;
  std::vector<int64_t> hptr;       // local CSR row pointers (host)
  std::vector<double> hl, hu;      // original bounds
  double hnorm = 0.0, cnorm = 0.0; // ||h||_inf, ||c||_inf (original data)
  // box-column order (plan_colperm): internal k holds the caller's column i2u[k]
  bool colperm = false;
  std::vector<int32_t> u2i, i2u;
  DBuf<int32_t> u2i_d, i2u_d;
  DBuf<double> permbuf;

  // device matrices
  DevCsr K, KT;
  DBuf<int32_t> Kptr, Kcol, KTptr, KTcol, planrows;
  DBuf<double> Kval, KTval;
  // device vectors (scaled space unless noted)
  DBuf<double> c0, h0, l0, u0;                 // original data
  DBuf<double> r, q, ct, ht, lt, ut;           // divisors, scaled data
  DBuf<double> x, xh, x0, xsum, kty, ktyh, xa, ktya, bx, candx, lam0, lam1, onesn;
  DBuf<double> y, yh, y0, ysum, kxh, kxd, ya, kxa, by, candy, res0, res1, onesm;
  DBuf<double> tmpn, tmpm, scal;
  DBuf<double> kxc, kx0;                       // K x of the current iterate and of the anchor (carried)
  // row sharding (comm.h): NCCL or in-process loopback communicator over the ranks
  bool dist = false;
  std::unique_ptr<Comm> comm;
  DBuf<double> ktyp;                           // local K~^T y partial before the all-reduce
  // the K~^T y partial in row chunks, each all-reduced on comm_st while the next
  // chunk's rows are summed (PDCS_AR_CHUNKS, default 4; CSR K~^T only)
  std::vector<SpmvPlan> ktc_plan;
  std::vector<int64_t> ktc_row;                // chunk c = rows [ktc_row[c], ktc_row[c+1])
  cudaStream_t comm_st = nullptr;
  std::vector<cudaEvent_t> ev_ar;
  cudaEvent_t ev_ar_done = nullptr;
  // column-tiled copies of K~ (pair gather) and K~^T (y gather), tiled.cuh
  struct TiledDev {
    bool on = false;
    TiledMat M;
    DBuf<TWork> work;
    DBuf<TBatch> batch;
    bool tma = true, sliced = false;
    DBuf<TChunk> chunk;
    DBuf<TSeg> seg;
    DBuf<int32_t> rowptr, col_d, blkb;
    DBuf<uint16_t> col_s, srow;
    DBuf<double> val_s, val_d, scratch;
    DBuf<TCItem> citem;
    int g_partial = 0, g_combine = 0;
    int64_t slot = 0;
    float tune_csr_ms = 0.f, tune_tiled_ms = 0.f;
    double build_ms = 0.0;                     // host build of the format
    double device_build_ms = 0.0;              // deferred build: device balancing + slicing
    TiledDevArrays dv;                         // device structure build (build_tiled_device)
    DBuf<int32_t> ccnt;                        // per-chunk arrival counters of the fused combine
    DBuf<TCItem> citem_w;                      // combine items of the chunks the fused kernel leaves
    TiledMat Mw;                               // M with citem = citem_w
    int g_combine_w = 0;
    bool fuse = false;                         // fused combine kept for this matrix
    float tune_fused_ms = 0.f;
  } tK, tKT;
  // Fused combine (tiled.cuh k_tiled_sliced<ELEM, Epi>): the last work item of a
  // chunk runs its epilogue.  Kept per matrix by the setup autotune when it is
  // >= 3% faster than partial + combine; PDCS_FUSED_COMBINE=1 / 0 forces it on / off.
  static int fused_env() {
    const char* e = std::getenv("PDCS_FUSED_COMBINE");
    return e ? (std::atoi(e) ? 1 : 0) : -1;
  }
  static bool fused(const TiledDev& D) { return D.fuse && D.sliced && !D.tma; }
  template <int ELEM, class Epi>
  void tiled_fused(const char* name, const char* wname, TiledDev& D, const double* xin, int guard, const Epi& e,
                   double* part, int64_t slot0) {
    launch(name, [&] {
      k_tiled_sliced<ELEM, Epi><<<D.g_partial, kTThreads, sliced_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard, e,
                                                                              D.ccnt.p, part, slot0);
    });
    if (D.Mw.ncitem)                           // chunks of many groups: combine over their items
      launch(wname, [&] {
        k_tiled_combine<Epi, ELEM><<<D.g_combine_w, kThreads, 0, st>>>(D.Mw, D.scratch.p, e, ctl, part,
                                                                        slot0 + D.M.nchunk);
      });
  }
  // accumulator slots a fused sweep writes (chunks, then the wide combine's CTAs)
  static int64_t fused_slots(const TiledDev& D) { return D.M.nchunk + D.g_combine_w; }
  // L2 column panels of K~ and K~^T (panels.cuh), kept by a setup autotune when
  // the gathered vector exceeds L2
  struct Panels {
    bool on = false;
    int P = 0;
    int64_t rows = 0, pcols = 0;
    int nx = 1;
    DBuf<int32_t> ptr, col, prow;
    DBuf<double> val, acc;
    std::vector<DevCsr> part;
    float tune_csr_ms = 0.f, tune_panel_ms = 0.f;
  } pK, pKT;
  double t_create_ms = 0.0, t_cones_ms = 0.0;  // wall time of pdcs_create / pdcs_set_cones
  // host builds of the tiled formats (build_tiled), started in pdcs_create
  TiledHost hK, hKT;
  std::thread thK, thKT;
  std::vector<int64_t> hKTptr;                 // K~^T structure for the background build
  std::vector<int32_t> hKTcol;
  DBuf<uint8_t> ek, rk;
  DBuf<Block> pblocks, rblocks;
  DBuf<double> warm_p, warm_r;                 // last SOC/RSOC multiplier of every block (trial ops)
  DBuf<int64_t> rsoc_offs_p, rsoc_offs_r;
  DBuf<double> tpart, kpart, gbuf;
  Ctl* ctl = nullptr;        // device
  Ctl* hctl = nullptr;       // pinned host mirror

  // block classes per side: [thread, warp, cta, grid] ranges into the block arrays
  struct BClass { int64_t begin = 0, count = 0; int grid = 0; int64_t slot = 0; int64_t kslot[2] = {0, 0}; };
  BClass pcls[kNClass], rcls[kNClass];   // thread, warp, cta, cluster, grid
  int64_t nslot_trial = 0, nslot_kkt = 0;
  int64_t slot_pe = 0, slot_spmv = 0, kslot_rows = 0, kslot_cols = 0;
  int g_pe = 0, g_m = 0, g_kr = 0, g_kc = 0, g_grid = 0;

  // CUDA graph of one accepted iteration: WHILE(rejected){trial} -> accept -> IF(check){check}
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_st = nullptr, cap_st2 = nullptr;
  // concurrent size-class kernels of one projection step (run_blocks): side
  // streams and fork/join events (graph branches when captured)
  cudaStream_t side[kNClass] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kNClass] = {};
  bool serial_blocks = false;
  unsigned long long g_retry = 0, g_check = 0;   // nonzero only while capturing / in the graph
  bool graph_failed = false;
  int64_t nodes_trial = 0, nodes_accept = 0, nodes_check = 0;

  // timing / counters
  bool timing = false;
  std::map<std::string, std::pair<double, int64_t>> ktimes;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  int64_t launches = 0;

  ~pdcs_ctx() {
    if (thK.joinable()) thK.join();
    if (thKT.joinable()) thKT.join();
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (cap_st) cudaStreamDestroy(cap_st);
    if (cap_st2) cudaStreamDestroy(cap_st2);
    for (int c = 0; c < kNClass; ++c) {
      if (side[c]) cudaStreamDestroy(side[c]);
      if (ev_join[c]) cudaEventDestroy(ev_join[c]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    for (auto e : ev_ar) cudaEventDestroy(e);
    if (ev_ar_done) cudaEventDestroy(ev_ar_done);
    if (comm_st) cudaStreamDestroy(comm_st);
    if (ctl) cudaFree(ctl);
    if (hctl) cudaFreeHost(hctl);
    for (auto e : evpool) cudaEventDestroy(e);
  }

  // ---------------------------------------------------------------- launch helpers
  cudaEvent_t ev() {
    if (evnext == evpool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      evpool.push_back(e);
    }
    return evpool[evnext++];
  }
  template <class F>
  void launch(const char* name, F&& f) {
    ++launches;
    if (!timing) {
      f();
      CK(cudaGetLastError());
      static const bool dbg = std::getenv("PDCS_DEBUG_SYNC") && std::atoi(std::getenv("PDCS_DEBUG_SYNC"));
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (dbg && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) fail(PDCS_ERR_CUDA, std::string("kernel '") + name + "': " + cudaGetErrorString(e));
      }
      return;
    }
    cudaEvent_t a = ev(), b = ev();
    CK(cudaEventRecord(a, st));
    f();
    CK(cudaGetLastError());
    CK(cudaEventRecord(b, st));
    pending.push_back({name, {a, b}});
  }
  void flush_timing() {
    if (!timing) return;
    CK(cudaStreamSynchronize(st));
    for (auto& p : pending) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
      auto& e = ktimes[p.first];
      e.first += ms;
      e.second += 1;
    }
    pending.clear();
    evnext = 0;
  }

  template <class Epi>
  void spmv(const char* name, const DevCsr& A, const double* x1, const double* x2, Epi epi, double* part,
            int64_t slot0) {
    if (&A == &K && pK.on) { psweep(name, pK, x1, x2, epi, part, slot0); return; }
    if (&A == &KT && pKT.on) { psweep(name, pKT, x1, x2, epi, part, slot0); return; }
    if (A.plan.total_cta == 0) return;
    launch(name, [&] {
      if (A.csr_u == 4)
        spmv_kernel<Epi, 4><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, x1, x2, A.plan, epi, ctl,
                                                                   part, slot0);
      else
        spmv_kernel<Epi><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, x1, x2, A.plan, epi, ctl,
                                                                part, slot0);
    });
  }
  // Entries in flight per lane of the CSR kernel for a matrix whose sweep
  // stays on the CSR path: 4 for K (the dual-trial sweep: MPO 227.6 -> 215.9
  // us, mixed 1527 -> 1503 us per step, Fisher unchanged), 8 for K^T (MPO's K^T
  // is slower with 4).  A timing of the plain product at setup did not predict
  // it (it kept 8 for MPO's K), so the rule is fixed.  PDCS_CSR_U4 = K | KT |
  // both | 0 overrides.
  void tune_csr_u(DevCsr& A, int64_t) {
    const bool isK = &A == &K;
    A.csr_u = isK ? 4 : 8;
    if (const char* e = std::getenv("PDCS_CSR_U4")) {
      const std::string v(e);
      A.csr_u = (v == "both" || (v == "K" && isK) || (v == "KT" && !isK)) ? 4 : 8;
    }
  }
  // A sweep through the L2 panels: one accumulating pass per panel, then the
  // sweep's epilogue over the accumulated rows (panels.cuh).
  template <class Epi>
  void psweep(const char* name, Panels& PA, const double* x1, const double* x2, Epi epi, double* part,
              int64_t slot0) {
    const char* pname = &PA == &pK ? "panel_K_partial" : "panel_KT_partial";
    int passes = 0;
    for (int p = 0; p < PA.P; ++p) {
      const DevCsr& A = PA.part[p];
      if (A.plan.total_cta == 0) continue;
      EpiPanelAcc<Epi> ea{epi, PA.acc.p, passes++ == 0 ? 1 : 0};
      launch(pname, [&] {
        spmv_kernel<EpiPanelAcc<Epi>><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, x1, x2, A.plan, ea,
                                                                             ctl, nullptr, 0);
      });
    }
    launch(name, [&] {
      k_panel_finish<Epi><<<(int)std::min<int64_t>(grid_for(PA.rows, sms), (int64_t)sms * 4), kThreads, 0, st>>>(
          PA.rows, PA.acc.p, epi, ctl, part, slot0);
    });
  }
  void spmv_store(const DevCsr& A, const double* xin, double* out, bool accepted_only = false) {
    EpiStore e{out};
    if (accepted_only) {
      EpiStoreAcc ea{out, 0};
      spmv("spmv_KT_partial", A, xin, nullptr, ea, nullptr, 0);
      return;
    }
    spmv("spmv_store", A, xin, nullptr, e, nullptr, 0);
  }

  // Product sweeps of the Eq. 9 check: the tiled copies when the autotune kept
  // them, else CSR.
  void spmv_check_KT(const double* yin, double* out) {
    if (!tKT.on) { spmv_store(KT, yin, out); return; }
    tiled_partial("tiled_check_partial", tKT, 1, yin, 0);
    EpiStore e{out};
    launch("check_combine", [&] {
      k_tiled_combine<EpiStore, 1><<<tKT.g_combine, kThreads, 0, st>>>(tKT.M, tKT.scratch.p, e, ctl, nullptr, 0);
    });
  }
  void spmv_check_K(const double* xin, double* out) {
    if (!tK.on) { spmv_store(K, xin, out); return; }
    tiled_partial("tiled_check_partial", tK, 1, xin, 0);
    EpiStore e{out};
    launch("check_combine", [&] {
      k_tiled_combine<EpiStore, 1><<<tK.g_combine, kThreads, 0, st>>>(tK.M, tK.scratch.p, e, ctl, nullptr, 0);
    });
  }

  void read_ctl() {
    CK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  void write_ctl() {
    CK(cudaMemcpyAsync(ctl, hctl, sizeof(Ctl), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  // In-place all-reduce over the row shards (no-op on a single rank).
  void allreduce(double* buf, size_t count, RedOp op, cudaStream_t s_ = nullptr) {
    if (!dist || count == 0) return;
    ++launches;
    const std::string e = comm->allreduce(buf, count, op, s_ ? s_ : st);
    if (!e.empty()) fail(PDCS_ERR_NCCL, e);
  }
  // n-vectors between the stored column order and the caller's (plan_colperm;
  // identity when no order was chosen).  to_caller returns a device pointer.
  const double* to_caller(const double* src) {
    if (!colperm) return src;
    k_gather_vals<<<grid_for(n, sms), kThreads, 0, st>>>(n, u2i_d.p, src, permbuf.p);
    CK(cudaGetLastError());
    return permbuf.p;
  }
  void from_caller(double* dst, const double* src, cudaMemcpyKind kind) {
    if (!n) return;
    if (!colperm) { CK(cudaMemcpyAsync(dst, src, n * sizeof(double), kind, st)); return; }
    CK(cudaMemcpyAsync(permbuf.p, src, n * sizeof(double), kind, st));
    k_gather_vals<<<grid_for(n, sms), kThreads, 0, st>>>(n, i2u_d.p, permbuf.p, dst);
    CK(cudaGetLastError());
  }
  // Time-limit stop, decided collectively so that every rank leaves at the
  // same Eq. 9 check (a rank-local clock would strand its peers in the next
  // collective).
  bool time_up(std::chrono::steady_clock::time_point t0, double limit) {
    if (!(limit > 0)) return false;
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return allreduce_host(el > limit ? 1.0 : 0.0, RedOp::Max) > 0.0;
  }
  // Host scalar all-reduce (setup values, collective stop decisions).
  double allreduce_host(double v, RedOp op) {
    if (!dist) return v;
    CK(cudaMemcpyAsync(scal.p + 7, &v, sizeof(double), cudaMemcpyHostToDevice, st));
    allreduce(scal.p + 7, 1, op);
    CK(cudaMemcpyAsync(&v, scal.p + 7, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return v;
  }

  // ---------------------------------------------------------------- block kernels
  BlockArgs bargs(bool primal, int op) {
    BlockArgs A{};
    A.blocks = primal ? pblocks.p : rblocks.p;
    A.op = op;
    A.x = x.p; A.c = ct.p; A.kty = kty.p; A.xh = xh.p;
    A.D = primal ? q.p : r.p;
    A.y = y.p; A.yh = yh.p; A.kxd = kxd.p;
    // warm-started multipliers for the trial projections (soc_team); env
    // PDCS_WARM=0 starts every Newton iteration at 0
    static const bool warm_off = std::getenv("PDCS_WARM") && std::atoi(std::getenv("PDCS_WARM")) == 0;
    if (!warm_off && (op == BOP_TRIAL_PRIMAL || op == BOP_TRIAL_DUAL)) A.warm = primal ? warm_p.p : warm_r.p;
    return A;
  }
  // The size classes of one side are independent (disjoint coordinates and
  // partial-sum slots): outside per-kernel timing the thread / warp / CTA /
  // cluster kernels run concurrently on side streams (each alone fills only a
  // fraction of the GPU: profiles/r1_ncu_blocks_mixed.txt), joined before the
  // grid-team kernel, which runs last on the main stream.
  // extra (optional): one more independent kernel of the same phase (the
  // trial's elementwise primal update), run as its own graph branch next to
  // the size classes; joined before the grid-team kernel like them.
  void run_blocks(bool primal, BlockArgs A, bool kkt, int cand,
                  const std::function<void(cudaStream_t)>* extra = nullptr) {
    BClass* cl = primal ? pcls : rcls;
    static const char* names[kNClass] = {"blocks_thread", "blocks_warp", "blocks_cta", "blocks_cluster",
                                         "blocks_grid"};
    int act[kNClass], na = 0;
    for (int c = 0; c < kNClass - 1; ++c)
      if (cl[c].count) act[na++] = c;
    const bool par = !timing && !serial_blocks && na + (extra ? 1 : 0) > 1;
    if (par) {
      if (!ev_fork) {
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        for (int c = 0; c < kNClass; ++c) {
          CK(cudaStreamCreateWithFlags(&side[c], cudaStreamNonBlocking));
          CK(cudaEventCreateWithFlags(&ev_join[c], cudaEventDisableTiming));
        }
      }
      CK(cudaEventRecord(ev_fork, st));
    }
    if (extra) {
      if (par) {
        CK(cudaStreamWaitEvent(side[kNClass - 1], ev_fork, 0));
        (*extra)(side[kNClass - 1]);
        CK(cudaEventRecord(ev_join[kNClass - 1], side[kNClass - 1]));
      } else {
        (*extra)(st);
      }
    }
    auto args = [&](int c) {
      BlockArgs B = A;
      B.blocks = A.blocks + cl[c].begin;
      B.nblocks = cl[c].count;
      B.cand = cand;
      B.part = kkt ? kpart.p : tpart.p;
      B.slot0 = kkt ? cl[c].kslot[cand] : cl[c].slot;
      if (A.warm) B.warm = A.warm + cl[c].begin;
      return B;
    };
    for (int i = 0; i < na; ++i) {
      const int c = act[i];
      const BlockArgs B = args(c);
      if (!par || i == 0) {
        launch(names[c], [&] { CK(launch_blocks(c, cl[c].grid, B, ctl, gbuf.p, st)); });
        continue;
      }
      CK(cudaStreamWaitEvent(side[i], ev_fork, 0));
      ++launches;
      CK(launch_blocks(c, cl[c].grid, B, ctl, gbuf.p, side[i]));
      CK(cudaEventRecord(ev_join[i], side[i]));
    }
    if (par) {
      for (int i = 1; i < na; ++i) CK(cudaStreamWaitEvent(st, ev_join[i], 0));
      if (extra) CK(cudaStreamWaitEvent(st, ev_join[kNClass - 1], 0));
    }
    if (cl[kNClass - 1].count) {
      const int c = kNClass - 1;
      const BlockArgs B = args(c);
      launch(names[c], [&] { CK(launch_blocks(c, cl[c].grid, B, ctl, gbuf.p, st)); });
    }
  }

  // ---------------------------------------------------------------- Alg. 1 pieces
  // One trial of AdaptiveStepPDHG (PDHG step Eq. 5 + accept test).
  void trial() {
    const std::function<void(cudaStream_t)> pe = [&](cudaStream_t s_) {
      launch("primal_elem", [&] {
        k_primal_elem<<<g_pe, kThreads, 0, s_>>>(n, ek.p, x.p, ct.p, kty.p, lt.p, ut.p, xh.p, ctl,
                                                 tpart.p, slot_pe);
      });
    };
    run_blocks(true, bargs(true, BOP_TRIAL_PRIMAL), false, 0, &pe);
    EpiDualTrial e{y.p, ht.p, rk.p, kxh.p, kxd.p, yh.p, kxc.p, 0.0, 0};
    if (tK.on && fused(tK)) {
      tiled_fused<1>("spmv_K_dual", "tiled_K_wide_combine", tK, xh.p, 1, e,
                     tpart.p, slot_spmv);
    } else if (tK.on) {
      tiled_partial("tiled_K_partial", tK, 1, xh.p, 1);
      launch("spmv_K_dual", [&] {
        k_tiled_combine<EpiDualTrial, 1><<<tK.g_combine, kThreads, 0, st>>>(tK.M, tK.scratch.p, e, ctl, tpart.p,
                                                                          slot_spmv);
      });
    } else {
      spmv("spmv_K_dual", K, xh.p, nullptr, e, tpart.p, slot_spmv);
    }
    run_blocks(false, bargs(false, BOP_TRIAL_DUAL), false, 0);
    if (dist) {
      launch("reduce_trial", [&] { k_reduce_trial<<<1, kDecideThreads, 0, st>>>(tpart.p, nslot_trial, ctl); });
      allreduce(&ctl->red3[1], 2, RedOp::Sum);     // ||dy||^2 and <dy, K dx> over the row shards
      launch("decide", [&] { k_decide<<<1, kDecideThreads, 0, st>>>(tpart.p, 0, ctl, g_retry, g_check, 1, FusedY{}); });
    } else {
      const FusedY fy = fuse_y() ? FusedY{m, yh.p, y0.p, y.p, ysum.p, kxh.p, kx0.p, kxc.p} : FusedY{};
      launch("decide", [&] { k_decide<<<1, kDecideThreads, 0, st>>>(tpart.p, nslot_trial, ctl, g_retry, g_check, 0, fy); });
    }
  }
  // Accepted step: y+ (Halpern/average on y), then K^T y+ with the fused
  // Halpern/average on x.
  // y-side Halpern update folded into k_decide (small m, single GPU; PDCS_FUSE_Y=0 disables)
  bool fuse_y_off = std::getenv("PDCS_FUSE_Y") && !std::atoi(std::getenv("PDCS_FUSE_Y"));   // read at create
  bool fuse_y() const { return !dist && m > 0 && m <= kFuseYMax && !fuse_y_off; }
  void accept() {
    if (!fuse_y())
      launch("halpern_y", [&] {
        k_halpern_y<<<g_m, kThreads, 0, st>>>(m, yh.p, y0.p, y.p, ysum.p, kxh.p, kx0.p, kxc.p, ctl);
      });
    if (dist) {
      // local K~^T y+ partial -> all-reduce -> x-side Halpern
      if (tKT.on) {
        tiled_partial("tiled_KT_partial", tKT, 1, y.p, 2);
        EpiStoreAcc ea{ktyp.p, 0};
        launch("spmv_KT_partial", [&] {
          k_tiled_combine<EpiStoreAcc, 1><<<tKT.g_combine, kThreads, 0, st>>>(tKT.M, tKT.scratch.p, ea, ctl, nullptr, 0);
        });
      } else if (!ktc_plan.empty() && !pKT.on) {
        // chunk c's rows summed, then all-reduced on comm_st while chunk c+1 runs
        for (size_t c = 0; c < ktc_plan.size(); ++c) {
          const SpmvPlan& pl = ktc_plan[c];
          EpiStoreAcc ea{ktyp.p, 0};
          if (pl.total_cta)
            launch("spmv_KT_partial", [&] {
              spmv_kernel<EpiStoreAcc><<<pl.total_cta, kThreads, 0, st>>>(KT.ptr, KT.col, KT.val, y.p, nullptr, pl, ea,
                                                                          ctl, nullptr, 0);
            });
          CK(cudaEventRecord(ev_ar[c], st));
          CK(cudaStreamWaitEvent(comm_st, ev_ar[c], 0));
          allreduce(ktyp.p + ktc_row[c], (size_t)(ktc_row[c + 1] - ktc_row[c]), RedOp::Sum, comm_st);
        }
        CK(cudaEventRecord(ev_ar_done, comm_st));
        CK(cudaStreamWaitEvent(st, ev_ar_done, 0));
      } else {
        spmv_store(KT, y.p, ktyp.p, true);
        allreduce(ktyp.p, n, RedOp::Sum);
      }
      if (tKT.on) allreduce(ktyp.p, n, RedOp::Sum);
      launch("halpern_x", [&] {
        k_halpern_x<<<g_pe, kThreads, 0, st>>>(n, xh.p, x0.p, ktyp.p, x.p, kty.p, xsum.p, ctl);
      });
      return;
    }
    EpiHalpernX e{xh.p, x0.p, x.p, kty.p, xsum.p, 0, 0, 0, 0, 0};
    if (tKT.on && fused(tKT)) {
      tiled_fused<1>("spmv_KT_halpern", "tiled_KT_wide_combine", tKT, y.p, 2, e, nullptr, 0);
    } else if (tKT.on) {
      tiled_partial("tiled_KT_partial", tKT, 1, y.p, 2);
      launch("spmv_KT_halpern", [&] {
        k_tiled_combine<EpiHalpernX, 1><<<tKT.g_combine, kThreads, 0, st>>>(tKT.M, tKT.scratch.p, e, ctl, nullptr, 0);
      });
    } else {
      spmv("spmv_KT_halpern", KT, y.p, nullptr, e, nullptr, 0);
    }
  }
  void kkt_launch(KktCand ca, KktCand cb, int ncand, int mode) {
    launch("kkt_rows", [&] {
      k_kkt_rows<<<g_kr, kThreads, 0, st>>>(m, rk.p, r.p, h0.p, y0.p, ca, cb, ncand, kpart.p, kslot_rows);
    });
    launch("kkt_cols", [&] {
      k_kkt_cols<<<g_kc, kThreads, 0, st>>>(n, ek.p, q.p, c0.p, l0.p, u0.p, x0.p, ca, cb, ncand, kpart.p,
                                            kslot_cols);
    });
    for (int c = 0; c < ncand; ++c) {
      const KktCand& C = c ? cb : ca;
      BlockArgs A = bargs(false, BOP_KKT_ROWS);
      A.scratch = C.res;
      run_blocks(false, A, true, c);
      BlockArgs B = bargs(true, BOP_KKT_COLS);
      B.scratch = C.lam;
      run_blocks(true, B, true, c);
    }
    // zero the slots of a candidate that was not evaluated
    if (ncand == 1) zero_cand1_kslots();
    launch("kkt_reduce", [&] { k_kkt_reduce<<<1, kThreads, 0, st>>>(kpart.p, nslot_kkt, ctl); });
    for (int c = 0; c < ncand; ++c) {             // row-side Eq. 9 terms over the shards
      allreduce(&ctl->kred[10 * c], 3, RedOp::Max);
      allreduce(&ctl->kred[10 * c + 3], 2, RedOp::Sum);
    }
    launch("kkt_decide", [&] { k_kkt_decide<<<1, 32, 0, st>>>(ncand, mode, hnorm, cnorm, ctl); });
  }
  void zero_cand1_kslots() {
    for (int side = 0; side < 2; ++side) {
      BClass* cl = side ? pcls : rcls;
      for (int c = 0; c < kNClass; ++c)
        if (cl[c].count)
          CK(cudaMemsetAsync(kpart.p + cl[c].kslot[1] * kKAcc, 0, (size_t)cl[c].grid * kKAcc * sizeof(double), st));
    }
  }
  // Eq. 9 check every check_interval accepted iterations.
  void check() {
    const bool van = prm.vanilla_pdhg != 0;
    KktCand c0{xh.p, yh.p, kxh.p, ktyh.p, res0.p, lam0.p};
    KktCand c1{xa.p, ya.p, kxa.p, ktya.p, res1.p, lam1.p};
    spmv_check_KT(yh.p, ktyh.p);    // K^T y^ of the current candidate (K x^ kept by the K pass)
    allreduce(ktyh.p, n, RedOp::Sum);
    if (!van) {
      launch("avg_elem", [&] { k_avg_elem<<<g_pe, kThreads, 0, st>>>(n, ek.p, xsum.p, lt.p, ut.p, xa.p, ctl); });
      BlockArgs A = bargs(true, BOP_AVG_PRIMAL);
      A.sum = xsum.p; A.out = xa.p;
      run_blocks(true, A, false, 0);
      launch("avg_elem", [&] { k_avg_elem<<<g_m, kThreads, 0, st>>>(m, rk.p, ysum.p, nullptr, nullptr, ya.p, ctl); });
      BlockArgs B = bargs(false, BOP_AVG_DUAL);
      B.sum = ysum.p; B.out = ya.p;
      run_blocks(false, B, false, 0);
      spmv_check_K(xa.p, kxa.p);
      spmv_check_KT(ya.p, ktya.p);
      allreduce(ktya.p, n, RedOp::Sum);
    }
    kkt_launch(c0, c1, van ? 1 : 2, 1);
    RestartArgs R{};
    R.n = n; R.m = m;
    R.cx[0] = xh.p; R.cy[0] = yh.p; R.ckty[0] = ktyh.p;
    R.cx[1] = xa.p; R.cy[1] = ya.p; R.ckty[1] = ktya.p;
    R.ckx[0] = kxh.p; R.ckx[1] = kxa.p; R.kxc = kxc.p; R.kx0 = kx0.p;
    R.x = x.p; R.x0 = x0.p; R.y = y.p; R.y0 = y0.p; R.kty = kty.p;
    R.xsum = xsum.p; R.ysum = ysum.p; R.bx = bx.p; R.by = by.p; R.candx = candx.p;
    R.candy = candy.p;
    launch("restart_copy", [&] {
      k_restart_copy<<<grid_for(std::max(n, m), sms), kThreads, 0, st>>>(R, ctl);
    });
    // the carried K x is refreshed with a fresh product at every check, so its
    // drift (O(k eps) |K x| through the Halpern recursion, P6) spans
    // at most one check interval
    spmv_check_K(x.p, kxc.p);
  }

  // Add a conditional node (WHILE / IF) at the current capture position of `st`
  // and capture body() into its body graph on a second stream.
  template <class F>
  void capture_conditional(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type, F&& body,
                           int64_t& nodes) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, cg, deps, ndeps, &np));
    CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t bodyg = np.conditional.phGraph_out[0];
    cudaStream_t saved = st;
    st = cap_st2;
    const int64_t l0 = launches;
    CK(cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body();
    CK(cudaStreamEndCapture(st, &bodyg));
    nodes = launches - l0;
    st = saved;
  }

  // Build the per-iteration graph once (after setup); on failure fall back to
  // the host-driven loop.
  void build_graph() {
    if (gexec || graph_failed) return;
    const cudaStream_t saved_st = st;
    const bool tsave_ = timing;
    try {
      if (!cap_st) CK(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
      if (!cap_st2) CK(cudaStreamCreateWithFlags(&cap_st2, cudaStreamNonBlocking));
      CK(cudaGraphCreate(&graph, 0));
      cudaGraphConditionalHandle hr, hc;
      CK(cudaGraphConditionalHandleCreate(&hr, graph, 1, cudaGraphCondAssignDefault));
      CK(cudaGraphConditionalHandleCreate(&hc, graph, 0, cudaGraphCondAssignDefault));
      cudaStream_t saved = st;
      const bool tsave = timing;
      timing = false;
      st = cap_st;
      g_retry = (unsigned long long)hr;
      g_check = (unsigned long long)hc;
      CK(cudaStreamBeginCaptureToGraph(st, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      capture_conditional(hr, cudaGraphCondTypeWhile, [&] { trial(); }, nodes_trial);
      const int64_t l0 = launches;
      accept();
      nodes_accept = launches - l0;
      capture_conditional(hc, cudaGraphCondTypeIf, [&] { check(); }, nodes_check);
      cudaGraph_t out;
      CK(cudaStreamEndCapture(st, &out));
      st = saved;
      timing = tsave;
      g_retry = g_check = 0;
      CK(cudaGraphInstantiate(&gexec, graph, 0));
    } catch (const CudaErr& e) {
      graph_abandon(saved_st, tsave_, std::string(cudaGetErrorString(e.e)) + " at " + e.what);
    } catch (const StatusErr& e) {                 // e.g. a collective refused under capture
      graph_abandon(saved_st, tsave_, e.msg);
    }
  }
  void graph_abandon(cudaStream_t saved, bool tsave, const std::string& why) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cap_st && cudaStreamIsCapturing(cap_st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t g2 = nullptr;
      cudaStreamEndCapture(cap_st, &g2);
    }
    st = saved;
    timing = tsave;
    graph_failed = true;
    g_retry = g_check = 0;
    cudaGetLastError();
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
    err = "graph build failed (host loop used): " + why;
  }

  // dynamic shared memory of the partial kernels, from the matrix's own tile size
  static size_t tile_bytes(const TiledDev& D) { return (size_t)D.M.T * D.M.elem * sizeof(double); }
  static size_t tma_smem(const TiledDev& D) {
    return 2 * tile_bytes(D) + (size_t)kNST * kBQ * 32 + (size_t)kNST * (kBQ + 2) * 8 +
           (size_t)kNST * kBR * 4 + (size_t)kTRows * D.M.elem * sizeof(double);
  }
  // launch the partial products of a tiled matrix (TMA pipeline or the plain kernel)
  void tiled_partial(const char* name, TiledDev& D, int elem, const double* xin, int guard) {
    launch(name, [&] {
      if (elem == 2) {
        if (D.tma) k_tiled_tma<2><<<D.g_partial, kTThreads, tma_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
        else if (D.sliced) k_tiled_sliced<2><<<D.g_partial, kTThreads, sliced_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
        else k_tiled_partial<2><<<D.g_partial, kTThreads, tiled_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
      } else {
        if (D.tma) k_tiled_tma<1><<<D.g_partial, kTThreads, tma_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
        else if (D.sliced) k_tiled_sliced<1><<<D.g_partial, kTThreads, sliced_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
        else k_tiled_partial<1><<<D.g_partial, kTThreads, tiled_smem(D), st>>>(D.M, xin, D.scratch.p, ctl, guard);
      }
    });
  }
  static size_t sliced_smem(const TiledDev& D) { return 2 * tile_bytes(D) + (size_t)kTRows * D.M.elem * sizeof(double); }
  static size_t tiled_smem(const TiledDev& D) { return tile_bytes(D) + (size_t)kTRows * D.M.elem * sizeof(double); }

  // Build the tiled copy of a CSR (structure on the host, scaled values on the device).
  void make_tiled(TiledDev& D, TiledHost& H, int64_t rows, int64_t nvec, int elem, const double* dval) {
    const double frac = H.nnz ? (double)H.staged / (double)H.nnz : 0.0;
    const char* env = std::getenv("PDCS_TILED");
    const bool want = H.devbuilt || (env ? std::atoi(env) != 0 : frac >= kTiledMinFrac);
    D.on = want && H.nnz > 0;
    if (!D.on) { H = TiledHost(); return; }
    SetupTrace tr;
    upload(D.work, H.work, st);
    upload(D.batch, H.batch, st);
    upload(D.chunk, H.chunk, st);
    upload(D.seg, H.seg, st);
    DBuf<int32_t> perm;
    if (H.devbuilt) {
      // built on the device (build_tiled_device): take its arrays, gather the values
      take(D.rowptr, D.dv.rowptr); take(D.srow, D.dv.srow); take(D.col_s, D.dv.col_s);
      take(D.col_d, D.dv.col_d); take(D.blkb, D.dv.blkb);
      D.val_s.alloc(std::max<size_t>(H.tot_s, 1));
      D.val_d.alloc(std::max<size_t>(H.tot_d, 1));
      if (H.tot_s)
        k_gather_vals<<<grid_for((int64_t)H.tot_s, sms, 32), kThreads, 0, st>>>((int64_t)H.tot_s, D.dv.perm_s.p, dval, D.val_s.p);
      if (H.tot_d)
        k_gather_vals<<<grid_for((int64_t)H.tot_d, sms, 32), kThreads, 0, st>>>((int64_t)H.tot_d, D.dv.perm_d.p, dval, D.val_d.p);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(st));
      D.dv.perm_s.free_();
      D.dv.perm_d.free_();
      tr.mark("  tiled: gather values (device-built)", st);
    } else if (H.parts.empty()) {
      upload(D.rowptr, H.rowptr, st);
      upload(D.srow, H.srow, st);
      upload(D.col_s, H.col_s, st);
      upload(D.col_d, H.col_d, st);
      upload(D.blkb, H.blkb, st);
    } else {
      // slices of the parts at their offsets; the gaps and tails hold the
      // padding values of the concatenated layout (ids 0, permutation -1)
      D.rowptr.alloc(H.tot_rp); D.srow.alloc(H.tot_rp); D.col_s.alloc(H.tot_s);
      D.col_d.alloc(std::max<size_t>(H.tot_d, 1)); D.blkb.alloc(H.tot_bb);
      perm.alloc(std::max<size_t>(H.tot_s, 1));
      CK(cudaMemsetAsync(D.rowptr.p, 0, H.tot_rp * sizeof(int32_t), st));
      CK(cudaMemsetAsync(D.srow.p, 0, H.tot_rp * sizeof(uint16_t), st));
      CK(cudaMemsetAsync(D.col_s.p, 0, H.tot_s * sizeof(uint16_t), st));
      CK(cudaMemsetAsync(D.blkb.p, 0, H.tot_bb * sizeof(int32_t), st));
      CK(cudaMemsetAsync(perm.p, 0xff, H.tot_s * sizeof(int32_t), st));
      auto put = [&](auto* dst, const auto& v, size_t off) {
        if (!v.empty()) CK(cudaMemcpyAsync(dst + off, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, st));
      };
      DBuf<uint16_t> pcol;                     // deferred build: the unbalanced row-major quads
      DBuf<int32_t> pperm;
      if (H.defer) {
        pcol.alloc(std::max<size_t>(H.tot_pre, 1));
        pperm.alloc(std::max<size_t>(H.tot_pre, 1));
      }
      for (size_t w = 0; w < H.parts.size(); ++w) {
        const TiledHost& P = H.parts[w];
        put(D.rowptr.p, P.rowptr, H.o_rp[w]);
        put(D.srow.p, P.srow, H.o_rp[w]);
        if (H.defer) {
          put(pcol.p, P.col_s, H.o_pre[w]);
          put(pperm.p, P.perm_s, H.o_pre[w]);
        } else {
          put(D.col_s.p, P.col_s, H.o_s[w]);
          put(perm.p, P.perm_s, H.o_s[w]);
        }
        put(D.col_d.p, P.col_d, H.o_d[w]);
        put(D.blkb.p, P.blkb, H.o_bb[w]);
      }
      tr.mark("  tiled: part uploads", st);
      if (H.defer && !H.dblk.empty()) {
        // bank balancing and sliced re-layout on the device (tiled.cuh)
        const auto t0 = std::chrono::steady_clock::now();
        DBuf<TDefer> dseg;
        DBuf<int2> dblk;
        upload(dseg, H.dseg, st);
        upload(dblk, H.dblk, st);
        DBuf<uint16_t> bcol, ncol;
        DBuf<int32_t> bperm, nperm;
        bcol.alloc(H.tot_pre); ncol.alloc(H.tot_pre); bperm.alloc(H.tot_pre); nperm.alloc(H.tot_pre);
        const int64_t nb = (int64_t)H.dblk.size();
        const int tb = 128;
        launch_tile_balance(dseg.p, H.dseg, dblk.p, nb, elem, D.rowptr.p, pcol.p, pperm.p, bcol.p, bperm.p, ncol.p,
                            nperm.p, st);
        k_tile_slice<<<(int)((nb + tb - 1) / tb), tb, 0, st>>>(dseg.p, dblk.p, nb, D.rowptr.p, D.blkb.p, ncol.p,
                                                               nperm.p, D.col_s.p, perm.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
        D.device_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        tr.mark("  tiled: balance + slice", st);
      }
    }
    if (!H.devbuilt) {
    D.val_s.alloc(std::max<size_t>(H.n_s(), 1));
    D.val_d.alloc(std::max<size_t>(H.n_d(), 1));
    if (H.n_s()) {
      if (H.parts.empty()) upload(perm, H.perm_s, st);
      k_gather_vals<<<grid_for((int64_t)H.n_s(), sms, 32), kThreads, 0, st>>>((int64_t)H.n_s(), perm.p, dval, D.val_s.p);
      CK(cudaStreamSynchronize(st));
    }
    if (H.n_d()) {
      if (H.parts.empty()) upload(perm, H.perm_d, st);
      else {
        perm.alloc(H.tot_d);
        for (size_t w = 0; w < H.parts.size(); ++w)
          if (!H.parts[w].perm_d.empty())
            CK(cudaMemcpyAsync(perm.p + H.o_d[w], H.parts[w].perm_d.data(), H.parts[w].perm_d.size() * sizeof(int32_t),
                               cudaMemcpyHostToDevice, st));
      }
      k_gather_vals<<<grid_for((int64_t)H.n_d(), sms, 32), kThreads, 0, st>>>((int64_t)H.n_d(), perm.p, dval, D.val_d.p);
      CK(cudaStreamSynchronize(st));
    }
    tr.mark("  tiled: gather values", st);
    }
    D.scratch.alloc(std::max<int64_t>(H.scratch, 1));
    TiledMat& M = D.M;
    M.m = rows; M.nvec = nvec; M.nwork = (int64_t)H.work.size(); M.nchunk = (int64_t)H.chunk.size();
    M.T = H.T; M.elem = elem;
    M.work = D.work.p; M.chunk = D.chunk.p; M.seg = D.seg.p; M.rowptr = D.rowptr.p; M.srow = D.srow.p;
    M.val_s = D.val_s.p; M.col_s = D.col_s.p; M.val_d = D.val_d.p; M.col_d = D.col_d.p;
    M.batch = D.batch.p;
    M.blkb = D.blkb.p;
    // TMA-pipelined variant (k_tiled_tma) is opt-in: on B200 it measured slower than
    // the 4-CTA/SM register-streaming kernel, PDCS_TMA=1 enables it.
    D.tma = H.tma;
    D.sliced = H.sliced;
    int occ = 1;
    if (elem == 2) {
      CK(cudaFuncSetAttribute(k_tiled_partial<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiled_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<2, EpiStore2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem(D)));
      if (D.tma) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_tma<2>, kTThreads, tma_smem(D)));
      else if (D.sliced) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_sliced<2>, kTThreads, sliced_smem(D)));
      else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_partial<2>, kTThreads, tiled_smem(D)));
    } else {
      CK(cudaFuncSetAttribute(k_tiled_partial<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiled_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<1, EpiHalpernX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<1, EpiDualTrial>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_sliced<1, EpiStore>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sliced_smem(D)));
      CK(cudaFuncSetAttribute(k_tiled_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tma_smem(D)));
      if (D.tma) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_tma<1>, kTThreads, tma_smem(D)));
      else if (D.sliced) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_sliced<1>, kTThreads, sliced_smem(D)));
      else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled_partial<1>, kTThreads, tiled_smem(D)));
    }
    D.g_partial = (int)std::max<int64_t>(1, std::min<int64_t>(M.nwork, (int64_t)sms * std::max(occ, 1)));
    std::vector<TCItem> citems;                // combine items (k_tiled_combine)
    for (size_t c = 0; c < H.chunk.size(); ++c) {
      const TChunk& C = H.chunk[c];
      const int step = C.ngroups >= kCombWideG ? kCombRowsWide : C.ngroups <= kCombNarrowG ? kCombRowsNarrow : kThreads;
      for (int32_t r0 = 0; r0 < C.nrows; r0 += step) citems.push_back(TCItem{(int32_t)c, r0});
    }
    upload(D.citem, citems, st);
    {
      std::vector<TCItem> wide;
      for (const TCItem& I : citems)
        if (H.chunk[I.chunk].ngroups >= kCombWideG) wide.push_back(I);
      upload(D.citem_w, wide, st);
      D.Mw = M;
      D.Mw.citem = D.citem_w.p;
      D.Mw.ncitem = (int64_t)wide.size();
      D.g_combine_w = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)wide.size(), (int64_t)sms * 8));
    }
    D.ccnt.alloc(std::max<int64_t>(M.nchunk, 1));
    CK(cudaMemsetAsync(D.ccnt.p, 0, std::max<int64_t>(M.nchunk, 1) * sizeof(int32_t), st));
    M.citem = D.citem.p;
    M.ncitem = (int64_t)citems.size();
    H = TiledHost();                           // host copy no longer needed
    D.g_combine = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)citems.size(), (int64_t)sms * 8));
    D.fuse = fused_env() == 1;
    // Setup-time autotune: keep the tiled copy only if it beats the CSR kernel
    // by >= 10% on this matrix (gather locality decides).
    if (!env) {
      const DevCsr& A = &D == &tK ? K : KT;      // the CSR this tiled copy stands for
      DBuf<double> xin, out;
      xin.alloc(std::max<int64_t>(nvec * elem, 1) + 2);
      out.alloc(std::max<int64_t>(rows, 1));
      k_fill<<<grid_for(nvec * elem, sms), kThreads, 0, st>>>(nvec * elem, 1.0, xin.p);
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      auto run_csr = [&] {
        if (elem == 2) {
          EpiStore2 e{out.p};
          spmv_kernel<EpiStore2><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, xin.p, nullptr, A.plan, e, ctl, nullptr, 0);
        } else {
          EpiStore e{out.p};
          spmv_kernel<EpiStore><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, xin.p, nullptr, A.plan, e, ctl, nullptr, 0);
        }
      };
      auto run_fused = [&] {
        if (elem == 2) tiled_fused<2>("autotune", "autotune", D, xin.p, 0, EpiStore2{out.p}, nullptr, 0);
        else tiled_fused<1>("autotune", "autotune", D, xin.p, 0, EpiStore{out.p}, nullptr, 0);
      };
      auto run_tiled = [&] {
        if (elem == 2) {
          tiled_partial("autotune", D, 2, xin.p, 0);
          EpiStore2 e{out.p};
          k_tiled_combine<EpiStore2, 2><<<D.g_combine, kThreads, 0, st>>>(M, D.scratch.p, e, ctl, nullptr, 0);
        } else {
          tiled_partial("autotune", D, 1, xin.p, 0);
          EpiStore e{out.p};
          k_tiled_combine<EpiStore, 1><<<D.g_combine, kThreads, 0, st>>>(M, D.scratch.p, e, ctl, nullptr, 0);
        }
      };
      static const bool dbg = std::getenv("PDCS_DEBUG_SYNC") && std::atoi(std::getenv("PDCS_DEBUG_SYNC"));
      auto timeit = [&](auto&& f) {   // median of 5 after 2 warm-ups
        f();
        if (dbg) { CK(cudaStreamSynchronize(st)); CK(cudaGetLastError()); }
        f();
        float v[5];
        for (int i = 0; i < 5; ++i) {
          CK(cudaEventRecord(a, st));
          f();
          CK(cudaEventRecord(b, st));
          if (dbg) {
            const cudaError_t e = cudaEventSynchronize(b);
            if (e != cudaSuccess) fail(PDCS_ERR_CUDA, "autotune rep " + std::to_string(i) + ": " + cudaGetErrorString(e));
          }
          CK(cudaEventSynchronize(b));
          CK(cudaEventElapsedTime(&v[i], a, b));
        }
        std::sort(v, v + 5);
        return v[2];
      };
      if (dbg) std::fprintf(stderr, "[pdcs debug] autotune csr, elem %d\n", elem);
      const float tc = timeit(run_csr);
      if (dbg) std::fprintf(stderr, "[pdcs debug] autotune tiled\n");
      float tt = timeit(run_tiled);
      if (dbg) std::fprintf(stderr, "[pdcs debug] autotune fused\n");
      const int fe = fused_env();
      if (D.sliced && !D.tma && fe != 0) {
        D.tune_fused_ms = timeit(run_fused);
        D.fuse = fe == 1 || D.tune_fused_ms < 0.97f * tt;
        if (D.fuse) tt = std::min(tt, D.tune_fused_ms);
      }
      CK(cudaGetLastError());
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      D.tune_csr_ms = tc;
      D.tune_tiled_ms = tt;
      if (!(tt < 0.9f * tc)) {
        D.on = false;
        D.work.free_(); D.chunk.free_(); D.seg.free_(); D.rowptr.free_(); D.srow.free_(); D.col_d.free_(); D.col_s.free_();
        D.blkb.free_();
        D.val_s.free_(); D.val_d.free_(); D.scratch.free_(); D.citem.free_();
      }
    }
  }

  // L2 column panels of A (rows x cols, gathering nx doubles per column) when
  // the gathered vector exceeds L2 and the tiled copy is off (panels.cuh).
  // PDCS_PANELS=0 disables, =P forces P panels (no autotune); PDCS_PANEL_MB
  // sets the vector slice per panel (default 24 MB of the 126 MB L2).  Kept only
  // if the setup autotune measures it >= 10% faster than the CSR sweep.
  void build_panels(Panels& PA, const DevCsr& A, bool tiled_on, int nx) {
    const char* e = std::getenv("PDCS_PANELS");
    const int force = e ? std::atoi(e) : -1;
    if (force == 0 || A.nnz == 0 || A.m == 0 || A.n == 0) return;
    if (force < 0 && tiled_on) return;
    const double vec_bytes = (double)A.n * 8.0 * nx;
    const double panel_mb = std::getenv("PDCS_PANEL_MB") ? std::atof(std::getenv("PDCS_PANEL_MB")) : 24.0;
    if (force < 0 && vec_bytes < 64.0 * (1 << 20)) return;
    const int P = force > 0 ? force : (int)std::ceil(vec_bytes / (panel_mb * (1 << 20)));
    if (P < 1 || (force < 0 && P < 2)) return;
    const int64_t rows = A.m, pcols = (A.n + P - 1) / P;
    PA.P = P; PA.rows = rows; PA.pcols = pcols; PA.nx = nx;
    DBuf<int32_t> cnt;
    cnt.alloc((int64_t)P * rows + 1);
    CK(cudaMemsetAsync(cnt.p, 0, ((int64_t)P * rows + 1) * sizeof(int32_t), st));
    k_panel_count<<<grid_for(rows, sms, 32), kThreads, 0, st>>>(rows, A.ptr, A.col, pcols, cnt.p);
    PA.ptr.alloc((int64_t)P * rows + 1);
    size_t tmpb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmpb, cnt.p, PA.ptr.p, (int)(P * rows + 1), st));
    DBuf<char> tmp;
    tmp.alloc((int64_t)tmpb);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmpb, cnt.p, PA.ptr.p, (int)(P * rows + 1), st));
    PA.col.alloc(A.nnz);
    PA.val.alloc(A.nnz);
    k_panel_scatter<<<grid_for(rows, sms, 32), kThreads, 0, st>>>(rows, A.ptr, A.col, A.val, pcols, PA.ptr.p,
                                                                  PA.col.p, PA.val.p);
    CK(cudaGetLastError());
    std::vector<int32_t> hp((size_t)P * rows + 1);
    CK(cudaMemcpyAsync(hp.data(), PA.ptr.p, hp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int32_t> rowstore;
    std::vector<size_t> offs;
    PA.part.assign(P, DevCsr{});
    std::vector<int64_t> pp(rows + 1);
    for (int p = 0; p < P; ++p) {
      for (int64_t i = 0; i <= rows; ++i) pp[i] = hp[(size_t)p * rows + i] - hp[(size_t)p * rows];
      DevCsr& D = PA.part[p];
      D.m = rows; D.n = A.n; D.nnz = pp[rows];
      D.ptr = PA.ptr.p + (size_t)p * rows; D.col = PA.col.p; D.val = PA.val.p;
      build_plan(D, pp, rowstore, offs);
    }
    upload(PA.prow, rowstore, st);
    for (DevCsr& D : PA.part)
      for (int c = 0; c < D.plan.ncls; ++c)
        if (D.plan.cls[c].rows) D.plan.cls[c].rows = PA.prow.p + ((size_t)(uintptr_t)D.plan.cls[c].rows - 1);
    PA.acc.alloc(rows * nx);
    PA.on = true;
    if (force > 0) return;
    // setup autotune: the panelled product against the CSR one, on this matrix
    DBuf<double> xin, out;
    xin.alloc(A.n * nx + 2);
    out.alloc(rows);
    k_fill<<<grid_for(A.n * nx, sms), kThreads, 0, st>>>(A.n * nx, 1.0, xin.p);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto timeit = [&](auto&& f) {   // median of 5 after 2 warm-ups
      f();
      f();
      float v[5];
      for (int i = 0; i < 5; ++i) {
        CK(cudaEventRecord(a, st));
        f();
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&v[i], a, b));
      }
      std::sort(v, v + 5);
      return v[2];
    };
    const bool was_timing = timing;
    timing = false;
    float tc, tp;
    if (nx == 2) {
      EpiStore2 es{out.p};
      tc = timeit([&] { spmv_kernel<EpiStore2><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, xin.p, nullptr,
                                                                                 A.plan, es, ctl, nullptr, 0); });
      tp = timeit([&] { psweep("autotune", PA, xin.p, nullptr, es, nullptr, 0); });
    } else {
      EpiStore es{out.p};
      tc = timeit([&] { spmv_kernel<EpiStore><<<A.plan.total_cta, kThreads, 0, st>>>(A.ptr, A.col, A.val, xin.p, nullptr,
                                                                                A.plan, es, ctl, nullptr, 0); });
      tp = timeit([&] { psweep("autotune", PA, xin.p, nullptr, es, nullptr, 0); });
    }
    timing = was_timing;
    CK(cudaGetLastError());
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    PA.tune_csr_ms = tc;
    PA.tune_panel_ms = tp;
    if (!(tp < 0.9f * tc)) {
      PA.on = false;
      PA.ptr.free_(); PA.col.free_(); PA.val.free_(); PA.prow.free_(); PA.acc.free_();
      PA.part.clear();
    }
  }

  // products of (x, y) into (kx, kty)
  void products(const double* xs, const double* ys, double* kxo, double* ktyo) {
    spmv_store(K, xs, kxo);
    spmv_store(KT, ys, ktyo);
    allreduce(ktyo, n, RedOp::Sum);
  }

  // ---------------------------------------------------------------- setup helpers
  void build_plan(DevCsr& A, const std::vector<int64_t>& ptr, std::vector<int32_t>& rowstore,
                  std::vector<size_t>& offs, int64_t row_a = 0, int64_t row_b = -1) {
    const int64_t rows = row_b >= 0 ? row_b : (int64_t)ptr.size() - 1;
    // V classes: 1, 4, 8, 16, 32 lanes per row, 0 = one CTA per row.  Upper
    // row-length bounds per class (PDCS_SPMV_BINS="b1,b4,b8,b16,b32" overrides).
    const int Vs[kMaxClasses] = {1, 4, 8, 16, 32, 0};
    int64_t bound[5] = {2, 12, 48, 96, (int64_t)1 << 40};   // measured on B200 (profiles/)
    bool fixed_bins = false;
    if (const char* env = std::getenv("PDCS_SPMV_BINS")) {
      int64_t b[5];
      if (std::sscanf(env, "%ld,%ld,%ld,%ld,%ld", &b[0], &b[1], &b[2], &b[3], &b[4]) == 5) {
        for (int i = 0; i < 5; ++i) bound[i] = b[i];
        fixed_bins = true;
      }
    }
    // class of every row (one byte each), then per class its count and row
    // range; row lists are materialised only for classes whose rows are not
    // contiguous (Fisher's K^T: 1e7 rows, one class, had been pushed into a
    // 1e7-entry list: ~0.14 s)
    std::vector<uint8_t> cls_of((size_t)std::max<int64_t>(rows - row_a, 0));
    int64_t nlong = 0;
    for (int64_t i = row_a; i < rows; ++i) {
      const int64_t L = ptr[i + 1] - ptr[i];
      int c = 5;
      for (int k = 0; k < 5; ++k)
        if (L <= bound[k]) { c = k; break; }
      cls_of[i - row_a] = (uint8_t)c;
      nlong += c == 4 && L > 1024;
    }
    // Few very long rows (> 1024 nnz; fewer than 16 per SM): one warp per row
    // leaves the SMs idle while each warp walks a long serial chain of gathers
    // (Fisher's 1000 supply rows of 1e4 nnz), so they get a CTA each.  With
    // many of them (Lasso K^T: 1e4 rows) warp-per-row is faster
    // (profiles/r1_sweep_v0.txt).
    if (!fixed_bins && nlong && nlong < (int64_t)sms * 16)
      for (int64_t i = row_a; i < rows; ++i)
        if (cls_of[i - row_a] == 4 && ptr[i + 1] - ptr[i] > 1024) cls_of[i - row_a] = 5;
    int64_t ccount[kMaxClasses] = {0}, cfirst[kMaxClasses], clast[kMaxClasses];
    for (int c = 0; c < kMaxClasses; ++c) { cfirst[c] = -1; clast[c] = -1; }
    for (int64_t i = row_a; i < rows; ++i) {
      const int c = cls_of[i - row_a];
      if (cfirst[c] < 0) cfirst[c] = i;
      clast[c] = i;
      ++ccount[c];
    }
    SpmvPlan P{};
    P.ncls = 0;
    int total = 0;
    // The one-CTA-per-row class goes first, one row per CTA: CTAs are
    // dispatched in index order, so the long rows start at once and the short
    // classes fill the SMs behind them (last, with a grid stride over 4 CTAs
    // per SM, they had made a tail of second rows: Fisher's 1000 supply rows)
    static const int order[kMaxClasses] = {5, 0, 1, 2, 3, 4};
    for (int oc = 0; oc < kMaxClasses; ++oc) {
      const int c = order[oc];
      if (ccount[c] == 0) continue;
      SpmvClass& K_ = P.cls[P.ncls++];
      K_.V = Vs[c];
      K_.nrows = ccount[c];
      const bool contiguous = clast[c] - cfirst[c] + 1 == K_.nrows;
      K_.range_begin = contiguous ? cfirst[c] : 0;
      K_.rows = nullptr;
      if (!contiguous) {
        offs.push_back(rowstore.size());
        for (int64_t i = cfirst[c]; i <= clast[c]; ++i)
          if (cls_of[i - row_a] == c) rowstore.push_back((int32_t)i);
        K_.rows = (const int32_t*)(uintptr_t)(offs.back() + 1);   // patched after upload
      }
      int64_t rows_per_cta = K_.V == 0 ? 1 : K_.V == 1 ? kThreads : kThreads / K_.V;
      int64_t g = (K_.nrows + rows_per_cta - 1) / rows_per_cta;
      const int64_t cap = K_.V == 0 ? (int64_t)sms * 16 : (int64_t)sms * 8;
      K_.ncta = (int32_t)std::max<int64_t>(1, std::min(g, cap));
      total += K_.ncta;
    }
    P.total_cta = total;
    A.plan = P;
  }
  void patch_plan(DevCsr& A) {
    for (int c = 0; c < A.plan.ncls; ++c)
      if (A.plan.cls[c].rows) {
        const size_t off = (size_t)(uintptr_t)A.plan.cls[c].rows - 1;
        A.plan.cls[c].rows = planrows.p + off;
      }
  }
};

// ============================================================================
namespace {

pdcs_status guard_impl(pdcs_ctx* ctx, const std::function<void()>& f) {
  try {
    f();
    return PDCS_OK;
  } catch (const CudaErr& e) {
    std::string msg = std::string("CUDA error ") + cudaGetErrorString(e.e) + " at line " +
                      std::to_string(e.line) + ": " + e.what;
    if (ctx) ctx->err = msg; else g_create_error = msg;
    return PDCS_ERR_CUDA;
  } catch (const StatusErr& e) {
    if (ctx) ctx->err = e.msg; else g_create_error = e.msg;
    return e.st;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what(); else g_create_error = e.what();
    return PDCS_ERR_ARG;
  }
}
// A failing rank tells its peers (loopback: they leave their rendezvous with an
// error instead of waiting for a collective this rank will never join).
pdcs_status guard(pdcs_ctx* ctx, const std::function<void()>& f) {
  const pdcs_status s = guard_impl(ctx, f);
  if (s != PDCS_OK && ctx && ctx->comm) ctx->comm->on_error(ctx->err);
  return s;
}

template <class T>
std::vector<T> to_host(const T* p, int64_t count, int mem_kind) {
  if (count <= 0) return std::vector<T>();
  if (!p) fail(PDCS_ERR_ARG, "null input pointer");
  if (mem_kind != PDCS_MEM_DEVICE) return std::vector<T>(p, p + count);   // one pass, no zero-fill first
  std::vector<T> v((size_t)count);
  CK(cudaMemcpy(v.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost));
  return v;
}


}  // namespace

// Internal: (re)initialise z, z0, products, sums and e_anchor from the current x, y.
static void reset_from_current(pdcs_ctx* ctx) {
  cudaStream_t st = ctx->st;
  const int64_t n = ctx->n, m = ctx->m;
  ctx->products(ctx->x.p, ctx->y.p, ctx->kxh.p, ctx->kty.p);
  auto cp = [&](double* d, const double* s, int64_t cnt) {
    if (cnt) CK(cudaMemcpyAsync(d, s, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
  };
  cp(ctx->x0.p, ctx->x.p, n); cp(ctx->xh.p, ctx->x.p, n);
  cp(ctx->ktyh.p, ctx->kty.p, n); cp(ctx->candx.p, ctx->x.p, n);
  cp(ctx->y0.p, ctx->y.p, m); cp(ctx->yh.p, ctx->y.p, m); cp(ctx->candy.p, ctx->y.p, m);
  cp(ctx->kxc.p, ctx->kxh.p, m); cp(ctx->kx0.p, ctx->kxh.p, m);   // carried K x, K x0 (x0 = x)
  CK(cudaMemsetAsync(ctx->xsum.p, 0, n * sizeof(double), st));
  CK(cudaMemsetAsync(ctx->ysum.p, 0, m * sizeof(double), st));
  KktCand c0{ctx->x.p, ctx->y.p, ctx->kxh.p, ctx->kty.p, ctx->res0.p, ctx->lam0.p};
  ctx->kkt_launch(c0, c0, 1, 0);
  ctx->read_ctl();
  Ctl& C = *ctx->hctl;
  C.e_anchor = std::max(C.kkt[0][0], std::max(C.kkt[0][1], C.kkt[0][2]));
  C.k = 0;
  C.Wsum = 0.0;
  C.beta = ctx->prm.beta_max;
  C.e_prev = -1.0;
  ctx->write_ctl();
}

// ============================================================================
extern "C" {

void pdcs_default_params(pdcs_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->tol = 1e-6;
  p->max_iters = 1000000;
  p->time_limit_s = 0.0;
  p->ruiz_iters = 10;
  p->pock_chambolle = 1;
  p->check_interval = 40;
  p->vanilla_pdhg = 0;
  p->eta0 = 0.0;
  p->omega0 = 0.0;
  p->beta_max = 1.0;
  p->refl_window = 40;
  p->restart_suff = 0.2;
  p->restart_nec = 0.8;
  p->restart_art = 0.36;
  p->ls_shrink = 0.5;
  p->ls_grow = 1.05;
  p->ls_max_rejects = 60;
  p->verbose = 0;
}

const char* pdcs_last_error(const pdcs_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

}  // extern "C"


// pdcs_create / pdcs_create_loopback: the communicator is NCCL (nccl_unique_id),
// an in-process loopback group (loop), or none.
static pdcs_status create_impl(pdcs_ctx** out, int64_t m_global, int64_t n, int64_t n1, int64_t row_begin,
                               int64_t row_end, const int64_t* row_ptr, const int32_t* col_idx,
                               const double* vals, const double* c, const double* h, const double* l,
                               const double* u, const pdcs_params* p, int device, void* cuda_stream,
                               int mem_kind, const void* nccl_unique_id, LoopbackGroup* loop, int rank,
                               int world) {
  if (!out) return PDCS_ERR_ARG;
  *out = nullptr;
  pdcs_ctx* ctx = new pdcs_ctx();
  const auto t_start = std::chrono::steady_clock::now();
  pdcs_status s = guard(nullptr, [&] {
    if (m_global < 0 || n < 0 || n1 < 0 || n1 > n) fail(PDCS_ERR_DIM, "bad sizes m/n/n1");
    if (row_begin < 0 || row_end < row_begin || row_end > m_global) fail(PDCS_ERR_DIM, "bad row range");
    if (mem_kind != PDCS_MEM_HOST && mem_kind != PDCS_MEM_DEVICE) fail(PDCS_ERR_ARG, "bad mem_kind");
    if (world < 1 || rank < 0 || rank >= world) fail(PDCS_ERR_ARG, "bad rank / world");
    if (world > 1 && !nccl_unique_id && !loop) fail(PDCS_ERR_ARG, "world > 1 needs an nccl_unique_id");
    if (loop && (world != loop->world || world > kLoopMaxRanks)) fail(PDCS_ERR_ARG, "world does not match the loopback group");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(PDCS_ERR_CUDA, "no CUDA device");
    if (device < 0 || device >= ndev) fail(PDCS_ERR_ARG, "bad device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(PDCS_ERR_CUDA, "libpdcs is built for sm_100a; device is sm_" +
                                              std::to_string(prop.major * 10 + prop.minor));
    ctx->device = device;
    ctx->sms = prop.multiProcessorCount;
    if (loop) {                                    // in-process loopback ranks (tests)
      auto lc = std::make_unique<LoopbackComm>();
      lc->g = loop;
      lc->rank = rank;
      lc->world = world;
      ctx->comm = std::move(lc);
      ctx->dist = true;
    } else if (nccl_unique_id) {                   // row-sharded context (also world == 1, for testing)
      auto nc = std::make_unique<NcclComm>();
      const std::string e = nc->init(nccl_unique_id, rank, world);
      if (!e.empty()) fail(PDCS_ERR_NCCL, e);
      ctx->comm = std::move(nc);
      ctx->dist = true;
    }
    ctx->st = (cudaStream_t)cuda_stream;
    ctx->serial_blocks = std::getenv("PDCS_SERIAL_BLOCKS") && std::atoi(std::getenv("PDCS_SERIAL_BLOCKS")) != 0;
    ctx->mem_kind = mem_kind;
    ctx->rank = rank;
    ctx->world = world;
    ctx->mg = m_global;
    ctx->m = row_end - row_begin;
    ctx->row_begin = row_begin;
    ctx->n = n;
    ctx->n1 = n1;
    if (p) ctx->prm = *p; else pdcs_default_params(&ctx->prm);
    if (ctx->prm.check_interval < 1 || ctx->prm.refl_window < 1) fail(PDCS_ERR_ARG, "bad cadence params");
    const int64_t m = ctx->m;
    // ---- host copies + validation
    ctx->hptr = to_host(row_ptr, m + 1, mem_kind);
    if (ctx->hptr[0] != 0) fail(PDCS_ERR_DIM, "row_ptr[0] must be 0");
    for (int64_t i = 0; i < m; ++i)
      if (ctx->hptr[i + 1] < ctx->hptr[i]) fail(PDCS_ERR_DIM, "row_ptr not monotone at row " + std::to_string(i));
    const int64_t nnz = ctx->hptr[m];
    if (nnz >= ((int64_t)1 << 31)) fail(PDCS_ERR_DIM, "local nnz must be < 2^31 (shard the rows)");
    // host view of the matrix: the caller's buffers (host) or copies (device)
    std::vector<int32_t> colcopy;
    std::vector<double> valcopy;
    const int32_t* hcolp = col_idx;
    const double* hvalp = vals;
    if (mem_kind == PDCS_MEM_DEVICE) {
      colcopy = to_host(col_idx, nnz, mem_kind);
      valcopy = to_host(vals, nnz, mem_kind);
      hcolp = colcopy.data();
      hvalp = valcopy.data();
    } else if (nnz && (!col_idx || !vals)) {
      fail(PDCS_ERR_ARG, "null input pointer");
    }
    SetupTrace tr;
    validate_csr(ctx->hptr.data(), hcolp, hvalp, m, n);
    tr.mark("validate", nullptr, false);
    // box-column order for gather locality (single context only: every rank of a
    // sharded run must store x identically, and the order depends on all rows)
    std::vector<int32_t> pcol;
    std::vector<double> pval;
    {
      const char* e = std::getenv("PDCS_COLPERM");
      const bool allow = (e ? std::atoi(e) != 0 : true) && !ctx->dist;
      const bool cp = allow && plan_colperm(ctx->hptr.data(), hcolp, m, n, n1, ctx->sms, ctx->u2i, ctx->i2u);
      tr.mark("  colperm plan", nullptr, false);
      if (cp) {
        permute_csr(ctx->hptr.data(), hcolp, hvalp, m, ctx->u2i, pcol, pval);
        tr.mark("  colperm: permute CSR", nullptr, false);
        hcolp = pcol.data();
        hvalp = pval.data();
        ctx->colperm = true;
      }
    }
    // tiled format of K~ (structure only) on host threads, overlapping the uploads
    // and the device transpose below; joined before this call returns
    // (PDCS_TILE_DEVBUILD=0: on host threads, overlapping the uploads and the
    // device transpose below; else on the device once K is there)
    const bool devb = tiled_devbuild_env();
    if (!devb)
      ctx->thK = std::thread([ctx, hcolp, m, n] {
        build_tiled(ctx->hptr.data(), hcolp, m, n, 1, ctx->hK, true, true);
      });
    struct Joiner {
      std::thread& t;
      ~Joiner() { if (t.joinable()) t.join(); }
    } join_k{ctx->thK};
    std::vector<double> hc = to_host(c, n, mem_kind), hh = to_host(h, m, mem_kind);
    ctx->hl = to_host(l, n1, mem_kind);
    ctx->hu = to_host(u, n1, mem_kind);
    tr.mark("  c, h, l, u to host", nullptr, false);
    if (ctx->colperm) {                           // c, l, u in the stored column order
      auto perm = [&](std::vector<double>& v, int64_t cnt) {   // random gathers: on host threads
        std::vector<double> o(cnt);
        parallel_chunks(cnt, [&](int64_t a, int64_t b) {
          for (int64_t k = a; k < b; ++k) o[k] = v[ctx->i2u[k]];
        });
        v.swap(o);
      };
      perm(hc, n);
      perm(ctx->hl, n1);
      perm(ctx->hu, n1);
      tr.mark("  c, l, u permuted", nullptr, false);
    }
    for (double v : hc) if (!std::isfinite(v)) fail(PDCS_ERR_NONFINITE, "non-finite c");
    for (double v : hh) if (!std::isfinite(v)) fail(PDCS_ERR_NONFINITE, "non-finite h");
    for (int64_t j = 0; j < n1; ++j) {
      if (std::isnan(ctx->hl[j]) || std::isnan(ctx->hu[j]) || ctx->hl[j] > ctx->hu[j] ||
          ctx->hl[j] == INFINITY || ctx->hu[j] == -INFINITY)
        fail(PDCS_ERR_BOUNDS, "bound inversion at index " + std::to_string(j));
    }
    double hn = 0.0, cn = 0.0;
    for (double v : hh) hn = std::max(hn, std::fabs(v));
    for (double v : hc) cn = std::max(cn, std::fabs(v));
    ctx->hnorm = hn;
    ctx->cnorm = cn;
    cudaStream_t st = ctx->st;
    tr.mark("colperm + host data", nullptr, false);
    // ---- device CSR(K)
    std::vector<int32_t> p32(m + 1);
    for (int64_t i = 0; i <= m; ++i) p32[i] = (int32_t)ctx->hptr[i];
    upload(ctx->Kptr, p32, st);
    ctx->Kcol.alloc(nnz);
    ctx->Kval.alloc(nnz);
    if (nnz) {
      CK(cudaMemcpyAsync(ctx->Kcol.p, ctx->colperm ? hcolp : col_idx, nnz * sizeof(int32_t), cudaMemcpyDefault, st));
      CK(cudaMemcpyAsync(ctx->Kval.p, ctx->colperm ? hvalp : vals, nnz * sizeof(double), cudaMemcpyDefault, st));
    }
    if (ctx->colperm) {
      upload(ctx->u2i_d, ctx->u2i, st);
      upload(ctx->i2u_d, ctx->i2u, st);
      ctx->permbuf.alloc(n);
      CK(cudaStreamSynchronize(st));             // pcol / pval are pageable and die with this scope
    }
    upload(ctx->c0, hc, st);
    upload(ctx->h0, hh, st);
    upload(ctx->l0, ctx->hl, st);
    upload(ctx->u0, ctx->hu, st);
    ctx->K.m = m; ctx->K.n = n; ctx->K.nnz = nnz;
    ctx->K.ptr = ctx->Kptr.p; ctx->K.col = ctx->Kcol.p; ctx->K.val = ctx->Kval.p;
    tr.mark("upload K", st);
    if (devb) {
      build_tiled_device(ctx->Kptr.p, ctx->Kcol.p, ctx->hptr.data(), m, n, 1, kTiledMinFrac, ctx->hK, ctx->tK.dv, st,
                         ctx->sms);
      tr.mark("tiled K (device build)", st);
    }
    // ---- device CSR(K^T) by a stable radix sort of the entries on column id
    ctx->KTptr.alloc(n + 1);
    ctx->KTcol.alloc(nnz);
    ctx->KTval.alloc(nnz);
    {
      DBuf<int32_t> keys_in, keys_out, perm_in, perm_out, rid, cnt;
      keys_in.alloc(nnz); keys_out.alloc(nnz); perm_in.alloc(nnz); perm_out.alloc(nnz); rid.alloc(nnz);
      cnt.alloc(n + 1);
      const int G = grid_for(nnz, ctx->sms, 32);
      if (nnz) {
        CK(cudaMemcpyAsync(keys_in.p, ctx->Kcol.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        k_iota<<<G, kThreads, 0, st>>>(nnz, perm_in.p);
        k_row_ids<<<grid_for(m, ctx->sms, 32), kThreads, 0, st>>>(m, ctx->Kptr.p, rid.p);
        int bits = 1;
        while (((int64_t)1 << bits) < n) ++bits;
        size_t tmpb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmpb, keys_in.p, keys_out.p, perm_in.p, perm_out.p,
                                           (int)nnz, 0, bits, st));
        DBuf<char> tmp;
        tmp.alloc(tmpb);
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmpb, keys_in.p, keys_out.p, perm_in.p, perm_out.p,
                                           (int)nnz, 0, bits, st));
        k_gather_t<<<G, kThreads, 0, st>>>(nnz, perm_out.p, rid.p, ctx->Kval.p, ctx->KTcol.p, ctx->KTval.p);
      }
      CK(cudaMemsetAsync(cnt.p, 0, (n + 1) * sizeof(int32_t), st));
      if (nnz) k_count_cols<<<G, kThreads, 0, st>>>(nnz, ctx->Kcol.p, cnt.p);
      size_t tmpb = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmpb, cnt.p, ctx->KTptr.p, (int)(n + 1), st));
      DBuf<char> tmp;
      tmp.alloc(tmpb);
      CK(cub::DeviceScan::ExclusiveSum(tmp.p, tmpb, cnt.p, ctx->KTptr.p, (int)(n + 1), st));
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(st));
    }
    ctx->KT.m = n; ctx->KT.n = m; ctx->KT.nnz = nnz;
    ctx->KT.ptr = ctx->KTptr.p; ctx->KT.col = ctx->KTcol.p; ctx->KT.val = ctx->KTval.p;
    tr.mark("transpose", st);
    // ---- SpMV plans (row-length binning)
    std::vector<int32_t> tptr32(n + 1);
    CK(cudaMemcpy(tptr32.data(), ctx->KTptr.p, (n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    std::vector<int64_t> tptr(tptr32.begin(), tptr32.end());
    std::vector<int32_t> rowstore;
    std::vector<size_t> offs;
    ctx->build_plan(ctx->K, ctx->hptr, rowstore, offs);
    ctx->build_plan(ctx->KT, tptr, rowstore, offs);
    tr.mark("  SpMV plans", nullptr, false);
    // sharded: K~^T in row chunks whose all-reduces overlap the next chunk's sums
    if (ctx->dist) {
      const char* e = std::getenv("PDCS_AR_CHUNKS");
      const int C = e ? std::max(1, std::atoi(e)) : (n * 8 >= (8 << 20) ? 4 : 1);
      if (C > 1 && n >= C) {
        for (int c = 0; c <= C; ++c) ctx->ktc_row.push_back(n * c / C);
        for (int c = 0; c < C; ++c) {
          DevCsr tmpA;
          ctx->build_plan(tmpA, tptr, rowstore, offs, ctx->ktc_row[c], ctx->ktc_row[c + 1]);
          ctx->ktc_plan.push_back(tmpA.plan);
        }
        CK(cudaStreamCreateWithFlags(&ctx->comm_st, cudaStreamNonBlocking));
        ctx->ev_ar.resize(C);
        for (auto& ev : ctx->ev_ar) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_ar_done, cudaEventDisableTiming));
      }
    }
    // tiled format of K~^T from the transposed structure, in the background
    // (joined in pdcs_set_cones, which uses it after the Ruiz scaling)
    if (devb) {
      build_tiled_device(ctx->KTptr.p, ctx->KTcol.p, tptr.data(), n, m, 1, kTiledMinFrac, ctx->hKT, ctx->tKT.dv, st,
                         ctx->sms);
      tr.mark("  tiled K^T (device build)", st);
    } else {
      ctx->hKTptr = std::move(tptr);
      ctx->hKTcol.resize(nnz);
      if (nnz) CK(cudaMemcpy(ctx->hKTcol.data(), ctx->KTcol.p, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
      tr.mark("  K^T ids to host", nullptr, false);
      ctx->thKT = std::thread([ctx, m, n] {
        build_tiled(ctx->hKTptr.data(), ctx->hKTcol.data(), n, m, 1, ctx->hKT, true, true);
      });
    }
    upload(ctx->planrows, rowstore, st);
    ctx->patch_plan(ctx->K);
    ctx->patch_plan(ctx->KT);
    for (SpmvPlan& pl : ctx->ktc_plan) {
      DevCsr tmpA;
      tmpA.plan = pl;
      ctx->patch_plan(tmpA);
      pl = tmpA.plan;
    }
    // ---- L1 / shared-memory split for the gathering kernels (PDCS_CARVEOUT, % smem)
    if (const char* env = std::getenv("PDCS_CARVEOUT")) {
      const int pc = std::atoi(env);
      CK(cudaFuncSetAttribute(spmv_kernel<EpiDualTrial>, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
      CK(cudaFuncSetAttribute(spmv_kernel<EpiHalpernX>, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
      CK(cudaFuncSetAttribute(spmv_kernel<EpiStore>, cudaFuncAttributePreferredSharedMemoryCarveout, pc));
    }
    // ---- control block
    CK(cudaMalloc(&ctx->ctl, sizeof(Ctl)));
    CK(cudaMallocHost(&ctx->hctl, sizeof(Ctl)));
    std::memset(ctx->hctl, 0, sizeof(Ctl));
    CK(cudaStreamSynchronize(st));
    tr.mark("plans + K^T to host", st);
    if (ctx->thK.joinable()) ctx->thK.join();
    tr.mark("join tiled K build", nullptr, false);
    ctx->tK.build_ms = ctx->hK.build_ms;
    ctx->t_create_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  });
  if (s != PDCS_OK) {
    delete ctx;
    return s;
  }
  *out = ctx;
  return PDCS_OK;
}

extern "C" {

pdcs_status pdcs_create(pdcs_ctx** out, int64_t m_global, int64_t n, int64_t n1, int64_t row_begin,
                        int64_t row_end, const int64_t* row_ptr, const int32_t* col_idx,
                        const double* vals, const double* c, const double* h, const double* l,
                        const double* u, const pdcs_params* p, int device, void* cuda_stream,
                        int mem_kind, const void* nccl_unique_id, int rank, int world) {
  return create_impl(out, m_global, n, n1, row_begin, row_end, row_ptr, col_idx, vals, c, h, l, u, p, device,
                     cuda_stream, mem_kind, nccl_unique_id, nullptr, rank, world);
}

pdcs_status pdcs_create_loopback(pdcs_ctx** out, int64_t m_global, int64_t n, int64_t n1, int64_t row_begin,
                                 int64_t row_end, const int64_t* row_ptr, const int32_t* col_idx,
                                 const double* vals, const double* c, const double* h, const double* l,
                                 const double* u, const pdcs_params* p, int device, void* cuda_stream,
                                 int mem_kind, pdcs_loopback* group, int rank) {
  if (!group) { g_create_error = "null loopback group"; return PDCS_ERR_ARG; }
  LoopbackGroup* g = reinterpret_cast<LoopbackGroup*>(group);
  return create_impl(out, m_global, n, n1, row_begin, row_end, row_ptr, col_idx, vals, c, h, l, u, p, device,
                     cuda_stream, mem_kind, nullptr, g, rank, g->world);
}

pdcs_status pdcs_set_allocator(pdcs_alloc_fn alloc, pdcs_free_fn free_fn, void* user) {
  if ((alloc == nullptr) != (free_fn == nullptr)) {
    g_create_error = "pdcs_set_allocator needs both functions or neither";
    return PDCS_ERR_ARG;
  }
  g_alloc_user.store(user);
  g_free.store(free_fn);
  g_alloc.store(alloc);
  return PDCS_OK;
}

int64_t pdcs_trim_memory(void) {
  int64_t released = 0;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (int d = 0; d < 64; ++d) {
    DevPool& P = g_pool[d];
    if (!P.pool) continue;
    uint64_t before = 0, after = 0;
    cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrReservedMemCurrent, &before);
    if (cudaMemPoolTrimTo(P.pool, 0) != cudaSuccess) return -1;
    cudaMemPoolGetAttribute(P.pool, cudaMemPoolAttrReservedMemCurrent, &after);
    released += (int64_t)(before - after);
  }
  return released;
}

pdcs_status pdcs_loopback_create(pdcs_loopback** out, int world) {
  if (!out || world < 1 || world > kLoopMaxRanks) {
    g_create_error = "loopback world must be 1..16";
    return PDCS_ERR_ARG;
  }
  *out = reinterpret_cast<pdcs_loopback*>(new LoopbackGroup(world));
  return PDCS_OK;
}

void pdcs_loopback_destroy(pdcs_loopback* group) { delete reinterpret_cast<LoopbackGroup*>(group); }

pdcs_status pdcs_set_cones(pdcs_ctx* ctx, const int32_t* pk, const int64_t* pdim, int64_t npc,
                           const int32_t* rkind, const int64_t* rdim, int64_t nrc) {
  if (!ctx) return PDCS_ERR_ARG;
  const auto t_start = std::chrono::steady_clock::now();
  return guard(ctx, [&] {
    if (ctx->cones_set) fail(PDCS_ERR_STATE, "cones already set");
    if (npc < 0 || nrc < 0 || (npc && (!pk || !pdim)) || (nrc && (!rkind || !rdim)))
      fail(PDCS_ERR_ARG, "bad cone arrays");
    const int64_t n = ctx->n, n1 = ctx->n1, m = ctx->m, mg = ctx->mg;
    cudaStream_t st = ctx->st;
    auto dim_ok = [](int32_t k, int64_t d) {
      switch (k) {
        case C_ZERO: case C_NONNEG: return d >= 1;
        case C_SOC: return d >= 2;
        case C_RSOC: return d >= 3;
        case C_EXP: case C_DEXP: return d == 3;
        default: return false;
      }
    };
    // element kinds
    std::vector<uint8_t> ek(n), rk(m);
    for (int64_t j = 0; j < n1; ++j) {
      const bool fl = std::isfinite(ctx->hl[j]), fu = std::isfinite(ctx->hu[j]);
      ek[j] = !fl && !fu ? EK_FREE : (fl && !fu) ? (ctx->hl[j] == 0.0 ? EK_LO0 : EK_LO) : (!fl ? EK_UP : EK_BOTH);
    }
    std::vector<Block> pb, rb;
    std::vector<int64_t> prs, rrs;
    int64_t off = n1;
    for (int64_t b = 0; b < npc; ++b) {
      if (!dim_ok(pk[b], pdim[b])) fail(PDCS_ERR_CONE, "bad primal cone " + std::to_string(b));
      if (off + pdim[b] > n) fail(PDCS_ERR_CONE, "primal cone dims exceed n2");
      const uint8_t e = pk[b] == C_ZERO ? EK_ZERO : pk[b] == C_NONNEG ? EK_NONNEG : EK_BLOCK;
      for (int64_t j = off; j < off + pdim[b]; ++j) ek[j] = e;
      if (e == EK_BLOCK) pb.push_back(Block{off, pk[b], (int32_t)pdim[b]});
      if (pk[b] == C_RSOC) prs.push_back(off);
      off += pdim[b];
    }
    if (off != n) fail(PDCS_ERR_CONE, "primal cone dims do not sum to n2");
    off = 0;
    for (int64_t b = 0; b < nrc; ++b) {
      if (!dim_ok(rkind[b], rdim[b])) fail(PDCS_ERR_CONE, "bad row cone " + std::to_string(b));
      const int64_t lo = off - ctx->row_begin, hi = lo + rdim[b];
      if (hi > 0 && lo < m) {
        const uint8_t e = rkind[b] == C_ZERO ? EK_FREE : rkind[b] == C_NONNEG ? EK_NONNEG : EK_BLOCK;
        // Zero / NonNeg rows are elementwise and may be cut by a shard; a cone block may not
        if (e == EK_BLOCK && (lo < 0 || hi > m))
          fail(PDCS_ERR_SHARD, "row cone " + std::to_string(b) + " straddles the rank's rows");
        for (int64_t i = std::max<int64_t>(lo, 0); i < std::min<int64_t>(hi, m); ++i) rk[i] = e;
        if (e == EK_BLOCK) rb.push_back(Block{lo, rkind[b], (int32_t)rdim[b]});
        if (rkind[b] == C_RSOC) rrs.push_back(lo);
      }
      off += rdim[b];
    }
    if (off != mg) fail(PDCS_ERR_CONE, "row cone dims do not sum to m");
    // Size classes (class_policy): thread (exp, soc <= 32), warp, CTA, cluster
    // of kClusterCtas CTAs (<= 131072), grid.  Within a class blocks are
    // ordered by (kind, dim) so that the lanes / warps of a launch run the same
    // code path with similar trip counts.
    auto classify = [&](std::vector<Block>& v, pdcs_ctx::BClass* cl) {
      const ClassPolicy pol = class_policy(v, ctx->sms);
      auto cls = [&](const Block& b) { return pol.of(b); };
      std::stable_sort(v.begin(), v.end(), [&](const Block& a, const Block& b) {
        const int ca = cls(a), cb = cls(b);
        if (ca != cb) return ca < cb;
        if (a.kind != b.kind) return a.kind < b.kind;
        return a.dim < b.dim;
      });
      for (int c = 0; c < kNClass; ++c) cl[c] = pdcs_ctx::BClass{};
      for (size_t i = 0; i < v.size(); ++i) {
        const int c = cls(v[i]);
        if (cl[c].count == 0) cl[c].begin = (int64_t)i;
        cl[c].count++;
      }
      for (int c = 0; c < kNClass; ++c) {
        const int64_t cnt = cl[c].count;
        if (!cnt) continue;
        if (c == 0) {
          // PDCS_THREAD_CPT: cones per thread of the thread class (default 1);
          // more per thread averages the exp root finder's iteration counts
          // within a lane (the warp waits for its slowest lane) at lower occupancy
          const int64_t cpt = std::getenv("PDCS_THREAD_CPT") ? std::max(1, std::atoi(std::getenv("PDCS_THREAD_CPT"))) : 1;
          cl[c].grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + cpt * kThreadsSmall - 1) / (cpt * kThreadsSmall),
                                                                  (int64_t)ctx->sms * 32));
        }
        else if (c == 1) cl[c].grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 7) / 8, (int64_t)ctx->sms * 8));
        else if (c == 2) cl[c].grid = (int)std::min<int64_t>(cnt, (int64_t)ctx->sms * 4);
        else if (c == 3) cl[c].grid = kClusterCtas * (int)std::min<int64_t>(cnt, (int64_t)ctx->sms * 2 / kClusterCtas);
        else {
          int nb = 0;
          CK(grid_team_occupancy(&nb));
          // PDCS_GRID_CTAS (per SM) lowers the grid team's size: fewer CTAs
          // to synchronise per reduction, more elements per thread
          if (const char* e = std::getenv("PDCS_GRID_CTAS")) nb = std::min(nb, std::max(1, std::atoi(e)));
          cl[c].grid = std::max(1, std::min(nb, 4)) * ctx->sms;
        }
      }
    };
    classify(pb, ctx->pcls);
    classify(rb, ctx->rcls);
    upload(ctx->pblocks, pb, st);
    upload(ctx->rblocks, rb, st);
    for (auto* w : {&ctx->warm_p, &ctx->warm_r}) {
      const size_t nb = std::max<size_t>(w == &ctx->warm_p ? pb.size() : rb.size(), 1);
      w->alloc(nb);
      CK(cudaMemsetAsync(w->p, 0, nb * sizeof(double), st));
    }
    upload(ctx->ek, ek, st);
    upload(ctx->rk, rk, st);
    std::vector<int64_t> prs64(prs.begin(), prs.end()), rrs64(rrs.begin(), rrs.end());
    upload(ctx->rsoc_offs_p, prs64, st);
    upload(ctx->rsoc_offs_r, rrs64, st);
    // ---- partial-sum slots
    ctx->g_pe = grid_for(n, ctx->sms);
    ctx->g_m = grid_for(m, ctx->sms);
    ctx->g_kr = grid_for(m, ctx->sms, 4);
    ctx->g_kc = grid_for(n, ctx->sms, 4);
    int64_t s = 0;
    ctx->slot_pe = s; s += ctx->g_pe;
    for (int c = 0; c < kNClass; ++c) if (ctx->pcls[c].count) { ctx->pcls[c].slot = s; s += ctx->pcls[c].grid; }
    ctx->slot_spmv = s;   // also the tiled combine and panel finish grids, and the fused combine's chunks
    s += std::max<int64_t>({ctx->K.plan.total_cta, (int64_t)ctx->sms * 8, ctx->tK.on ? pdcs_ctx::fused_slots(ctx->tK) : 0});
    for (int c = 0; c < kNClass; ++c) if (ctx->rcls[c].count) { ctx->rcls[c].slot = s; s += ctx->rcls[c].grid; }
    ctx->nslot_trial = s;
    int64_t ks = 0;
    ctx->kslot_rows = ks; ks += ctx->g_kr;
    ctx->kslot_cols = ks; ks += ctx->g_kc;
    for (int cand = 0; cand < 2; ++cand)
      for (int side = 0; side < 2; ++side) {
        pdcs_ctx::BClass* cl = side ? ctx->pcls : ctx->rcls;
        for (int c = 0; c < kNClass; ++c)
          if (cl[c].count) {
            cl[c].kslot[cand] = ks;
            ks += cl[c].grid;
          }
      }
    ctx->nslot_kkt = ks;
    ctx->tpart.alloc(s * kAcc);
    ctx->kpart.alloc(ks * kKAcc);
    CK(cudaMemsetAsync(ctx->tpart.p, 0, s * kAcc * sizeof(double), st));
    CK(cudaMemsetAsync(ctx->kpart.p, 0, ks * kKAcc * sizeof(double), st));
    ctx->gbuf.alloc(4 * (size_t)ctx->sms * 8);
    // ---- vectors
    ctx->y.alloc(m + 2);   // +pad: TMA tile copies round up to 16 B
    for (auto* b : {&ctx->r, &ctx->onesm, &ctx->ht, &ctx->yh, &ctx->y0, &ctx->ysum,
                    &ctx->kxh, &ctx->kxd, &ctx->ya, &ctx->kxa, &ctx->by, &ctx->candy, &ctx->res0,
                    &ctx->res1, &ctx->tmpm})
      b->alloc(std::max<int64_t>(m, 1));
    ctx->xh.alloc(n + 2);  // +pad: gathered by the K sweep (TMA tile copies round up to 16 B)
    for (auto* b : {&ctx->q, &ctx->onesn, &ctx->ct, &ctx->x, &ctx->x0, &ctx->xsum, &ctx->kty,
                    &ctx->ktyh, &ctx->xa, &ctx->ktya, &ctx->bx, &ctx->candx, &ctx->lam0,
                    &ctx->lam1, &ctx->tmpn})
      b->alloc(std::max<int64_t>(n, 1));
    ctx->kxc.alloc(std::max<int64_t>(m, 1) + 1);
    ctx->kx0.alloc(std::max<int64_t>(m, 1) + 1);
    ctx->ktyp.alloc(std::max<int64_t>(n, 1));
    ctx->lt.alloc(std::max<int64_t>(n1, 1));
    ctx->ut.alloc(std::max<int64_t>(n1, 1));
    ctx->scal.alloc(8);
    // ||h||_inf of Eq. 9's err_p denominator over ALL rows (every rank must score
    // candidates, restarts and termination identically)
    ctx->hnorm = ctx->allreduce_host(ctx->hnorm, RedOp::Max);
    const int Gm = grid_for(m, ctx->sms), Gn = grid_for(n, ctx->sms);
    k_fill<<<Gm, kThreads, 0, st>>>(m, 1.0, ctx->r.p);
    k_fill<<<Gm, kThreads, 0, st>>>(m, 1.0, ctx->onesm.p);
    k_fill<<<Gn, kThreads, 0, st>>>(n, 1.0, ctx->q.p);
    k_fill<<<Gn, kThreads, 0, st>>>(n, 1.0, ctx->onesn.p);
    for (auto* b : {&ctx->y, &ctx->yh, &ctx->y0, &ctx->ysum, &ctx->kxh, &ctx->kxd, &ctx->ya,
                    &ctx->kxa, &ctx->by, &ctx->candy, &ctx->res0, &ctx->res1})
      CK(cudaMemsetAsync(b->p, 0, b->n * sizeof(double), st));
    for (auto* b : {&ctx->x, &ctx->xh, &ctx->x0, &ctx->xsum, &ctx->kty, &ctx->ktyh, &ctx->xa,
                    &ctx->ktya, &ctx->bx, &ctx->candx, &ctx->lam0, &ctx->lam1})
      CK(cudaMemsetAsync(b->p, 0, b->n * sizeof(double), st));
    const bool van = ctx->prm.vanilla_pdhg != 0;
    SetupTrace tr;
    tr.mark("set_cones: cones + slots", st);
    // ---- Ruiz + Pock-Chambolle (readings A2, A3, A21)
    const int Grm = grid_for(m * 32, ctx->sms, 16), Grn = grid_for(n * 32, ctx->sms, 16);
    if (!van) {
      for (int it = 0; it < ctx->prm.ruiz_iters + (ctx->prm.pock_chambolle ? 1 : 0); ++it) {
        const int mode = it < ctx->prm.ruiz_iters ? 0 : 1;
        k_row_norms<<<Grm, kThreads, 0, st>>>(m, ctx->K.ptr, ctx->K.col, ctx->K.val, ctx->r.p, ctx->q.p, mode,
                                             ctx->tmpm.p);
        k_row_norms<<<Grn, kThreads, 0, st>>>(n, ctx->KT.ptr, ctx->KT.col, ctx->KT.val, ctx->q.p, ctx->r.p,
                                             mode, ctx->tmpn.p);
        ctx->allreduce(ctx->tmpn.p, n, mode ? RedOp::Sum : RedOp::Max);   // column norms over all rows
        k_apply_root<<<Gm, kThreads, 0, st>>>(m, ctx->tmpm.p, ctx->r.p);
        k_apply_root<<<Gn, kThreads, 0, st>>>(n, ctx->tmpn.p, ctx->q.p);
      }
      if (!prs64.empty()) k_rsoc_geomean<<<1, kThreads, 0, st>>>(ctx->rsoc_offs_p.p, (int64_t)prs64.size(), ctx->q.p);
      if (!rrs64.empty()) k_rsoc_geomean<<<1, kThreads, 0, st>>>(ctx->rsoc_offs_r.p, (int64_t)rrs64.size(), ctx->r.p);
      k_scale_vals<<<Grm, kThreads, 0, st>>>(m, ctx->K.ptr, ctx->K.col, ctx->K.val, ctx->r.p, ctx->q.p);
      k_scale_vals<<<Grn, kThreads, 0, st>>>(n, ctx->KT.ptr, ctx->KT.col, ctx->KT.val, ctx->q.p, ctx->r.p);
    }
    CK(cudaGetLastError());
    // column-tiled copies of K~ and K~^T for the hot SpMVs (tiled.cuh)
    {
      tr.mark("ruiz", st);
      ctx->make_tiled(ctx->tK, ctx->hK, m, n, 1, ctx->K.val);
      tr.mark("tiled K (device part)", st);
      if (ctx->thKT.joinable()) ctx->thKT.join();
      tr.mark("join tiled K^T build", nullptr, false);
      ctx->tKT.build_ms = ctx->hKT.build_ms;
      ctx->make_tiled(ctx->tKT, ctx->hKT, n, m, 1, ctx->KT.val);
      ctx->hKTptr = std::vector<int64_t>();
      ctx->hKTcol = std::vector<int32_t>();
    }
    // L2 column panels where the gathered vector exceeds L2 (panels.cuh)
    tr.mark("tiled K^T (device part)", st);
    ctx->build_panels(ctx->pK, ctx->K, ctx->tK.on, 1);
    ctx->build_panels(ctx->pKT, ctx->KT, ctx->tKT.on, 1);
    if (!ctx->tK.on && !ctx->pK.on) ctx->tune_csr_u(ctx->K, n);
    if (!ctx->tKT.on && !ctx->pKT.on) ctx->tune_csr_u(ctx->KT, m);
    tr.mark("panels", st);
    // scaled data (reading A2): c~ = c/q, h~ = h/r, l~ = q l, u~ = q u
    k_ewise<<<Gn, kThreads, 0, st>>>(n, ctx->c0.p, ctx->q.p, 0, ctx->ct.p);
    k_ewise<<<Gm, kThreads, 0, st>>>(m, ctx->h0.p, ctx->r.p, 0, ctx->ht.p);
    if (n1) k_bounds<<<grid_for(n1, ctx->sms), kThreads, 0, st>>>(n1, ctx->q.p, ctx->l0.p, ctx->u0.p, ctx->lt.p, ctx->ut.p);
    // ---- control block (reading A4-A6)
    Ctl& C = *ctx->hctl;
    std::memset(&C, 0, sizeof(Ctl));
    const pdcs_params& P = ctx->prm;
    C.vanilla = van ? 1 : 0;
    C.ls_shrink = P.ls_shrink; C.ls_grow = P.ls_grow; C.beta_max = P.beta_max;
    C.suff = P.restart_suff; C.nec = P.restart_nec; C.art = P.restart_art;
    C.ls_max_rejects = P.ls_max_rejects; C.refl_window = P.refl_window; C.check_interval = P.check_interval;
    C.tol = P.tol;
    C.beta = P.beta_max;
    C.e_prev = -1.0;
    C.best_e = INFINITY;
    C.status = ST_RUNNING;
    double eta = 1.0, omega = 1.0;
    if (van) {
      if (P.eta0 > 0.0) eta = P.eta0;
      else {
        // tau = sigma = 0.9/||G||_2, power iteration on G^T G
        const double v0 = 1.0 / std::sqrt((double)std::max<int64_t>(n, 1));
        k_fill<<<Gn, kThreads, 0, st>>>(n, v0, ctx->tmpn.p);
        double lam = 0.0;
        for (int it = 0; it < 20; ++it) {
          ctx->spmv_store(ctx->K, ctx->tmpn.p, ctx->tmpm.p);
          ctx->spmv_store(ctx->KT, ctx->tmpm.p, ctx->lam0.p);
          ctx->allreduce(ctx->lam0.p, n, RedOp::Sum);
          k_reduce<<<1, kThreads, 0, st>>>(n, ctx->lam0.p, 1, ctx->scal.p);
          double s2 = 0.0;
          CK(cudaMemcpyAsync(&s2, ctx->scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          const double nw = std::sqrt(s2);
          if (nw == 0.0) { lam = 0.0; break; }
          const double prev = lam;
          lam = nw;
          // v = w / ||w||
          CK(cudaMemcpyAsync(ctx->tmpn.p, ctx->lam0.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
          k_fill<<<Gn, kThreads, 0, st>>>(n, nw, ctx->lam1.p);
          k_ewise<<<Gn, kThreads, 0, st>>>(n, ctx->tmpn.p, ctx->lam1.p, 0, ctx->tmpn.p);
          if (it > 0 && std::fabs(lam - prev) < 1e-4 * lam) break;
        }
        const double nrm = std::sqrt(lam);
        eta = nrm > 0.0 ? 0.9 / nrm : 1.0;
      }
      omega = 1.0;
    } else {
      // eta0 = 1/||K~||_inf (A5); omega0 = ||c~||/||h~|| clipped (A6)
      k_row_norms<<<Grm, kThreads, 0, st>>>(m, ctx->K.ptr, ctx->K.col, ctx->K.val, ctx->onesm.p, ctx->onesn.p, 1,
                                           ctx->tmpm.p);
      k_reduce<<<1, kThreads, 0, st>>>(m, ctx->tmpm.p, 2, ctx->scal.p);
      k_reduce<<<1, kThreads, 0, st>>>(n, ctx->ct.p, 0, ctx->scal.p + 1);
      k_reduce<<<1, kThreads, 0, st>>>(m, ctx->ht.p, 0, ctx->scal.p + 2);
      ctx->allreduce(ctx->scal.p, 1, RedOp::Max);        // ||K~||_inf over the row shards
      ctx->allreduce(ctx->scal.p + 2, 1, RedOp::Max);    // ||h~||_inf
      double hs[3];
      CK(cudaMemcpyAsync(hs, ctx->scal.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      eta = P.eta0 > 0.0 ? P.eta0 : (hs[0] > 0.0 ? 1.0 / hs[0] : 1.0);
      if (P.omega0 > 0.0) omega = P.omega0;
      else if (hs[1] > 0.0 && hs[2] > 0.0) omega = std::min(std::max(hs[1] / hs[2], 1e-4), 1e4);
      else omega = 1.0;
    }
    C.eta = eta; C.eta_init = eta; C.omega = omega;
    C.tau = eta / omega; C.sigma = eta * omega;
    ctx->write_ctl();
    ctx->cones_set = true;
    // initial point z00 = (P_X(0), 0) (reading A4): average of a zero sum with W = 1
    C.Wsum = 1.0;
    ctx->write_ctl();
    k_avg_elem<<<Gn, kThreads, 0, st>>>(n, ctx->ek.p, ctx->xsum.p, ctx->lt.p, ctx->ut.p, ctx->x.p, ctx->ctl);
    C.Wsum = 0.0;
    ctx->write_ctl();
    CK(cudaGetLastError());
    // anchor / products / e_anchor
    reset_from_current(ctx);
    CK(cudaStreamSynchronize(st));
    tr.mark("eta0/omega0 + anchor KKT", st);
    ctx->t_cones_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  });
}

pdcs_status pdcs_set_iterate(pdcs_ctx* ctx, const double* x, const double* y) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    cudaStream_t st = ctx->st;
    const int64_t n = ctx->n, m = ctx->m;
    const cudaMemcpyKind kind = ctx->mem_kind == PDCS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (x) {
      ctx->from_caller(ctx->tmpn.p, x, kind);
      k_ewise<<<grid_for(n, ctx->sms), kThreads, 0, st>>>(n, ctx->tmpn.p, ctx->q.p, 1, ctx->x.p);
    }
    if (y) {
      CK(cudaMemcpyAsync(ctx->tmpm.p, y, m * sizeof(double), kind, st));
      k_ewise<<<grid_for(m, ctx->sms), kThreads, 0, st>>>(m, ctx->tmpm.p, ctx->r.p, 1, ctx->y.p);
    }
    CK(cudaGetLastError());
    reset_from_current(ctx);
  });
}

static void finish_result(pdcs_ctx* ctx, pdcs_result_t* out, double secs) {
  if (!out) return;
  const Ctl& C = *ctx->hctl;
  std::memset(out, 0, sizeof(*out));
  out->status = C.status == ST_RUNNING ? PDCS_RUNNING : C.status;
  out->kkt.err_p = C.best_kkt[0]; out->kkt.err_d = C.best_kkt[1]; out->kkt.err_gap = C.best_kkt[2];
  out->kkt.pobj = C.best_kkt[3]; out->kkt.dobj = C.best_kkt[4];
  out->iters = C.total; out->trials = C.trials; out->restarts = C.restarts;
  // matrix passes: one K sweep per trial (K x^ and K x together), one K^T sweep
  // per accepted step, and per Eq. 9 check K^T y^ plus (PDCS) K xbar, K^T ybar
  out->spmv_K = C.trials + (C.vanilla ? 0 : C.checks);
  out->spmv_KT = C.total + C.checks * (C.vanilla ? 1 : 2);
  out->eta = C.eta; out->omega = C.omega; out->beta = C.beta;
  out->solve_seconds = secs;
}

// Graph-driven loop of Alg. 1: one graph launch per accepted iteration; the
// host synchronises only every check_interval launches (to test termination)
// or at the end.
static bool run_steps_graph(pdcs_ctx* ctx, int64_t n_inner, bool stop_at_tol, double time_limit) {
  if (ctx->timing || std::getenv("PDCS_NO_GRAPH")) return false;
  // sharded: the collectives are recorded into the graph when the communicator
  // allows it (NCCL; PDCS_DIST_GRAPH=0 keeps the host loop), else the host loop
  if (ctx->dist && (!ctx->comm->capturable() ||
                    (std::getenv("PDCS_DIST_GRAPH") && !std::atoi(std::getenv("PDCS_DIST_GRAPH")))))
    return false;
  ctx->build_graph();
  if (!ctx->gexec) return false;
  auto t0 = std::chrono::steady_clock::now();
  ctx->read_ctl();
  ctx->hctl->stop_at_tol = stop_at_tol ? 1 : 0;
  ctx->write_ctl();
  const Ctl before = *ctx->hctl;
  const int64_t batch = stop_at_tol ? ctx->prm.check_interval : n_inner;
  int64_t done = 0;
  while (done < n_inner) {
    const int64_t b = std::min(batch, n_inner - done);
    for (int64_t i = 0; i < b; ++i) CK(cudaGraphLaunch(ctx->gexec, ctx->st));
    done += b;
    ctx->read_ctl();
    if (ctx->hctl->status == ST_NUMERICAL) fail(PDCS_ERR_NUMERICAL, "line search failed (eta underflow / too many rejects)");
    if (ctx->hctl->status != ST_RUNNING) break;
    if (stop_at_tol && ctx->time_up(t0, time_limit)) { ctx->hctl->status = ST_TIME; ctx->write_ctl(); break; }
  }
  const Ctl& C = *ctx->hctl;
  const int64_t trials = C.trials - before.trials, iters = C.total - before.total;
  ctx->launches += trials * ctx->nodes_trial + iters * ctx->nodes_accept +
                   (iters / std::max(1, ctx->prm.check_interval)) * ctx->nodes_check;
  ctx->hctl->stop_at_tol = 0;
  ctx->write_ctl();
  return true;
}

// Host loop of Alg. 1 (the accept flag is read back after each trial); used
// with per-kernel timing, with a non-capturable communicator (loopback) and as
// the fallback when graphs are unavailable.
static void run_steps(pdcs_ctx* ctx, int64_t n_inner, bool stop_at_tol, double time_limit) {
  if (run_steps_graph(ctx, n_inner, stop_at_tol, time_limit)) return;
  auto t0 = std::chrono::steady_clock::now();
  for (int64_t s = 0; s < n_inner; ++s) {
    for (;;) {
      ctx->trial();
      CK(cudaMemcpyAsync(ctx->hctl, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->st));
      CK(cudaStreamSynchronize(ctx->st));
      if (ctx->hctl->status == ST_NUMERICAL) fail(PDCS_ERR_NUMERICAL, "line search failed (eta underflow / too many rejects)");
      if (ctx->hctl->accepted) break;
    }
    const bool chk = ctx->hctl->need_check;
    ctx->accept();
    if (chk) {
      ctx->check();
      if (stop_at_tol) {
        ctx->read_ctl();
        if (ctx->hctl->done) { ctx->hctl->status = ST_OPTIMAL; ctx->write_ctl(); return; }
        if (ctx->time_up(t0, time_limit)) { ctx->hctl->status = ST_TIME; ctx->write_ctl(); return; }
      }
    }
  }
}

// pdcs_iterate / pdcs_solve on a context whose last solve ended: NUMERICAL_ERROR
// is final; OPTIMAL / ITERATION_ / TIME_LIMIT need pdcs_set_tolerance first.
static int finished_status(pdcs_ctx* ctx) {
  ctx->read_ctl();
  return ctx->hctl->status;
}

pdcs_status pdcs_iterate(pdcs_ctx* ctx, int64_t n_inner, pdcs_result_t* out) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    if (n_inner < 0) fail(PDCS_ERR_ARG, "n_inner < 0");
    const int fs = finished_status(ctx);
    if (fs == ST_NUMERICAL) fail(PDCS_ERR_STATE, "solver is in NUMERICAL_ERROR");
    if (fs != ST_RUNNING) fail(PDCS_ERR_STATE, "the last pdcs_solve finished; pdcs_set_tolerance continues it");
    ctx->launches = 0;
    auto t0 = std::chrono::steady_clock::now();
    run_steps(ctx, n_inner, false, 0.0);
    ctx->flush_timing();
    ctx->read_ctl();
    finish_result(ctx, out, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  });
}

pdcs_status pdcs_solve(pdcs_ctx* ctx, pdcs_result_t* out) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    auto t0 = std::chrono::steady_clock::now();
    ctx->launches = 0;
    const int fs = finished_status(ctx);
    if (fs == ST_NUMERICAL) fail(PDCS_ERR_STATE, "solver is in NUMERICAL_ERROR");
    if (fs != ST_RUNNING) {                        // already finished: report it again
      finish_result(ctx, out, 0.0);
      return;
    }
    const int64_t remaining = std::max<int64_t>(0, ctx->prm.max_iters - ctx->hctl->total);
    try {
      run_steps(ctx, remaining, true, ctx->prm.time_limit_s);
    } catch (const StatusErr& e) {
      if (e.st != PDCS_ERR_NUMERICAL) throw;
      ctx->read_ctl();
      ctx->hctl->status = ST_NUMERICAL;
      ctx->write_ctl();
    }
    ctx->flush_timing();
    ctx->read_ctl();
    if (ctx->hctl->status == ST_RUNNING) { ctx->hctl->status = ST_ITER; ctx->write_ctl(); }
    finish_result(ctx, out, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  });
}

// Tighten or loosen the stopping tolerance between solves (multi-tolerance
// runs: time to 1e-3, then continue to 1e-6 from the same state).  Clears a
// finished status so the next pdcs_solve continues; NUMERICAL_ERROR stays.
pdcs_status pdcs_set_tolerance(pdcs_ctx* ctx, double tol, double time_limit_s) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    if (!(tol >= 0.0) || !(time_limit_s >= 0.0)) fail(PDCS_ERR_ARG, "tol and time_limit_s must be >= 0");
    ctx->read_ctl();
    if (ctx->hctl->status == ST_NUMERICAL) fail(PDCS_ERR_STATE, "solver is in NUMERICAL_ERROR");
    ctx->prm.tol = tol;
    ctx->prm.time_limit_s = time_limit_s;
    ctx->hctl->tol = tol;
    ctx->hctl->done = 0;
    ctx->hctl->status = ST_RUNNING;
    ctx->write_ctl();
  });
}

pdcs_status pdcs_kkt(pdcs_ctx* ctx, int which, pdcs_kkt_t* out) {
  if (!ctx || !out) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    const double *xs, *ys;
    switch (which) {
      case PDCS_CURRENT: xs = ctx->x.p; ys = ctx->y.p; break;
      case PDCS_PDHG_OUT: xs = ctx->xh.p; ys = ctx->yh.p; break;
      case PDCS_ANCHOR: xs = ctx->x0.p; ys = ctx->y0.p; break;
      case PDCS_BEST: xs = ctx->bx.p; ys = ctx->by.p; break;
      case PDCS_CANDIDATE: xs = ctx->candx.p; ys = ctx->candy.p; break;
      default: fail(PDCS_ERR_ARG, "bad which");
    }
    ctx->products(xs, ys, ctx->tmpm.p, ctx->tmpn.p);
    KktCand c0{xs, ys, ctx->tmpm.p, ctx->tmpn.p, ctx->res0.p, ctx->lam0.p};
    // finalize in evaluate mode writes kkt[0]; keep the rest of the control block
    ctx->read_ctl();
    Ctl saved = *ctx->hctl;
    ctx->kkt_launch(c0, c0, 1, 0);
    ctx->read_ctl();
    out->err_p = ctx->hctl->kkt[0][0]; out->err_d = ctx->hctl->kkt[0][1]; out->err_gap = ctx->hctl->kkt[0][2];
    out->pobj = ctx->hctl->kkt[0][3]; out->dobj = ctx->hctl->kkt[0][4];
    *ctx->hctl = saved;
    ctx->write_ctl();
  });
}

pdcs_status pdcs_get_iterate(pdcs_ctx* ctx, int which, int space, double* x, double* y) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    const double *xs, *ys;
    switch (which) {
      case PDCS_CURRENT: xs = ctx->x.p; ys = ctx->y.p; break;
      case PDCS_PDHG_OUT: xs = ctx->xh.p; ys = ctx->yh.p; break;
      case PDCS_ANCHOR: xs = ctx->x0.p; ys = ctx->y0.p; break;
      case PDCS_BEST: xs = ctx->bx.p; ys = ctx->by.p; break;
      case PDCS_CANDIDATE: xs = ctx->candx.p; ys = ctx->candy.p; break;
      default: fail(PDCS_ERR_ARG, "bad which");
    }
    cudaStream_t st = ctx->st;
    const int64_t n = ctx->n, m = ctx->m;
    const double* xo = xs;
    const double* yo = ys;
    if (space == PDCS_ORIGINAL) {
      k_ewise<<<grid_for(n, ctx->sms), kThreads, 0, st>>>(n, xs, ctx->q.p, 0, ctx->tmpn.p);
      k_ewise<<<grid_for(m, ctx->sms), kThreads, 0, st>>>(m, ys, ctx->r.p, 0, ctx->tmpm.p);
      CK(cudaGetLastError());
      xo = ctx->tmpn.p;
      yo = ctx->tmpm.p;
    } else if (space != PDCS_SCALED) {
      fail(PDCS_ERR_ARG, "bad space");
    }
    const cudaMemcpyKind kind = ctx->mem_kind == PDCS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (x && n) CK(cudaMemcpyAsync(x, ctx->to_caller(xo), n * sizeof(double), kind, st));
    if (y && m) CK(cudaMemcpyAsync(y, yo, m * sizeof(double), kind, st));
    CK(cudaStreamSynchronize(st));
  });
}

pdcs_status pdcs_get_state(pdcs_ctx* ctx, double* x, double* y, double* x0, double* y0, double* xsum,
                           double* ysum, double* sc) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    const cudaMemcpyKind kind = ctx->mem_kind == PDCS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const int64_t n = ctx->n, m = ctx->m;
    auto get = [&](double* dst, const DBuf<double>& src, int64_t cnt) {
      if (dst && cnt) CK(cudaMemcpyAsync(dst, src.p, cnt * sizeof(double), kind, ctx->st));
    };
    auto getx = [&](double* dst, const DBuf<double>& src) {
      if (dst && n) CK(cudaMemcpyAsync(dst, ctx->to_caller(src.p), n * sizeof(double), kind, ctx->st));
    };
    getx(x, ctx->x); get(y, ctx->y, m); getx(x0, ctx->x0); get(y0, ctx->y0, m);
    getx(xsum, ctx->xsum); get(ysum, ctx->ysum, m);
    ctx->read_ctl();
    if (sc) {
      const Ctl& C = *ctx->hctl;
      const double v[13] = {C.eta, C.eta_init, C.omega, C.beta, C.Wsum, C.r_start, C.e_anchor, C.e_prev,
                            C.best_e, (double)C.k, (double)C.total, (double)C.trials, (double)C.restarts};
      std::memcpy(sc, v, sizeof(v));
    }
  });
}

pdcs_status pdcs_set_state(pdcs_ctx* ctx, const double* x, const double* y, const double* x0,
                           const double* y0, const double* xsum, const double* ysum, const double* sc) {
  if (!ctx || !x || !y || !x0 || !y0 || !xsum || !ysum || !sc) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    const cudaMemcpyKind kind = ctx->mem_kind == PDCS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const int64_t n = ctx->n, m = ctx->m;
    cudaStream_t st = ctx->st;
    auto put = [&](DBuf<double>& dst, const double* src, int64_t cnt) {
      if (cnt) CK(cudaMemcpyAsync(dst.p, src, cnt * sizeof(double), kind, st));
    };
    ctx->from_caller(ctx->x.p, x, kind); put(ctx->y, y, m); ctx->from_caller(ctx->x0.p, x0, kind);
    put(ctx->y0, y0, m); ctx->from_caller(ctx->xsum.p, xsum, kind); put(ctx->ysum, ysum, m);
    ctx->products(ctx->x.p, ctx->y.p, ctx->kxh.p, ctx->kty.p);
    ctx->spmv_store(ctx->K, ctx->x0.p, ctx->kx0.p);      // fresh K x0 (the carried products restart here)
    auto cp = [&](double* d, const double* s_, int64_t cnt) {
      if (cnt) CK(cudaMemcpyAsync(d, s_, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st));
    };
    cp(ctx->xh.p, ctx->x.p, n); cp(ctx->yh.p, ctx->y.p, m); cp(ctx->kxc.p, ctx->kxh.p, m);
    cp(ctx->ktyh.p, ctx->kty.p, n);
    ctx->read_ctl();
    Ctl& C = *ctx->hctl;
    C.eta = sc[0]; C.eta_init = sc[1]; C.omega = sc[2]; C.beta = sc[3]; C.Wsum = sc[4]; C.r_start = sc[5];
    C.e_anchor = sc[6]; C.e_prev = sc[7]; C.best_e = sc[8]; C.k = (int64_t)sc[9]; C.total = (int64_t)sc[10];
    C.trials = (int64_t)sc[11]; C.restarts = (int64_t)sc[12];
    C.tau = C.eta / C.omega; C.sigma = C.eta * C.omega;
    C.status = ST_RUNNING; C.rejects = 0; C.accepted = 0; C.need_check = 0; C.store_kty = 0;
    ctx->write_ctl();
  });
}

pdcs_status pdcs_get_scaling(pdcs_ctx* ctx, double* r, double* q) {
  if (!ctx) return PDCS_ERR_ARG;
  return guard(ctx, [&] {
    if (!ctx->cones_set) fail(PDCS_ERR_STATE, "call pdcs_set_cones first");
    const cudaMemcpyKind kind = ctx->mem_kind == PDCS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (r && ctx->m) CK(cudaMemcpyAsync(r, ctx->r.p, ctx->m * sizeof(double), kind, ctx->st));
    if (q && ctx->n) CK(cudaMemcpyAsync(q, ctx->to_caller(ctx->q.p), ctx->n * sizeof(double), kind, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
  });
}

void pdcs_enable_timing(pdcs_ctx* ctx, int on) {
  if (!ctx) return;
  ctx->timing = on != 0;
  ctx->ktimes.clear();
}

int pdcs_kernel_times(pdcs_ctx* ctx, char (*names)[32], double* ms, int64_t* launches, int cap) {
  if (!ctx) return 0;
  int i = 0;
  for (auto& kv : ctx->ktimes) {
    if (i >= cap) break;
    if (names) { std::strncpy(names[i], kv.first.c_str(), 31); names[i][31] = 0; }
    if (ms) ms[i] = kv.second.first;
    if (launches) launches[i] = kv.second.second;
    ++i;
  }
  return i;
}

int pdcs_get_scalars(pdcs_ctx* ctx, double* out, int cap) {
  if (!ctx || !out || !ctx->ctl) return 0;
  if (guard(ctx, [&] { ctx->read_ctl(); }) != PDCS_OK) return 0;
  const Ctl& C = *ctx->hctl;
  double v[49] = {C.eta, C.omega, C.beta, (double)C.k, (double)C.total, (double)C.trials,
                  (double)C.restarts, C.e_anchor, C.Wsum, C.eta_init,
                  C.kkt[0][0], C.kkt[0][1], C.kkt[0][2], C.kkt[0][3], C.kkt[0][4],
                  C.kkt[1][0], C.kkt[1][1], C.kkt[1][2], C.kkt[1][3], C.kkt[1][4],
                  C.e_prev, C.best_e, (double)C.use_avg, (double)C.restart, C.last_num, C.last_cross,
                  (double)ctx->tK.on, ctx->tK.tune_csr_ms, ctx->tK.tune_tiled_ms,
                  (double)ctx->tKT.on, ctx->tKT.tune_csr_ms, ctx->tKT.tune_tiled_ms,
                  ctx->tK.build_ms, ctx->tKT.build_ms, ctx->t_create_ms, ctx->t_cones_ms,
                  (double)ctx->colperm, (double)(ctx->pK.on ? ctx->pK.P : 0), ctx->pK.tune_csr_ms,
                  ctx->pK.tune_panel_ms, (double)(ctx->pKT.on ? ctx->pKT.P : 0), ctx->pKT.tune_csr_ms,
                  ctx->pKT.tune_panel_ms, (double)pdcs_ctx::fused(ctx->tK), ctx->tK.tune_fused_ms,
                  (double)pdcs_ctx::fused(ctx->tKT), ctx->tKT.tune_fused_ms, (double)ctx->K.csr_u,
                  (double)ctx->KT.csr_u};
  const int k = std::min(cap, 49);
  for (int i = 0; i < k; ++i) out[i] = v[i];
  return k;
}

int64_t pdcs_launch_count(const pdcs_ctx* ctx) { return ctx ? ctx->launches : 0; }

void pdcs_destroy(pdcs_ctx* ctx) { delete ctx; }

// Host-only timing of the tiled-format build (setup diagnostics; no device).
// out[0] = total ms, out[1] = ms in the threaded per-range builds, out[2] = staged nnz.
int pdcs_tiled_build_host(const int64_t* row_ptr, const int32_t* col, int64_t rows, int64_t nvec, int elem,
                          double* out) {
  if (!row_ptr || (!col && row_ptr[rows] > 0) || rows < 0 || nvec <= 0 || (elem != 1 && elem != 2) || !out)
    return 0;
  TiledHost H;
  build_tiled(row_ptr, col, rows, nvec, elem, H, true);
  out[0] = H.build_ms; out[1] = H.ranges_ms; out[2] = (double)H.staged;
  return 3;
}

// Device check of the deferred tiled build: the layout built by the host with
// the bank balancing and slicing on the device (the solver's default) against
// the all-host build, entry by entry.  out[0] = mismatching entries over the
// column ids, value permutation, row pointers, block bases and segment
// descriptors; out[1] = all-host build ms; out[2] = deferred host ms; out[3] =
// device ms; out[4] = final layout entries.  Returns 5, 0 on bad arguments, -1
// on a CUDA error.
int pdcs_tiled_device_check(const int64_t* row_ptr, const int32_t* col, int64_t rows, int64_t nvec, int elem,
                            double* out) {
  if (!row_ptr || (!col && row_ptr[rows] > 0) || rows < 0 || nvec <= 0 || (elem != 1 && elem != 2) || !out)
    return 0;
  try {
    TiledHost A, B;
    build_tiled(row_ptr, col, rows, nvec, elem, A);                  // all host
    build_tiled(row_ptr, col, rows, nvec, elem, B, true, true);      // deferred, parts
    if (!B.defer) return 0;
    cudaStream_t st = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    DBuf<int32_t> rp, bb, perm, pperm, bperm, nperm;
    DBuf<uint16_t> cs, pcol, bcol, ncol;
    rp.alloc(B.tot_rp); bb.alloc(B.tot_bb); cs.alloc(B.tot_s); perm.alloc(B.tot_s);
    pcol.alloc(std::max<size_t>(B.tot_pre, 1)); pperm.alloc(std::max<size_t>(B.tot_pre, 1));
    CK(cudaMemset(rp.p, 0, B.tot_rp * sizeof(int32_t)));
    CK(cudaMemset(bb.p, 0, B.tot_bb * sizeof(int32_t)));
    CK(cudaMemset(cs.p, 0, B.tot_s * sizeof(uint16_t)));
    CK(cudaMemset(perm.p, 0xff, B.tot_s * sizeof(int32_t)));
    auto put = [&](auto* dst, const auto& v, size_t off) {
      if (!v.empty()) CK(cudaMemcpy(dst + off, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice));
    };
    for (size_t w = 0; w < B.parts.size(); ++w) {
      put(rp.p, B.parts[w].rowptr, B.o_rp[w]);
      put(bb.p, B.parts[w].blkb, B.o_bb[w]);
      put(pcol.p, B.parts[w].col_s, B.o_pre[w]);
      put(pperm.p, B.parts[w].perm_s, B.o_pre[w]);
    }
    const int64_t nb = (int64_t)B.dblk.size();
    if (nb) {
      DBuf<TDefer> dseg;
      DBuf<int2> dblk;
      upload(dseg, B.dseg, st);
      upload(dblk, B.dblk, st);
      bcol.alloc(B.tot_pre); ncol.alloc(B.tot_pre); bperm.alloc(B.tot_pre); nperm.alloc(B.tot_pre);
      launch_tile_balance(dseg.p, B.dseg, dblk.p, nb, elem, rp.p, pcol.p, pperm.p, bcol.p, bperm.p, ncol.p, nperm.p,
                          nullptr);
      k_tile_slice<<<(int)((nb + 127) / 128), 128>>>(dseg.p, dblk.p, nb, rp.p, bb.p, ncol.p, nperm.p, cs.p, perm.p);
      CK(cudaGetLastError());
    }
    CK(cudaDeviceSynchronize());
    const double dev_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::vector<uint16_t> hc(B.tot_s);
    std::vector<int32_t> hp(B.tot_s), hr(B.tot_rp), hb(B.tot_bb);
    CK(cudaMemcpy(hc.data(), cs.p, B.tot_s * sizeof(uint16_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hp.data(), perm.p, B.tot_s * sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), rp.p, B.tot_rp * sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb.data(), bb.p, B.tot_bb * sizeof(int32_t), cudaMemcpyDeviceToHost));
    double bad = 0;
    if (A.col_s.size() != hc.size() || A.rowptr.size() != hr.size() || A.blkb.size() != hb.size() ||
        A.seg.size() != B.seg.size())
      bad = 1e18;
    else {
      for (size_t i = 0; i < hc.size(); ++i) bad += (A.col_s[i] != hc[i]) + (A.perm_s[i] != hp[i]);
      for (size_t i = 0; i < hr.size(); ++i) bad += A.rowptr[i] != hr[i];
      for (size_t i = 0; i < hb.size(); ++i) bad += A.blkb[i] != hb[i];
      for (size_t i = 0; i < A.seg.size(); ++i)
        bad += A.seg[i].nz != B.seg[i].nz || A.seg[i].bb != B.seg[i].bb || A.seg[i].rp != B.seg[i].rp ||
               A.seg[i].V != B.seg[i].V || A.seg[i].tile != B.seg[i].tile;
    }
    out[0] = bad; out[1] = A.build_ms; out[2] = B.build_ms; out[3] = dev_ms; out[4] = (double)hc.size();
    return 5;
  } catch (...) {
    return -1;
  }
}

// Device structure build (build_tiled_device, the solver's default) against
// the all-host build, entry by entry: column ids and value permutation of the
// staged and direct entries, row pointers, row order, block bases, segment
// descriptors, work items, batches and chunks.  out[0] = mismatches; out[1] =
// all-host ms; out[2] = device-build ms; out[3] = staged entries; out[4] =
// layout entries.  Returns 5, 0 on bad arguments (or when the layout is not
// the sliced, balanced one), -1 on a CUDA error.
int pdcs_tiled_devbuild_check(const int64_t* row_ptr, const int32_t* col, int64_t rows, int64_t nvec, int elem,
                              double* out) {
  if (!row_ptr || (!col && row_ptr[rows] > 0) || rows < 0 || nvec <= 0 || (elem != 1 && elem != 2) || !out)
    return 0;
  if (!tiled_devbuild_env() || row_ptr[rows] >= ((int64_t)1 << 31)) return 0;
  try {
    TiledHost A, B;
    build_tiled(row_ptr, col, rows, nvec, elem, A);                  // all host
    cudaStream_t st = nullptr;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int64_t nnz = row_ptr[rows];
    std::vector<int32_t> p32(rows + 1);
    for (int64_t i = 0; i <= rows; ++i) p32[i] = (int32_t)row_ptr[i];
    DBuf<int32_t> dptr, dcol;
    upload(dptr, p32, st);
    dcol.alloc(std::max<int64_t>(nnz, 1));
    if (nnz) CK(cudaMemcpy(dcol.p, col, nnz * sizeof(int32_t), cudaMemcpyHostToDevice));
    TiledDevArrays D;
    build_tiled_device(dptr.p, dcol.p, row_ptr, rows, nvec, elem, -1.0, B, D, st, sms);
    CK(cudaDeviceSynchronize());
    double bad = 0;
    auto dl = [](const auto& d, size_t n, auto* tag) {
      std::vector<std::remove_pointer_t<decltype(tag)>> h(n);
      if (n) CK(cudaMemcpy(h.data(), d.p, n * sizeof(h[0]), cudaMemcpyDeviceToHost));
      return h;
    };
    const auto hc = dl(D.col_s, B.tot_s, (uint16_t*)nullptr);
    const auto hp = dl(D.perm_s, B.tot_s, (int32_t*)nullptr);
    const auto hr = dl(D.rowptr, B.tot_rp, (int32_t*)nullptr);
    const auto hs = dl(D.srow, B.tot_rp, (uint16_t*)nullptr);
    const auto hb = dl(D.blkb, B.tot_bb, (int32_t*)nullptr);
    const auto hcd = dl(D.col_d, B.tot_d, (int32_t*)nullptr);
    const auto hpd = dl(D.perm_d, B.tot_d, (int32_t*)nullptr);
    // staged entries: equal up to the shorter array; the longer one's tail is
    // padding (the host build rounds part ends up to 64 entries)
    const size_t ns = std::min(A.col_s.size(), hc.size());
    for (size_t i = 0; i < ns; ++i) bad += (A.col_s[i] != hc[i]) + (A.perm_s[i] != hp[i]);
    for (size_t i = ns; i < A.col_s.size(); ++i) bad += A.col_s[i] != 0 || A.perm_s[i] != -1;
    for (size_t i = ns; i < hc.size(); ++i) bad += hc[i] != 0 || hp[i] != -1;
    if (A.rowptr.size() != hr.size() || A.srow.size() != hs.size() || A.blkb.size() != hb.size() ||
        A.col_d.size() != hcd.size() || A.seg.size() != B.seg.size() || A.work.size() != B.work.size() ||
        A.chunk.size() != B.chunk.size() || A.batch.size() != B.batch.size() || A.scratch != B.scratch ||
        A.staged != B.staged)
      bad += 1e18;
    else {
      for (size_t i = 0; i < hr.size(); ++i) bad += (A.rowptr[i] != hr[i]) + (A.srow[i] != hs[i]);
      for (size_t i = 0; i < hb.size(); ++i) bad += A.blkb[i] != hb[i];
      for (size_t i = 0; i < hcd.size(); ++i) bad += (A.col_d[i] != hcd[i]) + (A.perm_d[i] != hpd[i]);
      for (size_t i = 0; i < A.seg.size(); ++i)
        bad += A.seg[i].nz != B.seg[i].nz || A.seg[i].bb != B.seg[i].bb || A.seg[i].rp != B.seg[i].rp ||
               A.seg[i].V != B.seg[i].V || A.seg[i].tile != B.seg[i].tile;
      for (size_t i = 0; i < A.work.size(); ++i)
        bad += std::memcmp(&A.work[i], &B.work[i], sizeof(TWork)) != 0;
      for (size_t i = 0; i < A.batch.size(); ++i)
        bad += std::memcmp(&A.batch[i], &B.batch[i], sizeof(TBatch)) != 0;
      for (size_t i = 0; i < A.chunk.size(); ++i)
        bad += A.chunk[i].row0 != B.chunk[i].row0 || A.chunk[i].nrows != B.chunk[i].nrows ||
               A.chunk[i].ngroups != B.chunk[i].ngroups || A.chunk[i].scratch != B.chunk[i].scratch;
    }
    out[0] = bad; out[1] = A.build_ms; out[2] = B.build_ms; out[3] = (double)B.staged; out[4] = (double)hc.size();
    return 5;
  } catch (...) {
    return -1;
  }
}

int pdcs_tiled_layout_stats(const int64_t* row_ptr, const int32_t* col, int64_t rows, int64_t nvec, int elem,
                            double* out, int cap) {
  if (!row_ptr || (!col && row_ptr[rows] > 0) || rows < 0 || nvec <= 0 || (elem != 1 && elem != 2) || !out)
    return 0;
  TiledHost H;
  build_tiled(row_ptr, col, rows, nvec, elem, H);
  // simulate the shared-memory gathers of k_tiled_partial along the schedule
  // of tiled_block_schedule: per (block, time step, quad position) one
  // ld.shared; a phase of P lanes costs the largest number of distinct
  // addresses in one bank group
  const int P = elem == 2 ? 8 : 16;
  double quads = 0, pads = 0, inst = 0, wav = 0, segs = 0, bound = 0;
  std::vector<int32_t> brows;
  std::vector<std::vector<std::pair<int32_t, int32_t>>> lanes;
  for (size_t si = 0; si < H.seg.size(); ++si) {
    const TSeg& S = H.seg[si];
    if (S.tile < 0) continue;
    segs += 1;
    const int32_t* rp = H.rowptr.data() + S.rp;
    int32_t nr = 0;
    for (const TWork& W : H.work)
      if ((int64_t)si >= W.s0 && (int64_t)si < W.s1) { nr = H.chunk[W.chunk].nrows; break; }
    quads += rp[nr] - rp[0];
    for (int32_t pos = 0; pos < nr; ++pos)
      for (int32_t j = 0; j < rp[pos + 1] - rp[pos]; ++j)
        for (int k = 0; k < 4; ++k) pads += H.perm_s[S.nz + 4 * quad_slot(H.blkb, S, rp, pos, j) + k] < 0;
    const int nblk = tiled_blocks(nr, S.V);
    for (int blk = 0; blk < nblk; ++blk) {
      tiled_block_schedule(rp, nr, S.V, blk, brows, lanes);
      size_t tmax = 0;
      for (const auto& ln : lanes) tmax = std::max(tmax, ln.size());
      for (int ph = 0; ph < 32 / P; ++ph) {
        int load[16] = {0};
        double active_slots = 0;
        for (size_t t = 0; t < tmax; ++t)
          for (int k = 0; k < 4; ++k) {
            int cnt[16] = {0};
            int seen[16][16];
            int active = 0;
            for (int lane = ph * P; lane < ph * P + P; ++lane) {
              if (t >= lanes[lane].size()) continue;
              ++active;
              const int64_t e = S.nz + 4 * quad_slot(H.blkb, S, rp, brows[lanes[lane][t].first], lanes[lane][t].second) + k;
              const int c = H.col_s[e];
              const int g = c % P;
              if (H.perm_s[e] >= 0) ++load[g];
              bool dup = false;
              for (int z = 0; z < cnt[g]; ++z) dup |= seen[g][z] == c;
              if (!dup) seen[g][cnt[g]++] = c;
            }
            if (active) { wav += *std::max_element(cnt, cnt + P); active_slots += 1; }
          }
        bound += std::max<double>(active_slots, (double)*std::max_element(load, load + P));
      }
      inst += 4.0 * (double)tmax;
    }
  }
  // structure check: every CSR entry stored exactly once, under its own column
  const int64_t nnz = H.nnz;
  std::vector<uint8_t> hit(nnz, 0);
  double bad = 0;
  for (size_t si = 0; si < H.seg.size(); ++si) {
    const TSeg& S = H.seg[si];
    int32_t nr = 0;
    for (const TWork& W : H.work)
      if ((int64_t)si >= W.s0 && (int64_t)si < W.s1) { nr = H.chunk[W.chunk].nrows; break; }
    const int32_t* rp = H.rowptr.data() + S.rp;
    auto visit = [&](int64_t e) {
      const int32_t pp = S.tile >= 0 ? H.perm_s[S.nz + e] : H.perm_d[S.nz + e];
      if (pp < 0) return;
      const int64_t c = S.tile >= 0 ? (int64_t)S.tile * H.T + H.col_s[S.nz + e] : H.col_d[S.nz + e];
      if (pp >= nnz || hit[pp] || c != col[pp]) { bad += 1; return; }
      hit[pp] = 1;
    };
    if (S.tile >= 0) {
      for (int32_t pos = 0; pos < nr; ++pos)
        for (int32_t j = 0; j < rp[pos + 1] - rp[pos]; ++j)
          for (int k = 0; k < 4; ++k) visit(4 * quad_slot(H.blkb, S, rp, pos, j) + k);
    } else {
      for (int64_t e = 0; e < rp[nr]; ++e) visit(e);
    }
  }
  for (int64_t q = 0; q < nnz; ++q) bad += hit[q] == 0;
  const double v[11] = {(double)H.nnz, (double)H.staged, quads, pads, segs, (double)H.work.size(), inst, wav,
                        H.build_ms, bound, bad};
  const int k = std::min(cap, 11);
  for (int i = 0; i < k; ++i) out[i] = v[i];
  return k;
}

// ---------------------------------------------------------------- standalone projections
// Multi-cone projection plan (Figs. 3-4):
// the block descriptors of one cone product, grouped into the solver's size
// classes (or all SOC/RSOC blocks forced into one team), uploaded once.
struct pdcs_proj {
  int device = 0, sms = 0;
  DBuf<Block> blocks;
  pdcs_ctx::BClass cls[kNClass];
  DBuf<double> gbuf;
  int64_t len = 0;
  std::string err;
};

pdcs_status pdcs_proj_create(pdcs_proj** out, int device, const int32_t* kinds, const int64_t* dims,
                             int64_t nblocks, int team) {
  if (!out) return PDCS_ERR_ARG;
  *out = nullptr;
  pdcs_proj* P = new pdcs_proj();
  pdcs_status s = guard(nullptr, [&] {
    if (nblocks < 0 || (nblocks > 0 && (!kinds || !dims))) fail(PDCS_ERR_ARG, "bad block list");
    if (team < -1 || team >= kNClass) fail(PDCS_ERR_ARG, "team must be -1 (auto) or 0..4");
    std::vector<Block> v;
    v.reserve((size_t)nblocks);
    int64_t off = 0;
    for (int64_t b = 0; b < nblocks; ++b) {
      const int32_t k = kinds[b];
      const int64_t d = dims[b];
      const bool ok = ((k == C_SOC && d >= 2) || (k == C_RSOC && d >= 3) || ((k == C_EXP || k == C_DEXP) && d == 3)) &&
                      d <= INT32_MAX;
      if (!ok) fail(PDCS_ERR_CONE, "block " + std::to_string(b) + ": kind must be SOC (dim>=2), RSOC (>=3), EXP/DEXP (3)");
      v.push_back(Block{off, k, (int32_t)d});
      off += d;
    }
    P->len = off;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) fail(PDCS_ERR_CUDA, "no CUDA device");
    if (device < 0 || device >= ndev) fail(PDCS_ERR_ARG, "bad device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(PDCS_ERR_CUDA, "libpdcs is built for sm_100a");
    P->device = device;
    P->sms = prop.multiProcessorCount;
    const ClassPolicy pol = class_policy(v, P->sms);
    auto cls = [&](const Block& b) {
      if (b.kind == C_EXP || b.kind == C_DEXP) return 0;
      if (team >= 0) return team;
      return pol.of(b);
    };
    std::stable_sort(v.begin(), v.end(), [&](const Block& a, const Block& b) {
      const int ca = cls(a), cb = cls(b);
      if (ca != cb) return ca < cb;
      if (a.kind != b.kind) return a.kind < b.kind;
      return a.dim < b.dim;
    });
    for (size_t i = 0; i < v.size(); ++i) {
      const int c = cls(v[i]);
      if (P->cls[c].count == 0) P->cls[c].begin = (int64_t)i;
      P->cls[c].count++;
    }
    for (int c = 0; c < kNClass; ++c) {
      const int64_t cnt = P->cls[c].count;
      if (!cnt) continue;
      if (c == 0) P->cls[c].grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + kThreadsSmall - 1) / kThreadsSmall, (int64_t)P->sms * 32));
      else if (c == 1) P->cls[c].grid = (int)std::max<int64_t>(1, std::min<int64_t>((cnt + 7) / 8, (int64_t)P->sms * 8));
      else if (c == 2) P->cls[c].grid = (int)std::min<int64_t>(cnt, (int64_t)P->sms * 4);
      else if (c == 3) P->cls[c].grid = kClusterCtas * (int)std::min<int64_t>(cnt, (int64_t)P->sms * 2 / kClusterCtas);
      else {
        int nb = 0;
        CK(grid_team_occupancy(&nb));
        P->cls[c].grid = std::max(1, std::min(nb, 4)) * P->sms;
      }
    }
    if (!v.empty()) {
      P->blocks.alloc(v.size());
      CK(cudaMemcpy(P->blocks.p, v.data(), v.size() * sizeof(Block), cudaMemcpyHostToDevice));
    }
    P->gbuf.alloc(4 * (size_t)P->sms * 8);
  });
  if (s != PDCS_OK) { delete P; return s; }
  *out = P;
  return PDCS_OK;
}

pdcs_status pdcs_proj_run(pdcs_proj* P, const double* D, const double* v, double* out, void* stream) {
  if (!P || (P->len > 0 && (!v || !out))) return PDCS_ERR_ARG;
  return guard(nullptr, [&] {
    CK(cudaSetDevice(P->device));
    cudaStream_t st = (cudaStream_t)stream;
    BlockArgs A{};
    A.op = BOP_PROJECT;
    A.D = D;
    A.scratch = v;
    A.out = out;
    for (int c = 0; c < kNClass; ++c) {
      if (P->cls[c].count == 0) continue;
      BlockArgs B = A;
      B.blocks = P->blocks.p + P->cls[c].begin;
      B.nblocks = P->cls[c].count;
      const int g = P->cls[c].grid;
      CK(launch_blocks(c, g, B, nullptr, P->gbuf.p, st));
      CK(cudaGetLastError());
    }
  });
}

int pdcs_proj_info(const pdcs_proj* P, int64_t* counts, int64_t* grids) {
  if (!P) return 0;
  for (int c = 0; c < kNClass; ++c) {
    if (counts) counts[c] = P->cls[c].count;
    if (grids) grids[c] = P->cls[c].grid;
  }
  return kNClass;
}

void pdcs_proj_destroy(pdcs_proj* P) { delete P; }

pdcs_status pdcs_nccl_unique_id(void* out128) {
  if (!out128) return PDCS_ERR_ARG;
  std::string e;
  if (!nccl().load(e)) { g_create_error = e; return PDCS_ERR_NCCL; }
  ncclUniqueId id;
  const ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) { g_create_error = nccl().GetErrorString(r); return PDCS_ERR_NCCL; }
  std::memcpy(out128, &id, sizeof(id));
  return PDCS_OK;
}

}  // extern "C"
