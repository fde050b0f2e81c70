// tiled.cuh — column-tiled SpMV with shared-memory vector tiles (fp64).
//
// Why: the two products of Eq. 5 gather a vector at random
// column ids.  Every fp64 gather costs a 32-byte L2 sector, and L1 allocates a
// 128-byte line per random sector, so its useful capacity for gathers is ~1/4
// of its size.  On B200 the CSR kernels of spmv.cuh are bound by L2 sector
// throughput, not HBM (profiles/r1_ncu_spmv_lasso.txt).
//
// Format (built at setup): rows are cut into chunks of <= kTRows
// rows; the gathered vector into tiles of T elements (64 KB).  For every
// (chunk, tile) pair with enough nonzeros the entries form a *staged segment*
// (tile-local uint16 column ids, 10 bytes per nonzero instead of 12, stored in
// zero-padded quads of 4 entries with row pointers counted in quads); the rest
// of a chunk's entries form one *direct segment* (int32 global ids, gathered
// from L2).  Each segment is a small CSR over the chunk's rows.  A work item is
// (chunk, group of consecutive segments); it stages each tile in shared memory,
// accumulates per-row partial dot products in shared memory and writes them to
// a scratch buffer.  The combine kernel sums a row's partials in a fixed order
// and applies the fused epilogue (dual update / Halpern step), so results are
// deterministic.
#pragma once
#include <type_traits>
#include "spmv.cuh"

namespace pdcs {

#ifndef PDCS_TP_MINB
#define PDCS_TP_MINB 2                // min resident CTAs/SM of k_tiled_partial<2>: caps registers at 64
#endif
#ifndef PDCS_TP_MINB1
#define PDCS_TP_MINB1 3               // k_tiled_partial<1>: 40 registers, 3 CTAs/SM (-10% time on Lasso)
#endif
constexpr int kTRows = 1024;          // rows per chunk (shared accumulator size)
constexpr int kTThreads = 512;        // CTA size of the partial kernel
constexpr int kTileBytes = 65536;     // one vector tile in shared memory

struct TSeg {
  int32_t tile;      // >= 0: staged tile index; -1: direct segment
  int32_t V;         // lanes per row (1, 2, 4, 8, 16, 32)
  int64_t rp;        // offset of the segment's row pointers (nrows + 1 entries)
  int64_t nz;        // offset of the segment's entries in its pool (staged: in entries, = 4 * quads)
  int64_t bb;        // staged, >= 0: sliced layout, offset of the segment's warp-block bases in blkb
};
// A staged segment of the deferred build: its bank balancing and
// sliced re-layout run on the device.  src: first entry of its unbalanced
// row-major quads in the "pre" arrays; dst: first entry in the final sliced
// arrays; rp / bb: its row pointers and warp-block bases; nr rows, V lanes.
struct TDefer {
  int64_t src, dst, rp, bb;
  int32_t nr, V;
};
struct TChunk {
  int64_t row0;
  int32_t nrows;
  int32_t ngroups;
  int64_t scratch;   // offset (in doubles) of the chunk's partials: ngroups * nrows * ELEM
};
// One item of the combine: rows [r0, r0 + kCombRowsNarrow) of a chunk with <= 4
// groups (4 rows per thread), rows [r0, r0 + kThreads) of a chunk with a few
// more, or rows [r0, r0 + kCombRowsWide) of a chunk with >= kCombWideG groups,
// whose group sums are split over kCombLanes lanes per row (Lasso K^T: ~150).
struct TCItem {
  int32_t chunk, r0;
};
constexpr int kCombLanes = 8;
constexpr int kCombRowsWide = 256 / kCombLanes;
constexpr int kCombWideG = 16;
constexpr int kCombRowsNarrow = 4 * 256;   // rows of an item of a chunk with <= kCombNarrowG groups
#ifndef PDCS_COMB_NARROW
#define PDCS_COMB_NARROW 2
#endif
constexpr int kCombNarrowG = PDCS_COMB_NARROW;   // 4 measured slower on Lasso K with pairs (3 groups, 80 registers): 26.6 -> 29.2 us
struct TWork {
  int32_t chunk, group, s0, s1;   // segments [s0, s1): direct ones run first, staged via batches
  int32_t b0, b1;                 // TMA batches [b0, b1) of the staged segments
};
// A TMA batch: quads [qa, qb) (segment-relative, qb - qa <= kBQ) of rows [ra, rb)
// of segment `seg`; `first` marks the first batch of that segment in the item.
struct TBatch {
  int32_t seg, ra, rb, qa, qb, first, ord, pad;   // ord: segment ordinal within the work item
};
constexpr int kBQ = 1024;             // quads per TMA batch (32 KB values + 8 KB column ids)
constexpr int kBR = kTRows + 8;       // row pointers per TMA batch (16-B aligned slice)
constexpr int kNST = 3;               // TMA pipeline stages
struct TiledMat {
  int64_t m = 0, nvec = 0, nwork = 0, nchunk = 0;
  int32_t T = 0, elem = 1;
  const TWork* work = nullptr;
  const TChunk* chunk = nullptr;
  const TSeg* seg = nullptr;
  const int32_t* rowptr = nullptr;
  const uint16_t* srow = nullptr;     // segment position -> chunk-local row (parallel to rowptr)
  const double* val_s = nullptr;
  const uint16_t* col_s = nullptr;
  const double* val_d = nullptr;
  const int32_t* col_d = nullptr;
  const TBatch* batch = nullptr;
  const int32_t* blkb = nullptr;      // sliced staged segments: first quad of every warp block
  const TCItem* citem = nullptr;      // combine items (k_tiled_combine)
  int64_t ncitem = 0;
};

// Shared-memory loads with 32-bit shared addresses (the tile pointer would
// otherwise reach the loop as a generic pointer: 64-bit generic loads).
__device__ __forceinline__ double2 lds_v2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// Streaming 16-byte loads of the matrix (no L1 allocation).
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
// 32-byte load (sm_100: LDG.256): one quad of values, one L2 sector, one request
__device__ __forceinline__ double4 ld_stream4(const double* p) {
  double4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// Staged segment row, quad layout: the row's entries are packed in quads of 4
// (32 B of values, 8 B of uint16 tile-local column ids, zero padded), so every
// load a lane issues is a full 16/8-byte vector and a warp touches whole
// sectors.  Lane l of the V-lane group takes quads qb+l, qb+l+V, ...
template <int V, int ELEM>
__device__ __forceinline__ void seg_row_dot_quad(const double* __restrict__ val4, const uint16_t* __restrict__ col4,
                                                 uint32_t xs_s, int32_t qb, int32_t qe, int lane, double& s1,
                                                 double& s2) {
  constexpr int U = 2;   // quads per lane per batch
  s1 = 0.0;
  s2 = 0.0;
  for (int32_t q0 = qb + lane; q0 < qe; q0 += U * V) {
    double a[U][4];
    uint32_t c[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int32_t q = q0 + u * V;
      if (q < qe) {
        const double4 v = ld_stream4(val4 + 4 * (int64_t)q);
        const uint2 cc = ld_stream_u2(col4 + 4 * (int64_t)q);
        a[u][0] = v.x; a[u][1] = v.y; a[u][2] = v.z; a[u][3] = v.w;
        c[u][0] = cc.x & 0xffffu; c[u][1] = cc.x >> 16; c[u][2] = cc.y & 0xffffu; c[u][3] = cc.y >> 16;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { a[u][k] = 0.0; c[u][k] = 0u; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * V < qe)                 // no shared-memory wavefronts for slots past the row
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (ELEM == 2) {
            const double2 v = lds_v2(xs_s + c[u][k] * 16u);
            s1 += a[u][k] * v.x;
            s2 += a[u][k] * v.y;
          } else {
            s1 += a[u][k] * lds_f64(xs_s + c[u][k] * 8u);
          }
        }
  }
  if (V > 1) {
#pragma unroll
    for (int o = V / 2; o >= 1; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
      if (ELEM == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
    }
  }
}

// Direct segment row (global gathers, int32 column ids): predicated batches of
// U entries per lane, all loads of a batch issued before any gather.
template <int V, int ELEM>
__device__ __forceinline__ void seg_row_dot_direct(const double* __restrict__ val, const int32_t* __restrict__ c32,
                                                   const double* __restrict__ xs, int32_t b, int32_t e, int lane,
                                                   double& s1, double& s2) {
  constexpr int U = 8;
  s1 = 0.0;
  s2 = 0.0;
  for (int32_t p = b + lane; p < e; p += U * V) {
    int32_t c[U];
    double a[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int32_t q = p + k * V;
      const bool ok = q < e;
      a[k] = ok ? ld_stream(val + q) : 0.0;
      c[k] = ok ? ld_stream(c32 + q) : 0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (ELEM == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xs) + c[k]);
        s1 += a[k] * v.x;
        s2 += a[k] * v.y;
      } else {
        s1 += a[k] * __ldg(xs + c[k]);
      }
    }
  }
  if (V > 1) {
#pragma unroll
    for (int o = V / 2; o >= 1; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
      if (ELEM == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
    }
  }
}

template <int V, int ELEM>
__device__ __forceinline__ void seg_rows(const TiledMat& M, const TSeg& S, const TChunk& C,
                                         const double* xs, uint32_t xs_s, bool staged, double* acc) {
  const int G = blockDim.x / V;
  const int g = threadIdx.x / V, lane = threadIdx.x % V;
  const int32_t* rp = M.rowptr + S.rp;
  for (int rb = 0; rb < C.nrows; rb += G) {        // uniform trip count per warp
    const int r = rb + g;
    double s1 = 0.0, s2 = 0.0;
    int32_t b = 0, e = 0;
    if (r < C.nrows) { b = __ldg(rp + r); e = __ldg(rp + r + 1); }
    if (staged) seg_row_dot_quad<V, ELEM>(M.val_s + S.nz, M.col_s + S.nz, xs_s, b, e, lane, s1, s2);
    else seg_row_dot_direct<V, ELEM>(M.val_d + S.nz, M.col_d + S.nz, xs, b, e, lane, s1, s2);
    if (lane == 0 && r < C.nrows) {
      const int rr = __ldg(M.srow + S.rp + r);
      acc[rr * ELEM] += s1;
      if (ELEM == 2) acc[rr * ELEM + 1] += s2;
    }
  }
}

// Partial dot products of every work item -> scratch.
// guard: 0 always run, 1 only while running, 2 only on an accepted step
template <int ELEM>
__global__ void __launch_bounds__(kTThreads, ELEM == 1 ? PDCS_TP_MINB1 : PDCS_TP_MINB) k_tiled_partial(TiledMat M, const double* __restrict__ x,
                                                             double* __restrict__ scratch, const Ctl* ctl,
                                                             int guard) {
  if (guard >= 1 && ctl->status != 4) return;
  if (guard == 2 && !ctl->accepted) return;
  extern __shared__ double smem[];
  double* tile = smem;                                  // T * ELEM doubles
  double* acc = smem + (size_t)M.T * ELEM;              // kTRows * ELEM doubles
  for (int64_t w = blockIdx.x; w < M.nwork; w += gridDim.x) {
    const TWork W = M.work[w];
    const TChunk C = M.chunk[W.chunk];
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    for (int s = W.s0; s < W.s1; ++s) {
      const TSeg S = M.seg[s];
      const bool staged = S.tile >= 0;
      if (staged) {
        const int64_t base = (int64_t)S.tile * M.T;
        const int64_t len = (M.nvec - base < M.T ? M.nvec - base : M.T) * ELEM;   // doubles
        const double2* src = reinterpret_cast<const double2*>(x + base * ELEM);
        double2* dst = reinterpret_cast<double2*>(tile);
        for (int64_t i = threadIdx.x; i < len / 2; i += blockDim.x) dst[i] = __ldg(src + i);
        if ((len & 1) && threadIdx.x == 0) tile[len - 1] = __ldg(x + base * ELEM + len - 1);
        __syncthreads();
      }
      const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(tile);
      switch (S.V) {
        case 1: seg_rows<1, ELEM>(M, S, C, x, xs_s, staged, acc); break;
        case 2: seg_rows<2, ELEM>(M, S, C, x, xs_s, staged, acc); break;
        case 4: seg_rows<4, ELEM>(M, S, C, x, xs_s, staged, acc); break;
        case 8: seg_rows<8, ELEM>(M, S, C, x, xs_s, staged, acc); break;
        case 16: seg_rows<16, ELEM>(M, S, C, x, xs_s, staged, acc); break;
        default: seg_rows<32, ELEM>(M, S, C, x, xs_s, staged, acc); break;
      }
      __syncthreads();
    }
    double* out = scratch + C.scratch + (int64_t)W.group * C.nrows * ELEM;
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) out[i] = acc[i];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ TMA pipeline
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA), completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int V, int ELEM>
__device__ __forceinline__ void batch_rows(const TiledMat& M, const TSeg& S, const TBatch& B, uint32_t tile_s,
                                           const double* sval, const uint16_t* scol, int32_t qcopy,
                                           const int32_t* rp, double* acc) {
  const int G = blockDim.x / V;
  const int g = threadIdx.x / V, lane = threadIdx.x % V;
  for (int rb = B.ra; rb < B.rb; rb += G) {              // uniform trip count per warp
    const int r = rb + g;
    double s1 = 0.0, s2 = 0.0;
    if (r < B.rb) {
      const int32_t qb = max(rp[r], B.qa), qe = min(rp[r + 1], B.qb);
      for (int32_t q = qb + lane; q < qe; q += V) {
        const int32_t l = q - qcopy;
        const double2 v01 = *reinterpret_cast<const double2*>(sval + 4 * l);
        const double2 v23 = *reinterpret_cast<const double2*>(sval + 4 * l + 2);
        const uint2 cc = *reinterpret_cast<const uint2*>(scol + 4 * l);
        const uint32_t c0 = cc.x & 0xffffu, c1 = cc.x >> 16, c2 = cc.y & 0xffffu, c3 = cc.y >> 16;
        if (ELEM == 2) {
          const double2 x0 = lds_v2(tile_s + c0 * 16u), x1 = lds_v2(tile_s + c1 * 16u);
          const double2 x2 = lds_v2(tile_s + c2 * 16u), x3 = lds_v2(tile_s + c3 * 16u);
          s1 += v01.x * x0.x; s2 += v01.x * x0.y;
          s1 += v01.y * x1.x; s2 += v01.y * x1.y;
          s1 += v23.x * x2.x; s2 += v23.x * x2.y;
          s1 += v23.y * x3.x; s2 += v23.y * x3.y;
        } else {
          s1 += v01.x * lds_f64(tile_s + c0 * 8u);
          s1 += v01.y * lds_f64(tile_s + c1 * 8u);
          s1 += v23.x * lds_f64(tile_s + c2 * 8u);
          s1 += v23.y * lds_f64(tile_s + c3 * 8u);
        }
      }
    }
    if (V > 1) {
#pragma unroll
      for (int o = V / 2; o >= 1; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
        if (ELEM == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
      }
    }
    if (lane == 0 && r < B.rb) {
      const int rr = __ldg(M.srow + S.rp + r);
      acc[rr * ELEM] += s1;
      if (ELEM == 2) acc[rr * ELEM + 1] += s2;
    }
  }
}

// Partial products with the staged segments streamed by TMA: thread 0 keeps
// kNST batches (values + column ids, and the segment's vector tile) in flight;
// all warps consume from shared memory.  Direct segments run first from global.
template <int ELEM>
__global__ void __launch_bounds__(kTThreads) k_tiled_tma(TiledMat M, const double* __restrict__ x,
                                                         double* __restrict__ scratch, const Ctl* ctl, int guard) {
  if (guard >= 1 && ctl->status != 4) return;
  if (guard == 2 && !ctl->accepted) return;
  extern __shared__ __align__(128) double smem[];
  const int tile_doubles = M.T * ELEM;
  double* tiles = smem;                                       // 2 * tile_doubles
  double* vals = tiles + 2 * tile_doubles;                    // kNST * kBQ * 4
  uint16_t* cols = reinterpret_cast<uint16_t*>(vals + kNST * kBQ * 4);   // kNST * kBQ * 4 (+ 8 pad)
  int32_t* rps = reinterpret_cast<int32_t*>(cols + kNST * (kBQ + 2) * 4);  // kNST * kBR
  double* acc = reinterpret_cast<double*>(rps + kNST * kBR);               // kTRows * ELEM
  __shared__ __align__(8) uint64_t full[kNST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t uses[kNST] = {0, 0, 0};   // completed phases per stage (thread 0 and consumers agree)
  for (int64_t w = blockIdx.x; w < M.nwork; w += gridDim.x) {
    const TWork W = M.work[w];
    const TChunk C = M.chunk[W.chunk];
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    // direct segments (global gathers)
    for (int s = W.s0; s < W.s1; ++s) {
      const TSeg S = M.seg[s];
      if (S.tile >= 0) continue;
      switch (S.V) {
        case 1: seg_rows<1, ELEM>(M, S, C, x, 0u, false, acc); break;
        case 2: seg_rows<2, ELEM>(M, S, C, x, 0u, false, acc); break;
        case 4: seg_rows<4, ELEM>(M, S, C, x, 0u, false, acc); break;
        case 8: seg_rows<8, ELEM>(M, S, C, x, 0u, false, acc); break;
        case 16: seg_rows<16, ELEM>(M, S, C, x, 0u, false, acc); break;
        default: seg_rows<32, ELEM>(M, S, C, x, 0u, false, acc); break;
      }
      __syncthreads();
    }
    const int nb = W.b1 - W.b0;
    auto issue = [&](int j) {
      const TBatch B = M.batch[W.b0 + j];
      const TSeg S = M.seg[B.seg];
      const int st = j % kNST;
      const int32_t qc = B.qa & ~1;                        // 16-B aligned column-id copy
      const uint32_t vbytes = (uint32_t)(B.qb - B.qa) * 32u;
      const uint32_t cbytes = (uint32_t)(((B.qb - qc + 1) & ~1) * 8);
      uint32_t tbytes = 0;
      if (B.first) {
        const int64_t base = (int64_t)S.tile * M.T;
        const int64_t len = (M.nvec - base < M.T ? M.nvec - base : M.T) * ELEM * 8;
        tbytes = (uint32_t)((len + 15) & ~15);
      }
      const int64_t r0 = (S.rp + B.ra) & ~(int64_t)3;      // 16-B aligned row-pointer slice
      const uint32_t rbytes = (uint32_t)(((S.rp + B.rb + 1 - r0) * 4 + 15) & ~15);
      mbar_expect_tx(&full[st], vbytes + cbytes + tbytes + rbytes);
      tma_load_1d(rps + (size_t)st * kBR, M.rowptr + r0, rbytes, &full[st]);
      tma_load_1d(vals + (size_t)st * kBQ * 4, M.val_s + S.nz + 4 * (int64_t)B.qa, vbytes, &full[st]);
      tma_load_1d(cols + (size_t)st * (kBQ + 2) * 4, M.col_s + S.nz + 4 * (int64_t)qc, cbytes, &full[st]);
      if (B.first)
        tma_load_1d(tiles + (size_t)(B.ord & 1) * tile_doubles, x + (int64_t)S.tile * M.T * ELEM, tbytes,
                    &full[st]);
    };
    // thread 0 issues batch j when a stage is free (j <= i + kNST) and the tile
    // buffer it opens is free: segment ordinal ord_j <= ord(oldest unfinished) + 1
    int next = 0;
    auto pump = [&](int oldest) {
      if (threadIdx.x != 0) return;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int oord = oldest < nb ? M.batch[W.b0 + oldest].ord : 0x7fffffff;
      while (next < nb && next < oldest + kNST) {
        const TBatch Bn = M.batch[W.b0 + next];
        if (Bn.first && Bn.ord > oord + 1) break;
        issue(next);
        ++next;
      }
    };
    pump(0);
    for (int i = 0; i < nb; ++i) {
      const TBatch B = M.batch[W.b0 + i];
      const int st = i % kNST;
      mbar_wait(&full[st], uses[st] & 1u);
      ++uses[st];
      const TSeg S = M.seg[B.seg];
      const uint32_t tile_s = smem_u32(tiles + (size_t)(B.ord & 1) * tile_doubles);
      const double* sv = vals + (size_t)st * kBQ * 4;
      const uint16_t* sc = cols + (size_t)st * (kBQ + 2) * 4;
      const int32_t qc = B.qa & ~1;
      const double* svb = sv - 4 * (B.qa - qc);            // values were copied from qa
      // row pointers were copied from (S.rp + ra) & ~3: index them by chunk row
      const int32_t* rpb = rps + (size_t)st * kBR - ((S.rp + B.ra) & ~(int64_t)3) + S.rp;
      switch (S.V) {
        case 1: batch_rows<1, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
        case 2: batch_rows<2, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
        case 4: batch_rows<4, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
        case 8: batch_rows<8, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
        case 16: batch_rows<16, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
        default: batch_rows<32, ELEM>(M, S, B, tile_s, svb, sc, qc, rpb, acc); break;
      }
      __syncthreads();                       // stage st (and a finished segment's tile) is free
      pump(i + 1);
    }
    double* out = scratch + C.scratch + (int64_t)W.group * C.nrows * ELEM;
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) out[i] = acc[i];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ sliced layout
// Staged segments in the sliced layout (pdcs.cu slice_segments): the quads of
// a warp block of 32/V consecutive segment rows are stored time step by time
// step, lane by lane, so the quad lane l of the block reads at step t sits at
// blkb[block] + l + 32 t.  A warp-wide LDG.256 then reads 1 KB of consecutive
// values (8 full lines) and the column-id load 256 consecutive bytes.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Asynchronous copy (LDGSTS) of vector tile `tile` into shared buffer dst.
template <int ELEM>
__device__ __forceinline__ void tile_fetch_async(const TiledMat& M, const double* __restrict__ x, int32_t tile,
                                                 double* dst) {
  const int64_t base = (int64_t)tile * M.T;
  const int64_t len = (M.nvec - base < M.T ? M.nvec - base : M.T) * ELEM;   // doubles
  const double* src = x + base * ELEM;
  const uint32_t d = smem_u32(dst);
  for (int64_t i = threadIdx.x; i < len / 2; i += blockDim.x) cp_async16(d + 16u * (uint32_t)i, src + 2 * i);
  if ((len & 1) && threadIdx.x == 0) dst[len - 1] = __ldg(src + len - 1);
}

#ifndef PDCS_SL_U2
#define PDCS_SL_U2 4                  // quads in flight per lane, pair gather (B200 sweep: 2 -> 4 is -2% / -21%)
#endif
#ifndef PDCS_SL_U1
#define PDCS_SL_U1 4                  // quads in flight per lane, single gather
#endif
#ifndef PDCS_SL_PIPE
#define PDCS_SL_PIPE 0                // > 0: software-pipelined loop, this many quads per stage
#endif
// One staged segment, warp per block of 32/V rows.  Blocks go to warps in
// snake order (rows are sorted longest first, so this balances the warps);
// the next block's row lengths, base and output rows are loaded before the
// current block's data loop, so the only exposed latency is the data's.
template <int V, int ELEM>
__device__ __forceinline__ void sliced_blocks(const TiledMat& M, const TSeg& S, int32_t nrows, uint32_t xs_s,
                                              double* acc) {
  constexpr int RPW = 32 / V;
  constexpr int U = ELEM == 2 ? PDCS_SL_U2 : PDCS_SL_U1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int a = lane / V, l = lane % V;
  const int32_t* rp = M.rowptr + S.rp;
  const uint16_t* srow = M.srow + S.rp;
  const int32_t* bb = M.blkb + S.bb;
  const double* val = M.val_s + S.nz;
  const uint16_t* col = M.col_s + S.nz;
  const int nblk = (nrows + RPW - 1) / RPW;
  auto blk_of = [&](int i) { return i * nw + ((i & 1) ? nw - 1 - warp : warp); };
  auto meta = [&](int blk, int32_t& nq, int32_t& base, int& rr) {
    nq = 0; base = 0; rr = -1;
    if (blk < nblk) {
      const int pos = blk * RPW + a;
      base = __ldg(bb + blk);
      if (pos < nrows) { nq = __ldg(rp + pos + 1) - __ldg(rp + pos); rr = __ldg(srow + pos); }
    }
  };
  int i = 0, blk = blk_of(0);
  int32_t nq, base;
  int rr;
  meta(blk, nq, base, rr);
  while (blk < nblk) {
    const int blk2 = blk_of(i + 1);
    int32_t nq2, base2;
    int rr2;
    meta(blk2, nq2, base2, rr2);
    const int32_t nt = nq > l ? (nq - l + V - 1) / V : 0;     // quads of this lane
    const int32_t tmax = (int32_t)__reduce_max_sync(0xffffffffu, (unsigned)nt);
    const double* vp = val + 4 * ((int64_t)base + lane);
    const uint16_t* cp = col + 4 * ((int64_t)base + lane);
    double s1 = 0.0, s2 = 0.0;
#if PDCS_SL_PIPE
    // software-pipelined: the next PU quads' loads are in flight while the
    // current ones are gathered and summed (same entry order, same sums)
    {
      constexpr int PU = PDCS_SL_PIPE;
      double q[PU][4];
      uint2 c[PU];
#define PDCS_SL_FETCH(TT, QQ, CC)                                             \
  _Pragma("unroll") for (int u = 0; u < PU; ++u) {                            \
    if ((TT) + u < nt) {                                                      \
      const double4 v_ = ld_stream4(vp + 128 * (int64_t)((TT) + u));          \
      CC[u] = ld_stream_u2(cp + 128 * (int64_t)((TT) + u));                   \
      QQ[u][0] = v_.x; QQ[u][1] = v_.y; QQ[u][2] = v_.z; QQ[u][3] = v_.w;     \
    } else {                                                                  \
      CC[u] = make_uint2(0u, 0u);                                             \
      QQ[u][0] = QQ[u][1] = QQ[u][2] = QQ[u][3] = 0.0;                        \
    }                                                                         \
  }
      PDCS_SL_FETCH(0, q, c)
      for (int32_t t0 = 0; t0 < tmax; t0 += PU) {
        double qn[PU][4];
        uint2 cn[PU];
        PDCS_SL_FETCH(t0 + PU, qn, cn)
#pragma unroll
        for (int u = 0; u < PU; ++u)
          if (t0 + u < nt) {
            const uint32_t cc[4] = {c[u].x & 0xffffu, c[u].x >> 16, c[u].y & 0xffffu, c[u].y >> 16};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (ELEM == 2) {
                const double2 v = lds_v2(xs_s + cc[k] * 16u);
                s1 += q[u][k] * v.x;
                s2 += q[u][k] * v.y;
              } else {
                s1 += q[u][k] * lds_f64(xs_s + cc[k] * 8u);
              }
            }
          }
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          c[u] = cn[u];
#pragma unroll
          for (int k = 0; k < 4; ++k) q[u][k] = qn[u][k];
        }
      }
#undef PDCS_SL_FETCH
    }
#else
    for (int32_t t0 = 0; t0 < tmax; t0 += U) {
      double q[U][4];
      uint2 c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < nt) {
          const double4 v = ld_stream4(vp + 128 * (int64_t)(t0 + u));
          c[u] = ld_stream_u2(cp + 128 * (int64_t)(t0 + u));
          q[u][0] = v.x; q[u][1] = v.y; q[u][2] = v.z; q[u][3] = v.w;
        } else {
          c[u] = make_uint2(0u, 0u);
          q[u][0] = q[u][1] = q[u][2] = q[u][3] = 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u < nt) {
          const uint32_t cc[4] = {c[u].x & 0xffffu, c[u].x >> 16, c[u].y & 0xffffu, c[u].y >> 16};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (ELEM == 2) {
              const double2 v = lds_v2(xs_s + cc[k] * 16u);
              s1 += q[u][k] * v.x;
              s2 += q[u][k] * v.y;
            } else {
              s1 += q[u][k] * lds_f64(xs_s + cc[k] * 8u);
            }
          }
        }
    }
#endif
    if (V > 1) {
#pragma unroll
      for (int o = V / 2; o >= 1; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
        if (ELEM == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
      }
    }
    if (l == 0 && rr >= 0) {
      acc[rr * ELEM] += s1;
      if (ELEM == 2) acc[rr * ELEM + 1] += s2;
    }
    blk = blk2; nq = nq2; base = base2; rr = rr2;
    ++i;
  }
}

__device__ __forceinline__ int32_t next_staged(const TiledMat& M, int32_t s, int32_t e) {
  for (; s < e; ++s)
    if (M.seg[s].tile >= 0) return s;
  return -1;
}

// Partial products, sliced layout.  The vector tile of the next staged segment
// (in this work item, else in the CTA's next item) is copied asynchronously
// into the second shared buffer while the current segment runs.
#ifndef PDCS_TS_MINB1
#define PDCS_TS_MINB1 2               // k_tiled_sliced<1>: 64 registers (40 spills)
#endif
// EpiNone: the partial kernel alone (k_tiled_combine runs the epilogue).
struct EpiNone {
  static constexpr int NA = 1;
  static constexpr int NX = 1;
  __device__ void init(const Ctl*) {}
  __device__ bool active() const { return true; }
  __device__ void row(int64_t, double, double, Acc<1>&) {}
};

// Fused combine (Epi != EpiNone): the CTA that completes a chunk's last work
// item (per-chunk arrival counter, reset by that CTA) sums the chunk's group
// partials in k_tiled_combine's order and runs the epilogue on its rows; the
// epilogue's accumulators go to slot slot0 + chunk.  A chunk of one work item
// takes its sums straight from shared memory.  Same sums, bit for bit, as
// partial + combine; one launch and one scratch round trip fewer.  Chunks of
// >= kCombWideG groups (Lasso K^T's long rows: ~150) would leave one CTA
// reading ~1 MB of partials at the end of the sweep: their partials are
// written as before and a combine launch over their items only follows.
template <class Epi, int ELEM>
__device__ __forceinline__ void chunk_epilogue(const TChunk& C, const double* __restrict__ src, const double* acc,
                                               Epi& epi, double* part, int64_t slot) {
  Acc<Epi::NA> a;
  a.zero();
  if (!src) {                                        // one group: the sums are in shared memory
    for (int r = threadIdx.x; r < C.nrows; r += blockDim.x) {
      double s1 = 0.0, s2 = 0.0;
      s1 += acc[r * ELEM];
      if (ELEM == 2) s2 += acc[r * ELEM + 1];
      epi.row(C.row0 + r, s1, s2, a);
    }
  } else {                                           // groups added in order (ngroups < kCombWideG)
    for (int r = threadIdx.x; r < C.nrows; r += blockDim.x) {
      double s1 = 0.0, s2 = 0.0;
      for (int g = 0; g < C.ngroups; ++g) {
        s1 += __ldcg(src + ((int64_t)g * C.nrows + r) * ELEM);
        if (ELEM == 2) s2 += __ldcg(src + ((int64_t)g * C.nrows + r) * ELEM + 1);
      }
      epi.row(C.row0 + r, s1, s2, a);
    }
  }
  if (part) {                                        // fixed-order CTA reduction (up to 32 warps)
    __shared__ double red[Epi::NA][32];
#pragma unroll
    for (int i = 0; i < Epi::NA; ++i) {
      double v = a.v[i];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < Epi::NA) {
      double v = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
      part[slot * Epi::NA + threadIdx.x] = v;
    }
    __syncthreads();
  }
}

template <int ELEM, class Epi = EpiNone>
__global__ void __launch_bounds__(kTThreads, ELEM == 1 ? PDCS_TS_MINB1 : PDCS_TP_MINB)
    k_tiled_sliced(TiledMat M, const double* __restrict__ x, double* __restrict__ scratch, const Ctl* ctl, int guard,
                   Epi epi = Epi(), int32_t* chunk_cnt = nullptr, double* part = nullptr, int64_t slot0 = 0) {
  constexpr bool kFused = !std::is_same<Epi, EpiNone>::value;
  if (guard >= 1 && ctl->status != 4) return;
  if (guard == 2 && !ctl->accepted) return;
  if (kFused) {
    epi.init(ctl);
    if (!epi.active()) return;
  }
  extern __shared__ __align__(128) double smem[];
  const int64_t TE = (int64_t)M.T * ELEM;
  double* tiles = smem;                              // 2 buffers of T * ELEM doubles
  double* acc = smem + 2 * TE;                       // kTRows * ELEM doubles
  int buf = 0;                                       // buffer of the tile in flight
  int32_t inflight = -1;                             // segment whose tile is in flight
  if (blockIdx.x < M.nwork) {
    const TWork W = M.work[blockIdx.x];
    inflight = next_staged(M, W.s0, W.s1);
    if (inflight >= 0) tile_fetch_async<ELEM>(M, x, M.seg[inflight].tile, tiles + buf * TE);
  }
  for (int64_t w = blockIdx.x; w < M.nwork; w += gridDim.x) {
    const TWork W = M.work[w];
    const TChunk C = M.chunk[W.chunk];
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    for (int s = W.s0; s < W.s1; ++s) {
      const TSeg S = M.seg[s];
      if (S.tile >= 0) {
        if (s != inflight) tile_fetch_async<ELEM>(M, x, S.tile, tiles + buf * TE);
        cp_async_wait_all();
        __syncthreads();                               // tile visible; the other buffer is free
        const uint32_t xs_s = smem_u32(tiles + buf * TE);
        buf ^= 1;
        inflight = next_staged(M, s + 1, W.s1);
        if (inflight < 0 && w + gridDim.x < M.nwork) {
          const TWork W2 = M.work[w + gridDim.x];
          inflight = next_staged(M, W2.s0, W2.s1);
        }
        if (inflight >= 0) tile_fetch_async<ELEM>(M, x, M.seg[inflight].tile, tiles + buf * TE);
#define PDCS_SLB sliced_blocks
        switch (S.V) {
          case 1: PDCS_SLB<1, ELEM>(M, S, C.nrows, xs_s, acc); break;
          case 2: PDCS_SLB<2, ELEM>(M, S, C.nrows, xs_s, acc); break;
          case 4: PDCS_SLB<4, ELEM>(M, S, C.nrows, xs_s, acc); break;
          case 8: PDCS_SLB<8, ELEM>(M, S, C.nrows, xs_s, acc); break;
          case 16: PDCS_SLB<16, ELEM>(M, S, C.nrows, xs_s, acc); break;
          default: PDCS_SLB<32, ELEM>(M, S, C.nrows, xs_s, acc); break;
        }
      } else {
        switch (S.V) {
          case 1: seg_rows<1, ELEM>(M, S, C, x, 0u, false, acc); break;
          case 2: seg_rows<2, ELEM>(M, S, C, x, 0u, false, acc); break;
          case 4: seg_rows<4, ELEM>(M, S, C, x, 0u, false, acc); break;
          case 8: seg_rows<8, ELEM>(M, S, C, x, 0u, false, acc); break;
          case 16: seg_rows<16, ELEM>(M, S, C, x, 0u, false, acc); break;
          default: seg_rows<32, ELEM>(M, S, C, x, 0u, false, acc); break;
        }
      }
      __syncthreads();                                 // acc rows are shared across segments
    }
    double* out = scratch + C.scratch + (int64_t)W.group * C.nrows * ELEM;
    if (!kFused || C.ngroups >= kCombWideG) {
      // partials only (chunks of many groups: k_tiled_combine over their items)
      for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) out[i] = acc[i];
      __syncthreads();
    } else if (C.ngroups == 1) {
      chunk_epilogue<Epi, ELEM>(C, nullptr, acc, epi, part, slot0 + W.chunk);
      __syncthreads();
    } else {
      __shared__ int s_last;
      for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) __stcg(out + i, acc[i]);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        s_last = atomicAdd(chunk_cnt + W.chunk, 1) == C.ngroups - 1;
        if (s_last) chunk_cnt[W.chunk] = 0;          // ready for the next launch
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        chunk_epilogue<Epi, ELEM>(C, scratch + C.scratch, acc, epi, part, slot0 + W.chunk);
      }
      __syncthreads();
    }
  }
  cp_async_wait_all();
}

// ---- Deferred build on the device -------------------------
// The host builds the segments' unbalanced row-major quads; these two kernels
// do what balance_banks and slice_segments (pdcs.cu) do on the host, one
// thread per warp block, with the same arithmetic and tie-breaks, so the final
// layout is bit-identical (tests/test_tiled_layout.py, device check).
//
// Bank balancing of one warp block (balance_banks): at every time step each
// lane reads one quad, and position k of those quads is one warp-wide
// ld.shared served in 32/G phases of G lanes; per phase, lanes with the fewest
// choices go first and take the free bank group with the most entries left.
// pcol / pperm: the pre layout (read); bcol / bperm: bucket scratch at the same
// offsets; ncol / nperm: the balanced quads at the same offsets (written).
// Bank balancing, one WARP per warp block (the solver's device builds).  The
// same greedy as balance_banks (pdcs.cu), decision for decision:
// lane a < R owns row a's state (group mask, entries left, slots left, quads);
// the per-(row, group) bucket counts and the block's per-group totals live in
// shared memory.  Per phase the units (schedule lanes with a quad at this step)
// are taken in (popcount of the row's groups at the phase start, lane) order,
// one at a time: the owner's current state is broadcast and every lane computes
// the same choice (the free group with the most entries left, lowest on ties;
// a forced conflict when the row has no pad to spare; else a pad).  Each unit's
// lane then moves its entry: bucket (a, g) is consumed from the back, as on the
// host.  Pads re-read the first unit's column (0 if that unit was a pad).
constexpr int kBalWarps = 4;                          // warps per CTA of k_tile_balance_w
constexpr int kBalRG = 32 * 16;                       // max rows x groups of a warp block
__global__ void __launch_bounds__(32 * kBalWarps)
    k_tile_balance_w(const TDefer* __restrict__ dseg, const int2* __restrict__ dblk, int64_t nblk, int elem,
                     const int32_t* __restrict__ rowptr, const uint16_t* __restrict__ pcol,
                     const int32_t* __restrict__ pperm, uint16_t* __restrict__ bcol, int32_t* __restrict__ bperm,
                     uint16_t* __restrict__ ncol, int32_t* __restrict__ nperm) {
  __shared__ int32_t s_cnt[kBalWarps][kBalRG];        // bucket sizes, then entries left per bucket
  __shared__ int32_t s_start[kBalWarps][kBalRG + 1];  // bucket starts (exclusive prefix, row-major)
  __shared__ int32_t s_cur[kBalWarps][kBalRG];        // fill cursors
  __shared__ int32_t s_rem[kBalWarps][16];            // entries left per group in the block
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  int32_t* cnt = s_cnt[w];
  int32_t* bst = s_start[w];
  int32_t* cur = s_cur[w];
  int32_t* rem = s_rem[w];
  const int G = elem == 2 ? 8 : 16;
  const int64_t nwarps = (int64_t)gridDim.x * kBalWarps;
  for (int64_t it = (int64_t)blockIdx.x * kBalWarps + w; it < nblk; it += nwarps) {
    const int2 db = dblk[it];
    const TDefer S = dseg[db.x];
    const int V = S.V, rpw = 32 / V;
    const int32_t* rp = rowptr + S.rp;
    const int32_t i0 = db.y * rpw;
    const int R = min(rpw, S.nr - i0);
    const uint16_t* cols = pcol + S.src;
    const int32_t* perm = pperm + S.src;
    const int64_t bbase = S.src + 4 * (int64_t)rp[i0];
    const int RG = R * G;
    // ---- row state (owner lanes)
    int32_t q0 = 0, nq = 0;
    if (lane < R) { q0 = rp[i0 + lane]; nq = rp[i0 + lane + 1] - q0; }
    const int32_t tmax = (int32_t)__reduce_max_sync(FULL, (unsigned)((nq + V - 1) / V));
    for (int z = lane; z < RG; z += 32) { cnt[z] = 0; cur[z] = 0; }
    if (lane < 16) rem[lane] = 0;
    __syncwarp();
    // ---- bucket sizes (integer counts: order-free)
    for (int a = 0; a < R; ++a) {
      const int32_t qa = __shfl_sync(FULL, q0, a), na = __shfl_sync(FULL, nq, a);
      for (int64_t e = 4 * (int64_t)qa + lane; e < 4 * (int64_t)(qa + na); e += 32)
        if (perm[e] >= 0) {
          const int g = cols[e] % G;
          atomicAdd(cnt + a * G + g, 1);
          atomicAdd(rem + g, 1);
        }
    }
    __syncwarp();
    // ---- bucket starts: exclusive prefix over (row, group), row-major
    {
      const int per = (RG + 31) / 32;
      const int z0 = min(RG, lane * per), z1 = min(RG, z0 + per);
      int32_t loc = 0;
      for (int z = z0; z < z1; ++z) loc += cnt[z];
      int32_t inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
      }
      int32_t run = inc - loc;
      for (int z = z0; z < z1; ++z) { bst[z] = run; run += cnt[z]; }
      if (lane == 31) bst[RG] = inc;
    }
    __syncwarp();
    // ---- buckets filled in entry order (stable within a bucket)
    for (int a = 0; a < R; ++a) {
      const int32_t qa = __shfl_sync(FULL, q0, a), na = __shfl_sync(FULL, nq, a);
      for (int64_t e0 = 4 * (int64_t)qa; e0 < 4 * (int64_t)(qa + na); e0 += 32) {
        const int64_t e = e0 + lane;
        const bool ok = e < 4 * (int64_t)(qa + na) && perm[e] >= 0;
        const int g = ok ? cols[e] % G : -1 - lane;
        const unsigned same = __match_any_sync(FULL, g);
        if (ok) {
          const int bi = a * G + g;
          const int32_t z = bst[bi] + cur[bi] + __popc(same & ((1u << lane) - 1u));
          bcol[bbase + z] = cols[e];
          bperm[bbase + z] = perm[e];
        }
        __syncwarp();
        if (ok && lane == 31 - __clz(same)) cur[a * G + g] += __popc(same);
        __syncwarp();
      }
    }
    // ---- owner state: group mask, entries left, slots left
    uint32_t mask = 0;
    int32_t left = 0, slots = 4 * nq;
    if (lane < R)
      for (int g = 0; g < G; ++g) {
        const int32_t c = cnt[lane * G + g];
        if (c) mask |= 1u << g;
        left += c;
      }
    __syncwarp();
    // ---- the greedy, phase by phase
    for (int32_t t = 0; t < tmax; ++t)
      for (int k = 0; k < 4; ++k)
        for (int ph = 0; ph < 32 / G; ++ph) {
          const int a = lane / V, l = lane % V;
          const bool inph = lane >= ph * G && lane < ph * G + G;
          const int32_t na = __shfl_sync(FULL, nq, a < 32 ? a : 0);
          const int32_t qa = __shfl_sync(FULL, q0, a < 32 ? a : 0);
          const uint32_t m0 = __shfl_sync(FULL, mask, a < 32 ? a : 0);
          const bool unit = inph && a < R && l + t * V < na;
          unsigned key = unit ? ((unsigned)__popc(m0) << 5) | (unsigned)lane : 0xffffffffu;
          uint32_t used = 0;
          int32_t z_src = -1;                          // this lane's entry (bucket index), -1: pad
          int first = -1, first_pad = 0;               // first unit processed; whether it was a pad
          for (;;) {
            const unsigned kmin = __reduce_min_sync(FULL, key);
            if (kmin == 0xffffffffu) break;
            const int wl = (int)(kmin & 31u);
            const int aw = wl / V;
            const uint32_t m = __shfl_sync(FULL, mask, aw);
            const int32_t lf = __shfl_sync(FULL, left, aw);
            const int32_t sl = __shfl_sync(FULL, slots, aw);
            const uint32_t avail = m & ~used;
            const uint32_t from = avail ? avail : ((lf > 0 && sl == lf) ? m : 0u);
            unsigned cand = 0;
            if (lane < G && ((from >> lane) & 1u)) cand = ((unsigned)rem[lane] << 5) | (unsigned)(31 - lane) | 0x80000000u;
            const unsigned best = __reduce_max_sync(FULL, cand);
            const int g = best ? 31 - (int)(best & 31u) : -1;
            if (first < 0) { first = wl; first_pad = g < 0; }
            if (g >= 0) {
              const int bi = aw * G + g;
              int32_t nleft = 0;
              if (lane == aw) {
                nleft = --cnt[bi];
                if (nleft == 0) mask &= ~(1u << g);
                --left;
              }
              nleft = __shfl_sync(FULL, nleft, aw);
              if (lane == wl) z_src = bst[bi] + nleft;
              if (lane == 0) --rem[g];
              used |= 1u << g;
            }
            if (lane == aw) --slots;
            if (lane == wl) key = 0xffffffffu;
            __syncwarp();
          }
          // move the entries (loads issued for every unit together)
          uint16_t c = 0;
          int32_t pv = -1;
          if (unit && z_src >= 0) { c = bcol[bbase + z_src]; pv = bperm[bbase + z_src]; }
          const uint16_t fc = (uint16_t)__shfl_sync(FULL, (int)c, first >= 0 ? first : 0);
          if (unit) {
            const int64_t slot = 4 * (int64_t)(qa + l + t * V) + k;
            if (z_src >= 0) { ncol[S.src + slot] = c; nperm[S.src + slot] = pv; }
            else { ncol[S.src + slot] = first_pad ? (uint16_t)0 : fc; nperm[S.src + slot] = -1; }
          }
        }
    __syncwarp();
  }
}

// Sliced re-layout of one warp block (slice_segments / quad_slot): quad j of
// block row a goes to blkb[block] + a V + j % V + 32 (j / V).
__global__ void k_tile_slice(const TDefer* __restrict__ dseg, const int2* __restrict__ dblk, int64_t nblk,
                             const int32_t* __restrict__ rowptr, const int32_t* __restrict__ blkb,
                             const uint16_t* __restrict__ ncol, const int32_t* __restrict__ nperm,
                             uint16_t* __restrict__ col_s, int32_t* __restrict__ perm_s) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= nblk) return;
  const int2 db = dblk[it];
  const TDefer S = dseg[db.x];
  const int V = S.V, rpw = 32 / V;
  const int32_t* rp = rowptr + S.rp;
  const int32_t i0 = db.y * rpw;
  const int R = min(rpw, S.nr - i0);
  const int64_t base = blkb[S.bb + db.y];
  for (int a = 0; a < R; ++a) {
    const int32_t pos = i0 + a, nq = rp[pos + 1] - rp[pos];
    for (int32_t j = 0; j < nq; ++j) {
      const int64_t to = S.dst + 4 * (base + a * V + j % V + 32 * (int64_t)(j / V));
      const int64_t from = S.src + 4 * ((int64_t)rp[pos] + j);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        col_s[to + k] = ncol[from + k];
        perm_s[to + k] = nperm[from + k];
      }
    }
  }
}

// ---- Device structure build -------------------------------
// The column-tiled layout built from a device CSR without the entries passing
// through the host: k_tile_hist counts the entries of every (chunk, tile),
// the host picks the staged tiles per chunk; k_tile_rowcnt counts every row's
// entries per segment, the host orders the rows and lays out the segments
// (only O(segments x rows) work); k_tile_fill writes the column ids and CSR
// positions of every entry at their slots of the unbalanced row-major quads
// (staged segments) or of col_d (direct).  k_tile_balance_w / k_tile_slice then
// finish as in the deferred build.  Same layout, bit for bit, as build_tiled
// (tests/test_tiled_layout.py, pdcs_tiled_devbuild_check).
struct TBChunk {
  int64_t sbase;      // global index of the chunk's first segment
  int32_t soff, nst;  // its staged tiles, ascending: stl[soff, soff + nst)
  int32_t direct;     // 1: the chunk's segment 0 is its direct segment
  int32_t pad;
};
struct TFillSeg {
  int64_t off;        // staged: first entry of its pre quads; direct: first entry in col_d
  int64_t rp;         // its row pointers (and posof)
  int32_t tile;       // -1: direct
  int32_t nr;         // rows of its chunk
};

// Chunk-local segment of an entry in tile t: the staged tile's slot, else the
// direct segment (index 0; it exists whenever a touched tile is not staged).
__device__ __forceinline__ int tb_seg_of(const TBChunk& C, const int32_t* __restrict__ stl, int32_t t) {
  int lo = 0, hi = C.nst;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(stl + C.soff + mid) < t) lo = mid + 1; else hi = mid;
  }
  return (lo < C.nst && __ldg(stl + C.soff + lo) == t) ? C.direct + lo : 0;
}

// Entries per (chunk, tile): out[(chunk - c0) * ntiles + t] (zeroed by the
// caller).  One CTA per item = a range of at most 65536 entries of one chunk
// (a chunk of 1024 long rows holds ~1e7 entries on Lasso's K^T: one CTA per
// chunk had taken 27 ms), a shared-memory histogram when ntiles fits, added
// into the chunk's row of out.
struct THistItem {
  int64_t chunk, p0, p1;
};
__global__ void k_tile_hist(const int32_t* __restrict__ col, const THistItem* __restrict__ items, int32_t T,
                            int64_t ntiles, int64_t c0, int32_t* __restrict__ out, int use_smem) {
  extern __shared__ int32_t hist[];
  const THistItem I = items[blockIdx.x];
  int32_t* dst = out + (I.chunk - c0) * ntiles;
  if (use_smem) {
    for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x) hist[t] = 0;
    __syncthreads();
  }
  // entries are sorted by column within a row, so neighbouring lanes mostly
  // share a tile: one atomic per (warp step, tile) instead of one per entry
  for (int64_t q0 = I.p0; q0 < I.p1; q0 += blockDim.x) {
    const int64_t p = q0 + threadIdx.x;
    const int32_t t = p < I.p1 ? __ldg(col + p) / T : -1 - (int32_t)(threadIdx.x & 31);
    const unsigned same = __match_any_sync(0xffffffffu, t);
    if (p < I.p1 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(use_smem ? hist + t : dst + t, __popc(same));
  }
  if (use_smem) {
    __syncthreads();
    for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x)
      if (hist[t]) atomicAdd(dst + t, hist[t]);
  }
}

// Entries of every row per segment: rc[(sbase + k) * kTRows + i] (zeroed by
// the caller).  One warp per row; lanes of one segment add once.
__global__ void k_tile_rowcnt(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col, int64_t rows,
                              int32_t T, const TBChunk* __restrict__ cb, const int32_t* __restrict__ stl,
                              int32_t* __restrict__ rc) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarp) {
    const TBChunk C = cb[r / kTRows];
    const int64_t i = r % kTRows;
    const int32_t b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    for (int32_t p0 = b; p0 < e; p0 += 32) {
      const int32_t p = p0 + lane;
      const bool ok = p < e;
      const int k = ok ? tb_seg_of(C, stl, __ldg(col + p) / T) : -1 - lane;
      const unsigned same = __match_any_sync(0xffffffffu, k);
      if (ok && lane == __ffs(same) - 1) atomicAdd(rc + (C.sbase + k) * kTRows + i, __popc(same));
    }
  }
}

// Inverse of every segment's row order: posof[rp + srow[rp + pos]] = pos.
__global__ void k_tile_posof(const TFillSeg* __restrict__ fs, int64_t nseg, const uint16_t* __restrict__ srow,
                             uint16_t* __restrict__ posof) {
  for (int64_t g = blockIdx.x; g < nseg; g += gridDim.x) {
    const TFillSeg S = fs[g];
    for (int pos = threadIdx.x; pos < S.nr; pos += blockDim.x) posof[S.rp + srow[S.rp + pos]] = (uint16_t)pos;
  }
}

// Column id and CSR position of every entry at its slot: entry f of row i in
// segment k (f counted in CSR order within the row) goes to unit
// rowptr[rp + posof[rp + i]] of the segment (quads for staged segments).
__global__ void k_tile_fill(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col, int64_t rows,
                            int32_t T, const TBChunk* __restrict__ cb, const int32_t* __restrict__ stl,
                            const TFillSeg* __restrict__ fs, const int32_t* __restrict__ rowptr,
                            const uint16_t* __restrict__ posof, uint16_t* __restrict__ pcol,
                            int32_t* __restrict__ pperm, int32_t* __restrict__ col_d, int32_t* __restrict__ perm_d) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarp) {
    const TBChunk C = cb[r / kTRows];
    const int64_t i = r % kTRows;
    const int32_t b = __ldg(ptr + r), e = __ldg(ptr + r + 1);
    int32_t carry_t = -1, carry_start = 0, carry_d = 0;
    for (int32_t p0 = b; p0 < e; p0 += 32) {
      const int32_t p = p0 + lane;
      const bool ok = p < e;
      const unsigned act = __ballot_sync(0xffffffffu, ok);
      const int32_t cv = ok ? __ldg(col + p) : 0;
      const int32_t t = ok ? cv / T : -1 - lane;
      const int k = ok ? tb_seg_of(C, stl, t) : 0;
      const TFillSeg S = fs[C.sbase + k];
      const bool staged = ok && S.tile >= 0;
      // staged: position within the row's run of tile t (columns ascend, so a
      // tile's entries are contiguous in the row)
      const unsigned same = __match_any_sync(0xffffffffu, t);
      const int lead = __ffs(same) - 1;
      const int32_t start = (lead == 0 && t == carry_t) ? carry_start : p0 + lead;
      // direct: rank among the row's direct entries
      const unsigned dm = __ballot_sync(0xffffffffu, ok && !staged);
      const int32_t fd = carry_d + __popc(dm & ((1u << lane) - 1u));
      if (ok) {
        const int32_t unit = __ldg(rowptr + S.rp + __ldg(posof + S.rp + i));
        if (staged) {
          const int64_t q = S.off + 4 * (int64_t)unit + (p - start);
          pcol[q] = (uint16_t)(cv - t * T);
          pperm[q] = p;
        } else {
          const int64_t q = S.off + unit + fd;
          col_d[q] = cv;
          perm_d[q] = p;
        }
      }
      const int last = 31 - __clz(act);
      carry_t = __shfl_sync(0xffffffffu, t, last);
      carry_start = __shfl_sync(0xffffffffu, start, last);
      carry_d += __popc(dm);
    }
  }
}

// Sum the partials of every row (fixed order) and run the fused epilogue.
// Items of chunks with few groups: one thread per row, the groups summed in
// order with loads batched 8 deep.  Items of chunks with many groups (the long
// rows of Lasso's K^T have ~150 per chunk; one thread per row serialised ~20
// dependent load batches and made the tail of the kernel): kCombLanes lanes per
// row, lane l summing groups l, l+8, ..., then a fixed shuffle tree.  Both
// orders are fixed, so results are reproducible run to run.
template <class Epi, int ELEM>
__global__ void __launch_bounds__(kThreads) k_tiled_combine(TiledMat M, const double* __restrict__ scratch,
                                                            Epi epi, const Ctl* ctl, double* part,
                                                            int64_t slot0) {
  epi.init(ctl);
  if (!epi.active()) return;
  Acc<Epi::NA> acc;
  acc.zero();
  for (int64_t it = blockIdx.x; it < M.ncitem; it += gridDim.x) {
    const TCItem I = M.citem[it];
    const TChunk C = M.chunk[I.chunk];
    const double* src = scratch + C.scratch;
    if (C.ngroups <= kCombNarrowG) {
      // the common case (chunks of a few work items): the item is
      // kCombRowsNarrow rows, kCombRowsNarrow / blockDim per thread, every
      // partial load of the thread issued before the first epilogue
      constexpr int RPT = kCombRowsNarrow / kThreads;
      double u1[RPT][kCombNarrowG], u2[RPT][kCombNarrowG];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int r = I.r0 + threadIdx.x + k * kThreads;
#pragma unroll
        for (int g = 0; g < kCombNarrowG; ++g) {
          const bool ok = r < C.nrows && g < C.ngroups;
          u1[k][g] = ok ? src[((int64_t)g * C.nrows + r) * ELEM] : 0.0;
          u2[k][g] = ok && ELEM == 2 ? src[((int64_t)g * C.nrows + r) * ELEM + 1] : 0.0;
        }
      }
      double s1[RPT], s2[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        s1[k] = 0.0;
        s2[k] = 0.0;
#pragma unroll
        for (int g = 0; g < kCombNarrowG; ++g) {       // groups added in order (zeros past the end)
          if (g < C.ngroups) { s1[k] += u1[k][g]; s2[k] += u2[k][g]; }
        }
      }
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int r = I.r0 + threadIdx.x + k * kThreads;
        if (r < C.nrows) epi.row(C.row0 + r, s1[k], s2[k], acc);
      }
    } else if (C.ngroups < kCombWideG) {
      const int r = I.r0 + threadIdx.x;
      if (r < C.nrows) {
        double s1 = 0.0, s2 = 0.0;
        int g = 0;
        for (; g + 8 <= C.ngroups; g += 8) {
          double u1[8], u2[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            u1[k] = src[((int64_t)(g + k) * C.nrows + r) * ELEM];
            if (ELEM == 2) u2[k] = src[((int64_t)(g + k) * C.nrows + r) * ELEM + 1];
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            s1 += u1[k];
            if (ELEM == 2) s2 += u2[k];
          }
        }
        for (; g < C.ngroups; ++g) {
          s1 += src[((int64_t)g * C.nrows + r) * ELEM];
          if (ELEM == 2) s2 += src[((int64_t)g * C.nrows + r) * ELEM + 1];
        }
        epi.row(C.row0 + r, s1, s2, acc);
      }
    } else {
      const int lane = threadIdx.x % kCombLanes;
      const int r = I.r0 + threadIdx.x / kCombLanes;
      double s1 = 0.0, s2 = 0.0;
      if (r < C.nrows) {
        int g = lane;
        for (; g + 3 * kCombLanes < C.ngroups; g += 4 * kCombLanes) {
          double u1[4], u2[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            u1[k] = src[((int64_t)(g + k * kCombLanes) * C.nrows + r) * ELEM];
            if (ELEM == 2) u2[k] = src[((int64_t)(g + k * kCombLanes) * C.nrows + r) * ELEM + 1];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            s1 += u1[k];
            if (ELEM == 2) s2 += u2[k];
          }
        }
        for (; g < C.ngroups; g += kCombLanes) {
          s1 += src[((int64_t)g * C.nrows + r) * ELEM];
          if (ELEM == 2) s2 += src[((int64_t)g * C.nrows + r) * ELEM + 1];
        }
      }
#pragma unroll
      for (int o = kCombLanes / 2; o >= 1; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o, kCombLanes);
        if (ELEM == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, kCombLanes);
      }
      if (lane == 0 && r < C.nrows) epi.row(C.row0 + r, s1, s2, acc);
    }
  }
  if (part) cta_write_partials<Epi::NA>(acc, part, slot0 + blockIdx.x);
}

}  // namespace pdcs
