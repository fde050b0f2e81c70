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
// (tile-local uint16 column ids, 10 bytes per nonzero instead of 12); the rest
// of a chunk's entries form one *direct segment* (int32 global ids, gathered
// from L2).  Each segment is a small CSR over the chunk's rows.  A work item is
// (chunk, group of consecutive segments); it stages each tile in shared memory,
// accumulates per-row partial dot products in shared memory and writes them to
// a scratch buffer.  The combine kernel sums a row's partials in a fixed order
// and applies the fused epilogue (dual update / Halpern step), so results are
// deterministic.
#pragma once
#include "spmv.cuh"

namespace pdcs {

constexpr int kTRows = 1024;          // rows per chunk (shared accumulator size)
constexpr int kTThreads = 512;        // CTA size of the partial kernel
constexpr int kTileBytes = 65536;     // one vector tile in shared memory

struct TSeg {
  int32_t tile;      // >= 0: staged tile index; -1: direct segment
  int32_t V;         // lanes per row (1, 2, 4, 8, 16, 32)
  int64_t rp;        // offset of the segment's row pointers (nrows + 1 entries)
  int64_t nz;        // offset of the segment's entries in its pool
};
struct TChunk {
  int64_t row0;
  int32_t nrows;
  int32_t ngroups;
  int64_t scratch;   // offset (in doubles) of the chunk's partials: ngroups * nrows * ELEM
};
struct TWork {
  int32_t chunk, group, s0, s1;
};
struct TiledMat {
  int64_t m = 0, nvec = 0, nwork = 0, nchunk = 0;
  int32_t T = 0, elem = 1;
  const TWork* work = nullptr;
  const TChunk* chunk = nullptr;
  const TSeg* seg = nullptr;
  const int32_t* rowptr = nullptr;
  const double* val_s = nullptr;
  const uint16_t* col_s = nullptr;
  const double* val_d = nullptr;
  const int32_t* col_d = nullptr;
};

// Dot of one segment row with V lanes; xs is the gathered source (shared tile or
// global vector), ELEM 1 or 2 (interleaved pairs).
template <int V, int ELEM, bool STAGED>
__device__ __forceinline__ void seg_row_dot(const double* __restrict__ val, const uint16_t* __restrict__ c16,
                                            const int32_t* __restrict__ c32, const double* xs, int32_t b,
                                            int32_t e, int lane, double& s1, double& s2) {
  constexpr int U = 4;
  s1 = 0.0;
  s2 = 0.0;
  int32_t p = b + lane;
  for (; p + (U - 1) * V < e; p += U * V) {
    int32_t c[U];
    double a[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      a[k] = ld_stream(val + p + k * V);
      c[k] = STAGED ? (int32_t)__ldg(c16 + p + k * V) : ld_stream(c32 + p + k * V);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (ELEM == 2) {
        const double2 v = STAGED ? reinterpret_cast<const double2*>(xs)[c[k]]
                                 : __ldg(reinterpret_cast<const double2*>(xs) + c[k]);
        s1 += a[k] * v.x;
        s2 += a[k] * v.y;
      } else {
        s1 += a[k] * (STAGED ? xs[c[k]] : __ldg(xs + c[k]));
      }
    }
  }
  for (; p < e; p += V) {
    const double a = ld_stream(val + p);
    const int32_t c = STAGED ? (int32_t)__ldg(c16 + p) : ld_stream(c32 + p);
    if (ELEM == 2) {
      const double2 v = STAGED ? reinterpret_cast<const double2*>(xs)[c]
                               : __ldg(reinterpret_cast<const double2*>(xs) + c);
      s1 += a * v.x;
      s2 += a * v.y;
    } else {
      s1 += a * (STAGED ? xs[c] : __ldg(xs + c));
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
                                         const double* xs, bool staged, double* acc) {
  const int G = blockDim.x / V;
  const int g = threadIdx.x / V, lane = threadIdx.x % V;
  const int32_t* rp = M.rowptr + S.rp;
  for (int rb = 0; rb < C.nrows; rb += G) {        // uniform trip count per warp
    const int r = rb + g;
    double s1 = 0.0, s2 = 0.0;
    int32_t b = 0, e = 0;
    if (r < C.nrows) { b = __ldg(rp + r); e = __ldg(rp + r + 1); }
    if (staged) seg_row_dot<V, ELEM, true>(M.val_s + S.nz, M.col_s + S.nz, nullptr, xs, b, e, lane, s1, s2);
    else seg_row_dot<V, ELEM, false>(M.val_d + S.nz, nullptr, M.col_d + S.nz, xs, b, e, lane, s1, s2);
    if (lane == 0 && r < C.nrows) {
      acc[r * ELEM] += s1;
      if (ELEM == 2) acc[r * ELEM + 1] += s2;
    }
  }
}

// Partial dot products of every work item -> scratch.
// guard: 0 always run, 1 only while running, 2 only on an accepted step
template <int ELEM>
__global__ void __launch_bounds__(kTThreads) k_tiled_partial(TiledMat M, const double* __restrict__ x,
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
      const double* xs = staged ? tile : x;
      switch (S.V) {
        case 1: seg_rows<1, ELEM>(M, S, C, xs, staged, acc); break;
        case 2: seg_rows<2, ELEM>(M, S, C, xs, staged, acc); break;
        case 4: seg_rows<4, ELEM>(M, S, C, xs, staged, acc); break;
        case 8: seg_rows<8, ELEM>(M, S, C, xs, staged, acc); break;
        case 16: seg_rows<16, ELEM>(M, S, C, xs, staged, acc); break;
        default: seg_rows<32, ELEM>(M, S, C, xs, staged, acc); break;
      }
      __syncthreads();
    }
    double* out = scratch + C.scratch + (int64_t)W.group * C.nrows * ELEM;
    for (int i = threadIdx.x; i < C.nrows * ELEM; i += blockDim.x) out[i] = acc[i];
    __syncthreads();
  }
}

// Sum the partials of every row (fixed order) and run the fused epilogue.
template <class Epi, int ELEM>
__global__ void __launch_bounds__(kThreads) k_tiled_combine(TiledMat M, const double* __restrict__ scratch,
                                                            Epi epi, const Ctl* ctl, double* part,
                                                            int64_t slot0) {
  epi.init(ctl);
  if (!epi.active()) return;
  Acc<Epi::NA> acc;
  acc.zero();
  // items are (chunk, slab of blockDim rows); slabs of one chunk are consecutive
  const int64_t per = (kTRows + blockDim.x - 1) / blockDim.x;   // slabs per chunk (upper bound)
  for (int64_t it = blockIdx.x; it < M.nchunk * per; it += gridDim.x) {
    const int64_t c = it / per;
    const int slab = (int)(it % per);
    const TChunk C = M.chunk[c];
    const int r = slab * blockDim.x + threadIdx.x;
    if (r < C.nrows) {
      const double* src = scratch + C.scratch;
      double s1 = 0.0, s2 = 0.0;
      for (int g = 0; g < C.ngroups; ++g) {
        s1 += src[((int64_t)g * C.nrows + r) * ELEM];
        if (ELEM == 2) s2 += src[((int64_t)g * C.nrows + r) * ELEM + 1];
      }
      epi.row(C.row0 + r, s1, s2, acc);
    }
  }
  if (part) cta_write_partials<Epi::NA>(acc, part, slot0 + blockIdx.x);
}

}  // namespace pdcs
