// spmv.cuh — row-binned CSR SpMV (fp64) with fused per-row epilogues.
//
// The two products of Eq. 5, K x^ and K^T y^, dominate
// PDCS.  Rows are binned by length at setup (SpmvPlan):
//   V = 1            one thread per row         (rows of <= 2 nnz)
//   V = 4, 8, 16, 32 V lanes per row, segmented shuffle reduction (warp-
//                    segmented rows; 32/V rows per warp).  Thresholds are
//                    set at setup (PDCS_SPMV_BINS overrides them for tuning).
//   V = 0            one CTA per row (rows of > 4096 nnz)
// Matrix values / column ids are streamed with evict-first loads; the
// gathered vector goes through the read-only path and stays in L2.  Each CTA
// iteration covers a contiguous slice of a class's rows; dot products are
// staged in shared memory so that the epilogue (the fused dual update,
// Halpern step, ...) reads and writes the row-indexed vectors coalesced.
// Epilogue accumulators (line-search sums) are reduced per CTA in a fixed
// order and written to one slot per CTA -> deterministic results.
#pragma once
#include "internal.cuh"

namespace pdcs {

template <int N>
struct Acc {
  double v[N];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = 0.0;
  }
};

// Reduce NA accumulators across the CTA and write them to part[slot*NA + i].
template <int NA>
__device__ __forceinline__ void cta_write_partials(Acc<NA>& a, double* part, int64_t slot) {
  __shared__ double red[NA][kThreads / 32];
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    double s = a.v[i];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x < NA) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
    part[slot * NA + threadIdx.x] = s;
  }
}

// Streaming loads of the matrix (read once per pass): no L1 allocation, so the
// L1 keeps the gathered vector(s).
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Dot products of one row with V lanes (lane in [0, V)) against NX gathered
// vectors: NX == 1 x1; NX == 2 x1 and x2; NX == 3 x1 holds interleaved pairs
// (x^_j, x_j) so that K x^ and K x share one sweep and one 16-byte gather.
// Software-pipelined: the column ids / values of chunk i+1 are in flight while
// chunk i's gathers are served; tails are predicated.  Results valid in all
// lanes of the group.
#ifndef PDCS_CSR_U
#define PDCS_CSR_U 8                  // entries in flight per lane, V >= 8 (B200: 4 -> 8 with the 64-register cap, MPO +13%, mixed +7%)
#endif
template <int V, int NX, int UU = PDCS_CSR_U>
__device__ __forceinline__ void row_dot(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                        const double* __restrict__ val, const double* __restrict__ x1,
                                        const double* __restrict__ x2, int64_t row, int lane, double& s1,
                                        double& s2) {
  constexpr int U = (V >= 8 && V <= 32) ? UU : 4;   // entries in flight per lane
  s1 = 0.0;
  s2 = 0.0;
  if (row >= 0) {
    const int32_t b = __ldg(ptr + row), e = __ldg(ptr + row + 1);
    int32_t p = b + lane;
    int32_t c[U];
    double a[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int32_t q = p + k * V;
      c[k] = q < e ? ld_stream(col + q) : -1;
      a[k] = q < e ? ld_stream(val + q) : 0.0;
    }
    for (; p < e; p += U * V) {
      int32_t cn[U];
      double an[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int32_t q = p + (U + k) * V;
        cn[k] = q < e ? ld_stream(col + q) : -1;
        an[k] = q < e ? ld_stream(val + q) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (c[k] >= 0) {
          if (NX == 3) {   // interleaved pair: one 16-byte gather serves both products
            const double2 v = __ldg(reinterpret_cast<const double2*>(x1) + c[k]);
            s1 += a[k] * v.x;
            s2 += a[k] * v.y;
          } else {
            s1 += a[k] * __ldg(x1 + c[k]);
            if (NX == 2) s2 += a[k] * __ldg(x2 + c[k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) { c[k] = cn[k]; a[k] = an[k]; }
    }
  }
  if (V > 1 && V <= 32) {
#pragma unroll
    for (int o = V / 2; o >= 1; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
      if (NX >= 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
    }
  }
}

// Epi: struct with
//   static constexpr int NA;                       accumulators per CTA
//   static constexpr int NX;                       gathered vectors (1 or 2)
//   __device__ void init(const Ctl*);              read scalars once
//   __device__ bool active() const;                predicate (false: kernel is a no-op)
//   __device__ void row(int64_t i, double dot1, double dot2, Acc<NA>&);
#ifndef PDCS_CSR_MINB
#define PDCS_CSR_MINB 4               // 64 registers: 4 CTAs of 256 threads per SM
#endif
// UU: entries in flight per lane for the V >= 8 classes (a per-matrix setup
// choice between 8 and 4: MPO's K sweep 227.6 -> 216.1 us with 4, its K^T
// sweep slower with 4).
template <class Epi, int UU = PDCS_CSR_U>
__global__ void __launch_bounds__(kThreads, PDCS_CSR_MINB) spmv_kernel(const int32_t* __restrict__ ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x1,
                                                        const double* __restrict__ x2,
                                                        SpmvPlan plan, Epi epi, const Ctl* ctl,
                                                        double* part, int64_t slot0) {
  constexpr int NX = Epi::NX;
  epi.init(ctl);
  if (!epi.active()) return;
  Acc<Epi::NA> acc;
  acc.zero();
  __shared__ double sdot[2][kThreads];
  __shared__ int64_t srow[kThreads];
  // locate the class of this CTA
  int c = 0, base = 0;
  while (c < plan.ncls - 1 && (int)blockIdx.x >= base + plan.cls[c].ncta) { base += plan.cls[c].ncta; ++c; }
  const SpmvClass K = plan.cls[c];
  const int lcta = blockIdx.x - base;
  auto rowid = [&](int64_t idx) -> int64_t { return K.rows ? (int64_t)K.rows[idx] : K.range_begin + idx; };
  if (K.V == 0) {
    // one CTA per row
    __shared__ double red[2][kThreads / 32];
    for (int64_t idx = lcta; idx < K.nrows; idx += K.ncta) {
      const int64_t row = rowid(idx);
      double s1, s2;
      row_dot<kThreads, NX>(ptr, col, val, x1, x2, row, threadIdx.x, s1, s2);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        if (NX >= 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s1; red[1][threadIdx.x >> 5] = s2; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) { t1 += red[0][w]; t2 += red[1][w]; }
        epi.row(row, t1, t2, acc);
      }
      __syncthreads();
    }
  } else if (K.V == 1) {
    // one thread per row (rows of <= 2 nnz as binned): R rows per thread and
    // step, their pointers, first two entries and gathers issued together so
    // that the dependent latencies of the R rows overlap
    constexpr int R = 4;
    const int64_t stride = (int64_t)K.ncta * kThreads;
    auto gather = [&](int32_t c, double a, double& s1, double& s2) {
      if (c < 0) return;
      if (NX == 3) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(x1) + c);
        s1 += a * v.x;
        s2 += a * v.y;
      } else {
        s1 += a * __ldg(x1 + c);
        if (NX == 2) s2 += a * __ldg(x2 + c);
      }
    };
    for (int64_t i0 = (int64_t)lcta * kThreads + threadIdx.x; i0 < K.nrows; i0 += R * stride) {
      int64_t rw[R];
      int32_t b[R], e[R], c0[R], c1[R];
      double a0[R], a1[R], s1[R], s2[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int64_t idx = i0 + k * stride;
        rw[k] = idx < K.nrows ? rowid(idx) : -1;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        b[k] = rw[k] >= 0 ? __ldg(ptr + rw[k]) : 0;
        e[k] = rw[k] >= 0 ? __ldg(ptr + rw[k] + 1) : 0;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        c0[k] = b[k] < e[k] ? ld_stream(col + b[k]) : -1;
        a0[k] = b[k] < e[k] ? ld_stream(val + b[k]) : 0.0;
        c1[k] = b[k] + 1 < e[k] ? ld_stream(col + b[k] + 1) : -1;
        a1[k] = b[k] + 1 < e[k] ? ld_stream(val + b[k] + 1) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        s1[k] = 0.0;
        s2[k] = 0.0;
        gather(c0[k], a0[k], s1[k], s2[k]);
        gather(c1[k], a1[k], s1[k], s2[k]);
        for (int32_t p = b[k] + 2; p < e[k]; ++p) gather(ld_stream(col + p), ld_stream(val + p), s1[k], s2[k]);
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (rw[k] >= 0) epi.row(rw[k], s1[k], s2[k], acc);
    }
  } else if (K.V >= 8) {
    // V lanes per row, epilogue run directly by the group leader (matrix bytes
    // per row >> epilogue bytes, so no staging / barriers are needed).
    const int V = K.V;
    const int G = kThreads / V;                  // row groups per CTA
    const int g = threadIdx.x / V, lane = threadIdx.x % V;
    for (int64_t ib = (int64_t)lcta * G; ib < K.nrows; ib += (int64_t)K.ncta * G) {
      const int64_t idx = ib + g;
      const int64_t row = idx < K.nrows ? rowid(idx) : -1;
      double s1, s2;
      switch (V) {
        case 8: row_dot<8, NX, UU>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
        case 16: row_dot<16, NX, UU>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
        default: row_dot<32, NX, UU>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
      }
      if (lane == 0 && row >= 0) epi.row(row, s1, s2, acc);
    }
  } else {
    // V = 4: short rows; dot products staged in shared memory so that the
    // epilogue of consecutive rows is coalesced.
    const int V = K.V;
    const int R = kThreads / V;                  // rows per CTA iteration
    const int g = threadIdx.x / V, lane = threadIdx.x % V;
    for (int64_t ib = (int64_t)lcta * R; ib < K.nrows; ib += (int64_t)K.ncta * R) {
      const int64_t idx = ib + g;
      const int64_t row = idx < K.nrows ? rowid(idx) : -1;
      double s1, s2;
      row_dot<4, NX>(ptr, col, val, x1, x2, row, lane, s1, s2);
      if (lane == 0) { sdot[0][g] = s1; sdot[1][g] = s2; srow[g] = row; }
      __syncthreads();
      if (threadIdx.x < R && srow[threadIdx.x] >= 0)
        epi.row(srow[threadIdx.x], sdot[0][threadIdx.x], sdot[1][threadIdx.x], acc);
      __syncthreads();
    }
  }
  if (part) cta_write_partials<Epi::NA>(acc, part, slot0 + blockIdx.x);
}

}  // namespace pdcs
