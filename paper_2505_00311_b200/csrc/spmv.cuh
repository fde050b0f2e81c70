// spmv.cuh — row-binned CSR SpMV (fp64) with fused per-row epilogues.
//
// The two products of Eq. 5, K x^ and K^T y^, dominate
// PDCS.  Rows are binned by length at setup (SpmvPlan):
//   V = 1            one thread per row         (rows of <= 2 nnz)
//   V = 4, 8, 16, 32 V lanes per row, segmented shuffle reduction (warp-
//                    segmented rows; 32/V rows per warp)
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

__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }

// Dot products of one row with V lanes (lane in [0, V)) against NX gathered
// vectors (x1, and x2 when NX == 2: K x^ and K x share one sweep over the row).
// Results valid in all lanes of the group.
template <int V, int NX>
__device__ __forceinline__ void row_dot(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                        const double* __restrict__ val, const double* __restrict__ x1,
                                        const double* __restrict__ x2, int64_t row, int lane, double& s1,
                                        double& s2) {
  s1 = 0.0;
  s2 = 0.0;
  if (row >= 0) {
    const int32_t b = __ldg(ptr + row), e = __ldg(ptr + row + 1);
    int32_t p = b + lane;
    for (; p + 3 * V < e; p += 4 * V) {
      const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + V);
      const int32_t c2 = ld_stream(col + p + 2 * V), c3 = ld_stream(col + p + 3 * V);
      const double a0 = ld_stream(val + p), a1 = ld_stream(val + p + V);
      const double a2 = ld_stream(val + p + 2 * V), a3 = ld_stream(val + p + 3 * V);
      s1 += a0 * __ldg(x1 + c0);
      s1 += a1 * __ldg(x1 + c1);
      s1 += a2 * __ldg(x1 + c2);
      s1 += a3 * __ldg(x1 + c3);
      if (NX == 2) {
        s2 += a0 * __ldg(x2 + c0);
        s2 += a1 * __ldg(x2 + c1);
        s2 += a2 * __ldg(x2 + c2);
        s2 += a3 * __ldg(x2 + c3);
      }
    }
    for (; p < e; p += V) {
      const double a = ld_stream(val + p);
      const int32_t c = ld_stream(col + p);
      s1 += a * __ldg(x1 + c);
      if (NX == 2) s2 += a * __ldg(x2 + c);
    }
  }
  if (V > 1) {
#pragma unroll
    for (int o = V / 2; o >= 1; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o, V);
      if (NX == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, V);
    }
  }
}

// Epi: struct with
//   static constexpr int NA;                       accumulators per CTA
//   static constexpr int NX;                       gathered vectors (1 or 2)
//   __device__ void init(const Ctl*);              read scalars once
//   __device__ bool active() const;                predicate (false: kernel is a no-op)
//   __device__ void row(int64_t i, double dot1, double dot2, Acc<NA>&);
template <class Epi>
__global__ void __launch_bounds__(kThreads) spmv_kernel(const int32_t* __restrict__ ptr,
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
      const int32_t b = __ldg(ptr + row), e = __ldg(ptr + row + 1);
      double s1 = 0.0, s2 = 0.0;
      int32_t p = b + threadIdx.x;
      for (; p + 3 * kThreads < e; p += 4 * kThreads) {
        const int32_t c0 = ld_stream(col + p), c1 = ld_stream(col + p + kThreads);
        const int32_t c2 = ld_stream(col + p + 2 * kThreads), c3 = ld_stream(col + p + 3 * kThreads);
        const double a0 = ld_stream(val + p), a1 = ld_stream(val + p + kThreads);
        const double a2 = ld_stream(val + p + 2 * kThreads), a3 = ld_stream(val + p + 3 * kThreads);
        s1 += a0 * __ldg(x1 + c0);
        s1 += a1 * __ldg(x1 + c1);
        s1 += a2 * __ldg(x1 + c2);
        s1 += a3 * __ldg(x1 + c3);
        if (NX == 2) {
          s2 += a0 * __ldg(x2 + c0);
          s2 += a1 * __ldg(x2 + c1);
          s2 += a2 * __ldg(x2 + c2);
          s2 += a3 * __ldg(x2 + c3);
        }
      }
      for (; p < e; p += kThreads) {
        const double a = ld_stream(val + p);
        const int32_t cc = ld_stream(col + p);
        s1 += a * __ldg(x1 + cc);
        if (NX == 2) s2 += a * __ldg(x2 + cc);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        if (NX == 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
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
    for (int64_t idx = (int64_t)lcta * kThreads + threadIdx.x; idx < K.nrows;
         idx += (int64_t)K.ncta * kThreads) {
      const int64_t row = rowid(idx);
      double s1, s2;
      row_dot<1, NX>(ptr, col, val, x1, x2, row, 0, s1, s2);
      epi.row(row, s1, s2, acc);
    }
  } else {
    const int V = K.V;
    const int R = kThreads / V;                  // rows per CTA iteration
    const int g = threadIdx.x / V, lane = threadIdx.x % V;
    for (int64_t ib = (int64_t)lcta * R; ib < K.nrows; ib += (int64_t)K.ncta * R) {
      const int64_t idx = ib + g;
      const int64_t row = idx < K.nrows ? rowid(idx) : -1;
      double s1, s2;
      switch (V) {
        case 4: row_dot<4, NX>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
        case 8: row_dot<8, NX>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
        case 16: row_dot<16, NX>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
        default: row_dot<32, NX>(ptr, col, val, x1, x2, row, lane, s1, s2); break;
      }
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
