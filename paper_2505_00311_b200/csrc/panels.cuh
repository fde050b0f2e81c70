// panels.cuh — L2 column panels for SpMV sweeps whose gathered vector does not
// fit in L2.
//
// The CSR kernels gather x (or the (x^, x) pairs) at random columns.  When that
// vector is larger than the 126 MB L2 (configs[4] at its stated size: 1e7
// pairs = 160 MB for K x^; 2e7 doubles = 160 MB for K^T y), almost every gather
// misses L2 and costs a whole 32-byte DRAM sector for 8 or 16 useful bytes: the
// K sweep of the 2e9-nnz instance moved ~88 GB for 24 GB of matrix.  Splitting
// the matrix into P column panels whose slice of the vector fits in L2 and
// running the panels one after another turns those misses into L2 hits; the
// price is P passes over a row accumulator (16 or 8 B per row and panel).
//
// Layout: entries regrouped panel-major (panel p holds the columns
// [p*pcols, (p+1)*pcols)), each panel a CSR over all rows with absolute offsets
// into the shared col / val arrays; row order and the order of entries within
// a row are kept, so a row's dot product is the same sum split into P partial
// sums added in panel order (deterministic).
#pragma once
#include "spmv.cuh"

namespace pdcs {

// cnt[p*rows + r] = entries of row r in panel p (rows' columns ascending, so a
// row's panels come in runs).
__global__ void k_panel_count(int64_t rows, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                              int64_t pcols, int32_t* __restrict__ cnt) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = -1;
    int32_t c = 0;
    for (int32_t q = ptr[r]; q < ptr[r + 1]; ++q) {
      const int64_t p = col[q] / pcols;
      if (p != prev) {
        if (prev >= 0) cnt[prev * rows + r] = c;
        prev = p;
        c = 0;
      }
      ++c;
    }
    if (prev >= 0) cnt[prev * rows + r] = c;
  }
}

// Scatter each row's entries to their panels (pptr = exclusive scan of cnt).
__global__ void k_panel_scatter(int64_t rows, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                const double* __restrict__ val, int64_t pcols, const int32_t* __restrict__ pptr,
                                int32_t* __restrict__ pcol, double* __restrict__ pval) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = -1;
    int32_t d = 0;
    for (int32_t q = ptr[r]; q < ptr[r + 1]; ++q) {
      const int64_t p = col[q] / pcols;
      if (p != prev) { prev = p; d = pptr[p * rows + r]; }
      pcol[d] = col[q];
      pval[d] = val[q];
      ++d;
    }
  }
}

// One panel's pass: the row's partial dot products are stored (first panel) or
// added (later panels) into acc (nx doubles per row).  init / active follow the
// sweep's own epilogue, so a pass is skipped exactly when the sweep would be.
template <class Base>
struct EpiPanelAcc {
  static constexpr int NA = 1;
  static constexpr int NX = Base::NX;
  Base base;
  double* acc;
  int first;
  __device__ void init(const Ctl* c) { base.init(c); }
  __device__ bool active() const { return base.active(); }
  __device__ void row(int64_t i, double d1, double d2, Acc<NA>&) {
    if (NX >= 2) {
      double2* a2 = reinterpret_cast<double2*>(acc);
      if (first) { a2[i] = make_double2(d1, d2); return; }
      double2 a = a2[i];
      a.x += d1;
      a.y += d2;
      a2[i] = a;
    } else {
      acc[i] = first ? d1 : acc[i] + d1;
    }
  }
};

// The sweep's epilogue over the accumulated dot products (coalesced, one row
// per thread), with its per-CTA accumulator slots as in spmv_kernel.
template <class Epi>
__global__ void __launch_bounds__(kThreads) k_panel_finish(int64_t rows, const double* __restrict__ acc, Epi epi,
                                                           const Ctl* ctl, double* part, int64_t slot0) {
  epi.init(ctl);
  if (!epi.active()) return;
  Acc<Epi::NA> a;
  a.zero();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    if (Epi::NX >= 2) {
      const double2 v = reinterpret_cast<const double2*>(acc)[i];
      epi.row(i, v.x, v.y, a);
    } else {
      epi.row(i, acc[i], 0.0, a);
    }
  }
  if (part) cta_write_partials<Epi::NA>(a, part, slot0 + blockIdx.x);
}

}  // namespace pdcs
