// stream_probe.cu — the read-only HBM ceiling of this B200, next to the copy
// peak of MEASURED_PEAKS.json (read + write).  The SpMV sweeps are read-
// dominated (≈97% of their bytes are loads), so their roofline fraction is
// also reported against the best read-only stream measured here.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/stream_probe tools/stream_probe.cu
//   tools/bin/stream_probe [GiB=2.4]
// Prints GB/s for: 32-B loads (v4.f64, L1::no_allocate, as the tiled kernel
// streams values), 16-B loads, with 1..4 loads in flight per thread, grids of
// 1..8 CTAs/SM x 512 threads; and a plain copy for comparison.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double4 ld4(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int W, int U>   // W doubles per load (2 or 4), U loads in flight per thread
__global__ void rd(const double* __restrict__ a, int64_t n, double* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * W * U;
  double s = 0.0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n; i += stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + (int64_t)u * gridDim.x * blockDim.x * W;
      if (j + W <= n) {
        if (W == 4) { const double4 v = ld4(a + j); s += v.x + v.y + v.z + v.w; }
        else { const double2 v = ld2(a + j); s += v.x + v.y; }
      }
    }
  }
  if (s == 12345.678) out[0] = s;   // keep the loads
}

__global__ void cp(const double4* __restrict__ a, double4* __restrict__ b, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <class F>
float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  f();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 2.4;
  const int64_t n = (int64_t)(gib * (1ull << 30) / 8) & ~(int64_t)63;
  double *a, *b, *out;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)n * 8;
  printf("{\"bytes\": %.0f, \"sms\": %d, \"runs\": [\n", bytes, sms);
  bool first = true;
  auto rep = [&](const char* name, int per_sm, float ms, double moved) {
    printf("%s {\"kernel\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", first ? "" : ",", name, per_sm,
           ms, moved / (ms * 1e-3) / 1e9);
    first = false;
  };
  for (int per_sm : {1, 2, 4, 8}) {
    const int g = sms * per_sm;
    rep("v4.f64 U1", per_sm, best_ms([&] { rd<4, 1><<<g, 512>>>(a, n, out); }), bytes);
    rep("v4.f64 U2", per_sm, best_ms([&] { rd<4, 2><<<g, 512>>>(a, n, out); }), bytes);
    rep("v4.f64 U4", per_sm, best_ms([&] { rd<4, 4><<<g, 512>>>(a, n, out); }), bytes);
    rep("v2.f64 U4", per_sm, best_ms([&] { rd<2, 4><<<g, 512>>>(a, n, out); }), bytes);
  }
  rep("copy v4 (read+write bytes)", 4, best_ms([&] { cp<<<sms * 4, 512>>>((const double4*)a, (double4*)b, n / 4); }),
      2 * bytes);
  printf("]}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
