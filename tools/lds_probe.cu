// lds_probe.cu — how many shared-memory wavefronts does one warp-wide
// ld.shared.v2.f64 / ld.shared.f64 cost for a given lane -> address pattern?
// Run under ncu and divide l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum
// by smsp__sass_inst_executed_op_shared_ld.sum (one kernel per pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_probe tools/lds_probe.cu
#include <cstdio>
#include <cstdint>

template <int W>   // W = 16 (v2.f64) or 8 (f64)
__global__ void probe(const uint32_t* __restrict__ idx, double* out, int reps) {
  __shared__ __align__(16) double tile[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tile[i] = i;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tile);
  const uint32_t a = base + idx[threadIdx.x & 31] * W;
  double s = 0.0;
  for (int r = 0; r < reps; ++r) {
    if (W == 16) {
      double x, y;
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
      s += x + y;
    } else {
      double x;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a));
      s += x;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  uint32_t pat[8][32];
  uint32_t st = 12345;
  for (int l = 0; l < 32; ++l) {
    pat[0][l] = l;                                  // consecutive: conflict-free
    pat[1][l] = (l % 8) + (l / 8) * 8 * 7;          // each quarter: groups 0..7, different lines
    pat[2][l] = l * 8;                              // all lanes group 0 (v2) / group 0,8 (f64)
    pat[3][l] = (l / 4) + (l % 4) * 8;              // quarter: 4 lanes per group; warp: 4 per group (v2)
    pat[4][l] = (l % 4) * 8 + (l / 4) % 2 + (l / 8) * 2 * 8 * 0 + (l / 8) * 2;   // mixed
    st = st * 1103515245u + 12345u;
    pat[5][l] = (st >> 8) % 2048;                   // random
    pat[6][l] = (l % 8) * 8 + (l / 8);              // quarter: all 8 lanes same group? no: group = l/8 (v2)
    pat[7][l] = l * 2;                              // f64: 2-lane stride
  }
  uint32_t* d;
  double* o;
  cudaMalloc(&d, sizeof(pat));
  cudaMalloc(&o, 148 * 256 * sizeof(double));
  cudaMemcpy(d, pat, sizeof(pat), cudaMemcpyHostToDevice);
  for (int p = 0; p < 8; ++p) probe<16><<<1, 32>>>(d + 32 * p, o, 1000);
  for (int p = 0; p < 8; ++p) probe<8><<<1, 32>>>(d + 32 * p, o, 1000);
  cudaDeviceSynchronize();
  for (int p = 0; p < 8; ++p) {
    printf("pattern %d:", p);
    for (int l = 0; l < 32; ++l) printf(" %u", pat[p][l]);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
