// DMMA (mma.sync.m8n8k4.f64) throughput vs resident warps per SM and independent
// accumulator chains per warp: how many DMMAs must be in flight to reach peak.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[CH][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < CH; ++j) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(double* out, int warps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000 / CH * 4, grid = 148, bs = 32 * warps;
  k<CH><<<grid, bs>>>(out, 10);
  cudaEventRecord(e0);
  k<CH><<<grid, bs>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256.0 * CH * (double)iters * grid * warps;
  printf("warps/SM %2d chains/warp %2d: %6.1f TFLOP/s\n", warps, CH, flops / ms / 1e9);
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  for (int w : {4, 8, 16, 32}) {
    run<1>(out, w); run<2>(out, w); run<4>(out, w); run<6>(out, w); run<12>(out, w);
  }
  return 0;
}
