// Measure FP64 throughput on the B200: DMMA (mma.sync m8n8k4 f64, the FP64
// tensor-core path) vs DFMA (SIMT).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[j][0]), "+d"(d[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[16] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) d[j] = fma(a, d[j], b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += d[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int bs : {128, 256, 512}) {
    int grid = 148 * 4;
    k_dmma<<<grid, bs>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8 * iters * (double)grid * (bs / 32);
    printf("DMMA bs=%d: %.1f TFLOP/s\n", bs, flops / ms / 1e9);
    k_dfma<<<grid, bs>>>(out, 100);
    cudaEventRecord(e0);
    k_dfma<<<grid, bs>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)grid * bs;
    printf("DFMA bs=%d: %.1f TFLOP/s\n", bs, flops / ms / 1e9);
  }
  return 0;
}
