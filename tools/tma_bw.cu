// Per-SM streaming bandwidth of TMA bulk copies (cp.async.bulk) versus plain
// vectorised loads, for L2-resident and HBM-resident sources.  Used to size the
// projector pipeline (how many SMs must stream Phi to hide L2 latency).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_tma(const char* src, size_t per_cta, size_t span, int stage_bytes, int nstage,
                      unsigned long long* sink) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nstage * stage_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = ((size_t)blockIdx.x * per_cta) % span;
  const int n = (int)(per_cta / stage_bytes);
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n + nstage; ++i) {
      if (i >= nstage) {   // consume stage i - nstage
        const int s = (i - nstage) % nstage;
        const uint32_t par = ((i - nstage) / nstage) & 1;
        asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(su32(&bar[s])), "r"(par) : "memory");
        acc += sm[(size_t)s * stage_bytes];
      }
      if (i < n) {
        const int s = i % nstage;
        const char* p = src + (base + (size_t)i * stage_bytes) % span;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)s * stage_bytes)), "l"(p), "r"(stage_bytes), "r"(su32(&bar[s])) : "memory");
      }
    }
    sink[blockIdx.x] = acc;
  }
}

__global__ void k_ldg(const double2* src, size_t per_cta, size_t span, unsigned long long* sink) {
  const size_t n = per_cta / 16, sp = span / 16;
  const size_t base = ((size_t)blockIdx.x * n) % sp;
  double acc = 0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x * 4) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcg(&src[(base + i + (size_t)u * blockDim.x) % sp]);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x;
  }
  if (acc == 12345.0) sink[blockIdx.x] = 1;
}

// one stage = ncopy bulk copies of stage_bytes / ncopy each, issued by ncopy lanes
__global__ void k_tma_multi(const char* src, size_t per_cta, size_t span, int stage_bytes,
                            int nstage, int ncopy, unsigned long long* sink) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)nstage * stage_bytes);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < nstage; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = ((size_t)blockIdx.x * per_cta) % span;
  const int n = (int)(per_cta / stage_bytes);
  const int cb = stage_bytes / ncopy;
  unsigned long long acc = 0;
  for (int i = 0; i < n + nstage; ++i) {
    if (i >= nstage) {
      const int s = (i - nstage) % nstage;
      const uint32_t par = ((i - nstage) / nstage) & 1;
      asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}" ::"r"(su32(&bar[s])), "r"(par) : "memory");
      acc += sm[(size_t)s * stage_bytes];
    }
    __syncwarp();
    if (i < n) {
      const int s = i % nstage;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(stage_bytes) : "memory");
      __syncwarp();
      for (int c = lane; c < ncopy; c += 32) {
        // scattered sources (like gathered rows): copy c of stage i from a distant address
        const char* p = src + (base + ((size_t)c * 1048576 + (size_t)i * cb)) % span;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)s * stage_bytes + (size_t)c * cb)), "l"(p), "r"(cb), "r"(su32(&bar[s])) : "memory");
      }
    }
  }
  if (lane == 0) sink[blockIdx.x] = acc;
}

int main() {
  const size_t big = 2ull << 30;
  char* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  cudaMalloc(&sink, 4096 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const size_t spans[2] = {16ull << 20, big};
  const char* names[2] = {"L2 (16 MB span)", "HBM (2 GB span)"};
  for (int si = 0; si < 2; ++si) {
    for (int grid : {1, 8, 16, 148}) {
      for (int sb : {8192, 36864}) {
        for (int ns : {2, 4}) {
          if ((size_t)sb * ns > 190 * 1024) continue;
          const size_t per = (size_t)sb * 256;
          k_tma<<<grid, 32, (size_t)sb * ns + 64>>>(buf, per, spans[si], sb, ns, sink);
          cudaEventRecord(e0);
          k_tma<<<grid, 32, (size_t)sb * ns + 64>>>(buf, per, spans[si], sb, ns, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double gbs = (double)per * grid / (ms * 1e-3) / 1e9;
          printf("TMA %-16s grid %3d stage %6d x%d: %8.1f GB/s total, %6.1f GB/s per SM\n",
                 names[si], grid, sb, ns, gbs, gbs / grid);
        }
      }
      const size_t per = 36864ull * 256;
      k_ldg<<<grid, 256>>>((const double2*)buf, per, spans[si], sink);
      cudaEventRecord(e0);
      k_ldg<<<grid, 256>>>((const double2*)buf, per, spans[si], sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = (double)per * grid / (ms * 1e-3) / 1e9;
      printf("LDG %-16s grid %3d 256 thr x4 in flight: %8.1f GB/s total, %6.1f GB/s per SM\n",
             names[si], grid, gbs, gbs / grid);
    }
  }
  cudaFuncSetAttribute(k_tma_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {8, 148}) {
    for (int nc : {1, 4, 16, 36}) {
      const int sb = 36864, ns = 3;
      const size_t per = (size_t)sb * 128;
      k_tma_multi<<<grid, 32, (size_t)sb * ns + 64>>>(buf, per, spans[0], sb, ns, nc, sink);
      cudaEventRecord(e0);
      k_tma_multi<<<grid, 32, (size_t)sb * ns + 64>>>(buf, per, spans[0], sb, ns, nc, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gbs = (double)per * grid / (ms * 1e-3) / 1e9;
      printf("TMA-multi L2 grid %3d stage 36 KB as %2d copies x3 stages: %8.1f GB/s total, %6.1f GB/s per SM, %.3f us/stage\n",
             grid, nc, gbs, gbs / grid, ms * 1e3 / 128);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
