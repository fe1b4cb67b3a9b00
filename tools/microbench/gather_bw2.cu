// Random 128-byte-row gathers over an 8 GB buffer (the C5 SpMM's access pattern after the fold:
// 32 fp32 probes per row): how much in-flight depth does the B200 need, and do cp.async copies into
// shared memory (no registers held per load) beat register loads?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_bw2.cu -o gather_bw2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd_row(uint32_t& x, uint32_t mask) {
  x = x * 1664525u + 1013904223u;
  const uint32_t h = (x ^ (x >> 15)) * 2246822519u;
  return (h ^ (h >> 13)) & mask;
}

// register loads: 8 lanes x float4 per row (4 rows per warp instruction), U loads in flight per lane
template <int U>
__global__ void ld_kernel(const float4* __restrict__ buf, uint32_t mask, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 8 * 7919u + 1;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) v[q] = __ldg(buf + static_cast<int64_t>(rnd_row(x, mask)) * 8 + (lane & 7));
#pragma unroll
    for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

// cp.async: each warp keeps D groups of 4 x 8 rows (one 16-byte copy per lane per row-quad) in a
// shared-memory ring; waits for the oldest group, sums it, refills
template <int D>
__global__ void cpasync_kernel(const float4* __restrict__ buf, uint32_t mask, int iters, float* out) {
  extern __shared__ __align__(16) float4 ring[];   // [warps][D][8 quads][32 lanes]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* my = ring + static_cast<int64_t>(warp) * D * 8 * 32;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 8 * 7919u + 1;
  float acc = 0.f;
  auto issue = [&](int slot) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4* src = buf + static_cast<int64_t>(rnd_row(x, mask)) * 8 + (lane & 7);
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(my + (slot * 8 + k) * 32 + lane));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < D; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % D;
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 v = my[(s * 8 + k) * 32 + lane];
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    issue(s);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const int64_t bytes = 8ll << 30;
  const int64_t nrows = bytes / 128;
  const uint32_t mask = static_cast<uint32_t>(nrows - 1);
  float4* buf = nullptr; float* out = nullptr;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 64);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto report = [&](const char* name, int ctas_per_sm, int threads, int depth, double rows, float ms) {
    printf("{\"kernel\": \"%s\", \"ctas_per_sm\": %d, \"threads\": %d, \"depth\": %d, \"GBps\": %.1f}\n", name, ctas_per_sm,
           threads, depth, rows * 128 / (ms * 1e-3) / 1e9);
  };
#define LD(U, CPS)                                                                                        \
  {                                                                                                       \
    const int ctas = 148 * CPS, thr = 256, iters = 256 / U * 4;                                           \
    ld_kernel<U><<<ctas, thr>>>(buf, mask, 2, out);                                                       \
    cudaEventRecord(e0); ld_kernel<U><<<ctas, thr>>>(buf, mask, iters, out); cudaEventRecord(e1);         \
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);                                 \
    report("ld_float4", CPS, thr, U, static_cast<double>(ctas) * thr / 8 * iters * U, ms);                \
  }
  LD(4, 4) LD(8, 4) LD(16, 4) LD(8, 8) LD(16, 8)
#define CPA(D, CPS, THR)                                                                                  \
  {                                                                                                       \
    const int ctas = 148 * CPS, thr = THR, iters = 512;                                                   \
    const size_t smem = static_cast<size_t>(thr / 32) * D * 8 * 32 * 16;                                  \
    cudaFuncSetAttribute(cpasync_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    cpasync_kernel<D><<<ctas, thr, smem>>>(buf, mask, 2, out);                                            \
    cudaEventRecord(e0); cpasync_kernel<D><<<ctas, thr, smem>>>(buf, mask, iters, out); cudaEventRecord(e1); \
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);                                 \
    report("cp_async", CPS, thr, D * 32, static_cast<double>(ctas) * thr / 8 * iters * 8, ms);            \
  }
  CPA(2, 2, 256) CPA(2, 3, 256) CPA(3, 2, 256) CPA(6, 2, 128) CPA(4, 3, 128)
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
