// Random-row gathers of R-byte rows (R = 16*CH) from a buffer of B bytes: register loads vs cp.async
// into shared memory, to size the in-flight depth the SpMM needs when the gathered block is
// L2-resident (C2: 800-byte fp64 rows of an 80 MB block) or not.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_bw3.cu -o gather_bw3 ; ./gather_bw3 MB CH
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd_row(uint32_t& x, uint32_t nrows) {
  x = x * 1664525u + 1013904223u;
  const uint32_t h = (x ^ (x >> 15)) * 2246822519u;
  return (h ^ (h >> 13)) % nrows;
}

// register loads: a warp reads U rows per round (lane covers chunks lane, lane+32, ...)
template <int U, int CH>
__global__ void ld_kernel(const float4* __restrict__ buf, uint32_t nrows, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 7919u + 1;
  constexpr int PL = (CH + 31) / 32;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[U][PL];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const float4* row = buf + static_cast<int64_t>(rnd_row(x, nrows)) * CH;
#pragma unroll
      for (int j = 0; j < PL; ++j) v[q][j] = (lane + 32 * j < CH) ? __ldg(row + lane + 32 * j) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
#pragma unroll
      for (int j = 0; j < PL; ++j) acc += v[q][j].x + v[q][j].w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

// cp.async: per warp a ring of D groups of G rows; wait for the oldest group, consume, refill
template <int D, int G, int CH>
__global__ void cpasync_kernel(const float4* __restrict__ buf, uint32_t nrows, int iters, float* out) {
  extern __shared__ __align__(16) float4 ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* my = ring + static_cast<int64_t>(warp) * D * G * CH;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 7919u + 1;
  float acc = 0.f;
  auto issue = [&](int slot) {
    for (int k = 0; k < G; ++k) {
      const float4* row = buf + static_cast<int64_t>(rnd_row(x, nrows)) * CH;
      for (int c = lane; c < CH; c += 32) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(my + (slot * G + k) * CH + c));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(row + c) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < D; ++s) issue(s);
  for (int it = 0; it < iters; ++it) {
    const int s = it % D;
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    __syncwarp();
    for (int k = 0; k < G; ++k)
      for (int c = lane; c < CH; c += 32) {
        const float4 v = my[(s * G + k) * CH + c];
        acc += v.x + v.w;
      }
    __syncwarp();
    issue(s);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (acc == 1.2345f) out[0] = acc;
}

template <int CH>
void run(int64_t mb) {
  const int64_t bytes = mb << 20;
  const uint32_t nrows = static_cast<uint32_t>(bytes / (16 * CH));
  float4* buf = nullptr; float* out = nullptr;
  cudaMalloc(&buf, bytes); cudaMalloc(&out, 64);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto report = [&](const char* name, int ctas_per_sm, int threads, int depth, double rows, float ms) {
    printf("{\"kernel\": \"%s\", \"buf_MB\": %lld, \"row_bytes\": %d, \"ctas_per_sm\": %d, \"threads\": %d, \"rows_in_flight_per_warp\": %d, \"GBps\": %.1f}\n",
           name, (long long)mb, 16 * CH, ctas_per_sm, threads, depth, rows * 16 * CH / (ms * 1e-3) / 1e9);
  };
#define LD(U, CPS)                                                                                          \
  {                                                                                                         \
    const int ctas = 148 * CPS, thr = 256, iters = 64;                                                      \
    ld_kernel<U, CH><<<ctas, thr>>>(buf, nrows, 2, out);                                                    \
    cudaEventRecord(e0); ld_kernel<U, CH><<<ctas, thr>>>(buf, nrows, iters, out); cudaEventRecord(e1);      \
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);                                   \
    report("ld", CPS, thr, U, static_cast<double>(ctas) * thr / 32 * iters * U, ms);                         \
  }
  LD(1, 4) LD(2, 3) LD(2, 4) LD(4, 2) LD(4, 4)
#define CPA(D, G, CPS, THR)                                                                                 \
  {                                                                                                         \
    const int ctas = 148 * CPS, thr = THR, iters = 64;                                                      \
    const size_t smem = static_cast<size_t>(thr / 32) * D * G * CH * 16;                                    \
    if (smem <= 227 * 1024) {                                                                               \
      cudaFuncSetAttribute(cpasync_kernel<D, G, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      cpasync_kernel<D, G, CH><<<ctas, thr, smem>>>(buf, nrows, 2, out);                                    \
      cudaEventRecord(e0); cpasync_kernel<D, G, CH><<<ctas, thr, smem>>>(buf, nrows, iters, out);           \
      cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);            \
      report("cp_async", CPS, thr, D * G, static_cast<double>(ctas) * thr / 32 * iters * G, ms);           \
    }                                                                                                       \
  }
  CPA(2, 2, 4, 128) CPA(3, 2, 2, 256) CPA(4, 2, 2, 128) CPA(2, 4, 2, 128) CPA(4, 4, 1, 128) CPA(3, 4, 2, 64)
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
  cudaFree(buf); cudaFree(out);
}

int main(int argc, char** argv) {
  const int64_t mb = argc > 1 ? atoll(argv[1]) : 80;
  run<50>(mb);   // 800-byte rows (C2: 100 fp64 probes)
  run<8>(mb);    // 128-byte rows
  return 0;
}
