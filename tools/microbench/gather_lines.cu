// Random 128-byte line gathers (the C5 SpMM's access: one 32-probe fp32 row per nonzero) over a
// buffer of a given size: the line-request rate the B200 sustains when the lines come from DRAM
// (buffer >> L2) and when they hit L2 (buffer < L2).  This is the ceiling of the narrow-chunk SpMM,
// which issues one 128-byte line request per nonzero.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_lines.cu -o gather_lines
//   ./gather_lines <buffer MB> ...   -> one JSON line per (size, depth, ctas/SM)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd_row(uint32_t& x, uint32_t mask) {
  x = x * 1664525u + 1013904223u;
  const uint32_t h = (x ^ (x >> 15)) * 2246822519u;
  return (h ^ (h >> 13)) & mask;
}

// 8 lanes x float4 per 128-byte line (4 lines per warp instruction), U loads in flight per lane
template <int U>
__global__ void __launch_bounds__(256) lines_kernel(const float4* __restrict__ buf, uint32_t mask, int iters,
                                                    float* out) {
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

int main(int argc, char** argv) {
  float* out = nullptr;
  cudaMalloc(&out, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int a = 1; a < argc; ++a) {
    const int64_t mb = atoll(argv[a]);
    int64_t nrows = 1;
    while (nrows * 2 * 128 <= mb * (1ll << 20)) nrows *= 2;   // power-of-two rows (mask)
    const int64_t bytes = nrows * 128;
    float4* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("{\"error\": \"alloc %lld MB\"}\n", (long long)mb); return 1; }
    cudaMemset(buf, 0, bytes);
    const uint32_t mask = static_cast<uint32_t>(nrows - 1);
#define RUN(U, CPS)                                                                                         \
    {                                                                                                       \
      const int ctas = 148 * CPS, thr = 256, iters = 1024 / U;                                              \
      lines_kernel<U><<<ctas, thr>>>(buf, mask, 2, out);                                                    \
      cudaEventRecord(e0);                                                                                  \
      lines_kernel<U><<<ctas, thr>>>(buf, mask, iters, out);                                                \
      cudaEventRecord(e1);                                                                                  \
      cudaEventSynchronize(e1);                                                                             \
      float ms;                                                                                             \
      cudaEventElapsedTime(&ms, e0, e1);                                                                    \
      const double lines = static_cast<double>(ctas) * thr / 8 * iters * U;                                \
      printf("{\"buffer_MB\": %.1f, \"depth\": %d, \"ctas_per_sm\": %d, \"Glines_per_s\": %.2f, \"GBps\": %.1f}\n", \
             bytes / 1048576.0, U, CPS, lines / (ms * 1e-3) / 1e9, lines * 128 / (ms * 1e-3) / 1e9);        \
    }
    RUN(4, 4) RUN(8, 4) RUN(16, 4) RUN(8, 8)
    cudaFree(buf);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
