// Does vertex relabelling pay for the C5 SpMM?  Random 128-byte line gathers over an 8 GB buffer
// where a fraction f of the accesses hit a hot set of H lines (R-MAT hubs: the top 500K rows of
// 63M take 53% of the column references) -- hot lines either CONTIGUOUS (the first H lines: what a
// degree-ordered relabelling produces, few 2 MB pages) or SCATTERED uniformly over the buffer (R-MAT
// vertex ids as generated).  Same lines, same reuse: any difference is page (TLB) locality.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_hot.cu -o gather_hot && ./gather_hot
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t& x) {
  x = x * 1664525u + 1013904223u;
  const uint32_t h = (x ^ (x >> 15)) * 2246822519u;
  return h ^ (h >> 13);
}

template <int U, bool SCATTER>
__global__ void __launch_bounds__(256) hot_kernel(const float4* __restrict__ buf, uint32_t mask, uint32_t hot,
                                                  uint32_t stride, uint32_t fthresh, int iters, float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 8 * 7919u + 1;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const uint32_t h = hash32(x);
      uint32_t row;
      if ((h >> 16) < fthresh) {                    // hot access
        const uint32_t k = hash32(x) % hot;
        row = SCATTER ? (k * stride) & mask : k;
      } else {
        row = hash32(x) & mask;
      }
      v[q] = __ldg(buf + static_cast<int64_t>(row) * 8 + (lane & 7));
    }
#pragma unroll
    for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const int64_t nrows = 1ll << 26;                  // 8 GB of 128-byte lines
  const uint32_t mask = static_cast<uint32_t>(nrows - 1);
  float4* buf = nullptr;
  float* out = nullptr;
  cudaMalloc(&buf, nrows * 128);
  cudaMalloc(&out, 64);
  cudaMemset(buf, 0, nrows * 128);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t hots[] = {250000, 500000, 1000000};
  const double fracs[] = {0.0, 0.42, 0.53, 0.63};
  for (uint32_t hot : hots) {
    const uint32_t stride = static_cast<uint32_t>(nrows / hot) | 1u;
    for (double f : fracs) {
      const uint32_t ft = static_cast<uint32_t>(f * 65536.0);
      for (int sc = 0; sc < 2; ++sc) {
        const int ctas = 148 * 4, thr = 256, iters = 128;
        auto launch = [&](int it) {
          if (sc) hot_kernel<8, true><<<ctas, thr>>>(buf, mask, hot, stride, ft, it, out);
          else hot_kernel<8, false><<<ctas, thr>>>(buf, mask, hot, stride, ft, it, out);
        };
        launch(2);
        cudaEventRecord(e0);
        launch(iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double lines = static_cast<double>(ctas) * thr / 8 * iters * 8;
        printf("{\"hot_lines\": %u, \"hot_MB\": %.0f, \"hot_fraction\": %.2f, \"hot_layout\": \"%s\", \"Glines_per_s\": %.2f}\n",
               hot, hot * 128.0 / 1e6, f, sc ? "scattered" : "contiguous", lines / (ms * 1e-3) / 1e9);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
