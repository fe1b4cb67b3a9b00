// Random-row gather bandwidth on one GPU: warps read rows of `row_bytes` at uniformly random row
// indices of a `buf_gb` buffer (the SpMM's access pattern on a graph with no locality).  Reports
// useful GB/s for several row sizes and loads in flight.  nvcc -O3 -arch=sm_100a gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

// each group of G lanes reads one row of G*4 bytes (G = 8, 16, 32); U rows in flight per group
template <int G, int U>
__global__ void gather(const float* __restrict__ buf, int64_t nrows, int64_t iters, float* out) {
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  float acc = 0.f;
  // cheap 32-bit index stream (nrows is a power of two): a few integer ops per row
  const uint32_t mask = static_cast<uint32_t>(nrows - 1);
  uint32_t x = static_cast<uint32_t>(mix(gid + 1));
  for (int64_t it = 0; it < iters; ++it) {
    float v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      x = x * 1664525u + 1013904223u;
      const uint32_t h = (x ^ (x >> 15)) * 2246822519u;
      const int64_t row = static_cast<int64_t>((h ^ (h >> 13)) & mask);
      v[q] = __ldg(buf + row * G + gl);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) acc += v[q];
  }
  if (acc == 12345.f) out[0] = acc;
  (void)grp;
}

template <int G, int U>
void run(const float* buf, int64_t bytes, float* out, int blocks, int threads) {
  const int64_t nrows = bytes / (G * 4);
  const int64_t iters = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  gather<G, U><<<blocks, threads>>>(buf, nrows, 8, out);
  cudaEventRecord(e0);
  gather<G, U><<<blocks, threads>>>(buf, nrows, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const double groups = static_cast<double>(blocks) * threads / G;
  const double useful = groups * iters * U * G * 4;
  printf("{\"buf_GB\": %.2f, \"row_bytes\": %d, \"in_flight_per_group\": %d, \"blocks\": %d, \"GBps\": %.1f}\n",
         bytes / 1e9, G * 4, U, blocks, useful / (ms * 1e-3) / 1e9);
}

int main() {
  const int64_t maxbytes = 32ll << 30;
  float* buf = nullptr; float* out = nullptr;
  cudaMalloc(&buf, maxbytes); cudaMalloc(&out, 64);
  cudaMemset(buf, 0, maxbytes);
  for (int64_t mb : {64ll, 256ll, 1024ll, 2048ll, 4096ll, 8192ll, 32768ll}) {
    const int64_t bytes = mb << 20;
    const int blocks = 148 * 8, threads = 256;
    run<16, 8>(buf, bytes, out, blocks, threads);
    run<32, 8>(buf, bytes, out, blocks, threads);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
