// TMA tile::gather4 on sm_100a: correctness of the smem layout and random-row gather throughput
// against plain warp loads, for rows of `cols` fp64 (the SpMM's gathered probe rows).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather4_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(phase) : "memory");
  }
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3,
                                        uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}

__global__ void layout_kernel(const __grid_constant__ CUtensorMap map, int cols, double* out) {
  __shared__ alignas(128) double buf[4 * 256];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect(&bar, 4 * cols * 8);
    gather4(buf, &map, 0, 5, 17, 2, 9, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 4 * cols; i += blockDim.x) out[i] = buf[i];
}

// each CTA: one producer lane keeps D gather4s in flight into a ring; all threads then sum the rows
template <int D>
__global__ void tma_bw_kernel(const __grid_constant__ CUtensorMap map, int cols, uint32_t mask, int iters, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  double* ring = reinterpret_cast<double*>(sm + 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t x = blockIdx.x * 7919u + 1;
  auto rnd = [&]() { x = x * 1664525u + 1013904223u; uint32_t h = (x ^ (x >> 15)) * 2246822519u; return (h ^ (h >> 13)) & mask; };
  double acc = 0.0;
  if (threadIdx.x == 0)
    for (int s = 0; s < D; ++s) {
      mbar_expect(&bars[s], 4 * cols * 8);
      gather4(ring + s * 4 * cols, &map, 0, rnd(), rnd(), rnd(), rnd(), &bars[s]);
    }
  for (int it = 0; it < iters; ++it) {
    const int s = it % D;
    mbar_wait(&bars[s], (it / D) & 1);
    for (int i = threadIdx.x; i < 4 * cols; i += blockDim.x) acc += ring[s * 4 * cols + i];
    __syncthreads();
    if (threadIdx.x == 0 && it + D < iters) {
      mbar_expect(&bars[s], 4 * cols * 8);
      gather4(ring + s * 4 * cols, &map, 0, rnd(), rnd(), rnd(), rnd(), &bars[s]);
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

// plain loads: each warp reads rows (lane = column chunk) with U rows in flight per lane
template <int U>
__global__ void ld_bw_kernel(const double* __restrict__ u, int cols, uint32_t mask, int iters, double* out) {
  const int lane = threadIdx.x & 31;
  uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 7919u + 1;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    double v[U][4];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      x = x * 1664525u + 1013904223u;
      uint32_t h = (x ^ (x >> 15)) * 2246822519u;
      const uint32_t row = (h ^ (h >> 13)) & mask;
#pragma unroll
      for (int j = 0; j < 4; ++j) v[q][j] = (lane + 32 * j < cols) ? __ldg(u + static_cast<int64_t>(row) * cols + lane + 32 * j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc += v[q][j];
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  if (!encode) { printf("{\"error\": \"no cuTensorMapEncodeTiled\"}\n"); return 1; }
  for (int cols : {100, 16, 128}) {
    for (int64_t nrows : {1ll << 17, 1ll << 23}) {   // 100k-row L2-resident block vs 8M rows (> L2)
      double* u = nullptr; double* out = nullptr;
      cudaMalloc(&u, nrows * cols * 8); cudaMalloc(&out, 4096 * 8);
      std::vector<double> h(static_cast<size_t>(nrows) * cols);
      for (int64_t r = 0; r < nrows; ++r) for (int c = 0; c < cols; ++c) h[r * cols + c] = r * 1000.0 + c;
      cudaMemcpy(u, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      CUtensorMap map;
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(nrows)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 8};
      cuuint32_t box[2] = {static_cast<cuuint32_t>(cols), 1};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, u, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("{\"cols\": %d, \"encode_error\": %d}\n", cols, (int)r); continue; }
      layout_kernel<<<1, 128>>>(map, cols, out);
      std::vector<double> o(4 * cols);
      cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
      const int rows[4] = {5, 17, 2, 9};
      bool ok = cudaGetLastError() == cudaSuccess;
      for (int i = 0; i < 4; ++i) for (int c = 0; c < cols; ++c) ok = ok && o[i * cols + c] == rows[i] * 1000.0 + c;
      const uint32_t mask = static_cast<uint32_t>(nrows - 1);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      const int iters = 2000;
      const int D = 8;
      const size_t smem = 128 + D * 4 * cols * 8;
      cudaFuncSetAttribute(tma_bw_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int ctas = 148 * 4;
      tma_bw_kernel<D><<<ctas, 128, smem>>>(map, cols, mask, 10, out);
      cudaEventRecord(e0);
      tma_bw_kernel<D><<<ctas, 128, smem>>>(map, cols, mask, iters, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms_tma = 0; cudaEventElapsedTime(&ms_tma, e0, e1);
      const double bytes_tma = static_cast<double>(ctas) * iters * 4 * cols * 8;
      ld_bw_kernel<2><<<148 * 8, 256>>>(u, cols, mask, 10, out);
      cudaEventRecord(e0);
      ld_bw_kernel<2><<<148 * 8, 256>>>(u, cols, mask, iters / 4, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms_ld = 0; cudaEventElapsedTime(&ms_ld, e0, e1);
      const double bytes_ld = static_cast<double>(148 * 8 * 8) * (iters / 4) * 2 * cols * 8;
      cudaError_t err = cudaGetLastError();
      printf("{\"cols\": %d, \"rows\": %lld, \"layout_ok\": %s, \"tma_gather4_GBps\": %.0f, \"ld_GBps\": %.0f, \"err\": \"%s\"}\n",
             cols, (long long)nrows, ok ? "true" : "false", bytes_tma / (ms_tma * 1e6), bytes_ld / (ms_ld * 1e6),
             cudaGetErrorString(err));
      cudaFree(u); cudaFree(out);
    }
  }
  return 0;
}
