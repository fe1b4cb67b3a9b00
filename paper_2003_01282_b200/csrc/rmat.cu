// Device R-MAT generator + canonical CSR build (BASELINE C4/C5 shapes).
//
// Samples: edge_factor * 2^scale; sample j draws `scale` uniforms from a counter-based stream
// (splitmix64 of (seed, j, level)) and picks the quadrant per level with probabilities
// (a, b, c, d = 1-a-b-c), exactly as synth.rmat does on the host (but with this RNG).  The canonical
// CSR of graphs.py:110-132 (both directions, no self-loops, duplicates collapsed, rows and columns
// ascending) is built from directed keys row*n + col: radix sort, unique, then row offsets by binary
// search.  Peak memory is about 2 x 8 bytes x (2 * samples) + CUB scratch; the graph then owns
// int64 offsets and int32 columns only.  synth.rmat_device_reference() restates the same RNG on the
// host so small scales can be checked edge for edge.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

#include "slq_common.cuh"

namespace slq {

int graph_adopt(slq_graph* g, int64_t* offsets, int32_t* cols, cudaStream_t st, double* weights = nullptr);   // graph.cu

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// uniform in [0, 1) with 53 random bits, for (seed, sample, level)
__host__ __device__ __forceinline__ double rmat_uniform(uint64_t seed, uint64_t sample, int level) {
  const uint64_t h = splitmix64(splitmix64(seed ^ 0xD1B54A32D192ED03ull) ^ (sample * 64 + level));
  return static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void rmat_keys_kernel(uint64_t seed, int scale, int64_t samples, double a, double ab, double abc,
                                 uint64_t* __restrict__ keys) {
  const uint64_t n = 1ull << scale;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < samples;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t u = 0, v = 0;
    for (int level = 0; level < scale; ++level) {
      const double r = rmat_uniform(seed, static_cast<uint64_t>(j), level);
      const uint64_t bit = 1ull << (scale - 1 - level);
      if (r >= ab) u |= bit;                               // quadrants c, d: row bit
      if ((r >= a && r < ab) || r >= abc) v |= bit;        // quadrants b, d: column bit
    }
    // self-loops become a sentinel that sorts last and is dropped with the duplicates
    const uint64_t sentinel = ~0ull;
    keys[2 * j] = u == v ? sentinel : u * n + v;
    keys[2 * j + 1] = u == v ? sentinel : v * n + u;
  }
}

__global__ void keys_to_cols_kernel(const uint64_t* __restrict__ keys, int64_t nnz, int64_t n,
                                    int32_t* __restrict__ cols) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cols[i] = static_cast<int32_t>(keys[i] % static_cast<uint64_t>(n));
}

// offsets[r] = first key >= r*n (lower bound), r in [0, n]
__global__ void offsets_kernel(const uint64_t* __restrict__ keys, int64_t nnz, int64_t n, int64_t* __restrict__ off) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t target = static_cast<uint64_t>(r) * static_cast<uint64_t>(n);
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    off[r] = lo;
  }
}

}  // namespace slq

using namespace slq;

extern "C" int slq_graph_create_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                                     void* stream, slq_graph** out) {
  if (!out) return fail(SLQ_ERR_VALUE, "out must not be NULL");
  *out = nullptr;
  if (scale < 1 || scale > 30 || edge_factor < 1) return fail(SLQ_ERR_VALUE, "need 1 <= scale <= 30, edge_factor >= 1");
  if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return fail(SLQ_ERR_VALUE, "bad quadrant probabilities");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = 1ll << scale;
  const int64_t samples = static_cast<int64_t>(edge_factor) * n;
  const int64_t nkeys = 2 * samples;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  int64_t* d_count = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k0), sizeof(uint64_t) * nkeys, st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k1), sizeof(uint64_t) * nkeys, st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_count), sizeof(int64_t), st));
  {
    LaunchScope ls(K_PREPARE, st);
    rmat_keys_kernel<<<148 * 32, 256, 0, st>>>(seed, scale, samples, a, a + b, a + b + c, k0);
  }
  // sort directed keys (the sentinel needs all 64 bits); the DoubleBuffer form needs no third buffer
  cub::DoubleBuffer<uint64_t> db(k0, k1);
  size_t tb_sort = 0, tb_uniq = 0;
  SLQ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, db, nkeys, 0, 64, st));
  SLQ_CUDA(cub::DeviceSelect::Unique(nullptr, tb_uniq, k0, k1, d_count, nkeys, st));
  void* tmp = nullptr;
  SLQ_CUDA(cudaMallocAsync(&tmp, std::max(tb_sort, tb_uniq) + 256, st));
  SLQ_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb_sort, db, nkeys, 0, 64, st));
  uint64_t* sorted = db.Current();
  uint64_t* uniq = db.Alternate();
  SLQ_CUDA(cub::DeviceSelect::Unique(tmp, tb_uniq, sorted, uniq, d_count, nkeys, st));
  SLQ_CUDA(cudaFreeAsync(tmp, st));
  SLQ_CUDA(cudaFreeAsync(sorted, st));
  k0 = uniq;
  int64_t nuniq = 0;
  SLQ_CUDA(cudaMemcpyAsync(&nuniq, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  SLQ_CUDA(cudaFreeAsync(d_count, st));
  // the self-loop sentinel (if any sample was a self-loop) is the last unique key
  uint64_t last = 0;
  if (nuniq > 0) {
    SLQ_CUDA(cudaMemcpyAsync(&last, k0 + nuniq - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SLQ_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t nnz = (nuniq > 0 && last == ~0ull) ? nuniq - 1 : nuniq;
  int64_t* off = nullptr;
  int32_t* cols = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&off), sizeof(int64_t) * (n + 1), st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cols), sizeof(int32_t) * std::max<int64_t>(nnz, 1), st));
  {
    LaunchScope ls(K_PREPARE, st);
    keys_to_cols_kernel<<<148 * 32, 256, 0, st>>>(k0, nnz, n, cols);
  }
  {
    LaunchScope ls(K_PREPARE, st);
    offsets_kernel<<<148 * 32, 256, 0, st>>>(k0, nnz, n, off);
  }
  SLQ_CUDA(cudaFreeAsync(k0, st));
  slq_graph* g = new slq_graph();
  g->n = n;
  g->nnz = nnz;
  g->stream = stream;
  cudaGetDevice(&g->device);
  ensure_pool(g->device);
  { size_t fr = 0; cudaMemGetInfo(&fr, &g->device_total_mem); }
  const int rc = graph_adopt(g, off, cols, st);
  if (rc != SLQ_OK) {
    slq_graph_destroy(g);
    return rc;
  }
  *out = g;
  return SLQ_OK;
}

namespace slq {

// directed keys of an edge list: both directions, self-loops and out-of-range endpoints become the
// sentinel (out of range also sets *bad); weights duplicated to both directions
__global__ void edge_keys_kernel(const int64_t* __restrict__ u, const int64_t* __restrict__ v,
                                 const double* __restrict__ w, int64_t m, int64_t n, uint64_t* __restrict__ keys,
                                 double* __restrict__ wout, int* __restrict__ bad) {
  const uint64_t sentinel = ~0ull;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t a = u[e], b = v[e];
    const bool range = a >= 0 && a < n && b >= 0 && b < n;
    if (!range) atomicOr(bad, 1);
    const bool keep = range && a != b;
    keys[2 * e] = keep ? static_cast<uint64_t>(a) * static_cast<uint64_t>(n) + static_cast<uint64_t>(b) : sentinel;
    keys[2 * e + 1] = keep ? static_cast<uint64_t>(b) * static_cast<uint64_t>(n) + static_cast<uint64_t>(a) : sentinel;
    if (wout) {
      const double x = w[e];
      wout[2 * e] = x;
      wout[2 * e + 1] = x;
    }
  }
}

struct MaxWeight {
  __device__ __forceinline__ double operator()(double a, double b) const { return a > b ? a : b; }
};

}  // namespace slq

// Edge list (u[m], v[m], optional w[m]; host or device pointers) -> canonical CSR on the device,
// the semantics of graphs.csr_from_edges (graphs.py:110-132): self-loops dropped, both directions
// stored, duplicates collapsed to the maximum weight, rows and columns ascending.
extern "C" int slq_graph_create_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v, const double* w,
                                      void* stream, slq_graph** out) {
  if (!out) return fail(SLQ_ERR_VALUE, "out must not be NULL");
  *out = nullptr;
  if (n < 0 || m < 0) return fail(SLQ_ERR_VALUE, "negative n or m");
  if (n >= (int64_t(1) << 31)) return fail(SLQ_ERR_VALUE, "n >= 2^31 is not supported (int32 columns)");
  if (m > 0 && (!u || !v)) return fail(SLQ_ERR_VALUE, "NULL edge array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nkeys = 2 * m;
  int64_t *du = nullptr, *dv = nullptr, *d_count = nullptr;
  double* dw = nullptr;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  double *w0 = nullptr, *w1 = nullptr;
  int* bad = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), 16, st));   // [0] bad flag, [8] unique count
  d_count = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(bad) + 8);
  SLQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  int64_t nuniq = 0;
  if (m > 0) {
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&du), sizeof(int64_t) * m, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dv), sizeof(int64_t) * m, st));
    SLQ_CUDA(cudaMemcpyAsync(du, u, sizeof(int64_t) * m, cudaMemcpyDefault, st));
    SLQ_CUDA(cudaMemcpyAsync(dv, v, sizeof(int64_t) * m, cudaMemcpyDefault, st));
    if (w) {
      SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dw), sizeof(double) * m, st));
      SLQ_CUDA(cudaMemcpyAsync(dw, w, sizeof(double) * m, cudaMemcpyDefault, st));
      SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w0), sizeof(double) * nkeys, st));
      SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w1), sizeof(double) * nkeys, st));
    }
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k0), sizeof(uint64_t) * nkeys, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k1), sizeof(uint64_t) * nkeys, st));
    {
      LaunchScope ls(K_PREPARE, st);
      edge_keys_kernel<<<148 * 32, 256, 0, st>>>(du, dv, dw, m, n, k0, w0, bad);
    }
    SLQ_CUDA(cudaFreeAsync(du, st));
    SLQ_CUDA(cudaFreeAsync(dv, st));
    if (dw) SLQ_CUDA(cudaFreeAsync(dw, st));
    size_t tb_sort = 0, tb_red = 0;
    void* tmp = nullptr;
    if (!w) {
      cub::DoubleBuffer<uint64_t> db(k0, k1);
      SLQ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb_sort, db, nkeys, 0, 64, st));
      SLQ_CUDA(cub::DeviceSelect::Unique(nullptr, tb_red, k0, k1, d_count, nkeys, st));
      SLQ_CUDA(cudaMallocAsync(&tmp, std::max(tb_sort, tb_red) + 256, st));
      SLQ_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb_sort, db, nkeys, 0, 64, st));
      uint64_t* sorted = db.Current();
      uint64_t* uniq = db.Alternate();
      SLQ_CUDA(cub::DeviceSelect::Unique(tmp, tb_red, sorted, uniq, d_count, nkeys, st));
      k0 = uniq;
      k1 = sorted;
    } else {
      // stable key sort carrying the weights, then max over equal keys
      cub::DoubleBuffer<uint64_t> db(k0, k1);
      cub::DoubleBuffer<double> dbw(w0, w1);
      SLQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, db, dbw, nkeys, 0, 64, st));
      SLQ_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tb_red, k0, k1, w0, w1, d_count, MaxWeight(), nkeys, st));
      SLQ_CUDA(cudaMallocAsync(&tmp, std::max(tb_sort, tb_red) + 256, st));
      SLQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_sort, db, dbw, nkeys, 0, 64, st));
      uint64_t* ks = db.Current();
      double* ws = dbw.Current();
      uint64_t* ku = db.Alternate();
      double* wu = dbw.Alternate();
      SLQ_CUDA(cub::DeviceReduce::ReduceByKey(tmp, tb_red, ks, ku, ws, wu, d_count, MaxWeight(), nkeys, st));
      k0 = ku;
      k1 = ks;
      w0 = wu;
      w1 = ws;
    }
    SLQ_CUDA(cudaFreeAsync(tmp, st));
    SLQ_CUDA(cudaFreeAsync(k1, st));
    if (w1) SLQ_CUDA(cudaFreeAsync(w1, st));
  }
  int hbad = 0;
  SLQ_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (m > 0) SLQ_CUDA(cudaMemcpyAsync(&nuniq, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  SLQ_CUDA(cudaFreeAsync(bad, st));
  if (hbad) {
    if (k0) cudaFreeAsync(k0, st);
    if (w0) cudaFreeAsync(w0, st);
    return fail(SLQ_ERR_VALUE, "edge endpoint out of range");
  }
  uint64_t last = 0;
  if (nuniq > 0) {
    SLQ_CUDA(cudaMemcpyAsync(&last, k0 + nuniq - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SLQ_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t nnz = (nuniq > 0 && last == ~0ull) ? nuniq - 1 : nuniq;
  int64_t* off = nullptr;
  int32_t* cols = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&off), sizeof(int64_t) * (n + 1), st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cols), sizeof(int32_t) * std::max<int64_t>(nnz, 1), st));
  if (nnz > 0) {
    LaunchScope ls(K_PREPARE, st);
    keys_to_cols_kernel<<<148 * 32, 256, 0, st>>>(k0, nnz, n, cols);
  }
  {
    LaunchScope ls(K_PREPARE, st);
    offsets_kernel<<<148 * 32, 256, 0, st>>>(k0, nnz, n, off);
  }
  if (k0) SLQ_CUDA(cudaFreeAsync(k0, st));
  slq_graph* g = new slq_graph();
  g->n = n;
  g->nnz = nnz;
  g->stream = stream;
  cudaGetDevice(&g->device);
  ensure_pool(g->device);
  { size_t fr = 0; cudaMemGetInfo(&fr, &g->device_total_mem); }
  const int rc = graph_adopt(g, off, cols, st, w0);   // w0: max weights aligned with the unique keys
  if (rc != SLQ_OK) {
    slq_graph_destroy(g);
    return rc;
  }
  *out = g;
  return SLQ_OK;
}

extern "C" int slq_rmat_uniform_host(uint64_t seed, uint64_t sample, int level, double* out) {
  if (!out) return fail(SLQ_ERR_VALUE, "NULL output");
  *out = rmat_uniform(seed, sample, level);
  return SLQ_OK;
}
