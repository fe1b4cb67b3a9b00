// Shared definitions for the sm_100a SLQ engine (libslq_b200.so).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/slq_b200.h"

namespace slq {

constexpr int kWarp = 32;
constexpr int kMaxSteps = 128;     // longest rule held in registers/local memory (longer: global scratch)
constexpr int kMaxStepsLong = 4096;   // largest Lanczos step budget accepted (the reference has no cap)
constexpr int kCgsBlock = 16;      // basis vectors handled per CGS sweep (register accumulators)
constexpr int64_t kLongRow = 1024;  // rows with more nonzeros are split into segments ...
constexpr int64_t kSeg = 1024;      // ... of this many nonzeros, one warp each

// --- error state (thread local, see slq_last_error) -------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SLQ_CUDA(call)                                         \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::slq::cuda_fail(_e, #call); \
  } while (0)

// --- launch accounting + optional per-class CUDA-event timing ----------------
enum KernelClass {
  K_PREPARE = 0,
  K_PROBE,
  K_SPMM,
  K_CGS_DOT,
  K_CGS_UPDATE,
  K_REDUCE,
  K_EIG,
  K_QUAD,
  K_ESTIMATE,
  K_BATCHED,
  K_NUM_CLASSES
};

void ensure_pool(int dev);   // keep the stream-ordered allocator's memory cached
}  // namespace slq
struct slq_graph;
namespace slq {
int fetch_host_scalars(slq_graph* g);
// single small graph on the batched kernel (batched.cu); slq_rules routes n <= small_graph_max_n()
int64_t small_graph_max_n();
struct SeedKey;
int small_rules(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, int64_t count, int S, int dtype,
                double* nodes, double* weights, int32_t* steps_out, int32_t* status, cudaStream_t st);

void launch_begin(KernelClass k, cudaStream_t s);
void launch_end(KernelClass k, cudaStream_t s);

struct LaunchScope {
  KernelClass k;
  cudaStream_t s;
  LaunchScope(KernelClass k_, cudaStream_t s_) : k(k_), s(s_) { launch_begin(k, s); }
  ~LaunchScope() { launch_end(k, s); }
};

// --- device helpers ----------------------------------------------------------
template <typename T>
__device__ __forceinline__ double to_f64(T x) { return static_cast<double>(x); }

template <typename T>
__device__ __forceinline__ T from_f64(double x) { return static_cast<T>(x); }

__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }
__device__ __forceinline__ double ldg_f64(const float* p) { return static_cast<double>(__ldg(p)); }

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace slq

// Opaque graph handle (definition shared by the .cu files).
struct slq_graph {
  int64_t n = 0;
  int64_t nnz = 0;
  int64_t m = 0;                 // undirected edges = nnz / 2 for simple graphs
  int device = 0;
  size_t device_total_mem = 0;       // recorded at creation (chunk budget while a stream is captured)
  void* stream = nullptr;            // creation stream: owned buffers are freed on it
  const int64_t* offsets = nullptr;  // [n+1] device (owned copy)
  const int32_t* cols = nullptr;     // [nnz] device, narrowed to int32
  const double* weights = nullptr;   // [nnz] device, nullptr when every weight is 1.0
  double* degree = nullptr;          // [n]
  double* dinv = nullptr;            // [n]  1/sqrt(d) (0 for isolated)
  // SpMM tiles: contiguous row ranges with bounded (nnz + row) cost, fixed per graph
  int ntiles = 0;
  int64_t* tile_rows = nullptr;      // [ntiles+1] device
  int nftiles = 0;                   // fine tiles of the flat SpMM (large graphs; same allocation)
  int64_t* ftile_rows = nullptr;     // [nftiles+1] device
  // streaming tiles (pass B): contiguous equal row ranges
  int ntiles_stream = 0;
  int64_t rows_per_stream_tile = 0;
  // device scalars: [0] tr L, [1] max degree, [2] #isolated, [3] 1/tr L, [4] 2*max degree
  double* dscal = nullptr;
  int* dflags = nullptr;    // [0] out-of-range column seen, [1] a weight != 1.0
  // host copies of the scalars (filled lazily by fetch_host_scalars)
  int host_valid = 0;
  int bad_columns = 0;
  double trace_l = 0.0;     // sum of degrees (tr L)
  double max_degree = 0.0;
  int64_t isolated = 0;
  int unit_weights = 1;
  // long rows split into kSeg-nonzero segments (device counts: [0] long rows, [1] segments)
  int64_t max_long = 0, max_seg = 0;   // host upper bounds
  int64_t* long_counts = nullptr;
  int32_t* long_rows = nullptr;        // [max_long]
  int64_t* long_seg_first = nullptr;   // [max_long+1] first segment of each long row
  int32_t* seg_row = nullptr;          // [max_seg]
  int64_t* seg_begin = nullptr;        // [max_seg] first nonzero of each segment
  // isolated-vertex fold (slq_graph_fold_isolated): the graph without its unreferenced empty rows
  // plus ONE trailing empty row that stands for all of them (see graph.cu)
  slq_graph* folded = nullptr;
  int32_t* fold_remap = nullptr;       // [n] original vertex -> folded row, -1 for folded-away rows
  int64_t fold_m = 0;                  // vertices folded into the trailing row
  int degree_ordered = 0;              // (a fold) rows renumbered by descending degree: hubs first
  // owned device allocations
  void* owned[12] = {nullptr};
  int n_owned = 0;
};
