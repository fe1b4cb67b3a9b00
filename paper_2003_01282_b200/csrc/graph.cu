// Device graph preparation: the work of operators.py:52-62 (_adjacency, degrees) and the
// per-operator set-up of make_operator (operators.py:65-102), done once per graph on the GPU:
//   * int64 -> int32 column narrowing (+ range check),
//   * unit-weight detection (weights dropped when all are 1.0: implicit CSR values),
//   * degrees d = A.1 as sequential in-row sums (bit-identical to scipy csr_matvec),
//   * dinv = 1/sqrt(d) with IEEE sqrt then divide (operators.py:85-86), 0 for isolated rows,
//   * tr L = sum d, max degree and isolated count (deterministic fixed-order reductions),
//   * the fixed SpMM row-tile partition (depends on the graph only, never on probe counts).
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "slq_common.cuh"

namespace slq {

constexpr int kMaxTiles = 148 * 256;  // SpMM warp tiles (dynamically scheduled): ~8 per resident warp
constexpr int kMaxStreamTiles = 148 * 16;
constexpr int64_t kMinTileCost = 64;
constexpr int64_t kFlatTileCost = 4096;   // flat SpMM work item (nonzeros + kRowCost per row)
constexpr int64_t kFlatMinNnz = int64_t(1) << 24;
constexpr int64_t kRowCost = 2;       // per-row overhead in nonzero-equivalents
constexpr int64_t kMinStreamRows = 128;

__global__ void narrow_cols_kernel(const int64_t* __restrict__ cols, int32_t* __restrict__ out,
                                   int64_t nnz, int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cols[i];
    const bool ok = c >= 0 && c < n;
    if (!ok) *bad = 1;
    out[i] = ok ? static_cast<int32_t>(c) : 0;   // clamped: no out-of-range gather ever happens
  }
}

// int32 columns given by the caller: range check in place (out-of-range -> flag, clamped to 0)
__global__ void check_cols_kernel(int32_t* __restrict__ cols, int64_t nnz, int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cols[i];
    if (c < 0 || c >= n) {
      *bad = 1;
      cols[i] = 0;
    }
  }
}

__global__ void unit_weight_kernel(const double* __restrict__ w, int64_t nnz, int* __restrict__ nonunit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x)
    if (w[i] != 1.0) *nonunit = 1;
}

// One thread per row: sequential sum in stored order (scipy csr_matvec with x = ones).
__global__ void degree_kernel(const int64_t* __restrict__ off, const double* __restrict__ w,
                              int64_t n, double* __restrict__ deg, double* __restrict__ dinv) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = off[r], e = off[r + 1];
    double s = 0.0;
    if (w) {
      for (int64_t k = b; k < e; ++k) s = __dadd_rn(s, __dmul_rn(w[k], 1.0));
    } else {
      s = static_cast<double>(e - b);   // exact: sum of ones, < 2^53
    }
    deg[r] = s;
    dinv[r] = s > 0.0 ? __ddiv_rn(1.0, __dsqrt_rn(s)) : 0.0;
  }
}

// Fixed-order block partials of (sum d, max d, #isolated); final pass in one block.
constexpr int kScalBlock = 256;
__global__ void degree_stats_kernel(const double* __restrict__ deg, int64_t n, int64_t per_block,
                                    double* __restrict__ psum, double* __restrict__ pmax,
                                    long long* __restrict__ piso) {
  __shared__ double ss[kScalBlock], sm[kScalBlock];
  __shared__ long long si[kScalBlock];
  const int64_t b = blockIdx.x * per_block, e = min(n, b + per_block);
  double s = 0.0, mx = 0.0;
  long long iso = 0;
  for (int64_t r = b + threadIdx.x; r < e; r += blockDim.x) {
    const double d = deg[r];
    s += d;
    mx = fmax(mx, d);
    iso += (d == 0.0);
  }
  ss[threadIdx.x] = s; sm[threadIdx.x] = mx; si[threadIdx.x] = iso;
  __syncthreads();
  for (int h = kScalBlock / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      ss[threadIdx.x] += ss[threadIdx.x + h];
      sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + h]);
      si[threadIdx.x] += si[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { psum[blockIdx.x] = ss[0]; pmax[blockIdx.x] = sm[0]; piso[blockIdx.x] = si[0]; }
}

__global__ void degree_stats_final(const double* psum, const double* pmax, const long long* piso,
                                   int nb, double* out3) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0, mx = 0.0;
    long long iso = 0;
    for (int i = 0; i < nb; ++i) { s += psum[i]; mx = fmax(mx, pmax[i]); iso += piso[i]; }
    out3[0] = s; out3[1] = mx; out3[2] = static_cast<double>(iso);
    out3[3] = s > 0.0 ? 1.0 / s : 0.0;    // density scale 1/tr L (operators.py:96)
    out3[4] = 2.0 * mx;                   // Laplacian interval hi (operators.py:79)
  }
}

// Long rows (degree > kLongRow) are split into kSeg-nonzero segments processed by separate warps
// (R-MAT hubs reach 64k nonzeros at scale 20).  Per-row segment counts, then exclusive scans.
__global__ void long_row_count_kernel(const int64_t* __restrict__ off, int64_t n, int64_t* __restrict__ nseg_row,
                                      int64_t* __restrict__ is_long) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = r < n ? off[r + 1] - off[r] : 0;
    const bool lng = d > kLongRow;
    nseg_row[r] = lng ? (d + kSeg - 1) / kSeg : 0;
    is_long[r] = lng ? 1 : 0;
  }
}

__global__ void long_row_fill_kernel(const int64_t* __restrict__ off, int64_t n, const int64_t* __restrict__ seg_first,
                                     const int64_t* __restrict__ long_idx, int32_t* __restrict__ long_rows,
                                     int64_t* __restrict__ long_seg_first, int32_t* __restrict__ seg_row,
                                     int64_t* __restrict__ seg_begin, int64_t* __restrict__ counts) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n;
       r += (int64_t)gridDim.x * blockDim.x) {
    if (r == n) {
      counts[0] = long_idx[n];
      counts[1] = seg_first[n];
      long_seg_first[long_idx[n]] = seg_first[n];
      continue;
    }
    const int64_t d = off[r + 1] - off[r];
    if (d <= kLongRow) continue;
    const int64_t lr = long_idx[r], sf = seg_first[r];
    long_rows[lr] = static_cast<int32_t>(r);
    long_seg_first[lr] = sf;
    const int64_t ns = (d + kSeg - 1) / kSeg;
    for (int64_t k = 0; k < ns; ++k) {
      seg_row[sf + k] = static_cast<int32_t>(r);
      seg_begin[sf + k] = off[r] + k * kSeg;
    }
  }
}

// tile_rows[t] = first row r with offsets[r] + kRowCost*r >= t*target (lower bound), t <= ntiles.
__global__ void tile_kernel(const int64_t* __restrict__ off, int64_t n, int64_t target, int ntiles,
                            int64_t* __restrict__ tile_rows) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  if (t == ntiles) { tile_rows[t] = n; return; }
  const int64_t key = static_cast<int64_t>(t) * target;
  int64_t lo = 0, hi = n;   // search in [0, n]
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] + kRowCost * mid >= key) hi = mid; else lo = mid + 1;
  }
  tile_rows[t] = lo;
}

static int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

static void* track(slq_graph* g, void* p) {
  g->owned[g->n_owned++] = p;
  return p;
}

// Fully stream-ordered: no host synchronisation.  Scalars stay on the device (g->dscal); the host
// mirror is fetched lazily by fetch_host_scalars() (slq_graph_info, Laplacian interval).
// Either copies (offsets, int64 cols) or adopts device buffers the caller allocated with
// cudaMallocAsync (adopt_off, adopt_cols: the graph frees them).
static int graph_build(slq_graph* g, const int64_t* offsets, const int64_t* cols, const double* weights,
                       cudaStream_t st, int64_t* adopt_off = nullptr, int32_t* adopt_cols = nullptr,
                       double* adopt_w = nullptr, bool check_adopted = false) {
  const int64_t n = g->n, nnz = g->nnz;
  void* p = nullptr;
  if (adopt_off) {
    g->offsets = static_cast<int64_t*>(track(g, adopt_off));
    g->cols = static_cast<int32_t*>(track(g, adopt_cols));
  } else {
    SLQ_CUDA(cudaMallocAsync(&p, sizeof(int64_t) * (n + 1), st));
    g->offsets = static_cast<int64_t*>(track(g, p));
    SLQ_CUDA(cudaMemcpyAsync(const_cast<int64_t*>(g->offsets), offsets, sizeof(int64_t) * (n + 1),
                             cudaMemcpyDefault, st));
    SLQ_CUDA(cudaMallocAsync(&p, sizeof(int32_t) * std::max<int64_t>(nnz, 1), st));
    g->cols = static_cast<int32_t*>(track(g, p));
  }
  // degree and dinv, each padded to an even length + 2 (16-byte aligned; bulk copies of dinv windows
  // may read one element past n)
  const int64_t dstride = ((std::max<int64_t>(n, 1) + 1) / 2) * 2 + 2;
  SLQ_CUDA(cudaMallocAsync(&p, sizeof(double) * dstride * 2, st));
  SLQ_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * dstride * 2, st));
  track(g, p);
  g->degree = static_cast<double*>(p);
  g->dinv = g->degree + dstride;
  SLQ_CUDA(cudaMallocAsync(&p, sizeof(double) * 8 + sizeof(int) * 4, st));
  track(g, p);
  g->dscal = static_cast<double*>(p);
  g->dflags = reinterpret_cast<int*>(g->dscal + 8);
  SLQ_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * 8 + sizeof(int) * 4, st));
  if (nnz > 0 && !adopt_cols) {
    LaunchScope ls(K_PREPARE, st);
    narrow_cols_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(cols, const_cast<int32_t*>(g->cols), nnz, n, g->dflags);
  } else if (nnz > 0 && check_adopted) {
    LaunchScope ls(K_PREPARE, st);
    check_cols_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(const_cast<int32_t*>(g->cols), nnz, n, g->dflags);
  }
  if ((weights || adopt_w) && nnz > 0) {
    // explicit weights are kept even if all are 1.0 (w * t == t exactly, so results are identical)
    if (adopt_w) {
      g->weights = static_cast<double*>(track(g, adopt_w));
    } else {
      SLQ_CUDA(cudaMallocAsync(&p, sizeof(double) * nnz, st));
      g->weights = static_cast<double*>(track(g, p));
      SLQ_CUDA(cudaMemcpyAsync(const_cast<double*>(g->weights), weights, sizeof(double) * nnz, cudaMemcpyDefault, st));
    }
    LaunchScope ls(K_PREPARE, st);
    unit_weight_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(g->weights, nnz, g->dflags + 1);
  }
  if (n > 0) {
    LaunchScope ls(K_PREPARE, st);
    degree_kernel<<<grid_for(n, 256), 256, 0, st>>>(g->offsets, g->weights, n, g->degree, g->dinv);
  }
  // degree statistics -> dscal
  const int64_t per_block = std::max<int64_t>(4096, (n + 1023) / 1024);
  const int nb = std::max(1, ceil_div(n, per_block));
  double* scratch = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * (3 * nb + 3), st));
  if (n > 0) {
    {
      LaunchScope ls(K_PREPARE, st);
      degree_stats_kernel<<<nb, kScalBlock, 0, st>>>(g->degree, n, per_block, scratch, scratch + nb,
                                                     reinterpret_cast<long long*>(scratch + 2 * nb));
    }
    LaunchScope ls(K_PREPARE, st);
    degree_stats_final<<<1, 32, 0, st>>>(scratch, scratch + nb, reinterpret_cast<long long*>(scratch + 2 * nb),
                                         nb, g->dscal);
  }
  SLQ_CUDA(cudaFreeAsync(scratch, st));
  // tiles
  const int64_t total = nnz + kRowCost * n;
  // small graphs get smaller tiles (down to 16 cost units) so their few rows still spread over
  // ~4 warps per SM; large graphs keep >= kMinTileCost per tile (scheduling overhead)
  const int64_t min_cost = std::min<int64_t>(kMinTileCost, std::max<int64_t>(16, total / (148 * 32)));
  int64_t target = std::max<int64_t>(min_cost, (total + kMaxTiles - 1) / kMaxTiles);
  g->ntiles = std::max(1, ceil_div(total, target));
  // fine tiles for the flat SpMM (spmm_flat.cu): large graphs only (SLQ_SPMM_FLAT=0 off, =1 any graph)
  static const int flat_env = [] { const char* e = getenv("SLQ_SPMM_FLAT"); return e ? atoi(e) : -1; }();
  const bool flat = flat_env != 0 && n > 0 && nnz > 0 && (flat_env > 0 || nnz >= kFlatMinNnz);
  g->nftiles = flat ? std::max(1, ceil_div(total, kFlatTileCost)) : 0;
  SLQ_CUDA(cudaMallocAsync(&p, sizeof(int64_t) * (g->ntiles + 1 + (flat ? g->nftiles + 1 : 0)), st));
  g->tile_rows = static_cast<int64_t*>(track(g, p));
  g->ftile_rows = flat ? g->tile_rows + g->ntiles + 1 : nullptr;
  {
    LaunchScope ls(K_PREPARE, st);
    tile_kernel<<<ceil_div(g->ntiles + 1, 256), 256, 0, st>>>(g->offsets, n, target, g->ntiles, g->tile_rows);
  }
  if (flat) {
    LaunchScope ls(K_PREPARE, st);
    tile_kernel<<<ceil_div(g->nftiles + 1, 256), 256, 0, st>>>(g->offsets, n, kFlatTileCost, g->nftiles, g->ftile_rows);
  }
  g->rows_per_stream_tile = std::max<int64_t>(kMinStreamRows, (n + kMaxStreamTiles - 1) / kMaxStreamTiles);
  g->ntiles_stream = std::max(1, ceil_div(n, g->rows_per_stream_tile));
  g->m = nnz / 2;
  // long-row segments (device-side counts; host-side upper bounds size the buffers)
  g->max_long = nnz / (kLongRow + 1) + 1;
  g->max_seg = nnz / kSeg + g->max_long + 1;
  SLQ_CUDA(cudaMallocAsync(&p, sizeof(int64_t) * (2 + (g->max_long + 1) + g->max_seg) +
                                   sizeof(int32_t) * (g->max_long + g->max_seg) + 64, st));
  track(g, p);
  g->long_counts = static_cast<int64_t*>(p);
  g->long_seg_first = g->long_counts + 2;
  g->seg_begin = g->long_seg_first + g->max_long + 1;
  g->long_rows = reinterpret_cast<int32_t*>(g->seg_begin + g->max_seg);
  g->seg_row = g->long_rows + g->max_long;
  SLQ_CUDA(cudaMemsetAsync(g->long_counts, 0, 2 * sizeof(int64_t), st));
  if (n > 0 && nnz > kLongRow) {
    int64_t* tmp = nullptr;   // [n+1] nseg_row, [n+1] is_long, [n+1] seg_first, [n+1] long_idx
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(int64_t) * 4 * (n + 1), st));
    {
      LaunchScope ls(K_PREPARE, st);
      long_row_count_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(g->offsets, n, tmp, tmp + (n + 1));
    }
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, tmp, tmp + 2 * (n + 1), static_cast<int>(n + 1), st);
    void* cubtmp = nullptr;
    SLQ_CUDA(cudaMallocAsync(&cubtmp, tb + 16, st));
    SLQ_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, tb, tmp, tmp + 2 * (n + 1), static_cast<int>(n + 1), st));
    SLQ_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, tb, tmp + (n + 1), tmp + 3 * (n + 1), static_cast<int>(n + 1), st));
    {
      LaunchScope ls(K_PREPARE, st);
      long_row_fill_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(g->offsets, n, tmp + 2 * (n + 1), tmp + 3 * (n + 1),
                                                                g->long_rows, g->long_seg_first, g->seg_row,
                                                                g->seg_begin, g->long_counts);
    }
    SLQ_CUDA(cudaFreeAsync(cubtmp, st));
    SLQ_CUDA(cudaFreeAsync(tmp, st));
  }
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

int graph_adopt(slq_graph* g, int64_t* offsets, int32_t* cols, cudaStream_t st, double* weights) {
  if (weights && g->nnz == 0) {
    cudaFreeAsync(weights, st);
    weights = nullptr;
  }
  return graph_build(g, nullptr, nullptr, nullptr, st, offsets, cols, weights);
}

// Host mirror of the device scalars (synchronises the creation stream once).
int fetch_host_scalars(slq_graph* g) {
  if (g->host_valid) return SLQ_OK;
  double sc[8];
  int fl[4];
  cudaStream_t st = static_cast<cudaStream_t>(g->stream);
  SLQ_CUDA(cudaMemcpyAsync(sc, g->dscal, sizeof(sc), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaMemcpyAsync(fl, g->dflags, sizeof(fl), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  g->trace_l = sc[0];
  g->max_degree = sc[1];
  g->isolated = static_cast<int64_t>(sc[2]);
  g->bad_columns = fl[0];
  g->unit_weights = fl[1] ? 0 : 1;
  g->host_valid = 1;
  return SLQ_OK;
}

// ----------------------------------------------------------------------------- isolated-vertex fold
// A vertex whose row is empty and which no row references is isolated in the operator sense: every
// operator kind gives y_v = 0 (operators.py:76-99: d_v = 0, dinv_v = 0, no neighbours).  In the
// Lanczos recurrence such a row only ever sees row-local linear updates (three-term, CGS
// subtraction, 1/beta), whose arithmetic is sign-symmetric, so u_k[v] = z_v * e_k with the probe sign
// z_v = +-1 and ONE per-probe scalar sequence e_k shared by all isolated rows (bit for bit).  The fold
// drops those rows and appends a single empty row that carries sqrt(m) * e_k for the m of them: every
// dot product over the original rows equals the folded one up to rounding (m e_k e_l), while the
// vectors shrink by m rows.  The relabelling is monotone, so rows keep their stored column order and
// the SpMM's in-row sums are bitwise those of the unfolded graph.
__global__ void fold_mark_rows_kernel(const int64_t* __restrict__ off, int64_t n, int32_t* __restrict__ keep) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x)
    keep[v] = v < n && off[v + 1] > off[v] ? 1 : 0;
}

__global__ void fold_mark_cols_kernel(const int32_t* __restrict__ cols, int64_t nnz, int32_t* __restrict__ keep) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cols[e];
    if (!keep[c]) keep[c] = 1;   // benign race: every writer stores 1
  }
}

// keep[] becomes the remap (folded row or -1) in place; off_f[newid[v]] = off[v] for kept rows and
// the trailing row n' is empty.
__global__ void fold_offsets_kernel(const int64_t* __restrict__ off, int32_t* __restrict__ keep_remap,
                                    const int32_t* __restrict__ newid, int64_t n, int64_t nprime, int64_t nnz,
                                    int64_t* __restrict__ off_f) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x) {
    if (v == n) {
      off_f[nprime] = nnz;
      off_f[nprime + 1] = nnz;
      continue;
    }
    const bool k = keep_remap[v] != 0;
    if (k) off_f[newid[v]] = off[v];
    keep_remap[v] = k ? newid[v] : -1;
  }
}

__global__ void fold_cols_kernel(const int32_t* __restrict__ cols, const int32_t* __restrict__ newid, int64_t nnz,
                                 int32_t* __restrict__ cols_f) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    cols_f[e] = newid[cols[e]];
}

// Degree-ordered fold (default): the kept vertices are renumbered by DESCENDING degree (ties: original
// order), so the rows most nonzeros reference (R-MAT hubs: the top 1M of 63M rows take 63% of the
// column references) sit in the first few hundred MB of every Lanczos vector.  The SpMM's random
// 128-byte row gathers then touch few 2 MB pages for most nonzeros: measured (gather_hot.cu) 36 ->
// 52-56 G lines/s for 53-63% of gathers on a contiguous 64 MB hot set, no gain when the same hot set is
// scattered (the gather rate over an 8 GB vector is bound by address translation, not by DRAM or L2).
// Each row keeps its stored column order, so its in-row sum is bitwise the unfolded one; the
// reductions over rows run in the new row order (equal to rounding).
__global__ void fold_sort_keys_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ keep, int64_t n,
                                      int32_t* __restrict__ keys, int32_t* __restrict__ ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    keys[v] = keep[v] ? static_cast<int32_t>(off[v + 1] - off[v]) : -1;   // dropped vertices sort last
    ids[v] = static_cast<int32_t>(v);
  }
}

// perm[r] = old vertex of new row r (r < n'): newid[old] = r, -1 for dropped vertices; row lengths in
// the new order for the offsets scan (the trailing virtual row and the scan's end entry are empty)
__global__ void fold_perm_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ perm, int64_t n,
                                 int64_t nprime, int32_t* __restrict__ newid, int64_t* __restrict__ len_new) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n + 2; r += (int64_t)gridDim.x * blockDim.x) {
    if (r < n) {
      const int32_t v = perm[r];
      newid[v] = r < nprime ? static_cast<int32_t>(r) : -1;
    }
    if (r <= nprime + 1) len_new[r] = r < nprime ? off[perm[r] + 1] - off[perm[r]] : 0;
  }
}

// one warp per new row: copy the old row's columns (stored order) relabelled, and its weights
__global__ void fold_rows_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ cols,
                                 const double* __restrict__ w, const int32_t* __restrict__ perm,
                                 const int32_t* __restrict__ newid, const int64_t* __restrict__ off_f, int64_t nprime,
                                 int32_t* __restrict__ cols_f, double* __restrict__ w_f) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < nprime; r += warps) {
    const int64_t src = off[perm[r]], dst = off_f[r], len = off_f[r + 1] - dst;
    for (int64_t k = lane; k < len; k += 32) {
      cols_f[dst + k] = newid[cols[src + k]];
      if (w) w_f[dst + k] = w[src + k];
    }
  }
}

static bool fold_by_degree() {
  static const bool v = [] { const char* e = getenv("SLQ_FOLD_ORDER"); return !(e && e[0] == 'm'); }();
  return v;   // SLQ_FOLD_ORDER=monotone keeps the original vertex order (A/B)
}

static void drop_fold(slq_graph* g) {
  if (g->folded) slq_graph_destroy(g->folded);
  if (g->fold_remap) cudaFreeAsync(g->fold_remap, static_cast<cudaStream_t>(g->stream));
  g->folded = nullptr;
  g->fold_remap = nullptr;
  g->fold_m = 0;
}

static int graph_fold(slq_graph* g, double min_fraction, int64_t* folded_out) {
  *folded_out = 0;
  if (min_fraction < 0.0) {
    drop_fold(g);
    return SLQ_OK;
  }
  if (g->folded) {
    *folded_out = g->fold_m;
    return SLQ_OK;
  }
  int rc = fetch_host_scalars(g);
  if (rc) return rc;
  const int64_t n = g->n, nnz = g->nnz;
  // Large unit-weight graphs are "folded" even without (enough) isolated vertices: the fold's degree
  // order is what the flat SpMM (spmm_flat.cu) needs, the trailing row then stands for m >= 0 vertices
  // (m = 0: a row that stays 0).  SLQ_FOLD_RELABEL=0 turns this off.
  static const bool relabel_env = [] { const char* e = getenv("SLQ_FOLD_RELABEL"); return !(e && e[0] == '0'); }();
  const bool relabel = relabel_env && fold_by_degree() && nnz >= kFlatMinNnz && !g->weights && n < (int64_t(1) << 29);
  // degree-0 vertices bound the foldable ones from above; nothing to do below the threshold
  if (g->bad_columns || nnz == 0) return SLQ_OK;
  if (!relabel && (g->isolated < 1 || static_cast<double>(g->isolated) < min_fraction * static_cast<double>(n)))
    return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(g->stream);
  {
    // the fold holds a second CSR: skip it (not an error) when the device cannot hold it comfortably
    size_t freeb = 0, total = 0;
    cudaMemGetInfo(&freeb, &total);
    double avail = static_cast<double>(freeb);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
      uint64_t reserved = 0, used = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      if (reserved > used) avail += static_cast<double>(reserved - used);
    }
    const double need = 40.0 * static_cast<double>(n) + (g->weights ? 12.0 : 4.0) * static_cast<double>(nnz) +
                        static_cast<double>(1ull << 28);
    if (need > 0.9 * avail) return SLQ_OK;
  }
  int32_t* keep = nullptr;    // [n+1] keep flags, then the remap
  int32_t* newid = nullptr;   // [n+1] exclusive scan of keep
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keep), sizeof(int32_t) * (n + 1), st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&newid), sizeof(int32_t) * (n + 1), st));
  {
    LaunchScope ls(K_PREPARE, st);
    fold_mark_rows_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(g->offsets, n, keep);
    fold_mark_cols_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(g->cols, nnz, keep);
  }
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, newid, static_cast<int>(n + 1), st);
  void* cubtmp = nullptr;
  SLQ_CUDA(cudaMallocAsync(&cubtmp, tb + 16, st));
  SLQ_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp, tb, keep, newid, static_cast<int>(n + 1), st));
  SLQ_CUDA(cudaFreeAsync(cubtmp, st));
  int32_t nprime32 = 0;
  SLQ_CUDA(cudaMemcpyAsync(&nprime32, newid + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  const int64_t nprime = nprime32, m = n - nprime;
  if (!relabel && (m < 1 || static_cast<double>(m) < min_fraction * static_cast<double>(n))) {
    cudaFreeAsync(keep, st);
    cudaFreeAsync(newid, st);
    return SLQ_OK;
  }
  int64_t* off_f = nullptr;
  int32_t* cols_f = nullptr;
  double* w_f = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&off_f), sizeof(int64_t) * (nprime + 2), st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cols_f), sizeof(int32_t) * nnz, st));
  if (g->weights) SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w_f), sizeof(double) * nnz, st));
  if (fold_by_degree()) {
    // keys/ids -> sorted by descending degree (stable: ties keep the original order)
    int32_t *keys = nullptr, *ids = nullptr, *keys_s = nullptr, *perm = nullptr;
    int64_t* len_new = nullptr;
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys), sizeof(int32_t) * n, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ids), sizeof(int32_t) * n, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys_s), sizeof(int32_t) * n, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&perm), sizeof(int32_t) * n, st));
    {
      LaunchScope ls(K_PREPARE, st);
      fold_sort_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(g->offsets, keep, n, keys, ids);
    }
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, sb, keys, keys_s, ids, perm, static_cast<int>(n), 0, 32, st);
    void* sorttmp = nullptr;
    SLQ_CUDA(cudaMallocAsync(&sorttmp, sb + 16, st));
    SLQ_CUDA(cub::DeviceRadixSort::SortPairsDescending(sorttmp, sb, keys, keys_s, ids, perm, static_cast<int>(n), 0,
                                                       32, st));
    SLQ_CUDA(cudaFreeAsync(sorttmp, st));
    SLQ_CUDA(cudaFreeAsync(keys, st));
    SLQ_CUDA(cudaFreeAsync(ids, st));
    SLQ_CUDA(cudaFreeAsync(keys_s, st));
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&len_new), sizeof(int64_t) * (nprime + 2), st));
    {
      LaunchScope ls(K_PREPARE, st);
      fold_perm_kernel<<<grid_for(n + 2, 256), 256, 0, st>>>(g->offsets, perm, n, nprime, newid, len_new);
    }
    size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, len_new, off_f, static_cast<int>(nprime + 2), st);
    void* scantmp = nullptr;
    SLQ_CUDA(cudaMallocAsync(&scantmp, tb2 + 16, st));
    SLQ_CUDA(cub::DeviceScan::ExclusiveSum(scantmp, tb2, len_new, off_f, static_cast<int>(nprime + 2), st));
    SLQ_CUDA(cudaFreeAsync(scantmp, st));
    SLQ_CUDA(cudaFreeAsync(len_new, st));
    {
      LaunchScope ls(K_PREPARE, st);
      fold_rows_kernel<<<grid_for(nprime * 32, 256), 256, 0, st>>>(g->offsets, g->cols, g->weights, perm, newid, off_f,
                                                                   nprime, cols_f, w_f);
    }
    SLQ_CUDA(cudaFreeAsync(perm, st));
    // the remap (original vertex -> folded row, -1 dropped) is newid; keep[] is no longer needed
    SLQ_CUDA(cudaFreeAsync(keep, st));
    keep = newid;
    newid = nullptr;
  } else {
    {
      LaunchScope ls(K_PREPARE, st);
      fold_offsets_kernel<<<grid_for(n + 1, 256), 256, 0, st>>>(g->offsets, keep, newid, n, nprime, nnz, off_f);
      fold_cols_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(g->cols, newid, nnz, cols_f);
    }
    SLQ_CUDA(cudaFreeAsync(newid, st));
    newid = nullptr;
    if (g->weights) SLQ_CUDA(cudaMemcpyAsync(w_f, g->weights, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st));
  }
  slq_graph* f = new slq_graph();
  f->n = nprime + 1;
  f->nnz = nnz;
  f->stream = g->stream;
  f->device = g->device;
  f->device_total_mem = g->device_total_mem;
  rc = graph_adopt(f, off_f, cols_f, st, w_f);
  if (rc) {
    slq_graph_destroy(f);
    cudaFreeAsync(keep, st);
    return rc;
  }
  // the operator scalars are the original graph's (tr L, max degree, 1/tr L, interval): the same
  // values, and for weighted graphs the same summation order
  SLQ_CUDA(cudaMemcpyAsync(f->dscal, g->dscal, sizeof(double) * 8, cudaMemcpyDeviceToDevice, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  SLQ_CUDA(cudaGetLastError());
  f->degree_ordered = fold_by_degree() ? 1 : 0;
  g->folded = f;
  g->fold_remap = keep;
  g->fold_m = m;
  *folded_out = m;
  return SLQ_OK;
}

}  // namespace slq

using namespace slq;

extern "C" int slq_graph_create(int64_t n, int64_t nnz, const int64_t* offsets, const int64_t* cols,
                                const double* weights, void* stream, slq_graph** out) {
  if (!out) return fail(SLQ_ERR_VALUE, "out must not be NULL");
  *out = nullptr;
  if (n < 0 || nnz < 0) return fail(SLQ_ERR_VALUE, "negative n or nnz");
  if (n >= (int64_t(1) << 31)) return fail(SLQ_ERR_VALUE, "n >= 2^31 is not supported (int32 columns)");
  if (!offsets || (nnz > 0 && !cols)) return fail(SLQ_ERR_VALUE, "NULL CSR array");
  slq_graph* g = new slq_graph();
  g->n = n;
  g->nnz = nnz;
  g->stream = stream;
  cudaGetDevice(&g->device);
  ensure_pool(g->device);
  { size_t fr = 0; cudaMemGetInfo(&fr, &g->device_total_mem); }
  int rc = graph_build(g, offsets, cols, weights, static_cast<cudaStream_t>(stream));
  if (rc != SLQ_OK) {
    slq_graph_destroy(g);
    return rc;
  }
  *out = g;
  return SLQ_OK;
}

extern "C" int slq_graph_create_host(int64_t n, int64_t nnz, const int64_t* offsets_host,
                                     const int64_t* cols_host, const double* weights_host, void* stream,
                                     slq_graph** out) {
  // H2D staging of the canonical CSR, then the device build.
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t* d_off = nullptr;
  int64_t* d_cols = nullptr;
  double* d_w = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_off), sizeof(int64_t) * (n + 1), st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_cols), sizeof(int64_t) * std::max<int64_t>(nnz, 1), st));
  SLQ_CUDA(cudaMemcpyAsync(d_off, offsets_host, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
  if (nnz > 0) SLQ_CUDA(cudaMemcpyAsync(d_cols, cols_host, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
  if (weights_host && nnz > 0) {
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_w), sizeof(double) * nnz, st));
    SLQ_CUDA(cudaMemcpyAsync(d_w, weights_host, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  }
  int rc = slq_graph_create(n, nnz, d_off, d_cols, d_w, stream, out);
  cudaFreeAsync(d_off, st);
  cudaFreeAsync(d_cols, st);
  if (d_w) cudaFreeAsync(d_w, st);
  return rc;
}

// int32 columns (the C5 data format: "int32 indices with fp32 values", implicit unit weights when
// weights == NULL); host or device pointers.  The copies land in buffers the graph adopts, so the
// device holds one int32 copy of the columns (no int64 staging).
extern "C" int slq_graph_create_i32(int64_t n, int64_t nnz, const int64_t* offsets, const int32_t* cols,
                                    const double* weights, void* stream, slq_graph** out) {
  if (!out) return fail(SLQ_ERR_VALUE, "out must not be NULL");
  *out = nullptr;
  if (n < 0 || nnz < 0) return fail(SLQ_ERR_VALUE, "negative n or nnz");
  if (n >= (int64_t(1) << 31)) return fail(SLQ_ERR_VALUE, "n >= 2^31 is not supported (int32 columns)");
  if (!offsets || (nnz > 0 && !cols)) return fail(SLQ_ERR_VALUE, "NULL CSR array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  slq_graph* g = new slq_graph();
  g->n = n;
  g->nnz = nnz;
  g->stream = stream;
  cudaGetDevice(&g->device);
  ensure_pool(g->device);
  { size_t fr = 0; cudaMemGetInfo(&fr, &g->device_total_mem); }
  int64_t* off = nullptr;
  int32_t* c = nullptr;
  double* w = nullptr;
  auto cleanup = [&]() {
    if (off) cudaFreeAsync(off, st);
    if (c) cudaFreeAsync(c, st);
    if (w) cudaFreeAsync(w, st);
    delete g;
  };
  if (cudaMallocAsync(reinterpret_cast<void**>(&off), sizeof(int64_t) * (n + 1), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&c), sizeof(int32_t) * std::max<int64_t>(nnz, 1), st) != cudaSuccess ||
      (weights && nnz > 0 && cudaMallocAsync(reinterpret_cast<void**>(&w), sizeof(double) * nnz, st) != cudaSuccess)) {
    cleanup();
    return fail(SLQ_ERR_ALLOC, "device allocation failed for the CSR");
  }
  if (cudaMemcpyAsync(off, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyDefault, st) != cudaSuccess ||
      (nnz > 0 && cudaMemcpyAsync(c, cols, sizeof(int32_t) * nnz, cudaMemcpyDefault, st) != cudaSuccess) ||
      (w && cudaMemcpyAsync(w, weights, sizeof(double) * nnz, cudaMemcpyDefault, st) != cudaSuccess)) {
    cleanup();
    return cuda_fail(cudaGetLastError(), "CSR copy");
  }
  const int rc = graph_build(g, nullptr, nullptr, nullptr, st, off, c, w, /*check_adopted=*/true);
  if (rc != SLQ_OK) {
    slq_graph_destroy(g);
    return rc;
  }
  *out = g;
  return SLQ_OK;
}

// Diagnostics: the first `count` row lengths of the Lanczos graph (the fold when there is one), host
// array; returns the number of rows of that graph in *rows_host.  Synchronous.
extern "C" int slq_graph_lanczos_rows(const slq_graph* g, int64_t* lengths_host, int64_t count, int64_t* rows_host) {
  if (!g || !lengths_host || !rows_host || count < 0) return fail(SLQ_ERR_VALUE, "bad argument");
  const slq_graph* f = g->folded ? g->folded : g;
  cudaStream_t st = static_cast<cudaStream_t>(g->stream);
  count = std::min<int64_t>(count, f->n);
  std::vector<int64_t> off(static_cast<size_t>(count + 1));
  if (count > 0) {
    SLQ_CUDA(cudaMemcpyAsync(off.data(), f->offsets, sizeof(int64_t) * (count + 1), cudaMemcpyDeviceToHost, st));
    SLQ_CUDA(cudaStreamSynchronize(st));
  }
  for (int64_t r = 0; r < count; ++r) lengths_host[r] = off[r + 1] - off[r];
  *rows_host = f->n;
  return SLQ_OK;
}

extern "C" int slq_graph_info(const slq_graph* g, slq_graph_info_t* out) {
  if (!g || !out) return fail(SLQ_ERR_VALUE, "NULL argument");
  int rc = fetch_host_scalars(const_cast<slq_graph*>(g));
  if (rc) return rc;
  if (g->bad_columns) return fail(SLQ_ERR_VALUE, "column index out of range [0, n)");
  out->n = g->n;
  out->nnz = g->nnz;
  out->trace_l = g->trace_l;
  out->max_degree = g->max_degree;
  out->isolated = g->isolated;
  out->unit_weights = g->unit_weights;
  out->ntiles = g->ntiles;
  return SLQ_OK;
}

extern "C" void slq_graph_destroy(slq_graph* g) {
  if (!g) return;
  drop_fold(g);
  // stream-ordered frees on the creation stream (it must outlive the graph)
  for (int i = 0; i < g->n_owned; ++i) cudaFreeAsync(g->owned[i], static_cast<cudaStream_t>(g->stream));
  delete g;
}

extern "C" int slq_graph_fold_isolated(slq_graph* g, double min_fraction, int64_t* folded_host) {
  if (!g || !folded_host) return fail(SLQ_ERR_VALUE, "NULL argument");
  return graph_fold(g, min_fraction, folded_host);
}

extern "C" int slq_operator_interval(const slq_graph* g, int kind, double* lo, double* hi) {
  if (!g || !lo || !hi) return fail(SLQ_ERR_VALUE, "NULL argument");
  *lo = 0.0;
  switch (kind) {
    case SLQ_LAPLACIAN: {
      int rc = fetch_host_scalars(const_cast<slq_graph*>(g));
      if (rc) return rc;
      *hi = 2.0 * g->max_degree;
      return SLQ_OK;
    }
    case SLQ_NORMALIZED_LAPLACIAN: *hi = 2.0; return SLQ_OK;
    case SLQ_DENSITY:
      // weights are strictly positive, so tr L > 0 exactly when there is an edge
      if (g->nnz == 0) return fail(SLQ_ERR_VALUE, "density matrix undefined for a graph without edges");
      *hi = 1.0;
      return SLQ_OK;
  }
  return fail(SLQ_ERR_VALUE, "unknown operator kind");
}

extern "C" int slq_graph_csr(const slq_graph* g, int64_t* offsets, int32_t* cols, void* stream) {
  if (!g) return fail(SLQ_ERR_VALUE, "NULL graph");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (offsets) SLQ_CUDA(cudaMemcpyAsync(offsets, g->offsets, sizeof(int64_t) * (g->n + 1), cudaMemcpyDefault, st));
  if (cols && g->nnz > 0) SLQ_CUDA(cudaMemcpyAsync(cols, g->cols, sizeof(int32_t) * g->nnz, cudaMemcpyDefault, st));
  return SLQ_OK;
}

namespace slq {

// Partial sums of the squared-operator trace identities (operators.py:119-141) in a fixed order:
// thread t of block b owns rows [lo, hi) of a fixed partition; per row the stored entries in order.
//   s[0] = sum_r d_r^2, s[1] = sum_e w_e^2, s[2] = sum_e w_e^2 / (d_r d_c)
constexpr int kTrBlocks = 148 * 4, kTrThreads = 256;
__global__ void __launch_bounds__(kTrThreads) trace_sq_kernel(const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ cols,
                                                              const double* __restrict__ w,
                                                              const double* __restrict__ deg, int64_t n,
                                                              double* __restrict__ part) {
  __shared__ double red[3][kTrThreads];
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kTrThreads + threadIdx.x;
  const int64_t T = static_cast<int64_t>(kTrBlocks) * kTrThreads;
  const int64_t lo = n * t / T, hi = n * (t + 1) / T;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int64_t r = lo; r < hi; ++r) {
    const double dr = deg[r];
    s0 = fma(dr, dr, s0);
    for (int64_t e = off[r]; e < off[r + 1]; ++e) {
      const double we = w ? w[e] : 1.0;
      const double w2 = we * we;
      s1 += w2;
      s2 += w2 / (dr * deg[cols[e]]);
    }
  }
  red[0][threadIdx.x] = s0;
  red[1][threadIdx.x] = s1;
  red[2][threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int i = 0; i < kTrThreads; ++i) acc += red[threadIdx.x][i];
    part[blockIdx.x * 3 + threadIdx.x] = acc;
  }
}

__global__ void trace_sq_final(const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int b = 0; b < kTrBlocks; ++b) acc += part[b * 3 + threadIdx.x];
    out[threadIdx.x] = acc;
  }
}

}  // namespace slq

// Exact trace of the squared operator (operators.py:119-141): L: sum d^2 + sum w^2; normalized
// Laplacian: #non-isolated + sum_e w^2 / (d_r d_c); density: tr(L^2) / tr(L)^2.  Synchronises.
extern "C" int slq_trace_squared(const slq_graph* g, int kind, double* out_host) {
  if (!g || !out_host) return fail(SLQ_ERR_VALUE, "NULL argument");
  int rc = fetch_host_scalars(const_cast<slq_graph*>(g));
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(g->stream);
  double* part = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * (3 * kTrBlocks + 3), st));
  {
    LaunchScope ls(K_PREPARE, st);
    trace_sq_kernel<<<kTrBlocks, kTrThreads, 0, st>>>(g->offsets, g->cols, g->weights, g->degree, g->n, part);
    trace_sq_final<<<1, 32, 0, st>>>(part, part + 3 * kTrBlocks);
  }
  double s[3];
  SLQ_CUDA(cudaMemcpyAsync(s, part + 3 * kTrBlocks, sizeof(s), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  SLQ_CUDA(cudaFreeAsync(part, st));
  const double trl = g->trace_l;
  switch (kind) {
    case SLQ_LAPLACIAN: *out_host = s[0] + s[1]; break;
    case SLQ_NORMALIZED_LAPLACIAN:
      *out_host = static_cast<double>(g->n - g->isolated) + (g->nnz > 0 ? s[2] : 0.0);
      break;
    case SLQ_DENSITY:
      if (g->nnz == 0 || trl <= 0.0) return fail(SLQ_ERR_VALUE, "density matrix undefined for a graph without edges");
      *out_host = (s[0] + s[1]) / (trl * trl);
      break;
    default: return fail(SLQ_ERR_VALUE, "unknown operator kind");
  }
  return SLQ_OK;
}

extern "C" int slq_graph_weights(const slq_graph* g, double* weights, int32_t* has_weights_host, void* stream) {
  if (!g || !has_weights_host) return fail(SLQ_ERR_VALUE, "NULL argument");
  *has_weights_host = g->weights ? 1 : 0;
  if (g->weights && weights && g->nnz > 0)
    SLQ_CUDA(cudaMemcpyAsync(weights, g->weights, sizeof(double) * g->nnz, cudaMemcpyDefault,
                             static_cast<cudaStream_t>(stream)));
  return SLQ_OK;
}

extern "C" int slq_graph_degrees(const slq_graph* g, double* degree, double* dinv, void* stream) {
  if (!g) return fail(SLQ_ERR_VALUE, "NULL graph");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (g->n == 0) return SLQ_OK;
  if (degree) SLQ_CUDA(cudaMemcpyAsync(degree, g->degree, sizeof(double) * g->n, cudaMemcpyDeviceToDevice, st));
  if (dinv) SLQ_CUDA(cudaMemcpyAsync(dinv, g->dinv, sizeof(double) * g->n, cudaMemcpyDeviceToDevice, st));
  return SLQ_OK;
}
