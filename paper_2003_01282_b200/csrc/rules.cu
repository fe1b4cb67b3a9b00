// Gauss quadrature rules, grid quadrature and the probe aggregate.
//   slq_gauss_rules  <- quadrature_rule (lanczos.py:148-163) + np.clip (slq.py:76-77)
//                      batched symmetric tridiagonal implicit QL (Wilkinson shift), one thread per
//                      probe, accumulating only the FIRST ROW of the eigenvector matrix
//                      (weights = Z[0,:]^2), ascending nodes.
//   slq_quadrature   <- _apply_rule over the whole t grid (slq.py:89-95, 153-168)
//   slq_estimate     <- _estimate_from (slq.py:98-105)
#include <cfloat>
#include <algorithm>
#include <cmath>

#include "slq_common.cuh"
#include "pcg64.cuh"
#include "tridiag.cuh"

namespace slq {

// status bits (device int, OR-ed): 1 eigensolver failed, 2 non-finite tridiagonal, 4 non-finite integrand,
// 8 out-of-range column index in the graph.
constexpr int kStEigen = 1, kStNanTri = 2, kStNanF = 4, kStBadCol = 8;

// hi_kind >= 0: the clamp interval comes from the device graph scalars (no host round trip).
// One thread per probe; d, e, z are the thread's work arrays (local memory up to 128 steps, a global
// scratch slice beyond).
__device__ __forceinline__ void gauss_rule_one(const double* __restrict__ alpha, const double* __restrict__ beta,
                                               const int32_t* __restrict__ steps, int64_t p, int ld, double lo,
                                               double hi, double* __restrict__ nodes, double* __restrict__ weights,
                                               int32_t* __restrict__ info, int* __restrict__ status, double* d,
                                               double* e, double* z) {
  const int m = steps[p];
  const double* a = alpha + p * ld;
  const double* b = beta + p * ld;
  bool finite = true;
  for (int k = 0; k < m; ++k) {
    d[k] = a[k];
    e[k] = k + 1 < m ? b[k] : 0.0;
    z[k] = k == 0 ? 1.0 : 0.0;
    finite = finite && isfinite(d[k]) && isfinite(e[k]);
  }
  int rc = 0;
  if (!finite) rc = -1;                       // scipy check_finite -> ValueError
  else rc = tridiag_ql_first_row(d, e, z, m);
  if (info) info[p] = rc;
  if (rc) {
    atomicOr(status, rc < 0 ? kStNanTri : kStEigen);
    for (int k = 0; k < ld; ++k) { nodes[p * ld + k] = 0.0; weights[p * ld + k] = 0.0; }
    return;
  }
  // ascending sort of (node, weight) pairs
  for (int k = 0; k < m; ++k) z[k] = z[k] * z[k];
  for (int i = 1; i < m; ++i) {
    const double dv = d[i], zv = z[i];
    int j = i - 1;
    while (j >= 0 && d[j] > dv) { d[j + 1] = d[j]; z[j + 1] = z[j]; --j; }
    d[j + 1] = dv;
    z[j + 1] = zv;
  }
  for (int k = 0; k < ld; ++k) {
    nodes[p * ld + k] = k < m ? fmin(fmax(d[k], lo), hi) : 0.0;
    weights[p * ld + k] = k < m ? z[k] : 0.0;
  }
}

__device__ __forceinline__ double clamp_hi(double hi, const double* dscal, int hi_kind) {
  if (hi_kind < 0) return hi;
  return hi_kind == SLQ_NORMALIZED_LAPLACIAN ? 2.0 : (hi_kind == SLQ_DENSITY ? 1.0 : dscal[4]);
}

// MAXS: capacity of the per-thread work arrays (local memory): sized to the rule length so the
// arrays of a CTA stay L1-resident.
template <int MAXS>
__global__ void gauss_rules_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                                   const int32_t* __restrict__ steps, int64_t count, int ld, double lo,
                                   double hi, double* __restrict__ nodes, double* __restrict__ weights,
                                   int32_t* __restrict__ info, int* __restrict__ status, const double* dscal,
                                   int hi_kind, const int* gflags) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p == 0 && gflags && gflags[0]) atomicOr(status, kStBadCol);
  if (p >= count) return;
  double d[MAXS], e[MAXS], z[MAXS];
  gauss_rule_one(alpha, beta, steps, p, ld, lo, clamp_hi(hi, dscal, hi_kind), nodes, weights, info, status, d, e, z);
}

// Rules longer than kMaxSteps (s > 128: the reference accepts any step budget, lanczos.py:79-110):
// the same solver on a global scratch slice [3][ld] per probe.
__global__ void gauss_rules_long_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                                        const int32_t* __restrict__ steps, int64_t count, int ld, double lo,
                                        double hi, double* __restrict__ nodes, double* __restrict__ weights,
                                        int32_t* __restrict__ info, int* __restrict__ status, const double* dscal,
                                        int hi_kind, const int* gflags, double* __restrict__ scratch) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p == 0 && gflags && gflags[0]) atomicOr(status, kStBadCol);
  if (p >= count) return;
  double* d = scratch + p * 3 * static_cast<int64_t>(ld);
  gauss_rule_one(alpha, beta, steps, p, ld, lo, clamp_hi(hi, dscal, hi_kind), nodes, weights, info, status, d, d + ld,
                 d + 2 * ld);
}

template <int FN>
__device__ __forceinline__ double integrand(double t, double x) {
  if (FN == SLQ_FN_HEAT) return exp(-t * x);
  if (FN == SLQ_FN_WAVE_RE) return cos(t * x);
  if (FN == SLQ_FN_WAVE_IM) return -sin(t * x);
  if (FN == SLQ_FN_XLOGX) return x > 0.0 ? x * log(x) : 0.0;
  return x;
}

template <int FN>
__global__ void quadrature_kernel(const double* __restrict__ nodes, const double* __restrict__ weights,
                                  const int32_t* __restrict__ steps, int64_t count, int ld,
                                  const double* __restrict__ tgrid, int64_t T, double* __restrict__ pv,
                                  int* __restrict__ nonfinite) {
  const int64_t total = T * count;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ti = idx / count, p = idx - ti * count;
    const double t = tgrid ? tgrid[ti] : 0.0;
    const int m = steps[p];
    double acc = 0.0;
    bool ok = true;
    for (int k = 0; k < m; ++k) {
      const double f = integrand<FN>(t, nodes[p * ld + k]);
      ok = ok && isfinite(f);
      acc = fma(weights[p * ld + k], f, acc);
    }
    if (!ok) atomicOr(nonfinite, kStNanF);
    pv[ti * count + p] = acc;
  }
}

__global__ void estimate_kernel(const double* __restrict__ pv, int64_t T, int64_t count, double n,
                                double* __restrict__ value, double* __restrict__ std_error) {
  const int64_t ti = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (ti >= T) return;
  const double* row = pv + ti * count;
  double s = 0.0, sx = 0.0;
  for (int64_t p = 0; p < count; ++p) { s += row[p]; sx += n * row[p]; }
  value[ti] = n * (s / static_cast<double>(count));
  if (count > 1) {
    const double mean = sx / static_cast<double>(count);
    double ss = 0.0;
    for (int64_t p = 0; p < count; ++p) {
      const double dlt = n * row[p] - mean;
      ss += dlt * dlt;
    }
    std_error[ti] = sqrt(ss / static_cast<double>(count - 1)) / sqrt(static_cast<double>(count));
  } else {
    std_error[ti] = 0.0;
  }
}

// Fused quadrature + aggregate for up to 8 integrands: block (t, f); threads over probes; fixed-tree
// block sums for the mean and for sum (x - mean)^2 (the two passes of np.std, slq.py:98-105).
struct FnList {
  int fn[8];
  int n;
};

__device__ __forceinline__ double integrand_rt(int fn, double t, double x) {
  switch (fn) {
    case SLQ_FN_HEAT: return exp(-t * x);
    case SLQ_FN_WAVE_RE: return cos(t * x);
    case SLQ_FN_WAVE_IM: return -sin(t * x);
    case SLQ_FN_XLOGX: return x > 0.0 ? x * log(x) : 0.0;
    default: return x;
  }
}

__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double tot = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += sh[w];
    sh[32] = tot;
  }
  __syncthreads();
  tot = sh[32];
  __syncthreads();
  return tot;
}

__global__ void __launch_bounds__(256)
integrate_kernel(const double* __restrict__ nodes, const double* __restrict__ weights,
                 const int32_t* __restrict__ steps, int64_t count, int ld, const double* __restrict__ tgrid, int64_t T,
                 FnList fl, double n, double* __restrict__ values, double* __restrict__ stds,
                 double* __restrict__ per_vector, int* __restrict__ status) {
  __shared__ double sh[33];
  const int64_t ti = blockIdx.x;
  const int f = blockIdx.y;
  const int fn = fl.fn[f];
  const double t = tgrid ? tgrid[ti] : 0.0;
  double s = 0.0;
  bool ok = true;
  for (int64_t p = threadIdx.x; p < count; p += blockDim.x) {
    const int m = steps[p];
    double acc = 0.0;
    for (int k = 0; k < m; ++k) {
      const double v = integrand_rt(fn, t, nodes[p * ld + k]);
      ok = ok && isfinite(v);
      acc = fma(weights[p * ld + k], v, acc);
    }
    if (per_vector) per_vector[(static_cast<int64_t>(f) * T + ti) * count + p] = acc;
    s += acc;
  }
  if (!ok) atomicOr(status, kStNanF);
  const double sp = block_sum(s, sh);
  const double value = n * (sp / static_cast<double>(count));   // n * mean(per_vector), slq.py:100
  const double mean = value;                                     // mean of n * per_vector
  double ss = 0.0;
  for (int64_t p = threadIdx.x; p < count; p += blockDim.x) {
    const int m = steps[p];
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc = fma(weights[p * ld + k], integrand_rt(fn, t, nodes[p * ld + k]), acc);
    const double dl = n * acc - mean;
    ss += dl * dl;
  }
  const double sq = block_sum(ss, sh);
  if (threadIdx.x == 0) {
    values[static_cast<int64_t>(f) * T + ti] = value;
    stds[static_cast<int64_t>(f) * T + ti] =
        count > 1 ? sqrt(sq / static_cast<double>(count - 1)) / sqrt(static_cast<double>(count)) : 0.0;
  }
}

static int launch_gauss_rules(const double* alpha, const double* beta, const int32_t* steps, int64_t count, int ld,
                              double lo, double hi, double* nodes, double* weights, int32_t* info, int* status,
                              const double* dscal, int hi_kind, const int* gflags, cudaStream_t st) {
  const int grid = ceil_div(count, 32);
  LaunchScope ls(K_EIG, st);
#define SLQ_RULES(M) gauss_rules_kernel<M><<<grid, 32, 0, st>>>(alpha, beta, steps, count, ld, lo, hi, nodes, weights, \
                                                                 info, status, dscal, hi_kind, gflags)
  if (ld <= 16) SLQ_RULES(16);
  else if (ld <= 32) SLQ_RULES(32);
  else if (ld <= 64) SLQ_RULES(64);
  else if (ld <= kMaxSteps) SLQ_RULES(kMaxSteps);
  else {
    double* scratch = nullptr;
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * 3 * ld * count, st));
    gauss_rules_long_kernel<<<grid, 32, 0, st>>>(alpha, beta, steps, count, ld, lo, hi, nodes, weights, info, status,
                                                 dscal, hi_kind, gflags, scratch);
    SLQ_CUDA(cudaFreeAsync(scratch, st));
  }
#undef SLQ_RULES
  return SLQ_OK;
}

}  // namespace slq

using namespace slq;

extern "C" int slq_gauss_rules(const double* alpha, const double* beta, const int32_t* steps, int64_t count,
                               int ld, double lo, double hi, double* nodes, double* weights, int32_t* info,
                               void* stream) {
  if (count < 0 || ld < 1 || ld > kMaxStepsLong) return fail(SLQ_ERR_VALUE, "bad rule shape (ld must be in [1,4096])");
  if (count == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* status = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&status), sizeof(int), st));
  SLQ_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
  int rc = launch_gauss_rules(alpha, beta, steps, count, ld, lo, hi, nodes, weights, info, status, nullptr, -1, nullptr, st);
  if (rc) return rc;
  int h = 0;
  SLQ_CUDA(cudaMemcpyAsync(&h, status, sizeof(int), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(status, st);
  SLQ_CUDA(cudaGetLastError());
  if (h & kStNanTri) return fail(SLQ_ERR_VALUE, "array must not contain infs or NaNs");
  if (h & kStEigen) return fail(SLQ_ERR_EIGEN, "tridiagonal eigensolver failed: no convergence");
  return SLQ_OK;
}

extern "C" int slq_quadrature(const double* nodes, const double* weights, const int32_t* steps, int64_t count,
                              int ld, const double* t, int64_t T, int fn, double* per_vector, void* stream) {
  if (count < 0 || T < 0) return fail(SLQ_ERR_VALUE, "negative size");
  if (count == 0 || T == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* flag = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), st));
  SLQ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  const int64_t total = T * count;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  {
    LaunchScope ls(K_QUAD, st);
    switch (fn) {
      case SLQ_FN_HEAT: quadrature_kernel<SLQ_FN_HEAT><<<grid, 256, 0, st>>>(nodes, weights, steps, count, ld, t, T, per_vector, flag); break;
      case SLQ_FN_WAVE_RE: quadrature_kernel<SLQ_FN_WAVE_RE><<<grid, 256, 0, st>>>(nodes, weights, steps, count, ld, t, T, per_vector, flag); break;
      case SLQ_FN_WAVE_IM: quadrature_kernel<SLQ_FN_WAVE_IM><<<grid, 256, 0, st>>>(nodes, weights, steps, count, ld, t, T, per_vector, flag); break;
      case SLQ_FN_XLOGX: quadrature_kernel<SLQ_FN_XLOGX><<<grid, 256, 0, st>>>(nodes, weights, steps, count, ld, t, T, per_vector, flag); break;
      case SLQ_FN_IDENTITY: quadrature_kernel<SLQ_FN_IDENTITY><<<grid, 256, 0, st>>>(nodes, weights, steps, count, ld, t, T, per_vector, flag); break;
      default: cudaFreeAsync(flag, st); return fail(SLQ_ERR_VALUE, "unknown integrand");
    }
  }
  int h = 0;
  SLQ_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  SLQ_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(flag, st);
  SLQ_CUDA(cudaGetLastError());
  if (h) return fail(SLQ_ERR_NONFINITE, "f returned a non-finite value at quadrature nodes");
  return SLQ_OK;
}

extern "C" int slq_estimate(const double* per_vector, int64_t T, int64_t count, double n, double* value,
                            double* std_error, void* stream) {
  if (count < 1 || T < 0) return fail(SLQ_ERR_VALUE, "need at least one probe");
  if (T == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  {
    LaunchScope ls(K_ESTIMATE, st);
    estimate_kernel<<<ceil_div(T, 128), 128, 0, st>>>(per_vector, T, count, n, value, std_error);
  }
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

// ------------------------------------------------------------------ asynchronous composite entry points
int lanczos_seeded_key(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, int64_t count,
                       int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out, void* stream);

static int rules_entry(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, int64_t count, int steps,
                       int reorth, int dtype, double* nodes, double* weights, int32_t* steps_out, int32_t* status,
                       void* stream) {
  if (!g || !status) return fail(SLQ_ERR_VALUE, "NULL argument");
  if (count == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int S = static_cast<int>(std::min<int64_t>(steps, std::max<int64_t>(g->n, 1)));
  // small graphs: one CTA per probe block runs the whole recurrence (batched.cu)
  const int ro = reorth < 0 ? (S <= 100 ? 1 : 0) : reorth;
  if (g->n > 0 && g->n <= small_graph_max_n() && ro == 1 && steps >= 1 && S <= kMaxSteps && count > 0 &&
      probe_begin >= 0 && (dtype == SLQ_F64 || dtype == SLQ_F32) &&
      (kind == SLQ_NORMALIZED_LAPLACIAN || (kind == SLQ_DENSITY && g->nnz > 0))) {
    const size_t ws = static_cast<size_t>((count + 63) / 64) * (S + 1) * g->n * std::min<int64_t>(count, 64) *
                      (dtype == SLQ_F64 ? 8 : 4);
    if (ws <= (size_t(1) << 30))
      return small_rules(g, kind, seed, probe_begin, count, S, dtype, nodes, weights, steps_out, status, st);
  }
  double* ab = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ab), sizeof(double) * 2 * count * S, st));
  int rc = lanczos_seeded_key(g, kind, seed, probe_begin, count, steps, reorth, dtype, ab, ab + count * S, steps_out,
                              stream);
  if (rc == SLQ_OK)
    rc = launch_gauss_rules(ab, ab + count * S, steps_out, count, S, 0.0, 0.0, nodes, weights, nullptr, status, g->dscal,
                            kind, g->dflags, st);
  cudaFreeAsync(ab, st);
  if (rc) return rc;
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

int lanczos_pair_key(const slq_graph* g, const SeedKey& seed, int64_t probe_begin, int64_t count, int steps, int reorth,
                     int dtype, double* alpha_a, double* beta_a, int32_t* steps_a, double* alpha_b, double* beta_b,
                     int32_t* steps_b, void* stream, int* paired);

extern "C" int slq_rules_pair_seeded(const slq_graph* g, const slq_seed* seed, int64_t probe_begin, int64_t count,
                                     int steps, int reorth, int dtype, double* nodes_nl, double* weights_nl,
                                     int32_t* steps_nl, double* nodes_p, double* weights_p, int32_t* steps_p,
                                     int32_t* status, int32_t* paired, void* stream) {
  if (!g || !status) return fail(SLQ_ERR_VALUE, "NULL argument");
  SeedKey k;
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  if (steps < 1) return fail(SLQ_ERR_VALUE, "step budget must be >= 1");
  if (count < 0 || probe_begin < 0) return fail(SLQ_ERR_VALUE, "negative probe range");
  if (g->nnz == 0) return fail(SLQ_ERR_VALUE, "density matrix undefined for a graph without edges");
  if (paired) *paired = 0;
  if (count == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int S = static_cast<int>(std::min<int64_t>(steps, std::max<int64_t>(g->n, 1)));
  if (g->n <= small_graph_max_n()) {   // small graphs: the batched kernel, one operator at a time
    int rc = rules_entry(g, SLQ_NORMALIZED_LAPLACIAN, k, probe_begin, count, steps, reorth, dtype, nodes_nl, weights_nl,
                         steps_nl, status, stream);
    if (rc) return rc;
    return rules_entry(g, SLQ_DENSITY, k, probe_begin, count, steps, reorth, dtype, nodes_p, weights_p, steps_p, status,
                       stream);
  }
  double* ab = nullptr;
  const int64_t cs = count * S;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ab), sizeof(double) * 4 * cs, st));
  int used = 0;
  int rc = lanczos_pair_key(g, k, probe_begin, count, steps, reorth, dtype, ab, ab + cs, steps_nl, ab + 2 * cs, ab + 3 * cs,
                            steps_p, stream, &used);
  if (rc == SLQ_OK)
    rc = launch_gauss_rules(ab, ab + cs, steps_nl, count, S, 0.0, 0.0, nodes_nl, weights_nl, nullptr, status, g->dscal,
                            SLQ_NORMALIZED_LAPLACIAN, g->dflags, st);
  if (rc == SLQ_OK)
    rc = launch_gauss_rules(ab + 2 * cs, ab + 3 * cs, steps_p, count, S, 0.0, 0.0, nodes_p, weights_p, nullptr, status,
                            g->dscal, SLQ_DENSITY, g->dflags, st);
  cudaFreeAsync(ab, st);
  if (rc) return rc;
  if (paired) *paired = used;
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

extern "C" int slq_rules(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count, int steps,
                         int reorth, int dtype, double* nodes, double* weights, int32_t* steps_out, int32_t* status,
                         void* stream) {
  return rules_entry(g, kind, seed_key_u64(seed), probe_begin, count, steps, reorth, dtype, nodes, weights, steps_out,
                     status, stream);
}

extern "C" int slq_rules_seeded(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin, int64_t count,
                                int steps, int reorth, int dtype, double* nodes, double* weights, int32_t* steps_out,
                                int32_t* status, void* stream) {
  SeedKey k;
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  return rules_entry(g, kind, k, probe_begin, count, steps, reorth, dtype, nodes, weights, steps_out, status, stream);
}

extern "C" int slq_integrate(const double* nodes, const double* weights, const int32_t* steps, int64_t count, int ld,
                             const double* t, int64_t T, const int* fns_host, int nfn, double n, double* values,
                             double* std_errors, double* per_vector, int32_t* status, void* stream) {
  if (count < 1 || T < 0 || nfn < 0 || !status) return fail(SLQ_ERR_VALUE, "bad integrate arguments");
  if (T == 0 || nfn == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int f0 = 0; f0 < nfn; f0 += 8) {
    FnList fl{};
    fl.n = std::min(8, nfn - f0);
    for (int f = 0; f < fl.n; ++f) {
      if (fns_host[f0 + f] < 0 || fns_host[f0 + f] > SLQ_FN_IDENTITY) return fail(SLQ_ERR_VALUE, "unknown integrand");
      fl.fn[f] = fns_host[f0 + f];
    }
    LaunchScope ls(K_QUAD, st);
    integrate_kernel<<<dim3(static_cast<unsigned>(T), fl.n), 256, 0, st>>>(
        nodes, weights, steps, count, ld, t, T, fl, n, values + static_cast<int64_t>(f0) * T,
        std_errors + static_cast<int64_t>(f0) * T,
        per_vector ? per_vector + static_cast<int64_t>(f0) * T * count : nullptr, status);
  }
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

extern "C" int slq_signature(const slq_graph* g, int kind, uint64_t seed, int64_t count, int steps, int reorth,
                             int dtype, const double* t, int64_t T, const int* fns_host, int nfn, double* values,
                             double* std_errors, int32_t* status, void* stream) {
  if (!g || !status) return fail(SLQ_ERR_VALUE, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int S = static_cast<int>(std::min<int64_t>(steps, std::max<int64_t>(g->n, 1)));
  char* buf = nullptr;
  const size_t bn = sizeof(double) * count * S;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * bn + sizeof(int32_t) * count + 16, st));
  double* nodes = reinterpret_cast<double*>(buf);
  double* weights = nodes + count * S;
  int32_t* stp = reinterpret_cast<int32_t*>(buf + 2 * bn);
  int rc = slq_rules(g, kind, seed, 0, count, steps, reorth, dtype, nodes, weights, stp, status, stream);
  if (rc == SLQ_OK)
    rc = slq_integrate(nodes, weights, stp, count, S, t, T, fns_host, nfn, static_cast<double>(g->n), values,
                       std_errors, nullptr, status, stream);
  cudaFreeAsync(buf, st);
  return rc;
}

// Synchronous host-buffer variant of slq_rules_seeded for FFI bindings without a device allocator
// (the reference's ctypes stub): probes [probe_begin, +count) of `seed`, rules
// copied to host arrays nodes_host/weights_host [count][s'] and steps_host [count],
// s' = min(steps, n).  The device status word is mapped to the return code (SLQ_ERR_EIGEN,
// SLQ_ERR_VALUE for non-finite tridiagonals or out-of-range columns).  Runs on the graph's stream.
extern "C" int slq_rules_host(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin, int64_t count,
                              int steps, int reorth, int dtype, double* nodes_host, double* weights_host,
                              int32_t* steps_host) {
  if (!g || !nodes_host || !weights_host || !steps_host) return fail(SLQ_ERR_VALUE, "NULL argument");
  if (steps < 1) return fail(SLQ_ERR_VALUE, "step budget must be >= 1");
  if (count <= 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(g->stream);
  const int64_t S = std::min<int64_t>(steps, std::max<int64_t>(g->n, 1));
  char* buf = nullptr;
  const size_t bn = sizeof(double) * count * S;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * bn + sizeof(int32_t) * (count + 1) + 16, st));
  double* nodes = reinterpret_cast<double*>(buf);
  double* weights = nodes + count * S;
  int32_t* stp = reinterpret_cast<int32_t*>(buf + 2 * bn);
  int32_t* status = stp + count;
  int rc = cudaMemsetAsync(status, 0, sizeof(int32_t), st) == cudaSuccess ? SLQ_OK : SLQ_ERR_CUDA;
  if (rc == SLQ_OK)
    rc = slq_rules_seeded(g, kind, seed, probe_begin, count, steps, reorth, dtype, nodes, weights, stp, status, st);
  int32_t hstatus = 0;
  if (rc == SLQ_OK) {
    if (cudaMemcpyAsync(nodes_host, nodes, bn, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(weights_host, weights, bn, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(steps_host, stp, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(&hstatus, status, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rc = cuda_fail(cudaGetLastError(), "rules D2H");
  }
  cudaFreeAsync(buf, st);
  if (rc) return rc;
  SLQ_CUDA(cudaStreamSynchronize(st));
  if (hstatus & kStBadCol) return fail(SLQ_ERR_VALUE, "column index out of range [0, n)");
  if (hstatus & kStNanTri) return fail(SLQ_ERR_VALUE, "array must not contain infs or NaNs");
  if (hstatus & kStEigen) return fail(SLQ_ERR_EIGEN, "tridiagonal eigensolver failed: no convergence");
  return SLQ_OK;
}
