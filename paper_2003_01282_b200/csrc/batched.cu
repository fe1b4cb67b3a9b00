// Batched block-diagonal path (BASELINE C3): many small graphs stacked in one block-diagonal CSR,
// one CTA per graph running the reference's per-graph netlsd_slq / vnge_slq recurrence
// (slq.py:63-86, lanczos.py:70-163) for all probes of that graph at once:
//   * probes are prefixes of the same PCG64 streams (entry k of probe p does not depend on n), so
//     q0 = v/||v|| = +-1/fl(sqrt(n_g)) per graph, exactly as the reference draws them per graph;
//   * thread (p, slot) owns probe p and the rows == slot (mod kRows): every per-probe sum runs in a
//     fixed order and is combined over the kRows slots in order (deterministic);
//   * the literal CGS of lanczos.py:70-76 (dots with w', one subtraction, conditional second pass);
//   * breakdown at 1e-12 * interval_hi; per-probe implicit-QL Gauss rules, node clamp.
// Vectors live in a global workspace [S+1][N][c] (N = total vertices): each CTA touches only its
// own rows, so the working set of the resident CTAs stays in L2.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "pcg64.cuh"
#include "slq_common.cuh"
#include "tridiag.cuh"

namespace slq {

constexpr int kRows = 8;         // row slots per probe
constexpr int kBatchMaxProbes = 64;

struct BatchArgs {
  const int64_t* offsets;
  const int32_t* cols;
  const double* weights;
  const double* degree;
  const double* dinv;
  const double* dscal;
  const int64_t* voff;     // [G+1]
  int64_t G;
  int kind;
  SeedKey seed;
  int c;                   // probes per graph
  int S;                   // requested steps
  int64_t N;               // total vertices
  void* vec;               // [gridDim.y][S+1][N][c] workspace (slot S = w)
  double* nodes;           // [G][Y*c][S] (Y = gridDim.y probe blocks)
  double* weights_out;     // [G][Y*c][S]
  int32_t* steps_out;      // [G][Y*c]
  int* status;
  uint64_t probe0;         // stream index of probe 0 of probe block 0
  int64_t count;           // probes stored per graph (<= Y*c; the tail of the last block is dropped)
  const int* dflags;       // graph flags (bad columns -> status bit 8), may be null
};

template <typename VT>
__device__ __forceinline__ VT* vslot(const BatchArgs& a, int k) {
  return static_cast<VT*>(a.vec) + (static_cast<int64_t>(blockIdx.y) * (a.S + 1) + k) * a.N * a.c;
}

// Sum the kRows slot partials of quantity q (smem part[kRows][nq][c]) in slot order.
__device__ __forceinline__ double slot_sum(const double* part, int nq, int c, int q, int p) {
  double s = part[(0 * nq + q) * c + p];
  for (int r = 1; r < kRows; ++r) s += part[(r * nq + q) * c + p];
  return s;
}

// MAXS: capacity of the per-thread eigensolver arrays (local memory), >= the rule length
template <typename VT, int KIND, int MAXS = kMaxSteps>
#ifndef SLQ_BATCH_MINB
#define SLQ_BATCH_MINB 2   // 64 registers: 2x the resident CTAs (C3 fp32 -8%)
#endif
__global__ void __launch_bounds__(kRows * kBatchMaxProbes, SLQ_BATCH_MINB)
batched_lanczos_kernel(BatchArgs a) {
  extern __shared__ double sm[];
  const int c = a.c;
  const int t = threadIdx.x;
  const int p = t % c, rs = t / c;
  const bool act = rs < kRows;                         // threads beyond c*kRows idle
  const int nqmax = kCgsBlock + 1;
  double* part = sm;                                   // [kRows][nqmax][c]
  double* alpha = part + kRows * nqmax * c;            // [S][c]
  double* beta = alpha + a.S * c;                      // [S][c]
  double* rsc = beta + a.S * c;                        // [S+1][c]
  double* h = rsc + (a.S + 1) * c;                     // [S][c]
  double* nb = h + a.S * c;                            // [c]
  int* flags = reinterpret_cast<int*>(nb + c);         // [c] alive, [c] again, [c] steps, [1] any_again
  int* alive = flags;
  int* again = flags + c;
  int* steps = flags + 2 * c;
  int* any_again = flags + 3 * c;
  const double hi_int = KIND == SLQ_NORMALIZED_LAPLACIAN ? 2.0 : 1.0;
  const double tol = 1e-12 * hi_int;                   // lanczos.py:36,110

  for (int64_t gi = blockIdx.x; gi < a.G; gi += gridDim.x) {
    const int64_t v0 = a.voff[gi], v1 = a.voff[gi + 1];
    const int n = static_cast<int>(v1 - v0);
    const int S = n < a.S ? n : a.S;                   // lanczos.py:105
    __syncthreads();
    if (n <= 0) continue;
    // per-graph operator scalars: density scale 1/tr L_g (operators.py:93-96)
    double scale = 0.0;
    if (KIND == SLQ_DENSITY) {
      double trl = 0.0;
      for (int row = 0; row < n; ++row) trl += a.degree[v0 + row];   // same value in every thread
      scale = trl > 0.0 ? 1.0 / trl : 0.0;
    }
    // probes: u_0 = +-1 (stream prefix), r_0 = 1/fl(sqrt(n))
    VT* u0 = vslot<VT>(a, 0);
    if (act) {
      u128 st, inc;
      pcg64_seed_state(a.seed, a.probe0 + static_cast<uint64_t>(blockIdx.y) * c + p, &st, &inc);
      const u128 mult = pcg_mult();
      // rows rs, rs+kRows, ...: output m holds entries 2m (bit 31) and 2m+1 (bit 63)
      int row = rs;
      u128 cur = pcg_advance(st, inc, static_cast<uint64_t>(row / 2));
      int m_cur = row / 2;
      for (; row < n; row += kRows) {
        const int m = row / 2;
        if (m != m_cur) { cur = pcg_advance(cur, inc, static_cast<uint64_t>(m - m_cur)); m_cur = m; }
        const u128 s1 = cur * mult + inc;
        const uint64_t out = pcg_output(s1);
        const int bit = (row & 1) ? 63 : 31;
        u0[(v0 + row) * c + p] = from_f64<VT>(((out >> bit) & 1u) ? 1.0 : -1.0);
      }
    }
    if (t < c) {
      rsc[t] = __ddiv_rn(1.0, __dsqrt_rn(static_cast<double>(n)));
      alive[t] = 1;
      again[t] = 0;
      steps[t] = S;
      for (int k = 0; k < S; ++k) { alpha[k * c + t] = 0.0; beta[k * c + t] = 0.0; }
    }
    __syncthreads();
    VT* wv = vslot<VT>(a, a.S);
    for (int i = 0; i < S; ++i) {
      VT* ui = vslot<VT>(a, i);
      const VT* uim1 = vslot<VT>(a, i > 0 ? i - 1 : 0);
      const double ri = act ? rsc[i * c + p] : 0.0;
      // ---- w = Op(q_i) (sequential in-row sums), alpha partials
      double ap = 0.0;
      if (act) {
        for (int row = rs; row < n; row += kRows) {
          const int64_t gr = v0 + row;
          const int64_t b = a.offsets[gr], e = a.offsets[gr + 1];
          double acc = 0.0;
          for (int64_t k = b; k < e; ++k) {
            const int64_t col = a.cols[k];
            double tt = __dmul_rn(to_f64(ui[col * c + p]), ri);
            if (KIND == SLQ_NORMALIZED_LAPLACIAN) tt = __dmul_rn(a.dinv[col], tt);
            if (a.weights) tt = __dmul_rn(a.weights[k], tt);
            acc = __dadd_rn(acc, tt);
          }
          const double x = __dmul_rn(to_f64(ui[gr * c + p]), ri);
          const double d = a.degree[gr];
          double y;
          if (KIND == SLQ_NORMALIZED_LAPLACIAN) {
            y = __dsub_rn(__dmul_rn(d > 0.0 ? 1.0 : 0.0, x), __dmul_rn(a.dinv[gr], acc));
          } else if (KIND == SLQ_DENSITY) {
            y = __dmul_rn(scale, __dsub_rn(__dmul_rn(d, x), acc));
          } else {
            y = __dsub_rn(__dmul_rn(d, x), acc);
          }
          wv[gr * c + p] = from_f64<VT>(y);
          ap = fma(x, y, ap);
        }
        part[(rs * nqmax + 0) * c + p] = ap;
      }
      __syncthreads();
      if (t < c && alive[t]) alpha[i * c + t] = slot_sum(part, nqmax, c, 0, t);
      if (t == 0) *any_again = 0;
      __syncthreads();
      if (i == S - 1) break;
      // ---- w' = (w - alpha q_i) - beta q_{i-1}; CGS dots h_k = q_k . w' (k <= i), ||w'||^2
      const int nk = i + 1;
      const double al = act ? alpha[i * c + p] : 0.0;
      const double bp = (act && i > 0) ? beta[(i - 1) * c + p] : 0.0;
      const double rim1 = (act && i > 0) ? rsc[(i - 1) * c + p] : 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1 && *any_again == 0) break;
        const bool second = pass == 1;
        const bool pv = act && (!second || again[p]);
        VT* un = vslot<VT>(a, i + 1);
        for (int k0 = 0; k0 < nk; k0 += kCgsBlock) {
          const int kb = nk - k0 < kCgsBlock ? nk - k0 : kCgsBlock;
          double hp[kCgsBlock];
#pragma unroll
          for (int kk = 0; kk < kCgsBlock; ++kk) hp[kk] = 0.0;
          double nbp = 0.0;
          if (pv) {
            for (int row = rs; row < n; row += kRows) {
              const int64_t idx = (v0 + row) * c + p;
              double wp;
              if (second) wp = to_f64(un[idx]);
              else {
                const double qi = __dmul_rn(to_f64(ui[idx]), ri);
                const double qp = i > 0 ? __dmul_rn(to_f64(uim1[idx]), rim1) : 0.0;
                wp = __dsub_rn(__dsub_rn(to_f64(wv[idx]), __dmul_rn(al, qi)), __dmul_rn(bp, qp));
              }
              nbp = fma(wp, wp, nbp);
#pragma unroll
              for (int kk = 0; kk < kCgsBlock; ++kk) {
                if (kk < kb) {
                  const int k = k0 + kk;
                  const double qk = __dmul_rn(to_f64(vslot<VT>(a, k)[idx]), rsc[k * c + p]);
                  hp[kk] = fma(qk, wp, hp[kk]);
                }
              }
            }
          }
          if (act) {
#pragma unroll
            for (int kk = 0; kk < kCgsBlock; ++kk)
              if (kk < kb) part[(rs * nqmax + kk) * c + p] = hp[kk];
            part[(rs * nqmax + kCgsBlock) * c + p] = nbp;
          }
          __syncthreads();
          if (t < c) {
            for (int kk = 0; kk < kb; ++kk) h[(k0 + kk) * c + t] = slot_sum(part, nqmax, c, kk, t);
            if (!second && k0 == 0) nb[t] = slot_sum(part, nqmax, c, kCgsBlock, t);
          }
          __syncthreads();
        }
        // ---- u_{i+1} = w' - sum_k h_k q_k ; ||u_{i+1}||^2
        double np = 0.0;
        if (pv) {
          for (int row = rs; row < n; row += kRows) {
            const int64_t idx = (v0 + row) * c + p;
            double wp;
            if (second) wp = to_f64(un[idx]);
            else {
              const double qi = __dmul_rn(to_f64(ui[idx]), ri);
              const double qp = i > 0 ? __dmul_rn(to_f64(uim1[idx]), rim1) : 0.0;
              wp = __dsub_rn(__dsub_rn(to_f64(wv[idx]), __dmul_rn(al, qi)), __dmul_rn(bp, qp));
            }
            double proj = 0.0;
            for (int k = 0; k < nk; ++k)
              proj = __dadd_rn(proj, __dmul_rn(__dmul_rn(to_f64(vslot<VT>(a, k)[idx]), rsc[k * c + p]), h[k * c + p]));
            const VT v = from_f64<VT>(__dsub_rn(wp, proj));
            un[idx] = v;
            const double vd = to_f64(v);
            np = fma(vd, vd, np);
          }
        }
        if (act) part[(rs * nqmax + 0) * c + p] = np;
        __syncthreads();
        if (t < c && alive[t] && (!second || again[t])) {
          const double b = sqrt(slot_sum(part, nqmax, c, 0, t));
          bool commit = true;
          if (!second) {
            if (b < 0.5 * sqrt(nb[t])) {                 // lanczos.py:75
              again[t] = 1;
              *any_again = 1;
              if (a.dflags) atomicAdd(const_cast<int*>(a.dflags) + 2, 1);   // second-pass counter
              commit = false;
            }
          } else {
            again[t] = 0;
          }
          if (commit) {
            if (b <= tol) {                              // lanczos.py:133-134
              steps[t] = i + 1;
              alive[t] = 0;
              rsc[(i + 1) * c + t] = 0.0;
            } else {
              beta[i * c + t] = b;
              rsc[(i + 1) * c + t] = __ddiv_rn(1.0, b);
            }
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();
    // ---- Gauss rules per probe (lanczos.py:148-163 + slq.py:76-77)
    const int64_t pg = static_cast<int64_t>(blockIdx.y) * c + t;   // probe index within the graph's output
    const int64_t ow = static_cast<int64_t>(gridDim.y) * c;
    if (t < c && pg < a.count) {
      double d[MAXS], e[MAXS], z[MAXS];
      const int m = steps[t];
      bool finite = true;
      for (int k = 0; k < m; ++k) {
        d[k] = alpha[k * c + t];
        e[k] = k + 1 < m ? beta[k * c + t] : 0.0;
        z[k] = k == 0 ? 1.0 : 0.0;
        finite = finite && isfinite(d[k]) && isfinite(e[k]);
      }
      int rc = finite ? tridiag_ql_first_row(d, e, z, m) : -1;
      double* nd = a.nodes + (gi * ow + pg) * a.S;
      double* wt = a.weights_out + (gi * ow + pg) * a.S;
      if (rc) {
        atomicOr(a.status, rc < 0 ? 2 : 1);
        for (int k = 0; k < a.S; ++k) { nd[k] = 0.0; wt[k] = 0.0; }
      } else {
        for (int k = 0; k < m; ++k) z[k] = z[k] * z[k];
        for (int ii = 1; ii < m; ++ii) {
          const double dv = d[ii], zv = z[ii];
          int j = ii - 1;
          while (j >= 0 && d[j] > dv) { d[j + 1] = d[j]; z[j + 1] = z[j]; --j; }
          d[j + 1] = dv;
          z[j + 1] = zv;
        }
        for (int k = 0; k < a.S; ++k) {
          nd[k] = k < m ? fmin(fmax(d[k], 0.0), hi_int) : 0.0;
          wt[k] = k < m ? z[k] : 0.0;
        }
      }
      a.steps_out[gi * ow + pg] = m;
      if (a.dflags && a.dflags[0]) atomicOr(a.status, 8);
    }
  }
}

// Per-graph quadrature + aggregate: values[g][t] = n_g * mean_p sum_k w f(t, x), std like slq.py:98-105.
template <int FN>
__global__ void batched_integrate_kernel(const double* __restrict__ nodes, const double* __restrict__ weights,
                                         const int32_t* __restrict__ steps, int64_t G, int c, int ld,
                                         const int64_t* __restrict__ voff, const double* __restrict__ tgrid, int64_t T,
                                         double* __restrict__ values, double* __restrict__ stds, int* status) {
  extern __shared__ double pv[];   // [c]
  for (int64_t job = blockIdx.x; job < G * T; job += gridDim.x) {
    const int64_t gi = job / T, ti = job - gi * T;
    const double t = tgrid ? tgrid[ti] : 0.0;
    const double n = static_cast<double>(voff[gi + 1] - voff[gi]);
    for (int p = threadIdx.x; p < c; p += blockDim.x) {
      const int64_t o = (gi * c + p) * ld;
      const int m = steps[gi * c + p];
      double acc = 0.0;
      bool ok = true;
      for (int k = 0; k < m; ++k) {
        const double x = nodes[o + k];
        double f;
        if (FN == SLQ_FN_HEAT) f = exp(-t * x);
        else if (FN == SLQ_FN_WAVE_RE) f = cos(t * x);
        else if (FN == SLQ_FN_WAVE_IM) f = -sin(t * x);
        else if (FN == SLQ_FN_XLOGX) f = x > 0.0 ? x * log(x) : 0.0;
        else f = x;
        ok = ok && isfinite(f);
        acc = fma(weights[o + k], f, acc);
      }
      if (!ok) atomicOr(status, 4);
      pv[p] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0, sx = 0.0;
      for (int p = 0; p < c; ++p) { s += pv[p]; sx += n * pv[p]; }
      values[gi * T + ti] = n * (s / c);
      if (c > 1) {
        const double mean = sx / c;
        double ss = 0.0;
        for (int p = 0; p < c; ++p) { const double dl = n * pv[p] - mean; ss += dl * dl; }
        stds[gi * T + ti] = sqrt(ss / (c - 1)) / sqrt(static_cast<double>(c));
      } else {
        stds[gi * T + ti] = 0.0;
      }
    }
    __syncthreads();
  }
}

}  // namespace slq

using namespace slq;

static int lanczos_batched_entry(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs, int kind,
                                 const SeedKey& seed, int n_v, int steps, int dtype, double* nodes, double* weights,
                                 int32_t* steps_out, int32_t* status, void* stream) {
  if (!g || !vertex_offsets || !status) return fail(SLQ_ERR_VALUE, "NULL argument");
  if (n_v < 1 || n_v > kBatchMaxProbes) return fail(SLQ_ERR_VALUE, "batched path: 1 <= n_v <= 64");
  if (steps < 1 || steps > kMaxSteps) return fail(SLQ_ERR_VALUE, "steps must be in [1, 128]");
  if (kind != SLQ_NORMALIZED_LAPLACIAN && kind != SLQ_DENSITY && kind != SLQ_LAPLACIAN)
    return fail(SLQ_ERR_VALUE, "unknown operator kind");
  if (kind == SLQ_LAPLACIAN) return fail(SLQ_ERR_VALUE, "batched path: Laplacian interval is per graph; use kind 1 or 2");
  if (num_graphs <= 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ensure_pool(g->device);
  const int vb = dtype == SLQ_F64 ? 8 : 4;
  void* vec = nullptr;
  SLQ_CUDA(cudaMallocAsync(&vec, static_cast<size_t>(steps + 1) * std::max<int64_t>(g->n, 1) * n_v * vb, st));
  BatchArgs a{};
  a.offsets = g->offsets; a.cols = g->cols; a.weights = g->weights; a.degree = g->degree; a.dinv = g->dinv;
  a.dscal = g->dscal; a.voff = vertex_offsets; a.G = num_graphs; a.kind = kind; a.seed = seed; a.c = n_v;
  a.S = steps; a.N = g->n; a.vec = vec; a.nodes = nodes; a.weights_out = weights; a.steps_out = steps_out;
  a.status = status; a.probe0 = 0; a.count = n_v; a.dflags = nullptr;
  const int threads = ((kRows * n_v + 31) / 32) * 32;
  const size_t smem = sizeof(double) * (kRows * (kCgsBlock + 1) * n_v + (4 * steps + 3) * n_v) +
                      sizeof(int) * (3 * n_v + 4);
  const int grid = static_cast<int>(std::min<int64_t>(num_graphs, 148 * 16));
  {
    LaunchScope ls(K_BATCHED, st);
#define SLQ_BATCH(VT, K)                                                                                       \
  do {                                                                                                         \
    if (smem > 48 * 1024)                                                                                      \
      cudaFuncSetAttribute(a.S <= 16 ? batched_lanczos_kernel<VT, K, 16> : batched_lanczos_kernel<VT, K>,     \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));               \
    if (a.S <= 16) batched_lanczos_kernel<VT, K, 16><<<grid, threads, smem, st>>>(a);                          \
    else batched_lanczos_kernel<VT, K><<<grid, threads, smem, st>>>(a);                                        \
  } while (0)
    if (dtype == SLQ_F64) {
      if (kind == SLQ_NORMALIZED_LAPLACIAN) SLQ_BATCH(double, SLQ_NORMALIZED_LAPLACIAN);
      else SLQ_BATCH(double, SLQ_DENSITY);
    } else {
      if (kind == SLQ_NORMALIZED_LAPLACIAN) SLQ_BATCH(float, SLQ_NORMALIZED_LAPLACIAN);
      else SLQ_BATCH(float, SLQ_DENSITY);
    }
#undef SLQ_BATCH
  }
  SLQ_CUDA(cudaGetLastError());
  SLQ_CUDA(cudaFreeAsync(vec, st));
  return SLQ_OK;
}

// Single small graph (slq_rules for n <= small_graph_max_n()): the batched kernel with one graph
// and one CTA per block of <= 64 probes (grid.y), so the whole Lanczos run stays on one SM per probe
// block instead of ~2 grid-wide kernels per step.  Per-probe arithmetic does not depend on the
// block, so a probe's rule is the same for every probe range and count.
namespace slq {

int64_t small_graph_max_n() {
  static const int64_t v = [] {
    const char* e = getenv("SLQ_SMALL_N");
    return e ? static_cast<int64_t>(atoll(e)) : static_cast<int64_t>(128);   // measured crossover ~130 rows
  }();
  return v;
}

// Vertex offsets {0, n} of the single graph, written on the device: no host buffer is read inside
// the call, so it can be captured into a CUDA graph (a pageable memcpy from a stack array cannot).
static __global__ void single_graph_offsets_kernel(int64_t* voff, int64_t n) {
  voff[0] = 0;
  voff[1] = n;
}

int small_rules(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, int64_t count, int S, int dtype,
                double* nodes, double* weights, int32_t* steps_out, int32_t* status, cudaStream_t st) {
  const int c = static_cast<int>(std::min<int64_t>(count, kBatchMaxProbes));
  const int64_t blocks = (count + c - 1) / c;
  const int vb = dtype == SLQ_F64 ? 8 : 4;
  void* vec = nullptr;
  int64_t* voff = nullptr;
  SLQ_CUDA(cudaMallocAsync(&vec, static_cast<size_t>(blocks) * (S + 1) * std::max<int64_t>(g->n, 1) * c * vb, st));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&voff), 2 * sizeof(int64_t), st));
  single_graph_offsets_kernel<<<1, 1, 0, st>>>(voff, g->n);
  BatchArgs a{};
  a.offsets = g->offsets; a.cols = g->cols; a.weights = g->weights; a.degree = g->degree; a.dinv = g->dinv;
  a.dscal = g->dscal; a.voff = voff; a.G = 1; a.kind = kind; a.seed = seed; a.c = c;
  a.S = S; a.N = g->n; a.vec = vec; a.nodes = nodes; a.weights_out = weights; a.steps_out = steps_out;
  a.status = status; a.probe0 = static_cast<uint64_t>(probe_begin); a.count = count; a.dflags = g->dflags;
  const int threads = ((kRows * c + 31) / 32) * 32;
  const size_t smem = sizeof(double) * (kRows * (kCgsBlock + 1) * c + (4 * S + 3) * c) + sizeof(int) * (3 * c + 4);
  const dim3 grid(1, static_cast<unsigned>(blocks));
  {
    LaunchScope ls(K_BATCHED, st);
#define SLQ_SMALL(VT, K)                                                                                       \
  do {                                                                                                         \
    if (smem > 48 * 1024)                                                                                      \
      cudaFuncSetAttribute(a.S <= 16 ? batched_lanczos_kernel<VT, K, 16> : batched_lanczos_kernel<VT, K>,     \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));               \
    if (a.S <= 16) batched_lanczos_kernel<VT, K, 16><<<grid, threads, smem, st>>>(a);                          \
    else batched_lanczos_kernel<VT, K><<<grid, threads, smem, st>>>(a);                                        \
  } while (0)
    if (dtype == SLQ_F64) {
      if (kind == SLQ_NORMALIZED_LAPLACIAN) SLQ_SMALL(double, SLQ_NORMALIZED_LAPLACIAN);
      else SLQ_SMALL(double, SLQ_DENSITY);
    } else {
      if (kind == SLQ_NORMALIZED_LAPLACIAN) SLQ_SMALL(float, SLQ_NORMALIZED_LAPLACIAN);
      else SLQ_SMALL(float, SLQ_DENSITY);
    }
#undef SLQ_SMALL
  }
  SLQ_CUDA(cudaGetLastError());
  SLQ_CUDA(cudaFreeAsync(vec, st));
  SLQ_CUDA(cudaFreeAsync(voff, st));
  return SLQ_OK;
}

}  // namespace slq

extern "C" int slq_lanczos_batched(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs, int kind,
                                   uint64_t seed, int n_v, int steps, int dtype, double* nodes, double* weights,
                                   int32_t* steps_out, int32_t* status, void* stream) {
  return lanczos_batched_entry(g, vertex_offsets, num_graphs, kind, seed_key_u64(seed), n_v, steps, dtype, nodes,
                               weights, steps_out, status, stream);
}

extern "C" int slq_lanczos_batched_seeded(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs,
                                          int kind, const slq_seed* seed, int n_v, int steps, int dtype, double* nodes,
                                          double* weights, int32_t* steps_out, int32_t* status, void* stream) {
  SeedKey k;
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  return lanczos_batched_entry(g, vertex_offsets, num_graphs, kind, k, n_v, steps, dtype, nodes, weights, steps_out,
                               status, stream);
}

extern "C" int slq_integrate_batched(const double* nodes, const double* weights, const int32_t* steps,
                                     int64_t num_graphs, int n_v, int ld, const int64_t* vertex_offsets,
                                     const double* t, int64_t T, int fn, double* values, double* std_errors,
                                     int32_t* status, void* stream) {
  if (num_graphs < 0 || n_v < 1 || T < 0 || !status) return fail(SLQ_ERR_VALUE, "bad batched integrate arguments");
  if (num_graphs == 0 || T == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = static_cast<int>(std::min<int64_t>(num_graphs * T, 148 * 32));
  const size_t smem = sizeof(double) * n_v;
  LaunchScope ls(K_QUAD, st);
  switch (fn) {
    case SLQ_FN_HEAT: batched_integrate_kernel<SLQ_FN_HEAT><<<grid, 32, smem, st>>>(nodes, weights, steps, num_graphs, n_v, ld, vertex_offsets, t, T, values, std_errors, status); break;
    case SLQ_FN_WAVE_RE: batched_integrate_kernel<SLQ_FN_WAVE_RE><<<grid, 32, smem, st>>>(nodes, weights, steps, num_graphs, n_v, ld, vertex_offsets, t, T, values, std_errors, status); break;
    case SLQ_FN_WAVE_IM: batched_integrate_kernel<SLQ_FN_WAVE_IM><<<grid, 32, smem, st>>>(nodes, weights, steps, num_graphs, n_v, ld, vertex_offsets, t, T, values, std_errors, status); break;
    case SLQ_FN_XLOGX: batched_integrate_kernel<SLQ_FN_XLOGX><<<grid, 32, smem, st>>>(nodes, weights, steps, num_graphs, n_v, ld, vertex_offsets, t, T, values, std_errors, status); break;
    default: return fail(SLQ_ERR_VALUE, "unknown integrand");
  }
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}
