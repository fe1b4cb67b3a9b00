// Block Lanczos engine: all probes of a chunk advance together through the reference's
// per-probe recurrence (lanczos.py:79-145) with full CGS reorthogonalisation (lanczos.py:70-76).
//
// HBM layout: every Lanczos vector of a chunk is an [n][ldc] row-major block, probes
// interleaved (ldc >= c), so one gathered CSR row reads c contiguous values.  The basis keeps
// the UNNORMALISED vectors u_k plus a per-probe scale r_k = 1/beta_{k-1}; every reader forms
// q_k = u_k * r_k on the fly (no normalisation pass over HBM).  u_0 is the +-1 probe and
// r_0 = 1/fl(sqrt(n)), so q_0 equals the reference's v/||v|| bit for bit (slq.py:73).
//
// One Lanczos step i, per chunk:
//   A   spmm     w = Op(q_i) (sequential in-row sums, no FMA: bit-exact operator) ; alpha partials
//   R   reduce   alpha_i (fixed-order tree over tiles: deterministic, independent of chunking)
//   B1  cgs_dot  w' = (w - alpha q_i) - beta_{i-1} q_{i-1} recomputed per row;
//                partials of h_k = q_k . w' (k <= i) and ||w'||^2
//   R   reduce   h, ||w'||
//   B2  cgs_upd  u_{i+1} = w' - sum_k h_k q_k ; ||u_{i+1}||^2 partials
//   R   reduce + finalize: beta_i, breakdown (beta <= 1e-12 * interval_hi), second-pass flag
//   [B1', R, B2', R] second CGS pass for probes with ||w''|| < 0.5 ||w'|| (grid-stride kernels
//                that exit at once when no probe asked for it)
// Every per-probe reduction order depends only on the graph's fixed tiles, so a probe's rule is
// bitwise independent of the chunk width, probe range and GPU count (reference prefix property).
#include <algorithm>
#include <cmath>
#include <vector>

#include "pcg64.cuh"
#include "slq_common.cuh"

namespace slq {

constexpr int kSpmmWarps = 4;
constexpr int kStreamWarps = 4;
constexpr int kReduceWarps = 32;
constexpr int kProbeRun = 32;        // 64-bit PCG outputs per thread in probe_init (64 rows)
constexpr int kSecondPassGrid = 148 * 4;
constexpr int kMaxChunk = 512;       // probes per chunk (16 probe groups)

// ----------------------------------------------------------------------------- probes
template <typename VT>
__global__ void probe_init_kernel(uint64_t seed, int64_t probe_begin, int c, int64_t n, VT* __restrict__ u,
                                  int64_t ldc) {
  const int lane = threadIdx.x & 31;
  const int64_t run = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int p = blockIdx.y * 32 + lane;
  const int64_t row0 = run * (2 * kProbeRun);
  if (p >= c || row0 >= n) return;
  u128 st, inc;
  pcg64_seed_state(seed, static_cast<uint64_t>(probe_begin + p), &st, &inc);
  st = pcg_advance(st, inc, static_cast<uint64_t>(run) * kProbeRun);
  const u128 mult = pcg_mult();
  for (int m = 0; m < kProbeRun; ++m) {
    st = st * mult + inc;
    const uint64_t out = pcg_output(st);
    const int64_t r = row0 + 2 * m;
    if (r < n) u[r * ldc + p] = from_f64<VT>(((out >> 31) & 1u) ? 1.0 : -1.0);
    if (r + 1 < n) u[(r + 1) * ldc + p] = from_f64<VT>(((out >> 63) & 1u) ? 1.0 : -1.0);
  }
}

template <typename VT>
static void launch_probes(uint64_t seed, int64_t probe_begin, int c, int64_t n, VT* u, int64_t ldc,
                          cudaStream_t st) {
  const int64_t runs = (n + 2 * kProbeRun - 1) / (2 * kProbeRun);
  dim3 grid(ceil_div(runs, 4), ceil_div(c, 32));
  LaunchScope ls(K_PROBE, st);
  probe_init_kernel<VT><<<grid, 128, 0, st>>>(seed, probe_begin, c, n, u, ldc);
}

template <typename VT>
__global__ void copy_start_kernel(const double* __restrict__ q0, int64_t ldq, int c, int64_t n, VT* __restrict__ u,
                                  int64_t ldc) {
  const int64_t total = n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = idx / c;
    const int p = static_cast<int>(idx - r * c);
    u[r * ldc + p] = from_f64<VT>(q0[r * ldq + p]);
  }
}

// ----------------------------------------------------------------------------- per-probe state
struct ChunkState {
  int c = 0, cpad = 0, S = 0;
  double* rsc = nullptr;    // [S+1][cpad]  r_k = 1/beta_{k-1}, r_0 = 1/sqrt(n)
  double* alpha = nullptr;  // [S][cpad]
  double* beta = nullptr;   // [S][cpad]
  double* h = nullptr;      // [S][cpad]    CGS coefficients of the current step
  double* nb2 = nullptr;    // [cpad]       ||w'||^2
  int* steps = nullptr;     // [cpad]
  int* alive = nullptr;     // [cpad]
  int* again = nullptr;     // [cpad]
  int* any_again = nullptr; // [1]
};

__global__ void state_init_kernel(ChunkState s, int64_t n, int given_start) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s.cpad) return;
  const bool pv = p < s.c;
  // r_0: the probe +-1 block is scaled by 1/fl(sqrt(n)) (= 1/||v||); a caller-given unit start
  // vector is used as is.
  s.rsc[p] = pv ? (given_start ? 1.0 : __ddiv_rn(1.0, __dsqrt_rn(static_cast<double>(n)))) : 0.0;
  s.steps[p] = s.S;
  s.alive[p] = pv ? 1 : 0;
  s.again[p] = 0;
  for (int k = 0; k < s.S; ++k) { s.alpha[k * s.cpad + p] = 0.0; s.beta[k * s.cpad + p] = 0.0; }
  if (p == 0) *s.any_again = 0;
}

// ----------------------------------------------------------------------------- pass A: SpMM
struct SpmmArgs {
  const int64_t* offsets;
  const int32_t* cols;
  const double* weights;   // nullptr = unit
  const double* degree;
  const double* dinv;
  const int64_t* tile_rows;
  int ntiles;
  double scale;            // density: 1/trL
  const void* u;           // [n][ldc] input (unnormalised)
  const double* r;         // [cpad] per-probe scale (nullptr = 1.0)
  void* w;                 // [n][ldc] output
  int64_t ldc_in, ldc_out;
  int c, cpad;
  double* partial;         // [ntiles][cpad] alpha partials (nullptr = none)
};

template <int KIND>
__device__ __forceinline__ double op_epilogue(double x, double acc, double d, double dis, double scale) {
  if (KIND == SLQ_NORMALIZED_LAPLACIAN) {
    // nonisolated * x - dinv_sqrt * (A @ (dinv_sqrt * x))       operators.py:88-89
    const double keep = d > 0.0 ? 1.0 : 0.0;
    return __dsub_rn(__dmul_rn(keep, x), __dmul_rn(dis, acc));
  } else if (KIND == SLQ_DENSITY) {
    // scale * (d * x - A @ x)                                   operators.py:98-99
    return __dmul_rn(scale, __dsub_rn(__dmul_rn(d, x), acc));
  } else {
    // d * x - A @ x                                             operators.py:76-78
    return __dsub_rn(__dmul_rn(d, x), acc);
  }
}

template <typename VT, int KIND, bool WEIGHTED>
__global__ void __launch_bounds__(kSpmmWarps * 32)
spmm_kernel(SpmmArgs a) {
  __shared__ double red[kSpmmWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.y * 32 + lane;
  const bool pv = p < a.c;
  const double r = (a.r && pv) ? a.r[p] : 1.0;
  const VT* __restrict__ u = static_cast<const VT*>(a.u);
  VT* __restrict__ w = static_cast<VT*>(a.w);
  const int64_t* __restrict__ off = a.offsets;
  const int32_t* __restrict__ cols = a.cols;
  const double* __restrict__ dinv = a.dinv;
  const double* __restrict__ wts = a.weights;
  const int64_t ldi = a.ldc_in;

  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t rb = a.tile_rows[tile], re = a.tile_rows[tile + 1];
    double dot = 0.0;
    for (int64_t row = rb + warp; row < re; row += kSpmmWarps) {
      const int64_t beg = off[row], end = off[row + 1];
      double acc = 0.0;
      for (int64_t base = beg; base < end; base += 32) {
        const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
        int mycol = 0;
        double mys = 1.0, myw = 1.0;
        if (lane < cnt) {
          mycol = __ldg(cols + base + lane);
          if (KIND == SLQ_NORMALIZED_LAPLACIAN) mys = __ldg(dinv + mycol);
          if (WEIGHTED) myw = __ldg(wts + base + lane);
        }
        int k = 0;
        for (; k + 8 <= cnt; k += 8) {
          double xv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int cc = __shfl_sync(0xffffffffu, mycol, k + j);
            xv[j] = pv ? ldg_f64(u + static_cast<int64_t>(cc) * ldi + p) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double t = __dmul_rn(xv[j], r);
            if (KIND == SLQ_NORMALIZED_LAPLACIAN) t = __dmul_rn(__shfl_sync(0xffffffffu, mys, k + j), t);
            if (WEIGHTED) t = __dmul_rn(__shfl_sync(0xffffffffu, myw, k + j), t);
            acc = __dadd_rn(acc, t);
          }
        }
        for (; k < cnt; ++k) {
          const int cc = __shfl_sync(0xffffffffu, mycol, k);
          const double sk = __shfl_sync(0xffffffffu, mys, k);
          const double wk = __shfl_sync(0xffffffffu, myw, k);
          double t = __dmul_rn(pv ? ldg_f64(u + static_cast<int64_t>(cc) * ldi + p) : 0.0, r);
          if (KIND == SLQ_NORMALIZED_LAPLACIAN) t = __dmul_rn(sk, t);
          if (WEIGHTED) t = __dmul_rn(wk, t);
          acc = __dadd_rn(acc, t);
        }
      }
      if (pv) {
        const double x = __dmul_rn(ldg_f64(u + row * ldi + p), r);
        const double y = op_epilogue<KIND>(x, acc, __ldg(a.degree + row),
                                           KIND == SLQ_NORMALIZED_LAPLACIAN ? __ldg(dinv + row) : 0.0, a.scale);
        w[row * a.ldc_out + p] = from_f64<VT>(y);
        dot = fma(x, y, dot);
      }
    }
    if (a.partial) {
      red[warp][lane] = dot;
      __syncthreads();
      if (warp == 0) {
        double s = red[0][lane];
#pragma unroll
        for (int j = 1; j < kSpmmWarps; ++j) s += red[j][lane];
        a.partial[static_cast<int64_t>(tile) * a.cpad + blockIdx.y * 32 + lane] = s;
      }
      __syncthreads();
    }
  }
}

template <typename VT>
static void launch_spmm(int kind, const slq_graph* g, SpmmArgs a, int ngroups, cudaStream_t st) {
  dim3 grid(a.ntiles, ngroups);
  LaunchScope ls(K_SPMM, st);
  const bool wt = a.weights != nullptr;
#define SLQ_SPMM(K, W) spmm_kernel<VT, K, W><<<grid, kSpmmWarps * 32, 0, st>>>(a)
  if (kind == SLQ_NORMALIZED_LAPLACIAN) { if (wt) SLQ_SPMM(SLQ_NORMALIZED_LAPLACIAN, true); else SLQ_SPMM(SLQ_NORMALIZED_LAPLACIAN, false); }
  else if (kind == SLQ_DENSITY) { if (wt) SLQ_SPMM(SLQ_DENSITY, true); else SLQ_SPMM(SLQ_DENSITY, false); }
  else { if (wt) SLQ_SPMM(SLQ_LAPLACIAN, true); else SLQ_SPMM(SLQ_LAPLACIAN, false); }
#undef SLQ_SPMM
}

// ----------------------------------------------------------------------------- pass B: CGS
struct CgsArgs {
  int64_t n, ldc, vec_stride;      // vec_stride = n*ldc elements between basis vectors
  int64_t rows_per_tile;
  int ntiles;
  int c, cpad;
  int i;                           // current Lanczos step
  int k0, nk;                      // basis block [k0, k0+nk) handled by this launch
  int second;                      // 1: second CGS pass on u_{i+1}
  int reorth;
  const void* basis;               // u_0 .. u_S (S+1 vectors; u_{i+1} is the output slot)
  const void* w;                   // Op(q_i)
  ChunkState s;
  double* partial;                 // [ntiles][nq][cpad]
};

template <typename VT>
__device__ __forceinline__ double qval(const VT* basis, int64_t vs, int k, int64_t idx, double rk) {
  return __dmul_rn(ldg_f64(basis + k * vs + idx), rk);
}

// w' = (w - alpha q_i) - beta_{i-1} q_{i-1}    (lanczos.py:129, numpy left-to-right evaluation)
template <typename VT>
__device__ __forceinline__ double three_term(const CgsArgs& a, const VT* basis, const VT* w, int64_t idx,
                                             double al, double bp, double ri, double rim1) {
  const double wv = ldg_f64(w + idx);
  const double qi = qval(basis, a.vec_stride, a.i, idx, ri);
  const double qp = a.i > 0 ? qval(basis, a.vec_stride, a.i - 1, idx, rim1) : 0.0;
  return __dsub_rn(__dsub_rn(wv, __dmul_rn(al, qi)), __dmul_rn(bp, qp));
}

template <typename VT>
__global__ void __launch_bounds__(kStreamWarps * 32)
cgs_dot_kernel(CgsArgs a) {
  __shared__ double red[kStreamWarps][kCgsBlock + 1][32];
  if (a.second && *a.s.any_again == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.y * 32 + lane;
  const bool pv = p < a.c;
  const VT* basis = static_cast<const VT*>(a.basis);
  const VT* w = static_cast<const VT*>(a.w);
  const int cp = a.cpad;
  const double al = pv ? a.s.alpha[a.i * cp + p] : 0.0;
  const double bp = (pv && a.i > 0) ? a.s.beta[(a.i - 1) * cp + p] : 0.0;
  const double ri = pv ? a.s.rsc[a.i * cp + p] : 0.0;
  const double rim1 = (pv && a.i > 0) ? a.s.rsc[(a.i - 1) * cp + p] : 0.0;
  double rk[kCgsBlock];
#pragma unroll
  for (int kk = 0; kk < kCgsBlock; ++kk) rk[kk] = (pv && kk < a.nk) ? a.s.rsc[(a.k0 + kk) * cp + p] : 0.0;
  const int nq = a.nk + 1;

  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t rb = static_cast<int64_t>(tile) * a.rows_per_tile;
    const int64_t re = min(a.n, rb + a.rows_per_tile);
    double acc[kCgsBlock];
#pragma unroll
    for (int kk = 0; kk < kCgsBlock; ++kk) acc[kk] = 0.0;
    double nb = 0.0;
    if (pv) {
      for (int64_t row = rb + warp; row < re; row += kStreamWarps) {
        const int64_t idx = row * a.ldc + p;
        const double wp = a.second ? ldg_f64(basis + (a.i + 1) * a.vec_stride + idx)
                                   : three_term(a, basis, w, idx, al, bp, ri, rim1);
        nb = fma(wp, wp, nb);
#pragma unroll
        for (int kk = 0; kk < kCgsBlock; ++kk)
          if (kk < a.nk) acc[kk] = fma(qval(basis, a.vec_stride, a.k0 + kk, idx, rk[kk]), wp, acc[kk]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < kCgsBlock; ++kk) red[warp][kk][lane] = acc[kk];
    red[warp][kCgsBlock][lane] = nb;
    __syncthreads();
    for (int q = warp; q < nq; q += kStreamWarps) {
      const int slot = q < a.nk ? q : kCgsBlock;
      double s = red[0][slot][lane];
#pragma unroll
      for (int j = 1; j < kStreamWarps; ++j) s += red[j][slot][lane];
      a.partial[(static_cast<int64_t>(tile) * nq + q) * cp + blockIdx.y * 32 + lane] = s;
    }
    __syncthreads();
  }
}

template <typename VT>
__global__ void __launch_bounds__(kStreamWarps * 32)
cgs_update_kernel(CgsArgs a) {
  extern __shared__ double dyn[];          // [nk][32] h, then [nk][32] r
  __shared__ double red[kStreamWarps][32];
  if (a.second && *a.s.any_again == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = blockIdx.y * 32 + lane;
  const int cp = a.cpad;
  const bool pv = p < a.c && (!a.second || a.s.again[p]);
  const VT* basis = static_cast<const VT*>(a.basis);
  VT* out = const_cast<VT*>(basis) + (a.i + 1) * a.vec_stride;
  const VT* w = static_cast<const VT*>(a.w);
  const int nk = a.reorth ? a.i + 1 : 0;
  double* hs = dyn;
  double* rs = dyn + nk * 32;
  for (int k = warp; k < nk; k += kStreamWarps) {
    hs[k * 32 + lane] = pv ? a.s.h[k * cp + p] : 0.0;
    rs[k * 32 + lane] = pv ? a.s.rsc[k * cp + p] : 0.0;
  }
  __syncthreads();
  const double al = pv ? a.s.alpha[a.i * cp + p] : 0.0;
  const double bp = (pv && a.i > 0) ? a.s.beta[(a.i - 1) * cp + p] : 0.0;
  const double ri = pv ? a.s.rsc[a.i * cp + p] : 0.0;
  const double rim1 = (pv && a.i > 0) ? a.s.rsc[(a.i - 1) * cp + p] : 0.0;

  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t rb = static_cast<int64_t>(tile) * a.rows_per_tile;
    const int64_t re = min(a.n, rb + a.rows_per_tile);
    double nrm = 0.0;
    if (pv) {
      for (int64_t row = rb + warp; row < re; row += kStreamWarps) {
        const int64_t idx = row * a.ldc + p;
        const double wp = a.second ? ldg_f64(out + idx) : three_term(a, basis, w, idx, al, bp, ri, rim1);
        // basis.T @ h, accumulated over k in order, then one subtraction (lanczos.py:73)
        double proj = 0.0;
        for (int k = 0; k < nk; ++k)
          proj = __dadd_rn(proj, __dmul_rn(qval(basis, a.vec_stride, k, idx, rs[k * 32 + lane]), hs[k * 32 + lane]));
        const VT v = from_f64<VT>(nk ? __dsub_rn(wp, proj) : wp);
        out[idx] = v;
        const double vd = to_f64(v);
        nrm = fma(vd, vd, nrm);
      }
    }
    red[warp][lane] = nrm;
    __syncthreads();
    if (warp == 0) {
      double s = red[0][lane];
#pragma unroll
      for (int j = 1; j < kStreamWarps; ++j) s += red[j][lane];
      a.partial[static_cast<int64_t>(tile) * cp + blockIdx.y * 32 + lane] = s;
    }
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------- reductions
enum ReduceMode { RED_ALPHA = 0, RED_CGS = 1, RED_NORM = 2, RED_NORM2 = 3 };

struct ReduceArgs {
  const double* partial;   // [ntiles][nq][cpad]
  int ntiles, nq, cpad, c;
  int mode;
  int i, k0, nk, reorth;
  int second;              // 1: reduction of the conditional second CGS pass
  double tol;              // breakdown tolerance 1e-12 * interval_hi
  ChunkState s;
};

__global__ void __launch_bounds__(kReduceWarps * 32)
reduce_kernel(ReduceArgs a) {
  __shared__ double red[kReduceWarps][32];
  if (a.second && *a.s.any_again == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = blockIdx.x;
  const int p = blockIdx.y * 32 + lane;
  double s = 0.0;
  for (int t = warp; t < a.ntiles; t += kReduceWarps)
    s += a.partial[(static_cast<int64_t>(t) * a.nq + q) * a.cpad + p];
  red[warp][lane] = s;
  __syncthreads();
  if (warp != 0) return;
  double tot = red[0][lane];
  for (int j = 1; j < kReduceWarps; ++j) tot += red[j][lane];
  const int cp = a.cpad;
  const bool pv = p < a.c;
  switch (a.mode) {
    case RED_ALPHA:
      if (pv && a.s.alive[p]) a.s.alpha[a.i * cp + p] = tot;
      if (blockIdx.y == 0 && lane == 0) *a.s.any_again = 0;
      break;
    case RED_CGS:
      if (q < a.nk) a.s.h[(a.k0 + q) * cp + p] = tot;
      else if (!a.second) a.s.nb2[p] = tot;
      break;
    case RED_NORM:
    case RED_NORM2: {
      if (!pv || !a.s.alive[p]) break;
      const double b = sqrt(tot);
      if (a.mode == RED_NORM) {
        if (a.reorth && b < 0.5 * sqrt(a.s.nb2[p])) {    // lanczos.py:75
          a.s.again[p] = 1;
          *a.s.any_again = 1;
          break;
        }
      } else {
        if (!a.s.again[p]) break;
        a.s.again[p] = 0;
      }
      if (b <= a.tol) {                                  // lanczos.py:133-134
        a.s.steps[p] = a.i + 1;
        a.s.alive[p] = 0;
        a.s.rsc[(a.i + 1) * cp + p] = 0.0;
      } else {
        a.s.beta[a.i * cp + p] = b;
        a.s.rsc[(a.i + 1) * cp + p] = __ddiv_rn(1.0, b);
      }
      break;
    }
  }
}

static void launch_reduce(ReduceArgs a, int ngroups, cudaStream_t st) {
  dim3 grid(a.nq, ngroups);
  LaunchScope ls(K_REDUCE, st);
  reduce_kernel<<<grid, kReduceWarps * 32, 0, st>>>(a);
}

// ----------------------------------------------------------------------------- outputs
__global__ void scatter_out_kernel(ChunkState s, int64_t col0, int S, double* alpha, double* beta,
                                   int32_t* steps) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= s.c) return;
  const int64_t o = (col0 + p) * S;
  const int st = s.steps[p];
  for (int k = 0; k < S; ++k) {
    alpha[o + k] = k < st ? s.alpha[k * s.cpad + p] : 0.0;
    beta[o + k] = k + 1 < st ? s.beta[k * s.cpad + p] : 0.0;
  }
  steps[col0 + p] = st;
}

// ----------------------------------------------------------------------------- engine
static void ensure_pool(int dev) {
  static bool done[64] = {false};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

static int choose_chunk(const slq_graph* g, int64_t count, int S, int vbytes) {
  size_t freeb = 0, total = 0;
  cudaMemGetInfo(&freeb, &total);
  const double budget = 0.85 * static_cast<double>(freeb);
  const double per_probe = static_cast<double>(S + 2) * static_cast<double>(std::max<int64_t>(g->n, 1)) * vbytes;
  int64_t c = static_cast<int64_t>(budget / std::max(per_probe, 1.0));
  c = std::min<int64_t>({c, count, kMaxChunk});
  return static_cast<int>(std::max<int64_t>(c, 1));
}

template <typename VT>
static int run_chunk(const slq_graph* g, int kind, uint64_t seed, int64_t probe0, const double* q0, int64_t ldq,
                     int c, int S, int reorth, double* alpha_out, double* beta_out, int32_t* steps_out, int64_t col0,
                     cudaStream_t st) {
  const int64_t n = g->n;
  const int vb = sizeof(VT);
  // ldc: probes padded to a 32-byte sector multiple
  const int64_t ldc = ((c * vb + 31) / 32) * 32 / vb;
  const int ngroups = ceil_div(c, 32);
  const int cpad = ngroups * 32;
  const int64_t vs = n * ldc;
  double lo = 0, hi = 0;
  int rc = slq_operator_interval(g, kind, &lo, &hi);
  if (rc) return rc;
  const double tol = 1e-12 * hi;                           // lanczos.py:36,109-110

  // workspace: S+1 basis slots + w, state arrays, partials
  const int nq_max = std::max(kCgsBlock + 1, 1);
  const int64_t ptiles = std::max(g->ntiles, g->ntiles_stream);
  size_t bytes_vec = static_cast<size_t>(vs) * vb * (S + 2);
  size_t bytes_state = sizeof(double) * cpad * (4 * (S + 1) + 2) + sizeof(int) * (3 * cpad + 4);
  size_t bytes_part = sizeof(double) * ptiles * nq_max * cpad;
  char* ws = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes_vec + bytes_state + bytes_part + 256, st));
  VT* basis = reinterpret_cast<VT*>(ws);
  VT* wv = basis + (S + 1) * vs;
  double* dstate = reinterpret_cast<double*>(ws + ((bytes_vec + 127) / 128) * 128);
  ChunkState s;
  s.c = c; s.cpad = cpad; s.S = S;
  s.rsc = dstate;
  s.alpha = s.rsc + (S + 1) * cpad;
  s.beta = s.alpha + (S + 1) * cpad;
  s.h = s.beta + (S + 1) * cpad;
  s.nb2 = s.h + (S + 1) * cpad;
  int* istate = reinterpret_cast<int*>(s.nb2 + cpad);
  s.steps = istate;
  s.alive = istate + cpad;
  s.again = istate + 2 * cpad;
  s.any_again = istate + 3 * cpad;
  double* partial = reinterpret_cast<double*>(ws + ((bytes_vec + 127) / 128) * 128 + ((bytes_state + 127) / 128) * 128);

  {
    LaunchScope ls(K_PROBE, st);
    state_init_kernel<<<ceil_div(cpad, 128), 128, 0, st>>>(s, n, q0 != nullptr);
  }
  if (q0) {
    LaunchScope ls(K_PROBE, st);
    copy_start_kernel<VT><<<std::max(1, std::min(ceil_div(n * c, 256), 148 * 16)), 256, 0, st>>>(q0, ldq, c, n, basis, ldc);
  } else {
    launch_probes<VT>(seed, probe0, c, n, basis, ldc, st);
  }

  SpmmArgs sa{};
  sa.offsets = g->offsets; sa.cols = g->cols; sa.weights = g->weights; sa.degree = g->degree; sa.dinv = g->dinv;
  sa.tile_rows = g->tile_rows; sa.ntiles = g->ntiles;
  sa.scale = kind == SLQ_DENSITY ? 1.0 / g->trace_l : 0.0;
  sa.w = wv; sa.ldc_in = ldc; sa.ldc_out = ldc; sa.c = c; sa.cpad = cpad; sa.partial = partial;

  CgsArgs ca{};
  ca.n = n; ca.ldc = ldc; ca.vec_stride = vs; ca.rows_per_tile = g->rows_per_stream_tile;
  ca.ntiles = g->ntiles_stream; ca.c = c; ca.cpad = cpad; ca.basis = basis; ca.w = wv; ca.s = s;
  ca.partial = partial; ca.reorth = reorth;

  ReduceArgs ra{};
  ra.partial = partial; ra.cpad = cpad; ra.c = c; ra.s = s; ra.tol = tol; ra.reorth = reorth;

  const dim3 sgrid(g->ntiles_stream, ngroups);
  const size_t upd_smem = reorth ? sizeof(double) * 2 * 32 * S : 0;
  if (upd_smem > 48 * 1024)
    SLQ_CUDA(cudaFuncSetAttribute(cgs_update_kernel<VT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(upd_smem)));
  const dim3 sgrid2(std::min(g->ntiles_stream, kSecondPassGrid), ngroups);

  for (int i = 0; i < S; ++i) {
    sa.u = basis + i * vs;
    sa.r = s.rsc + i * cpad;
    launch_spmm<VT>(kind, g, sa, ngroups, st);
    ra.mode = RED_ALPHA; ra.ntiles = g->ntiles; ra.nq = 1; ra.i = i;
    launch_reduce(ra, ngroups, st);
    if (i == S - 1) break;
    ca.i = i;
    ca.second = 0;
    if (reorth) {
      for (int k0 = 0; k0 <= i; k0 += kCgsBlock) {
        ca.k0 = k0; ca.nk = std::min(kCgsBlock, i + 1 - k0);
        {
          LaunchScope ls(K_CGS_DOT, st);
          cgs_dot_kernel<VT><<<sgrid, kStreamWarps * 32, 0, st>>>(ca);
        }
        ra.mode = RED_CGS; ra.ntiles = g->ntiles_stream; ra.nq = ca.nk + 1; ra.k0 = k0; ra.nk = ca.nk;
        launch_reduce(ra, ngroups, st);
      }
    }
    {
      LaunchScope ls(K_CGS_UPDATE, st);
      cgs_update_kernel<VT><<<sgrid, kStreamWarps * 32, upd_smem, st>>>(ca);
    }
    ra.mode = RED_NORM; ra.ntiles = g->ntiles_stream; ra.nq = 1;
    launch_reduce(ra, ngroups, st);
    if (reorth) {
      // conditional second CGS pass (lanczos.py:75-76); kernels exit unless a probe asked for it
      ca.second = 1;
      ra.second = 1;
      for (int k0 = 0; k0 <= i; k0 += kCgsBlock) {
        ca.k0 = k0; ca.nk = std::min(kCgsBlock, i + 1 - k0);
        {
          LaunchScope ls(K_CGS_DOT, st);
          cgs_dot_kernel<VT><<<sgrid2, kStreamWarps * 32, 0, st>>>(ca);
        }
        ra.mode = RED_CGS; ra.ntiles = g->ntiles_stream; ra.nq = ca.nk + 1; ra.k0 = k0; ra.nk = ca.nk;
        launch_reduce(ra, ngroups, st);
      }
      {
        LaunchScope ls(K_CGS_UPDATE, st);
        cgs_update_kernel<VT><<<sgrid2, kStreamWarps * 32, upd_smem, st>>>(ca);
      }
      ra.mode = RED_NORM2; ra.ntiles = g->ntiles_stream; ra.nq = 1;
      launch_reduce(ra, ngroups, st);
      ca.second = 0;
      ra.second = 0;
    }
  }
  {
    LaunchScope ls(K_REDUCE, st);
    scatter_out_kernel<<<ceil_div(c, 128), 128, 0, st>>>(s, col0, S, alpha_out, beta_out, steps_out);
  }
  SLQ_CUDA(cudaGetLastError());
  SLQ_CUDA(cudaFreeAsync(ws, st));
  return SLQ_OK;
}

}  // namespace slq

using namespace slq;

static int lanczos_entry(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, const double* q0,
                         int64_t ldq, int64_t count, int steps, int reorth, int dtype, double* alpha, double* beta,
                         int32_t* steps_out, void* stream) {
  if (!g) return fail(SLQ_ERR_VALUE, "NULL graph");
  if (steps < 1) return fail(SLQ_ERR_VALUE, "step budget must be >= 1");
  if (count < 0 || probe_begin < 0) return fail(SLQ_ERR_VALUE, "negative probe range");
  if (kind < 0 || kind > 2) return fail(SLQ_ERR_VALUE, "unknown operator kind");
  if (dtype != SLQ_F64 && dtype != SLQ_F32) return fail(SLQ_ERR_VALUE, "dtype must be SLQ_F64 or SLQ_F32");
  if (g->n == 0) return fail(SLQ_ERR_VALUE, "start vector must have unit norm");
  double lo, hi;
  int rc = slq_operator_interval(g, kind, &lo, &hi);
  if (rc) return rc;
  const int S = static_cast<int>(std::min<int64_t>(steps, g->n));   // lanczos.py:105
  if (S > kMaxSteps) return fail(SLQ_ERR_VALUE, "steps > 128 not supported");
  if (reorth < 0) reorth = S <= 100 ? 1 : 0;                          // lanczos.py:106-107
  if (count == 0) return SLQ_OK;
  if (q0 && ldq < count) return fail(SLQ_ERR_VALUE, "ldq < count");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ensure_pool(g->device);
  const int vb = dtype == SLQ_F64 ? 8 : 4;
  const int cmax = choose_chunk(g, count, S, vb);
  for (int64_t done = 0; done < count;) {
    const int c = static_cast<int>(std::min<int64_t>(cmax, count - done));
    const double* qc = q0 ? q0 + done : nullptr;
    rc = dtype == SLQ_F64
             ? run_chunk<double>(g, kind, seed, probe_begin + done, qc, ldq, c, S, reorth, alpha, beta, steps_out, done, st)
             : run_chunk<float>(g, kind, seed, probe_begin + done, qc, ldq, c, S, reorth, alpha, beta, steps_out, done, st);
    if (rc) return rc;
    done += c;
  }
  return SLQ_OK;
}

extern "C" int slq_lanczos(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count,
                           int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                           void* stream) {
  return lanczos_entry(g, kind, seed, probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha, beta, steps_out,
                       stream);
}

extern "C" int slq_lanczos_start(const slq_graph* g, int kind, const double* q0, int64_t ldq, int64_t count,
                                 int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                                 void* stream) {
  if (!q0) return fail(SLQ_ERR_VALUE, "NULL start block");
  return lanczos_entry(g, kind, 0, 0, q0, ldq, count, steps, reorth, dtype, alpha, beta, steps_out, stream);
}

extern "C" int slq_operator_apply(const slq_graph* g, int kind, const double* x, double* y, int64_t ncols,
                                  int64_t ld, void* stream) {
  if (!g || (!x && g->n) || (!y && g->n)) return fail(SLQ_ERR_VALUE, "NULL argument");
  if (kind < 0 || kind > 2) return fail(SLQ_ERR_VALUE, "unknown operator kind");
  double lo, hi;
  int rc = slq_operator_interval(g, kind, &lo, &hi);
  if (rc) return rc;
  if (ncols <= 0 || g->n == 0) return SLQ_OK;
  if (ld < ncols) return fail(SLQ_ERR_VALUE, "ld < ncols");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SpmmArgs sa{};
  sa.offsets = g->offsets; sa.cols = g->cols; sa.weights = g->weights; sa.degree = g->degree; sa.dinv = g->dinv;
  sa.tile_rows = g->tile_rows; sa.ntiles = g->ntiles;
  sa.scale = kind == SLQ_DENSITY ? 1.0 / g->trace_l : 0.0;
  sa.u = x; sa.r = nullptr; sa.w = y; sa.ldc_in = ld; sa.ldc_out = ld;
  sa.c = static_cast<int>(ncols); sa.cpad = ceil_div(ncols, 32) * 32; sa.partial = nullptr;
  launch_spmm<double>(kind, g, sa, ceil_div(ncols, 32), st);
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

extern "C" int slq_probes(uint64_t seed, int64_t probe_begin, int64_t count, int64_t n, double* out, int64_t ld,
                          void* stream) {
  if (count < 0 || n < 0 || ld < count) return fail(SLQ_ERR_VALUE, "bad probe block shape");
  if (count == 0 || n == 0) return SLQ_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int64_t done = 0; done < count; done += 1024) {
    const int c = static_cast<int>(std::min<int64_t>(1024, count - done));
    launch_probes<double>(seed, probe_begin + done, c, n, out + done, ld, st);
  }
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

extern "C" int slq_probe_state(uint64_t seed, uint64_t index, uint64_t out_host[4]) {
  if (!out_host) return fail(SLQ_ERR_VALUE, "NULL output");
  u128 st, inc;
  pcg64_seed_state(seed, index, &st, &inc);
  out_host[0] = static_cast<uint64_t>(st >> 64);
  out_host[1] = static_cast<uint64_t>(st);
  out_host[2] = static_cast<uint64_t>(inc >> 64);
  out_host[3] = static_cast<uint64_t>(inc);
  return SLQ_OK;
}
