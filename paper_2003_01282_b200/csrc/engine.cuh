// Shared engine definitions: chunk state, reductions, the SpMM pass and the staged CGS step
// kernel (templates).  lanczos.cu runs the engine; spmm_*.cu and step_*.cu instantiate the
// heavy kernel families per vector type so the library builds in parallel translation units.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>
#include "bulk_pipe.cuh"
#include "pcg64.cuh"
#include "slq_common.cuh"

namespace slq {



constexpr int kProbeRun = 32;        // 64-bit PCG outputs per thread in probe_init (64 rows)
constexpr int kSecondPassGrid = 148 * 4;
constexpr int kMaxChunk = 256;       // probes per chunk (flat CGS CTAs of <= 512 threads)

// ----------------------------------------------------------------------------- probes
// Rademacher probes: u (if not null) gets +-1 values; bits (if not null) gets one bit per probe,
// bits[row][kBitWords] with word g = probes 32g..32g+31 (bit set = +1).  A warp = 32 probes of one
// group over a run of 2*kProbeRun rows.
constexpr int kBitWords = 4;   // bitmask row stride in 32-bit words (16 B: bulk-copy aligned; c <= 128)
// Step-0 records of the normalized Laplacian on large graphs: [bits (4 words) | dinv (2 words) | pad],
// 32 bytes per row, so the first SpMM fetches one sector per nonzero instead of bits + dinv[col]
constexpr int kRecWords = 8;

template <typename VT>
__global__ void probe_init_kernel(SeedKey seed, int64_t probe_begin, int c, int64_t n, VT* __restrict__ u,
                                  int64_t ldc, uint32_t* __restrict__ bits,
                                  const int32_t* __restrict__ remap) {
  const int lane = threadIdx.x & 31;
  const int64_t run = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int p = blockIdx.y * 32 + lane;
  const int64_t row0 = run * (2 * kProbeRun);
  if (row0 >= n) return;                       // warp-uniform
  const bool pv = p < c;
  u128 st = 0, inc = 0;
  if (pv) {
    pcg64_seed_state(seed, static_cast<uint64_t>(probe_begin + p), &st, &inc);
    st = pcg_advance(st, inc, static_cast<uint64_t>(run) * kProbeRun);
  }
  const u128 mult = pcg_mult();
  for (int m = 0; m < kProbeRun; ++m) {
    uint64_t out = 0;
    if (pv) {
      st = st * mult + inc;
      out = pcg_output(st);
    }
    const int64_t r = row0 + 2 * m;
    const bool b0 = (out >> 31) & 1u, b1 = (out >> 63) & 1u;
    if (u && pv) {
      if (r < n) u[r * ldc + p] = from_f64<VT>(b0 ? 1.0 : -1.0);
      if (r + 1 < n) u[(r + 1) * ldc + p] = from_f64<VT>(b1 ? 1.0 : -1.0);
    }
    if (bits) {
      const uint32_t w0 = __ballot_sync(0xffffffffu, pv && b0);
      const uint32_t w1 = __ballot_sync(0xffffffffu, pv && b1);
      if (lane == 0) {
        // remap (isolated-vertex fold): stream position r -> folded row, -1 = folded away
        const int64_t d0 = r < n ? (remap ? remap[r] : r) : -1;
        const int64_t d1 = r + 1 < n ? (remap ? remap[r + 1] : r + 1) : -1;
        if (d0 >= 0) bits[d0 * kBitWords + blockIdx.y] = w0;
        if (d1 >= 0) bits[d1 * kBitWords + blockIdx.y] = w1;
      }
    }
  }
}

template <typename VT>
static void launch_probes(const SeedKey& seed, int64_t probe_begin, int c, int64_t n, VT* u, int64_t ldc,
                          cudaStream_t st, uint32_t* bits = nullptr, const int32_t* remap = nullptr) {
  const int64_t runs = (n + 2 * kProbeRun - 1) / (2 * kProbeRun);
  dim3 grid(ceil_div(runs, 4), ceil_div(c, 32));
  LaunchScope ls(K_PROBE, st);
  probe_init_kernel<VT><<<grid, 128, 0, st>>>(seed, probe_begin, c, n, u, ldc, bits, remap);
}

// [bits | dinv | pad] records of every row (kRecWords words) for the first normalized-Laplacian SpMM
static __global__ void step0_records_kernel(const uint32_t* __restrict__ bits, const double* __restrict__ dinv,
                                            int64_t n, uint32_t* __restrict__ rec) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const uint4 b = *reinterpret_cast<const uint4*>(bits + r * kBitWords);
    const double d = dinv[r];
    uint4 t;
    t.x = static_cast<uint32_t>(__double_as_longlong(d));
    t.y = static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(d)) >> 32);
    t.z = 0u;
    t.w = 0u;
    reinterpret_cast<uint4*>(rec + r * kRecWords)[0] = b;
    reinterpret_cast<uint4*>(rec + r * kRecWords)[1] = t;
  }
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
  // staged path (Gram form of CGS): raw sums and the Gram matrix of the stored basis
  double* cdot = nullptr;   // [S+1][cpad]  sum_rows u_k . w            (k <= i)
  double* gram = nullptr;   // [S+1][cpad]  sum_rows u_k . u_{i+1}      (k <= i), row of the new vector
  double* nrm2 = nullptr;   // [cpad]       ||u_{i+1}||^2
  double* G = nullptr;      // [gstride*gstride][cpad]  G(k,j) = q_k . q_j (staged steps only: k, j <= 17)
  int gstride = 0;          // min(S + 1, kCgsBlock + 2)
  int* steps = nullptr;     // [cpad]
  int* alive = nullptr;     // [cpad]
  int* again = nullptr;     // [cpad]
  int* any_again = nullptr; // [1]
  int* second_passes = nullptr;   // graph counter: probe-steps that ran the second CGS pass (diagnostics)
  unsigned int* barrier = nullptr;   // [S] grid-barrier counters of the persistent step kernels
  unsigned long long* work = nullptr;   // [S][4] SpMM work counters
};

static __global__ void state_init_kernel(ChunkState s, int64_t n, int given_start) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < s.S) s.barrier[p] = 0u;
  if (p < 4 * s.S) s.work[p] = 0ull;
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

// ----------------------------------------------------------------------------- reductions
enum ReduceMode { RED_ALPHA = 0, RED_CGS = 1, RED_NORM = 2, RED_NORM2 = 3 };

struct ReduceArgs {
  const double* partial;   // [ntiles][nq][cpad]
  int ntiles, nq, cpad, c;
  int mode;
  int i, k0, nk, reorth;
  int second;              // 1: reduction of the conditional second CGS pass
  int kind;                // operator kind: breakdown tolerance 1e-12 * interval_hi (lanczos.py:36,110)
  const double* dscal;     // device graph scalars (Laplacian interval_hi = dscal[4])
  ChunkState s;
  // operator-pair chunk (slq_rules_pair): columns >= split belong to kind2 (same probes, second
  // operator); split >= c: a plain chunk
  int kind2 = -1;
  int split = 1 << 30;
};
__host__ __device__ __forceinline__ int kind_of_column(const ReduceArgs& a, int p) { return p < a.split ? a.kind : a.kind2; }

constexpr int kReduceWarps = 16;
constexpr int kStripes = 16;   // fixed partition of the partial rows: the sum order never depends on
                               // the CTA shape that runs the reduction

// Per-probe scalar logic applied to a fully reduced quantity (lanczos.py:123-137).
static __device__ void apply_reduced(const ReduceArgs& a, int q, int p, double tot, bool first_slice) {
  const int cp = a.cpad;
  const bool pv = p < a.c;
  switch (a.mode) {
    case RED_ALPHA:
      if (pv && a.s.alive[p]) a.s.alpha[a.i * cp + p] = tot;
      if (first_slice && p == 0) *a.s.any_again = 0;
      break;
    case RED_CGS:
      if (q < a.nk) a.s.h[(a.k0 + q) * cp + p] = tot * a.s.rsc[(a.k0 + q) * cp + p];
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
          if (a.s.second_passes) atomicAdd(a.s.second_passes, 1);
          break;
        }
      } else {
        if (!a.s.again[p]) break;
        a.s.again[p] = 0;
      }
      const int kd = kind_of_column(a, p);
      const double hi = kd == SLQ_NORMALIZED_LAPLACIAN ? 2.0 : (kd == SLQ_DENSITY ? 1.0 : a.dscal[4]);
      if (b <= 1e-12 * hi) {                             // lanczos.py:133-134
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

// Reduce quantity q for the 32 probes of `group` over a.ntiles partial rows, with any number of
// warps (>= 1).  All threads of the CTA must call it.  red: kStripes*32 doubles of shared memory.
static __device__ void reduce_slice(const ReduceArgs& a, int q, int group, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int p = group * 32 + lane;
  const int64_t stride = static_cast<int64_t>(a.nq) * a.cpad;
  const double* src = a.partial + static_cast<int64_t>(q) * a.cpad + p;
  for (int sidx = warp; sidx < kStripes; sidx += nw) {
    double s = 0.0;
    int t = sidx;
    for (; t + 3 * kStripes < a.ntiles; t += 4 * kStripes) {
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = src[(t + j * kStripes) * stride];
#pragma unroll
      for (int j = 0; j < 4; ++j) s += v[j];
    }
    for (; t < a.ntiles; t += kStripes) s += src[t * stride];
    red[sidx * 32 + lane] = s;
  }
  __syncthreads();
  if (warp == 0) {
    double tot = red[lane];
    for (int j = 1; j < kStripes; ++j) tot += red[j * 32 + lane];
    apply_reduced(a, q, p, tot, group == 0 && q == 0);
  }
  __syncthreads();
}

static __global__ void __launch_bounds__(kReduceWarps * 32)
reduce_kernel(ReduceArgs a) {
  __shared__ double red[kStripes * 32];
  if (a.second && *a.s.any_again == 0) return;
  reduce_slice(a, blockIdx.x, blockIdx.y, red);
}

// ----------------------------------------------------------------------------- launch geometry
// A CTA covers one block of up to kBlk = 128 probes; lane l owns probes l, l+32, l+64, l+96 of the
// block (PPL = probes per lane), so one shuffled column index feeds PPL coalesced 256-byte gathers.
// Which thread owns a probe never changes its arithmetic: every per-probe sum runs in a fixed order
// set by the graph's tiles and the warp count, never by c.
constexpr int kBlk = 128;
// probes per SpMM CTA block (grid.y = ceil(c / kSpmmBlk)): 64 gives each lane <= 2 probes, so a warp
// keeps twice the gathered rows in flight in the same registers
#ifndef SLQ_SPMM_BLK
#define SLQ_SPMM_BLK 128
#endif
constexpr int kSpmmBlk = SLQ_SPMM_BLK;
constexpr int kSpmmWarps = 8;
#ifndef SLQ_SPMM_UNRF
#define SLQ_SPMM_UNRF 8    // gathered values in flight per lane in the full-warp mapping (UNR * PPL)
#endif

__device__ __forceinline__ bool probe_ok(int p, int c) { return p < c; }

// ----------------------------------------------------------------------------- pass A: SpMM
struct SpmmArgs {
  const int64_t* offsets;
  const int32_t* cols;
  const double* weights;   // nullptr = unit
  const double* degree;
  const double* dinv;
  const int64_t* tile_rows;
  int ntiles;
  // fine row tiles + sizes for the flat kernel (spmm_flat.cu); ftile_rows = nullptr: not used
  const int64_t* ftile_rows = nullptr;
  int nftiles = 0;
  int64_t n_rows = 0, nnz_total = 0;
  const double* dscal;     // device graph scalars; density scale 1/tr L = dscal[3]
  const void* u;           // [n][ldc] input (unnormalised)
  const double* r;         // [cpad] per-probe scale (nullptr = 1.0)
  void* w;                 // [n][ldc] output
  int64_t ldc_in, ldc_out;
  int c, cpad;
  ReduceArgs red;          // operator kind / scalars for the step kernel's long-row finish
  // long rows (graph.cu): device counts, segment table, per-segment partial sums [max_seg][cpad]
  const int64_t* long_counts;
  const int32_t* long_rows;
  const int64_t* long_seg_first;
  const int32_t* seg_row;
  const int64_t* seg_begin;
  int64_t max_long;
  int64_t max_seg;           // host upper bound of the segment count (grid sizing)
  double* segpart;
  unsigned long long* work;  // [probe blocks] zeroed work counters of this launch
  const uint32_t* bits;      // first step: u_0 as a probe bitmask [n][kBitWords] (nullptr = use u)
  const uint32_t* rec = nullptr;   // first step, normalized Laplacian: [n][kRecWords] bits + dinv records
                                   // for the gathers (bits still serves the own-row values)
  const void* upre;          // normalized Laplacian: dinv (.) u to gather (nullptr = gather u, times dinv[col])
  // L2 persisting window over the gathered vector's first rows (degree-ordered fold: the hub rows);
  // win_rows = 0: no window
  int64_t win_rows = 0;
  // operator-pair chunk: columns >= split use the density epilogue (and plain gathers); flat kernel only
  int split = 1 << 30;
};

bool launch_spmm_flat_f32(int kind, const SpmmArgs& a, cudaStream_t st);   // spmm_flat.cu
bool launch_spmm_flat_f64(int kind, const SpmmArgs& a, cudaStream_t st);

// SpMM-internal kind: the normalized Laplacian gathering the PRESCALED vector dinv (.) u (written by
// the previous step kernel), so no dinv[col] gather per nonzero; the epilogue is the normalized one.
constexpr int kNLPre = 3;
template <int KIND>
__host__ __device__ constexpr bool nl_kind() { return KIND == SLQ_NORMALIZED_LAPLACIAN || KIND == kNLPre; }

template <int KIND>
__device__ __forceinline__ double op_epilogue(double x, double acc, double d, double dis, double scale) {
  if (nl_kind<KIND>()) {
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

// One term of the in-row sum: A_jk * (dinv_k * x_k) with x_k = u_k * r (operators.py:89 order).
template <int KIND, bool WEIGHTED>
__device__ __forceinline__ double gather_term(double xraw, double r, double sk, double wk) {
  double t = __dmul_rn(xraw, r);
  if (KIND == SLQ_NORMALIZED_LAPLACIAN) t = __dmul_rn(sk, t);
  if (WEIGHTED) t = __dmul_rn(wk, t);
  return t;
}

// acc[j] = sum over nonzeros [beg, end) of one row (beg is a row start, or a segment start a
// multiple of kSeg after it).
//  EXACT (operator apply, r == 1): t = fl(dinv_c * u_c) [* w], acc = fl(acc + t) in stored order:
//        the reference's csr_matvec order and rounding, bit for bit.
//  !EXACT (Lanczos): FMA sums with s_c = dinv_c [* w]; the caller multiplies by the probe scale r
//        (q = r u is never formed per gathered value).  Narrow chunks (c <= 32, PPL = 1) sum a row
//        as two chains, s_even over its even positions and s_odd over the odd ones, acc = s_even +
//        s_odd — the same order in the full-warp mapping (lane = probe, both chains in one lane)
//        and the HALF mapping (c <= 16: each half-warp gathers every other nonzero, so one warp
//        instruction fetches two rows' worth of probes).  Wide chunks (PPL >= 2) use one
//        sequential chain (fewer registers, one more resident CTA per SM).  Results are bitwise
//        independent of the chunk width within each class, like the step kernel's slot classes.
// Columns are loaded 32 at a time; each lane turns its column into an element offset once and the
// warp broadcasts offsets with one shuffle per nonzero.  Probe slots beyond c are clamped to a valid
// column (loaded, never stored), so the loads need no predicates.
template <typename VT, int KIND, bool WEIGHTED, int PPL, bool BITS, bool EXACT, bool HALF, bool V2 = false>
__device__ __forceinline__ void gather_range(const int32_t* __restrict__ cols, const double* __restrict__ dinv,
                                             const double* __restrict__ wts, const VT* __restrict__ u, int64_t ldi,
                                             const uint32_t* __restrict__ bits, const int* pidx, int64_t beg,
                                             int64_t end, double* acc) {
  // EXACT runs only for the operator apply (probe scale r == 1: fl(x * 1) == x)
  constexpr unsigned FULL = 0xffffffffu;
  // narrow chunks (PPL == 1, full-warp or HALF) sum a row as two chains (even / odd positions);
  // wide chunks (PPL >= 2) as one sequential chain: each order is fixed within its class
  constexpr bool TWO = PPL == 1;
  const int lane = threadIdx.x & 31;
  const int plane = HALF ? (lane & 15) : lane;   // probe lane
  const int sub = HALF ? (lane >> 4) : 0;        // HALF: chain (position parity) of this half
  const int boff = blockIdx.y * (kSpmmBlk / 32);  // bitmask word of this CTA's first probe
  constexpr bool SK = KIND == SLQ_NORMALIZED_LAPLACIAN || (!EXACT && WEIGHTED);   // kNLPre: weights only
  double a0[PPL], a1[PPL];
#pragma unroll
  for (int j = 0; j < PPL; ++j) a0[j] = a1[j] = 0.0;
  auto value = [&](const VT* src, const uint32_t* brow, int j) -> double {
    if (BITS) return ((__ldg(brow + boff + j) >> plane) & 1u) ? 1.0 : -1.0;
    return ldg_f64(src + pidx[j]);
  };
  for (int64_t base = beg; base < end; base += 32) {
    const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
    int64_t myoff = 0;
    double mys = 1.0, myw = 1.0;
    if (lane < cnt) {
      const int32_t raw = __ldg(cols + base + lane);
      const int64_t col = raw;
      myoff = col * ldi;   // BITS: ldi is the bitmask row stride (kBitWords, or kRecWords for records)
      if (KIND == SLQ_NORMALIZED_LAPLACIAN) {
        // step-0 records [bits | dinv]: dinv comes from the same 32-byte sector as the gathered bits
        mys = (BITS && ldi == kRecWords) ? __ldg(reinterpret_cast<const double*>(bits + col * kRecWords + kBitWords))
                                         : __ldg(dinv + col);
      }
      if (WEIGHTED) myw = __ldg(wts + base + lane);
      if (!EXACT && WEIGHTED) mys *= myw;   // s_c = dinv_c * w (or w)
    }
    if (HALF && PPL == 2) {
      // HALF2 (16 < c <= 32): lane (plane) holds probes 2 plane, 2 plane + 1 and reads them with one
      // 2-element vector load, so a half-warp gathers a whole row and a warp instruction two rows;
      // this half takes positions 2m + sub (its chain), U pairs in flight
      using V2 = typename std::conditional<std::is_same<VT, double>::value, double2, float2>::type;
      constexpr int U = 8;
      const int npairs = (cnt + 1) >> 1;
      int m = 0;
      for (; m + U <= npairs; m += U) {
        V2 xv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int64_t o = __shfl_sync(FULL, myoff, 2 * (m + q) + sub);
          if (BITS) {
            const uint32_t wd = __ldg(bits + o);
            xv[q].x = ((wd >> (2 * plane)) & 1u) ? VT(1) : VT(-1);
            xv[q].y = ((wd >> (2 * plane + 1)) & 1u) ? VT(1) : VT(-1);
          } else {
            xv[q] = __ldg(reinterpret_cast<const V2*>(u + o + pidx[0]));
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int kk = 2 * (m + q) + sub;
          const double sk = SK ? __shfl_sync(FULL, mys, kk) : 1.0;
          if (kk < cnt) {
            const double x0 = static_cast<double>(xv[q].x), x1 = static_cast<double>(xv[q].y);
            a0[0] = SK ? fma(sk, x0, a0[0]) : a0[0] + x0;
            a0[1] = SK ? fma(sk, x1, a0[1]) : a0[1] + x1;
          }
        }
      }
      for (; m < npairs; ++m) {
        const int kk = 2 * m + sub;
        const int64_t o = __shfl_sync(FULL, myoff, kk);
        const double sk = SK ? __shfl_sync(FULL, mys, kk) : 1.0;
        V2 xv;
        if (BITS) {
          const uint32_t wd = __ldg(bits + o);
          xv.x = ((wd >> (2 * plane)) & 1u) ? VT(1) : VT(-1);
          xv.y = ((wd >> (2 * plane + 1)) & 1u) ? VT(1) : VT(-1);
        } else {
          xv = __ldg(reinterpret_cast<const V2*>(u + o + pidx[0]));
        }
        if (kk < cnt) {
          const double x0 = static_cast<double>(xv.x), x1 = static_cast<double>(xv.y);
          a0[0] = SK ? fma(sk, x0, a0[0]) : a0[0] + x0;
          a0[1] = SK ? fma(sk, x1, a0[1]) : a0[1] + x1;
        }
      }
      continue;
    }
    if (HALF) {
      // pair m: this half takes position 2m + sub; U pairs in flight
      constexpr int U = 8;
      const int npairs = (cnt + 1) >> 1;
      int m = 0;
      for (; m + U <= npairs; m += U) {
        double xv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int64_t o = __shfl_sync(FULL, myoff, 2 * (m + q) + sub);
          xv[q] = value(u + o, bits + o, 0);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int kk = 2 * (m + q) + sub;
          const double sk = SK ? __shfl_sync(FULL, mys, kk) : 1.0;
          if (kk < cnt) a0[0] = SK ? fma(sk, xv[q], a0[0]) : a0[0] + xv[q];
        }
      }
      for (; m < npairs; ++m) {
        const int kk = 2 * m + sub;
        const int64_t o = __shfl_sync(FULL, myoff, kk);
        const double sk = SK ? __shfl_sync(FULL, mys, kk) : 1.0;
        const double x = value(u + o, bits + o, 0);
        if (kk < cnt) a0[0] = SK ? fma(sk, x, a0[0]) : a0[0] + x;
      }
      continue;
    }
    if constexpr (V2 && !HALF && !BITS && !EXACT && PPL >= 2) {
      // VEC2 (wide chunks): lane l holds probe pairs (64 j + 2 l, 64 j + 2 l + 1) and reads each pair
      // with one 2-element vector load (half the load instructions of the scalar mapping); every
      // probe is still one sequential chain, so results equal the scalar mapping bit for bit
      using P2 = typename std::conditional<std::is_same<VT, double>::value, double2, float2>::type;
      constexpr int NP = PPL / 2;
      constexpr int U2 = SLQ_SPMM_UNRF / PPL;
      int k = 0;
      for (; k + U2 <= cnt; k += U2) {
        P2 xv[U2][NP];
#pragma unroll
        for (int q = 0; q < U2; ++q) {
          const int64_t o = __shfl_sync(FULL, myoff, k + q);
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) xv[q][jj] = __ldg(reinterpret_cast<const P2*>(u + o + pidx[jj]));
        }
#pragma unroll
        for (int q = 0; q < U2; ++q) {
          const double sk = SK ? __shfl_sync(FULL, mys, k + q) : 1.0;
#pragma unroll
          for (int jj = 0; jj < NP; ++jj) {
            const double x0 = static_cast<double>(xv[q][jj].x), x1 = static_cast<double>(xv[q][jj].y);
            a0[2 * jj] = SK ? fma(sk, x0, a0[2 * jj]) : a0[2 * jj] + x0;
            a0[2 * jj + 1] = SK ? fma(sk, x1, a0[2 * jj + 1]) : a0[2 * jj + 1] + x1;
          }
        }
      }
      for (; k < cnt; ++k) {
        const int64_t o = __shfl_sync(FULL, myoff, k);
        const double sk = SK ? __shfl_sync(FULL, mys, k) : 1.0;
#pragma unroll
        for (int jj = 0; jj < NP; ++jj) {
          const P2 xv = __ldg(reinterpret_cast<const P2*>(u + o + pidx[jj]));
          const double x0 = static_cast<double>(xv.x), x1 = static_cast<double>(xv.y);
          a0[2 * jj] = SK ? fma(sk, x0, a0[2 * jj]) : a0[2 * jj] + x0;
          a0[2 * jj + 1] = SK ? fma(sk, x1, a0[2 * jj + 1]) : a0[2 * jj + 1] + x1;
        }
      }
      continue;
    }
    constexpr int UNR = SLQ_SPMM_UNRF / PPL;   // gathers in flight per lane (even: chain = q & 1)
    int k = 0;
    for (; k + UNR <= cnt; k += UNR) {
      double xv[UNR][PPL];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int64_t o = __shfl_sync(FULL, myoff, k + q);
        if (BITS) {
          // u_0 = +-1 from the probe bitmask: one uniform 16-byte load covers 128 probes
          const uint4 wv = __ldg(reinterpret_cast<const uint4*>(bits + o));
          const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
          for (int j = 0; j < PPL; ++j) xv[q][j] = ((wd[boff + j] >> lane) & 1u) ? 1.0 : -1.0;
        } else {
          const VT* src = u + o;
#pragma unroll
          for (int j = 0; j < PPL; ++j) xv[q][j] = ldg_f64(src + pidx[j]);
        }
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const double sk = SK ? __shfl_sync(FULL, mys, k + q) : 1.0;
        const double wk = (EXACT && WEIGHTED) ? __shfl_sync(FULL, myw, k + q) : 1.0;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
          if (EXACT) a0[j] = __dadd_rn(a0[j], gather_term<KIND, WEIGHTED>(xv[q][j], 1.0, sk, wk));
          else if (TWO && (q & 1)) a1[j] = SK ? fma(sk, xv[q][j], a1[j]) : a1[j] + xv[q][j];
          else a0[j] = SK ? fma(sk, xv[q][j], a0[j]) : a0[j] + xv[q][j];
        }
      }
    }
    for (; k < cnt; ++k) {
      const int64_t o = __shfl_sync(FULL, myoff, k);
      const double sk = SK ? __shfl_sync(FULL, mys, k) : 1.0;
      const double wk = (EXACT && WEIGHTED) ? __shfl_sync(FULL, myw, k) : 1.0;
      double xr[PPL];
      if (BITS) {
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(bits + o));
        const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int j = 0; j < PPL; ++j) xr[j] = ((wd[boff + j] >> lane) & 1u) ? 1.0 : -1.0;
      } else {
        const VT* src = u + o;
#pragma unroll
        for (int j = 0; j < PPL; ++j) xr[j] = ldg_f64(src + pidx[j]);
      }
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        if (EXACT) a0[j] = __dadd_rn(a0[j], gather_term<KIND, WEIGHTED>(xr[j], 1.0, sk, wk));
        else if (TWO && (k & 1)) a1[j] = SK ? fma(sk, xr[j], a1[j]) : a1[j] + xr[j];
        else a0[j] = SK ? fma(sk, xr[j], a0[j]) : a0[j] + xr[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < PPL; ++j) {
    if (EXACT) acc[j] = a0[j];
    else if (HALF) acc[j] = a0[j] + __shfl_xor_sync(FULL, a0[j], 16);   // s_even + s_odd in both halves
    else acc[j] = TWO ? a0[j] + a1[j] : a0[j];
  }
}

#ifndef SLQ_HALF2_PIPE
#define SLQ_HALF2_PIPE 0    // pipelined HALF2 gather: pairs in flight per half-warp (0: off; measured slower)
#endif
// HALF2 (fp32 chunks of 17..32 probes, 128-byte rows), software-pipelined: the column indices of the
// next 32 nonzeros are loaded before this batch's gathers are issued, and every pair of a batch is
// issued in one predicated round of U loads (no serial tail loop), so a row costs about one gather
// latency per 32 nonzeros instead of ~3.  Each half-warp still sums the positions of one parity of
// the row in ascending order, and the halves are combined at the end: bitwise the two-chain order
// of the narrow class (gather_range).
template <typename VT, int KIND, bool WEIGHTED, int U>
__device__ __forceinline__ void gather_half2_pipe(const int32_t* __restrict__ cols, const double* __restrict__ dinv,
                                                  const double* __restrict__ wts, const VT* __restrict__ u,
                                                  int64_t ldi, int pidx0, int64_t beg, int64_t end, double* acc) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr bool SK = KIND == SLQ_NORMALIZED_LAPLACIAN || WEIGHTED;
  using V2 = typename std::conditional<std::is_same<VT, double>::value, double2, float2>::type;
  const int lane = threadIdx.x & 31;
  const int sub = lane >> 4;
  double a0 = 0.0, a1 = 0.0;
  // 32-bit column indices travel through the shuffles (one shuffle per gather); offsets are formed
  // by the consumer lane
  auto load = [&](int64_t b, int32_t& col, double& sc) {
    col = 0;
    sc = 1.0;
    if (b + lane < end) {
      col = __ldg(cols + b + lane);
      if (KIND == SLQ_NORMALIZED_LAPLACIAN) sc = __ldg(dinv + col);
      if (WEIGHTED) sc *= __ldg(wts + b + lane);
    }
  };
  const VT* __restrict__ up = u + pidx0;
  int32_t mycol;
  double mys;
  load(beg, mycol, mys);
  for (int64_t base = beg; base < end; base += 32) {
    const int cnt = static_cast<int>(end - base < 32 ? end - base : 32);
    int32_t ncol = 0;
    double ns = 1.0;
    if (base + 32 < end) load(base + 32, ncol, ns);   // prefetch: independent of this batch's gathers
    const int npairs = (cnt + 1) >> 1;
    for (int m = 0; m < npairs; m += U) {
      V2 xv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int c = __shfl_sync(FULL, mycol, (2 * (m + q) + sub) & 31);
        if (m + q < npairs) xv[q] = __ldg(reinterpret_cast<const V2*>(up + static_cast<int64_t>(c) * ldi));
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int kk = 2 * (m + q) + sub;
        const double sk = SK ? __shfl_sync(FULL, mys, kk & 31) : 1.0;
        if (m + q < npairs && kk < cnt) {
          const double x0 = static_cast<double>(xv[q].x), x1 = static_cast<double>(xv[q].y);
          a0 = SK ? fma(sk, x0, a0) : a0 + x0;
          a1 = SK ? fma(sk, x1, a1) : a1 + x1;
        }
      }
    }
    mycol = ncol;
    mys = ns;
  }
  acc[0] = a0 + __shfl_xor_sync(FULL, a0, 16);   // s_even + s_odd in both halves
  acc[1] = a1 + __shfl_xor_sync(FULL, a1, 16);
}

// own-row value u[row][probe j of this lane] (from the bitmask on the first step).  u points at the
// lane's first probe; probe j of the lane is PS j further, and `probe` is its index within the
// 128-probe block (the bitmask word probe / 32, bit probe % 32).
template <typename VT, int PPL, bool BITS, int PS = 32>
__device__ __forceinline__ double own_value(const VT* u, int64_t ldi, const uint32_t* bits, int64_t row, int j,
                                            int probe) {
  if (BITS) {
    const uint32_t wd = __ldg(bits + row * kBitWords + (probe >> 5));
    return ((wd >> (probe & 31)) & 1u) ? 1.0 : -1.0;
  }
  return ldg_f64(u + row * ldi + PS * j);
}

// Pass A.  Warp-level work items taken from an atomic counter: first the long-row segments (partial
// sums to a.segpart), then the graph-fixed row tiles (one warp per tile: rows in order, alpha
// partial per tile).  Which warp runs an item never changes its arithmetic, so results are
// deterministic; dynamic scheduling removes the tail left by hub rows.  Long rows are finished by
// spmm_long_finish_kernel or the step kernel's phase 0.
#ifndef SLQ_SPMM_MINB4
#define SLQ_SPMM_MINB4 3   // resident CTAs per SM for PPL = 4 (80 registers: no spills in the 4-probe lanes)
#endif
#ifndef SLQ_SPMM_MINB_H2
#define SLQ_SPMM_MINB_H2 4   // resident CTAs per SM for the pipelined HALF2 mapping
#endif
#ifndef SLQ_SPMM_MINB1
#define SLQ_SPMM_MINB1 4   // resident CTAs per SM for PPL = 1 and 2
#endif
template <typename VT, int KIND, bool WEIGHTED, int PPL, bool BITS, bool EXACT, bool HALF, bool V2 = false>
__global__ void __launch_bounds__(kSpmmWarps * 32,
                                  PPL == 4 ? SLQ_SPMM_MINB4 : ((HALF && PPL == 2 && !BITS) ? SLQ_SPMM_MINB_H2 : SLQ_SPMM_MINB1))
spmm_kernel(SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  const int plane = HALF ? (lane & 15) : lane;   // HALF: two half-warps share probes 0..15 (0..31)
  const bool writer = !HALF || lane < 16;
  // probe j of this lane: pbase + poff(j).  HALF2 (HALF, PPL = 2): probes 2 plane, 2 plane + 1;
  // VEC2: probes 64 (j / 2) + 2 lane + (j % 2); otherwise plane + 32 j.
  constexpr int PS = HALF ? 1 : 32;
  auto poff = [](int j) { return V2 ? 64 * (j >> 1) + (j & 1) : PS * j; };
  const int pbase = blockIdx.y * kSpmmBlk + ((HALF || V2) ? (HALF ? PPL : 2) : 1) * plane;
  bool pv[PPL];
  int pidx[PPL];   // column offsets within a gathered row, clamped to a valid probe
#pragma unroll
  for (int j = 0; j < PPL; ++j) {
    pv[j] = probe_ok(pbase + poff(j), a.c);
    pidx[j] = pv[j] ? poff(j) : (a.c - 1 - (pbase - blockIdx.y * kSpmmBlk));
  }
  if (V2) {
    // pair jj: one vector load at offset 64 jj; a pair past the row's end reads the row's first pair
#pragma unroll
    for (int jj = 0; jj < PPL / 2; ++jj)
      pidx[jj] = blockIdx.y * kSpmmBlk + 64 * jj + 2 * plane + 1 < a.ldc_in ? 64 * jj : -2 * plane;
  }
  if (HALF && PPL == 2) {
    // one vector load per pair: a pair past the row's end (2 plane + 1 >= ldc) reads the row's first
    // pair instead (a valid address; those probes are never stored)
    pidx[0] = 2 * plane + 1 < a.ldc_in ? 0 : -2 * plane;
    pidx[1] = pidx[0] + 1;
  }
  const VT* __restrict__ u = static_cast<const VT*>(a.u) + pbase;
  // gathered rows: u, or the prescaled dinv (.) u (kNLPre); own-row values always from u
  const VT* __restrict__ ug = KIND == kNLPre ? static_cast<const VT*>(a.upre) + pbase : u;
  VT* __restrict__ w = static_cast<VT*>(a.w) + pbase;
  const int64_t* __restrict__ off = a.offsets;
  const double* __restrict__ dinv = a.dinv;
  const int64_t ldi = a.ldc_in;
  // gathered bitmask rows: the step-0 records when present (stride kRecWords), else the bitmask
  const uint32_t* gbits = (BITS && a.rec) ? a.rec : a.bits;
  const int64_t gld = BITS ? (a.rec ? kRecWords : kBitWords) : ldi;
  const double scale = KIND == SLQ_DENSITY ? a.dscal[3] : 0.0;
  const int64_t nseg = a.long_counts ? a.long_counts[1] : 0;
  unsigned long long* counter = a.work + blockIdx.y;   // [0..1] segments, [2..3] tiles (per probe block)

  // phase 1: long-row segments, one warp each (dynamic)
  for (;;) {
    long long item = 0;
    if (lane == 0) item = static_cast<long long>(atomicAdd(counter, 1ull));
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= nseg) break;
    const int64_t row = a.seg_row[item];
    const int64_t beg = a.seg_begin[item];
    const int64_t rend = off[row + 1];
    const int64_t end = beg + kSeg < rend ? beg + kSeg : rend;
    double acc[PPL];
#pragma unroll
    for (int j = 0; j < PPL; ++j) acc[j] = 0.0;
    gather_range<VT, KIND, WEIGHTED, PPL, BITS, EXACT, HALF, V2>(a.cols, dinv, a.weights, ug, gld, gbits, pidx, beg,
                                                                end, acc);
    double* dst = a.segpart + item * a.cpad + pbase;
#pragma unroll
    for (int j = 0; j < PPL; ++j)
      if (pv[j] && writer) dst[poff(j)] = acc[j];
  }
  // phase 2: row tiles, one warp each (dynamic); rows in order
  unsigned long long* tcounter = counter + 2;
  for (;;) {
    long long item = 0;
    if (lane == 0) item = static_cast<long long>(atomicAdd(tcounter, 1ull));
    const int tile = static_cast<int>(__shfl_sync(0xffffffffu, item, 0));
    if (tile >= a.ntiles) break;
    const int64_t rb = a.tile_rows[tile], re = a.tile_rows[tile + 1];
    for (int64_t row = rb; row < re; ++row) {
      const int64_t beg = off[row], end = off[row + 1];
      if (a.long_counts && end - beg > kLongRow) continue;   // finished from its segments
      double acc[PPL];
#pragma unroll
      for (int j = 0; j < PPL; ++j) acc[j] = 0.0;
      if constexpr (SLQ_HALF2_PIPE > 0 && HALF && PPL == 2 && !BITS && !EXACT) {
        gather_half2_pipe<VT, KIND == kNLPre ? SLQ_LAPLACIAN : KIND, WEIGHTED, SLQ_HALF2_PIPE>(
            a.cols, dinv, a.weights, ug, ldi, pidx[0], beg, end, acc);
      } else {
        gather_range<VT, KIND, WEIGHTED, PPL, BITS, EXACT, HALF, V2>(a.cols, dinv, a.weights, ug, gld, gbits, pidx, beg,
                                                                    end, acc);
      }
      const double d = __ldg(a.degree + row);
      const double dis = nl_kind<KIND>() ? __ldg(dinv + row) : 0.0;
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        if (!pv[j] || !writer) continue;
        const double rj = EXACT ? 1.0 : __ldg(a.r + pbase + poff(j));
        const double own = BITS ? own_value<VT, PPL, BITS, PS>(u, ldi, a.bits, row, j, pbase + poff(j))
                                : ldg_f64(u + row * ldi + poff(j));
        const double x = __dmul_rn(own, rj);
        const double y = op_epilogue<KIND>(x, EXACT ? acc[j] : acc[j] * rj, d, dis, scale);
        w[row * a.ldc_out + poff(j)] = from_f64<VT>(y);
      }
    }
  }
}

// Long rows: sum the segment partials in segment order, then the operator epilogue.
template <typename VT, int KIND, int PPL>
__global__ void __launch_bounds__(kSpmmWarps * 32)
spmm_long_finish_kernel(SpmmArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pbase = blockIdx.y * kSpmmBlk + lane;
  const int64_t nlong = a.long_counts[0];
  const VT* __restrict__ u = static_cast<const VT*>(a.u) + pbase;
  VT* __restrict__ w = static_cast<VT*>(a.w) + pbase;
  const double scale = KIND == SLQ_DENSITY ? a.dscal[3] : 0.0;
  for (int64_t lr = static_cast<int64_t>(blockIdx.x) * kSpmmWarps + warp; lr < a.max_long;
       lr += static_cast<int64_t>(gridDim.x) * kSpmmWarps) {
    if (lr < nlong) {
      const int64_t row = a.long_rows[lr];
      const int64_t s0 = a.long_seg_first[lr], s1 = a.long_seg_first[lr + 1];
      const double d = __ldg(a.degree + row);
      const double dis = KIND == SLQ_NORMALIZED_LAPLACIAN ? __ldg(a.dinv + row) : 0.0;
#pragma unroll
      for (int j = 0; j < PPL; ++j) {
        const int p = pbase + 32 * j;
        if (p >= a.c) continue;
        double acc = 0.0;
        for (int64_t sg = s0; sg < s1; ++sg) acc = __dadd_rn(acc, a.segpart[sg * a.cpad + p]);
        if (a.r) acc *= a.r[p];   // Lanczos path: segments hold unscaled sums
        const double rj = a.r ? a.r[p] : 1.0;
        const double own = a.bits ? (((a.bits[row * kBitWords + (p >> 5)] >> (p & 31)) & 1u) ? 1.0 : -1.0)
                                  : ldg_f64(u + row * a.ldc_in + 32 * j);
        const double x = __dmul_rn(own, rj);
        const double y = p < a.split ? op_epilogue<KIND>(x, acc, d, dis, a.dscal[3])
                                     : op_epilogue<SLQ_DENSITY>(x, acc, d, dis, a.dscal[3]);
        w[row * a.ldc_out + 32 * j] = from_f64<VT>(y);
      }
    }
  }
}

// VEC2 mapping for wide chunks (SLQ_SPMM_VEC2=0 keeps the scalar mapping; same arithmetic)
static bool vec2_on() {
  static const bool v = [] { const char* e = getenv("SLQ_SPMM_VEC2"); return !(e && e[0] == '0'); }();
  return v;
}

static int ppl_for(int c) {
  const int cb = c < kSpmmBlk ? c : kSpmmBlk;
  return cb <= 32 ? 1 : (cb <= 64 ? 2 : 4);
}

// Demote the window's persisting lines back to normal after the SpMM (a read of one word per 128-byte
// line, launched with a Normal-hitProp window over the same bytes), so the L2 carve-out does not
// shrink the cache of the CGS step kernel that follows.
static __global__ void l2_demote_kernel(const uint32_t* __restrict__ p, int64_t lines, uint32_t* sink) {
  uint32_t acc = 0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < lines; l += (int64_t)gridDim.x * blockDim.x)
    acc ^= __ldcg(p + l * 32);
  if (acc == 0x9e3779b9u) *sink = acc;   // never true in practice: keeps the loads
}

static void l2_demote(const void* base, size_t bytes, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  const int64_t lines = static_cast<int64_t>(bytes / 128);
  cfg.gridDim = dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(148 * 8, (lines + 255) / 256))));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  at[0].val.accessPolicyWindow.num_bytes = bytes;
  at[0].val.accessPolicyWindow.hitRatio = 1.0f;
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, l2_demote_kernel, static_cast<const uint32_t*>(base), lines, static_cast<uint32_t*>(nullptr));
}

// Launch one SpMM kernel; with a window, as cudaLaunchKernelEx carrying an access-policy window that
// marks the hub rows of the gathered vector (u, the prescaled dinv (.) u, or the probe bitmask)
// persisting in L2 and everything else streaming.
template <typename VT, int KIND, bool W, int PPL, bool BITS, bool EXACT, bool HALF, bool V2 = false>
static void spmm_go(const SpmmArgs& a, dim3 grid, cudaStream_t st) {
  if (a.win_rows <= 0 || EXACT) {
    spmm_kernel<VT, KIND, W, PPL, BITS, EXACT, HALF, V2><<<grid, kSpmmWarps * 32, 0, st>>>(a);
    return;
  }
  const void* base = BITS ? static_cast<const void*>(a.rec ? a.rec : a.bits) : (KIND == kNLPre ? a.upre : a.u);
  const size_t row_bytes = BITS ? sizeof(uint32_t) * (a.rec ? kRecWords : kBitWords)
                                : sizeof(VT) * static_cast<size_t>(a.ldc_in);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kSpmmWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeAccessPolicyWindow;
  at[0].val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  at[0].val.accessPolicyWindow.num_bytes = row_bytes * static_cast<size_t>(a.win_rows);
  at[0].val.accessPolicyWindow.hitRatio = 1.0f;
  at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, spmm_kernel<VT, KIND, W, PPL, BITS, EXACT, HALF, V2>, a);
  l2_demote(base, at[0].val.accessPolicyWindow.num_bytes, st);
}

template <typename VT, int KIND, bool W, int PPL>
static void spmm_launch_one(SpmmArgs& a, int gy, cudaStream_t st) {
  // persistent: work is taken from the atomic counters; small graphs launch only the warps they can use
  const int64_t items = static_cast<int64_t>(a.ntiles) + (a.long_counts ? a.max_seg : 0);
  dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(148 * 4, (items + kSpmmWarps - 1) / kSpmmWarps))),
            gy);
  // EXACT (bit-identical operator apply) only for the apply entry (r == nullptr, double);
  // HALF (two nonzeros per warp instruction) for Lanczos chunks of <= 16 probes.
  const bool half = PPL == 1 && a.c <= 16 && a.ldc_in <= 16;
  // HALF2 for 16 < c <= 32 (SLQ_SPMM_HALF2=0 keeps the full-warp mapping; same arithmetic)
  static const bool half2_on = [] { const char* e = getenv("SLQ_SPMM_HALF2"); return !(e && e[0] == '0'); }();
  const bool half2 = half2_on && std::is_same<VT, float>::value && PPL == 1 && !half && a.c <= 32 && a.ldc_in <= 32;
  if (!a.r) {
    if constexpr (std::is_same<VT, double>::value)
      spmm_go<VT, KIND, W, PPL, false, true, false>(a, grid, st);
  } else if (half2) {
    // fp32 rows only: fp64 pairs (16-byte loads) do not fit the register budget without spills
    if constexpr (std::is_same<VT, float>::value) {
      if (a.bits) spmm_go<VT, KIND, W, 2, true, false, true>(a, grid, st);
      else spmm_go<VT, KIND, W, 2, false, false, true>(a, grid, st);
    }
  } else if (half) {
    if (a.bits) spmm_go<VT, KIND, W, 1, true, false, true>(a, grid, st);
    else spmm_go<VT, KIND, W, 1, false, false, true>(a, grid, st);
  } else if (a.bits) {
    spmm_go<VT, KIND, W, PPL, true, false, false>(a, grid, st);
  } else if (PPL >= 2 && std::is_same<VT, double>::value && vec2_on()) {
    // fp64 rows only (measured: fp32 pairs are ~1.5% slower than the scalar mapping at C2 fp32)
    if constexpr (std::is_same<VT, double>::value)
      spmm_go<VT, KIND, W, PPL, false, false, false, true>(a, grid, st);
  } else {
    spmm_go<VT, KIND, W, PPL, false, false, false>(a, grid, st);
  }
}

template <typename VT, int KIND>
static void long_finish_dispatch(SpmmArgs& a, int gy, cudaStream_t st) {
  dim3 g2(static_cast<unsigned>(std::min<int64_t>((a.max_long + kSpmmWarps - 1) / kSpmmWarps, 148 * 8)), gy);
  switch (ppl_for(a.c)) {
    case 1: spmm_long_finish_kernel<VT, KIND, 1><<<g2, kSpmmWarps * 32, 0, st>>>(a); break;
    case 2: spmm_long_finish_kernel<VT, KIND, 2><<<g2, kSpmmWarps * 32, 0, st>>>(a); break;
    default: spmm_long_finish_kernel<VT, KIND, 4><<<g2, kSpmmWarps * 32, 0, st>>>(a); break;
  }
}

template <typename VT, int KIND, bool W>
static void spmm_dispatch(SpmmArgs& a, int gy, cudaStream_t st) {
  switch (ppl_for(a.c)) {
    case 1: spmm_launch_one<VT, KIND, W, 1>(a, gy, st); break;
    case 2: spmm_launch_one<VT, KIND, W, 2>(a, gy, st); break;
    default: spmm_launch_one<VT, KIND, W, 4>(a, gy, st); break;
  }
}

template <typename VT>
static void launch_spmm_main(int kind, SpmmArgs& a, int gy, cudaStream_t st) {
  LaunchScope ls(K_SPMM, st);
  const bool wt = a.weights != nullptr;
  if (kind == SLQ_NORMALIZED_LAPLACIAN && a.upre && !a.bits && a.r) {
    if (wt) spmm_dispatch<VT, kNLPre, true>(a, gy, st);
    else spmm_dispatch<VT, kNLPre, false>(a, gy, st);
  } else if (kind == SLQ_NORMALIZED_LAPLACIAN) {
    if (wt) spmm_dispatch<VT, SLQ_NORMALIZED_LAPLACIAN, true>(a, gy, st);
    else spmm_dispatch<VT, SLQ_NORMALIZED_LAPLACIAN, false>(a, gy, st);
  } else if (kind == SLQ_DENSITY) {
    if (wt) spmm_dispatch<VT, SLQ_DENSITY, true>(a, gy, st);
    else spmm_dispatch<VT, SLQ_DENSITY, false>(a, gy, st);
  } else {
    if (wt) spmm_dispatch<VT, SLQ_LAPLACIAN, true>(a, gy, st);
    else spmm_dispatch<VT, SLQ_LAPLACIAN, false>(a, gy, st);
  }
}

// The SpMM pass (short rows + long-row segments), then the long-row finish when the graph has any.
template <typename VT>
static void launch_spmm(int kind, SpmmArgs a, cudaStream_t st, bool finish = true) {
  const int gy = ceil_div(a.c, kSpmmBlk);
  bool flat = false;
  if constexpr (std::is_same<VT, float>::value) flat = launch_spmm_flat_f32(kind, a, st);
  else flat = launch_spmm_flat_f64(kind, a, st);
  if (!flat) launch_spmm_main<VT>(kind, a, gy, st);
  if (finish && a.long_counts && a.max_long > 0) {
    LaunchScope ls(K_SPMM, st);
    if (kind == SLQ_NORMALIZED_LAPLACIAN) long_finish_dispatch<VT, SLQ_NORMALIZED_LAPLACIAN>(a, gy, st);
    else if (kind == SLQ_DENSITY) long_finish_dispatch<VT, SLQ_DENSITY>(a, gy, st);
    else long_finish_dispatch<VT, SLQ_LAPLACIAN>(a, gy, st);
  }
}

// ----------------------------------------------------------------------------- pass B: CGS
struct CgsArgs {
  int64_t n, ldc, vec_stride;      // vec_stride = n*ldc elements between basis vectors
  int64_t rows_per_tile;
  int ntiles;
  int c, cpad;
  int i;                           // current Lanczos step
  int k0, nk;                      // basis block [k0, k0+nk) handled by this launch (dot kernel)
  int second;                      // 1: second CGS pass on u_{i+1}
  int reorth;
  const void* basis;               // u_0 .. u_S
  const void* w;                   // Op(q_i)
  ChunkState s;
  double* partial;                 // [ntiles][nq][cpad]
  // isolated-vertex fold: row virt_row stands for m isolated vertices; its u_0 is sqrt(m) (virt_root)
  // instead of a +-1 probe bit (-1: no such row)
  int64_t virt_row = -1;
  double virt_root = 0.0;
  // normalized Laplacian, prescaled gathers: the update also writes dinv (.) u_{i+1} into the (still
  // unused) slot i+2 for the next SpMM (nullptr: not this step)
  const double* pre_dinv = nullptr;
  void* pre_out = nullptr;         // where dinv (.) u_{i+1} goes (nullptr: the slot of u_{i+2}); the last
                                   // step kernel writes it over w, which the last SpMM no longer needs
  int pre_split = 1 << 30;         // operator-pair chunk: columns >= pre_split are copied unscaled
  unsigned long long* dbg = nullptr;   // SLQ_STEP_TIMING: %globaltimer of CTA 0 around each grid barrier
};

// w' = (w - alpha q_i) - beta_{i-1} q_{i-1}    (lanczos.py:129, numpy left-to-right evaluation)
__device__ __forceinline__ double three_term(double wv, double ui, double uim1, double al, double bp, double ri,
                                             double rim1) {
  const double qi = __dmul_rn(ui, ri);
  const double qp = __dmul_rn(uim1, rim1);
  return __dsub_rn(__dsub_rn(wv, __dmul_rn(al, qi)), __dmul_rn(bp, qp));
}

// Streaming CGS kernels use a flat layout: thread t of a CTA owns ONE probe column p = t % ldc and
// one of kRowSlots row slots, for a group of tiles; a warp reads 256 contiguous bytes per load and
// every per-probe scalar (alpha, beta, r, CGS coefficients) lives in registers.  The row slot of a
// row is its index mod kRowSlots, so per-probe sums never depend on the chunk width.
constexpr int kRowSlots = 2;
constexpr int kStreamThreads = 256;

struct FlatGeom {
  int ldc, G;    // tiles per CTA
};

static FlatGeom flat_geom(int64_t ldc) {
  FlatGeom f;
  f.ldc = static_cast<int>(ldc);
  f.G = std::max(1, static_cast<int>(kStreamThreads / (kRowSlots * ldc)));
  return f;
}

// Partials of sum_rows u_k . w' (CGS coefficient before the r_k scale, lanczos.py:73) for k in
// [k0, k0+nk) and of ||w'||^2 (lanczos.py:72).
template <typename VT>
__global__ void __launch_bounds__(512)
cgs_dot_kernel(CgsArgs a, int ldc_i, int G) {
  extern __shared__ double part[];   // [G][kRowSlots][nq][ldc]
  if (a.second && *a.s.any_again == 0) return;
  const int t = threadIdx.x;
  const int p = t % ldc_i;
  const int slot = (t / ldc_i) % kRowSlots;
  const int gt = t / (ldc_i * kRowSlots);
  const bool pv = p < a.c;
  const int cp = a.cpad;
  const int nq = a.nk + 1;
  const double al = pv ? a.s.alpha[a.i * cp + p] : 0.0;
  const double bp = (pv && a.i > 0) ? a.s.beta[(a.i - 1) * cp + p] : 0.0;
  const double ri = pv ? a.s.rsc[a.i * cp + p] : 0.0;
  const double rim1 = (pv && a.i > 0) ? a.s.rsc[(a.i - 1) * cp + p] : 0.0;
  const VT* basis = static_cast<const VT*>(a.basis) + p;
  const VT* w = static_cast<const VT*>(a.w) + p;
  const int64_t vs = a.vec_stride;
  const VT* ui = basis + static_cast<int64_t>(a.i) * vs;
  const VT* uim1 = basis + static_cast<int64_t>(a.i > 0 ? a.i - 1 : 0) * vs;
  const VT* unext = basis + static_cast<int64_t>(a.i + 1) * vs;
  const VT* uk0 = basis + static_cast<int64_t>(a.k0) * vs;

  for (int tb = blockIdx.x * G; tb < a.ntiles; tb += gridDim.x * G) {
    const int tile = tb + gt;
    double acc[kCgsBlock];
#pragma unroll
    for (int kk = 0; kk < kCgsBlock; ++kk) acc[kk] = 0.0;
    double nb = 0.0;
    if (pv && tile < a.ntiles) {
      const int64_t rb = static_cast<int64_t>(tile) * a.rows_per_tile;
      const int64_t re = min(a.n, rb + a.rows_per_tile);
      for (int64_t row = rb + slot; row < re; row += kRowSlots) {
        const int64_t idx = row * a.ldc;
        const double wp = a.second ? ldg_f64(unext + idx)
                                   : three_term(ldg_f64(w + idx), ldg_f64(ui + idx),
                                                a.i > 0 ? ldg_f64(uim1 + idx) : 0.0, al, bp, ri, rim1);
        nb = fma(wp, wp, nb);
#pragma unroll
        for (int kk = 0; kk < kCgsBlock; ++kk)
          if (kk < a.nk) acc[kk] = fma(ldg_f64(uk0 + kk * vs + idx), wp, acc[kk]);
      }
    }
    double* my = part + (static_cast<int64_t>(gt) * kRowSlots + slot) * nq * ldc_i + p;
#pragma unroll
    for (int kk = 0; kk < kCgsBlock; ++kk)
      if (kk < a.nk) my[kk * ldc_i] = acc[kk];
    my[a.nk * ldc_i] = nb;
    __syncthreads();
    // fixed-order combine of the row slots
    const int per_tile = nq * ldc_i;
    for (int e = t; e < G * per_tile; e += blockDim.x) {
      const int g2 = e / per_tile, rem = e - g2 * per_tile;
      const int q = rem / ldc_i, pp = rem - q * ldc_i;
      const int tl = tb + g2;
      if (tl >= a.ntiles || pp >= cp) continue;
      const double* src = part + static_cast<int64_t>(g2) * kRowSlots * per_tile + rem;
      double s = src[0];
#pragma unroll
      for (int rs = 1; rs < kRowSlots; ++rs) s += src[rs * per_tile];
      a.partial[(static_cast<int64_t>(tl) * nq + q) * cp + pp] = s;
    }
    __syncthreads();
  }
}

// u_{i+1} = w' - sum_k coef_k u_k (coef_k = h_k r_k, i.e. basis.T @ h with q_k = u_k r_k, lanczos.py:73);
// partials of ||u_{i+1}||^2.  Second pass: u_{i+1} -= sum_k coef2_k u_k for flagged probes only.
template <typename VT>
__global__ void __launch_bounds__(512)
cgs_update_kernel(CgsArgs a, int ldc_i, int G) {
  extern __shared__ double part[];   // [G][kRowSlots][ldc]
  if (a.second && *a.s.any_again == 0) return;
  const int t = threadIdx.x;
  const int p = t % ldc_i;
  const int slot = (t / ldc_i) % kRowSlots;
  const int gt = t / (ldc_i * kRowSlots);
  const int cp = a.cpad;
  const bool pv = p < a.c && (!a.second || a.s.again[p]);
  const int nk = a.reorth ? a.i + 1 : 0;
  double cf[kCgsBlock];
#pragma unroll
  for (int kk = 0; kk < kCgsBlock; ++kk) cf[kk] = (pv && kk < nk) ? a.s.h[kk * cp + p] * a.s.rsc[kk * cp + p] : 0.0;
  const double al = pv ? a.s.alpha[a.i * cp + p] : 0.0;
  const double bp = (pv && a.i > 0) ? a.s.beta[(a.i - 1) * cp + p] : 0.0;
  const double ri = pv ? a.s.rsc[a.i * cp + p] : 0.0;
  const double rim1 = (pv && a.i > 0) ? a.s.rsc[(a.i - 1) * cp + p] : 0.0;
  VT* basis = const_cast<VT*>(static_cast<const VT*>(a.basis)) + p;
  const VT* w = static_cast<const VT*>(a.w) + p;
  const int64_t vs = a.vec_stride;
  VT* out = basis + static_cast<int64_t>(a.i + 1) * vs;
  const VT* ui = basis + static_cast<int64_t>(a.i) * vs;
  const VT* uim1 = basis + static_cast<int64_t>(a.i > 0 ? a.i - 1 : 0) * vs;

  for (int tb = blockIdx.x * G; tb < a.ntiles; tb += gridDim.x * G) {
    const int tile = tb + gt;
    double nrm = 0.0;
    if (pv && tile < a.ntiles) {
      const int64_t rb = static_cast<int64_t>(tile) * a.rows_per_tile;
      const int64_t re = min(a.n, rb + a.rows_per_tile);
      for (int64_t row = rb + slot; row < re; row += kRowSlots) {
        const int64_t idx = row * a.ldc;
        const double wp = a.second ? ldg_f64(out + idx)
                                   : three_term(ldg_f64(w + idx), ldg_f64(ui + idx),
                                                a.i > 0 ? ldg_f64(uim1 + idx) : 0.0, al, bp, ri, rim1);
        double proj = 0.0;
#pragma unroll
        for (int kk = 0; kk < kCgsBlock; ++kk)
          if (kk < nk) proj = fma(ldg_f64(basis + kk * vs + idx), cf[kk], proj);
        for (int k = kCgsBlock; k < nk; ++k)   // s > 17 only
          proj = fma(ldg_f64(basis + k * vs + idx), a.s.h[k * cp + p] * a.s.rsc[k * cp + p], proj);
        const VT v = from_f64<VT>(nk ? __dsub_rn(wp, proj) : wp);
        out[idx] = v;
        const double vd = to_f64(v);
        nrm = fma(vd, vd, nrm);
      }
    }
    part[(gt * kRowSlots + slot) * ldc_i + p] = nrm;
    __syncthreads();
    for (int e = t; e < G * ldc_i; e += blockDim.x) {
      const int g2 = e / ldc_i, pp = e - g2 * ldc_i;
      const int tl = tb + g2;
      if (tl >= a.ntiles || pp >= cp) continue;
      double s = part[(g2 * kRowSlots) * ldc_i + pp];
#pragma unroll
      for (int rs = 1; rs < kRowSlots; ++rs) s += part[(g2 * kRowSlots + rs) * ldc_i + pp];
      a.partial[static_cast<int64_t>(tl) * cp + pp] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- staged (TMA bulk) CGS step kernel
// One persistent launch per Lanczos step does everything after the SpMM: kPersist CTAs, CTA b owns
// the contiguous rows [n*b/G, n*(b+1)/G).  Warp 0 lane 0 is the producer: it streams row chunks of
// every needed vector into a kStages-deep shared-memory ring with cp.async.bulk (completion on a
// "full" mbarrier).  Consumer thread p owns probe column p, walks its CTA's rows in ascending
// order from shared memory and releases each stage on an "empty" mbarrier (bytes in flight per SM
// = the whole ring, no register cost).
//
// CGS in Gram form.  With q_k = r_k u_k and G(k,j) = q_k . q_j (kept per probe), the reference's
// coefficient h_k = q_k . w' with w' = (w - alpha q_i) - beta q_{i-1} (lanczos.py:72-73,129) is
//     h_k = r_k (u_k . w) - alpha G(k,i) - beta G(k,i-1),   alpha = r_i (u_i . w),
// so one streaming phase (A) yields alpha and every h_k; the update phase (C) forms w' exactly as
// the reference, subtracts sum_k h_k q_k, and accumulates ||w'||^2, ||u_{i+1}||^2 and the Gram row
// u_k . u_{i+1} of the new vector.  The Gram row is also the second CGS pass's coefficients
// (lanczos.py:75-76), so that pass is a single update phase (C').  Phases are separated by a
// software grid barrier (all CTAs co-resident: one per SM).  Every per-probe sum runs in row order
// inside a fixed row range, reduced in fixed stripes: independent of c and of chunking.
//
// Consumer layout.  Three row slots (rows (row - lo) % 3) of T = round_up(M * ldc, 32) threads; in
// a slot, M threads share one probe column and part t of them handles basis vectors k = t, t + M,
// ... (step_parts picks M from ldc).  No per-(probe, k) sum depends on M.  The update's sum_k coef_k u_k runs as 8 chains (k mod 8) combined as
// ((c0 + c4) + (c2 + c6)) + ((c1 + c5) + (c3 + c7)) for every M (a butterfly over the M parts), so
// u_{i+1} is bitwise independent of M as well: narrow chunks keep the whole CTA busy without
// changing any result.
constexpr int kPersist = 148;
#ifndef SLQ_STEP_MIN_ROWS
#define SLQ_STEP_MIN_ROWS 64
#endif
constexpr int64_t kStepMinRows = SLQ_STEP_MIN_ROWS;   // small graphs use fewer step CTAs (cheaper grid barriers)

// CTAs of the step kernel for n rows: one per SM, or fewer for small graphs.  A function of n only,
// so every probe of a graph sees the same row partition.
inline int step_ctas(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kPersist, (n + kStepMinRows - 1) / kStepMinRows)));
}
constexpr int kStageSlots = 3;      // row slots of the wide class (ldc > 32)
constexpr int kNarrowSlots = 12;    // row slots of the narrow class (ldc <= 32)
constexpr int kSlotThreads = 128;                                 // max threads per row slot
constexpr int kStepThreads = 32 + kStageSlots * kSlotThreads;   // producer warp + <= 384 consumers
constexpr int kStagedMaxLdc = 128;
#ifndef SLQ_STEP_REVERSE
#define SLQ_STEP_REVERSE 1
#endif
// Streaming directions: phase A (dots) and the update phases run opposite ways, so each starts on
// what the previous pass left in L2.  SLQ_STEP_REVERSE=1: A forward, update backward; =2: A backward
// (the SpMM's tail of w), update forward.
constexpr bool kReverseUpdate = SLQ_STEP_REVERSE == 1;
constexpr bool kReverseDots = SLQ_STEP_REVERSE == 2;
constexpr int kStages = 3;
constexpr int kMaxStaged = kCgsBlock + 4;
constexpr size_t kStagedSmem = 200 * 1024;   // + 20 KB static: within the 227 KB per CTA

// Row slots and parts per probe column of the step kernel for a chunk of leading dimension ldc.
// Wide class (ldc > 32): 3 row slots, M = 1.  Narrow class (ldc <= 32): 12 row slots, M = 32 /
// round_up(ldc) so a slot is one full warp.  Per-probe sums depend on the class (the slot count)
// but not on M, so results are bitwise independent of the chunk width within a class.
struct StepGeom { int slots, parts; };
inline StepGeom step_geometry(int64_t ldc) {
  StepGeom g = ldc <= 32 ? StepGeom{kNarrowSlots, ldc <= 8 ? 4 : (ldc <= 16 ? 2 : 1)} : StepGeom{kStageSlots, 1};
  static const int forced = [] { const char* e = getenv("SLQ_STEP_M"); return e ? atoi(e) : 0; }();   // tuning
  const int cap = g.slots == kNarrowSlots ? 32 : kSlotThreads;
  if ((forced == 1 || forced == 2 || forced == 4 || forced == 8) && forced * ldc <= cap) g.parts = forced;
  return g;
}
inline int step_parts(int64_t ldc) { return step_geometry(ldc).parts; }

struct StagedArgs {
  CgsArgs a;
  int nvec;                       // VT vectors staged per chunk (source + u_1..u_{NK-1})
  const void* vec[kMaxStaged];    // global base of each staged vector
  const uint32_t* bits;           // u_0 as the probe bitmask [n][kBitWords], staged after the vectors
  int rt;                         // rows per chunk
  int vstride;                    // elements between vector slots in a stage (>= rt*ldc, bank-padded)
};

struct StepArgs {
  StagedArgs pass[2];             // [0]: src = w (phases A, C), [1]: src = u_{i+1} (phase C')
  ReduceArgs red;
  SpmmArgs spmm;                  // long rows of the preceding SpMM are finished in phase 0
};

template <typename VT>
struct StageRing {
  uint64_t* full;
  uint64_t* empty;
  VT* buf;
  __device__ explicit StageRing(unsigned char* smem) {
    full = reinterpret_cast<uint64_t*>(smem);
    empty = full + kStages;
    buf = reinterpret_cast<VT*>(smem + 128);
  }
};

// One ring stage: nvec VT row blocks [rt][ldc] at vstride spacing, then the bitmask rows
// [rt][kBitWords], then (prescaled gathers) a window of rt + 2 (even) dinv values starting at the even row
// at or below the chunk's first row (in VT units).
template <typename VT>
__host__ __device__ __forceinline__ int64_t stage_elems_of(int nvec, int rt, int vstride, bool dwin = false) {
  return static_cast<int64_t>(nvec) * vstride +
         (static_cast<int64_t>(rt) * kBitWords * 4 + (dwin ? 8 * ((static_cast<int64_t>(rt) + 3) & ~int64_t(1)) : 0) + sizeof(VT) - 1) /
             sizeof(VT);
}
template <typename VT>
__device__ __forceinline__ const double* stage_dinv(const VT* stage, int nvec, int rt, int vstride) {
  return reinterpret_cast<const double*>(reinterpret_cast<const unsigned char*>(stage + static_cast<int64_t>(nvec) * vstride) +
                                         static_cast<int64_t>(rt) * kBitWords * 4);
}

__device__ __forceinline__ int chunk_count(int64_t lo, int64_t hi, int rt) {
  return hi > lo ? static_cast<int>((hi - lo + rt - 1) / rt) : 0;
}

// Producer (one lane): chunk j of [lo, hi) goes to ring slot (ch0 + j) % kStages.
template <typename VT>
__device__ __forceinline__ void staged_produce(const StagedArgs& sa, StageRing<VT>& ring, int ch0, int64_t lo, int64_t hi,
                                               bool rev = false) {
  const int64_t ldc = sa.a.ldc;
  const bool dw = sa.a.pre_dinv != nullptr;
  const int64_t stage_elems = stage_elems_of<VT>(sa.nvec, sa.rt, sa.vstride, dw);
  int ch = ch0;
  const int nch = chunk_count(lo, hi, sa.rt);
  for (int jc = 0; jc < nch; ++jc, ++ch) {
    const int64_t r0 = lo + static_cast<int64_t>(rev ? nch - 1 - jc : jc) * sa.rt;
    const int s = ch % kStages;
    if (ch >= kStages) mbar_wait(&ring.empty[s], ((ch / kStages) - 1) & 1);
    const int rows = static_cast<int>(hi - r0 < sa.rt ? hi - r0 : sa.rt);
    const uint32_t bytes = static_cast<uint32_t>(rows * ldc * sizeof(VT));
    const uint32_t bbytes = static_cast<uint32_t>(rows * kBitWords * sizeof(uint32_t));
    // dinv window: even start (16-byte aligned source), even length (16-byte multiple)
    const int64_t d0 = r0 & ~int64_t(1);
    const uint32_t dbytes = dw ? static_cast<uint32_t>(((r0 - d0 + rows + 1) & ~int64_t(1)) * sizeof(double)) : 0u;
    mbar_arrive_expect_tx(&ring.full[s], bytes * sa.nvec + bbytes + dbytes);
    VT* dst = ring.buf + s * stage_elems;
    for (int v = 0; v < sa.nvec; ++v)
      bulk_g2s(dst + static_cast<int64_t>(v) * sa.vstride, static_cast<const VT*>(sa.vec[v]) + r0 * ldc, bytes,
               &ring.full[s]);
    bulk_g2s(dst + static_cast<int64_t>(sa.nvec) * sa.vstride, sa.bits + r0 * kBitWords, bbytes, &ring.full[s]);
    if (dw)
      bulk_g2s(const_cast<double*>(stage_dinv<VT>(dst, sa.nvec, sa.rt, sa.vstride)), sa.a.pre_dinv + d0, dbytes,
               &ring.full[s]);
  }
}

// Gram-matrix entry G(k, j) of probe p (G is symmetric; stored as [(S+1)*(S+1)][cpad]).
__device__ __forceinline__ double gram_at(const ChunkState& s, int k, int j, int p) {
  return s.G[(static_cast<int64_t>(k) * s.gstride + j) * s.cpad + p];
}

// Shared-memory stage layout: [slot][row][ldc] with slot 0 = source (w or u_{i+1}) and slot k = u_k
// for k >= 1, then the probe bitmask rows (u_0 = +-1).  NK = i + 1 basis vectors is a compile-time
// constant; each thread's basis indices k = q M + part are unrolled over q.

// Consumer coordinates of this thread (see the layout note above).
template <int M, int SL>
struct StepLane {
  int slot, p, part;
  __device__ __forceinline__ StepLane() {
    const int t = threadIdx.x - 32;
    const int per_slot = (blockDim.x - 32) / SL;
    slot = t / per_slot;
    const int e = t % per_slot;
    p = e / M;
    part = e % M;
  }
};

// Threads per row slot for M parts per probe column (a multiple of 32; M * ldc <= 128).
inline int step_slot_threads(int64_t ldc, int M) { return static_cast<int>(((M * ldc + 31) / 32) * 32); }

// Streaming arithmetic of the step kernel.  fp64 vectors: every per-row product and sum in fp64.
// fp32 vectors: per-row arithmetic in fp32 (no conversions in the row loop), and every running sum
// is a fp32 block over kFlush consecutive rows of the thread's row sequence added into a fp64 total
// (so a sum over n rows carries fp32 rounding of 8-term blocks only).  Blocks follow the row
// sequence of the slot, not the stage boundaries, so the order is still independent of rt and M.
template <typename VT>
struct StepArith {
  using T = double;
  static constexpr int kFlush = 0;
  static __device__ __forceinline__ T mul(T x, T y) { return __dmul_rn(x, y); }
  static __device__ __forceinline__ T sub(T x, T y) { return __dsub_rn(x, y); }
};
template <>
struct StepArith<float> {
  using T = float;
  static constexpr int kFlush = 8;
  static __device__ __forceinline__ T mul(T x, T y) { return __fmul_rn(x, y); }
  static __device__ __forceinline__ T sub(T x, T y) { return __fsub_rn(x, y); }
};

// u_k of row r in the arithmetic type (u_0 = +-1 from the bitmask row; sqrt(m) on the fold's
// trailing row, virt)
template <typename VT, typename T>
__device__ __forceinline__ T stage_u(const VT* e, const uint32_t* brow, int vstride, int p, int k, bool virt,
                                     T vroot) {
  if (k == 0) return virt ? vroot : (((brow[p >> 5] >> (p & 31)) & 1u) ? T(1) : T(-1));
  return static_cast<T>(e[k * vstride]);
}

// Per-CTA partials: the consumers' per-slot sums go to a shared-memory scratch [slot][nq][cp] (the
// idle stage ring), then are added over the slots in slot order and written as ONE partial row per
// CTA, [cta][nq][cp]: the grid-wide reductions read gridDim.x rows instead of gridDim.x * SL.
constexpr size_t kSlotScratchBytes = sizeof(double) * (kCgsBlock + 2) * (kStageSlots * kSlotThreads);
template <int SL>
__device__ __forceinline__ void cta_slot_reduce(const double* scratch, int nq, int cp, double* dst_cta) {
  named_barrier_sync(2, blockDim.x - 32);   // consumer warps only
  const int nt = blockDim.x - 32;
  for (int idx = threadIdx.x - 32; idx < nq * cp; idx += nt) {
    double v = scratch[idx];
#pragma unroll
    for (int sl = 1; sl < SL; ++sl) v += scratch[static_cast<int64_t>(sl) * nq * cp + idx];
    dst_cta[idx] = v;
  }
  // the scratch is the stage ring: order these generic accesses before later bulk copies into it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Phase A (consumer side): partials [cta*slots+slot][nq][cpad] of u_k . w (k < NK); at i == 0 also
// u_0 . u_0 (q = 1) for G(0,0).
template <typename VT, int NK, int M, int SL>
__device__ __forceinline__ void phase_dots(const StagedArgs& sa, StageRing<VT>& ring, int ch0, int64_t lo,
                                           int64_t hi, int nq) {
  using A = StepArith<VT>;
  using T = typename A::T;
  constexpr int NQ = (NK + M - 1) / M;
  const CgsArgs& a = sa.a;
  const StepLane<M, SL> L;
  const int lane = threadIdx.x & 31;
  const bool pv = L.p < a.c;
  const int cp = a.cpad, ldc = static_cast<int>(a.ldc);
  const int rt = sa.rt, vstride = sa.vstride;
  const int64_t stage_elems = stage_elems_of<VT>(sa.nvec, rt, vstride, a.pre_dinv != nullptr);
  double acc[NQ];
  T blk[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0, blk[q] = T(0);
  int nrow = 0;
  double g00 = 0.0;
  auto flush = [&]() {
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] += static_cast<double>(blk[q]), blk[q] = T(0);
    nrow = 0;
  };
  const T vroot = static_cast<T>(a.virt_root);
  auto row_dots = [&](T wv, const T* uv) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q * M + L.part < NK) blk[q] = fma(uv[q], wv, blk[q]);
    // u_0 . u_0: 1 per +-1 row (exact), m for the fold's trailing row
    if (NK == 1 && L.part == 0) g00 += static_cast<double>(uv[0]) * static_cast<double>(uv[0]);
    if (A::kFlush && ++nrow == A::kFlush) flush();
  };
  auto load_row = [&](const VT* stage, const uint32_t* sbits, int rr, int64_t grow, T& wv, T* uv) {
    const VT* e = stage + L.p + rr * ldc;
    const uint32_t* brow = sbits + rr * kBitWords;
    const bool virt = grow == a.virt_row;
    wv = static_cast<T>(e[0]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = q * M + L.part;
      uv[q] = kk < NK ? stage_u<VT, T>(e, brow, vstride, L.p, kk, virt, vroot) : T(0);
    }
  };
  int ch = ch0;
  // kReverseDots: chunks backwards and rows backwards within them (the SpMM just wrote the tail of w,
  // still in L2); every slot's row sequence is then the exact reverse of the ascending one
  const int nch = chunk_count(lo, hi, rt);
  for (int jc = 0; jc < nch; ++jc, ++ch) {
    const int64_t r0 = lo + static_cast<int64_t>(kReverseDots ? nch - 1 - jc : jc) * rt;
    const int s = ch % kStages;
    mbar_wait(&ring.full[s], (ch / kStages) & 1);
    const int rows = static_cast<int>(hi - r0 < rt ? hi - r0 : rt);
    if (pv) {
      const VT* stage = ring.buf + s * stage_elems;
      const uint32_t* sbits = reinterpret_cast<const uint32_t*>(stage + static_cast<int64_t>(sa.nvec) * vstride);
      // this thread's rows: (row - lo) % SL == slot; U rows per iteration (all shared-memory loads
      // first, then the arithmetic in row order)
      constexpr int U = NQ <= 2 ? 4 : (NQ <= 4 ? 2 : 1);
      constexpr int D = kReverseDots ? -SL : SL;
      const int first = static_cast<int>(((L.slot - (r0 - lo)) % SL + SL) % SL);
      const int last = first < rows ? first + SL * ((rows - 1 - first) / SL) : first - SL;
      const int cnt = first < rows ? (last - first) / SL + 1 : 0;
      int r = kReverseDots ? last : first;
      int k = 0;
      for (; k + U <= cnt; k += U, r += D * U) {
        T wv[U], uv[U][NQ];
#pragma unroll
        for (int j = 0; j < U; ++j) load_row(stage, sbits, r + D * j, r0 + r + D * j, wv[j], uv[j]);
#pragma unroll
        for (int j = 0; j < U; ++j) row_dots(wv[j], uv[j]);
      }
      for (; k < cnt; ++k, r += D) {
        T wv1, uv1[NQ];
        load_row(stage, sbits, r, r0 + r, wv1, uv1);
        row_dots(wv1, uv1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[s]);
  }
  flush();
  named_barrier_sync(2, blockDim.x - 32);   // every consumer warp is done reading the ring
  double* scratch = reinterpret_cast<double*>(ring.buf);
  if (L.p < cp) {
    double* dst = scratch + static_cast<int64_t>(L.slot) * nq * cp + L.p;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = q * M + L.part;
      if (kk < NK) dst[kk * cp] = acc[q];
    }
    if (NK == 1 && L.part == 0) dst[NK * cp] = g00;
  }
  cta_slot_reduce<SL>(scratch, nq, cp, a.partial + static_cast<int64_t>(blockIdx.x) * nq * cp);
}

// sum_k coef_k u_k from this thread's chains ch[j] (chain j M + part), combined in the canonical
// order ((c0 + c4) + (c2 + c6)) + ((c1 + c5) + (c3 + c7)) over the M parts of the probe column.
template <int M, typename T>
__device__ __forceinline__ T chain_total(const T* ch) {
  constexpr unsigned FULL = 0xffffffffu;
  if (M == 1) return ((ch[0] + ch[4]) + (ch[2] + ch[6])) + ((ch[1] + ch[5]) + (ch[3] + ch[7]));
  if (M == 2) {
    const T s = (ch[0] + ch[2]) + (ch[1] + ch[3]);   // (c_t + c_t+4) + (c_t+2 + c_t+6)
    return s + __shfl_xor_sync(FULL, s, 1);
  }
  if (M == 4) {
    T s = ch[0] + ch[1];                             // c_t + c_t+4
    s = s + __shfl_xor_sync(FULL, s, 2);
    return s + __shfl_xor_sync(FULL, s, 1);
  }
  T s = ch[0] + __shfl_xor_sync(FULL, ch[0], 4);
  s = s + __shfl_xor_sync(FULL, s, 2);
  return s + __shfl_xor_sync(FULL, s, 1);
}

// Phase C / C' (consumer side).  First pass: w' = three-term, u_{i+1} = w' - sum_k coef_k u_k.
// Second pass (flagged probes): u_{i+1} -= sum_k coef_k u_k.  Partials [cta*slots+slot][nq][cpad]:
// q=0 ||w'||^2, q=1 ||u_{i+1}||^2, q=2+k  u_k . u_{i+1}.  Every lane runs the row loop (the chain
// butterfly shuffles across the parts); lanes past the chunk read a valid column and store nothing.
template <typename VT, int NK, bool SECOND, int M, int SL>
__device__ __forceinline__ void phase_update(const StagedArgs& sa, StageRing<VT>& ring, int ch0, int64_t lo,
                                             int64_t hi, double* cf_sm) {
  using A = StepArith<VT>;
  using T = typename A::T;
  constexpr int NQ = (NK + M - 1) / M;
  constexpr int NC = 8 / M;
  const CgsArgs& a = sa.a;
  const ChunkState& S = a.s;
  const StepLane<M, SL> L;
  const int lane = threadIdx.x & 31;
  const int p = L.p;
  const int cp = a.cpad, ldc = static_cast<int>(a.ldc);
  const int pr = p < ldc ? p : ldc - 1;
  const bool pv = p < a.c && (!SECOND || S.again[p]);
  constexpr int nq = NK + 2;
  constexpr int i = NK - 1;
  double al = 0.0, bp = 0.0, ri = 0.0, rim1 = 0.0;
  if (pv) {
    ri = S.rsc[i * cp + p];
    rim1 = i > 0 ? S.rsc[(i - 1) * cp + p] : 0.0;
    bp = i > 0 ? S.beta[(i - 1) * cp + p] : 0.0;
    al = __dmul_rn(ri, S.cdot[i * cp + p]);
  }
  // CGS coefficients coef_k = h_k r_k into shared memory [NK][kSlotThreads] (slot 0 computes)
  if (L.slot == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = q * M + L.part;
      if (kk >= NK) continue;
      double c = 0.0;
      if (pv) {
        const double rk = S.rsc[kk * cp + p];
        double h;
        // explicit roundings: no FMA contraction, so every template instance (NK, M) computes the
        // same coefficient bits
        if (SECOND) {
          h = __dmul_rn(rk, S.gram[kk * cp + p]);                                  // q_k . w''
        } else {
          h = __dsub_rn(__dmul_rn(rk, S.cdot[kk * cp + p]), __dmul_rn(al, gram_at(S, kk, i, p)));
          if (i > 0) h = __dsub_rn(h, __dmul_rn(bp, gram_at(S, kk, i - 1, p)));
        }
        c = __dmul_rn(h, rk);
      }
      cf_sm[kk * kSlotThreads + p] = c;
    }
  }
  named_barrier_sync(1, blockDim.x - 32);   // consumers only
  T cf[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int kk = q * M + L.part;
    cf[q] = static_cast<T>(kk < NK ? cf_sm[kk * kSlotThreads + p] : 0.0);
  }
  const T al_t = static_cast<T>(al), bp_t = static_cast<T>(bp), ri_t = static_cast<T>(ri);
  const T rim1_t = static_cast<T>(rim1);
  const T vroot = static_cast<T>(a.virt_root);
  const int rt = sa.rt, vstride = sa.vstride;
  const int64_t stage_elems = stage_elems_of<VT>(sa.nvec, rt, vstride, a.pre_dinv != nullptr);
  VT* out = const_cast<VT*>(static_cast<const VT*>(a.basis)) + static_cast<int64_t>(NK) * a.vec_stride + p;
  // dinv (.) u_{i+1}: slot i+2, or (last step kernel) the rows of w this CTA has already consumed
  VT* out_pre = a.pre_dinv ? (a.pre_out ? static_cast<VT*>(a.pre_out) + p : out + a.vec_stride) : nullptr;
  double nb = 0.0, nrm = 0.0, gr[NQ];
  T bnb = T(0), bnrm = T(0), bgr[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) gr[q] = 0.0, bgr[q] = T(0);
  int nrow = 0;
  auto flush = [&]() {
    nb += static_cast<double>(bnb);
    nrm += static_cast<double>(bnrm);
    bnb = T(0);
    bnrm = T(0);
#pragma unroll
    for (int q = 0; q < NQ; ++q) gr[q] += static_cast<double>(bgr[q]), bgr[q] = T(0);
    nrow = 0;
  };
  // one row: w' (or the source), u_{i+1} = w' - sum_k coef_k u_k, and its sums (in row order)
  auto row_update = [&](T src, T ui, T uim1, const T* uk, int64_t grow, double dv) {
    T wp;
    if (SECOND) {
      wp = src;
    } else {
      // w' = (w - alpha q_i) - beta q_{i-1}, q = u r  (lanczos.py:72-73)
      wp = A::sub(A::sub(src, A::mul(al_t, A::mul(ui, ri_t))), A::mul(bp_t, A::mul(uim1, rim1_t)));
      bnb = fma(wp, wp, bnb);
    }
    T chn[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) chn[j] = T(0);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q * M + L.part < NK) chn[q % NC] = fma(uk[q], cf[q], chn[q % NC]);
    const VT vv = static_cast<VT>(A::sub(wp, chain_total<M, T>(chn)));
    if (pv && L.part == 0) {
      out[grow * a.ldc] = vv;
      if (out_pre) out_pre[grow * a.ldc] = static_cast<VT>(__dmul_rn(dv, static_cast<double>(vv)));
    }
    const T vd = static_cast<T>(vv);
    bnrm = fma(vd, vd, bnrm);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q * M + L.part < NK) bgr[q] = fma(uk[q], vd, bgr[q]);
    if (A::kFlush && ++nrow == A::kFlush) flush();
  };
  int ch = ch0;
  // chunks in REVERSE order: the first chunks of the update are the last ones phase A streamed, still
  // in L2 (rows keep their slots, so only the order of the per-slot partial sums changes)
  const int nch = chunk_count(lo, hi, rt);
  for (int jc = 0; jc < nch; ++jc, ++ch) {
    const int64_t r0 = lo + static_cast<int64_t>(kReverseUpdate ? nch - 1 - jc : jc) * rt;
    const int s = ch % kStages;
    mbar_wait(&ring.full[s], (ch / kStages) & 1);
    const int rows = static_cast<int>(hi - r0 < rt ? hi - r0 : rt);
    const VT* stage = ring.buf + s * stage_elems;
    const uint32_t* sbits = reinterpret_cast<const uint32_t*>(stage + static_cast<int64_t>(sa.nvec) * vstride);
    const double* sdinv = stage_dinv<VT>(stage, sa.nvec, rt, vstride);
    auto load_row = [&](int rr, T& src, T& ui, T& uim1, T* uk, double& dv) {
      const VT* e = stage + pr + rr * ldc;
      dv = out_pre ? (p < a.pre_split ? sdinv[(r0 & 1) + rr] : 1.0) : 0.0;   // staged dinv window
      const uint32_t* brow = sbits + rr * kBitWords;
      const bool virt = r0 + rr == a.virt_row;
      src = static_cast<T>(e[0]);
      if (!SECOND) {
        ui = stage_u<VT, T>(e, brow, vstride, pr, i, virt, vroot);
        uim1 = i > 0 ? stage_u<VT, T>(e, brow, vstride, pr, i > 0 ? i - 1 : 0, virt, vroot) : T(0);
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int kk = q * M + L.part;
        uk[q] = kk < NK ? stage_u<VT, T>(e, brow, vstride, pr, kk, virt, vroot) : T(0);
      }
    };
    // this slot's rows of the chunk; with kReverseUpdate they run in DESCENDING order (chunks
    // backwards and rows backwards within them), so every slot's row sequence is the reverse of its
    // ascending one whatever the chunk size rt (results stay independent of the chunk width)
    constexpr int U = NQ <= 2 ? 4 : (NQ <= 5 ? 2 : 1);
    constexpr int D = kReverseUpdate ? -SL : SL;   // row step
    const int first = static_cast<int>(((L.slot - (r0 - lo)) % SL + SL) % SL);
    const int last = first < rows ? first + SL * ((rows - 1 - first) / SL) : first - SL;
    const int cnt = first < rows ? (last - first) / SL + 1 : 0;
    int r = kReverseUpdate ? last : first;
    int k = 0;
    for (; k + U <= cnt; k += U, r += D * U) {
      T src[U], ui[U], uim1[U], uk[U][NQ];
      double dv[U];
#pragma unroll
      for (int j = 0; j < U; ++j) load_row(r + D * j, src[j], ui[j], uim1[j], uk[j], dv[j]);
#pragma unroll
      for (int j = 0; j < U; ++j) row_update(src[j], ui[j], uim1[j], uk[j], r0 + r + D * j, dv[j]);
    }
    for (; k < cnt; ++k, r += D) {
      T src1, ui1 = T(0), uim11 = T(0), uk1[NQ];
      double dv1;
      load_row(r, src1, ui1, uim11, uk1, dv1);
      row_update(src1, ui1, uim11, uk1, r0 + r, dv1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[s]);
  }
  flush();
  named_barrier_sync(2, blockDim.x - 32);   // every consumer warp is done reading the ring
  double* scratch = reinterpret_cast<double*>(ring.buf);
  if (p < cp) {
    double* dst = scratch + static_cast<int64_t>(L.slot) * nq * cp + p;
    if (L.part == 0) {
      dst[0] = pv ? nb : 0.0;
      dst[cp] = pv ? nrm : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int kk = q * M + L.part;
      if (kk < NK) dst[(2 + kk) * cp] = pv ? gr[q] : 0.0;
    }
  }
  cta_slot_reduce<SL>(scratch, nq, cp, a.partial + static_cast<int64_t>(blockIdx.x) * nq * cp);
}

// Fixed-order stripe reduction of quantity q for 32 probes; returns the total in warp 0's lanes.
static __device__ double stripe_sum(const double* partial, int ntiles, int nq, int cpad, int q, int group, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int p = group * 32 + lane;
  const int64_t stride = static_cast<int64_t>(nq) * cpad;
  const double* src = partial + static_cast<int64_t>(q) * cpad + p;
  for (int sidx = warp; sidx < kStripes; sidx += nw) {
    // 8 loads in flight, then the adds in the same sequential order (bitwise the plain loop)
    double s = 0.0;
    int t = sidx;
    for (; t + 7 * kStripes < ntiles; t += 8 * kStripes) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = src[static_cast<int64_t>(t + j * kStripes) * stride];
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; t < ntiles; t += kStripes) s += src[static_cast<int64_t>(t) * stride];
    red[sidx * 32 + lane] = s;
  }
  __syncthreads();
  double tot = 0.0;
  if (warp == 0) {
    tot = red[lane];
    for (int j = 1; j < kStripes; ++j) tot += red[j * 32 + lane];
  }
  __syncthreads();
  return tot;
}

// Phases C (or C'), D, E of one CGS pass (SECOND: the conditional second pass, lanczos.py:75-76).
template <typename VT, int NK, bool SECOND, int M, int SL, typename Sync>
__device__ __forceinline__ void update_pass(const StepArgs& sa, const StagedArgs& st, StageRing<VT>& ring, int& ch,
                                            int64_t lo, int64_t hi, int nrows_partial, double* cf_sm,
                                            double* red, Sync& sync_grid) {
  const CgsArgs& a = sa.pass[0].a;
  const ChunkState& S = a.s;
  const int ngroups = a.cpad / 32, cp = a.cpad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nk = a.i + 1, nq = nk + 2, nslot = S.gstride;
  // C / C': update
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) staged_produce<VT>(st, ring, ch, lo, hi, kReverseUpdate);
  } else {
    phase_update<VT, NK, SECOND, M, SL>(st, ring, ch, lo, hi, cf_sm);
  }
  ch += chunk_count(lo, hi, st.rt);
  asm volatile("fence.proxy.async.global;" ::: "memory");   // u_{i+1} is bulk-read by a second pass
  sync_grid();
  // D: reduce ||w'||^2, ||u_{i+1}||^2 and the Gram row
  for (int sl = blockIdx.x; sl < nq * ngroups; sl += gridDim.x) {
    const int q = sl % nq, gidx = sl / nq, p = gidx * 32 + lane;
    const double tot = stripe_sum(a.partial, nrows_partial, nq, cp, q, gidx, red);
    if (warp == 0 && p < a.c) {
      if (q == 0) { if (!SECOND) S.nb2[p] = tot; }
      else if (q == 1) S.nrm2[p] = tot;
      else S.gram[(q - 2) * cp + p] = tot;
    }
  }
  sync_grid();
  // E: beta, breakdown, second-pass flag, Gram column of q_{i+1} (lanczos.py:75,132-137)
  for (int gidx = blockIdx.x; gidx < ngroups; gidx += gridDim.x) {
    const int p = gidx * 32 + lane;
    if (warp != 0 || p >= a.c || !S.alive[p]) continue;
    if (SECOND && !S.again[p]) continue;
    const double b = sqrt(S.nrm2[p]);
    if (!SECOND && b < 0.5 * sqrt(S.nb2[p])) {
      S.again[p] = 1;
      *S.any_again = 1;
      if (S.second_passes) atomicAdd(S.second_passes, 1);
      continue;
    }
    if (SECOND) S.again[p] = 0;
    const int kd = kind_of_column(sa.red, p);
    const double hi_int = kd == SLQ_NORMALIZED_LAPLACIAN ? 2.0 : (kd == SLQ_DENSITY ? 1.0 : sa.red.dscal[4]);   // interval_hi
    if (b <= 1e-12 * hi_int) {
      S.steps[p] = a.i + 1;
      S.alive[p] = 0;
      S.rsc[(a.i + 1) * cp + p] = 0.0;
    } else {
      const double rn = __ddiv_rn(1.0, b);
      S.beta[a.i * cp + p] = b;
      S.rsc[(a.i + 1) * cp + p] = rn;
      const int j = a.i + 1;   // == NK
      // all loads first (the stores below could alias them for the compiler), then the stores
      double rk[NK], gk[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) { rk[k] = S.rsc[k * cp + p]; gk[k] = S.gram[k * cp + p]; }
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const double gkj = rk[k] * rn * gk[k];
        S.G[(static_cast<int64_t>(k) * nslot + j) * cp + p] = gkj;
        S.G[(static_cast<int64_t>(j) * nslot + k) * cp + p] = gkj;
      }
      S.G[(static_cast<int64_t>(j) * nslot + j) * cp + p] = rn * rn * S.nrm2[p];
    }
  }
  sync_grid();
}

template <typename VT, int NK, int M, int SL>
__global__ void __launch_bounds__(kStepThreads, 1)
cgs_step_kernel(StepArgs sa) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double red[kStripes * 32];
  __shared__ double cf_sm[kCgsBlock * kSlotThreads];
  StageRing<VT> ring(smem);
  const CgsArgs& a = sa.pass[0].a;
  const ChunkState& S = a.s;
  unsigned int* bar = S.barrier + a.i;
  unsigned int nbar = 0;
  auto stamp = [&](int k) {
    if (a.dbg && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (blockIdx.x == 0 && k < 32) a.dbg[k] = t;
      // every CTA: start and the entries of barriers 1 and 3 (ends of the two streaming phases)
      if (k == 0 || k == 1 || k == 5) a.dbg[32 + 4 * blockIdx.x + (k == 0 ? 0 : (k == 1 ? 1 : 2))] = t;
    }
  };
  stamp(0);
  auto sync_grid = [&]() {
    if (a.dbg) __syncthreads();   // diagnostics: stamp when the whole CTA has arrived
    stamp(2 * nbar + 1);   // entry of barrier nbar+1
    grid_barrier(bar, ++nbar);
    stamp(2 * nbar);       // exit
  };
  const int nwc = (blockDim.x - 32) / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&ring.full[s], 1); mbar_init(&ring.empty[s], nwc); }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t lo = a.n * blockIdx.x / gridDim.x, hi = a.n * (blockIdx.x + 1) / gridDim.x;
  const int ngroups = a.cpad / 32, cp = a.cpad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nk = a.i + 1;
  const int nrows_partial = gridDim.x;   // one pre-reduced partial row per CTA
  int ch = 0;
  const StagedArgs& st0 = sa.pass[0];
  const int nch0 = chunk_count(lo, hi, st0.rt);

  // 0: finish the SpMM's long rows (segment partials in order + epilogue); skipped when none
  const SpmmArgs& sp = sa.spmm;
  const int64_t nlong = sp.long_counts ? sp.long_counts[0] : 0;
  if (nlong > 0) {
    const int nw = blockDim.x >> 5;
    const VT* uu = static_cast<const VT*>(sp.u);
    VT* ww = static_cast<VT*>(sp.w);
    const double scale = sp.dscal[3];
    for (int64_t lr = static_cast<int64_t>(blockIdx.x) * nw + warp; lr < nlong;
         lr += static_cast<int64_t>(gridDim.x) * nw) {
      const int64_t row = sp.long_rows[lr];
      const int64_t s0 = sp.long_seg_first[lr], s1 = sp.long_seg_first[lr + 1];
      const double d = sp.degree[row], dis = sp.dinv[row];
      for (int p = lane; p < sp.c; p += 32) {
        double acc = 0.0;
        for (int64_t sg = s0; sg < s1; ++sg) acc = __dadd_rn(acc, sp.segpart[sg * sp.cpad + p]);
        acc *= sp.r[p];   // segments hold unscaled sums
        const double own = sp.bits ? (((sp.bits[row * kBitWords + (p >> 5)] >> (p & 31)) & 1u) ? 1.0 : -1.0)
                                   : to_f64(uu[row * sp.ldc_in + p]);
        const double x = __dmul_rn(own, sp.r[p]);
        double y;
        const int kd = kind_of_column(sa.red, p);
        if (kd == SLQ_NORMALIZED_LAPLACIAN) y = op_epilogue<SLQ_NORMALIZED_LAPLACIAN>(x, acc, d, dis, scale);
        else if (kd == SLQ_DENSITY) y = op_epilogue<SLQ_DENSITY>(x, acc, d, dis, scale);
        else y = op_epilogue<SLQ_LAPLACIAN>(x, acc, d, dis, scale);
        ww[row * sp.ldc_out + p] = from_f64<VT>(y);
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");   // w is bulk-read in phase A
    sync_grid();
  }
  // A: u_k . w for k <= i (and u_0 . u_0 at i == 0)
  const int nqa = nk + (a.i == 0 ? 1 : 0);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) staged_produce<VT>(st0, ring, ch, lo, hi, kReverseDots);
  } else {
    phase_dots<VT, NK, M, SL>(st0, ring, ch, lo, hi, nqa);
  }
  ch += nch0;
  sync_grid();
  // B: reduce them (fixed stripes); G(0,0) at the first step
  for (int sl = blockIdx.x; sl < nqa * ngroups; sl += gridDim.x) {
    const int q = sl % nqa, gidx = sl / nqa, p = gidx * 32 + lane;
    const double tot = stripe_sum(a.partial, nrows_partial, nqa, cp, q, gidx, red);
    if (warp == 0 && p < a.c) {
      if (q < nk) {
        S.cdot[q * cp + p] = tot;
        if (q == a.i && S.alive[p]) S.alpha[a.i * cp + p] = S.rsc[a.i * cp + p] * tot;   // alpha = q_i . w
      } else {
        const double r0 = S.rsc[p];
        S.G[p] = r0 * r0 * tot;                                                       // G(0,0)
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *S.any_again = 0;
  sync_grid();
  update_pass<VT, NK, false, M, SL>(sa, sa.pass[0], ring, ch, lo, hi, nrows_partial, cf_sm, red, sync_grid);
  if (*S.any_again) {   // uniform: read after a grid barrier
#ifdef SLQ_DEBUG_SECOND
    if (blockIdx.x == 0 && threadIdx.x == 0) printf("second pass at step %d\n", a.i);
#endif
    update_pass<VT, NK, true, M, SL>(sa, sa.pass[1], ring, ch, lo, hi, nrows_partial, cf_sm, red, sync_grid);
  }
}

// Build the staged-vector list of one pass; false when the geometry does not fit.  Vector slots
// of a stage are vstride elements apart, vstride = W / M (mod W) with W = 128 B / sizeof(VT), so the
// M parts of a probe column (reading M different slots of one row) hit distinct banks.
template <typename VT>
static bool staged_setup(const CgsArgs& a, bool second, const uint32_t* bits, StagedArgs* out) {
  StagedArgs s{};
  s.a = a;
  const VT* basis = static_cast<const VT*>(a.basis);
  const int nk = a.i + 1;
  if (!a.reorth || nk > kCgsBlock || !bits || a.ldc > kStagedMaxLdc) return false;
  int nv = 0;
  s.vec[nv++] = second ? static_cast<const void*>(basis + (a.i + 1) * a.vec_stride) : a.w;
  for (int kk = 1; kk < nk; ++kk) s.vec[nv++] = basis + static_cast<int64_t>(kk) * a.vec_stride;   // u_0: bitmask
  s.bits = bits;
  s.nvec = nv;
  const int M = step_parts(a.ldc);
  const int W = 128 / static_cast<int>(sizeof(VT));
  const int target = (W / M) % W;
  auto padded = [&](int64_t rt) {
    int64_t v = rt * a.ldc;
    while (v % W != target) ++v;
    return v;
  };
  const int64_t rows_per_cta = (a.n + step_ctas(a.n) - 1) / step_ctas(a.n);
  const bool dw = a.pre_dinv != nullptr;
  const size_t row_bytes = static_cast<size_t>(nv) * a.ldc * sizeof(VT) + kBitWords * sizeof(uint32_t) + (dw ? 8 : 0);
  int64_t rt = static_cast<int64_t>((kStagedSmem - 256) / (kStages * row_bytes));
  rt = std::min<int64_t>(rt, std::max<int64_t>(1, rows_per_cta));
  while (rt > 1 && 128 + kStages * sizeof(VT) * stage_elems_of<VT>(nv, static_cast<int>(rt),
                                                                    static_cast<int>(padded(rt)), dw) > kStagedSmem)
    --rt;
  if (rt < 1) return false;
  s.rt = static_cast<int>(rt);
  s.vstride = static_cast<int>(padded(rt));
  *out = s;
  return true;
}

// Whether the persistent step kernel can run on `dev`: the part must be able to hold its grid and
// support cooperative launches (the launch itself then guarantees co-residency).
static int coop_supported(int dev) {
  static std::atomic<int> v[64];
  if (dev < 0 || dev >= 64) return 0;
  int cur = v[dev].load(std::memory_order_acquire);
  if (cur == 0) {
    int sms = 0, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cur = (sms >= kPersist && coop) ? 1 : 2;
    v[dev].store(cur, std::memory_order_release);
  }
  return cur == 1;
}

// Class launchers (instantiated per vector type and slot class in step_{f32,f64}_{wide,narrow}.cu).
bool step_launch_f32_wide(const StepArgs& sa, int nk, int parts, int threads, size_t smem, cudaStream_t st, cudaError_t* e);
bool step_launch_f32_narrow(const StepArgs& sa, int nk, int parts, int threads, size_t smem, cudaStream_t st, cudaError_t* e);
bool step_launch_f64_wide(const StepArgs& sa, int nk, int parts, int threads, size_t smem, cudaStream_t st, cudaError_t* e);
bool step_launch_f64_narrow(const StepArgs& sa, int nk, int parts, int threads, size_t smem, cudaStream_t st, cudaError_t* e);

// The dynamic shared-memory opt-in is per device context: remember it per (instance, device).
inline bool smem_optin(const void* fn, int bytes, std::atomic<bool>* done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  if (!done[dev].load(std::memory_order_acquire)) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
    done[dev].store(true, std::memory_order_release);
  }
  return true;
}

// The step kernel spins on a software grid barrier, so every CTA must be resident at once: it is
// launched as a COOPERATIVE kernel (cudaLaunchAttributeCooperative), for which the driver guarantees
// co-residency or fails the launch (cudaErrorCooperativeLaunchTooLarge) instead of hanging -- also
// when other streams, processes (MPS) or green contexts hold part of the SMs.  Capturable in graphs.
template <typename VT, int NK, int MM, int SL>
inline cudaError_t launch_step_coop(const StepArgs& sa, int threads, size_t smem, cudaStream_t st) {
  static std::atomic<bool> attr[64];
  if (!smem_optin(reinterpret_cast<const void*>(cgs_step_kernel<VT, NK, MM, SL>), static_cast<int>(kStagedSmem), attr))
    return cudaErrorInvalidDevice;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(step_ctas(sa.pass[0].a.n));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, cgs_step_kernel<VT, NK, MM, SL>, sa);
}

template <typename VT, int SL, int MM>
bool step_launch_one(const StepArgs& sa, int nk, int threads, size_t smem, cudaStream_t st, cudaError_t* err) {
  switch (nk) {
#define SLQ_STEP_K(K) \
    case K: *err = launch_step_coop<VT, K, MM, SL>(sa, threads, smem, st); return true;
    SLQ_STEP_K(1) SLQ_STEP_K(2) SLQ_STEP_K(3) SLQ_STEP_K(4) SLQ_STEP_K(5) SLQ_STEP_K(6) SLQ_STEP_K(7)
    SLQ_STEP_K(8) SLQ_STEP_K(9) SLQ_STEP_K(10) SLQ_STEP_K(11) SLQ_STEP_K(12) SLQ_STEP_K(13) SLQ_STEP_K(14)
    SLQ_STEP_K(15) SLQ_STEP_K(16)
#undef SLQ_STEP_K
    default: return false;
  }
}

// Launch everything after the SpMM of step i as one persistent kernel; false when the staged path
// does not apply (the caller then runs the separate kernels).
template <typename VT>
static bool launch_cgs_step(const CgsArgs& a, const ReduceArgs& red, const SpmmArgs& spmm, const uint32_t* bits,
                            int dev, cudaStream_t st, int* rc) {
  *rc = SLQ_OK;
  if (!coop_supported(dev)) return false;
  StepArgs sa{};
  if (!staged_setup<VT>(a, false, bits, &sa.pass[0]) || !staged_setup<VT>(a, true, bits, &sa.pass[1])) return false;
  sa.red = red;
  sa.spmm = spmm;
  const size_t smem = 128 + std::max(kSlotScratchBytes,
                                     kStages * sizeof(VT) *
                                         std::max(stage_elems_of<VT>(sa.pass[0].nvec, sa.pass[0].rt, sa.pass[0].vstride,
                                                                     a.pre_dinv != nullptr),
                                                  stage_elems_of<VT>(sa.pass[1].nvec, sa.pass[1].rt, sa.pass[1].vstride,
                                                                     a.pre_dinv != nullptr)));
  LaunchScope ls(K_CGS_UPDATE, st);
  // at most one CTA per SM by shared memory; the cooperative launch makes co-residency a driver
  // guarantee (the software grid barrier never waits on a CTA that is not running)
  const StepGeom geo = step_geometry(a.ldc);
  const int threads = 32 + geo.slots * step_slot_threads(a.ldc, geo.parts);
  const bool narrow = geo.slots == kNarrowSlots;
  cudaError_t e = cudaSuccess;
  bool ok;
  if (sizeof(VT) == 4) ok = narrow ? step_launch_f32_narrow(sa, a.i + 1, geo.parts, threads, smem, st, &e)
                                   : step_launch_f32_wide(sa, a.i + 1, geo.parts, threads, smem, st, &e);
  else ok = narrow ? step_launch_f64_narrow(sa, a.i + 1, geo.parts, threads, smem, st, &e)
                   : step_launch_f64_wide(sa, a.i + 1, geo.parts, threads, smem, st, &e);
  if (!ok) return false;
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) *rc = cuda_fail(e, "cgs_step_kernel cooperative launch");
  return true;
}

template <typename VT>
static int launch_cgs_dot(CgsArgs a, int max_ctas, cudaStream_t st) {
  const FlatGeom f = flat_geom(a.ldc);
  const int threads = f.G * kRowSlots * f.ldc;
  const int ctas = std::max(1, std::min(ceil_div(a.ntiles, f.G), max_ctas));
  const size_t smem = sizeof(double) * threads * (a.nk + 1);
  LaunchScope ls(K_CGS_DOT, st);
  if (smem > 48 * 1024)
    SLQ_CUDA(cudaFuncSetAttribute(cgs_dot_kernel<VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cgs_dot_kernel<VT><<<ctas, threads, smem, st>>>(a, f.ldc, f.G);
  return SLQ_OK;
}

template <typename VT>
static int launch_cgs_update(CgsArgs a, int max_ctas, cudaStream_t st) {
  const FlatGeom f = flat_geom(a.ldc);
  const int threads = f.G * kRowSlots * f.ldc;
  const int ctas = std::max(1, std::min(ceil_div(a.ntiles, f.G), max_ctas));
  const size_t smem = sizeof(double) * threads;
  LaunchScope ls(K_CGS_UPDATE, st);
  cgs_update_kernel<VT><<<ctas, threads, smem, st>>>(a, f.ldc, f.G);
  return SLQ_OK;
}

static void launch_reduce(ReduceArgs a, cudaStream_t st) {
  dim3 grid(a.nq, a.cpad / 32);
  LaunchScope ls(K_REDUCE, st);
  reduce_kernel<<<grid, kReduceWarps * 32, 0, st>>>(a);
}

// Per-vector-type entry points instantiated in spmm_{f32,f64}.cu and step_{f32,f64}.cu.
void launch_spmm_f32(int kind, const SpmmArgs& a, cudaStream_t st, bool finish);
void launch_spmm_f64(int kind, const SpmmArgs& a, cudaStream_t st, bool finish);
template <typename VT>
inline void spmm_entry(int kind, const SpmmArgs& a, cudaStream_t st, bool finish = true) {
  if (sizeof(VT) == 4) launch_spmm_f32(kind, a, st, finish);
  else launch_spmm_f64(kind, a, st, finish);
}

template <typename VT>
inline bool cgs_step_entry(const CgsArgs& a, const ReduceArgs& red, const SpmmArgs& spmm, const uint32_t* bits,
                           int dev, cudaStream_t st, int* rc) {
  return launch_cgs_step<VT>(a, red, spmm, bits, dev, st, rc);
}

}  // namespace slq
