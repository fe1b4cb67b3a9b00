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



#include "engine.cuh"

namespace slq {

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

// Debug export of the Lanczos basis (lanczos.py:85,143-144 return_basis): q_k = u_k r_k
// into out[k][row][ldo] at column col0 + p; u_0 from the probe bitmask when the chunk kept it as bits.
template <typename VT>
__global__ void export_basis_kernel(const VT* __restrict__ basis, const uint32_t* __restrict__ bits,
                                    const double* __restrict__ rsc, int cpad, int64_t n, int64_t ldc, int c, int S,
                                    int64_t vs, double* __restrict__ out, int64_t ldo, int64_t col0) {
  const int64_t total = static_cast<int64_t>(S) * n * c;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(idx / (n * c));
    const int64_t rem = idx - static_cast<int64_t>(k) * n * c;
    const int64_t row = rem / c;
    const int p = static_cast<int>(rem - row * c);
    double u;
    if (k == 0 && bits) u = ((bits[row * kBitWords + (p >> 5)] >> (p & 31)) & 1u) ? 1.0 : -1.0;
    else u = static_cast<double>(basis[static_cast<int64_t>(k) * vs + row * ldc + p]);
    out[(static_cast<int64_t>(k) * n + row) * ldo + col0 + p] = u * rsc[static_cast<int64_t>(k) * cpad + p];
  }
}

// alpha_i = q_i . w for the steps that do not run the staged step kernel (the last step, s > 17,
// SLQ_STAGED=0): kAlphaCtas CTAs with fixed contiguous row ranges, 2 row slots per probe column,
// per-CTA partials reduced by reduce_kernel (fixed stripes): deterministic and independent of c.
constexpr int kAlphaCtas = 148 * 4;

template <typename VT>
__global__ void __launch_bounds__(256)
alpha_dot_kernel(const VT* __restrict__ u, const double* __restrict__ r, const VT* __restrict__ w, int64_t n,
                 int64_t ldc, int c, int cpad, double* __restrict__ partial) {
  __shared__ double red[2][kBlk];
  const int cols = (blockDim.x >> 1);
  const int pl = threadIdx.x % cols, slot = threadIdx.x / cols;
  const int p = blockIdx.y * kBlk + pl;
  const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  double s = 0.0;
  if (p < c) {
    const double rp = r[p];
    for (int64_t row = lo + slot; row < hi; row += 2) {
      const double x = __dmul_rn(ldg_f64(u + row * ldc + p), rp);
      s = fma(x, ldg_f64(w + row * ldc + p), s);
    }
  }
  red[slot][pl] = s;
  __syncthreads();
  if (slot == 0 && p < cpad) partial[static_cast<int64_t>(blockIdx.x) * cpad + p] = red[0][pl] + red[1][pl];
}

// ----------------------------------------------------------------------------- engine
static unsigned long long* g_step_dbg = nullptr;   // SLQ_STEP_TIMING buffer (diagnostics)
constexpr int kDbgStride = 32 + 4 * 160;           // per step: CTA 0's barrier stamps, then 4 per CTA
static void set_long_rows(SpmmArgs& sa, const slq_graph* g, double* segpart) {
  sa.long_counts = g->long_counts;
  sa.long_rows = g->long_rows;
  sa.long_seg_first = g->long_seg_first;
  sa.seg_row = g->seg_row;
  sa.seg_begin = g->seg_begin;
  sa.max_long = g->max_long;
  sa.max_seg = g->max_seg;
  sa.segpart = segpart;
}

static double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static bool trace_host() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("SLQ_TRACE_HOST"); v = (e && e[0] == '1') ? 1 : 0; }
  return v == 1;
}
#define SLQ_TRACE(label) do { if (trace_host()) fprintf(stderr, "[slq host] %-28s %9.3f ms\n", label, host_ms() - t_host0); } while (0)

static bool staged_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SLQ_STAGED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

void ensure_pool(int dev) {
  static std::atomic<bool> done[64];
  if (dev < 0 || dev >= 64 || done[dev].load(std::memory_order_acquire)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev].store(true, std::memory_order_release);
}

static int64_t partial_rows(const slq_graph* g);

// The all-staged schedule keeps u_0 as a bitmask and never stores u_S, so a chunk holds S vectors
// (u_1..u_{S-1} and w) instead of S + 2.
static bool lean_schedule(const slq_graph* g, bool start_block, int S, int reorth) {
  return !start_block && staged_enabled() && coop_supported(g->device) && reorth && S >= 2 && S - 1 <= kCgsBlock;
}

// Probes per chunk: as many as fit in 90% of the memory the device and this device's pool can
// still hand out (the pool keeps freed blocks), rounded down to a 32-byte sector multiple of
// columns when more than one sector fits (a narrower chunk gathers whole sectors; the padded
// tail of a wider chunk would not).  Results do not depend on the chunk width.
static int choose_chunk(const slq_graph* g, int64_t count, int S, int vbytes, bool lean, cudaStream_t st) {
  // Memory queries are not allowed while the stream is being captured into a CUDA graph: a capture
  // reuses the last value seen on this device by ANY host thread (process-wide, atomic), or, when no
  // eager call ran yet, a conservative fixed budget (1/4 of the device's memory).
  static std::atomic<double> last_avail[64];
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  double avail = 0.0;
  const int dev = g->device >= 0 && g->device < 64 ? g->device : 0;
  if (cap != cudaStreamCaptureStatusNone) {
    avail = last_avail[dev].load(std::memory_order_relaxed);
    if (avail <= 0.0) avail = static_cast<double>(g->device_total_mem) / 4.0;
  } else {
    size_t freeb = 0, total = 0;
    cudaMemGetInfo(&freeb, &total);
    avail = static_cast<double>(freeb);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, g->device) == cudaSuccess) {
      uint64_t reserved = 0, used = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      if (reserved > used) avail += static_cast<double>(reserved - used);
    }
    last_avail[dev].store(avail, std::memory_order_relaxed);
  }
  const double budget = 0.9 * avail - static_cast<double>(1ull << 30);
  const int nvec = lean ? S : S + 2;
  const double per_probe = static_cast<double>(nvec) * static_cast<double>(std::max<int64_t>(g->n, 1)) * vbytes +
                           8.0 * static_cast<double>(g->max_seg) +
                           8.0 * static_cast<double>(partial_rows(g)) * (kCgsBlock + 2);
  int64_t c = static_cast<int64_t>(budget / std::max(per_probe, 1.0));
  c = std::min<int64_t>({c, count, kMaxChunk});
  const int sector = 32 / vbytes;
  if (c < count && c > sector) c -= c % sector;
  return static_cast<int>(std::max<int64_t>(c, 1));
}

// Rows of reduction partials: flat fallback kernels (one per stream tile), the persistent step
// kernel (one per row slot) and alpha_dot_kernel (one per CTA).  The SpMM writes none.
static int64_t partial_rows(const slq_graph* g) {
  return std::max<int64_t>({static_cast<int64_t>(g->ntiles_stream), static_cast<int64_t>(kPersist) * kNarrowSlots,
                            static_cast<int64_t>(kAlphaCtas)});
}

// Bytes of the SpMM's persisting L2 window on graph g (0: none): degree-ordered folds only, capped by
// the device's persisting-L2 and window limits and SLQ_L2_WINDOW_MB; the persisting carve-out is set
// once per device.
static int64_t l2_window_bytes(const slq_graph* g) {
  if (!g->degree_ordered) return 0;
  // 32 MB by default (R-MAT-26, 32 probes: SpMM -2.7%, CGS step unchanged; the device maximum, 79 MB,
  // gives SpMM -5% but costs the step kernel +39% of its L2 reuse).  SLQ_L2_WINDOW_MB=0 turns
  // it off, -1 uses the device maximum (at most 64 MB), k sets k MB.  The carve-out (cudaLimitPersistingL2CacheSize,
  // a device-wide setting) is sized to the window.
  static const long long env_mb = [] { const char* e = getenv("SLQ_L2_WINDOW_MB"); return e ? atoll(e) : 32ll; }();
  if (env_mb == 0) return 0;
  const int dev = g->device >= 0 && g->device < 64 ? g->device : 0;
  static std::atomic<long long> cached[64];
  long long v = cached[dev].load(std::memory_order_acquire);
  if (v == 0) {
    int persist = 0, maxwin = 0;
    cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    long long bytes = std::min<long long>(persist, maxwin);
    if (env_mb > 0) bytes = std::min<long long>(bytes, env_mb << 20);
    else bytes = std::min<long long>(bytes, 64ll << 20);   // -1: the largest window the launches accept
    if (bytes > 0) {
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(static_cast<cudaStream_t>(g->stream), &cap);
      if (cap == cudaStreamCaptureStatusNone &&
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(bytes)) != cudaSuccess) {
        cudaGetLastError();
        bytes = 0;
      }
    }
    v = bytes > 0 ? bytes : -1;
    cached[dev].store(v, std::memory_order_release);
  }
  return v < 0 ? 0 : v;
}

// Operator-pair chunk: duplicate the probe bits of columns [0, split) into columns [split, 2 split)
// (word 0 of every bitmask row; 2 split <= 32).
static __global__ void pair_bits_kernel(uint32_t* __restrict__ bits, int64_t n, int split) {
  const uint32_t mask = (1u << split) - 1u;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w = bits[r * kBitWords] & mask;
    bits[r * kBitWords] = w | (w << split);
  }
}

// set when run_chunk refuses an operator-pair chunk (the caller then runs the two operators apart)
static thread_local bool tl_pair_refused = false;
static int pair_fail(const char* msg) {
  tl_pair_refused = true;
  return fail(SLQ_ERR_VALUE, msg);
}

// The recurrence runs on `g`; with an isolated-vertex fold, g is the folded graph and `orig` the
// graph the probes and the start-vector norm belong to (probe stream positions are original vertex
// ids, remapped to folded rows; the trailing row carries sqrt(m)).
struct FoldRun {
  const slq_graph* orig = nullptr;   // nullptr: no fold
};

template <typename VT>
static int run_chunk(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe0, const double* q0, int64_t ldq,
                     int c, int S, int reorth, double* alpha_out, double* beta_out, int32_t* steps_out, int64_t col0,
                     cudaStream_t st, FoldRun fold = FoldRun{}, double* basis_out = nullptr, int64_t basis_ld = 0,
                     int kind2 = -1, int split = 0) {
  // kind2 >= 0: an operator-PAIR chunk -- columns [0, split) run `kind` on probes probe0 .. probe0 +
  // split - 1, columns [split, c) run `kind2` on the SAME probes (column split + j = probe probe0 + j);
  // the flat SpMM serves both runs with one gather per nonzero (slq_rules_pair)
  const bool pair = kind2 >= 0;
  const double t_host0 = host_ms();
  const int64_t n = g->n;
  const int64_t n_probe = fold.orig ? fold.orig->n : n;   // probe length: ||v||^2 = n (slq.py:73)
  const int vb = sizeof(VT);
  // ldc: probes padded to a 32-byte sector multiple
  const int64_t ldc = ((c * vb + 31) / 32) * 32 / vb;
  const int cpad = ceil_div(c, 32) * 32;
  const int64_t vs = n * ldc;
  int rc = SLQ_OK;

  const int nq_max = kCgsBlock + 2;
  const int64_t ptiles = partial_rows(g);
  // u_0 as a probe bitmask (c <= 128): the first SpMM gathers bits and the staged step kernels
  // stream bits instead of u_0; the +-1 values are materialised only for the non-staged kernels.
  const bool coop_ok = staged_enabled() && coop_supported(g->device);
  const bool use_bits = !q0 && c <= kBlk;
  const bool all_staged = use_bits && coop_ok && reorth && S >= 2 && S - 1 <= kCgsBlock && ldc <= kStagedMaxLdc;
  // all_staged: slots u_1..u_{S-1} and w only (lean_schedule); basis[0] is never addressed
  const int64_t nvec = all_staged ? S : S + 2;
  const size_t bytes_vec = static_cast<size_t>(vs) * vb * nvec;
  const int gstride = std::min(S + 1, kCgsBlock + 2);   // Gram matrix of the staged steps (i + 1 <= kCgsBlock)
  const size_t bytes_state = sizeof(double) * cpad * (6 * (S + 1) + 3 + gstride * gstride) +
                             sizeof(int) * (3 * cpad + 4 + S + 4) + sizeof(unsigned long long) * (4 * S + 2);
  const size_t bytes_part = sizeof(double) * ptiles * nq_max * cpad;
  const size_t bytes_seg = sizeof(double) * g->max_seg * cpad;
  const size_t off_state = ((bytes_vec + 255) / 256) * 256;
  const size_t off_part = off_state + ((bytes_state + 255) / 256) * 256;
  char* ws = nullptr;
  SLQ_TRACE("before malloc");
  const size_t off_seg = off_part + ((bytes_part + 255) / 256) * 256;
  const size_t off_bits = off_seg + ((bytes_seg + 255) / 256) * 256;
  const size_t bytes_bits = sizeof(uint32_t) * kBitWords * static_cast<size_t>(std::max<int64_t>(n, 1));
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), off_bits + bytes_bits, st));
  // every early return below frees the workspace (the pool never releases it to the device)
  struct WsGuard {
    void* p;
    cudaStream_t s;
    ~WsGuard() { if (p) cudaFreeAsync(p, s); }
  } ws_guard{ws, st};
  SLQ_TRACE("after malloc");
  VT* basis = all_staged ? reinterpret_cast<VT*>(ws) - vs : reinterpret_cast<VT*>(ws);
  VT* wv = basis + (all_staged ? S : S + 1) * vs;
  double* dstate = reinterpret_cast<double*>(ws + off_state);
  ChunkState s;
  s.c = c; s.cpad = cpad; s.S = S;
  s.rsc = dstate;
  s.alpha = s.rsc + (S + 1) * cpad;
  s.beta = s.alpha + (S + 1) * cpad;
  s.h = s.beta + (S + 1) * cpad;
  s.nb2 = s.h + (S + 1) * cpad;
  s.cdot = s.nb2 + cpad;
  s.gram = s.cdot + (S + 1) * cpad;
  s.nrm2 = s.gram + (S + 1) * cpad;
  s.G = s.nrm2 + cpad;
  s.gstride = gstride;
  int* istate = reinterpret_cast<int*>(s.G + static_cast<int64_t>(gstride) * gstride * cpad);
  s.steps = istate;
  s.alive = istate + cpad;
  s.again = istate + 2 * cpad;
  s.any_again = istate + 3 * cpad;
  s.second_passes = (fold.orig ? fold.orig : g)->dflags + 2;
  s.barrier = reinterpret_cast<unsigned int*>(istate + 3 * cpad + 4);
  s.work = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(s.barrier + S) + 15) & ~static_cast<uintptr_t>(15));
  double* partial = reinterpret_cast<double*>(ws + off_part);

  {
    LaunchScope ls(K_PROBE, st);
    state_init_kernel<<<ceil_div(std::max(cpad, 4 * S), 128), 128, 0, st>>>(s, n_probe, q0 != nullptr);
  }
  uint32_t* bits = use_bits ? reinterpret_cast<uint32_t*>(ws + off_bits) : nullptr;
  if (q0) {
    LaunchScope ls(K_PROBE, st);
    copy_start_kernel<VT><<<std::max(1, std::min(ceil_div(n * c, 256), 148 * 16)), 256, 0, st>>>(q0, ldq, c, n, basis, ldc);
  } else if (fold.orig) {
    if (!all_staged) return fail(SLQ_ERR_VALUE, "isolated-vertex fold needs the all-staged schedule");
    launch_probes<VT>(seed, probe0, pair ? split : c, n_probe, nullptr, ldc, st, bits, fold.orig->fold_remap);
    SLQ_CUDA(cudaMemsetAsync(bits + (n - 1) * kBitWords, 0xff, sizeof(uint32_t) * kBitWords, st));
  } else {
    if (pair && !all_staged) return pair_fail("operator-pair chunk needs the all-staged schedule");
    launch_probes<VT>(seed, probe0, pair ? split : c, n, all_staged ? nullptr : basis, ldc, st, bits);
  }
  if (pair) {   // the second operator's columns carry the same probes
    LaunchScope ls(K_PROBE, st);
    pair_bits_kernel<<<std::max(1, std::min(ceil_div(n, 256), 148 * 16)), 256, 0, st>>>(bits, n, split);
  }

  SpmmArgs sa{};
  sa.offsets = g->offsets; sa.cols = g->cols; sa.weights = g->weights; sa.degree = g->degree; sa.dinv = g->dinv;
  sa.tile_rows = g->tile_rows; sa.ntiles = g->ntiles;
  // flat SpMM (spmm_flat.cu): walks quads of neighbouring rows in lockstep, so it needs the
  // degree-ordered fold (SLQ_SPMM_FLAT=1 forces it on any graph: same results, wasted slots)
  static const bool flat_forced = [] { const char* e = getenv("SLQ_SPMM_FLAT"); return e && atoi(e) > 0; }();
  if (g->ftile_rows && (g->degree_ordered || flat_forced)) { sa.ftile_rows = g->ftile_rows; sa.nftiles = g->nftiles; }
  sa.n_rows = n; sa.nnz_total = g->nnz;
  if (pair) {
    sa.split = split;
    if (!sa.ftile_rows || !std::is_same<VT, float>::value || ldc <= 16 || ldc > 32 || (split & 3) || g->weights ||
        !all_staged || c != 2 * split || n >= (int64_t(1) << 29) || g->max_seg >= (int64_t(1) << 29))
      return pair_fail("operator-pair chunk needs the flat SpMM (fp32, 17..32 columns, unit weights, staged steps)");
  }
  sa.dscal = g->dscal;
  sa.w = wv; sa.ldc_in = ldc; sa.ldc_out = ldc; sa.c = c; sa.cpad = cpad;
  set_long_rows(sa, g, reinterpret_cast<double*>(ws + off_seg));
  // Degree-ordered fold: the first rows of every gathered vector are the hubs; an L2 access-policy
  // window can keep them persisting across the SpMM (LRU alone evicts a hub row between its references
  // when the cold rows stream through).  SLQ_L2_WINDOW_MB sizes it (see l2_window_bytes).
  const int64_t win_bytes = l2_window_bytes(g);
  const int64_t win_rows_vec = win_bytes > 0 ? std::min<int64_t>(n, win_bytes / (ldc * vb)) : 0;

  CgsArgs ca{};
  ca.n = n; ca.ldc = ldc; ca.vec_stride = vs; ca.rows_per_tile = g->rows_per_stream_tile;
  ca.ntiles = g->ntiles_stream; ca.c = c; ca.cpad = cpad; ca.basis = basis; ca.w = wv; ca.s = s;
  ca.partial = partial; ca.reorth = reorth;
  if (fold.orig) {
    ca.virt_row = n - 1;
    ca.virt_root = std::sqrt(static_cast<double>(fold.orig->fold_m));
  }

  ReduceArgs ra{};
  ra.partial = partial; ra.cpad = cpad; ra.c = c; ra.s = s; ra.kind = kind; ra.dscal = g->dscal; ra.reorth = reorth;
  if (pair) { ra.kind2 = kind2; ra.split = split; ca.pre_split = split; }

  // Prescaled gathers (normalized Laplacian, narrow class, graphs whose dinv does not stay in L2):
  // step kernel i also writes dinv (.) u_{i+1} into the slot of u_{i+2} (unused until step kernel i+1),
  // and SpMM i+1 gathers it instead of u_{i+1} times a dinv[col] gather per nonzero.  Steps 1..S-2
  // (step 0 gathers the probe bitmask, the last SpMM has no free slot).  A function of the graph and
  // the step kernel's slot class only, so results stay bitwise independent of the chunk width.
  static const bool pre_env = [] { const char* e = getenv("SLQ_PRESCALE"); return !(e && e[0] == '0'); }();
  static const int64_t pre_min_n = [] {   // SLQ_PRESCALE_MIN_N: testing knob
    const char* e = getenv("SLQ_PRESCALE_MIN_N");
    return e ? static_cast<int64_t>(atoll(e)) : (int64_t(1) << 22);
  }();
  // ... or any graph the flat SpMM runs on (fine tiles + degree-ordered rows: a property of the graph
  // too): its normalized-Laplacian gathers are the prescaled ones (R-MAT-22, 32 probes: SpMM + step
  // kernels 67.1 -> 42.7 ms per run; R-MAT-20: 16.9 -> 14.7 ms)
  const bool pre_size = n >= pre_min_n || (g->ftile_rows && g->degree_ordered);
  const bool prescale = pre_env && kind == SLQ_NORMALIZED_LAPLACIAN && all_staged && ldc <= 32 && pre_size;
  // The last SpMM (step S-1) is prescaled too: the last step kernel writes dinv (.) u_{S-1} over w (each
  // CTA over rows it has already consumed), and that SpMM, which only feeds alpha_{S-1}, writes its
  // output into the slot of u_1 (no longer needed).  Needs S >= 3 and no basis export.
  const bool last_pre = prescale && S >= 3 && !basis_out;
  // Step 0 of the normalized Laplacian on large graphs gathers the probe bitmask AND dinv[col]: two
  // random line requests per nonzero.  32-byte [bits | dinv] records (built into the slot of u_1, free
  // until the first step kernel writes u_1) make it one; values and arithmetic are unchanged.
  if (pair && !(prescale && last_pre && kind == SLQ_NORMALIZED_LAPLACIAN && kind2 == SLQ_DENSITY))
    return pair_fail("operator-pair chunk needs prescaled normalized-Laplacian gathers + density");
  const bool rec_on = kind == SLQ_NORMALIZED_LAPLACIAN && all_staged && bits != nullptr && S >= 2 &&
                      ldc * vb >= static_cast<int64_t>(sizeof(uint32_t)) * kRecWords && pre_size && pre_env;
  if (pair && !rec_on) return pair_fail("operator-pair chunk needs the first-step records");
  // SLQ_STEP_TIMING=1 (diagnostics): the step kernels stamp %globaltimer around their grid barriers
  static unsigned long long* dbgbuf = [] {
    unsigned long long* p = nullptr;
    const char* e = getenv("SLQ_STEP_TIMING");
    if (e && e[0] == '1' && cudaMalloc(&p, sizeof(unsigned long long) * kDbgStride * kMaxSteps) != cudaSuccess) p = nullptr;
    return p;
  }();
  g_step_dbg = dbgbuf;
  const int gx = 1 << 30;                 // one CTA per tile group
  const bool coop = coop_ok && bits != nullptr;
  const int gx2 = kSecondPassGrid;        // second pass: small grid-stride launch

  // Non-staged path (s > 17, SLQ_STAGED=0 or no cooperative launch): separate kernels + reductions.
  auto dot_pass = [&](int i, int second, int grid_x) {
    for (int k0 = 0; k0 <= i; k0 += kCgsBlock) {
      ca.k0 = k0;
      ca.nk = std::min(kCgsBlock, i + 1 - k0);
      ca.second = second;
      launch_cgs_dot<VT>(ca, grid_x, st);
      ra.mode = RED_CGS; ra.ntiles = g->ntiles_stream; ra.nq = ca.nk + 1; ra.k0 = k0; ra.nk = ca.nk;
      ra.second = second;
      launch_reduce(ra, st);
    }
  };

  for (int i = 0; i < S; ++i) {
    sa.u = basis + i * vs;
    sa.r = s.rsc + i * cpad;
    ra.mode = RED_ALPHA; ra.ntiles = kAlphaCtas; ra.nq = 1; ra.i = i; ra.second = 0;
    ra.k0 = 0; ra.nk = 0;
    sa.red = ra;
    sa.work = s.work + 4 * i;
    sa.bits = (i == 0) ? bits : nullptr;
    sa.rec = nullptr;
    if (i == 0 && rec_on) {   // [bits | dinv] records in the (still unused) slot of u_1
      uint32_t* rec = reinterpret_cast<uint32_t*>(basis + vs);
      LaunchScope ls(K_PROBE, st);
      step0_records_kernel<<<std::max(1, std::min(ceil_div(n, 256), 148 * 16)), 256, 0, st>>>(bits, g->dinv, n, rec);
      sa.rec = rec;
    }
    sa.win_rows = sa.bits ? std::min<int64_t>(n, win_bytes / static_cast<int64_t>(sizeof(uint32_t) * kBitWords))
                          : win_rows_vec;
    if (win_bytes <= 0) sa.win_rows = 0;
    sa.upre = (prescale && i >= 1 && i <= S - 2) ? static_cast<const void*>(basis + (i + 1) * vs) : nullptr;
    sa.w = wv;
    ca.pre_dinv = (prescale && i + 1 <= S - 2) ? g->dinv : nullptr;
    ca.pre_out = nullptr;
    if (last_pre && i == S - 2) {   // the last step kernel: dinv (.) u_{S-1} over w
      ca.pre_dinv = g->dinv;
      ca.pre_out = wv;
    }
    if (last_pre && i == S - 1) {   // the last SpMM gathers it and writes into the slot of u_1
      sa.upre = wv;
      sa.w = basis + vs;
    }
    ca.dbg = (dbgbuf && i < kMaxSteps) ? dbgbuf + kDbgStride * i : nullptr;
    ca.i = i;
    ca.second = 0;
    // staged step kernel: alpha and the CGS coefficients come from its Gram form, so the SpMM only
    // writes w; otherwise (last step, s > 17, SLQ_STAGED=0) the SpMM also reduces alpha.
    const bool staged = coop && reorth && i < S - 1 && i + 1 <= kCgsBlock && ldc <= kStagedMaxLdc;
    // alpha: step kernel (staged) or alpha_dot_kernel
    SLQ_TRACE("spmm launch");
    spmm_entry<VT>(kind, sa, st, /*finish=*/!staged);   // staged: phase 0 finishes
    SLQ_TRACE("spmm launched");
    if (!staged) {
      // the long rows of w must be complete before alpha: finish kernel ran inside launch_spmm
      const int colsb = std::min(cpad, kBlk);
      {
        LaunchScope ls(K_REDUCE, st);
        alpha_dot_kernel<VT><<<dim3(kAlphaCtas, ceil_div(c, kBlk)), 2 * colsb, 0, st>>>(
            basis + i * vs, s.rsc + i * cpad, static_cast<const VT*>(sa.w), n, ldc, c, cpad, partial);
      }
      ReduceArgs rd = ra;
      rd.ntiles = kAlphaCtas;
      launch_reduce(rd, st);
    }
    if (i == S - 1) break;
    if (staged) {
      const bool done = cgs_step_entry<VT>(ca, ra, sa, bits, g->device, st, &rc);
      SLQ_TRACE("step launched");
      if (rc) return rc;
      if (done) continue;
      return fail(SLQ_ERR_CUDA, "staged step kernel unavailable after the SpMM skipped alpha");
    }
    if (reorth) dot_pass(i, 0, gx);
    ca.second = 0;
    rc = launch_cgs_update<VT>(ca, gx, st);
    if (rc) return rc;
    ra.mode = RED_NORM; ra.ntiles = g->ntiles_stream; ra.nq = 1; ra.second = 0;
    launch_reduce(ra, st);
    if (reorth) {
      // conditional second CGS pass (lanczos.py:75-76); kernels exit unless a probe asked for it
      dot_pass(i, 1, gx2);
      ca.second = 1;
      rc = launch_cgs_update<VT>(ca, gx2, st);
      if (rc) return rc;
      ca.second = 0;
      ra.mode = RED_NORM2; ra.ntiles = g->ntiles_stream; ra.nq = 1; ra.second = 1;
      launch_reduce(ra, st);
      ra.second = 0;
    }
  }
  {
    LaunchScope ls(K_REDUCE, st);
    scatter_out_kernel<<<ceil_div(c, 128), 128, 0, st>>>(s, col0, S, alpha_out, beta_out, steps_out);
  }
  if (basis_out) {
    LaunchScope ls(K_REDUCE, st);
    const int64_t total = static_cast<int64_t>(S) * n * c;
    export_basis_kernel<VT><<<std::max(1, std::min(ceil_div(total, 256), 148 * 16)), 256, 0, st>>>(
        basis, all_staged ? bits : nullptr, s.rsc, cpad, n, ldc, c, S, vs, basis_out, basis_ld, col0);
  }
  SLQ_CUDA(cudaGetLastError());
  ws_guard.p = nullptr;
  SLQ_CUDA(cudaFreeAsync(ws, st));
  SLQ_TRACE("chunk done");
  return SLQ_OK;
}

}  // namespace slq

using namespace slq;

static int lanczos_entry(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, const double* q0,
                         int64_t ldq, int64_t count, int steps, int reorth, int dtype, double* alpha, double* beta,
                         int32_t* steps_out, void* stream, double* basis_out = nullptr) {
  if (!g) return fail(SLQ_ERR_VALUE, "NULL graph");
  if (steps < 1) return fail(SLQ_ERR_VALUE, "step budget must be >= 1");
  if (count < 0 || probe_begin < 0) return fail(SLQ_ERR_VALUE, "negative probe range");
  if (kind < 0 || kind > 2) return fail(SLQ_ERR_VALUE, "unknown operator kind");
  if (dtype != SLQ_F64 && dtype != SLQ_F32) return fail(SLQ_ERR_VALUE, "dtype must be SLQ_F64 or SLQ_F32");
  if (g->n == 0) return fail(SLQ_ERR_VALUE, "start vector must have unit norm");
  if (kind == SLQ_DENSITY && g->nnz == 0) return fail(SLQ_ERR_VALUE, "density matrix undefined for a graph without edges");
  int rc = SLQ_OK;
  const int S = static_cast<int>(std::min<int64_t>(steps, g->n));   // lanczos.py:105
  if (S > kMaxStepsLong) return fail(SLQ_ERR_VALUE, "steps > 4096 not supported");
  if (reorth < 0) reorth = S <= 100 ? 1 : 0;                          // lanczos.py:106-107
  if (count == 0) return SLQ_OK;
  if (q0 && ldq < count) return fail(SLQ_ERR_VALUE, "ldq < count");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ensure_pool(g->device);
  const int vb = dtype == SLQ_F64 ? 8 : 4;
  const double t_host0 = host_ms();
  // isolated-vertex fold (slq_graph_fold_isolated): only under the all-staged schedule (u_0 as the
  // probe bitmask, which is where the trailing row's sqrt(m) is substituted)
  const bool lean = lean_schedule(g, q0 != nullptr, S, reorth);
  FoldRun fold;
  const slq_graph* gr = g;
  if (g->folded && lean && !basis_out) {   // the basis export runs on the unfolded graph
    fold.orig = g;
    gr = g->folded;
  }
  int cmax = choose_chunk(gr, count, S, vb, lean, st);
  if (fold.orig) cmax = std::min(cmax, kBlk);   // bitmask probes: <= 128 per chunk
  SLQ_TRACE("choose_chunk");
  for (int64_t done = 0; done < count;) {
    const int c = static_cast<int>(std::min<int64_t>(cmax, count - done));
    const double* qc = q0 ? q0 + done : nullptr;
    rc = dtype == SLQ_F64
             ? run_chunk<double>(gr, kind, seed, probe_begin + done, qc, ldq, c, S, reorth, alpha, beta, steps_out, done, st,
                                 fold, basis_out, count)
             : run_chunk<float>(gr, kind, seed, probe_begin + done, qc, ldq, c, S, reorth, alpha, beta, steps_out, done, st,
                                fold, basis_out, count);
    if (rc) return rc;
    done += c;
  }
  return SLQ_OK;
}

extern "C" int slq_lanczos(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count,
                           int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                           void* stream) {
  return lanczos_entry(g, kind, seed_key_u64(seed), probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha, beta,
                       steps_out, stream);
}

extern "C" int slq_lanczos_seeded(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin,
                                  int64_t count, int steps, int reorth, int dtype, double* alpha, double* beta,
                                  int32_t* steps_out, void* stream) {
  SeedKey k;
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  return lanczos_entry(g, kind, k, probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha, beta, steps_out,
                       stream);
}

extern "C" int slq_lanczos_start(const slq_graph* g, int kind, const double* q0, int64_t ldq, int64_t count,
                                 int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                                 void* stream) {
  if (!q0) return fail(SLQ_ERR_VALUE, "NULL start block");
  return lanczos_entry(g, kind, seed_key_u64(0), 0, q0, ldq, count, steps, reorth, dtype, alpha, beta, steps_out,
                       stream);
}

extern "C" int slq_operator_apply(const slq_graph* g, int kind, const double* x, double* y, int64_t ncols,
                                  int64_t ld, void* stream) {
  if (!g || (!x && g->n) || (!y && g->n)) return fail(SLQ_ERR_VALUE, "NULL argument");
  if (kind < 0 || kind > 2) return fail(SLQ_ERR_VALUE, "unknown operator kind");
  if (kind == SLQ_DENSITY && g->nnz == 0) return fail(SLQ_ERR_VALUE, "density matrix undefined for a graph without edges");
  if (ncols <= 0 || g->n == 0) return SLQ_OK;
  if (ld < ncols) return fail(SLQ_ERR_VALUE, "ld < ncols");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  constexpr int64_t kCols = 2 * kBlk;   // columns per pass (two 128-probe blocks)
  const int64_t passes = (ncols + kCols - 1) / kCols;
  double* segpart = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&segpart), sizeof(double) * g->max_seg * kCols + 64, st));
  unsigned long long* work = nullptr;
  SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&work), sizeof(unsigned long long) * 4 * passes, st));
  SLQ_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned long long) * 4 * passes, st));
  for (int64_t pi = 0; pi < passes; ++pi) {
    const int64_t j0 = pi * kCols;
    SpmmArgs sa{};
    sa.offsets = g->offsets; sa.cols = g->cols; sa.weights = g->weights; sa.degree = g->degree; sa.dinv = g->dinv;
    sa.tile_rows = g->tile_rows; sa.ntiles = g->ntiles;
    sa.dscal = g->dscal;
    sa.u = x + j0; sa.r = nullptr; sa.w = y + j0; sa.ldc_in = ld; sa.ldc_out = ld;
    sa.c = static_cast<int>(std::min<int64_t>(kCols, ncols - j0));
    sa.cpad = ceil_div(sa.c, 32) * 32;
    sa.work = work + 4 * pi;
    set_long_rows(sa, g, segpart);
    spmm_entry<double>(kind, sa, st);
  }
  SLQ_CUDA(cudaFreeAsync(segpart, st));
  SLQ_CUDA(cudaFreeAsync(work, st));
  SLQ_CUDA(cudaGetLastError());
  return SLQ_OK;
}

static int probes_entry(const SeedKey& seed, int64_t probe_begin, int64_t count, int64_t n, double* out, int64_t ld,
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

extern "C" int slq_probes(uint64_t seed, int64_t probe_begin, int64_t count, int64_t n, double* out, int64_t ld,
                          void* stream) {
  return probes_entry(seed_key_u64(seed), probe_begin, count, n, out, ld, stream);
}

extern "C" int slq_probes_seeded(const slq_seed* seed, int64_t probe_begin, int64_t count, int64_t n, double* out,
                                 int64_t ld, void* stream) {
  SeedKey k;
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  return probes_entry(k, probe_begin, count, n, out, ld, stream);
}

static void probe_state_words(const SeedKey& k, uint64_t index, uint64_t out_host[4]) {
  u128 st, inc;
  pcg64_seed_state(k, index, &st, &inc);
  out_host[0] = static_cast<uint64_t>(st >> 64);
  out_host[1] = static_cast<uint64_t>(st);
  out_host[2] = static_cast<uint64_t>(inc >> 64);
  out_host[3] = static_cast<uint64_t>(inc);
}

extern "C" int slq_probe_state(uint64_t seed, uint64_t index, uint64_t out_host[4]) {
  if (!out_host) return fail(SLQ_ERR_VALUE, "NULL output");
  probe_state_words(seed_key_u64(seed), index, out_host);
  return SLQ_OK;
}

extern "C" int slq_probe_state_seeded(const slq_seed* seed, uint64_t index, uint64_t out_host[4]) {
  SeedKey k;
  if (!out_host) return fail(SLQ_ERR_VALUE, "NULL output");
  if (!seed_key_of(seed, &k)) return fail(SLQ_ERR_VALUE, "seed must have 1..8 entropy words");
  probe_state_words(k, index, out_host);
  return SLQ_OK;
}

// Diagnostics (not part of the C ABI header): the SLQ_STEP_TIMING stamps of the last chunk,
// [step][kDbgStride] %globaltimer values (ns); returns the number of values copied.
extern "C" int slq_debug_step_times(unsigned long long* host, int n) {
  if (!g_step_dbg || !host) return 0;
  n = std::min(n, kDbgStride * kMaxSteps);
  if (cudaMemcpy(host, g_step_dbg, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

extern "C" int slq_lanczos_basis(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count,
                                 int steps, int reorth, int dtype, double* basis, double* alpha, double* beta,
                                 int32_t* steps_out, void* stream) {
  if (!basis) return fail(SLQ_ERR_VALUE, "NULL basis output");
  return lanczos_entry(g, kind, seed_key_u64(seed), probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha, beta,
                       steps_out, stream, basis);
}

// Diagnostics counter (slq_b200.h): probe-steps of this graph that ran the conditional second CGS
// pass (lanczos.py:75-76), summed over every Lanczos call since the graph was created.  Synchronous.
extern "C" int slq_graph_second_passes(const slq_graph* g, int64_t* out_host) {
  if (!g || !out_host) return fail(SLQ_ERR_VALUE, "NULL argument");
  int v = 0;
  SLQ_CUDA(cudaMemcpyAsync(&v, g->dflags + 2, sizeof(int), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(g->stream)));
  SLQ_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(g->stream)));
  *out_host = v;
  return SLQ_OK;
}

extern "C" int slq_lanczos_start_basis(const slq_graph* g, int kind, const double* q0, int64_t ldq, int64_t count,
                                       int steps, int reorth, int dtype, double* basis, double* alpha, double* beta,
                                       int32_t* steps_out, void* stream) {
  if (!q0) return fail(SLQ_ERR_VALUE, "NULL start block");
  if (!basis) return fail(SLQ_ERR_VALUE, "NULL basis output");
  return lanczos_entry(g, kind, seed_key_u64(0), 0, q0, ldq, count, steps, reorth, dtype, alpha, beta, steps_out,
                       stream, basis);
}

// C++ entry for rules.cu (seed as a SeedKey)
int lanczos_seeded_key(const slq_graph* g, int kind, const SeedKey& seed, int64_t probe_begin, int64_t count,
                       int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out, void* stream) {
  return lanczos_entry(g, kind, seed, probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha, beta, steps_out,
                       stream);
}

// Normalized Laplacian + density matrix on the SAME probes (heat/wave + VNGE of one signature).  With
// <= 16 probes (a rank's share of 128 probes on 8 GPUs) a single operator fills only half of a
// 128-byte gathered row, and the SpMM is bound by line requests, not bytes: the pair chunk interleaves
// both operators' columns in one row, so ONE pass over the graph per Lanczos step serves both runs.
// Per-probe arithmetic is that of the separate narrow-class runs (bitwise).  *paired = 1 when the pair
// chunk ran; otherwise (count > 16, fp64, small or unfolded graphs ...) the operators run apart.
int lanczos_pair_key(const slq_graph* g, const SeedKey& seed, int64_t probe_begin, int64_t count, int steps, int reorth,
                     int dtype, double* alpha_a, double* beta_a, int32_t* steps_a, double* alpha_b, double* beta_b,
                     int32_t* steps_b, void* stream, int* paired) {
  if (paired) *paired = 0;
  if (!g) return fail(SLQ_ERR_VALUE, "NULL graph");
  static const bool pair_env = [] { const char* e = getenv("SLQ_PAIR"); return !(e && e[0] == '0'); }();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int S = static_cast<int>(std::min<int64_t>(steps, std::max<int64_t>(g->n, 1)));
  const int ro = reorth < 0 ? (S <= 100 ? 1 : 0) : reorth;
  const int split = static_cast<int>((count + 3) / 4 * 4);
  if (pair_env && dtype == SLQ_F32 && count >= 9 && count <= 16 && steps >= 3 && probe_begin >= 0 && g->n > 0 &&
      g->nnz > 0 && S >= 3 && S <= kMaxStepsLong && lean_schedule(g, false, S, ro)) {
    ensure_pool(g->device);
    FoldRun fold;
    const slq_graph* gr = g;
    if (g->folded) {
      fold.orig = g;
      gr = g->folded;
    }
    // the pair block is ONE chunk of 2 * split columns: run the operators apart if it does not fit
    const bool fits = choose_chunk(gr, 2 * split, S, 4, true, st) >= 2 * split;
    char* tmp = nullptr;
    const size_t bn = sizeof(double) * 2 * split * S;
    SLQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), 2 * bn + sizeof(int32_t) * 2 * split + 16, st));
    double* ta = reinterpret_cast<double*>(tmp);
    double* tb = ta + 2 * split * S;
    int32_t* ts = reinterpret_cast<int32_t*>(tmp + 2 * bn);
    tl_pair_refused = false;
    int rc = fits ? run_chunk<float>(gr, SLQ_NORMALIZED_LAPLACIAN, seed, probe_begin, nullptr, 0, 2 * split, S, ro, ta, tb,
                                     ts, 0, st, fold, nullptr, 0, SLQ_DENSITY, split)
                  : pair_fail("operator-pair chunk does not fit the device memory");
    if (rc == SLQ_OK) {
      const size_t row = sizeof(double) * S;
      cudaMemcpyAsync(alpha_a, ta, row * count, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(beta_a, tb, row * count, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(steps_a, ts, sizeof(int32_t) * count, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(alpha_b, ta + static_cast<int64_t>(split) * S, row * count, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(beta_b, tb + static_cast<int64_t>(split) * S, row * count, cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(steps_b, ts + split, sizeof(int32_t) * count, cudaMemcpyDeviceToDevice, st);
    }
    cudaFreeAsync(tmp, st);
    if (rc == SLQ_OK) {
      SLQ_CUDA(cudaGetLastError());
      if (paired) *paired = 1;
      return SLQ_OK;
    }
    if (!tl_pair_refused) return rc;
    set_error("");   // refused: run the operators apart
  }
  int rc = lanczos_entry(g, SLQ_NORMALIZED_LAPLACIAN, seed, probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha_a,
                         beta_a, steps_a, stream);
  if (rc) return rc;
  return lanczos_entry(g, SLQ_DENSITY, seed, probe_begin, nullptr, 0, count, steps, reorth, dtype, alpha_b, beta_b,
                       steps_b, stream);
}

// Return the memory the library's stream-ordered pool keeps cached on the current device to the
// driver (the pool's release threshold is "never", so freed workspaces are reused across calls).
extern "C" int slq_trim_pool(void) {
  int dev = 0;
  SLQ_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  SLQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  SLQ_CUDA(cudaDeviceSynchronize());
  SLQ_CUDA(cudaMemPoolTrimTo(pool, 0));
  return SLQ_OK;
}

// Diagnostics: the device's persisting-L2 and access-policy-window limits (bytes).
extern "C" int slq_l2_limits(int64_t* persist_max, int64_t* window_max) {
  int dev = 0, p = 0, w = 0;
  SLQ_CUDA(cudaGetDevice(&dev));
  SLQ_CUDA(cudaDeviceGetAttribute(&p, cudaDevAttrMaxPersistingL2CacheSize, dev));
  SLQ_CUDA(cudaDeviceGetAttribute(&w, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  if (persist_max) *persist_max = p;
  if (window_max) *window_max = w;
  return SLQ_OK;
}
