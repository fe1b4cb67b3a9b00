/*
 * slq_b200.h — C ABI of libslq_b200.so, the B200 (sm_100a) stochastic Lanczos
 * quadrature engine.  Plain pointers and sizes only; no torch types.
 *
 * Reference interfaces replaced (all paths under /root/reference/pkg/src/spectrace/):
 *
 *   slq_graph_create / _host     operators.py:52-62  (_adjacency, degrees) and the
 *                                operator set-up of make_operator, operators.py:65-102
 *   slq_operator_apply           LinearOperator.apply closures, operators.py:76-99
 *   slq_operator_interval        LinearOperator.interval, operators.py:79-101
 *   slq_lanczos                  slq._collect_rules/_probe_rule (slq.py:63-86) minus the
 *                                eigensolve: probe draw, lanczos_tridiagonalize
 *                                (lanczos.py:79-145) with CGS reorth (lanczos.py:70-76)
 *   slq_gauss_rules              quadrature_rule (lanczos.py:148-163) + node clip (slq.py:76-77)
 *   slq_quadrature               _apply_rule over the whole grid (slq.py:89-95, 153-168)
 *   slq_estimate                 _estimate_from (slq.py:98-105)
 *   slq_probes / slq_probe_state _draw_probe + seeding (slq.py:63-72)
 *
 * Conventions
 *   - Every data pointer is a DEVICE pointer unless the name ends in _host.
 *   - Matrices are row-major with an explicit leading dimension (ld, in elements).
 *   - Work is stream-ordered on the given cudaStream_t (passed as void*; NULL =
 *     legacy default stream).  No call synchronises the device except the
 *     _host variants and slq_profile_end.
 *   - Return value: SLQ_OK or an error code; slq_last_error() gives a
 *     thread-local message.  The Python layer maps codes to the reference's
 *     exceptions (ValueError, TridiagonalEigenError, RuntimeError).
 *   - Reentrant: a graph handle is immutable after creation; concurrent calls
 *     on one handle from different streams or host threads are allowed
 *     (workspace is stream-ordered, allocated per call; lazily initialised
 *     per-device state is atomic).  The persistent step kernel, which syncs
 *     its CTAs through a software grid barrier, is launched as a COOPERATIVE
 *     kernel: the driver makes all its CTAs co-resident or fails the launch,
 *     so concurrent calls never deadlock (they may serialise on the SMs).
 */
#ifndef SLQ_B200_H
#define SLQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SLQ_OK 0
#define SLQ_ERR_VALUE 1      /* invalid argument / undefined operator  -> ValueError           */
#define SLQ_ERR_EIGEN 2      /* tridiagonal eigensolver did not converge -> TridiagonalEigenError */
#define SLQ_ERR_CUDA 3       /* CUDA runtime error                     -> RuntimeError          */
#define SLQ_ERR_NONFINITE 4  /* f non-finite at a node (slq.py:91-94)  -> ValueError           */
#define SLQ_ERR_ALLOC 5      /* device allocation failed               -> MemoryError           */

/* operator kinds (operators.py:31-34) */
#define SLQ_LAPLACIAN 0
#define SLQ_NORMALIZED_LAPLACIAN 1
#define SLQ_DENSITY 2

/* vector storage precision inside the Lanczos recurrence (reductions are always fp64) */
#define SLQ_F64 0
#define SLQ_F32 1

/* integrands for slq_quadrature: f(t, x) at clamped nodes x */
#define SLQ_FN_HEAT 0      /* exp(-t x)                 descriptors.py:132-134 */
#define SLQ_FN_WAVE_RE 1   /* cos(t x)                  Re exp(-i t x)          */
#define SLQ_FN_WAVE_IM 2   /* -sin(t x)                 Im exp(-i t x)          */
#define SLQ_FN_XLOGX 3     /* x ln x (0 at x<=0)        descriptors.py:220-224  */
#define SLQ_FN_IDENTITY 4  /* x                                                  */

typedef struct slq_graph slq_graph;

/* A probe seed of any size: the reference passes SlqConfig.seed (any non-negative Python int,
 * slq.py:28-35,63-72) to numpy's SeedSequence, which splits it into little-endian uint32 words
 * (0 -> one zero word).  The *_seeded entry points take that word list (seeds < 2^256); the plain
 * uint64_t-seed entry points are the same streams for seeds < 2^64. */
typedef struct slq_seed {
  uint32_t words[8];
  int32_t nwords;   /* 1..8 */
} slq_seed;

typedef struct slq_graph_info_t {
  int64_t n;
  int64_t nnz;          /* stored nonzeros = row_offsets[n] */
  double trace_l;       /* tr L = sum of degrees (operators.py:93) */
  double max_degree;
  int64_t isolated;     /* vertices of degree 0 */
  int32_t unit_weights; /* 1 when every weight is exactly 1.0 (weights dropped on device) */
  int32_t ntiles;       /* SpMM row tiles (fixed per graph; reduction order depends only on them) */
} slq_graph_info_t;

/* Build the device graph from DEVICE CSR arrays (canonical layout of graphs.py:110-132):
 * int64 offsets[n+1], int64 cols[nnz] (sorted per row), float64 weights[nnz] or NULL
 * (NULL = every weight 1.0).  The arrays are copied/narrowed; the caller keeps ownership.
 * Stream-ordered and asynchronous: input errors (out-of-range columns) surface in
 * slq_graph_info() and in the status word of the asynchronous calls.  `stream` must outlive
 * the graph (its buffers are freed on it). */
int slq_graph_create(int64_t n, int64_t nnz, const int64_t* offsets, const int64_t* cols,
                     const double* weights, void* stream, slq_graph** out);
/* Same from HOST arrays (the end-to-end plugin entry: H2D copies happen inside). */
int slq_graph_create_host(int64_t n, int64_t nnz, const int64_t* offsets_host,
                          const int64_t* cols_host, const double* weights_host, void* stream,
                          slq_graph** out);
/* Same from int32 column indices (host or device pointers): the compact CSR of the scale-27 workload
 * ("int32 indices", BASELINE configs[4]); weights == NULL means implicit 1.0.  The column copy is
 * adopted by the graph (no int64 staging); out-of-range columns are flagged as in slq_graph_create. */
int slq_graph_create_i32(int64_t n, int64_t nnz, const int64_t* offsets, const int32_t* cols,
                         const double* weights, void* stream, slq_graph** out);
int slq_graph_info(const slq_graph* g, slq_graph_info_t* out);
void slq_graph_destroy(slq_graph* g);

/* Generate an R-MAT graph on the device and build its canonical CSR there (no host arrays; the
 * C4/C5 workloads of BASELINE.json, whose CSR does not fit a host round trip at scale 27).
 * n = 2^scale, edge_factor * n samples, quadrant probabilities (a, b, c, 1-a-b-c); both directions,
 * self-loops dropped, duplicates collapsed, rows/columns ascending (graphs.py canonical form, the
 * reference's graph ingestion at operators.py:52-62 via scipy.sparse.csr_matrix).  Sample j, level l
 * draws slq_rmat_uniform_host(seed, j, l).  Synchronises `stream` (the unique-key count). */
int slq_graph_create_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                          void* stream, slq_graph** out);
/* Canonical CSR built on the device from an edge list u[m], v[m] (int64) and optional weights w[m]
 * (host or device pointers): self-loops dropped, both directions stored, duplicate edges collapsed
 * to the maximum weight, rows and columns ascending — graphs.py:110-132 (`_build_csr`).  Endpoints
 * outside [0, n) -> SLQ_ERR_VALUE.  Synchronises `stream` (the unique-edge count). */
int slq_graph_create_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v, const double* w,
                           void* stream, slq_graph** out);
/* Stored edge weights [nnz] into `weights` (device or host; may be NULL); *has_weights_host = 0
 * when the graph uses implicit unit weights (nothing is copied). */
int slq_graph_weights(const slq_graph* g, double* weights, int32_t* has_weights_host, void* stream);
/* Copy the prepared CSR (int64 offsets [n+1], int32 columns [nnz]) into caller buffers (device or
 * host; either may be NULL), stream-ordered. */
int slq_graph_csr(const slq_graph* g, int64_t* offsets, int32_t* cols, void* stream);
/* The generator's uniform for (seed, sample, level), for host restatements of the generator. */
int slq_rmat_uniform_host(uint64_t seed, uint64_t sample, int level, double* out);

/* Isolated-vertex fold.  Vertices with an empty row that no row references (degree 0: every
 * operator gives 0 there, operators.py:76-99) evolve in the Lanczos recurrence as the probe sign times
 * one per-probe scalar, so the recurrence can run on the graph without them plus ONE trailing empty
 * row standing for all m of them (value sqrt(m) times that scalar): dot products agree with the
 * unfolded ones to rounding, the Lanczos vectors lose m rows.  The kept rows are renumbered by
 * descending degree (every row keeps its columns in stored order, so row sums are bitwise the
 * unfolded ones).  Builds the fold when m >= 1 and m >= min_fraction * n (min_fraction < 0 drops an
 * existing fold); unit-weight graphs with >= 2^24 nonzeros are folded for ANY m >= 0, because the
 * degree order is what the flat SpMM needs (m = 0: the trailing row stays zero).  *folded_host = m.
 * Afterwards slq_lanczos / slq_rules / slq_signature on g use the fold whenever the all-staged
 * schedule runs (generated probes, reorth on, 2 <= s' <= 17, <= 128 probes per chunk); the operator
 * apply, degrees, CSR export and the batched path keep using g itself.  Synchronises the creation
 * stream; the fold holds a second copy of the CSR. */
int slq_graph_fold_isolated(slq_graph* g, double min_fraction, int64_t* folded_host);

/* Copy the prepared degree vector d = A.1 and dinv = 1/sqrt(d) (0 if isolated) into [n]
 * device buffers (either may be NULL).  operators.py:58-62, 84-86. */
int slq_graph_degrees(const slq_graph* g, double* degree, double* dinv, void* stream);

/* Exact trace of the squared operator from one edge pass (operators.py:119-141; the control-variate
 * companion of the degree identity tr M = slq_graph_info): writes the host double *out_host. */
int slq_trace_squared(const slq_graph* g, int kind, double* out_host);

/* Spectrum bounds used for node clamping (operators.py:79,90,101). */
int slq_operator_interval(const slq_graph* g, int kind, double* lo, double* hi);

/* Y = Op(X) for ncols columns; X, Y are [n][ld] float64.  Bit-identical to the
 * reference closure on each column (sequential in-row sums, no FMA). */
int slq_operator_apply(const slq_graph* g, int kind, const double* x, double* y, int64_t ncols,
                       int64_t ld, void* stream);

/* Lanczos tridiagonals for probes [probe_begin, probe_begin+count) of seed `seed`.
 * Probes: Rademacher from PCG64(SeedSequence(seed, spawn_key=(i,))) (slq.py:63-73).
 * steps: requested s (clamped to n, lanczos.py:105); reorth: 1 on, 0 off, -1 = reference
 * default (on iff s <= 100, lanczos.py:106-107).  dtype: SLQ_F64 / SLQ_F32 vector storage.
 * Outputs (ld = steps): alpha[count][steps], beta[count][steps] (entries >= steps_out-1 unused),
 * steps_out[count] = achieved steps (breakdown shortens, lanczos.py:133-134).
 * Per-probe results do not depend on count, probe_begin or chunking. */
int slq_lanczos(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count,
                int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                void* stream);

int slq_lanczos_seeded(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin, int64_t count,
                       int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                       void* stream);

/* Debug export (lanczos_tridiagonalize(..., return_basis=True), lanczos.py:85,143-144): slq_lanczos
 * plus the Lanczos vectors q_k = u_k / beta_{k-1} of every probe, basis[k][row][count] (k < s',
 * float64; zero after a probe's breakdown).  Runs on the unfolded graph. */
int slq_lanczos_basis(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count, int steps,
                      int reorth, int dtype, double* basis, double* alpha, double* beta, int32_t* steps_out,
                      void* stream);

/* Same recurrence from caller-given unit start vectors q0[n][ldq] (column j = start vector j);
 * the lanczos_tridiagonalize(op, q0, s) entry (lanczos.py:79-104). */
int slq_lanczos_start(const slq_graph* g, int kind, const double* q0, int64_t ldq, int64_t count,
                      int steps, int reorth, int dtype, double* alpha, double* beta, int32_t* steps_out,
                      void* stream);

/* slq_lanczos_start plus the basis export of slq_lanczos_basis: the
 * lanczos_tridiagonalize(op, q0, s, return_basis=True) entry (lanczos.py:79-145). */
int slq_lanczos_start_basis(const slq_graph* g, int kind, const double* q0, int64_t ldq, int64_t count, int steps,
                            int reorth, int dtype, double* basis, double* alpha, double* beta, int32_t* steps_out,
                            void* stream);

/* Gauss rules of `count` tridiagonals (alpha/beta rows of length ld <= 4096, steps[count]):
 * nodes ascending, clamped to [lo, hi]; weights = squared first eigenvector entries.
 * info[p] = 0 ok, else the eigensolver failed for probe p (returns SLQ_ERR_EIGEN). */
int slq_gauss_rules(const double* alpha, const double* beta, const int32_t* steps, int64_t count,
                    int ld, double lo, double hi, double* nodes, double* weights, int32_t* info,
                    void* stream);

/* per_vector[T][count] = sum_k weights[p][k] * f(t, nodes[p][k]) over k < steps[p]. */
int slq_quadrature(const double* nodes, const double* weights, const int32_t* steps, int64_t count,
                   int ld, const double* t, int64_t T, int fn, double* per_vector, void* stream);

/* value[t] = n * mean_p per_vector[t][p]; std_error[t] = std(n*pv, ddof=1)/sqrt(count). */
int slq_estimate(const double* per_vector, int64_t T, int64_t count, double n, double* value,
                 double* std_error, void* stream);

/* ---- asynchronous composite entry points (no host synchronisation; errors are OR-ed into a
 * device int32 *status: 1 eigensolver failed, 2 non-finite tridiagonal, 4 non-finite integrand,
 * 8 out-of-range column index).  The caller reads *status with the results. ---- */

/* Gauss rules of probes [probe_begin, +count): slq_lanczos + slq_gauss_rules with the operator's
 * clamp interval taken from the device graph scalars.  nodes/weights [count][s'], s' = min(steps, n). */
int slq_rules(const slq_graph* g, int kind, uint64_t seed, int64_t probe_begin, int64_t count, int steps,
              int reorth, int dtype, double* nodes, double* weights, int32_t* steps_out, int32_t* status,
              void* stream);

int slq_rules_seeded(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin, int64_t count,
                     int steps, int reorth, int dtype, double* nodes, double* weights, int32_t* steps_out,
                     int32_t* status, void* stream);

/* Heat/wave + VNGE of one signature share their probes (slq.py:63-72: same seed, same stream): the
 * normalized-Laplacian rules (netlsd_slq, descriptors.py:124-149) AND the density-matrix rules
 * (vnge_slq, descriptors.py:227-243) of probes [probe_begin, +count) in one call.  With 9..16 fp32
 * probes on a large folded graph (a rank's share of 128 probes on 8 GPUs) both Lanczos runs travel
 * in ONE block of 32 interleaved columns, so each step gathers one 128-byte row per nonzero for both
 * operators (half the passes over the graph); per-probe results are bitwise those of two
 * slq_rules_seeded calls.  Otherwise it is those two calls.  *paired (host, may be NULL) = 1 when
 * the fused block ran. */
int slq_rules_pair_seeded(const slq_graph* g, const slq_seed* seed, int64_t probe_begin, int64_t count, int steps,
                          int reorth, int dtype, double* nodes_nl, double* weights_nl, int32_t* steps_nl,
                          double* nodes_p, double* weights_p, int32_t* steps_p, int32_t* status, int32_t* paired,
                          void* stream);

/* Synchronous host-buffer form of slq_rules_seeded for FFI bindings that have no device allocator
 * (the reference's ctypes stub): the seam _collect_rules (slq.py:80-86) in one call.
 * nodes_host/weights_host [count][s'], steps_host [count], s' = min(steps, n); the device status is
 * mapped to the return code (SLQ_ERR_EIGEN / SLQ_ERR_VALUE).  Runs on (and synchronises) the graph's
 * creation stream. */
int slq_rules_host(const slq_graph* g, int kind, const slq_seed* seed, int64_t probe_begin, int64_t count,
                   int steps, int reorth, int dtype, double* nodes_host, double* weights_host, int32_t* steps_host);

/* For each integrand fns_host[f] (host array of SLQ_FN_*): quadrature over t[T] and the probe
 * aggregate: values[f][T], std_errors[f][T]; per_vector[f][T][count] if not NULL (slq.py:89-105). */
int slq_integrate(const double* nodes, const double* weights, const int32_t* steps, int64_t count, int ld,
                  const double* t, int64_t T, const int* fns_host, int nfn, double n, double* values,
                  double* std_errors, double* per_vector, int32_t* status, void* stream);

/* The whole signature (netlsd_slq / vnge_slq / wave): rules of probes 0..count-1, then every
 * integrand over the grid.  values/std_errors [nfn][T] on the device.  descriptors.py:124-149, 227-243. */
int slq_signature(const slq_graph* g, int kind, uint64_t seed, int64_t count, int steps, int reorth,
                  int dtype, const double* t, int64_t T, const int* fns_host, int nfn, double* values,
                  double* std_errors, int32_t* status, void* stream);

/* Rademacher probes as +-1.0 into out[n][ld] (column j = probe probe_begin+j). */
int slq_probes(uint64_t seed, int64_t probe_begin, int64_t count, int64_t n, double* out,
               int64_t ld, void* stream);
int slq_probes_seeded(const slq_seed* seed, int64_t probe_begin, int64_t count, int64_t n, double* out, int64_t ld,
                      void* stream);
/* Host: PCG64 (state_hi, state_lo, inc_hi, inc_lo) of SeedSequence(seed, spawn_key=(index,)). */
int slq_probe_state(uint64_t seed, uint64_t index, uint64_t out_host[4]);
int slq_probe_state_seeded(const slq_seed* seed, uint64_t index, uint64_t out_host[4]);

/* Batched block-diagonal path (C3): many small graphs stacked in one block-diagonal CSR, one CTA
 * per graph.  vertex_offsets[G+1] (device int64) delimit the graphs; graph g uses probes
 * 0..n_v-1 restricted to its own n_g vertices (stream prefixes, q0 = v/sqrt(n_g)) exactly as
 * netlsd_slq / vnge_slq on that graph alone (descriptors.py:124-149, 227-243).  kind: SLQ_NORMALIZED_LAPLACIAN
 * or SLQ_DENSITY; n_v <= 64.  Outputs: nodes/weights [G][n_v][steps] (clamped, ascending),
 * steps_out [G][n_v]; errors OR-ed into the device *status. */
int slq_lanczos_batched(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs,
                        int kind, uint64_t seed, int n_v, int steps, int dtype, double* nodes,
                        double* weights, int32_t* steps_out, int32_t* status, void* stream);

int slq_lanczos_batched_seeded(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs, int kind,
                               const slq_seed* seed, int n_v, int steps, int dtype, double* nodes, double* weights,
                               int32_t* steps_out, int32_t* status, void* stream);

/* Per-graph quadrature + probe aggregate of batched rules: values/std_errors [G][T]
 * (value = n_g * mean over the graph's probes). */
int slq_integrate_batched(const double* nodes, const double* weights, const int32_t* steps,
                          int64_t num_graphs, int n_v, int ld, const int64_t* vertex_offsets,
                          const double* t, int64_t T, int fn, double* values, double* std_errors,
                          int32_t* status, void* stream);

/* Diagnostics */
/* Probe-steps of graph g that ran the conditional second CGS pass (lanczos.py:75-76), summed over
 * every Lanczos call on g since it was created (synchronises the graph's creation stream). */
int slq_graph_second_passes(const slq_graph* g, int64_t* out_host);
/* Release the device memory the library's stream-ordered pool keeps cached on the current device
 * (synchronises the device). */
int slq_trim_pool(void);
/* The device's persisting-L2 capacity and access-policy-window limit (bytes; SpMM hub window). */
int slq_l2_limits(int64_t* persist_max, int64_t* window_max);
/* The first `count` row lengths of the graph the Lanczos recurrence runs on (the isolated-vertex fold,
 * degree-ordered, when there is one) and its row count. */
int slq_graph_lanczos_rows(const slq_graph* g, int64_t* lengths_host, int64_t count, int64_t* rows_host);
const char* slq_last_error(void);
uint64_t slq_launch_count(void);                /* kernels launched by this library so far */
void slq_profile_begin(void);                   /* start per-class CUDA-event timing */
/* Stop timing (synchronises the recorded events); fills ms[class] and launches[class] for
 * up to `n` classes: 0 prepare, 1 probe, 2 spmm, 3 cgs_dot, 4 cgs_update, 5 reduce, 6 eig,
 * 7 quad, 8 estimate, 9 batched.  Returns the number of classes. */
int slq_profile_end(double* ms, int64_t* launches, int n);
const char* slq_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SLQ_B200_H */
