// Batched block-diagonal path for collections of small graphs (C3). See slq_lanczos_batched.
#include "slq_common.cuh"

using namespace slq;

extern "C" int slq_lanczos_batched(const slq_graph* g, const int64_t* vertex_offsets, int64_t num_graphs, int kind,
                                   uint64_t seed, int n_v, int steps, int dtype, double* nodes, double* weights,
                                   int32_t* steps_out, void* stream) {
  (void)g; (void)vertex_offsets; (void)num_graphs; (void)kind; (void)seed; (void)n_v; (void)steps; (void)dtype;
  (void)nodes; (void)weights; (void)steps_out; (void)stream;
  return fail(SLQ_ERR_VALUE, "slq_lanczos_batched: not built yet");
}
