// SpMM pass instantiations for float vectors (engine.cuh: spmm_kernel, spmm_long_finish_kernel).
#include "engine.cuh"

namespace slq {

void launch_spmm_f32(int kind, const SpmmArgs& a, cudaStream_t st, bool finish) {
  launch_spmm<float>(kind, a, st, finish);
}

}  // namespace slq
