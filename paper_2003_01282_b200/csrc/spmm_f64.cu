// SpMM pass instantiations for double vectors (engine.cuh: spmm_kernel, spmm_long_finish_kernel).
#include "engine.cuh"

namespace slq {

void launch_spmm_f64(int kind, const SpmmArgs& a, cudaStream_t st, bool finish) {
  launch_spmm<double>(kind, a, st, finish);
}

}  // namespace slq
