// Staged CGS step kernel instantiations for float vectors (engine.cuh: cgs_step_kernel).
#include "engine.cuh"

namespace slq {

bool launch_cgs_step_f32(const CgsArgs& a, const ReduceArgs& red, const SpmmArgs& spmm, const uint32_t* bits, int dev,
                        cudaStream_t st, int* rc) {
  return launch_cgs_step<float>(a, red, spmm, bits, dev, st, rc);
}

}  // namespace slq
