// Staged CGS step kernels, double vectors, narrow class (12 row slots; engine.cuh: cgs_step_kernel).
#include "engine.cuh"

namespace slq {

bool step_launch_f64_narrow(const StepArgs& sa, int nk, int parts, int threads, size_t smem, cudaStream_t st, cudaError_t* e) {
  switch (parts) {
    case 1: return step_launch_one<double, kNarrowSlots, 1>(sa, nk, threads, smem, st, e);
    case 2: return step_launch_one<double, kNarrowSlots, 2>(sa, nk, threads, smem, st, e);
    case 4: return step_launch_one<double, kNarrowSlots, 4>(sa, nk, threads, smem, st, e);
    default: return false;
  }
}

}  // namespace slq
