// Instantiation of the fused step for world groups of 1 warp(s) (parallel build unit).
#include "step_impl.cuh"

namespace cf {
cudaError_t launch_step_w1(const StepParams& p, cudaStream_t s) { return launch_wpw<1>(p, s); }
}  // namespace cf
