// Instantiation of the fused step for one world per 16-warp CTA (parallel build unit).
#include "step_impl.cuh"

namespace cf {
cudaError_t launch_step_w16(const StepParams& p, cudaStream_t s) { return launch_cfg<16, 16>(p, s); }
}  // namespace cf
