// Instantiation of the deterministic step (one warp and one world per CTA).
#include "step_impl.cuh"

namespace cf {
cudaError_t launch_step_det(const StepParams& p, cudaStream_t s) { return launch_cfg<1, 1, true>(p, s); }
}  // namespace cf
