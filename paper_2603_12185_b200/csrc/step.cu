// step.cu — dispatch of the fused step kernel (see step_impl.cuh).
#include "step_impl.cuh"

namespace cf {

cudaError_t launch_step_w1(const StepParams& p, cudaStream_t s);
cudaError_t launch_step_w2(const StepParams& p, cudaStream_t s);
cudaError_t launch_step_w4(const StepParams& p, cudaStream_t s);
cudaError_t launch_step_w8(const StepParams& p, cudaStream_t s);
cudaError_t launch_step_w16(const StepParams& p, cudaStream_t s);

size_t step_world_floats(const SceneDev& sc) { return (size_t)group_layout(sc).total; }

size_t step_smem_bytes(const SceneDev& sc, int wpw) {
  return (size_t)(wpw >= kWarps ? 1 : kWarps / wpw) * group_layout(sc).total * sizeof(float);
}

cudaError_t launch_step(const StepParams& p, int wpw, cudaStream_t s) {
  switch (wpw) {
    case 1: return launch_step_w1(p, s);
    case 2: return launch_step_w2(p, s);
    case 4: return launch_step_w4(p, s);
    case 16: return launch_step_w16(p, s);
    default: return launch_step_w8(p, s);
  }
}

}  // namespace cf
