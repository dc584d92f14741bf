// Instantiation of the persistent fused step (k_step_persist in step_impl.cuh):
// CTAs that step their worlds in turn, the next world TMA-staged into shared
// memory (STAGE) or prefetched into L2.
#include <cstdlib>

#include "step_impl.cuh"

namespace cf {

// COMFREE_PERSIST_MODE (tuning): 1 = 8 warps, L2 prefetch (default);
// 2 = 16 warps, TMA-staged slab; 3 = 32 warps, TMA-staged slab
static int persist_mode() {
  const char* e = getenv("COMFREE_PERSIST_MODE");
  const int m = e ? atoi(e) : 1;
  return (m >= 1 && m <= 3) ? m : 1;
}

size_t step_persist_smem_bytes(const SceneDev& sc) { return persist_smem_bytes(sc, persist_mode() != 1); }

template <int WPW, bool STAGE>
static cudaError_t launch_mode(const StepParams& p, cudaStream_t s, int n_sm) {
  const bool imp = p.impulses != nullptr || p.wstats != nullptr;
  if (p.n_t == 4 && p.power_is_2 && !p.exact_diag)
    return imp ? launch_persist_variant<WPW, STAGE, true, true>(p, s, n_sm)
               : launch_persist_variant<WPW, STAGE, true, false>(p, s, n_sm);
  return imp ? launch_persist_variant<WPW, STAGE, false, true>(p, s, n_sm)
             : launch_persist_variant<WPW, STAGE, false, false>(p, s, n_sm);
}

cudaError_t launch_step_persist(const StepParams& p, cudaStream_t s) {
  int dev = 0, n_sm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  switch (persist_mode()) {
    case 2: return launch_mode<16, true>(p, s, n_sm);
    case 3: return launch_mode<32, true>(p, s, n_sm);
    default: return launch_mode<8, false>(p, s, n_sm);
  }
}

}  // namespace cf
