// inst_f32.cu -- instantiations of the fused / pool kernel template (fused_kernel.cuh) for one table
// element type; compiled as its own translation unit so the instance set builds in parallel.
#include "fused_kernel.cuh"

namespace emba2a {

cudaError_t plan_f32(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl) {
  return plan_elem<0, false>(P, c, fused, pl);
}

}  // namespace emba2a
