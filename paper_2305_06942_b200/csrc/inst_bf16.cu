// inst_bf16.cu -- instantiations of the fused / pool kernel template (fused_kernel.cuh) for one table
// element type; compiled as its own translation unit so the instance set builds in parallel.
#include "fused_kernel.cuh"

namespace emba2a {

cudaError_t plan_bf16(const KParams& P, const LaunchCfg& c, bool fused, bool weighted,
                      LaunchPlan* pl) {
  return weighted ? plan_elem<1, true>(P, c, fused, pl) : plan_elem<1, false>(P, c, fused, pl);
}

}  // namespace emba2a
