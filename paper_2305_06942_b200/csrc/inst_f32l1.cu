// inst_f32l1.cu -- fp32 unweighted instances with L1-allocating row loads (ELEM 3 of the
// fused / pool kernel template, fused_kernel.cuh): chosen for forwards with enough lookups per SM
// that hot rows recur on the same SM (host.cpp ensure_chunk, option "l1_rows").
#include "fused_kernel.cuh"

namespace emba2a {

cudaError_t plan_f32l1(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl) {
  return plan_elem<3, false>(P, c, fused, pl);
}

}  // namespace emba2a
