// inst_f16l1.cu -- fp16 unweighted instances with L1-allocating row loads (ELEM 5 of the fused /
// pool kernel template, fused_kernel.cuh; option "l1_rows", host.cpp ensure_chunk).
#include "fused_kernel.cuh"

namespace emba2a {

cudaError_t plan_f16l1(const KParams& P, const LaunchCfg& c, bool fused, LaunchPlan* pl) {
  return plan_elem<5, false>(P, c, fused, pl);
}

}  // namespace emba2a
