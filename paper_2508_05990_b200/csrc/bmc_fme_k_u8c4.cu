// Instantiation unit: stage kernels for uint8_t, 4-word chunks (all TY, both shift modes).
#include "bmc_fme_ws.cuh"

namespace bmc {

int launch_stage_u8c4(bool shift, const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                      cudaStream_t st) {
  if (a.plan.ws && shift) {
    const int rc = dispatch_ws<uint8_t, 4, true>(tw, tc, a, st);
    if (rc != -1) return rc;  // -1: no work counter (first use inside a graph capture) -> classic kernel
    StageLaunch b = a;
    b.plan.ws = 0;
    return dispatch_ty<uint8_t, 4, true>(tw, tc, b, grid, st);
  }
  return shift ? dispatch_ty<uint8_t, 4, true>(tw, tc, a, grid, st) : dispatch_ty<uint8_t, 4, false>(tw, tc, a, grid, st);
}

}  // namespace bmc
