// Instantiation unit: stage kernels for uint8_t, 4-word chunks (all TY, both shift modes).
#include "bmc_fme_impl.cuh"

namespace bmc {

int launch_stage_u8c4(bool shift, const CUtensorMap& tw, const CUtensorMap& tc, const StageLaunch& a, dim3 grid,
                      cudaStream_t st) {
  return shift ? dispatch_ty<uint8_t, 4, true>(tw, tc, a, grid, st) : dispatch_ty<uint8_t, 4, false>(tw, tc, a, grid, st);
}

}  // namespace bmc
