// replay_l1.cu — replay kernels of the <16,16> shared-memory layout
// (replay.cuh). Kept in its own translation unit for parallel builds.
#include "replay.cuh"

namespace pdg {

ReplayKernel replay_kernels_l1(int variant) {
#if defined(PDG_TP_BUILD)
  // throughput build (namespace pdg_tp): attainment-only search kernels only
  return variant == 3 ? replay_kernel<false, 16, 16, false, true> : variant == 0 ? replay_kernel<false, 16, 16, false>
                                                               : nullptr;
#else
  switch (variant) {
    case 2:
      return replay_kernel<false, 16, 16, true>;
    case 3:
      return replay_kernel<false, 16, 16, false, true>;
    default:  // diagnostics are built for the <8,8> layout only
      return replay_kernel<false, 16, 16, false>;
  }
#endif
}

cudaError_t replay_set_profile_l1(const pdsim_profile* profile, cudaStream_t stream) {
  return cudaMemcpyToSymbolAsync(c_profile, profile, sizeof(pdsim_profile), 0, cudaMemcpyHostToDevice, stream);
}

}  // namespace pdg
