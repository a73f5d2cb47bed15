// replay_l2.cu — replay kernels of the <64,32> shared-memory layout
// (replay.cuh). Kept in its own translation unit for parallel builds.
#include "replay.cuh"

namespace pdg {

ReplayKernel replay_kernels_l2(int variant) {
#if defined(PDG_TP_BUILD)
  // throughput build (namespace pdg_tp): attainment-only search kernels only
  return variant == 3 ? replay_kernel<false, 64, 32, false, true> : variant == 0 ? replay_kernel<false, 64, 32, false>
                                                               : nullptr;
#else
  switch (variant) {
    case 2:
      return replay_kernel<false, 64, 32, true>;
    case 3:
      return replay_kernel<false, 64, 32, false, true>;
    default:  // diagnostics are built for the <8,8> layout only
      return replay_kernel<false, 64, 32, false>;
  }
#endif
}

cudaError_t replay_set_profile_l2(const pdsim_profile* profile, cudaStream_t stream) {
  return cudaMemcpyToSymbolAsync(c_profile, profile, sizeof(pdsim_profile), 0, cudaMemcpyHostToDevice, stream);
}

}  // namespace pdg
