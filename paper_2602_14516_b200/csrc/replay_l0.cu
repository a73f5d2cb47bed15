// replay_l0.cu — replay kernels of the <8,8> shared-memory layout
// (replay.cuh). Kept in its own translation unit for parallel builds.
#include "replay.cuh"

namespace pdg {

ReplayKernel replay_kernels_l0(int variant) {
#if defined(PDG_TP_BUILD)
  // throughput build (namespace pdg_tp): attainment-only search kernels only
  return variant == 3 ? replay_kernel<false, 8, 8, false, true> : variant == 0 ? replay_kernel<false, 8, 8, false>
                                                               : nullptr;
#else
  switch (variant) {
    case 1:
      return replay_kernel<true, 8, 8, false>;
    case 2:
      return replay_kernel<false, 8, 8, true>;
    case 3:
      return replay_kernel<false, 8, 8, false, true>;
    default:
      return replay_kernel<false, 8, 8, false>;
  }
#endif
}

cudaError_t replay_set_profile_l0(const pdsim_profile* profile, cudaStream_t stream) {
  return cudaMemcpyToSymbolAsync(c_profile, profile, sizeof(pdsim_profile), 0, cudaMemcpyHostToDevice, stream);
}

ReplayKernel replay_kernel_for(int layout, int variant) {
  return layout == 0 ? replay_kernels_l0(variant) : layout == 1 ? replay_kernels_l1(variant) : replay_kernels_l2(variant);
}

cudaError_t replay_set_profile(const pdsim_profile* profile, cudaStream_t stream) {
  cudaError_t e = replay_set_profile_l0(profile, stream);
  if (e == cudaSuccess) e = replay_set_profile_l1(profile, stream);
  if (e == cudaSuccess) e = replay_set_profile_l2(profile, stream);
  return e;
}

}  // namespace pdg
