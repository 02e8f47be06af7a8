// Instantiation unit: managed planar kernels, f32.
#include "hf_dispatch.cuh"
namespace hfb {
int planar_managed_f32(int p, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_planar_managed_impl<float>(p, src, prm, st, info, dry);
}
}  // namespace hfb
