// Instantiation unit: mapped-element (non-constant Jacobian) kernels, f32.
#include "hf_dispatch.cuh"
namespace hfb {
int mapped_f32(int d, int p, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_mapped_impl<float>(d, p, src, prm, st, info, dry);
}
}  // namespace hfb
