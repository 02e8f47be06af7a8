// Instantiation unit: unfused stage-2/3/6 kernels, f32.
#include "hf_dispatch.cuh"
namespace hfb {
int unfused_f32(int d, int p, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_unfused_impl<float>(d, p, src, prm, st, info, dry);
}
}  // namespace hfb
