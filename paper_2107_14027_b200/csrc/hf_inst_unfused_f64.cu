// Instantiation unit: unfused stage-2/3/6 kernels, f64.
#include "hf_dispatch.cuh"
namespace hfb {
int unfused_f64(int d, int p, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_unfused_impl<double>(d, p, src, prm, st, info, dry);
}
}  // namespace hfb
