// Instantiation unit: managed planar kernels, f64.
#include "hf_dispatch.cuh"
namespace hfb {
int planar_managed_f64(int p, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_planar_managed_impl<double>(p, src, prm, st, info, dry);
}
}  // namespace hfb
