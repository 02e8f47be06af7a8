// Instantiation unit: mapped-element (non-constant Jacobian) kernels, f64.
#include "hf_dispatch.cuh"
namespace hfb {
int mapped_f64(int d, int p, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_mapped_impl<double>(d, p, src, prm, st, info, dry);
}
}  // namespace hfb
