// Instantiation unit: grouped-chunk lines kernels (whole caller groups per chunk), f64, d=3.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_grouped_f64_d3(int p, int gs, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info,
                          bool dry) {
    return run_lines_grouped<double, 3>(p, gs, src, prm, st, info, dry);
}
}  // namespace hfb
