// Instantiation unit: grouped-chunk lines kernels (whole caller groups per chunk), f32, d=2.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_grouped_f32_d2(int p, int gs, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info,
                          bool dry) {
    return run_lines_grouped<float, 2>(p, gs, src, prm, st, info, dry);
}
}  // namespace hfb
