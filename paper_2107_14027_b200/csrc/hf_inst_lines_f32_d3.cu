// Instantiation unit: lines kernels, f32, d=3.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_f32_d3(int p, int variant, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_lines_d3<float>(p, variant, src, prm, st, info, dry);
}
}  // namespace hfb
