// Instantiation unit: lines kernels, f32, d=2, variants 10-27.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_f32_d2_hi(int p, int variant, bool src, const Params<float>& prm, cudaStream_t st, KInfo* info,
                     bool dry, bool faces) {
    return run_lines_range<float, 2, 10, 27>(p, variant, src, prm, st, info, dry, faces);
}
}  // namespace hfb
