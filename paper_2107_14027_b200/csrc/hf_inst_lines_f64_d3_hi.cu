// Instantiation unit: lines kernels, f64, d=3, variants 10-27.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_f64_d3_hi(int p, int variant, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info,
                     bool dry, bool faces) {
    return run_lines_range<double, 3, 10, 27>(p, variant, src, prm, st, info, dry, faces);
}
}  // namespace hfb
