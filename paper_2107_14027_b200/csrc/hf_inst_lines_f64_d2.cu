// Instantiation unit: lines kernels, f64, d=2.
#include "hf_dispatch.cuh"
namespace hfb {
int lines_f64_d2(int p, int variant, bool src, const Params<double>& prm, cudaStream_t st, KInfo* info, bool dry) {
    return run_lines_d2<double>(p, variant, src, prm, st, info, dry);
}
}  // namespace hfb
