// Instantiation unit: FR stages 1 and 4+5 (hf_fr.cuh), f32.
#include "hf_fr.cuh"
namespace hfb {
int fr_f32(int which, int d, int p, const Params<float>& prm, const FrParams<float>& fp, float* uf, cudaStream_t st) {
    return run_fr_impl<float>(which, d, p, prm, fp, uf, st);
}
}  // namespace hfb
