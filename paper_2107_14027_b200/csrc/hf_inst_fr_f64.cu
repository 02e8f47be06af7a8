// Instantiation unit: FR stages 1 and 4+5 (hf_fr.cuh), f64.
#include "hf_fr.cuh"
namespace hfb {
int fr_f64(int which, int d, int p, const Params<double>& prm, const FrParams<double>& fp, double* uf, cudaStream_t st) {
    return run_fr_impl<double>(which, d, p, prm, fp, uf, st);
}
}  // namespace hfb
