// hf_unfused.cuh -- the unfused comparator: Table 1 stage 2 (pointwise flux),
// stage 3 (flux divergence) and stage 6 (source) as separate kernels, each a
// plain coalesced streaming kernel.  The reference only models their I/O
// (io_model.hpp:27-40: S2 reads n_v / writes d*n_v, S3 reads d*n_v / writes
// n_v, S6 reads n_v + d^2 / writes n_v).  They exist to measure the fused
// kernel's speed-up on the same hardware (BASELINE config 4).
//
// Flux workspace layout: the state's AoSoA layout with n_v replaced by d*n_v
// rows, row (a*n_v + v): ws[g*group*NP*d*NV + e_l + group*(pt + NP*(a*NV + v))].
#pragma once

#include "hf_common.cuh"

namespace hfb {

constexpr int kUnfusedBS = 256;

// Stage 2: F_a(U) at every point, all d*n_v entries (structural zeros included,
// as stage 2 writes d*n_v words per point in the model).
template <class R, int DIM, int M>
__global__ void __launch_bounds__(kUnfusedBS) hf_flux_kernel(const __grid_constant__ Params<R> p) {
    constexpr int NV = n_vars_c(DIM), NP = ipow_c(M, DIM);
    const long long g = blockIdx.x;
    const int G = p.group;
    const long long gwF = static_cast<long long>(G) * NP * DIM * NV;
    for (int rem = threadIdx.x; rem < G * NP; rem += kUnfusedBS) {
        const int pt = rem / G, el = rem - pt * G;
        if (g * G + el >= p.n_elem) continue;
        const R* __restrict__ u = p.u + g * p.group_words + el + static_cast<long long>(G) * pt;
        R* __restrict__ w = p.ws + g * gwF + el + static_cast<long long>(G) * pt;
        R s[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) s[v] = __ldcs(u + static_cast<long long>(G) * NP * v);
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            R f[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) f[v] = R(0);
            f[0] = p.zeta * s[1 + a];
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                const R gb = s[var_grad_c(DIM, b, a)];
                const R base = (a == b) ? fma(-p.nu, gb, s[0]) : (-p.nu) * gb;
                f[1 + b] = fma(s[1 + b], s[1 + a], base);
                f[var_grad_c(DIM, b, a)] = (-p.invT) * s[1 + b];
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) w[static_cast<long long>(G) * NP * (a * NV + v)] = f[v];
        }
    }
}

// Stage 3: -sum_a jac_a sum_t D(row_a, t) F_a(line point t), structural
// non-zeros only (oracle.hpp:36-50).  Neighbour re-reads hit L1/L2.
template <class R, int DIM, int M>
__global__ void __launch_bounds__(kUnfusedBS) hf_div_kernel(const __grid_constant__ Params<R> p) {
    constexpr int NV = n_vars_c(DIM), NP = ipow_c(M, DIM);
    const long long g = blockIdx.x;
    const int G = p.group;
    const long long gwF = static_cast<long long>(G) * NP * DIM * NV;
    for (int rem = threadIdx.x; rem < G * NP; rem += kUnfusedBS) {
        const int pt = rem / G, el = rem - pt * G;
        if (g * G + el >= p.n_elem) continue;
        const int ijk[3] = {pt % M, (pt / M) % M, DIM == 3 ? pt / (M * M) : 0};
        const R* __restrict__ w = p.ws + g * gwF + el;
        R acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = R(0);
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const int stride = (a == 0) ? 1 : (a == 1) ? M : M * M;
            const int row = ijk[a];
            const int pt0 = pt - row * stride;
            R s[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) s[v] = R(0);
#pragma unroll
            for (int t = 0; t < M; ++t) {
                const R c = p.D[row * M + t];
                const R* f = w + static_cast<long long>(G) * (pt0 + t * stride + NP * a * NV);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const bool nz = v <= DIM || ((v - 1 - DIM) % DIM == a);
                    if (nz) s[v] = fma(c, __ldg(f + static_cast<long long>(G) * NP * v), s[v]);
                }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const bool nz = v <= DIM || ((v - 1 - DIM) % DIM == a);
                if (nz) acc[v] = fma(p.jac[a], s[v], acc[v]);
            }
        }
        R* __restrict__ o = p.out + g * p.group_words + el + static_cast<long long>(G) * pt;
#pragma unroll
        for (int v = 0; v < NV; ++v) __stcs(o + static_cast<long long>(G) * NP * v, -acc[v]);
    }
}

// Stage 6: out += source(U): reads the divergence (n_v) and the d^2 gradient
// words of U, writes n_v (io_model.hpp:33).
template <class R, int DIM, int M>
__global__ void __launch_bounds__(kUnfusedBS) hf_source_kernel(const __grid_constant__ Params<R> p) {
    constexpr int NV = n_vars_c(DIM), NP = ipow_c(M, DIM);
    const long long g = blockIdx.x;
    const int G = p.group;
    for (int rem = threadIdx.x; rem < G * NP; rem += kUnfusedBS) {
        const int pt = rem / G, el = rem - pt * G;
        if (g * G + el >= p.n_elem) continue;
        const long long base = g * p.group_words + el + static_cast<long long>(G) * pt;
        R o[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) o[v] = __ldcs(p.out + base + static_cast<long long>(G) * NP * v);
#pragma unroll
        for (int v = 1 + DIM; v < NV; ++v)
            o[v] = fma(-p.invT, __ldcs(p.u + base + static_cast<long long>(G) * NP * v), o[v]);
#pragma unroll
        for (int v = 0; v < NV; ++v) __stcs(p.out + base + static_cast<long long>(G) * NP * v, o[v]);
    }
}

}  // namespace hfb
