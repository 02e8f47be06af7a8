// hf_planar.cuh -- the planar fused flux + divergence kernel (Alg. 1,
// codegen_planar.hpp:97-210) for sm_100a, d = 3.
//
// One thread per (element, z-plane kp); the thread walks x = i = 0..m-1:
//   * the y-line (i, *, kp) of all n_v variables is loaded from global into
//     registers rY[j][v] and mirrored into the y-z plane buffer in shared
//     memory (codegen_planar.hpp:113-139);
//   * x-lines (i2, j, kp) are read from global memory through the read-only
//     L1 path (:145-158); the i2 == i point comes from registers
//     (register_overlap, acceptance.cpp:375-402: p+1 reads per value);
//   * y-lines come from registers (:159-167);
//   * z-lines come from the shared plane buffer after one CTA barrier per
//     plane (:168-180; the reference re-barriers per j, which is redundant);
//   * the flux column of every neighbour is re-evaluated per line with the
//     reference's accumulation order (codegen_util.hpp:149-209), combined
//     per axis (:237-253) and written with the optional source (:181-191).
// Fully unrolled per order.  Threads are laid out element-fastest so every
// global access is a contiguous run of NE words (AoSoA, layout.hpp:128-134),
// and the plane buffer's kp stride is padded so the kp-strided stores are
// bank-conflict free (the banks.hpp:110-120 deconfliction, done statically).
#pragma once

#include "hf_common.cuh"

namespace hfb {

template <class R, int M, int NE>
struct PlanarShape {
    static constexpr int NV = 13;
    static constexpr int NP = M * M * M;
    static constexpr int BS = NE * M;
    static constexpr int BANKW = sizeof(R) == 4 ? 32 : 16;  // words per conflict-free wavefront
    static constexpr int KS0 = NE * NV * M;                  // natural kp stride (words)
    // smallest stride >= KS0 with KS == NE (mod BANKW): lanes (e_l, kp) tile the banks
    static constexpr int KS = KS0 + (((NE % BANKW) - (KS0 % BANKW)) % BANKW + BANKW) % BANKW;
    static constexpr size_t SMEM = size_t(KS) * M * sizeof(R);
};

// Running accumulators per output row (codegen_util.hpp:149-161): first
// contribution is a multiply, later ones fused multiply-adds.
template <class R>
__device__ __forceinline__ void acc_row(R& acc, bool first, R coef, R f) {
    acc = first ? coef * f : fma(coef, f, acc);
}

// Flux column `axis` of one point folded into the 13 row accumulators
// (codegen_util.hpp:177-209), only over the structural non-zeros
// (equations.hpp:97-103).
template <class R, int AXIS>
__device__ __forceinline__ void accumulate_column(R (&acc)[13], bool first, R coef, R P, const R (&V)[3],
                                                  const R (&G)[3], const Params<R>& p) {
    // continuity: zeta * V_a
    acc_row(acc[0], first, coef, p.zeta * V[AXIS]);
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        const R base = (b == AXIS) ? fma(-p.nu, G[b], P) : (-p.nu) * G[b];
        acc_row(acc[1 + b], first, coef, fma(V[b], V[AXIS], base));
    }
#pragma unroll
    for (int b = 0; b < 3; ++b) acc_row(acc[var_grad_c(3, b, AXIS)], first, coef, (-p.invT) * V[b]);
}

template <class R, int M, int NE, bool SRC>
__global__ void __launch_bounds__(PlanarShape<R, M, NE>::BS)
    hf_planar_kernel(const __grid_constant__ Params<R> p) {
    using S = PlanarShape<R, M, NE>;
    constexpr int NP = S::NP, NV = S::NV, KS = S::KS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    R* plane = reinterpret_cast<R*>(smem_raw);  // [kp][j][v][e_l], kp stride KS

    const int tid = threadIdx.x;
    const int el = tid % NE;
    const int kp = tid / NE;
    const long long e = static_cast<long long>(blockIdx.x) * NE + el;
    const bool act = e < p.n_elem;
    const long long ge = act ? e / p.group : 0;
    const R* __restrict__ ub = p.u + ge * p.group_words + (e - ge * p.group);
    R* __restrict__ ob = p.out + ge * p.group_words + (e - ge * p.group);
    const long long G = p.group;
    auto gofs = [&](int i, int j, int k, int v) -> long long {
        return G * static_cast<long long>(i + M * j + M * M * k + NP * v);
    };

    R rDz[M];
#pragma unroll
    for (int t = 0; t < M; ++t) rDz[t] = p.D[kp * M + t];

    R* __restrict__ myplane = plane + KS * kp + el;

#pragma unroll
    for (int i = 0; i < M; ++i) {
        // plane slice: y-line (i, *, kp) -> registers + shared
        R rY[M][NV];
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const R x = act ? __ldg(ub + gofs(i, j, kp, v)) : R(0);
                rY[j][v] = x;
                myplane[NE * (v + NV * j)] = x;
            }
        __syncthreads();

#pragma unroll
        for (int j = 0; j < M; ++j) {
            R tx[13], ty[13], tz[13];
            // x line from global (the i2 == i point from registers)
#pragma unroll
            for (int i2 = 0; i2 < M; ++i2) {
                R P, V[3], Gc[3];
                if (i2 == i) {
                    P = rY[j][0];
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        V[b] = rY[j][1 + b];
                        Gc[b] = rY[j][var_grad_c(3, b, 0)];
                    }
                } else {
                    P = act ? __ldg(ub + gofs(i2, j, kp, 0)) : R(0);
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        V[b] = act ? __ldg(ub + gofs(i2, j, kp, 1 + b)) : R(0);
                        Gc[b] = act ? __ldg(ub + gofs(i2, j, kp, var_grad_c(3, b, 0))) : R(0);
                    }
                }
                accumulate_column<R, 0>(tx, i2 == 0, p.D[i * M + i2], P, V, Gc, p);
            }
            // y line from registers
#pragma unroll
            for (int j2 = 0; j2 < M; ++j2) {
                const R V[3] = {rY[j2][1], rY[j2][2], rY[j2][3]};
                const R Gc[3] = {rY[j2][var_grad_c(3, 0, 1)], rY[j2][var_grad_c(3, 1, 1)],
                                 rY[j2][var_grad_c(3, 2, 1)]};
                accumulate_column<R, 1>(ty, j2 == 0, p.D[j * M + j2], rY[j2][0], V, Gc, p);
            }
            // z line from the shared y-z plane (only P, V, z-gradient column: zcol_needs :225-228)
#pragma unroll
            for (int k2 = 0; k2 < M; ++k2) {
                const R* q = plane + KS * k2 + el + NE * NV * j;
                const R V[3] = {q[NE * 1], q[NE * 2], q[NE * 3]};
                const R Gc[3] = {q[NE * var_grad_c(3, 0, 2)], q[NE * var_grad_c(3, 1, 2)],
                                 q[NE * var_grad_c(3, 2, 2)]};
                accumulate_column<R, 2>(tz, k2 == 0, rDz[k2], q[0], V, Gc, p);
            }
            // combine (codegen_util.hpp:237-253), negate, source, store
            if (act) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const bool hx = v <= 3 || (v >= 4 && (v - 4) % 3 == 0);
                    const bool hy = v <= 3 || (v >= 4 && (v - 4) % 3 == 1);
                    const bool hz = v <= 3 || (v >= 4 && (v - 4) % 3 == 2);
                    R r = R(0);
                    bool have = false;
                    if (hx) { r = p.jac[0] * tx[v]; have = true; }
                    if (hy) { r = have ? fma(p.jac[1], ty[v], r) : p.jac[1] * ty[v]; have = true; }
                    if (hz) { r = have ? fma(p.jac[2], tz[v], r) : p.jac[2] * tz[v]; }
                    R o = -r;
                    if constexpr (SRC)
                        if (v >= 4) o = fma(-p.invT, rY[j][v], o);
                    ob[gofs(i, j, kp, v)] = o;
                }
            }
        }
        if (i + 1 < M) __syncthreads();  // the next plane overwrites the buffer
    }
}

}  // namespace hfb
