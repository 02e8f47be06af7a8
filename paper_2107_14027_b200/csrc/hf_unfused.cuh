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

// Stage 3 as per-axis line contractions over staged flux blocks ("divergence matmuls",
// BASELINE config 4): the flux workspace of one group is d direction blocks F_a, each
// one contiguous range of G * NP * NV words ([v][pt][e_l]).  A persistent CTA streams
// the blocks (chunk c = one group, direction a) of its groups through a two-stage
// cp.async.bulk ring (the load of block k+1 is in flight while block k is contracted),
// each thread owns up to ITEMS (point, element) outputs and accumulates
// jac_a * sum_t D(row, t) F_a(line point t) over the structural rows in registers, and
// writes -acc (+ nothing else: stage 6 adds the source) once per group, coalesced.
// HBM traffic = d*n_v words read + n_v written per point: io_model S3 (io_model.hpp:32).
template <class R, int DIM, int M, int ITEMS>
struct DivStagedShape {
    static constexpr int NV = n_vars_c(DIM), NP = ipow_c(M, DIM);
    static constexpr int BS = 256;
    static constexpr int HDR = 128;  // two mbarriers
};

template <class R, int DIM, int M, int ITEMS>
__global__ void __launch_bounds__(256) hf_div_staged_kernel(const __grid_constant__ Params<R> p) {
    using S = DivStagedShape<R, DIM, M, ITEMS>;
    constexpr int NV = S::NV, NP = S::NP, BS = S::BS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    const int G = p.group;
    const int blk_words = G * NP * NV;                       // one direction block of one group
    const int blk_bytes = blk_words * int(sizeof(R));
    const int stage_bytes = (blk_bytes + 127) / 128 * 128;
    unsigned char* stage0 = smem_raw + S::HDR;
    const long long n_groups = (p.n_elem + G - 1) / G;
    const long long gwF = static_cast<long long>(G) * NP * DIM * NV;
    const int tid = threadIdx.x;
    // this CTA's groups: c = blockIdx.x + i * gridDim.x; blocks k = i * DIM + a
    const long long my_groups = blockIdx.x < n_groups ? (n_groups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long n_blocks = my_groups * DIM;
    auto src_of = [&](long long k) {
        const long long c = blockIdx.x + (k / DIM) * gridDim.x;
        const int a = static_cast<int>(k % DIM);
        return p.ws + c * gwF + static_cast<long long>(a) * blk_words;
    };
    auto issue = [&](long long k, int st) {  // one thread
        mbar_arrive_expect_tx(&full[st], uint32_t(blk_bytes));
        const unsigned char* src = reinterpret_cast<const unsigned char*>(src_of(k));
        for (int off = 0; off < blk_bytes; off += 65536) {
            const int n = blk_bytes - off < 65536 ? blk_bytes - off : 65536;
            bulk_g2s(stage0 + st * stage_bytes + off, src + off, n, &full[st]);
        }
    };
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        if (n_blocks > 0) issue(0, 0);
        if (n_blocks > 1) issue(1, 1);
    }
    R acc[ITEMS][NV];
    for (long long k = 0; k < n_blocks; ++k) {
        const int st = static_cast<int>(k & 1);
        const int a = static_cast<int>(k % DIM);
        const long long c = blockIdx.x + (k / DIM) * gridDim.x;
        mbar_wait_parity(&full[st], static_cast<uint32_t>((k >> 1) & 1));
        const R* F = reinterpret_cast<const R*>(stage0 + st * stage_bytes);
        const int stride = (a == 0) ? 1 : (a == 1) ? M : M * M;
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const int item = tid + it * BS;  // item = el + G * pt
            if (a == 0) {
#pragma unroll
                for (int v = 0; v < NV; ++v) acc[it][v] = R(0);
            }
            if (item < G * NP) {
                const int pt = item / G, el = item - pt * G;
                const int ijk = a == 0 ? pt % M : a == 1 ? (pt / M) % M : pt / (M * M);
                const R* f0 = F + el + G * (pt - ijk * stride);
                const R ja = p.jac[a];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    // structural rows of column a (equations.hpp:97-103): P, V, and g(b, a)
                    if (v > DIM && (v - 1 - DIM) % DIM != a) continue;
                    R sacc = R(0);
#pragma unroll
                    for (int t = 0; t < M; ++t) sacc = fma(p.D[ijk * M + t], f0[G * (t * stride + NP * v)], sacc);
                    acc[it][v] = fma(ja, sacc, acc[it][v]);
                }
                if (a == DIM - 1) {
                    const long long e = c * G + el;
                    if (e < p.n_elem) {
                        R* o = p.out + c * p.group_words + el + static_cast<long long>(G) * pt;
#pragma unroll
                        for (int v = 0; v < NV; ++v) __stcs(o + static_cast<long long>(G) * NP * v, -acc[it][v]);
                    }
                }
            }
        }
        __syncthreads();  // every thread is done with stage st
        if (tid == 0 && k + 2 < n_blocks) issue(k + 2, st);
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
