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

#include "hf_chunk_io.cuh"
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

// Unrolling of the per-thread y loop (j): whole at low order, where the loop body is small
// and the interleaved iterations hide latency; rolled from m = 5, where the unrolled body's
// registers cap the resident warps (managed FP64, same box: p4 0.47 -> 0.59, p5 0.22 -> 0.34,
// p6 0.11 -> 0.16 of the roofline rolled; p3 0.83 unrolled vs 0.76 rolled).
template <int M>
inline constexpr int kPlanarJUnroll = M <= 4 ? M : 1;
// ... and of the unmanaged kernel's x loop (i): whole up to m = 3 (p1 FP64 0.76 rolled vs
// 0.997 unrolled), rolled above (p3 FP64 0.22 -> 0.40, p5 0.10 -> 0.17).
template <int M>
inline constexpr int kPlanarIUnroll = M <= 3 ? M : 1;

// Resident CTAs the unmanaged planar kernel is compiled for (__launch_bounds__ min blocks):
// registers capped near 128 per thread at p1-p3 (FP64 from p2) -- fully unrolled, the
// kernel takes 236-255 and runs 2 CTAs per SM.  Same box, 1e7 points (planar_ab/): FP32 p1
// 0.73 -> 0.79, p2 0.45 -> 0.51, p3 0.20 -> 0.29; FP64 p2 0.64 -> 0.74, p3 0.39 -> 0.41;
// FP64 p1 126 registers either way; a 96-register cap spills.
// (0 from p4: no constraint, the compiler's own register choice.)
template <class R, int M, int BS>
inline constexpr int kPlanarMinBlocks = M <= 4 ? (65536 / (128 * BS) > 1 ? 65536 / (128 * BS) : 1) : 0;

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
__global__ void __launch_bounds__(PlanarShape<R, M, NE>::BS, kPlanarMinBlocks<R, M, PlanarShape<R, M, NE>::BS>)
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

#pragma unroll(kPlanarIUnroll<M>)
    for (int i = 0; i < M; ++i) {
        // plane slice: y-line (i, *, kp) -> shared, and its y-line operands (P, V, the
        // y-gradient column: 7 of the 13 rows) -> registers
        R rY[M][7];
#pragma unroll
        for (int j = 0; j < M; ++j)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const R x = act ? __ldg(ub + gofs(i, j, kp, v)) : R(0);
                if (v < 4) rY[j][v] = x;
                else if ((v - 4) % 3 == 1) rY[j][4 + (v - 4) / 3] = x;
                myplane[NE * (v + NV * j)] = x;
            }
        __syncthreads();

#pragma unroll(kPlanarJUnroll<M>)
        for (int j = 0; j < M; ++j) {
            R tx[13], ty[13], tz[13];
            const R* __restrict__ own = myplane + NE * NV * j;  // this thread's point (i, j, kp)
            // x line from global (the i2 == i point from the thread's own plane slice)
#pragma unroll
            for (int i2 = 0; i2 < M; ++i2) {
                R P, V[3], Gc[3];
                if (i2 == i) {
                    P = own[0];
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        V[b] = own[NE * (1 + b)];
                        Gc[b] = own[NE * var_grad_c(3, b, 0)];
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
                const R Gc[3] = {rY[j2][4], rY[j2][5], rY[j2][6]};
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
                        if (v >= 4) o = fma(-p.invT, own[NE * v], o);
                    ob[gofs(i, j, kp, v)] = o;
                }
            }
        }
        if (i + 1 < M) __syncthreads();  // the next plane overwrites the buffer
    }
}

// ---------------------------------------------------------------------------------------------
// Managed planar (Method::PlanarManaged, codegen_planar.hpp:276-300 + the
// generation-time MemoryManager, memory_manager.hpp:57-191).
//
// The reference's manager is a greedy allocator: with enough shared capacity
// every operand the planar emitter requests -- the y-z plane slices (high
// priority) and the x-line neighbours (low priority, load_x_value :229-240) --
// ends up resident in shared memory, and global memory is read exactly once.
// On B200 the per-CTA capacity (227 KB) holds whole element chunks, so the
// managed kernel realises the manager's fixed point directly: the CTA's NE
// elements are staged into shared memory with cp.async.bulk (hf_chunk_io.cuh),
// and the planar algorithm (same thread mapping, same accumulation order, hence
// bit-identical results to hf_planar_kernel) reads its y-line, x-line and
// z-line operands from the staged chunk.  Outputs go straight to global memory
// (coalesced over the element index), so the staged input stays intact for
// the neighbouring threads.
// ---------------------------------------------------------------------------------------------
template <class R, int M, int NE>
struct PlanarManagedShape {
    static constexpr int NV = 13;
    static constexpr int NP = M * M * M;
    static constexpr int NT = NE * M;                // compute threads: (element, z-plane)
    static constexpr int BS = ((NT + 31) / 32) * 32;  // whole warps: the bulk copies are split over 32 lanes
    static constexpr int HDR = 128;
    static constexpr int IN_BYTES = NE * NP * NV * int(sizeof(R));
    using IO = ChunkIO<R, NE, NP * NV, IN_BYTES>;
    static constexpr size_t SMEM = HDR + size_t(IO::BUF_BYTES);
};

template <class R, int M, int NE, bool SRC>
__global__ void __launch_bounds__(PlanarManagedShape<R, M, NE>::BS)
    hf_planar_managed_kernel(const __grid_constant__ Params<R> p) {
    using S = PlanarManagedShape<R, M, NE>;
    using IO = typename S::IO;
    constexpr int NP = S::NP, NV = S::NV, BS = S::BS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* buf = smem_raw + S::HDR;

    const int tid = threadIdx.x;
    const long long E0 = static_cast<long long>(blockIdx.x) * NE;
    const long long grp = E0 / p.group;
    const int el0 = static_cast<int>(E0 - grp * p.group);
    const long long gbase = grp * p.group_words + el0;
    const bool contiguous = (p.group == NE);
    bool fast = p.fast_ok && E0 + NE <= p.n_elem;
    if (fast && contiguous)  // the 16-byte superset must stay inside the allocation
        fast = ((gbase + NE * NP * NV) * (long long)sizeof(R) + 15) / 16 * 16 <= p.total_words * (long long)sizeof(R);
    const int head = fast ? IO::head_bytes(p.u + gbase, contiguous) : 0;

    // ---------------- stage the chunk (the manager's resident set) ----------------
    if (fast) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid < 32) {
            if (tid == 0) mbar_arrive_expect_tx(bar, IO::tx_bytes(p.u + gbase, contiguous));
            __syncwarp();
            IO::load(buf, p.u + gbase, p.group, contiguous, bar, tid);
        }
        mbar_wait_parity(bar, 0);
    } else {
        R* s0 = reinterpret_cast<R*>(buf);
        for (int idx = tid; idx < NE * NP * NV; idx += BS) {
            const long long e = E0 + idx % NE;
            R v = R(0);
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                v = ld_stream(p.u + ge * p.group_words + (e - ge * p.group) + static_cast<long long>(p.group) * (idx / NE));
            }
            s0[idx] = v;
        }
        __syncthreads();
    }
    const R* __restrict__ s = reinterpret_cast<const R*>(buf + head);
    if (tid >= S::NT) return;  // padding lanes of the last warp only help staging

    const int el = tid % NE;
    const int kp = tid / NE;
    const long long e = E0 + el;
    const bool act = e < p.n_elem;
    const long long ge = act ? e / p.group : 0;
    R* __restrict__ ob = p.out + ge * p.group_words + (e - ge * p.group);
    const long long G = p.group;
    auto sofs = [&](int i, int j, int k, int v) -> int { return el + NE * (i + M * j + M * M * k + NP * v); };
    auto gofs = [&](int i, int j, int k, int v) -> long long {
        return G * static_cast<long long>(i + M * j + M * M * k + NP * v);
    };

    R rDz[M];
#pragma unroll
    for (int t = 0; t < M; ++t) rDz[t] = p.D[kp * M + t];

#pragma unroll 1
    for (int i = 0; i < M; ++i) {
        // plane slice: the y-line (i, *, kp) operands P, V and the y-gradient column
        // (high-priority request, :118-131) -- 7 of the 13 rows
        R rY[M][7];
#pragma unroll
        for (int j = 0; j < M; ++j) {
#pragma unroll
            for (int v = 0; v < 4; ++v) rY[j][v] = s[sofs(i, j, kp, v)];
#pragma unroll
            for (int b = 0; b < 3; ++b) rY[j][4 + b] = s[sofs(i, j, kp, var_grad_c(3, b, 1))];
        }
#pragma unroll(kPlanarJUnroll<M>)
        for (int j = 0; j < M; ++j) {
            R tx[13], ty[13], tz[13];
#pragma unroll
            for (int i2 = 0; i2 < M; ++i2) {  // x line: resident neighbours (load_x_value, :229-240)
                R P, V[3], Gc[3];
                P = s[sofs(i2, j, kp, 0)];
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    V[b] = s[sofs(i2, j, kp, 1 + b)];
                    Gc[b] = s[sofs(i2, j, kp, var_grad_c(3, b, 0))];
                }
                accumulate_column<R, 0>(tx, i2 == 0, p.D[i * M + i2], P, V, Gc, p);
            }
#pragma unroll
            for (int j2 = 0; j2 < M; ++j2) {  // y line from registers
                const R V[3] = {rY[j2][1], rY[j2][2], rY[j2][3]};
                const R Gc[3] = {rY[j2][4], rY[j2][5], rY[j2][6]};
                accumulate_column<R, 1>(ty, j2 == 0, p.D[j * M + j2], rY[j2][0], V, Gc, p);
            }
#pragma unroll
            for (int k2 = 0; k2 < M; ++k2) {  // z line from the resident plane
                const R V[3] = {s[sofs(i, j, k2, 1)], s[sofs(i, j, k2, 2)], s[sofs(i, j, k2, 3)]};
                const R Gc[3] = {s[sofs(i, j, k2, var_grad_c(3, 0, 2))], s[sofs(i, j, k2, var_grad_c(3, 1, 2))],
                                 s[sofs(i, j, k2, var_grad_c(3, 2, 2))]};
                accumulate_column<R, 2>(tz, k2 == 0, rDz[k2], s[sofs(i, j, k2, 0)], V, Gc, p);
            }
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
                        if (v >= 4) o = fma(-p.invT, s[sofs(i, j, kp, v)], o);
                    ob[gofs(i, j, kp, v)] = o;
                }
            }
        }
    }
}

}  // namespace hfb
