// hf_lines.cuh -- the higher-parallelism ("lines") fused flux + divergence
// kernel for sm_100a.  B200 redesign of the reference's lines method
// (codegen_lines.hpp:143-262, Alg. 2): threads are split across the
// tensor-product lines of an element, and every solution point's flux column
// is evaluated exactly once per direction.
//
// One CTA owns a chunk of NE consecutive elements.
//
//   1. The chunk (NE * m^d * n_v words) is staged into shared memory with
//      cp.async.bulk (TMA bulk copies completing on one mbarrier).  When the
//      AoSoA group equals NE the chunk is one contiguous byte range of the
//      field (layout.hpp:128-134).
//   2. d sweeps, one per axis a.  In sweep a each thread owns one a-line
//      (element, two fixed indices) and holds, in registers, the m values of
//      V_b and of the momentum flux M_ba = V_b V_a + P delta_ab - nu g(b,a)
//      (equations.hpp:70-83) along its line.  The line derivative is then an
//      m x m register contraction with D rows taken from the parameter
//      constant bank -- no shared-memory re-reads per neighbour.
//        out[g(b,a)]  = (jac_a / T) (D V_b)                 [final in sweep a]
//                       (- g(b,a)/T with the source, equations.hpp:87-94)
//        cont partial += jac_a (D V_a)          -> out[P]  = -zeta * sum
//        mom_b partial += jac_a (D M_ba)        -> out[V_b] = -sum
//      The 1+d partials cross sweeps through a small shared accumulator
//      region; gradient outputs overwrite their own (dead) input slot in place.
//   3. After the last sweep the shared chunk holds the finished divergence in
//      the global layout; one set of bulk stores writes it back.
//
// HBM traffic is therefore exactly the algorithmic minimum (io_model Fused23,
// io_model.hpp:35): n_v words read and n_v words written per point.
//
// Partial chunks (the last group of a field, or layouts whose group/alignment
// rule out bulk copies) take a guarded LDG/STS + LDS/STG path in the same
// kernel; padding elements are neither read nor written (render.hpp:95,102).
#pragma once

#include "hf_common.cuh"

namespace hfb {

template <class R, int DIM, int M, int NE>
struct LinesShape {
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int NP = ipow_c(M, DIM);
    static constexpr int LINES = NE * ipow_c(M, DIM - 1);
    static constexpr int BS = ((LINES + 31) / 32) * 32 < 64 ? 64 : ((LINES + 31) / 32) * 32;
    static constexpr int NACC = 1 + DIM;  // continuity + d momentum partials
    static constexpr int IN_WORDS = NE * NP * NV;
    static constexpr int ACC_WORDS = NE * NP * NACC;
    static constexpr int HDR = 128;  // mbarrier + alignment pad
    static constexpr size_t SMEM = HDR + size_t(IN_WORDS + ACC_WORDS) * sizeof(R);
    static constexpr int IN_BYTES = IN_WORDS * int(sizeof(R));
    static constexpr int ROW_BYTES = NE * int(sizeof(R));
};

// One sweep along axis A.  PHASE: 0 = first sweep, 1 = middle, 2 = last.
template <class R, int DIM, int M, int NE, bool SRC, int A, int PHASE>
__device__ __forceinline__ void lines_sweep(R* __restrict__ s, R* __restrict__ acc, const Params<R>& p, int L) {
    using S = LinesShape<R, DIM, M, NE>;
    constexpr int NP = S::NP;
    constexpr int VS = NE * NP;  // word stride between variables
    constexpr int STRIDE = (A == 0) ? 1 : (A == 1) ? M : M * M;  // point stride along the line

    const int el = L % NE;
    const int r = L / NE;
    int base_pt;
    if constexpr (DIM == 3) {
        if constexpr (A == 0) base_pt = M * r;  // r = j + M k  ->  M j + M^2 k
        else if constexpr (A == 1) base_pt = (r % M) + M * M * (r / M);  // r = i + M k
        else base_pt = r;  // r = i + M j
    } else {
        if constexpr (A == 0) base_pt = M * r;  // r = j
        else base_pt = r;  // r = i
    }
    R* __restrict__ sb = s + el + NE * base_pt;
    R* __restrict__ ab = acc + el + NE * base_pt;

    const R nu = p.nu;
    R V[DIM][M];
    R Q[DIM][M];
#pragma unroll
    for (int t = 0; t < M; ++t) {
        const R* q = sb + NE * STRIDE * t;
        const R P = q[0];
#pragma unroll
        for (int b = 0; b < DIM; ++b) V[b][t] = q[VS * (1 + b)];
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
            const R g = q[VS * var_grad_c(DIM, b, A)];
            // codegen_util.hpp:191-202 operation order: base, then fma(V_b, V_a, base)
            const R base = (b == A) ? fma(-nu, g, P) : (-nu) * g;
            Q[b][t] = fma(V[b][t], V[A][t], base);
        }
    }

#pragma unroll
    for (int i = 0; i < M; ++i) {
        R dV[DIM], dQ[DIM];
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
            dV[b] = p.D[i * M] * V[b][0];
            dQ[b] = p.D[i * M] * Q[b][0];
        }
#pragma unroll
        for (int t = 1; t < M; ++t) {
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                dV[b] = fma(p.D[i * M + t], V[b][t], dV[b]);
                dQ[b] = fma(p.D[i * M + t], Q[b][t], dQ[b]);
            }
        }
        R* q = sb + NE * STRIDE * i;
        R* a = ab + NE * STRIDE * i;
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
            R o = p.jac_invT[A] * dV[b];
            if constexpr (SRC) o = fma(-p.invT, q[VS * var_grad_c(DIM, b, A)], o);
            q[VS * var_grad_c(DIM, b, A)] = o;
        }
        const R c = p.jac[A] * dV[A];
        if constexpr (PHASE == 0) {
            a[0] = c;
#pragma unroll
            for (int b = 0; b < DIM; ++b) a[VS * (1 + b)] = p.jac[A] * dQ[b];
        } else if constexpr (PHASE == 1) {
            a[0] = a[0] + c;
#pragma unroll
            for (int b = 0; b < DIM; ++b) a[VS * (1 + b)] = fma(p.jac[A], dQ[b], a[VS * (1 + b)]);
        } else {
            q[0] = -(p.zeta * (a[0] + c));
#pragma unroll
            for (int b = 0; b < DIM; ++b) q[VS * (1 + b)] = -fma(p.jac[A], dQ[b], a[VS * (1 + b)]);
        }
    }
}

template <class R, int DIM, int M, int NE, bool SRC>
__global__ void __launch_bounds__(LinesShape<R, DIM, M, NE>::BS)
    hf_lines_kernel(const __grid_constant__ Params<R> p) {
    using S = LinesShape<R, DIM, M, NE>;
    constexpr int BS = S::BS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    R* s = reinterpret_cast<R*>(smem_raw + S::HDR);
    R* acc = s + S::IN_WORDS;

    const int tid = threadIdx.x;
    const long long E0 = (p.chunk0 + static_cast<long long>(blockIdx.x)) * NE;
    const bool fast = p.fast_ok && (E0 + NE <= p.n_elem);
    const long long grp = E0 / p.group;
    const int el0 = static_cast<int>(E0 - grp * p.group);
    const long long gbase = grp * p.group_words + el0;

    // ---------------- stage the chunk into shared memory ----------------
    if (fast) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid < 32) {
            if (tid == 0) mbar_arrive_expect_tx(bar, S::IN_BYTES);
            __syncwarp();
            if (p.group == NE) {
                // contiguous chunk: split into 32 near-equal 16B-multiple pieces
                constexpr int PIECE = ((S::IN_BYTES / 32 + 15) / 16) * 16;
                const int off = tid * PIECE;
                if (off < S::IN_BYTES) {
                    const int len = (S::IN_BYTES - off) < PIECE ? (S::IN_BYTES - off) : PIECE;
                    bulk_g2s(reinterpret_cast<unsigned char*>(s) + off,
                             reinterpret_cast<const unsigned char*>(p.u + gbase) + off, len, bar);
                }
            } else {
                // one row per (point, variable): NE contiguous words at stride `group`
                for (int row = tid; row < S::NP * S::NV; row += 32)
                    bulk_g2s(s + NE * row, p.u + gbase + static_cast<long long>(p.group) * row, S::ROW_BYTES, bar);
            }
        }
        mbar_wait_parity(bar, 0);
    } else {
        for (int idx = tid; idx < S::IN_WORDS; idx += BS) {
            const int el = idx % NE;
            const int row = idx / NE;
            const long long e = E0 + el;
            R v = R(0);
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                v = ld_stream(p.u + ge * p.group_words + (e - ge * p.group) + static_cast<long long>(p.group) * row);
            }
            s[idx] = v;
        }
        __syncthreads();
    }

    // ---------------- d sweeps ----------------
    constexpr int LINES = S::LINES;
    if constexpr (DIM == 3) {
        for (int L = tid; L < LINES; L += BS) lines_sweep<R, 3, M, NE, SRC, 0, 0>(s, acc, p, L);
        __syncthreads();
        for (int L = tid; L < LINES; L += BS) lines_sweep<R, 3, M, NE, SRC, 1, 1>(s, acc, p, L);
        __syncthreads();
        for (int L = tid; L < LINES; L += BS) lines_sweep<R, 3, M, NE, SRC, 2, 2>(s, acc, p, L);
    } else {
        for (int L = tid; L < LINES; L += BS) lines_sweep<R, 2, M, NE, SRC, 0, 0>(s, acc, p, L);
        __syncthreads();
        for (int L = tid; L < LINES; L += BS) lines_sweep<R, 2, M, NE, SRC, 1, 2>(s, acc, p, L);
    }

    // ---------------- write the finished chunk ----------------
    if (fast) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid < 32) {
            if (p.group == NE) {
                constexpr int PIECE = ((S::IN_BYTES / 32 + 15) / 16) * 16;
                const int off = tid * PIECE;
                if (off < S::IN_BYTES) {
                    const int len = (S::IN_BYTES - off) < PIECE ? (S::IN_BYTES - off) : PIECE;
                    bulk_s2g(reinterpret_cast<unsigned char*>(p.out + gbase) + off,
                             reinterpret_cast<const unsigned char*>(s) + off, len);
                }
            } else {
                for (int row = tid; row < S::NP * S::NV; row += 32)
                    bulk_s2g(p.out + gbase + static_cast<long long>(p.group) * row, s + NE * row, S::ROW_BYTES);
            }
            bulk_commit();
            bulk_wait_read_all();
        }
    } else {
        __syncthreads();
        for (int idx = tid; idx < S::IN_WORDS; idx += BS) {
            const int el = idx % NE;
            const int row = idx / NE;
            const long long e = E0 + el;
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                p.out[ge * p.group_words + (e - ge * p.group) + static_cast<long long>(p.group) * row] = s[idx];
            }
        }
    }
}

}  // namespace hfb
