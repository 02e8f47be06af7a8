// hf_fr.cuh -- the FR stages either side of the fused kernel (Table 1,
// stages 1, 4, 5), on a periodic structured mesh with the
// reference's constant per-axis Jacobian.  EXTENSION beyond the reference,
// which models only their I/O; oracle: hfo_project_faces /
// hfo_fr_correct / hfo_fr_residual (oracle/hexfuse_oracle.c).
//
//   stage 1  hf_fr_project_kernel: each CTA stages a chunk of NE elements
//            (bulk copy, as the lines kernel) and extrapolates every a-line of
//            every variable to xi_a = -1, +1 (Lagrange basis at +-1) -> U_f.
//   stage 4+5 hf_fr_correct_kernel: per element, the common flux at both ends
//            of every line (own U_f against the neighbour's; PAPER.md:856:
//            Rusanov on the pressure / velocity rows with the inviscid wave
//            speed |V_a| + sqrt(V_a^2 + zeta), the mean of both sides on the
//            gradient rows of the hyperbolic diffusion), the jumps
//            F^I - F_a(U_f) into shared memory, then per solution point
//            out -= sum_a jac_a (g_L'(xi) jump_(-a) + g_R'(xi) jump_(+a)) over the
//            fused kernel's -div^D (+ source) in place.
//
// Face layout (AoSoA, the field's group; L = m^(d-1)):
//     word (e, a, s, l, v) = (e/group)*group*2*d*L*n_v + e%group + group*(l + L*(s + 2*(a + d*v))).
// Multi-GPU: a rank owns whole element layers (ex, ey planes of the mesh);
// the faces of the layers just below / above its slab arrive as ghost arrays
// (same layout, one layer each) through NCCL (multi_gpu.FrSlab).
#pragma once

#include <cstdlib>

#include "hf_launch.cuh"
#include "hf_lines.cuh"

namespace hfb {

struct FrMesh {
    int dims[3];         // elements per axis (dims[2] = 1 for d = 2)
    long long e_begin;   // first (global) element of this partition
    long long n_local;   // elements of this partition (whole layers unless single-partition)
    long long layer;     // elements per ghost layer (dims[0] * dims[1] for d = 3, dims[0] for d = 2)
};

template <class R>
struct FrParams {
    R lm[kMaxM], lp[kMaxM];  // Lagrange basis at xi = -1, +1
    R gl[kMaxM], gr[kMaxM];  // g_L'(x_i), g_R'(x_i) of the DG correction functions
    FrMesh mesh;
    const R* __restrict__ uf;       // local faces
    const R* __restrict__ ghost_lo;  // faces of the layer below the partition (or nullptr)
    const R* __restrict__ ghost_hi;  // faces of the layer above
};

template <int DIM, int M>
__host__ __device__ constexpr int fr_lines() {
    return ipow_c(M, DIM - 1);
}

// ---------------------------------------------------------------------------------------------
// stage 1
// ---------------------------------------------------------------------------------------------
template <class R, int DIM, int M, int NE>
struct FrProjShape {
    using L = LinesShape<R, DIM, M, NE>;
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int BS = L::BS;
    static constexpr int HDR = 128;
    static constexpr size_t SMEM = HDR + size_t(L::BUF_BYTES);
};

template <class R, int DIM, int M, int NE>
__global__ void __launch_bounds__(FrProjShape<R, DIM, M, NE>::BS)
    hf_fr_project_kernel(const __grid_constant__ Params<R> p, const __grid_constant__ FrParams<R> f, R* __restrict__ uf) {
    using S = FrProjShape<R, DIM, M, NE>;
    using L = typename S::L;
    using IO = typename L::IO;
    constexpr int BS = S::BS, NV = S::NV, NP = L::NP, LN = fr_lines<DIM, M>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* buf = smem_raw + S::HDR;
    const int tid = threadIdx.x;
    const long long E0 = static_cast<long long>(blockIdx.x) * NE;
    const long long grp = E0 / p.group;
    const long long gbase = grp * p.group_words + (E0 - grp * p.group);
    const bool contiguous = (p.group == NE);
    const bool fast = chunk_bulk_ok<R, L::IN_WORDS>(p, gbase, E0 + NE <= p.n_elem, contiguous);
    const int head = fast ? IO::head_bytes(p.u + gbase, contiguous) : 0;
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
        for (int idx = tid; idx < L::IN_WORDS; idx += BS) {
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
    const R* s = reinterpret_cast<const R*>(buf + head);
    // one task = (element, line, axis): both ends of the line for every variable (the
    // index arithmetic is paid once per line), stores coalesced over the element
    for (int task = tid; task < NE * LN * DIM; task += BS) {
        const int el = task % NE;
        const int l = (task / NE) % LN;
        const int a = task / (NE * LN);
        const long long e = E0 + el;
        if (e >= p.n_elem) continue;
        int pt[M];
#pragma unroll
        for (int t = 0; t < M; ++t) pt[t] = el + NE * fr_line_point<DIM, M>(a, l, t);
        const long long ge = e / p.group;
        R* ub = uf + ge * p.group * 2 * DIM * LN * NV + (e - ge * p.group) + (long long)p.group * (l + LN * 2 * a);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            R sm = R(0), sp = R(0);
#pragma unroll
            for (int t = 0; t < M; ++t) {
                const R u = s[pt[t] + NE * NP * v];
                sm = fma(f.lm[t], u, sm);
                sp = fma(f.lp[t], u, sp);
            }
            R* q = ub + (long long)p.group * LN * 2 * DIM * v;  // face_word(e, a, s, l, v)
            q[0] = sm;
            q[(long long)p.group * LN] = sp;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// stages 4 + 5
// ---------------------------------------------------------------------------------------------
// Locate the faces of global element eg: local buffer, or a ghost layer.
template <class R>
__device__ __forceinline__ const R* fr_faces_of(const FrParams<R>& f, long long eg, long long n_mesh, long long* e_loc) {
    const FrMesh& ms = f.mesh;
    long long rel = eg - ms.e_begin;
    if (rel < 0) rel += n_mesh;
    if (rel < ms.n_local) {
        *e_loc = rel;
        return f.uf;
    }
    if (rel < ms.n_local + ms.layer) {  // the layer above the partition
        *e_loc = rel - ms.n_local;
        return f.ghost_hi;
    }
    *e_loc = rel - (n_mesh - ms.layer);  // the layer below (wrapped)
    return f.ghost_lo;
}

template <class R, int DIM, int M, int NE>
struct FrCorrShape {
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int LN = fr_lines<DIM, M>();
    static constexpr int TASKS = NE * DIM * LN;  // (element, axis, line)
    // one thread per stage-4 task of an axis (NE * LN * 2: one round per axis, no
    // tail before the barrier); FP32 also at least one per two stage-5 points;
    // whole warps, 64..512
    static constexpr int T4 = NE * LN * 2, T5 = (NE * ipow_c(M, DIM) + 1) / 2;
    static constexpr int T = ((sizeof(R) == 8 || T4 > T5 ? T4 : T5) + 31) / 32 * 32;
    static constexpr int BS = T < 64 ? 64 : (T > 512 ? 512 : T);
    static constexpr size_t SMEM = size_t(TASKS) * 2 * NV * sizeof(R);  // jumps [v][s][a][l][el]
};

// Row V of the normal flux F_A (equations.hpp:70-83): zeta V_A on P,
// V_b V_A - nu g(b,A) (+P if b == A) on momentum b, -V_b/T on g(b,A), 0 elsewhere.
template <class R, int DIM, int A, int V>
__device__ __forceinline__ R fr_flux_row(const R (&U)[n_vars_c(DIM)], const Params<R>& p) {
    if constexpr (V == 0) {
        return p.zeta * U[1 + A];
    } else if constexpr (V <= DIM) {
        constexpr int b = V - 1;
        const R mom = U[1 + b] * U[1 + A] - p.nu * U[var_grad_c(DIM, b, A)];
        return (b == A) ? mom + U[0] : mom;
    } else {
        constexpr int b = (V - 1 - DIM) / DIM, c = (V - 1 - DIM) % DIM;
        if constexpr (c == A) return -U[1 + b] * p.invT;
        else return R(0);
    }
}

template <class R, int DIM, int A>
__device__ __forceinline__ R fr_wavespeed(const R (&U)[n_vars_c(DIM)], const Params<R>& p) {
    const R Va = U[1 + A];
    return fabs(Va) + sqrt(Va * Va + p.zeta);  // inviscid ACM spectral radius
}

// Jumps F^I - F_A(U_own) at both ends of one A-line, into the shared jump array.
template <class R, int DIM, int M, int NE, int A, int V = 0>
__device__ __forceinline__ void fr_jump_rows(const R (&Uo)[n_vars_c(DIM)], const R (&Un)[n_vars_c(DIM)], R lam,
                                             int s, const Params<R>& p, R* __restrict__ jrow) {
    if constexpr (V < n_vars_c(DIM)) {
        constexpr int LN = fr_lines<DIM, M>();
        const R fo = fr_flux_row<R, DIM, A, V>(Uo, p), fn = fr_flux_row<R, DIM, A, V>(Un, p);
        // U_L / U_R in the +x_A orientation of the face: own state is U_L on the +A face (s = 1)
        // Rusanov on the hyperbolic rows, the mean on the gradient rows
        R FI = R(0.5) * (fo + fn);
        if constexpr (V < 1 + DIM) FI -= R(0.5) * lam * (s ? (Un[V] - Uo[V]) : (Uo[V] - Un[V]));
        jrow[NE * LN * DIM * 2 * V] = FI - fo;
        fr_jump_rows<R, DIM, M, NE, A, V + 1>(Uo, Un, lam, s, p, jrow);
    }
}

// Element-local word offset of the AoSoA layouts: (e/group)*group*words + e%group.
__device__ __forceinline__ long long fr_elem_base(long long e, long long group, long long words_per_elem) {
    const long long g = e / group;
    return g * group * words_per_elem + (e - g * group);
}

template <class R, int DIM, int M, int NE>
__global__ void __launch_bounds__(FrCorrShape<R, DIM, M, NE>::BS)
    hf_fr_correct_kernel(const __grid_constant__ Params<R> p, const __grid_constant__ FrParams<R> f) {
    using S = FrCorrShape<R, DIM, M, NE>;
    constexpr int NV = S::NV, LN = S::LN, BS = S::BS, NP = ipow_c(M, DIM), FW = 2 * DIM * LN * NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    R* jump = reinterpret_cast<R*>(smem_raw);  // [v][s][a][l][el]
    // per element: own faces, the 2*DIM neighbour faces it meets (face (A, 1-s) of the
    // neighbour across side s of axis A) and its output words -- the 64-bit mesh and
    // group arithmetic once per element, 32-bit offsets in the task loops
    __shared__ const R* own_f[NE];
    __shared__ const R* nbr_f[NE][DIM][2];
    __shared__ R* out_e[NE];
    auto jidx = [](int el, int a, int s, int l, int v) { return el + NE * (l + LN * (a + DIM * (s + 2 * v))); };
    const int tid = threadIdx.x;
    const long long E0 = static_cast<long long>(blockIdx.x) * NE;
    const int ne = int(p.n_elem - E0 < NE ? p.n_elem - E0 : NE);
    const int G = int(p.group);
    const int VS = G * 2 * DIM * LN;  // face word stride between variables

    for (int q = tid; q < ne * 2 * DIM; q += BS) {
        const int el = q % ne, side = q / ne, A = side >> 1, s = side & 1;
        const long long e = E0 + el;
        const long long eg = f.mesh.e_begin + e;
        const long long nx = f.mesh.dims[0], ny = f.mesh.dims[1];
        const long long n_mesh = nx * ny * (DIM == 3 ? f.mesh.dims[2] : 1);
        long long c[3] = {eg % nx, (eg / nx) % ny, DIM == 3 ? eg / (nx * ny) : 0};
        c[A] = (c[A] + (s ? 1 : -1) + f.mesh.dims[A]) % f.mesh.dims[A];
        const long long en = c[0] + nx * (c[1] + ny * c[2]);
        long long enl;
        const R* nb = fr_faces_of(f, en, n_mesh, &enl);
        nbr_f[el][A][s] = nb + fr_elem_base(enl, G, FW) + (long long)G * LN * (1 - s + 2 * A);
        if (side == 0) {
            own_f[el] = f.uf + fr_elem_base(e, G, FW);
            out_e[el] = p.out + fr_elem_base(e, G, NP * NV);
        }
    }
    __syncthreads();

    // ---- stage 4: common fluxes and jumps at both ends of every line (axis unrolled)
    auto stage4 = [&](auto a_tag) {
        constexpr int A = decltype(a_tag)::value;
        for (int task = tid; task < NE * LN * 2; task += BS) {
            const int el = task % NE;
            const int l = (task / NE) % LN;
            const int s = task / (NE * LN);
            if (el >= ne) continue;
            const R* ow = own_f[el] + G * (l + LN * (s + 2 * A));
            const R* nw = nbr_f[el][A][s] + G * l;
            R Uo[NV], Un[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                Uo[v] = ow[VS * v];
                Un[v] = nw[VS * v];
            }
            const R lam = fmax(fr_wavespeed<R, DIM, A>(Uo, p), fr_wavespeed<R, DIM, A>(Un, p));
            fr_jump_rows<R, DIM, M, NE, A>(Uo, Un, lam, s, p, jump + jidx(el, A, s, l, 0));
        }
    };
    stage4(std::integral_constant<int, 0>{});
    stage4(std::integral_constant<int, 1>{});
    if constexpr (DIM == 3) stage4(std::integral_constant<int, 2>{});
    __syncthreads();

    // ---- stage 5: corrections at every solution point, over the fused kernel's result;
    // two points per thread and iteration, all 2 n_v loads in flight before the updates
    // (FP64 p4: 822 -> 753 us, FP32 p4: 434 -> 335 us)
    auto point = [&](int task, R (&cur)[NV], bool load) {
        const int el = task % NE;
        const int pt = task / NE;
        if (task >= NE * NP || el >= ne) return;
        R* ob = out_e[el] + G * pt;
        if (load) {
#pragma unroll
            for (int v = 0; v < NV; ++v) cur[v] = ob[G * NP * v];
            return;
        }
        const int i = pt % M, j = (pt / M) % M, k = pt / (M * M);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            R corr = R(0);
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const int t = a == 0 ? i : (a == 1 ? j : k);
                const int l = a == 0 ? (j + M * k) : (a == 1 ? (i + M * k) : (i + M * j));
                corr = fma(p.jac[a], fma(f.gl[t], jump[jidx(el, a, 0, l, v)], f.gr[t] * jump[jidx(el, a, 1, l, v)]), corr);
            }
            ob[G * NP * v] = cur[v] - corr;
        }
    };
    // (one point per iteration for FP32 blocks above 256 threads: the second point's
    // registers would cost a resident CTA -- p6 FP32: 92 registers, 336 -> 488 us)
    constexpr int ILP = (sizeof(R) == 8 || BS <= 256) ? 2 : 1;
    for (int task = tid; task < NE * NP; task += ILP * BS) {
        R c0[NV], c1[NV];
        point(task, c0, true);
        if constexpr (ILP == 2) point(task + BS, c1, true);
        point(task, c0, false);
        if constexpr (ILP == 2) point(task + BS, c1, false);
    }
}


// ---------------------------------------------------------------------------------------------
// stages 4 + 5, staged form: the residual chunk is bulk-copied into shared memory while
// stage 4 loads the faces; per axis one thread per (element, A-line) computes both line-end
// jumps in registers and applies out(t) -= jac_A (g_L'(x_t) jump_- + g_R'(x_t) jump_+) to the
// staged chunk (lines of one axis are disjoint; one barrier between axes); bulk copy out.
// Selected per (d, p, precision) where it beats hf_fr_correct_kernel (fr_correct_staged()).
// ---------------------------------------------------------------------------------------------
template <class R, int DIM, int M, int NE>
struct FrCorrStagedShape {
    using L = LinesShape<R, DIM, M, NE>;
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int LN = fr_lines<DIM, M>();
    static constexpr int T = (NE * LN + 31) / 32 * 32;
    static constexpr int BS = T < 64 ? 64 : T;
    static constexpr int HDR = 128;
    static constexpr size_t SMEM = HDR + size_t(L::BUF_BYTES);
};

template <class R, int DIM, int A, int V = 0>
__device__ __forceinline__ void fr_jump_regs(const R (&Uo)[n_vars_c(DIM)], const R (&Un)[n_vars_c(DIM)], R lam, int s,
                                             const Params<R>& p, R (&j)[n_vars_c(DIM)]) {
    if constexpr (V < n_vars_c(DIM)) {
        const R fo = fr_flux_row<R, DIM, A, V>(Uo, p), fn = fr_flux_row<R, DIM, A, V>(Un, p);
        // Rusanov on the hyperbolic rows, the mean on the gradient rows
        R FI = R(0.5) * (fo + fn);
        if constexpr (V < 1 + DIM) FI -= R(0.5) * lam * (s ? (Un[V] - Uo[V]) : (Uo[V] - Un[V]));
        j[V] = FI - fo;
        fr_jump_regs<R, DIM, A, V + 1>(Uo, Un, lam, s, p, j);
    }
}

// Stages 4+5 on a chunk of NE elements resident in shared memory (layout [v][pt][el], the
// elements E0 .. E0+ne-1): per axis one thread per (element, A-line) loads the own and the
// neighbour face values at both line ends (the neighbour's from f.uf or a ghost layer),
// forms the jumps F^I - F_A(U_own) in registers and applies
// out(t) -= jac_A (g_L'(x_t) jump_- + g_R'(x_t) jump_+) in place, one axis after the other.
// `before_update` runs once per thread ahead of its first shared-memory update (the staged
// correction kernel waits there for its chunk).  Ends with a CTA barrier.
// SH: the chunk's shared-memory layout (LinesShape; the padded layouts of lines variants 25-27
// included) -- word offsets of the line points and variables come from it.
template <class R, int DIM, int M, int NE, int BS, class SH = LinesShape<R, DIM, M, NE>, class Before>
__device__ __forceinline__ void fr_correct_smem(R* __restrict__ sm, const Params<R>& p, const FrParams<R>& f,
                                                long long E0, int ne, int tid, Before&& before_update) {
    constexpr int NV = n_vars_c(DIM), LN = fr_lines<DIM, M>(), NP = ipow_c(M, DIM), FW = 2 * DIM * LN * NV;
    __shared__ const R* own_f[NE];
    __shared__ const R* nbr_f[NE][DIM][2];
    const int G = int(p.group);
    const int VS = G * 2 * DIM * LN;
    for (int q = tid; q < ne * 2 * DIM; q += BS) {
        const int el = q % ne, side = q / ne, A = side >> 1, s = side & 1;
        const long long e = E0 + el;
        const long long eg = f.mesh.e_begin + e;
        const long long nx = f.mesh.dims[0], ny = f.mesh.dims[1];
        const long long n_mesh = nx * ny * (DIM == 3 ? f.mesh.dims[2] : 1);
        long long cx = eg % nx, cy = (eg / nx) % ny, cz = DIM == 3 ? eg / (nx * ny) : 0;
        const int step = s ? 1 : -1;
        if (A == 0) cx = (cx + step + nx) % nx;
        else if (A == 1) cy = (cy + step + ny) % ny;
        else cz = (cz + step + f.mesh.dims[2]) % f.mesh.dims[2];
        const long long en = cx + nx * (cy + ny * cz);
        long long enl;
        const R* nb = fr_faces_of(f, en, n_mesh, &enl);
        nbr_f[el][A][s] = nb + fr_elem_base(enl, G, FW) + (long long)G * LN * (1 - s + 2 * A);
        if (side == 0) own_f[el] = f.uf + fr_elem_base(e, G, FW);
    }
    __syncthreads();
    bool waited = false;
    auto axis = [&](auto a_tag) {
        constexpr int A = decltype(a_tag)::value;
        for (int task = tid; task < NE * LN; task += BS) {
            const int el = task % NE;
            const int l = task / NE;
            if (el >= ne) continue;
            R jm[NV], jp[NV];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const R* ow = own_f[el] + G * (l + LN * (s + 2 * A));
                const R* nw = nbr_f[el][A][s] + G * l;
                R Uo[NV], Un[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    Uo[v] = ow[VS * v];
                    Un[v] = nw[VS * v];
                }
                const R lam = fmax(fr_wavespeed<R, DIM, A>(Uo, p), fr_wavespeed<R, DIM, A>(Un, p));
                if (s == 0) fr_jump_regs<R, DIM, A>(Uo, Un, lam, 0, p, jm);
                else fr_jump_regs<R, DIM, A>(Uo, Un, lam, 1, p, jp);
            }
            if (!waited) {
                before_update();
                waited = true;
            }
            R* ln = sm + SH::word(el, fr_line_point<DIM, M>(A, l, 0), 0);
            constexpr int TS = SH::template step<A>();
            const R ja = p.jac[A];
#pragma unroll
            for (int t = 0; t < M; ++t) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    R* q = ln + TS * t + SH::VS * v;
                    *q = *q - ja * fma(f.gl[t], jm[v], f.gr[t] * jp[v]);
                }
            }
        }
        __syncthreads();
    };
    axis(std::integral_constant<int, 0>{});
    axis(std::integral_constant<int, 1>{});
    if constexpr (DIM == 3) axis(std::integral_constant<int, 2>{});
}

// Stages 2+3+6 and 4+5 in one pass (hf_fr_residual): the lines kernel's chunk, after the
// sweeps, gets the interface correction in shared memory and leaves it once -- the residual
// is written once instead of written, read back and rewritten by a second kernel.  The faces
// (stage 1) come from a projection launched just before (hf_fr_project_kernel).
template <class R, int DIM, int M, int NE, bool SRC, int XP = 0>
__global__ void __launch_bounds__(LinesShape<R, DIM, M, NE, 1, NE, false, XP>::BS)
    hf_lines_fr_kernel(const __grid_constant__ Params<R> p, const __grid_constant__ FrParams<R> f) {
    using SH = LinesShape<R, DIM, M, NE, 1, NE, false, XP>;
    constexpr int BS = SH::BS;
    auto hook = [&](R* sm, long long E0, int nvalid, int tid) {
        const long long left = p.n_elem - E0;
        const int ne = int(left < nvalid ? left : nvalid);
        fr_correct_smem<R, DIM, M, NE, BS, SH>(sm, p, f, E0, ne, tid, [] {});
    };
    lines_chunk<R, DIM, M, NE, SRC, 1, false, NE, false, decltype(hook)&, XP>(p, hook);
}

template <class R, int DIM, int M, int NE>
__global__ void __launch_bounds__(FrCorrStagedShape<R, DIM, M, NE>::BS)
    hf_fr_correct_staged_kernel(const __grid_constant__ Params<R> p, const __grid_constant__ FrParams<R> f) {
    using S = FrCorrStagedShape<R, DIM, M, NE>;
    using L = typename S::L;
    using IO = typename L::IO;
    constexpr int BS = S::BS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* buf = smem_raw + S::HDR;
    const int tid = threadIdx.x;
    const long long E0 = static_cast<long long>(blockIdx.x) * NE;
    const int ne = int(p.n_elem - E0 < NE ? p.n_elem - E0 : NE);
    const long long grp = E0 / p.group;
    const long long gbase = grp * p.group_words + (E0 - grp * p.group);
    const bool contiguous = (p.group == NE);
    const bool fast = chunk_bulk_ok<R, L::IN_WORDS>(p, gbase, E0 + NE <= p.n_elem, contiguous);
    const int head = fast ? IO::head_bytes(p.out + gbase, contiguous) : 0;

    if (fast) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid < 32) {
            if (tid == 0) mbar_arrive_expect_tx(bar, IO::tx_bytes(p.out + gbase, contiguous));
            __syncwarp();
            IO::load(buf, p.out + gbase, p.group, contiguous, bar, tid);
        }
    } else {
        R* s0 = reinterpret_cast<R*>(buf);
        for (int idx = tid; idx < L::IN_WORDS; idx += BS) {
            const long long e = E0 + idx % NE;
            R v = R(0);
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                v = p.out[ge * p.group_words + (e - ge * p.group) + static_cast<long long>(p.group) * (idx / NE)];
            }
            s0[idx] = v;
        }
    }
    fr_correct_smem<R, DIM, M, NE, BS>(reinterpret_cast<R*>(buf + head), p, f, E0, ne, tid, [&] {
        if (fast) mbar_wait_parity(bar, 0);  // the chunk has landed (overlapped with the face loads)
    });

    if (fast) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid < 32) {
            IO::store(p.out + gbase, buf, p.group, contiguous, tid);
            bulk_wait_read_all();
        }
    } else {
        const R* s0 = reinterpret_cast<const R*>(buf);
        for (int idx = tid; idx < L::IN_WORDS; idx += BS) {
            const long long e = E0 + idx % NE;
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                p.out[ge * p.group_words + (e - ge * p.group) + static_cast<long long>(p.group) * (idx / NE)] = s0[idx];
            }
        }
    }
}

}  // namespace hfb

// ---------------------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------------------
namespace hfb {

template <class R, int DIM, int M>
constexpr int fr_proj_ne() {
    int ne = 32;  // power of two, <= 72 KB of staged chunk
    while (ne > 1 && (size_t(ne) * ipow_c(M, DIM) * n_vars_c(DIM) * sizeof(R) > size_t(72 * 1024) ||
                      ne * ipow_c(M, DIM - 1) > 512))
        ne /= 2;
    return ne;
}

// power of two elements per CTA, <= KB kilobytes of jumps
template <class R, int DIM, int M, int KB>
constexpr int fr_corr_ne() {
    int ne = 32;
    while (ne > 1 && size_t(ne) * DIM * ipow_c(M, DIM - 1) * 2 * n_vars_c(DIM) * sizeof(R) > size_t(KB * 1024)) ne /= 2;
    return ne;
}

template <class R, int DIM, int M, int NE>
int fr_project_launch(const Params<R>& prm, const FrParams<R>& fp, R* uf, cudaStream_t st) {
    using S = FrProjShape<R, DIM, M, NE>;
    auto kernel = hf_fr_project_kernel<R, DIM, M, NE>;
    Params<R> p = prm;
    p.fast_ok = (p.group == NE || (p.group % NE == 0 && (NE * sizeof(R)) % 16 == 0 &&
                                   ((long long)p.group * sizeof(R)) % 16 == 0)) &&
                (reinterpret_cast<uintptr_t>(p.u) & 15u) == 0;
    if (S::SMEM > 40 * 1024) {  // (static shared memory counts against the default 48 KB)
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return int(e);
    }
    kernel<<<unsigned((p.n_elem + NE - 1) / NE), S::BS, S::SMEM, st>>>(p, fp, uf);
    return int(cudaGetLastError());
}

// Stage 1 stages whole chunks with bulk copies when the chunk is the AoSoA group
// (or whole 16-byte rows of it): the chunk size follows the caller's group.
template <class R, int DIM, int M, int NE = fr_proj_ne<R, DIM, M>()>
int fr_project_dispatch(const Params<R>& prm, const FrParams<R>& fp, R* uf, cudaStream_t st) {
    if constexpr (NE > 1) {
        if (prm.group != NE && prm.group % NE != 0) return fr_project_dispatch<R, DIM, M, NE / 2>(prm, fp, uf, st);
    }
    return fr_project_launch<R, DIM, M, NE>(prm, fp, uf, st);
}

template <class R, int DIM, int M, int NE>
int fr_correct_launch(const Params<R>& prm, const FrParams<R>& fp, cudaStream_t st) {
    using S = FrCorrShape<R, DIM, M, NE>;
    auto kernel = hf_fr_correct_kernel<R, DIM, M, NE>;
    if (S::SMEM > 40 * 1024) {  // (static shared memory counts against the default 48 KB)
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return int(e);
    }
    kernel<<<unsigned((prm.n_elem + NE - 1) / NE), S::BS, S::SMEM, st>>>(prm, fp);
    return int(cudaGetLastError());
}

template <class R, int DIM, int M, int NE>
int fr_correct_staged_launch(const Params<R>& prm, const FrParams<R>& fp, cudaStream_t st) {
    using S = FrCorrStagedShape<R, DIM, M, NE>;
    auto kernel = hf_fr_correct_staged_kernel<R, DIM, M, NE>;
    Params<R> p = prm;
    p.fast_ok = (p.group == NE || (p.group % NE == 0 && (NE * sizeof(R)) % 16 == 0 &&
                                   ((long long)p.group * sizeof(R)) % 16 == 0)) &&
                (reinterpret_cast<uintptr_t>(p.out) & 15u) == 0;
    if (S::SMEM > 40 * 1024) {  // (static shared memory counts against the default 48 KB)
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
        if (e != cudaSuccess) return int(e);
    }
    kernel<<<unsigned((p.n_elem + NE - 1) / NE), S::BS, S::SMEM, st>>>(p, fp);
    return int(cudaGetLastError());
}

// the chunk follows the caller's AoSoA group (bulk path), <= 72 KB, as stage 1
template <class R, int DIM, int M, int NE = fr_proj_ne<R, DIM, M>()>
int fr_correct_staged_dispatch(const Params<R>& prm, const FrParams<R>& fp, cudaStream_t st) {
    if constexpr (NE > 1) {
        if (prm.group != NE && prm.group % NE != 0) return fr_correct_staged_dispatch<R, DIM, M, NE / 2>(prm, fp, st);
    }
    return fr_correct_staged_launch<R, DIM, M, NE>(prm, fp, st);
}

// The one-chunk lines variant the fused residual kernel uses: the selected variant when it is
// a one-chunk form (a component-split one maps to its base chunk), else variant 0.
template <class R, int DIM, int M>
constexpr int fr_fused_variant() {
    for (const SelRow& r : kSelect)
        if (r.d == DIM && r.p == M - 1 && r.prec == (sizeof(R) == 8 ? 1 : 0) && r.method == 2) {
            if (is_one_chunk_variant(r.variant)) return r.variant;
            if (r.variant == 19) return 0;
            if (r.variant == 20) return 1;
            if (r.variant == 21) return 2;
            if (r.variant == 22) return 7;
            if (is_xpad_variant(r.variant)) return r.variant;  // the one-pass kernel runs padded too
        }
    return 0;
}

template <class R, int DIM, int M, int NE, bool SRC, int XP = 0>
int lines_fr_launch(Params<R> p, const FrParams<R>& f, cudaStream_t st) {
    using S = LinesShape<R, DIM, M, NE, 1, NE, false, XP>;
    if constexpr (XP > 0) {  // padded chunk (launch_lines): the group is the chunk, maps encoded
        if (!setup_xpad<R, DIM, M, NE, S>(p)) return lines_fr_launch<R, DIM, M, NE, SRC, 0>(p, f, st);
        p.fast_ok = 1;
        auto kernel = hf_lines_fr_kernel<R, DIM, M, NE, SRC, XP>;
        if (int e = set_smem_attr(kernel, S::SMEM)) return e;
        return int(launch_kernel(kernel, dim3(unsigned((p.n_elem + NE - 1) / NE)), dim3(S::BS), S::SMEM, st, p, f));
    }
    auto kernel = hf_lines_fr_kernel<R, DIM, M, NE, SRC>;
    const bool tile = tile_layout<R, NE>(p.group) && aligned16(p.u) && aligned16(p.out);
    const long long n_groups = (p.n_elem + p.group - 1) / p.group;
    const int sub = (p.group + NE - 1) / NE;
    const long long grid = tile ? n_groups * sub : (p.n_elem + NE - 1) / NE;
    p.fast_ok = (tile || bulk_layout<R, NE>(p.group)) && aligned16(p.u) && aligned16(p.out);
    if (tile) {
        p.tile = 1;
        p.sub_per_group = sub;
        if (!encode_chunk_map<R>(&p.tm_u, p.u, DIM, M, p.group, n_groups, NE) ||
            !encode_chunk_map<R>(&p.tm_out, p.out, DIM, M, p.group, n_groups, NE))
            p.fast_ok = 0;
    }
    if (int e = set_smem_attr(kernel, S::SMEM)) return e;
    return int(launch_kernel(kernel, dim3(unsigned(grid)), dim3(S::BS), S::SMEM, st, p, f));
}

// (d, p, precision) where the one-pass residual (projection, then the lines kernel with the
// correction in shared memory) beats the pair (lines kernel with the faces, then the
// correction kernel).  Decided under sustained (power-capped) load with the one-pass kernel
// on the selected chunk, padded where the selection pads (profiles/r02/fr_sustained/: every
// stage 0.5 s back to back, HF_FR_FUSED=1 / 0 alternating, two rounds): the one-pass form
// wins everywhere (1.01-1.22x) but at d3 FP32 p2, where the pair is 4.7 % ahead.
template <class R, int DIM, int M>
constexpr bool fr_residual_fused() {
    return !(DIM == 3 && sizeof(R) == 4 && M == 3);
}

template <class R, int DIM, int M>
int lines_fr_dispatch(const Params<R>& prm, const FrParams<R>& fp, bool src, cudaStream_t st) {
    constexpr int V = fr_fused_variant<R, DIM, M>();
    constexpr int NE = variant_ne<R, DIM, M, V>();
    constexpr int XP = is_xpad_variant(V) && NE >= 1 ? xpad_code<R, DIM, M, (NE >= 1 ? NE : 1)>() : 0;
    if constexpr (NE < 1 || LinesShape<R, DIM, M, NE, 1, NE, false, XP>::SMEM > size_t(kMaxSmemPerCta)) {
        return -1;
    } else {
        return src ? lines_fr_launch<R, DIM, M, NE, true, XP>(prm, fp, st)
                   : lines_fr_launch<R, DIM, M, NE, false, XP>(prm, fp, st);
    }
}

template <class R, int DIM, int M>
int fr_correct_dispatch_jumps(const Params<R>& prm, const FrParams<R>& fp, cudaStream_t st);

// (d, p, precision) where the staged correction wins by > 7 % (same box, 1e7 points,
// profiles/ext_r01f_fr_staged_{jumps,staged}.jsonl): d2 FP32 p2-p8 (1.09-1.38x), d2 FP64
// p4-p5 (1.24-1.27x), d3 FP32 p2 and p5 (1.39x, 1.19x); elsewhere the jump-array kernel
template <class R, int DIM, int M>
constexpr bool fr_correct_staged() {
    if constexpr (DIM == 2) return sizeof(R) == 4 ? M >= 3 : (M == 5 || M == 6);
    else return sizeof(R) == 4 && (M == 3 || M == 6);
}

template <class R, int DIM, int M>
int fr_stage(int which, const Params<R>& prm, const FrParams<R>& fp, R* uf, cudaStream_t st) {
    if (which == 5) return fr_residual_fused<R, DIM, M>() ? 1 : 0;
    if (prm.n_elem == 0) return 0;
    if (which == 1) return fr_project_dispatch<R, DIM, M>(prm, fp, uf, st);
    if (which == 3 || which == 4) return lines_fr_dispatch<R, DIM, M>(prm, fp, which == 4, st);  // 4: with source
    if (which == 5) return fr_residual_fused<R, DIM, M>() ? 1 : 0;  // query: the one-pass residual is preferred
#ifdef HF_FR_AB
    if (const char* ev = std::getenv("HF_FR_STAGED"))
        return ev[0] == '1' ? fr_correct_staged_dispatch<R, DIM, M>(prm, fp, st)
                            : fr_correct_dispatch_jumps<R, DIM, M>(prm, fp, st);
#endif
    if constexpr (fr_correct_staged<R, DIM, M>()) return fr_correct_staged_dispatch<R, DIM, M>(prm, fp, st);
    return fr_correct_dispatch_jumps<R, DIM, M>(prm, fp, st);
}

template <class R, int DIM, int M>
int fr_correct_dispatch_jumps(const Params<R>& prm, const FrParams<R>& fp, cudaStream_t st) {
    // <= 48 KB of jumps per CTA (occupancy), or <= 96 KB when the AoSoA group is at
    // least that many elements, so that stage 5's point loads cover whole 32-byte
    // sectors and rows (p6: FP32 486 -> 336 us, FP64 832 -> 744 us; p1 FP64, group 64:
    // 1297 -> 1091 us; a larger chunk with a smaller group only costs occupancy:
    // p4 FP64 822 -> 978 us)
    constexpr int NE1 = fr_corr_ne<R, DIM, M, 48>(), NE2 = fr_corr_ne<R, DIM, M, 96>();
    if constexpr (NE2 > NE1) {
        if (prm.group >= NE2) return fr_correct_launch<R, DIM, M, NE2>(prm, fp, st);
    }
    return fr_correct_launch<R, DIM, M, NE1>(prm, fp, st);
}


template <class R>
int run_fr_impl(int which, int d, int p, const Params<R>& prm, const FrParams<R>& fp, R* uf, cudaStream_t st) {
    if (d == 3) {
        switch (p) {
            case 1: return fr_stage<R, 3, 2>(which, prm, fp, uf, st);
            case 2: return fr_stage<R, 3, 3>(which, prm, fp, uf, st);
            case 3: return fr_stage<R, 3, 4>(which, prm, fp, uf, st);
            case 4: return fr_stage<R, 3, 5>(which, prm, fp, uf, st);
            case 5: return fr_stage<R, 3, 6>(which, prm, fp, uf, st);
            case 6: return fr_stage<R, 3, 7>(which, prm, fp, uf, st);
            case 7: return fr_stage<R, 3, 8>(which, prm, fp, uf, st);
            default: return -1;
        }
    }
    switch (p) {
        case 1: return fr_stage<R, 2, 2>(which, prm, fp, uf, st);
        case 2: return fr_stage<R, 2, 3>(which, prm, fp, uf, st);
        case 3: return fr_stage<R, 2, 4>(which, prm, fp, uf, st);
        case 4: return fr_stage<R, 2, 5>(which, prm, fp, uf, st);
        case 5: return fr_stage<R, 2, 6>(which, prm, fp, uf, st);
        case 6: return fr_stage<R, 2, 7>(which, prm, fp, uf, st);
        case 7: return fr_stage<R, 2, 8>(which, prm, fp, uf, st);
        case 8: return fr_stage<R, 2, 9>(which, prm, fp, uf, st);
        default: return -1;
    }
}

int fr_f32(int which, int d, int p, const Params<float>&, const FrParams<float>&, float*, cudaStream_t);
int fr_f64(int which, int d, int p, const Params<double>&, const FrParams<double>&, double*, cudaStream_t);

}  // namespace hfb
