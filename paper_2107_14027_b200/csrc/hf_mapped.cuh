// hf_mapped.cuh -- fused flux + divergence on elements with a non-constant
// Jacobian (bi/trilinear "linear" elements given by their 2^d corners).
//
// EXTENSION beyond the reference, which fixes a constant per-axis Jacobian
// (oracle.hpp:47).  PAPER.md:1111 names the next step:
// "linear elements, for which only the locations of the element corners need
// to be loaded".  Conservative FR form, collocated at the solution points
// (oracle: hfo_oracle_divergence_mapped, oracle/hexfuse_oracle.c):
//
//     out = -(1/|J|) sum_a D_a ( sum_b S_ab F_b )  (+ source),   S = adj(J) = |J| J^-1.
//
// With G_a = sum_b S_ab F_b (the contravariant flux) the rows are, per point,
//     continuity     zeta * W_a,                       W_a = sum_b S_ab V_b
//     momentum c     V_c W_a + S_ac P - nu sum_b S_ab g(c,b)
//     gradient (c,b) -S_ab V_c / T
// so unlike the constant-Jacobian kernel every output row receives a
// contribution from every sweep, and the metric varies along the line.
//
// One CTA per chunk of NE elements (hf_lines.cuh's staging):
//   1. U chunk -> shared (cp.async.bulk), the chunk's corners -> shared;
//   2. d sweeps, thread per a-line (bank-conflict-free LineMap order); row a
//      of S along the line from the corners (LineMetric: no stored metric); batch 0
//      contracts the 1+d continuity/momentum lines, then d batches of d
//      gradient lines S_ab V_c; partial sums of all n_v rows accumulate in a
//      shared region (n_v words/pt);
//   3. the last sweep finishes each point: out = -acc/|J| (+ -g/T) over the staged
//      input (|J| = row A of adj(J) . column A of J, the column constant along the line);
//      bulk store.
// HBM traffic stays n_v words in + n_v out per point plus 2^d d words per
// element of geometry.
#pragma once

#include "hf_lines.cuh"

namespace hfb {

template <class R, int DIM, int M, int NE>
struct MappedShape {
    using L = LinesShape<R, DIM, M, NE>;
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int NP = ipow_c(M, DIM);
    static constexpr int NC = 1 << DIM;  // corners
    static constexpr int BS = L::BS;
    static constexpr int HDR = 128;
    static constexpr size_t ACC_OFF = HDR + size_t(L::BUF_BYTES);
    static constexpr size_t GEO_OFF = ((ACC_OFF + size_t(NV) * NP * NE * sizeof(R) + 15) / 16) * 16;
    static constexpr size_t SMEM = GEO_OFF + size_t(NC) * DIM * NE * sizeof(R);
};

// adj(J) (row-major) and det(J) of the map at one point.
template <class R, int DIM>
__device__ __forceinline__ R mapped_adjugate(const R (&J)[DIM * DIM], R (&S)[DIM * DIM]) {
    if constexpr (DIM == 2) {
        S[0] = J[3];
        S[1] = -J[1];
        S[2] = -J[2];
        S[3] = J[0];
        return J[0] * J[3] - J[1] * J[2];
    } else {
        S[0] = J[4] * J[8] - J[5] * J[7];
        S[1] = J[2] * J[7] - J[1] * J[8];
        S[2] = J[1] * J[5] - J[2] * J[4];
        S[3] = J[5] * J[6] - J[3] * J[8];
        S[4] = J[0] * J[8] - J[2] * J[6];
        S[5] = J[2] * J[3] - J[0] * J[5];
        S[6] = J[3] * J[7] - J[4] * J[6];
        S[7] = J[1] * J[6] - J[0] * J[7];
        S[8] = J[0] * J[4] - J[1] * J[3];
        return J[0] * S[0] + J[1] * S[3] + J[2] * S[6];
    }
}

// The (bi/tri)linear map in monomial form: X(xi) = sum_k a_k prod_{i in k} xi_i
// over the 2^d axis subsets k, with a_k = 2^-d sum_c (-1)^popc(k & ~c) X_c (corner
// c at xi_i = bit i of c ? +1 : -1).  Converted once per element in shared memory
// ([k][x][el], in place of the corners), so that a Jacobian column costs 2^(d-1)
// FMAs per coordinate instead of 2^d corner shape-function derivatives.
template <class R, int DIM, int NE, int BS>
__device__ __forceinline__ void mapped_corners_to_monomials(R* __restrict__ geo, int tid) {
    constexpr int NC = 1 << DIM;
    for (int q = tid; q < DIM * NE; q += BS) {
        const int el = q % NE, x = q / NE;
        R X[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) X[c] = geo[el + NE * (x + DIM * c)];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            R a = R(0);
#pragma unroll
            for (int c = 0; c < NC; ++c) a = (__popc(k & ~c) & 1) ? a - X[c] : a + X[c];
            geo[el + NE * (x + DIM * k)] = a * (R(1) / R(NC));
        }
    }
}

// Column j of J = dx/dxi at reference point xi from the monomial coefficients:
// sum over subsets k containing j of a_k prod_{i in k, i != j} xi_i.
template <class R, int DIM, int NE>
__device__ __forceinline__ void mapped_jcol(const R* __restrict__ geo, int el, int j, const R (&xi)[3], R (&col)[DIM]) {
#pragma unroll
    for (int i = 0; i < DIM; ++i) col[i] = R(0);
#pragma unroll
    for (int k = 0; k < (1 << DIM); ++k) {
        if (!((k >> j) & 1)) continue;
        R mono = R(1);
        bool one = true;
#pragma unroll
        for (int i = 0; i < DIM; ++i)
            if (i != j && ((k >> i) & 1)) {
                mono = one ? xi[i] : mono * xi[i];
                one = false;
            }
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            const R a = geo[el + NE * (i + DIM * k)];
            col[i] = one ? col[i] + a : fma(a, mono, col[i]);
        }
    }
}

// Row A of adj(J) along one A-line.  The J columns transverse to A are linear
// in xi_A along the line (the map is (bi/tri)linear), so the thread evaluates
// them at xi_A = 0 and 1 once (P, P + Q) and the row at line point t is a
// cross product of P + xi_t Q terms: no per-point metric storage.
template <class R, int DIM, int NE, int A>
struct LineMetric {
    R P[DIM - 1][DIM], Q[DIM - 1][DIM];
    __device__ __forceinline__ LineMetric(const R* __restrict__ geo, int el, R (&xi)[3]) {
#pragma unroll
        for (int q = 0; q < DIM - 1; ++q) {
            const int b = (A + 1 + q) % DIM;
            R c0[DIM], c1[DIM];
            xi[A] = R(0);
            mapped_jcol<R, DIM, NE>(geo, el, b, xi, c0);
            xi[A] = R(1);
            mapped_jcol<R, DIM, NE>(geo, el, b, xi, c1);
#pragma unroll
            for (int i = 0; i < DIM; ++i) {
                P[q][i] = c0[i];
                Q[q][i] = c1[i] - c0[i];
            }
        }
    }
    // S(A, .) at xi_A = x
    __device__ __forceinline__ void row(R x, R (&Sa)[DIM]) const {
        if constexpr (DIM == 3) {
            R u[3], w[3];  // columns A+1, A+2: adj row A = col(A+1) x col(A+2)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                u[i] = fma(x, Q[0][i], P[0][i]);
                w[i] = fma(x, Q[1][i], P[1][i]);
            }
            Sa[0] = u[1] * w[2] - u[2] * w[1];
            Sa[1] = u[2] * w[0] - u[0] * w[2];
            Sa[2] = u[0] * w[1] - u[1] * w[0];
        } else {
            R u[2];  // the other column
#pragma unroll
            for (int i = 0; i < 2; ++i) u[i] = fma(x, Q[0][i], P[0][i]);
            // adj = [[J11, -J01], [-J10, J00]]: row 0 = (u1, -u0) with u = col 1; row 1 = (-u1, u0) with u = col 0
            if constexpr (A == 0) {
                Sa[0] = u[1];
                Sa[1] = -u[0];
            } else {
                Sa[0] = -u[1];
                Sa[1] = u[0];
            }
        }
    }
};

// Scalar / pair arithmetic for line_derivative (Pair<R>: FFMA2 for FP32).
template <class R>
__device__ __forceinline__ R t_mul(R s, R a) { return s * a; }
template <class R>
__device__ __forceinline__ R t_fma(R s, R a, R c) { return fma(s, a, c); }
template <class R>
__device__ __forceinline__ R t_add(R a, R b) { return a + b; }
template <class R>
__device__ __forceinline__ R t_sub(R a, R b) { return a - b; }
template <class R>
__device__ __forceinline__ Pair<R> t_mul(R s, Pair<R> a) { return pmul(s, a); }
template <class R>
__device__ __forceinline__ Pair<R> t_fma(R s, Pair<R> a, Pair<R> c) { return pfma(s, a, c); }
template <class R>
__device__ __forceinline__ Pair<R> t_add(Pair<R> a, Pair<R> b) { return padd(a, b); }
template <class R>
__device__ __forceinline__ Pair<R> t_sub(Pair<R> a, Pair<R> b) { return psub(a, b); }

// d = D y along one line (y is overwritten).  From m = HF_EVEN_ODD_MIN_M the
// even-odd split of D (Params::DE/DO/DC, as the lines kernel): about half the FMAs.
template <class R, int M, class T>
__device__ __forceinline__ void line_derivative(const Params<R>& p, T (&y)[M], T (&d)[M]) {
    if constexpr (M < HF_EVEN_ODD_MIN_M) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            T a = t_mul(p.D[i * M], y[0]);
#pragma unroll
            for (int t = 1; t < M; ++t) a = t_fma(p.D[i * M + t], y[t], a);
            d[i] = a;
        }
    } else {
        constexpr int H = M / 2, K = kMaxH;
#pragma unroll
        for (int t = 0; t < H; ++t) {
            const T y0 = y[t], y1 = y[M - 1 - t];
            y[t] = t_add(y0, y1);
            y[M - 1 - t] = t_sub(y0, y1);
        }
#pragma unroll
        for (int i = 0; i < H; ++i) {
            T x = t_mul(p.DE[i * K], y[0]);
            T z = t_mul(p.DO[i * K], y[M - 1]);
#pragma unroll
            for (int t = 1; t < H; ++t) {
                x = t_fma(p.DE[i * K + t], y[t], x);
                z = t_fma(p.DO[i * K + t], y[M - 1 - t], z);
            }
            if constexpr (M % 2 == 1) x = t_fma(p.DC[i], y[H], x);
            d[i] = t_add(x, z);
            d[M - 1 - i] = t_sub(z, x);
        }
        if constexpr (M % 2 == 1) {
            T z = t_mul(p.DO[H * K], y[M - 1]);
#pragma unroll
            for (int t = 1; t < H; ++t) z = t_fma(p.DO[H * K + t], y[M - 1 - t], z);
            d[H] = z;
        }
    }
}

// Accumulate d = D * Y (line rows of one batch) into the shared partial sums.
// Rows go through the contraction in pairs (same D row): FFMA2 for FP32.
template <class R, int M, int NE, int STRIDE, int NROW>
__device__ __forceinline__ void mapped_contract(const Params<R>& p, const R (&Y)[NROW][M], R* __restrict__ acc_line,
                                                const int (&rows)[NROW], R scale, bool first) {
    constexpr int NP_STRIDE = NE * STRIDE;
    using PR = Pair<R>;
#pragma unroll
    for (int r = 0; r < NROW; r += 2) {
        if (r + 1 < NROW) {
            PR y[M], d[M];
#pragma unroll
            for (int t = 0; t < M; ++t) y[t] = PR::make(Y[r][t], Y[r + 1][t]);
            line_derivative<R, M>(p, y, d);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                R* q0 = acc_line + rows[r] + NP_STRIDE * i;
                R* q1 = acc_line + rows[r + 1] + NP_STRIDE * i;
                *q0 = first ? scale * d[i].x() : fma(scale, d[i].x(), *q0);
                *q1 = first ? scale * d[i].y() : fma(scale, d[i].y(), *q1);
            }
        } else {
            R y[M], d[M];
#pragma unroll
            for (int t = 0; t < M; ++t) y[t] = Y[r][t];
            line_derivative<R, M>(p, y, d);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                R* q = acc_line + rows[r] + NP_STRIDE * i;
                *q = first ? scale * d[i] : fma(scale, d[i], *q);
            }
        }
    }
}

// The last sweep's contraction: the row's partial sum is complete at each point, so the
// output -(acc + scale d) / |J| (+ the source of gradient rows) goes straight over the staged
// input (this line's points, whose inputs the line has already read) -- no final pass.
template <class R, int M, int NE, int STRIDE, int NROW, bool SRCROWS>
__device__ __forceinline__ void mapped_contract_last(const Params<R>& p, const R (&Y)[NROW][M],
                                                     const R* __restrict__ acc_line, R* __restrict__ s_line,
                                                     const int (&rows)[NROW], R scale, const R (&inv)[M]) {
    constexpr int NP_STRIDE = NE * STRIDE;
    using PR = Pair<R>;
    auto fin = [&](int row, int i, R dv) {
        const int w = row + NP_STRIDE * i;
        R o = -fma(scale, dv, acc_line[w]) * inv[i];
        if constexpr (SRCROWS) o = fma(-p.invT, s_line[w], o);
        s_line[w] = o;
    };
#pragma unroll
    for (int r = 0; r < NROW; r += 2) {
        if (r + 1 < NROW) {
            PR y[M], d[M];
#pragma unroll
            for (int t = 0; t < M; ++t) y[t] = PR::make(Y[r][t], Y[r + 1][t]);
            line_derivative<R, M>(p, y, d);
#pragma unroll
            for (int i = 0; i < M; ++i) {
                fin(rows[r], i, d[i].x());
                fin(rows[r + 1], i, d[i].y());
            }
        } else {
            R y[M], d[M];
#pragma unroll
            for (int t = 0; t < M; ++t) y[t] = Y[r][t];
            line_derivative<R, M>(p, y, d);
#pragma unroll
            for (int i = 0; i < M; ++i) fin(rows[r], i, d[i]);
        }
    }
}

// One sweep along axis A for the line whose first point is word `o` of the chunk.
// LAST: the final sweep finishes the outputs in place (mapped_contract_last).
template <class R, int DIM, int M, int NE, int A, bool LAST = false, bool SRC = false>
__device__ __forceinline__ void mapped_sweep(R* __restrict__ s, R* __restrict__ acc, const R* __restrict__ geo,
                                             const Params<R>& p, int o) {
    constexpr int NP = ipow_c(M, DIM);
    constexpr int VS = NE * NP;  // word stride between variables (and metric entries)
    constexpr int STRIDE = (A == 0) ? 1 : (A == 1) ? M : M * M;
    constexpr int NV = n_vars_c(DIM);
    const bool first = (A == 0);
    R* sb = s + o;
    const int el = o % NE;
    const int bp = o / NE;  // the line's first point: its A index is 0
    R xi[3] = {p.xg[bp % M], p.xg[(bp / M) % M], DIM == 3 ? p.xg[bp / (M * M)] : R(0)};
    // row A of adj(J) at every point of the line, kept for all batches
    R SL[M][DIM];
    {
        const LineMetric<R, DIM, NE, A> lm(geo, el, xi);
#pragma unroll
        for (int t = 0; t < M; ++t) lm.row(p.xg[t], SL[t]);
    }
    // LAST: 1/|J| along the line.  Column A of J does not depend on xi_A (the map is
    // multilinear), and row A of adj(J) times column A of J is |J|.
    R inv[LAST ? M : 1];
    if constexpr (LAST) {
        R JA[DIM];
        mapped_jcol<R, DIM, NE>(geo, el, A, xi, JA);
#pragma unroll
        for (int t = 0; t < M; ++t) {
            R det = SL[t][0] * JA[0];
#pragma unroll
            for (int b = 1; b < DIM; ++b) det = fma(SL[t][b], JA[b], det);
            inv[t] = R(1) / det;
        }
    }
    // LAST: the velocity rows of the line, read before batch 0 overwrites them
    R VL[LAST ? M : 1][DIM];

    // batch 0: continuity + momentum rows
    {
        R Y[1 + DIM][M];
#pragma unroll
        for (int t = 0; t < M; ++t) {
            const int q = NE * STRIDE * t;
            const R(&Sa)[DIM] = SL[t];
            R V[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) V[b] = sb[q + VS * (1 + b)];
            if constexpr (LAST)
#pragma unroll
                for (int b = 0; b < DIM; ++b) VL[t][b] = V[b];
            const R P = sb[q];
            R W = Sa[0] * V[0];
#pragma unroll
            for (int b = 1; b < DIM; ++b) W = fma(Sa[b], V[b], W);
            Y[0][t] = p.zeta * W;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                R vg = Sa[0] * sb[q + VS * var_grad_c(DIM, c, 0)];
#pragma unroll
                for (int b = 1; b < DIM; ++b) vg = fma(Sa[b], sb[q + VS * var_grad_c(DIM, c, b)], vg);
                Y[1 + c][t] = fma(V[c], W, fma(Sa[c], P, -p.nu * vg));
            }
        }
        int rows[1 + DIM];
#pragma unroll
        for (int r = 0; r <= DIM; ++r) rows[r] = VS * r;
        if constexpr (LAST)
            mapped_contract_last<R, M, NE, STRIDE, 1 + DIM, false>(p, Y, acc + o, sb, rows, R(1), inv);
        else
            mapped_contract<R, M, NE, STRIDE, 1 + DIM>(p, Y, acc + o, rows, R(1), first);
    }
    // batches 1..d: gradient rows g(c, b) <- D (S_ab V_c) * (-1/T)
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        R Y[DIM][M];
#pragma unroll
        for (int t = 0; t < M; ++t) {
            const int q = NE * STRIDE * t;
            R Vc;
            if constexpr (LAST) Vc = VL[t][c];
            else Vc = sb[q + VS * (1 + c)];
#pragma unroll
            for (int b = 0; b < DIM; ++b) Y[b][t] = SL[t][b] * Vc;
        }
        int rows[DIM];
#pragma unroll
        for (int b = 0; b < DIM; ++b) rows[b] = VS * var_grad_c(DIM, c, b);
        if constexpr (LAST)
            mapped_contract_last<R, M, NE, STRIDE, DIM, SRC>(p, Y, acc + o, sb, rows, -p.invT, inv);
        else
            mapped_contract<R, M, NE, STRIDE, DIM>(p, Y, acc + o, rows, -p.invT, first);
    }
    (void)NV;
}

template <class R, int DIM, int M, int NE, bool SRC>
__global__ void __launch_bounds__(MappedShape<R, DIM, M, NE>::BS)
    hf_mapped_kernel(const __grid_constant__ Params<R> p) {
    using S = MappedShape<R, DIM, M, NE>;
    using L = LinesShape<R, DIM, M, NE>;
    using IO = typename L::IO;
    constexpr int BS = S::BS, NP = S::NP, NV = S::NV, NC = S::NC;
    constexpr int VS = NE * NP;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* buf = smem_raw + S::HDR;
    R* acc = reinterpret_cast<R*>(smem_raw + S::ACC_OFF);
    R* geo = reinterpret_cast<R*>(smem_raw + S::GEO_OFF);  // [c][x][el]

    const int tid = threadIdx.x;
    const long long E0 = static_cast<long long>(blockIdx.x) * NE;
    const long long grp = E0 / p.group;
    const int el0 = static_cast<int>(E0 - grp * p.group);
    const long long gbase = grp * p.group_words + el0;
    const bool contiguous = (p.group == NE);
    const bool fast = chunk_bulk_ok<R, L::IN_WORDS>(p, gbase, E0 + NE <= p.n_elem, contiguous);
    const int head = fast ? IO::head_bytes(p.u + gbase, contiguous) : 0;

    // ---------------- stage the chunk and its corners ----------------
    // With group == NE the chunk's corners are one contiguous, 16-byte-multiple
    // range (2^d d words per element): a second bulk copy on its own mbarrier,
    // so the sweeps' corner reads do not wait on a second round trip.
    constexpr int GEO_WORDS = NC * DIM * NE;
    const bool geo_bulk = fast && contiguous && (reinterpret_cast<uintptr_t>(p.geo) & 15u) == 0;
    if (fast) {
        if (tid == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (tid < 32) {
            if (tid == 0) {
                mbar_arrive_expect_tx(bar, IO::tx_bytes(p.u + gbase, contiguous));
                if (geo_bulk) {
                    mbar_arrive_expect_tx(bar + 1, uint32_t(GEO_WORDS * sizeof(R)));
                    bulk_g2s(geo, p.geo + E0 * NC * DIM, GEO_WORDS * sizeof(R), bar + 1);
                }
            }
            __syncwarp();
            IO::load(buf, p.u + gbase, p.group, contiguous, bar, tid);
        }
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
    }
    if (!geo_bulk) {
        for (int idx = tid; idx < GEO_WORDS; idx += BS) {
            const int el = idx % NE;
            const int cx = idx / NE;  // x + DIM * c
            const long long e = E0 + el;
            R v = R(0);
            if (e < p.n_elem) {
                const long long ge = e / p.group;
                v = p.geo[ge * p.group * NC * DIM + (e - ge * p.group) + static_cast<long long>(p.group) * cx];
            }
            geo[idx] = v;
        }
        __syncthreads();
    } else {
        mbar_wait_parity(bar + 1, 0);
    }

    if (fast) mbar_wait_parity(bar, 0);
    __syncthreads();
    mapped_corners_to_monomials<R, DIM, NE, BS>(geo, tid);
    __syncthreads();

    // ---------------- d sweeps ----------------
    R* s = reinterpret_cast<R*>(buf + head);
    auto sweep = [&](auto a_tag) {
        constexpr int A = decltype(a_tag)::value;
        constexpr bool LAST = (A == DIM - 1);
        using LM = LineMap<R, DIM, M, NE, A, BS>;
        const unsigned short* map = kLineMap<R, DIM, M, NE, A, BS>.off;
#pragma unroll 1
        for (int k = 0; k < LM::ITERS; ++k) {
            const int o = map[k * BS + tid];
            if (o != 0xFFFF) mapped_sweep<R, DIM, M, NE, A, LAST, SRC>(s, acc, geo, p, o);
        }
    };
    sweep(std::integral_constant<int, 0>{});
    __syncthreads();
    sweep(std::integral_constant<int, 1>{});
    if constexpr (DIM == 3) {
        __syncthreads();
        sweep(std::integral_constant<int, 2>{});
    }

    // ---------------- write the finished chunk ----------------
    if (fast) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid < 32) {
            IO::store(p.out + gbase, buf, p.group, contiguous, tid);
            bulk_wait_read_all();
        }
    } else {
        __syncthreads();
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
