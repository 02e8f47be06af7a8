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

#include <type_traits>

#include "hf_chunk_io.cuh"
#include "hf_common.cuh"

#ifndef HF_EVEN_ODD_MIN_M
#define HF_EVEN_ODD_MIN_M 6  // even-odd split of the line contraction from m = 6 (p = 5) up
#endif

namespace hfb {

// Padding (words) after each staged group of a grouped chunk (GS < NE): when the group's
// byte size is an even multiple of 16, successive groups would start in only a few bank
// classes (e.g. element-major p3: 832 words = 0 mod 32, every element in the same class),
// so each group is staged at a stride that is an odd multiple of 16 bytes (one bulk copy
// per group).  Groups whose size is not a multiple of 16 bytes stay one contiguous image.
constexpr int grouped_pad_words(int w, int blk_words) {
    if ((blk_words * w) % 16 != 0 || ((blk_words * w) / 16) % 2 == 1) return 0;
    return 16 / w;
}

// LPT: lines per thread of the one-chunk-per-CTA kernel (block = LINES / LPT
// threads): larger chunks per block without more threads, for the low-order
// cases whose per-line work is small and whose bytes in flight per SM are
// limited by the thread count.
// GS: the chunk's shared-memory layout.  GS = NE (default): [v][pt][el], the layout of
// one AoSoA group of NE elements.  GS < NE (NE a multiple of GS): the chunk is NE/GS
// whole groups of the caller's group size GS, staged as they lie in HBM,
// [el / GS][v][pt][el % GS] -- one contiguous byte range for any group that divides the
// chunk (grouped chunk, hf_launch.cuh launch_lines).
// CS: component split -- each a-line is worked by d threads, one per velocity component b
// (V_b and the momentum flux M_ba, lines_sweep_comp): d times the threads per chunk for the
// high orders whose chunks are few per SM (shared-memory bound), same arithmetic.
// Padding (words) of the x-rows of a padded chunk (lines variants 25-27, XP): the chunk is
// staged as rows of the m x NE words (i, el) of one (j, k, v), and x-lines (and the
// accumulator lines) all start at multiples of the row stride; a stride that is an odd
// multiple of 16 bytes spreads them over the banks.  The padded image is moved by one TMA
// tensor copy whose box is wider than the row -- the pad words are out of bounds, zero-filled
// on load and clipped on store -- so the copy engine does the deconfliction that the
// reference's planar kernels get from a padded plane stride (banks.hpp:59-120).
template <class R, int DIM, int M, int NE>
constexpr int xpad_words() {
    constexpr int gran = 16 / int(sizeof(R));
    int xp = 0;
    while ((M * NE + xp) % gran != 0 || ((M * NE + xp) / gran) % 2 == 0) ++xp;
    return xp;
}

// The padding code XP of a padded chunk: x-row pad words + 256 x pad rows per k-plane.  One-
// element chunks (NE = 1, element-major, vectorised x-lines) keep 16-byte rows unpadded and
// pad each k-plane by one row instead: their y-lines start at i + m^2 k, a few bank classes
// for every k (the x-lines are already spread by their vector reads).
template <class R, int DIM, int M, int NE>
constexpr int xpad_code() {
    if (DIM == 3 && NE == 1 && (M * int(sizeof(R))) % 16 == 0) return 256 * 1;
    return xpad_words<R, DIM, M, NE>();
}

template <class R, int DIM, int M, int NE, int LPT = 1, int GS = NE, bool CS = false, int XP = 0>
struct LinesShape {
    static_assert(NE % GS == 0, "a grouped chunk holds whole groups");
    static_assert(XP == 0 || (GS == NE && !CS), "padded chunks: plain chunks only");
    static constexpr int NV = n_vars_c(DIM);
    static constexpr int NP = ipow_c(M, DIM);
    static constexpr int LINES = NE * ipow_c(M, DIM - 1);
    static constexpr int TL = (LINES + LPT - 1) / LPT;
    static constexpr int NT = ((TL + 31) / 32) * 32;  // threads per component group (CS) / line slots
    static constexpr int BS = CS ? (DIM * NT < 64 ? 64 : DIM * NT) : (NT < 64 ? 64 : NT);
    static constexpr int NACC = 1 + DIM;  // continuity + d momentum partials
    static constexpr int IN_WORDS = NE * NP * NV;
    static constexpr int RW = M * NE;                   // x-row words (i, el)
    static constexpr int XW = XP % 256;                 // x-row pad words
    static constexpr int PJ = XP / 256;                 // pad rows per k-plane (d3)
    static_assert(PJ == 0 || DIM == 3, "plane padding is a d3 layout");
    static constexpr int RS = RW + XW;                  // staged x-row stride
    static constexpr int PR = M + PJ;                   // staged rows per k-plane
    static constexpr int PL = RS * PR;                  // staged k-plane stride
    static constexpr int XR = DIM == 3 ? PR * M : M;    // staged x-rows per variable
    static constexpr int AS = XP ? RS * XR : NE * NP;   // accumulator row stride
    static constexpr int ACC_WORDS = AS * NACC;
    static constexpr int HDR = 128;  // mbarrier + alignment pad
    static constexpr int IN_BYTES = IN_WORDS * int(sizeof(R));
    static constexpr int ROW_BYTES = NE * int(sizeof(R));
    using IO = ChunkIO<R, NE, NP * NV, IN_BYTES>;
    static constexpr int VS = XP ? RS * XR : GS * NP;  // word stride between variables
    static constexpr int BLK = GS * NP * NV;    // one group in HBM
    static constexpr int PADW = GS < NE ? grouped_pad_words(int(sizeof(R)), BLK) : 0;
    static constexpr int BLKP = BLK + PADW;     // one staged group (padded: one bulk copy per group)
    static constexpr int BUF_BYTES =            // chunk buffer incl. alignment slack
        XP ? (NV * VS * int(sizeof(R)) + 127) / 128 * 128
           : PADW ? ((NE / GS) * BLKP * int(sizeof(R)) + 15) / 16 * 16 : IO::BUF_BYTES;
    static constexpr size_t SMEM = HDR + size_t(BUF_BYTES) + size_t(ACC_WORDS) * sizeof(R);
    // word of (element, point, variable) in the staged chunk
    __host__ __device__ static constexpr int word(int el, int pt, int v) {
        if constexpr (XP > 0) return el + NE * (pt % M) + RS * ((pt / M) % M) + PL * (pt / (M * M)) + VS * v;
        return (el % GS) + GS * pt + VS * v + (el / GS) * BLKP;
    }
    // word step between consecutive points of an A-line (state; accumulators: acc_step)
    template <int A>
    __host__ __device__ static constexpr int step() {
        if constexpr (XP > 0) return A == 0 ? NE : A == 1 ? RS : PL;
        return GS * (A == 0 ? 1 : A == 1 ? M : M * M);
    }
    template <int A>
    __host__ __device__ static constexpr int acc_step() {
        if constexpr (XP > 0) return step<A>();
        return NE * (A == 0 ? 1 : A == 1 ? M : M * M);
    }
    // staged position of the li-th word of the chunk's HBM image (li = group * BLK + rem)
    __host__ __device__ static constexpr int staged(int li) {
        if constexpr (XP > 0) {
            const int v = li / (NE * NP), rem = li - v * (NE * NP);
            const int row = rem / RW, col = rem - row * RW;
            return col + RS * (row % M) + PL * (row / M) + VS * v;
        } else if constexpr (PADW == 0) {
            return li;
        } else {
            const int b = li / BLK;
            return li + b * PADW;
        }
    }
    // The accumulator region keeps the [row][pt][el] layout of NE elements whatever GS is
    // (its element classes then spread over the banks; a grouped chunk's state region
    // cannot be re-laid out -- it is the HBM image).  Offset of the line at chunk offset o:
    __host__ __device__ static constexpr int acc_of(int o) {
        if constexpr (GS == NE) {
            return o;  // (padded chunks: the accumulators share the padded layout)
        } else {
            const int blk = o / BLKP, rem = o - blk * BLKP;
            return blk * GS + rem % GS + NE * (rem / GS);
        }
    }
};

// Whether the chunk starting at word `gbase` can take the bulk path: full chunk,
// layout verified by the host, and (contiguous) the 16-byte superset stays inside
// the allocation.
template <class R, int IN_WORDS>
__device__ __forceinline__ bool chunk_bulk_ok(const Params<R>& p, long long gbase, bool full, bool contiguous) {
    if (!p.fast_ok || !full) return false;
    if (!contiguous) return true;
    return ((gbase + IN_WORDS) * (long long)sizeof(R) + 15) / 16 * 16 <= p.total_words * (long long)sizeof(R);
}

// Outputs of one line point (index i of the sweep's line): gradient rows final
// (+ source), continuity / momentum partials accumulated or finished.
// GRAD = false: the caller stores the gradient rows itself (vectorised x-lines, lines_sweep).
template <class R, int DIM, int M, int NE, bool SRC, int A, int PHASE, int GS = NE, bool GRAD = true, int XP = 0>
__device__ __forceinline__ void lines_emit(R* __restrict__ q, R* __restrict__ a, const Params<R>& p, const R (&dV)[DIM],
                                           const R (&dQ)[DIM]) {
    constexpr int VS = LinesShape<R, DIM, M, NE, 1, GS, false, XP>::VS;  // state rows
    constexpr int AS = LinesShape<R, DIM, M, NE, 1, GS, false, XP>::AS;  // accumulator rows
    if constexpr (GRAD)
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
        for (int b = 0; b < DIM; ++b) a[AS * (1 + b)] = p.jac[A] * dQ[b];
    } else if constexpr (PHASE == 1) {
        a[0] = a[0] + c;
#pragma unroll
        for (int b = 0; b < DIM; ++b) a[AS * (1 + b)] = fma(p.jac[A], dQ[b], a[AS * (1 + b)]);
    } else {
        q[0] = -(p.zeta * (a[0] + c));
#pragma unroll
        for (int b = 0; b < DIM; ++b) q[VS * (1 + b)] = -fma(p.jac[A], dQ[b], a[AS * (1 + b)]);
    }
}

// Word offset (inside a chunk) of the first point of line L of a sweep along A:
// L = el + NE * r, r enumerating the two fixed indices (layout.hpp:128-134).
template <int DIM, int M, int NE, int A, int GS = NE, int BLKS = GS * ipow_c(M, DIM) * n_vars_c(DIM), int RS = 0,
          int PL = RS * M>
__host__ __device__ constexpr int line_offset(int L) {
    const int el = L % NE;
    const int r = L / NE;
    if (RS > 0) {  // padded chunk (GS == NE): x-row stride RS, k-plane stride PL
        if (A == 0) return el + RS * (r % M) + PL * (r / M);          // r = j + M k
        if (DIM == 3 && A == 1) return el + NE * (r % M) + PL * (r / M);  // r = i + M k
        return el + NE * (r % M) + RS * (r / M);                        // d3 A=2: r = i + M j; d2 A=1: r = i
    }
    int base_pt = r;                                  // d3 A=2: r = i + M j;  d2 A=1: r = i
    if (A == 0) base_pt = M * r;                      // d3: r = j + M k;  d2: r = j
    if (DIM == 3 && A == 1) base_pt = (r % M) + M * M * (r / M);  // r = i + M k
    return (el % GS) + GS * base_pt + (el / GS) * BLKS;
}

// Vector width (words) of an x-line row read in an element-major chunk (GS = 1): every line
// starts at a multiple of M words inside its element's staged block, whose stride BLKP and
// the variable stride VS are byte multiples of the vector too.  1 = scalar reads.
template <class R, int M, int GS, int BLKP, int VS, int A>
__host__ __device__ constexpr int x_line_vec() {
    int best = 1;
    if (A == 0 && GS == 1)
        for (int vb = int(sizeof(R)) * 2; vb <= 16; vb *= 2) {
            const int vw = vb / int(sizeof(R));
            if (M % vw == 0 && (BLKP * int(sizeof(R))) % vb == 0 && (VS * int(sizeof(R))) % vb == 0) best = vw;
        }
    return best;
}

// Bank-conflict-free assignment of a sweep's lines to (iteration, thread).
// A warp's shared-memory access is one wavefront per 128 B only if its lanes
// hit distinct banks: for 4-byte words all 32 lanes need distinct word offsets
// mod 32, for 8-byte words each half-warp needs distinct offsets mod 16
// (measured on B200: a half-warp 2-way conflict doubles the wavefronts).  Every
// point of a line is the line offset plus a per-(point, variable) constant, so
// the class (offset mod 32 | 16) of the line decides.  The map deals the lines
// of class c to lane c of warps 0, 1, ... (and lane c + 16 for 8-byte words);
// a class with more lines than the slots of ITERS iterations spills into idle
// slots (a conflict, but no extra iteration).  With the natural order (L = t,
// t + NTHR, ...) the y-sweep conflicts whenever NE*m is not a multiple of the
// bank count (e.g. 2-way at p6 FP64).  Built at compile time; 0xFFFF = idle.
template <class R, int DIM, int M, int NE, int A, int NTHR, int GS = NE, int XP = 0>
struct LineMap {
    static constexpr int LINES = NE * ipow_c(M, DIM - 1);
    static constexpr int ITERS = (LINES + NTHR - 1) / NTHR;
    static constexpr int N = ITERS * NTHR;
    unsigned short off[N];
};

template <class R, int DIM, int M, int NE, int A, int NTHR, int GS = NE, int XP = 0>
constexpr LineMap<R, DIM, M, NE, A, NTHR, GS, XP> make_line_map() {
    using LM = LineMap<R, DIM, M, NE, A, NTHR, GS, XP>;
    using S = LinesShape<R, DIM, M, NE, 1, GS, false, XP>;
    // vectorised x-lines (x_line_vec): a VW-word access, 128 / (VW * sizeof(R)) lanes per wavefront
    constexpr int VW = x_line_vec<R, M, GS, S::BLKP, S::VS, A>();
    constexpr int B = VW > 1 ? 128 / (VW * int(sizeof(R))) : sizeof(R) == 4 ? 32 : 16;  // bank classes per phase
    constexpr int HALVES = 32 / B;
    constexpr int NW = NTHR / 32;
    LM m{};
    for (int i = 0; i < LM::N; ++i) m.off[i] = 0xFFFF;
    int next[B] = {};
    int spill[LM::LINES > 0 ? LM::LINES : 1] = {};
    int n_spill = 0;
    for (int L = 0; L < LM::LINES; ++L) {
        const int o = line_offset<DIM, M, NE, A, GS, S::BLKP, (XP ? S::RS : 0), (XP ? S::PL : 0)>(L);
        const int c = (o / VW) % B;
        const int idx = next[c]++;
        const int it = idx / (NW * HALVES);
        if (it >= LM::ITERS) {
            spill[n_spill++] = o;
            continue;
        }
        const int rem = idx % (NW * HALVES);
        const int slot = it * NTHR + (rem / HALVES) * 32 + (rem % HALVES) * B + c;
        m.off[slot] = static_cast<unsigned short>(o);
    }
    for (int i = 0, k = 0; k < n_spill && i < LM::N; ++i)
        if (m.off[i] == 0xFFFF) m.off[i] = static_cast<unsigned short>(spill[k++]);
    return m;
}

template <class R, int DIM, int M, int NE, int A, int NTHR, int GS = NE, int XP = 0>
__device__ const LineMap<R, DIM, M, NE, A, NTHR, GS, XP> kLineMap = make_line_map<R, DIM, M, NE, A, NTHR, GS, XP>();

template <class R, int M, int VW>
__device__ __forceinline__ void load_row(const R* __restrict__ q, R (&out)[M]) {
    static_assert(VW * sizeof(R) == 16 || VW * sizeof(R) == 8, "8- or 16-byte rows");
    if constexpr (sizeof(R) == 4 && VW == 4) {
#pragma unroll
        for (int t = 0; t < M; t += 4) {
            const float4 v = *reinterpret_cast<const float4*>(q + t);
            out[t] = v.x; out[t + 1] = v.y; out[t + 2] = v.z; out[t + 3] = v.w;
        }
    } else if constexpr (sizeof(R) == 4) {
#pragma unroll
        for (int t = 0; t < M; t += 2) {
            const float2 v = *reinterpret_cast<const float2*>(q + t);
            out[t] = v.x; out[t + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int t = 0; t < M; t += 2) {
            const double2 v = *reinterpret_cast<const double2*>(q + t);
            out[t] = v.x; out[t + 1] = v.y;
        }
    }
}

template <class R, int M, int VW>
__device__ __forceinline__ void store_row(R* __restrict__ q, const R (&in)[M]) {
    if constexpr (sizeof(R) == 4 && VW == 4) {
#pragma unroll
        for (int t = 0; t < M; t += 4) *reinterpret_cast<float4*>(q + t) = make_float4(in[t], in[t + 1], in[t + 2], in[t + 3]);
    } else if constexpr (sizeof(R) == 4) {
#pragma unroll
        for (int t = 0; t < M; t += 2) *reinterpret_cast<float2*>(q + t) = make_float2(in[t], in[t + 1]);
    } else {
#pragma unroll
        for (int t = 0; t < M; t += 2) *reinterpret_cast<double2*>(q + t) = make_double2(in[t], in[t + 1]);
    }
}

// One sweep along axis A.  PHASE: 0 = first sweep, 1 = middle, 2 = last.
// `o` = the line's first word inside the chunk (line_offset()).
template <class R, int DIM, int M, int NE, bool SRC, int A, int PHASE, int GS = NE, int XP = 0>
__device__ __forceinline__ void lines_sweep(R* __restrict__ s, R* __restrict__ acc, const Params<R>& p, int o) {
    using S = LinesShape<R, DIM, M, NE, 1, GS, false, XP>;
    constexpr int VS = S::VS;  // word stride between variables
    constexpr int PS = S::template step<A>();      // point step along the line (state)
    constexpr int APS = S::template acc_step<A>();  // ... and in the accumulator region

    R* __restrict__ sb = s + o;
    R* __restrict__ ab = acc + S::acc_of(o);
    const R nu = p.nu;
    using PR = Pair<R>;
    // W[b][t] = (V_b, M_ba) at line point t: both lines are contracted with the same D rows
    PR W[DIM][M];
    constexpr int VW = x_line_vec<R, M, GS, (XP ? S::RS : S::BLKP), VS, A>();
    // element-major chunk (GS = 1): an x-line's M points are consecutive words, so each
    // variable's row is read (and each gradient row of the first sweep written) with VW-wide
    // accesses -- a quarter-warp of LDS.128 covers the 32 banks, where scalar accesses of
    // lines at multiples of M words would collide M-way
    constexpr bool VEC_ST = VW > 1 && PHASE == 0;
    R G[DIM][M], Gout[DIM][VEC_ST ? M : 1];
    if constexpr (VW > 1) {
        R P[M], V[DIM][M];
        load_row<R, M, VW>(sb, P);
#pragma unroll
        for (int b = 0; b < DIM; ++b) {
            load_row<R, M, VW>(sb + VS * (1 + b), V[b]);
            load_row<R, M, VW>(sb + VS * var_grad_c(DIM, b, A), G[b]);
        }
#pragma unroll
        for (int t = 0; t < M; ++t)
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                const R base = (b == A) ? fma(-nu, G[b][t], P[t]) : (-nu) * G[b][t];
                W[b][t] = PR::make(V[b][t], fma(V[b][t], V[A][t], base));
            }
    } else {
#pragma unroll
        for (int t = 0; t < M; ++t) {
            const R* q = sb + PS * t;
            const R P = q[0];
            R V[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) V[b] = q[VS * (1 + b)];
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                const R g = q[VS * var_grad_c(DIM, b, A)];
                // codegen_util.hpp:191-202 operation order: base, then fma(V_b, V_a, base)
                const R base = (b == A) ? fma(-nu, g, P) : (-nu) * g;
                W[b][t] = PR::make(V[b], fma(V[b], V[A], base));
            }
        }
    }

    // Derivatives along the line.  m >= HF_EVEN_ODD_MIN_M: even-odd split of D
    // (Params::DE/DO/DC), about half the FMAs of the dense m x m contraction; it
    // lengthens the dependency chain, which only pays off at high order (measured:
    // p6 +14 % FP64, p3 -5 %), so lower orders use the dense contraction.
#define HF_EMIT(I, DP)                                                                                         \
    do {                                                                                                        \
        R dV_[DIM], dQ_[DIM];                                                                                  \
        _Pragma("unroll") for (int b_ = 0; b_ < DIM; ++b_) {                                                   \
            dV_[b_] = (DP)[b_].x();                                                                            \
            dQ_[b_] = (DP)[b_].y();                                                                            \
        }                                                                                                      \
        if constexpr (VEC_ST) {                                                                                \
            _Pragma("unroll") for (int b_ = 0; b_ < DIM; ++b_) {                                               \
                R o_ = p.jac_invT[A] * dV_[b_];                                                                \
                if constexpr (SRC) o_ = fma(-p.invT, G[b_][(I)], o_);                                          \
                Gout[b_][(I)] = o_;                                                                            \
            }                                                                                                   \
        }                                                                                                       \
        lines_emit<R, DIM, M, NE, SRC, A, PHASE, GS, !VEC_ST, XP>(sb + PS * (I), ab + APS * (I), p, dV_, dQ_);    \
    } while (0)
    if constexpr (M < HF_EVEN_ODD_MIN_M) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            PR d[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) d[b] = pmul(p.D[i * M], W[b][0]);
#pragma unroll
            for (int t = 1; t < M; ++t)
#pragma unroll
                for (int b = 0; b < DIM; ++b) d[b] = pfma(p.D[i * M + t], W[b][t], d[b]);
            HF_EMIT(i, d);
        }
    } else {
        constexpr int H = M / 2;
        constexpr int K = kMaxH;
        // symmetric / antisymmetric parts, in place: W[b][t] <- S_t, W[b][M-1-t] <- A_t
#pragma unroll
        for (int t = 0; t < H; ++t)
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                const PR w0 = W[b][t], w1 = W[b][M - 1 - t];
                W[b][t] = padd(w0, w1);
                W[b][M - 1 - t] = psub(w0, w1);
            }
#pragma unroll
        for (int i = 0; i < H; ++i) {
            PR x[DIM], y[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) {
                x[b] = pmul(p.DE[i * K], W[b][0]);
                y[b] = pmul(p.DO[i * K], W[b][M - 1]);
            }
#pragma unroll
            for (int t = 1; t < H; ++t)
#pragma unroll
                for (int b = 0; b < DIM; ++b) {
                    x[b] = pfma(p.DE[i * K + t], W[b][t], x[b]);
                    y[b] = pfma(p.DO[i * K + t], W[b][M - 1 - t], y[b]);
                }
            if constexpr (M % 2 == 1)
#pragma unroll
                for (int b = 0; b < DIM; ++b) x[b] = pfma(p.DC[i], W[b][H], x[b]);
            PR d[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) d[b] = padd(x[b], y[b]);
            HF_EMIT(i, d);
#pragma unroll
            for (int b = 0; b < DIM; ++b) d[b] = psub(y[b], x[b]);
            HF_EMIT(M - 1 - i, d);
        }
        if constexpr (M % 2 == 1) {
            PR d[DIM];
#pragma unroll
            for (int b = 0; b < DIM; ++b) d[b] = pmul(p.DO[H * K], W[b][M - 1]);
#pragma unroll
            for (int t = 1; t < H; ++t)
#pragma unroll
                for (int b = 0; b < DIM; ++b) d[b] = pfma(p.DO[H * K + t], W[b][M - 1 - t], d[b]);
            HF_EMIT(H, d);
        }
    }
    if constexpr (VEC_ST)
#pragma unroll
        for (int b = 0; b < DIM; ++b) store_row<R, M, VW>(sb + VS * var_grad_c(DIM, b, A), Gout[b]);
}

#undef HF_EMIT

// ---------------------------------------------------------------------------------------------
// Component-split sweep (LinesShape CS): the thread of component B of an A-line holds the
// pairs (V_B, M_BA) of its m points, M_BA = V_B V_A + P delta_AB - nu g(B,A) (the same
// operation order as lines_sweep), contracts them with the D rows and emits the gradient row
// (B,A), the momentum partial B and -- for B == A -- the continuity partial.  Every input word
// is read by the threads that need it; results are bit-identical to lines_sweep.
// ---------------------------------------------------------------------------------------------
template <class R, int DIM, int M, int NE, int A, int B, int GS>
__device__ __forceinline__ void comp_load(const R* __restrict__ s, const Params<R>& p, int o, Pair<R> (&W)[M]) {
    using S = LinesShape<R, DIM, M, NE, 1, GS>;
    constexpr int VS = S::VS;
    constexpr int STRIDE = (A == 0) ? 1 : (A == 1) ? M : M * M;
    const R* __restrict__ sb = s + o;
    const R nu = p.nu;
#pragma unroll
    for (int t = 0; t < M; ++t) {
        const R* q = sb + GS * STRIDE * t;
        const R Va = q[VS * (1 + A)];
        const R Vb = (B == A) ? Va : q[VS * (1 + B)];
        const R g = q[VS * var_grad_c(DIM, B, A)];
        // codegen_util.hpp:191-202 operation order: base, then fma(V_b, V_a, base)
        const R base = (B == A) ? fma(-nu, g, q[0]) : (-nu) * g;
        W[t] = Pair<R>::make(Vb, fma(Vb, Va, base));
    }
}

template <class R, int DIM, int M, int NE, bool SRC, int A, int B, int PHASE, int GS>
__device__ __forceinline__ void comp_emit(R* __restrict__ q, R* __restrict__ a, const Params<R>& p, R dV, R dQ) {
    constexpr int VS = GS * ipow_c(M, DIM);   // state rows
    constexpr int AS = NE * ipow_c(M, DIM);   // accumulator rows
    R o = p.jac_invT[A] * dV;
    if constexpr (SRC) o = fma(-p.invT, q[VS * var_grad_c(DIM, B, A)], o);
    q[VS * var_grad_c(DIM, B, A)] = o;
    if constexpr (B == A) {
        const R c = p.jac[A] * dV;
        if constexpr (PHASE == 0) a[0] = c;
        else if constexpr (PHASE == 1) a[0] = a[0] + c;
        else q[0] = -(p.zeta * (a[0] + c));
    }
    if constexpr (PHASE == 0) a[AS * (1 + B)] = p.jac[A] * dQ;
    else if constexpr (PHASE == 1) a[AS * (1 + B)] = fma(p.jac[A], dQ, a[AS * (1 + B)]);
    else q[VS * (1 + B)] = -fma(p.jac[A], dQ, a[AS * (1 + B)]);
}

template <class R, int DIM, int M, int NE, bool SRC, int A, int B, int PHASE, int GS>
__device__ __forceinline__ void comp_contract_emit(R* __restrict__ s, R* __restrict__ acc, const Params<R>& p, int o,
                                                   Pair<R> (&W)[M]) {
    using S = LinesShape<R, DIM, M, NE, 1, GS>;
    using PR = Pair<R>;
    constexpr int STRIDE = (A == 0) ? 1 : (A == 1) ? M : M * M;
    R* __restrict__ sb = s + o;
    R* __restrict__ ab = acc + S::acc_of(o);
    auto emit = [&](int i, PR d) {
        comp_emit<R, DIM, M, NE, SRC, A, B, PHASE, GS>(sb + GS * STRIDE * i, ab + NE * STRIDE * i, p, d.x(), d.y());
    };
    if constexpr (M < HF_EVEN_ODD_MIN_M) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
            PR d = pmul(p.D[i * M], W[0]);
#pragma unroll
            for (int t = 1; t < M; ++t) d = pfma(p.D[i * M + t], W[t], d);
            emit(i, d);
        }
    } else {
        constexpr int H = M / 2;
        constexpr int K = kMaxH;
#pragma unroll
        for (int t = 0; t < H; ++t) {
            const PR w0 = W[t], w1 = W[M - 1 - t];
            W[t] = padd(w0, w1);
            W[M - 1 - t] = psub(w0, w1);
        }
#pragma unroll
        for (int i = 0; i < H; ++i) {
            PR x = pmul(p.DE[i * K], W[0]);
            PR y = pmul(p.DO[i * K], W[M - 1]);
#pragma unroll
            for (int t = 1; t < H; ++t) {
                x = pfma(p.DE[i * K + t], W[t], x);
                y = pfma(p.DO[i * K + t], W[M - 1 - t], y);
            }
            if constexpr (M % 2 == 1) x = pfma(p.DC[i], W[H], x);
            emit(i, padd(x, y));
            emit(M - 1 - i, psub(y, x));
        }
        if constexpr (M % 2 == 1) {
            PR d = pmul(p.DO[H * K], W[M - 1]);
#pragma unroll
            for (int t = 1; t < H; ++t) d = pfma(p.DO[H * K + t], W[M - 1 - t], d);
            emit(H, d);
        }
    }
}

// All d sweeps of one chunk whose first word sits HEADB bytes into `buf`.
// HEADB is a template parameter so that every shared-memory address in the
// sweeps is a compile-time offset from the __shared__ window (a runtime base
// costs ~30 registers and ~10 % of HBM throughput, measured).  BAR: 0 = the
// whole CTA (__syncthreads), k > 0 = the NTHR threads of one consumer group
// (named barrier k), -1 = named barrier `bar_id` (runtime).
// FACES: FR stage 1 fused in (hf_fr.cuh): before the sweeps overwrite the staged
// chunk, every a-line of every variable is extrapolated to xi_a = -1, +1 and
// written to p.uf -- the face projection without a second read of the field.
template <class R, int DIM, int M, int NE, int GS = NE, int XP = 0>
__device__ __forceinline__ void lines_project_faces(const R* __restrict__ s, const Params<R>& p, long long E0, int t,
                                                    int nthr, int nvalid) {
    using S = LinesShape<R, DIM, M, NE, 1, GS, false, XP>;
    constexpr int NV = n_vars_c(DIM), LN = ipow_c(M, DIM - 1);
    for (int task = t; task < NE * LN * DIM; task += nthr) {
        const int el = task % NE;
        const int l = (task / NE) % LN;
        const int a = task / (NE * LN);
        const long long e = E0 + el;
        if (el >= nvalid || e >= p.n_elem) continue;
        int pt[M];
#pragma unroll
        for (int q = 0; q < M; ++q) pt[q] = S::word(el, fr_line_point<DIM, M>(a, l, q), 0);
        const long long ge = e / p.group;
        R* ub = p.uf + ge * p.group * 2 * DIM * LN * NV + (e - ge * p.group) + (long long)p.group * (l + LN * 2 * a);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            R sm = R(0), sp = R(0);
#pragma unroll
            for (int q = 0; q < M; ++q) {
                const R u = s[pt[q] + S::VS * v];
                sm = fma(p.lm[q], u, sm);
                sp = fma(p.lp[q], u, sp);
            }
            R* w = ub + (long long)p.group * LN * 2 * DIM * v;  // face_word(e, a, s, l, v)
            w[0] = sm;
            w[(long long)p.group * LN] = sp;
        }
    }
}

template <class R, int DIM, int M, int NE, bool SRC, int HEADB, int BAR, int NTHR, bool FACES = false, int GS = NE,
          bool CS = false, int XP = 0>
__device__ __forceinline__ void lines_sweeps(unsigned char* buf, R* acc, const Params<R>& p, int t, int bar_id = 0,
                                             long long E0 = 0, int nvalid = NE) {
    static_assert(XP == 0 || (!CS && HEADB == 0), "padded chunks: one thread per line, an aligned chunk");
    // NTHR: line slots per sweep iteration (LineMap); CS: d component groups of NTHR threads
    constexpr int NALL = CS ? DIM * NTHR : NTHR;
    R* s = reinterpret_cast<R*>(buf + HEADB);
#ifdef HF_IO_ONLY  // measurement build: chunk traffic only, no sweeps (tools/gpu_ab_io.sh)
    return;
#endif
    auto sync = [&] {
        if constexpr (BAR == 0) __syncthreads();
        else if constexpr (BAR < 0) named_bar_sync(bar_id, NALL);  // runtime barrier id (consumer groups)
        else named_bar_sync(BAR, NALL);
    };
    // lines of sweep A in the bank-conflict-free order of kLineMap
    auto sweep = [&](auto a_tag, auto phase_tag) {
        constexpr int A = decltype(a_tag)::value;
        constexpr int PH = decltype(phase_tag)::value;
        using LM = LineMap<R, DIM, M, NE, A, NTHR, GS, XP>;
        const unsigned short* map = kLineMap<R, DIM, M, NE, A, NTHR, GS, XP>.off;
        if constexpr (!CS) {
#pragma unroll 1
            for (int k = 0; k < LM::ITERS; ++k) {
                const int o = map[k * NTHR + t];
                if (o != 0xFFFF) lines_sweep<R, DIM, M, NE, SRC, A, PH, GS, XP>(s, acc, p, o);
            }
        } else {
            // warp-uniform component: component group b = threads [b*NTHR, (b+1)*NTHR)
            const int b = t / NTHR, tt = t - b * NTHR;
            auto load = [&](int o, Pair<R> (&W)[M]) {
                if (b == 0) comp_load<R, DIM, M, NE, A, 0, GS>(s, p, o, W);
                else if (DIM == 2 || b == 1) comp_load<R, DIM, M, NE, A, 1, GS>(s, p, o, W);
                else comp_load<R, DIM, M, NE, A, (DIM == 3 ? 2 : 1), GS>(s, p, o, W);
            };
            auto emit = [&](int o, Pair<R> (&W)[M]) {
                if (b == 0) comp_contract_emit<R, DIM, M, NE, SRC, A, 0, PH, GS>(s, acc, p, o, W);
                else if (DIM == 2 || b == 1) comp_contract_emit<R, DIM, M, NE, SRC, A, 1, PH, GS>(s, acc, p, o, W);
                else comp_contract_emit<R, DIM, M, NE, SRC, A, (DIM == 3 ? 2 : 1), PH, GS>(s, acc, p, o, W);
            };
#pragma unroll 1
            for (int k = 0; k < LM::ITERS; ++k) {
                const int o = map[k * NTHR + tt];
                Pair<R> W[M];
                if (o != 0xFFFF) load(o, W);
                // the last sweep overwrites V_A with its final value (component A's thread)
                // while the other components of the line still read it: all loads first
                if constexpr (PH == 2) sync();
                if (o != 0xFFFF) emit(o, W);
            }
        }
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    if constexpr (FACES) {
        lines_project_faces<R, DIM, M, NE, GS, XP>(s, p, E0, t, NALL, nvalid);
        sync();  // every line is read before sweep 0 writes in place
    }
    if constexpr (DIM == 3) {
        sweep(I0{}, I0{});
        sync();
        sweep(I1{}, I1{});
        sync();
        sweep(I2{}, I2{});
    } else {
        sweep(I0{}, I0{});
        sync();
        sweep(I1{}, I2{});
    }
}

// Runtime head (bytes, a multiple of sizeof(R), < 16) -> compile-time HEADB.
// Chunks whose byte size is a multiple of 16 always start aligned: one instance.
template <class R, int DIM, int M, int NE, bool SRC, int BAR, int NTHR, bool FACES = false, int GS = NE,
          bool CS = false, int XP = 0>
__device__ __forceinline__ void lines_sweeps_at(unsigned char* buf, int head, R* acc, const Params<R>& p, int t,
                                                int bar_id = 0, long long E0 = 0, int nv = NE) {
    if constexpr (XP > 0) {  // padded chunks are staged by a tensor copy or word by word: head 0
        lines_sweeps<R, DIM, M, NE, SRC, 0, BAR, NTHR, FACES, GS, CS, XP>(buf, acc, p, t, bar_id, E0, nv);
    } else if constexpr (LinesShape<R, DIM, M, NE>::IN_BYTES % 16 == 0) {
        lines_sweeps<R, DIM, M, NE, SRC, 0, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv);
    } else if constexpr (sizeof(R) == 8) {
        if (head == 0) lines_sweeps<R, DIM, M, NE, SRC, 0, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv);
        else lines_sweeps<R, DIM, M, NE, SRC, 8, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv);
    } else {
        switch (head) {
            case 0: lines_sweeps<R, DIM, M, NE, SRC, 0, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv); break;
            case 4: lines_sweeps<R, DIM, M, NE, SRC, 4, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv); break;
            case 8: lines_sweeps<R, DIM, M, NE, SRC, 8, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv); break;
            default: lines_sweeps<R, DIM, M, NE, SRC, 12, BAR, NTHR, FACES, GS, CS>(buf, acc, p, t, bar_id, E0, nv); break;
        }
    }
}

// No work between the sweeps and the store (the plain fused kernel).
struct NoChunkHook {};

// One chunk of the lines kernel: stage, sweeps, [hook], store.  `hook(chunk, E0, nvalid, tid)`
// runs on the finished divergence in shared memory (layout [v][pt][el] of NE elements, GS ==
// NE) between two CTA barriers -- the FR interface correction of hf_fr.cuh uses it to apply
// stages 4+5 before the chunk leaves shared memory.
template <class R, int DIM, int M, int NE, bool SRC, int LPT, bool FACES, int GS, bool CS, class Hook, int XP = 0>
__device__ __forceinline__ void lines_chunk(const Params<R>& p, Hook&& hook) {
    using S = LinesShape<R, DIM, M, NE, LPT, GS, CS, XP>;
    static_assert(XP == 0 || LPT == 1, "padded chunks: one line per thread");
    constexpr int BS = S::BS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using IO = typename S::IO;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    unsigned char* buf = smem_raw + S::HDR;
    R* acc = reinterpret_cast<R*>(buf + S::BUF_BYTES);

    const int tid = threadIdx.x;
    pdl_launch_dependents();  // the next kernel of the stream may take SM slots as chunks retire
    pdl_wait();               // ... and this one reads / writes HBM only after the previous kernel
    // chunk -> first element E0 and its nvalid elements: NE consecutive elements, or in
    // tile mode sub-chunk `sub` of group `grp` (the group's last sub-chunk may be short)
    const long long b = p.chunk0 + static_cast<long long>(blockIdx.x);
    long long grp, E0;
    int sub = 0, nvalid = NE;
    if (p.tile) {
        grp = b / p.sub_per_group;
        sub = static_cast<int>(b - grp * p.sub_per_group);
        E0 = grp * p.group + sub * NE;
        nvalid = p.group - sub * NE < NE ? p.group - sub * NE : NE;
    } else {
        E0 = b * NE;
        grp = E0 / p.group;
    }
    const int el0 = static_cast<int>(E0 - grp * p.group);
    const long long gbase = grp * p.group_words + el0;
    // one contiguous byte range: the chunk is one group (GS = NE) or NE / GS whole groups
    const bool contiguous = (p.group == GS);
    const bool full = E0 + nvalid <= p.n_elem;
    // padded grouped chunk (S::PADW): one exact 16-byte-multiple copy per group, no superset
    const bool fast = XP ? (p.xpad && full && contiguous)
                  : p.tile ? (p.fast_ok && full)
                           : (S::PADW ? (p.fast_ok && full && contiguous)
                                      : chunk_bulk_ok<R, S::IN_WORDS>(p, gbase, full, contiguous));
    const int head = (fast && !XP && !p.tile && !S::PADW) ? IO::head_bytes(p.u + gbase, contiguous) : 0;
    R* s = reinterpret_cast<R*>(smem_raw + S::HDR);  // guarded path (head == 0)
    __shared__ long long ebase[NE];                   // guarded path: element word bases, -1 = absent

    // ---------------- stage the chunk into shared memory ----------------
    if (fast) {
        if (tid == 0) {
            mbar_init(bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if constexpr (XP > 0) {  // one tensor copy: the box one pad wider than the row (and the
                                 // k-plane), the pad out of bounds and zero-filled
            if (tid == 0) {
                mbar_arrive_expect_tx(bar, uint32_t(S::NV * S::VS * int(sizeof(R))));
                if constexpr (DIM == 3) tma_load_5d(buf, &p.tm_u, 0, 0, 0, 0, static_cast<int>(grp), bar);
                else tma_load_4d(buf, &p.tm_u, 0, 0, 0, static_cast<int>(grp), bar);
            }
        } else if constexpr (S::PADW > 0) {  // one bulk copy per group, each to its padded slot
            if (tid == 0) mbar_arrive_expect_tx(bar, uint32_t(S::IN_BYTES));
            __syncthreads();
            for (int g = tid; g < NE / GS; g += BS)
                bulk_g2s(buf + g * S::BLKP * int(sizeof(R)), p.u + gbase + static_cast<long long>(g) * S::BLK,
                         S::BLK * int(sizeof(R)), bar);
        } else if (p.tile) {
            if (tid == 0) {  // one TMA tensor copy: the box {NE, m, m^(d-1), n_v, 1}; e_l >= group zero-filled
                mbar_arrive_expect_tx(bar, uint32_t(S::IN_BYTES));
                tma_load_5d(buf, &p.tm_u, sub * NE, 0, 0, 0, static_cast<int>(grp), bar);
            }
        } else if (tid < 32) {
            if (tid == 0) mbar_arrive_expect_tx(bar, IO::tx_bytes(p.u + gbase, contiguous));
            __syncwarp();
            IO::load(buf, p.u + gbase, p.group, contiguous, bar, tid);
        }
        mbar_wait_parity(bar, 0);
    } else {
        // guarded path (any group, alignment or partial chunk): the element's word base once per
        // element (the 64-bit group arithmetic), then one cp.async word copy per staged word
        // (LDGSTS: no register round trip, many in flight; consecutive threads read
        // consecutive words of a row wherever the group allows)
        for (int el = tid; el < NE; el += BS) {
            const long long e = E0 + el;
            long long b = -1;
            if (el < nvalid && e < p.n_elem) {
                const long long ge = e / p.group;
                b = ge * p.group_words + (e - ge * p.group);
            }
            ebase[el] = b;
        }
        __syncthreads();
        const long long G = p.group;
        for (int idx = tid; idx < S::IN_WORDS; idx += BS) {
            const int blk = idx / S::BLK, rem = idx - blk * S::BLK;  // image word -> (el, row)
            const int el = blk * GS + rem % GS;
            const int row = rem / GS;
            const long long b = ebase[el];
            R* dst = s + S::staged(idx);
            if (b >= 0) cp_async_word(dst, p.u + b + G * row);
            else *dst = R(0);
        }
        cp_async_wait_all();
        __syncthreads();
    }

    // ---------------- d sweeps ----------------
    lines_sweeps_at<R, DIM, M, NE, SRC, 0, (CS ? S::NT : BS), FACES, GS, CS, XP>(buf, head, acc, p, tid, 0, E0, nvalid);
    if constexpr (!std::is_same_v<std::decay_t<Hook>, NoChunkHook>) {
        __syncthreads();
        hook(reinterpret_cast<R*>(buf + head), E0, nvalid, tid);
    }

    // ---------------- write the finished chunk ----------------
    if (fast) {
        fence_proxy_async_smem();
        __syncthreads();
        if constexpr (XP > 0) {
            if (tid == 0) {  // the pad words are out of bounds: clipped
                if constexpr (DIM == 3) tma_store_5d(&p.tm_out, 0, 0, 0, 0, static_cast<int>(grp), buf);
                else tma_store_4d(&p.tm_out, 0, 0, 0, static_cast<int>(grp), buf);
                bulk_commit();
                bulk_wait_read_all();
            }
        } else if constexpr (S::PADW > 0) {
            for (int g = tid; g < NE / GS; g += BS)
                bulk_s2g(p.out + gbase + static_cast<long long>(g) * S::BLK, buf + g * S::BLKP * int(sizeof(R)),
                         S::BLK * int(sizeof(R)));
            bulk_commit();
            bulk_wait_read_all();
        } else if (p.tile) {
            if (tid == 0) {  // elements past the group's end are clipped by the tensor map
                tma_store_5d(&p.tm_out, sub * NE, 0, 0, 0, static_cast<int>(grp), buf);
                bulk_commit();
                bulk_wait_read_all();
            }
        } else if (tid < 32) {
            IO::store(p.out + gbase, buf, p.group, contiguous, tid);
            bulk_wait_read_all();
        }
    } else {
        __syncthreads();
        const long long G = p.group;
        for (int idx = tid; idx < S::IN_WORDS; idx += BS) {
            const int blk = idx / S::BLK, rem = idx - blk * S::BLK;
            const int el = blk * GS + rem % GS;
            const int row = rem / GS;
            const long long b = ebase[el];
            if (b >= 0) __stcs(p.out + b + G * row, s[S::staged(idx)]);
        }
    }
}

template <class R, int DIM, int M, int NE, bool SRC, int LPT = 1, bool FACES = false, int GS = NE, bool CS = false,
          int XP = 0>
__global__ void __launch_bounds__(LinesShape<R, DIM, M, NE, LPT, GS, CS, XP>::BS)
    hf_lines_kernel(const __grid_constant__ Params<R> p) {
    lines_chunk<R, DIM, M, NE, SRC, LPT, FACES, GS, CS, NoChunkHook, XP>(p, NoChunkHook{});
}

}  // namespace hfb
