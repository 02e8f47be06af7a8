// hf_common.cuh -- shared definitions for the B200 (sm_100a) fused flux +
// divergence kernels: the launch parameter block, the AoSoA layout
// (layout.hpp:128-134), and the PTX wrappers for mbarriers and bulk async
// copies (cp.async.bulk, TMA's non-tensor form).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace hfb {

constexpr int kMaxM = 9;  // m = p+1 <= 9 (d=2 p=8)
constexpr int kMaxH = 5;  // rows of the even-odd split: i <= m/2

__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }
__host__ __device__ constexpr int n_vars_c(int d) { return 1 + d + d * d; }
__host__ __device__ constexpr int var_grad_c(int d, int b, int a) { return 1 + d + b * d + a; }

// Everything a launch needs, passed by value as a __grid_constant__ so that the
// operator matrix and physical constants live in the kernel-parameter constant
// bank (immediate c[0x0][...] operands in DFMA/FFMA) and launches are
// reentrant across streams with no per-device __constant__ state.
template <class R>
struct Params {
    R D[kMaxM * kMaxM];  // derivative matrix, row-major m x m (operators.hpp:49-74)
    // Even-odd split of D for Gauss-Legendre nodes (x_{m-1-i} = -x_i, so
    // D(m-1-i, m-1-t) = -D(i, t)):  with S_t = f_t + f_{m-1-t}, A_t = f_t - f_{m-1-t} (t < m/2),
    //   X_i = sum_t DE[i][t] S_t + DC[i] f_mid,  Y_i = sum_t DO[i][t] A_t,
    //   (D f)_i = X_i + Y_i,  (D f)_{m-1-i} = Y_i - X_i   (i < m/2),  (D f)_mid = sum_t DO[mid][t] A_t.
    R DE[kMaxH * kMaxH];  // (D(i,t) + D(i,m-1-t)) / 2, row-major [i][t], i <= m/2, t < m/2
    R DO[kMaxH * kMaxH];  // (D(i,t) - D(i,m-1-t)) / 2
    R DC[kMaxH];          // D(i, mid) for odd m
    R nu, zeta, invT;    // PhysParams (equations.hpp:14-24), 1/T precomputed
    R jac[3];            // constant per-axis metric (oracle.hpp:47)
    R jac_invT[3];       // jac[a] / T : gradient-row scale
    R xg[kMaxM];         // Gauss-Legendre nodes (mapped elements: the reference point of each node)
    R lm[kMaxM], lp[kMaxM];  // Lagrange basis at xi = -1, +1 (FR stage 1 fused into the lines kernel)
    const R* __restrict__ u;  // input field, AoSoA (layout.hpp:128-134)
    R* __restrict__ out;      // divergence, same layout
    R* __restrict__ ws;       // unfused only: flux workspace
    const R* __restrict__ geo;  // mapped elements only: 2^d corners per element (hf_mapped.cuh)
    R* __restrict__ uf;         // lines kernel with FACES: the FR face array (stage 1) written beside the divergence
    long long n_elem;
    long long group_words;    // group * m^d * n_v
    long long total_words;    // n_groups * group_words (allocation size of u and out)
    long long chunk0;         // first chunk (of NE elements) this launch covers
    long long n_chunks;       // pipelined kernel: number of full chunks to process
    int group;
    int fast_ok;              // host-verified: bulk-copy alignment holds for full chunks
    // Tile mode (lines kernel, group != chunk): chunk b is sub-chunk b % sub_per_group of
    // group b / sub_per_group, a box of NE elements x all rows moved by ONE TMA tensor copy
    // per direction over the 5-d view {e_l, i, (j,k), v, group} of the AoSoA field.
    int tile;
    int sub_per_group;        // ceil(group / NE)
    // Padded chunks (lines variants 25-27): tm_u / tm_out hold the view {x-row, j, (k), v,
    // group} of a field whose group is the chunk, the box wider than the row / taller than the
    // k-plane by the pad (encode_xpad_map).
    int xpad;
    CUtensorMap tm_u;         // 64-byte aligned descriptors, read from the parameter space
    CUtensorMap tm_out;
};

// FR face array (stage 1 output, hf_fr.cuh): word of (element e, axis a, side s,
// line l = the line's transverse indices, variable v), AoSoA with the field's group.
__device__ __forceinline__ long long face_word(int dim, int m, long long group, long long e, int a, int s, int l,
                                               int v) {
    const int nv = 1 + dim + dim * dim;
    const int L = dim == 3 ? m * m : m;
    return (e / group) * group * 2 * dim * L * nv + e % group + group * (l + (long long)L * (s + 2 * (a + dim * v)));
}

// line l of axis a, point t -> point index i + m j + m^2 k
template <int DIM, int M>
__device__ __forceinline__ int fr_line_point(int a, int l, int t) {
    const int t0 = l % M, t1 = l / M;
    if (a == 0) return t + M * t0 + M * M * (DIM == 3 ? t1 : 0);
    if (a == 1) return t0 + M * t + M * M * (DIM == 3 ? t1 : 0);
    return t0 + M * t1 + M * M * t;
}

// ---------------------------------------------------------------------------------------------
// PTX: mbarrier + cp.async.bulk (SASS UBLKCP / SYNCS.*)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over a subset of the CTA's warps (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0, both ends 16B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// shared -> global bulk copy, bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// one word (4 or 8 bytes) global -> shared, async (LDGSTS)
template <class R>
__device__ __forceinline__ void cp_async_word(R* dst_smem, const R* src_gmem) {
    if constexpr (sizeof(R) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// TMA tensor copies (SASS UTMALDG / UTMASTG) of one 5-d box; `tmap` is the generic
// address of a CUtensorMap in the __grid_constant__ parameter block.
__device__ __forceinline__ void tma_load_5d(void* dst_smem, const CUtensorMap* tmap, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(smem_u32(dst_smem)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst_smem, const CUtensorMap* tmap, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst_smem)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* tmap, int c0, int c1, int c2, int c3,
                                             const void* src_smem) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src_smem))
                 : "memory");
}

__device__ __forceinline__ void tma_store_5d(const CUtensorMap* tmap, int c0, int c1, int c2, int c3, int c4,
                                             const void* src_smem) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
            reinterpret_cast<uint64_t>(tmap)),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src_smem))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}


// Programmatic dependent launch (launch_kernel in hf_launch.cuh sets the attribute): a
// kernel may be scheduled while the previous kernel of its stream drains; it waits for
// that kernel's completion and memory flush before its first global access.  No-ops for
// an ordinary launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// make generic-proxy shared-memory writes visible to the async proxy (bulk store)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------------------------
// Value pairs for the line contraction.  The lines kernel contracts two lines
// with the same D row at once (V_b and the momentum flux M_ba).  For FP32 the
// pair is a float2 driven by the sm_100 packed instructions (FFMA2 / FMUL2 /
// FADD2: two FP32 lanes per issued instruction, the scalar D operand broadcast
// from a uniform register), which halves the FP32 instruction count of the
// contraction; for FP64 it is two scalar DFMAs.
// ---------------------------------------------------------------------------------------------
template <class R>
struct Pair;

template <>
struct Pair<float> {
    float2 v;
    __device__ __forceinline__ float x() const { return v.x; }
    __device__ __forceinline__ float y() const { return v.y; }
    __device__ __forceinline__ static Pair make(float a, float b) { return {make_float2(a, b)}; }
};

template <>
struct Pair<double> {
    double a, b;
    __device__ __forceinline__ double x() const { return a; }
    __device__ __forceinline__ double y() const { return b; }
    __device__ __forceinline__ static Pair make(double x, double y) { return {x, y}; }
};

__device__ __forceinline__ unsigned long long f2_bits(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 f2_from(unsigned long long r) { return *reinterpret_cast<float2*>(&r); }

// s * a
__device__ __forceinline__ Pair<float> pmul(float s, Pair<float> a) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(make_float2(s, s))), "l"(f2_bits(a.v)));
    return {f2_from(r)};
}
__device__ __forceinline__ Pair<double> pmul(double s, Pair<double> a) { return {s * a.a, s * a.b}; }
// s * a + c
__device__ __forceinline__ Pair<float> pfma(float s, Pair<float> a, Pair<float> c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(f2_bits(make_float2(s, s))), "l"(f2_bits(a.v)), "l"(f2_bits(c.v)));
    return {f2_from(r)};
}
__device__ __forceinline__ Pair<double> pfma(double s, Pair<double> a, Pair<double> c) {
    return {fma(s, a.a, c.a), fma(s, a.b, c.b)};
}
__device__ __forceinline__ Pair<float> padd(Pair<float> a, Pair<float> b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a.v)), "l"(f2_bits(b.v)));
    return {f2_from(r)};
}
__device__ __forceinline__ Pair<double> padd(Pair<double> a, Pair<double> b) { return {a.a + b.a, a.b + b.b}; }
__device__ __forceinline__ Pair<float> psub(Pair<float> a, Pair<float> b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a.v)), "l"(f2_bits(b.v)));
    return {f2_from(r)};
}
__device__ __forceinline__ Pair<double> psub(Pair<double> a, Pair<double> b) { return {a.a - b.a, a.b - b.b}; }

// streaming (read-once) global load for the generic loader
template <class R>
__device__ __forceinline__ R ld_stream(const R* p) {
    return __ldcs(p);
}

}  // namespace hfb
