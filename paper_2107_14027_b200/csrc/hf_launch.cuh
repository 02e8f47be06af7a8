// hf_launch.cuh -- per-configuration launch shapes and the templated launchers.
//
// The reference picks one static configuration per (p, precision) from the
// paper's Volta measurements (preset_table, presets.hpp:25-37;
// default_lines_n, presets.hpp:86-103, sized for a 96 KiB shared-memory cap).
// On B200 (227 KB shared per CTA, 228 KB per SM) the lines kernel's default
// chunk (NE0) is sized for about three co-resident CTAs per SM, so one CTA can
// be staging its next chunk through the bulk-copy engine while the others
// compute; the variants below (chunk size, one chunk per CTA or a persistent
// TMA ring, consumer groups, lines per thread) are what the measured selection
// (hf_select_table.inc, tools/select_methods.py) chooses from.
#pragma once

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hf_common.cuh"
#include "hf_lines.cuh"
#include "hf_lines_pipe.cuh"
#include "hf_mapped.cuh"
#include "hf_planar.cuh"
#include "hf_unfused.cuh"

namespace hfb {

struct KInfo {
    int method = 0;
    int elems_per_cta = 0;
    int block_threads = 0;
    int shared_bytes = 0;
    int registers = 0;
    long long grid = 0;
    int bulk_path = 0;
    int blocks_per_sm = 0;
    char name[96] = {0};
};

constexpr int kLinesSmemBudget = 72 * 1024;
constexpr int kMaxSmemPerCta = 227 * 1024;

// NE0 of (word bytes w, d, m); constexpr and callable at run time (the host's choice of a
// variant for a caller's group, hf_capi.cu) so the two can never disagree.
constexpr int lines_ne0(int w, int dim, int m) {
    const int min_ne = 16 / w;  // a chunk row must be a 16-byte multiple
    int ne = (dim == 2) ? 128 : 64;
    while (ne > min_ne &&
           (128 + size_t(ne) * ipow_c(m, dim) * (n_vars_c(dim) + 1 + dim) * size_t(w) > size_t(kLinesSmemBudget) ||
            ne * ipow_c(m, dim - 1) > 512))
        ne /= 2;
    return ne;
}

template <class R, int DIM, int M>
constexpr int lines_ne_default() {
    static_assert(LinesShape<R, DIM, M, 1>::HDR == 128, "lines_ne0 assumes a 128-byte header");
    return lines_ne0(int(sizeof(R)), DIM, M);
}

// Lines variants.  NE0 = lines_ne_default (about three CTAs per SM).
//   one chunk per CTA (hf_lines_kernel):        0: NE0   1: NE0/2   2: 2*NE0   7: NE0/4
//   persistent TMA ring (hf_lines_pipe_kernel), (elements, stages, consumer groups):
//     3: (NE0, 2, 1)    4: (NE0/2, 3, 1)   5: (NE0/2, 2, 1)   6: (NE0, 3, 1)
//     8: (NE0/4, 3, 1)  9: (NE0/4, 4, 1)
//    10: (NE0/2, 4, 2) 11: (NE0/2, 6, 3)  12: (NE0/4, 8, 4)  13: (NE0/4, 6, 2)
//    14: (NE0, 4, 2)   15: (NE0/4, 6, 3)
//   one chunk per CTA with several lines per thread, (elements, lines per thread):
//    16: (2*NE0, 2)    17: (NE0, 2)       18: (4*NE0, 4)
//   component split (LinesShape CS: d threads per line, one per velocity component):
//    19: one chunk NE0   20: one chunk NE0/2   21: one chunk 2*NE0   22: one chunk NE0/4
//    23: TMA ring (NE0, 2)
// The contiguous bulk path accepts any NE >= 1 (hf_chunk_io.cuh), so the small-NE
// variants exist for every order; a variant whose shape does not fit (shared
// memory, 1024 threads) reports unsupported.
constexpr int kLinesVariants = 28;
constexpr bool is_cs_variant(int v) { return v >= 19 && v <= 23; }
constexpr int kTileRingVariant = 24;  // TMA ring, 2 NE0 elements, 2 stages, 1 group, tile mode
// 25 / 26 / 27: one chunk per CTA of NE0/4, NE0/2, NE0 elements staged padded (LinesShape XP,
// xpad_code): the chunk layout of variants 7 / 1 / 0 with an x-row stride (one-element
// chunks: a k-plane stride) that spreads the lines over the banks.
constexpr bool is_xpad_variant(int v) { return v >= 25 && v <= 27; }
constexpr int xpad_base_variant(int v) { return v == 25 ? 7 : v == 26 ? 1 : v == 27 ? 0 : v; }

// The measured selection (tools/select_methods.py -> hf_select_table.inc).
struct SelRow {
    int d, p, prec, method, variant;
};
constexpr SelRow kSelect[] = {
#include "hf_select_table.inc"
    {0, 0, 0, 0, 0}};

// Which lines variants the library instantiates.  The production build carries
// the selected variant of every (d, p, precision) plus variants 0 (one chunk per
// CTA), 3 (TMA ring) and 10 (grouped TMA ring), so that every kernel form stays
// parity-tested; the tuning build (make tuning, -DHF_TUNING) carries all of them
// for tools/select_methods.py.
// Lines variant for the FACES form where it differs from the selection: at d3 p6 the
// one-chunk-per-CTA kernel (variant 0, the same chunk as the selected ring) writes
// the faces faster than the TMA ring, whose consumers are the ring's bottleneck
// (fused stages 1+2+3+6, 1e7 points: FP64 657 -> 518 us, FP32 300 -> 288 us;
// profiles/ext_r01e_faces_variant_*.jsonl).  -1: the selected variant.
constexpr int faces_variant_override(int d, int p) { return (d == 3 && p == 6) ? 0 : -1; }

// The FACES (fused FR stage 1) form: the selected variant of each configuration.
template <class R, int DIM, int M, int VARIANT>
constexpr bool variant_faces_built() {
#ifdef HF_TUNING
    return VARIANT == 0 || VARIANT == 3;
#else
#ifdef HF_FACES_AB
    if (VARIANT == 0 || VARIANT == 3) return true;
#endif
    if (VARIANT == faces_variant_override(DIM, M - 1)) return true;
    for (const SelRow& r : kSelect)
        if (r.d == DIM && r.p == M - 1 && r.prec == (sizeof(R) == 8 ? 1 : 0) && r.method == 2 && r.variant == VARIANT)
            return true;
    return false;
#endif
}

// The one-chunk-per-CTA variants (NE0, NE0/2, 2*NE0, NE0/4): the chunk sizes the host
// chooses from for a caller's AoSoA group that is not the selected chunk (tile mode).
constexpr bool is_one_chunk_variant(int v) { return v == 0 || v == 1 || v == 2 || v == 7; }

template <class R, int DIM, int M, int VARIANT>
constexpr bool variant_built() {
#ifdef HF_TUNING
    return true;
#else
    if (is_one_chunk_variant(VARIANT) || VARIANT == 3 || VARIANT == 10) return true;
    // the tile ring (2 NE0 elements, 2 stages): caller groups of >= 32-byte rows at d3 p5,
    // where the one-chunk kernel of that chunk fits one CTA per SM (lines_variant_for_group)
    if (VARIANT == kTileRingVariant) return DIM == 3 && M == 6;
    // the padded one-chunk variants: all three at d3 p3 (parity coverage), else where selected
    if (is_xpad_variant(VARIANT) && DIM == 3 && M == 4) return true;
    for (const SelRow& r : kSelect)
        if (r.d == DIM && r.p == M - 1 && r.prec == (sizeof(R) == 8 ? 1 : 0) && r.method == 2 && r.variant == VARIANT)
            return true;
    return false;
#endif
}
template <int VARIANT>
constexpr bool is_pipe_variant() {
    return !(VARIANT == 0 || VARIANT == 1 || VARIANT == 2 || VARIANT == 7 || (VARIANT >= 16 && VARIANT <= 22) ||
             is_xpad_variant(VARIANT));
}
constexpr int variant_ne_of(int ne0, int v) {
    const int ne = (v == 0 || v == 3 || v == 6 || v == 14 || v == 19 || v == 23 || v == 27)     ? ne0
                   : (v == 1 || v == 4 || v == 5 || v == 10 || v == 11 || v == 20 || v == 26)  ? ne0 / 2
                   : (v == 2 || v == 16 || v == 21 || v == 24)                      ? ne0 * 2
                   : (v == 17)                                                      ? ne0
                   : (v == 18)                                                      ? ne0 * 4
                                                                                    : ne0 / 4;
    return ne >= 1 ? ne : 0;
}
template <class R, int DIM, int M, int VARIANT>
constexpr int variant_ne() {
    return variant_ne_of(lines_ne_default<R, DIM, M>(), VARIANT);
}
template <int VARIANT>
constexpr int pipe_stages() {
    switch (VARIANT) {
        case 4: case 6: case 8: return 3;
        case 9: case 10: case 14: return 4;
        case 11: case 13: case 15: return 6;
        case 12: return 8;
        default: return 2;
    }
}
template <int VARIANT>
constexpr int lines_per_thread() {
    return VARIANT == 16 || VARIANT == 17 ? 2 : (VARIANT == 18 ? 4 : 1);
}
template <int VARIANT>
constexpr int pipe_groups() {
    switch (VARIANT) {
        case 10: case 13: case 14: return 2;
        case 11: case 15: return 3;
        case 12: return 4;
        default: return 1;
    }
}

template <class R, int M>
constexpr int planar_ne() {
    int ne = 64;
    while (ne > 8 && ne * M > 128) ne /= 2;
    return ne;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Layouts whose full chunks take the bulk path (hf_chunk_io.cuh): the group is
// the chunk (one contiguous range, any alignment), or whole 16-byte rows.
template <class R, int NE>
inline bool bulk_layout(int group) {
    if (group == NE) return true;
    return (group % NE == 0) && (NE * sizeof(R)) % 16 == 0 && ((long long)group * sizeof(R)) % 16 == 0;
}

// Tile mode of the lines kernel (hf_lines.cuh): the caller's AoSoA group is not the
// kernel's chunk, so a chunk is NE elements x all rows of one group -- a strided box that
// one TMA tensor copy moves per direction.  TMA needs 16-byte global strides (group * w),
// a 16-byte box row (NE * w) and 16-byte aligned buffers.
template <class R, int NE>
inline bool tile_layout(int group) {
    return group != NE && (NE * sizeof(R)) % 16 == 0 && ((long long)group * sizeof(R)) % 16 == 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeTiled encode_tiled_fn() {
    static EncodeTiled fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return reinterpret_cast<EncodeTiled>(f);
    }();
    return fn;
}

// The 5-d view {e_l: group, i: m, (j,k): m^(d-1), v: n_v, group index: n_groups} of an
// AoSoA field (layout.hpp:128-134), box {NE, m, m^(d-1), n_v, 1}: the box lands in shared
// memory as [v][pt][e_l], exactly the chunk layout of the lines kernel.
template <class R>
inline bool encode_chunk_map(CUtensorMap* tm, const void* base, int dim, int m, int group, long long n_groups,
                             int ne) {
    EncodeTiled enc = encode_tiled_fn();
    if (!enc) return false;
    const int nv = n_vars_c(dim);
    const long long mh = dim == 3 ? (long long)m * m : m;
    const cuuint64_t w = sizeof(R);
    const cuuint64_t dims[5] = {cuuint64_t(group), cuuint64_t(m), cuuint64_t(mh), cuuint64_t(nv),
                                cuuint64_t(n_groups)};
    const cuuint64_t strides[4] = {group * w, group * w * m, group * w * m * mh, group * w * m * mh * nv};
    const cuuint32_t box[5] = {cuuint32_t(ne), cuuint32_t(m), cuuint32_t(mh), cuuint32_t(nv), 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = enc(tm, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The padded-chunk view of a field whose group is the chunk: d3 {x-row (i, e_l): m NE words,
// j: m, k: m, v: n_v, group} with box {rs, pr, m, n_v, 1}; d2 {x-row, j, v, group} with box
// {rs, m, n_v, 1}.  The words past each row (rs > m NE) and the rows past each k-plane
// (pr > m) are out of bounds -- zero-filled on load, clipped on store -- so the box lands in
// shared memory with the padded row and plane strides.  16-byte x-rows only.
template <class R>
inline bool encode_xpad_map(CUtensorMap* tm, const void* base, int dim, int m, int ne, long long n_groups, int rs,
                            int pr) {
    EncodeTiled enc = encode_tiled_fn();
    const cuuint64_t w = sizeof(R);
    const cuuint64_t rw = cuuint64_t(m) * ne;
    if (!enc || (rw * w) % 16 != 0 || rs > 256 || pr > 256) return false;
    const cuuint64_t nv = cuuint64_t(n_vars_c(dim));
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r;
    if (dim == 3) {  // {x-row, j, k, v, group}, box {rs, pr, m, n_v, 1}: rows j >= m are the plane pad
        const cuuint64_t dims[5] = {rw, cuuint64_t(m), cuuint64_t(m), nv, cuuint64_t(n_groups)};
        const cuuint64_t strides[4] = {rw * w, rw * w * m, rw * w * m * m, rw * w * m * m * nv};
        const cuuint32_t box[5] = {cuuint32_t(rs), cuuint32_t(pr), cuuint32_t(m), cuuint32_t(nv), 1};
        r = enc(tm, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t dims[4] = {rw, cuuint64_t(m), nv, cuuint64_t(n_groups)};
        const cuuint64_t strides[3] = {rw * w, rw * w * m, rw * w * m * nv};
        const cuuint32_t box[4] = {cuuint32_t(rs), cuuint32_t(m), cuuint32_t(nv), 1};
        r = enc(tm, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

// Padded-chunk launch set-up (lines variants 25-27, LinesShape XP): the group must be the
// chunk with 16-byte x-rows no wider than a tensor box and 16-byte aligned buffers; then both
// tensor maps are encoded and p.xpad set.  false: run the same chunk unpadded.
template <class R, int DIM, int M, int NE, class SX>
inline bool setup_xpad(Params<R>& p) {
    bool ok = p.group == NE && (M * NE * sizeof(R)) % 16 == 0 && SX::RS <= 256 &&
              (p.u == nullptr || (aligned16(p.u) && aligned16(p.out)));
    if (ok && p.u != nullptr && p.n_elem > 0) {
        const long long n_groups = (p.n_elem + p.group - 1) / p.group;
        ok = encode_xpad_map<R>(&p.tm_u, p.u, DIM, M, NE, n_groups, SX::RS, SX::PR) &&
             encode_xpad_map<R>(&p.tm_out, p.out, DIM, M, NE, n_groups, SX::RS, SX::PR);
        p.xpad = ok ? 1 : 0;
    }
    return ok;
}

// Kernel launch with programmatic dependent launch (PDL): consecutive fused launches on
// a stream overlap one kernel's launch and ramp-up with the previous one's tail; the
// kernels wait (griddepcontrol.wait) before touching HBM, so stream order is kept.
// HF_PDL=0 in the environment launches without the attribute (A/B measurements).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("HF_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <class... Args>
inline cudaError_t launch_kernel(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 const Args&... args) {
    if (!pdl_enabled()) {
        kernel<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <class K>
inline int set_smem_attr(K kernel, size_t smem) {
    // the default 48 KB limit counts static + dynamic shared memory; the kernels' static
    // arrays (element bases, FR face pointers) stay below 8 KB, so opt in from 40 KB of dynamic
    if (smem > 40 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return int(e);
    }
    return 0;
}

template <class K>
inline void fill_regs(K kernel, KInfo* info) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess) {
        info->registers = fa.numRegs;
        int b = 0;
        if (set_smem_attr(kernel, size_t(info->shared_bytes)) == 0 &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, info->block_threads, size_t(info->shared_bytes)) ==
                cudaSuccess)
            info->blocks_per_sm = b;
        else
            cudaGetLastError();
    } else {
        cudaGetLastError();
        info->registers = 0;
    }
}

inline const char* prec_name(size_t w) { return w == 4 ? "fp32" : "fp64"; }

// Launch (or, with dry = true, only describe) the lines kernel.
template <class R, int DIM, int M, int NE, bool SRC, int LPT = 1, bool FACES = false, int GS = NE, bool CS = false,
          int XP = 0>
cudaError_t launch_lines(Params<R> p, cudaStream_t st, KInfo* info, bool dry) {
    if constexpr (XP > 0) {
        // padded chunks: the group is the chunk, 16-byte x-rows no wider than a tensor box
        // (256 words with the pad), aligned buffers, both tensor maps encoded; else the same
        // chunk unpadded
        if (!setup_xpad<R, DIM, M, NE, LinesShape<R, DIM, M, NE, LPT, GS, CS, XP>>(p))
            return launch_lines<R, DIM, M, NE, SRC, LPT, FACES, GS, CS, 0>(p, st, info, dry);
    }
    using S = LinesShape<R, DIM, M, NE, LPT, GS, CS, XP>;
    auto kernel = hf_lines_kernel<R, DIM, M, NE, SRC, LPT, FACES, GS, CS, XP>;
    const bool tile = GS == NE && tile_layout<R, NE>(p.group) && (p.u == nullptr || (aligned16(p.u) && aligned16(p.out)));
    const long long n_groups = (p.n_elem + p.group - 1) / p.group;
    const int sub = (p.group + NE - 1) / NE;
    const long long grid = tile ? n_groups * sub : (p.n_elem + NE - 1) / NE;
    // grouped chunks: one contiguous image, or (S::PADW) one exact copy per group -- then every
    // group must start 16-byte aligned (group_words * w a multiple of 16, aligned buffers)
    const bool fast_layout =
        tile || (GS == NE ? bulk_layout<R, NE>(p.group)
                          : p.group == GS && (S::PADW == 0 || (p.group_words * (long long)sizeof(R)) % 16 == 0));
    if (info) {
        info->method = 2;
        info->elems_per_cta = NE;
        info->block_threads = S::BS;
        info->shared_bytes = int(S::SMEM);
        info->grid = grid;
        info->bulk_path = fast_layout ? 1 : 0;
        if (GS != NE)
            std::snprintf(info->name, sizeof(info->name), "hf_lines_d%d_p%d_%s_ne%d_g%d%s", DIM, M - 1,
                          prec_name(sizeof(R)), NE, GS, SRC ? "_src" : "");
        else if (LPT == 1)
            std::snprintf(info->name, sizeof(info->name), "hf_lines_d%d_p%d_%s_ne%d%s%s%s%s", DIM, M - 1,
                          prec_name(sizeof(R)), NE, CS ? "_cs" : "", XP ? "_xp" : "", tile ? "_tile" : "",
                          SRC ? "_src" : "");
        else
            std::snprintf(info->name, sizeof(info->name), "hf_lines_d%d_p%d_%s_ne%d_l%d%s", DIM, M - 1,
                          prec_name(sizeof(R)), NE, LPT, SRC ? "_src" : "");
        if (dry) fill_regs(kernel, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    p.fast_ok = fast_layout && aligned16(p.u) && aligned16(p.out);
    if (tile) {
        p.tile = 1;
        p.sub_per_group = sub;
        if (!encode_chunk_map<R>(&p.tm_u, p.u, DIM, M, p.group, n_groups, NE) ||
            !encode_chunk_map<R>(&p.tm_out, p.out, DIM, M, p.group, n_groups, NE))
            p.fast_ok = 0;  // every chunk takes the guarded path (same results)
    }
    size_t smem = S::SMEM;
#ifdef HF_OCC_PROBE  // measurement build: HF_LINES_MAXCTA=N pads shared memory to <= N CTAs per SM
    if (const char* cap = std::getenv("HF_LINES_MAXCTA")) {
        const size_t want = (228 * 1024) / size_t(std::atoi(cap)) - 1024;
        if (want > smem && want <= size_t(kMaxSmemPerCta)) smem = want;
    }
#endif
    if (int e = set_smem_attr(kernel, smem)) return cudaError_t(e);
    return launch_kernel(kernel, dim3(unsigned(grid)), dim3(S::BS), smem, st, p);
}

inline int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) ==
                                                      cudaSuccess)
            return v;
        cudaGetLastError();
        return 148;
    }();
    return n;
}

// Persistent pipelined lines kernel over the whole chunks, guarded tail through hf_lines_kernel.
template <class R, int DIM, int M, int NE, int STAGES, int GROUPS, bool SRC, bool FACES = false, bool CS = false,
          bool TILE = false>
cudaError_t launch_lines_pipe(Params<R> p, cudaStream_t st, KInfo* info, bool dry) {
    using S = PipeShape<R, DIM, M, NE, STAGES, GROUPS, CS, TILE>;
    using L = LinesShape<R, DIM, M, NE, 1, NE, CS>;
    auto kernel = hf_lines_pipe_kernel<R, DIM, M, NE, STAGES, GROUPS, SRC, FACES, CS, TILE>;
    // TILE ring: a group that is not the chunk goes through TMA tensor copies (tile_layout)
    const bool tile = TILE && !FACES && tile_layout<R, NE>(p.group) &&
                      (p.u == nullptr || (aligned16(p.u) && aligned16(p.out)));
    const bool fast_layout = tile || bulk_layout<R, NE>(p.group);
    const int sub = (p.group + NE - 1) / NE;
    const long long n_groups = (p.n_elem + p.group - 1) / p.group;
    long long n_full = p.n_elem / NE;
    long long n_chunks = (p.n_elem + NE - 1) / NE;
    if (tile) {
        // sub-chunks wholly inside n_elem: every one of the whole groups, and the leading ones
        // of a partial last group; the rest (guarded) go to the tail launch
        const long long whole = p.n_elem / p.group;
        n_full = whole * sub + (p.n_elem - whole * p.group) / NE;
        n_chunks = n_groups * sub;
    }
    // contiguous chunks load a 16-byte superset: keep the allocation's last chunk
    // (whose superset could run past the end) for the guarded tail launch
    if (!tile && p.group == NE && n_full > 0 && n_full * NE == p.n_elem &&
        (p.total_words * (long long)sizeof(R)) % 16 != 0)
        n_full -= 1;
    // resident CTAs per SM: measured once per device (thread-safe: atomics), the
    // shared-memory attribute set on every launch (it is per device)
    static std::atomic<int> bps_cache[16];
    int blocks_per_sm = 0;
    if (!dry) {
        if (int e = set_smem_attr(kernel, S::SMEM)) return cudaError_t(e);
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) {
            cudaGetLastError();
            dev = 0;
        }
        const int slot = dev & 15;
        blocks_per_sm = bps_cache[slot].load(std::memory_order_relaxed);
        if (blocks_per_sm < 1) {
            int b = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, S::BS, S::SMEM) != cudaSuccess || b < 1) {
                cudaGetLastError();
                b = 1;
            }
            bps_cache[slot].store(b, std::memory_order_relaxed);
            blocks_per_sm = b;
        }
    }
    const long long slots = (long long)(blocks_per_sm > 0 ? blocks_per_sm : 1) * num_sms();
    const long long grid = n_full < slots ? n_full : slots;
    if (info) {
        info->method = 2;
        info->elems_per_cta = NE;
        info->block_threads = S::BS;
        info->shared_bytes = int(S::SMEM);
        info->grid = grid;
        info->bulk_path = fast_layout ? 1 : 0;
        if (GROUPS == 1)
            std::snprintf(info->name, sizeof(info->name), "hf_lines_pipe_d%d_p%d_%s_ne%d_s%d%s%s%s", DIM, M - 1,
                          prec_name(sizeof(R)), NE, STAGES, CS ? "_cs" : "", tile ? "_tile" : "", SRC ? "_src" : "");
        else
            std::snprintf(info->name, sizeof(info->name), "hf_lines_pipe_d%d_p%d_%s_ne%d_s%d_g%d%s", DIM, M - 1,
                          prec_name(sizeof(R)), NE, STAGES, GROUPS, SRC ? "_src" : "");
        if (dry) fill_regs(kernel, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    p.fast_ok = fast_layout && aligned16(p.u) && aligned16(p.out);
    if (tile && p.fast_ok) {
        p.tile = 1;
        p.sub_per_group = sub;
        if (!encode_chunk_map<R>(&p.tm_u, p.u, DIM, M, p.group, n_groups, NE) ||
            !encode_chunk_map<R>(&p.tm_out, p.out, DIM, M, p.group, n_groups, NE))
            p.fast_ok = 0;
    }
    if (!p.fast_ok || n_full == 0) return launch_lines<R, DIM, M, NE, SRC, 1, FACES, NE, CS>(p, st, nullptr, false);
    p.chunk0 = 0;
    p.n_chunks = n_full;
    cudaError_t e = launch_kernel(kernel, dim3(unsigned(grid)), dim3(S::BS), S::SMEM, st, p);
    if (e != cudaSuccess) return e;
    if (n_full < n_chunks) {  // the partial (or allocation-final) chunk(s)
        auto tail = hf_lines_kernel<R, DIM, M, NE, SRC, 1, FACES, NE, CS>;
        if (int e2 = set_smem_attr(tail, L::SMEM)) return cudaError_t(e2);
        p.chunk0 = n_full;
        e = launch_kernel(tail, dim3(unsigned(n_chunks - n_full)), dim3(L::BS), L::SMEM, st, p);
    }
    return e;
}

template <class R, int M, int NE, bool SRC>
cudaError_t launch_planar(Params<R> p, cudaStream_t st, KInfo* info, bool dry) {
    using S = PlanarShape<R, M, NE>;
    auto kernel = hf_planar_kernel<R, M, NE, SRC>;
    const long long grid = (p.n_elem + NE - 1) / NE;
    if (info) {
        info->method = 1;
        info->elems_per_cta = NE;
        info->block_threads = S::BS;
        info->shared_bytes = int(S::SMEM);
        info->grid = grid;
        info->bulk_path = 0;
        std::snprintf(info->name, sizeof(info->name), "hf_planar_d3_p%d_%s_ne%d%s", M - 1, prec_name(sizeof(R)), NE,
                      SRC ? "_src" : "");
        if (dry) fill_regs(kernel, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    if (int e = set_smem_attr(kernel, S::SMEM)) return cudaError_t(e);
    kernel<<<dim3(unsigned(grid)), dim3(S::BS), S::SMEM, st>>>(p);
    return cudaGetLastError();
}

// Managed planar: the largest element count (<= planar_ne) whose staged chunk fits one CTA.
template <class R, int M>
constexpr int planar_managed_ne() {
    int ne = planar_ne<R, M>();
    while (ne > 1 && PlanarManagedShape<R, M, 1>::HDR + size_t(ne) * M * M * M * 13 * sizeof(R) + 48 >
                         size_t(kMaxSmemPerCta))
        ne /= 2;
    return ne;
}

template <class R, int M, int NE, bool SRC>
cudaError_t launch_planar_managed(Params<R> p, cudaStream_t st, KInfo* info, bool dry) {
    using S = PlanarManagedShape<R, M, NE>;
    auto kernel = hf_planar_managed_kernel<R, M, NE, SRC>;
    const long long grid = (p.n_elem + NE - 1) / NE;
    const bool fast_layout = bulk_layout<R, NE>(p.group);
    if (info) {
        info->method = 4;
        info->elems_per_cta = NE;
        info->block_threads = S::BS;
        info->shared_bytes = int(S::SMEM);
        info->grid = grid;
        info->bulk_path = fast_layout ? 1 : 0;
        std::snprintf(info->name, sizeof(info->name), "hf_planar_managed_d3_p%d_%s_ne%d%s", M - 1,
                      prec_name(sizeof(R)), NE, SRC ? "_src" : "");
        if (dry) fill_regs(kernel, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    p.fast_ok = fast_layout && aligned16(p.u) && aligned16(p.out);
    if (int e = set_smem_attr(kernel, S::SMEM)) return cudaError_t(e);
    kernel<<<dim3(unsigned(grid)), dim3(S::BS), S::SMEM, st>>>(p);
    return cudaGetLastError();
}

// Mapped elements: the largest power-of-two chunk (<= 64 / 128 elements) within
// the measured shared-memory budget and <= 512 lines.
template <class R, int DIM, int M>
constexpr int mapped_ne() {
    // shared-memory budget of the chunk (U + partial sums + corners), measured per
    // (d, p, precision) over 32 / 64 KB (profiles/ext_r01e_mapped_kb*.jsonl):
    // small chunks win where the element count then avoids bank-class collisions
    // of the x-lines and more CTAs hide the chunk loads (d3 p1 FP64 643 -> 522 us,
    // d2 p3 FP64 293 -> 225 us); HF_MAPPED_KB overrides it for such sweeps
#ifdef HF_MAPPED_KB
    constexpr int KB = HF_MAPPED_KB;
#else
    // re-checked under sustained (power-capped) load, profiles/r02/mapped_sustained/: d3 p2 FP64
    // and d2 p5 FP32 move to 64 KB (+5 %, +4 %); every other budget holds
    constexpr int KB = DIM == 3 ? ((M == 2 || (M == 3 && sizeof(R) == 4)) ? 32 : 64)
                                : (sizeof(R) == 4 ? ((M == 2 || M == 4 || M == 5) ? 32 : 64) : (M <= 4 ? 32 : 64));
#endif
    int ne = (DIM == 2) ? 128 : 64;
    while (ne > 1 && (MappedShape<R, DIM, M, 1>::HDR + 48 + size_t(ne) * ipow_c(M, DIM) *
                                                               (2 * n_vars_c(DIM)) * sizeof(R) +
                          size_t(ne) * (1 << DIM) * DIM * sizeof(R) >
                      size_t(KB * 1024) ||
                      ne * ipow_c(M, DIM - 1) > 512))
        ne /= 2;
    // NE*m a multiple of the bank period puts every x-line of a warp in a few bank
    // classes (e.g. p3 FP64, NE 4: 4 of 16); one element less spreads them
    const int bank_words = sizeof(R) == 4 ? 32 : 16;
    if (ne > 1 && (ne * M) % bank_words == 0) ne -= 1;
    return ne;
}

template <class R, int DIM, int M, int NE, bool SRC>
cudaError_t launch_mapped(Params<R> p, cudaStream_t st, KInfo* info, bool dry) {
    using S = MappedShape<R, DIM, M, NE>;
    auto kernel = hf_mapped_kernel<R, DIM, M, NE, SRC>;
    const long long grid = (p.n_elem + NE - 1) / NE;
    const bool fast_layout = bulk_layout<R, NE>(p.group);
    if (info) {
        info->method = 2;
        info->elems_per_cta = NE;
        info->block_threads = S::BS;
        info->shared_bytes = int(S::SMEM);
        info->grid = grid;
        info->bulk_path = fast_layout ? 1 : 0;
        std::snprintf(info->name, sizeof(info->name), "hf_mapped_d%d_p%d_%s_ne%d%s", DIM, M - 1,
                      prec_name(sizeof(R)), NE, SRC ? "_src" : "");
        if (dry) fill_regs(kernel, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    p.fast_ok = fast_layout && aligned16(p.u) && aligned16(p.out);
    if (int e = set_smem_attr(kernel, S::SMEM)) return cudaError_t(e);
    kernel<<<dim3(unsigned(grid)), dim3(S::BS), S::SMEM, st>>>(p);
    return cudaGetLastError();
}

// The staged stage-3 kernel takes a layout when one group's direction block (G * NP * NV
// words) fits a stage of the two-stage ring and moves with 16-byte bulk copies; a thread
// owns at most 4 (point, element) outputs.  Otherwise the gather kernel hf_div_kernel.
template <class R, int DIM, int M>
inline int div_staged_items(const Params<R>& p) {
    constexpr int NP = ipow_c(M, DIM), NV = n_vars_c(DIM);
    const long long blk = (long long)p.group * NP * NV * sizeof(R);
    if (blk % 16 != 0 || 2 * ((blk + 127) / 128 * 128) + 128 > 200 * 1024) return 0;
    if (p.u != nullptr && !(aligned16(p.ws) && aligned16(p.out))) return 0;
    const long long items = ((long long)p.group * NP + 255) / 256;
    return items <= 1 ? 1 : items <= 2 ? 2 : items <= 4 ? 4 : 0;
}

// the unfused method's own AoSoA group: the largest power of two whose direction block
// is at most 48 KB (two stages in flight, at least two CTAs per SM), at least 16-byte rows
template <class R, int DIM, int M>
constexpr int unfused_group() {
    int g = 64;
    while (g > 16 / int(sizeof(R)) && (long long)g * ipow_c(M, DIM) * n_vars_c(DIM) * sizeof(R) > 48 * 1024) g /= 2;
    return g;
}

template <class R, int DIM, int M, int ITEMS>
cudaError_t launch_div_staged(const Params<R>& p, cudaStream_t st) {
    using S = DivStagedShape<R, DIM, M, ITEMS>;
    auto kernel = hf_div_staged_kernel<R, DIM, M, ITEMS>;
    const int blk = p.group * ipow_c(M, DIM) * n_vars_c(DIM) * int(sizeof(R));
    const size_t smem = S::HDR + 2 * size_t((blk + 127) / 128 * 128);
    if (int e = set_smem_attr(kernel, smem)) return cudaError_t(e);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, S::BS, smem) != cudaSuccess || b < 1) {
        cudaGetLastError();
        b = 1;
    }
    const long long groups = (p.n_elem + p.group - 1) / p.group;
    const long long slots = (long long)b * num_sms();
    kernel<<<unsigned(groups < slots ? groups : slots), S::BS, smem, st>>>(p);
    return cudaGetLastError();
}

template <class R, int DIM, int M>
cudaError_t launch_unfused(Params<R> p, bool src, cudaStream_t st, KInfo* info, bool dry) {
    const long long groups = (p.n_elem + p.group - 1) / p.group;
    if (info) {
        info->method = 3;
        info->elems_per_cta = p.group;
        info->block_threads = kUnfusedBS;
        info->shared_bytes = 0;
        info->grid = groups;
        info->bulk_path = 0;
        std::snprintf(info->name, sizeof(info->name), "hf_flux+hf_div%s_d%d_p%d_%s", src ? "+hf_source" : "", DIM,
                      M - 1, prec_name(sizeof(R)));
        if (dry) fill_regs(hf_div_kernel<R, DIM, M>, info);
    }
    if (dry || p.n_elem == 0) return cudaSuccess;
    hf_flux_kernel<R, DIM, M><<<dim3(unsigned(groups)), dim3(kUnfusedBS), 0, st>>>(p);
    cudaError_t e = cudaSuccess;
    switch (div_staged_items<R, DIM, M>(p)) {
        case 1: e = launch_div_staged<R, DIM, M, 1>(p, st); break;
        case 2: e = launch_div_staged<R, DIM, M, 2>(p, st); break;
        case 4: e = launch_div_staged<R, DIM, M, 4>(p, st); break;
        default: hf_div_kernel<R, DIM, M><<<dim3(unsigned(groups)), dim3(kUnfusedBS), 0, st>>>(p);
    }
    if (e != cudaSuccess) return e;
    if (src) hf_source_kernel<R, DIM, M><<<dim3(unsigned(groups)), dim3(kUnfusedBS), 0, st>>>(p);
    return cudaGetLastError();
}

// Runtime -> template dispatch (hf_dispatch.cuh) returns this for a combination
// that is not instantiated; the C ABI maps it to HF_EINVAL.
constexpr int kUnsupported = -1;

}  // namespace hfb
