// hf_dispatch.cuh -- runtime (d, p, variant, source) -> kernel template.
// Included by the per-precision instantiation units hf_inst_*.cu so that the
// template instantiations compile in parallel.
#pragma once

#include "hf_launch.cuh"

namespace hfb {

template <class R, int DIM, int M, int VARIANT, bool FACES>
int lines_variant_f(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = variant_ne<R, DIM, M, VARIANT>();
    constexpr bool CS = is_cs_variant(VARIANT);
    if constexpr (is_pipe_variant<VARIANT>()) {
        constexpr int ST = pipe_stages<VARIANT>();
        constexpr int GR = pipe_groups<VARIANT>();
        constexpr bool TL = VARIANT == kTileRingVariant;
        return src ? int(launch_lines_pipe<R, DIM, M, NE, ST, GR, true, FACES, CS, TL>(prm, st, info, dry))
                   : int(launch_lines_pipe<R, DIM, M, NE, ST, GR, false, FACES, CS, TL>(prm, st, info, dry));
    } else {
        constexpr int LPT = lines_per_thread<VARIANT>();
        constexpr int XP = is_xpad_variant(VARIANT) ? xpad_code<R, DIM, M, NE>() : 0;
        return src ? int(launch_lines<R, DIM, M, NE, true, LPT, FACES, NE, CS, XP>(prm, st, info, dry))
                   : int(launch_lines<R, DIM, M, NE, false, LPT, FACES, NE, CS, XP>(prm, st, info, dry));
    }
}

// faces: FR stage 1 fused in (lines_sweeps<FACES>); instantiated for the selected
// variant only (and every variant in the tuning build).
template <class R, int DIM, int M, int VARIANT>
int lines_variant(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry, bool faces = false) {
    constexpr int NE = variant_ne<R, DIM, M, VARIANT>();
    if constexpr (NE == 0 || !variant_built<R, DIM, M, VARIANT>()) {
        return kUnsupported;
    } else if constexpr (is_pipe_variant<VARIANT>() &&
                         (PipeShape<R, DIM, M, NE, pipe_stages<VARIANT>(), pipe_groups<VARIANT>(),
                                    is_cs_variant(VARIANT), VARIANT == kTileRingVariant>::SMEM >
                              size_t(kMaxSmemPerCta) ||
                          PipeShape<R, DIM, M, NE, pipe_stages<VARIANT>(), pipe_groups<VARIANT>(),
                                    is_cs_variant(VARIANT)>::BS > 1024)) {
        return kUnsupported;
    } else if constexpr (!is_pipe_variant<VARIANT>() &&
                         (LinesShape<R, DIM, M, NE>::SMEM > size_t(kMaxSmemPerCta) ||
                          LinesShape<R, DIM, M, NE, lines_per_thread<VARIANT>(), NE, is_cs_variant(VARIANT)>::BS >
                              1024)) {
        return kUnsupported;
    } else {
        if (!faces) return lines_variant_f<R, DIM, M, VARIANT, false>(src, prm, st, info, dry);
        if constexpr (variant_faces_built<R, DIM, M, VARIANT>())
            return lines_variant_f<R, DIM, M, VARIANT, true>(src, prm, st, info, dry);
        return kUnsupported;
    }
}

// Variants [VLO, VHI] of one order (the instantiation units split the variant
// range so that the template instances compile in parallel).
template <class R, int DIM, int M, int VLO, int VHI, int V = VLO>
int lines_m(int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry, bool faces) {
    if (variant == V) return lines_variant<R, DIM, M, V>(src, prm, st, info, dry, faces);
    if constexpr (V < VHI) return lines_m<R, DIM, M, VLO, VHI, V + 1>(variant, src, prm, st, info, dry, faces);
    return kUnsupported;
}

template <class R, int DIM, int VLO, int VHI>
int run_lines_range(int p, int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry,
                    bool faces) {
    if (variant < VLO || variant > VHI) return kUnsupported;
    if constexpr (DIM == 3) {
        switch (p) {
            case 1: return lines_m<R, 3, 2, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 2: return lines_m<R, 3, 3, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 3: return lines_m<R, 3, 4, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 4: return lines_m<R, 3, 5, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 5: return lines_m<R, 3, 6, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 6: return lines_m<R, 3, 7, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 7: return lines_m<R, 3, 8, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            default: return kUnsupported;
        }
    } else {
        switch (p) {
            case 1: return lines_m<R, 2, 2, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 2: return lines_m<R, 2, 3, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 3: return lines_m<R, 2, 4, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 4: return lines_m<R, 2, 5, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 5: return lines_m<R, 2, 6, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 6: return lines_m<R, 2, 7, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 7: return lines_m<R, 2, 8, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            case 8: return lines_m<R, 2, 9, VLO, VHI>(variant, src, prm, st, info, dry, faces);
            default: return kUnsupported;
        }
    }
}

// Grouped chunks (hf_lines.cuh, LinesShape GS < NE): the chunk of variant 0 (NE0 elements)
// made of NE0 / GS whole groups of a caller's power-of-two group GS < NE0, one contiguous
// byte range.  Returns kUnsupported for a GS that is not instantiated.
template <class R, int DIM, int M, int GS = 1>
int lines_grouped_m(int gs, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = variant_ne<R, DIM, M, 0>();
    if constexpr (GS >= NE) {
        return kUnsupported;
    } else {
        if (gs == GS) {
            if constexpr (LinesShape<R, DIM, M, NE, 1, GS>::SMEM > size_t(kMaxSmemPerCta)) return kUnsupported;
            return src ? int(launch_lines<R, DIM, M, NE, true, 1, false, GS>(prm, st, info, dry))
                       : int(launch_lines<R, DIM, M, NE, false, 1, false, GS>(prm, st, info, dry));
        }
        return lines_grouped_m<R, DIM, M, GS * 2>(gs, src, prm, st, info, dry);
    }
}

template <class R, int DIM>
int run_lines_grouped(int p, int gs, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    if constexpr (DIM == 3) {
        switch (p) {
            case 1: return lines_grouped_m<R, 3, 2>(gs, src, prm, st, info, dry);
            case 2: return lines_grouped_m<R, 3, 3>(gs, src, prm, st, info, dry);
            case 3: return lines_grouped_m<R, 3, 4>(gs, src, prm, st, info, dry);
            case 4: return lines_grouped_m<R, 3, 5>(gs, src, prm, st, info, dry);
            case 5: return lines_grouped_m<R, 3, 6>(gs, src, prm, st, info, dry);
            case 6: return lines_grouped_m<R, 3, 7>(gs, src, prm, st, info, dry);
            case 7: return lines_grouped_m<R, 3, 8>(gs, src, prm, st, info, dry);
            default: return kUnsupported;
        }
    } else {
        switch (p) {
            case 1: return lines_grouped_m<R, 2, 2>(gs, src, prm, st, info, dry);
            case 2: return lines_grouped_m<R, 2, 3>(gs, src, prm, st, info, dry);
            case 3: return lines_grouped_m<R, 2, 4>(gs, src, prm, st, info, dry);
            case 4: return lines_grouped_m<R, 2, 5>(gs, src, prm, st, info, dry);
            case 5: return lines_grouped_m<R, 2, 6>(gs, src, prm, st, info, dry);
            case 6: return lines_grouped_m<R, 2, 7>(gs, src, prm, st, info, dry);
            case 7: return lines_grouped_m<R, 2, 8>(gs, src, prm, st, info, dry);
            case 8: return lines_grouped_m<R, 2, 9>(gs, src, prm, st, info, dry);
            default: return kUnsupported;
        }
    }
}

template <class R, int M>
int planar_m(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = planar_ne<R, M>();
    return src ? int(launch_planar<R, M, NE, true>(prm, st, info, dry))
               : int(launch_planar<R, M, NE, false>(prm, st, info, dry));
}

template <class R>
int run_planar_impl(int p, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    switch (p) {
        case 1: return planar_m<R, 2>(src, prm, st, info, dry);
        case 2: return planar_m<R, 3>(src, prm, st, info, dry);
        case 3: return planar_m<R, 4>(src, prm, st, info, dry);
        case 4: return planar_m<R, 5>(src, prm, st, info, dry);
        case 5: return planar_m<R, 6>(src, prm, st, info, dry);
        case 6: return planar_m<R, 7>(src, prm, st, info, dry);
        case 7: return planar_m<R, 8>(src, prm, st, info, dry);
        default: return kUnsupported;
    }
}

template <class R, int M>
int planar_managed_m(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = planar_managed_ne<R, M>();
    return src ? int(launch_planar_managed<R, M, NE, true>(prm, st, info, dry))
               : int(launch_planar_managed<R, M, NE, false>(prm, st, info, dry));
}

template <class R>
int run_planar_managed_impl(int p, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    switch (p) {
        case 1: return planar_managed_m<R, 2>(src, prm, st, info, dry);
        case 2: return planar_managed_m<R, 3>(src, prm, st, info, dry);
        case 3: return planar_managed_m<R, 4>(src, prm, st, info, dry);
        case 4: return planar_managed_m<R, 5>(src, prm, st, info, dry);
        case 5: return planar_managed_m<R, 6>(src, prm, st, info, dry);
        case 6: return planar_managed_m<R, 7>(src, prm, st, info, dry);
        case 7: return planar_managed_m<R, 8>(src, prm, st, info, dry);
        default: return kUnsupported;
    }
}

template <class R, int DIM, int M>
int mapped_m(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = mapped_ne<R, DIM, M>();
    if constexpr (MappedShape<R, DIM, M, NE>::SMEM > size_t(kMaxSmemPerCta)) {
        return kUnsupported;
    } else {
        return src ? int(launch_mapped<R, DIM, M, NE, true>(prm, st, info, dry))
                   : int(launch_mapped<R, DIM, M, NE, false>(prm, st, info, dry));
    }
}

template <class R>
int run_mapped_impl(int d, int p, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    if (d == 3) {
        switch (p) {
            case 1: return mapped_m<R, 3, 2>(src, prm, st, info, dry);
            case 2: return mapped_m<R, 3, 3>(src, prm, st, info, dry);
            case 3: return mapped_m<R, 3, 4>(src, prm, st, info, dry);
            case 4: return mapped_m<R, 3, 5>(src, prm, st, info, dry);
            case 5: return mapped_m<R, 3, 6>(src, prm, st, info, dry);
            case 6: return mapped_m<R, 3, 7>(src, prm, st, info, dry);
            case 7: return mapped_m<R, 3, 8>(src, prm, st, info, dry);
            default: return kUnsupported;
        }
    }
    switch (p) {
        case 1: return mapped_m<R, 2, 2>(src, prm, st, info, dry);
        case 2: return mapped_m<R, 2, 3>(src, prm, st, info, dry);
        case 3: return mapped_m<R, 2, 4>(src, prm, st, info, dry);
        case 4: return mapped_m<R, 2, 5>(src, prm, st, info, dry);
        case 5: return mapped_m<R, 2, 6>(src, prm, st, info, dry);
        case 6: return mapped_m<R, 2, 7>(src, prm, st, info, dry);
        case 7: return mapped_m<R, 2, 8>(src, prm, st, info, dry);
        case 8: return mapped_m<R, 2, 9>(src, prm, st, info, dry);
        default: return kUnsupported;
    }
}

template <class R>
int run_unfused_impl(int d, int p, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    if (d == 3) {
        switch (p) {
            case 1: return int(launch_unfused<R, 3, 2>(prm, src, st, info, dry));
            case 2: return int(launch_unfused<R, 3, 3>(prm, src, st, info, dry));
            case 3: return int(launch_unfused<R, 3, 4>(prm, src, st, info, dry));
            case 4: return int(launch_unfused<R, 3, 5>(prm, src, st, info, dry));
            case 5: return int(launch_unfused<R, 3, 6>(prm, src, st, info, dry));
            case 6: return int(launch_unfused<R, 3, 7>(prm, src, st, info, dry));
            case 7: return int(launch_unfused<R, 3, 8>(prm, src, st, info, dry));
            default: return kUnsupported;
        }
    }
    switch (p) {
        case 1: return int(launch_unfused<R, 2, 2>(prm, src, st, info, dry));
        case 2: return int(launch_unfused<R, 2, 3>(prm, src, st, info, dry));
        case 3: return int(launch_unfused<R, 2, 4>(prm, src, st, info, dry));
        case 4: return int(launch_unfused<R, 2, 5>(prm, src, st, info, dry));
        case 5: return int(launch_unfused<R, 2, 6>(prm, src, st, info, dry));
        case 6: return int(launch_unfused<R, 2, 7>(prm, src, st, info, dry));
        case 7: return int(launch_unfused<R, 2, 8>(prm, src, st, info, dry));
        case 8: return int(launch_unfused<R, 2, 9>(prm, src, st, info, dry));
        default: return kUnsupported;
    }
}

// Entry points defined in the instantiation units (lines: variants 0-9 in *_lo, 10-27 in *_hi).
#define HF_LINES_DECL(NAME, R)                                                                        \
    int NAME##_lo(int p, int variant, bool src, const Params<R>&, cudaStream_t, KInfo*, bool, bool);   \
    int NAME##_hi(int p, int variant, bool src, const Params<R>&, cudaStream_t, KInfo*, bool, bool);   \
    inline int NAME(int p, int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info,   \
                    bool dry, bool faces = false) {                                                   \
        return variant < 10 ? NAME##_lo(p, variant, src, prm, st, info, dry, faces)                   \
                            : NAME##_hi(p, variant, src, prm, st, info, dry, faces);                  \
    }
HF_LINES_DECL(lines_f32_d3, float)
HF_LINES_DECL(lines_f64_d3, double)
HF_LINES_DECL(lines_f32_d2, float)
HF_LINES_DECL(lines_f64_d2, double)
#undef HF_LINES_DECL
int lines_grouped_f32_d3(int p, int gs, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int lines_grouped_f64_d3(int p, int gs, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int lines_grouped_f32_d2(int p, int gs, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int lines_grouped_f64_d2(int p, int gs, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int planar_f32(int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int planar_f64(int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int planar_managed_f32(int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int planar_managed_f64(int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int mapped_f32(int d, int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int mapped_f64(int d, int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int unfused_f32(int d, int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int unfused_f64(int d, int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);

}  // namespace hfb
