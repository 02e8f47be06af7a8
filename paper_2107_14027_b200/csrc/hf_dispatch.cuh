// hf_dispatch.cuh -- runtime (d, p, variant, source) -> kernel template.
// Included by the per-precision instantiation units hf_inst_*.cu so that the
// template instantiations compile in parallel.
#pragma once

#include "hf_launch.cuh"

namespace hfb {

template <class R, int DIM, int M, int VARIANT>
int lines_variant(bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    constexpr int NE = variant_ne<R, DIM, M, VARIANT>();
    if constexpr (NE == 0) {
        return kUnsupported;
    } else if constexpr (is_pipe_variant<VARIANT>()) {
        constexpr int ST = pipe_stages<VARIANT>();
        if constexpr (PipeShape<R, DIM, M, NE, ST>::SMEM > size_t(kMaxSmemPerCta) ||
                      PipeShape<R, DIM, M, NE, ST>::BS > 1024) {
            return kUnsupported;
        } else {
            return src ? int(launch_lines_pipe<R, DIM, M, NE, ST, true>(prm, st, info, dry))
                       : int(launch_lines_pipe<R, DIM, M, NE, ST, false>(prm, st, info, dry));
        }
    } else if constexpr (LinesShape<R, DIM, M, NE>::SMEM > size_t(kMaxSmemPerCta) ||
                         LinesShape<R, DIM, M, NE>::BS > 1024) {
        return kUnsupported;
    } else {
        return src ? int(launch_lines<R, DIM, M, NE, true>(prm, st, info, dry))
                   : int(launch_lines<R, DIM, M, NE, false>(prm, st, info, dry));
    }
}

template <class R, int DIM, int M>
int lines_m(int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    switch (variant) {
        case 0: return lines_variant<R, DIM, M, 0>(src, prm, st, info, dry);
        case 1: return lines_variant<R, DIM, M, 1>(src, prm, st, info, dry);
        case 2: return lines_variant<R, DIM, M, 2>(src, prm, st, info, dry);
        case 3: return lines_variant<R, DIM, M, 3>(src, prm, st, info, dry);
        case 4: return lines_variant<R, DIM, M, 4>(src, prm, st, info, dry);
        case 5: return lines_variant<R, DIM, M, 5>(src, prm, st, info, dry);
        case 6: return lines_variant<R, DIM, M, 6>(src, prm, st, info, dry);
        case 7: return lines_variant<R, DIM, M, 7>(src, prm, st, info, dry);
        case 8: return lines_variant<R, DIM, M, 8>(src, prm, st, info, dry);
        case 9: return lines_variant<R, DIM, M, 9>(src, prm, st, info, dry);
        default: return kUnsupported;
    }
}

template <class R>
int run_lines_d3(int p, int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    switch (p) {
        case 1: return lines_m<R, 3, 2>(variant, src, prm, st, info, dry);
        case 2: return lines_m<R, 3, 3>(variant, src, prm, st, info, dry);
        case 3: return lines_m<R, 3, 4>(variant, src, prm, st, info, dry);
        case 4: return lines_m<R, 3, 5>(variant, src, prm, st, info, dry);
        case 5: return lines_m<R, 3, 6>(variant, src, prm, st, info, dry);
        case 6: return lines_m<R, 3, 7>(variant, src, prm, st, info, dry);
        case 7: return lines_m<R, 3, 8>(variant, src, prm, st, info, dry);
        default: return kUnsupported;
    }
}

template <class R>
int run_lines_d2(int p, int variant, bool src, const Params<R>& prm, cudaStream_t st, KInfo* info, bool dry) {
    switch (p) {
        case 1: return lines_m<R, 2, 2>(variant, src, prm, st, info, dry);
        case 2: return lines_m<R, 2, 3>(variant, src, prm, st, info, dry);
        case 3: return lines_m<R, 2, 4>(variant, src, prm, st, info, dry);
        case 4: return lines_m<R, 2, 5>(variant, src, prm, st, info, dry);
        case 5: return lines_m<R, 2, 6>(variant, src, prm, st, info, dry);
        case 6: return lines_m<R, 2, 7>(variant, src, prm, st, info, dry);
        case 7: return lines_m<R, 2, 8>(variant, src, prm, st, info, dry);
        case 8: return lines_m<R, 2, 9>(variant, src, prm, st, info, dry);
        default: return kUnsupported;
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

// Entry points defined in the instantiation units.
int lines_f32_d3(int p, int variant, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int lines_f64_d3(int p, int variant, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int lines_f32_d2(int p, int variant, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int lines_f64_d2(int p, int variant, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int planar_f32(int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int planar_f64(int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);
int unfused_f32(int d, int p, bool src, const Params<float>&, cudaStream_t, KInfo*, bool);
int unfused_f64(int d, int p, bool src, const Params<double>&, cudaStream_t, KInfo*, bool);

}  // namespace hfb
