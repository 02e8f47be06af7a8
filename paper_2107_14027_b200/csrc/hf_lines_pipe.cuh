// hf_lines_pipe.cuh -- persistent, warp-specialised form of the lines kernel.
//
// Same arithmetic as hf_lines.cuh (three register-line sweeps per chunk), but
// the chunk traffic is decoupled from the compute with a STAGES-deep ring of
// shared-memory chunk buffers fed by cp.async.bulk:
//
//   warp 0 (producer)  : keeps up to STAGES chunks in flight.  For each chunk
//                        it waits for the consumers to finish the stage, issues
//                        the bulk store of the finished divergence from that
//                        stage, waits for the store to have read shared memory,
//                        and refills the stage with the chunk STAGES ahead
//                        (mbarrier complete_tx).
//   warps 1.. (consumers): wait full[s], run the d sweeps on stage s (named
//                        barrier 1 between sweeps), fence the generic-proxy
//                        writes for the async proxy, arrive computed[s].
//
// One CTA per SM slot, chunks assigned round-robin (all chunks cost the same).
// Only whole chunks inside one AoSoA group run here (group % NE == 0, 16-byte
// rows); the guarded tail goes through hf_lines_kernel with chunk0 = n_chunks.
#pragma once

#include "hf_lines.cuh"

namespace hfb {

template <class R, int DIM, int M, int NE, int STAGES>
struct PipeShape {
    using L = LinesShape<R, DIM, M, NE>;
    static constexpr int NCONS = ((L::LINES + 31) / 32) * 32;  // consumer threads
    static constexpr int BS = NCONS + 32;                     // + producer warp
    static constexpr int HDR = 128;                           // 2*STAGES mbarriers (<= 16)
    static constexpr size_t STAGE_BYTES = size_t(L::IN_WORDS) * sizeof(R);
    static constexpr size_t SMEM = HDR + STAGES * STAGE_BYTES + size_t(L::ACC_WORDS) * sizeof(R);
    static constexpr int PIECE = 8192;  // contiguous-chunk bulk copies are split into 8 KB pieces
    static_assert(2 * STAGES * 8 <= HDR, "mbarrier header too small");
};

template <class R, int NE, int ROWS, int IN_BYTES, int PIECE>
__device__ __forceinline__ void pipe_load(R* dst, const R* src, long long group, bool contiguous, uint64_t* bar,
                                          int lane) {
    if (lane == 0) mbar_arrive_expect_tx(bar, IN_BYTES);
    __syncwarp();
    if (contiguous) {
        for (int off = lane * PIECE; off < IN_BYTES; off += 32 * PIECE) {
            const int len = (IN_BYTES - off) < PIECE ? (IN_BYTES - off) : PIECE;
            bulk_g2s(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off,
                     len, bar);
        }
    } else {
        for (int row = lane; row < ROWS; row += 32)
            bulk_g2s(dst + NE * row, src + group * row, NE * int(sizeof(R)), bar);
    }
}

template <class R, int NE, int ROWS, int IN_BYTES, int PIECE>
__device__ __forceinline__ void pipe_store(R* dst, const R* src, long long group, bool contiguous, int lane) {
    if (contiguous) {
        for (int off = lane * PIECE; off < IN_BYTES; off += 32 * PIECE) {
            const int len = (IN_BYTES - off) < PIECE ? (IN_BYTES - off) : PIECE;
            bulk_s2g(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off,
                     len);
        }
    } else {
        for (int row = lane; row < ROWS; row += 32) bulk_s2g(dst + group * row, src + NE * row, NE * int(sizeof(R)));
    }
    bulk_commit();
}

template <class R, int DIM, int M, int NE, int STAGES, bool SRC>
__global__ void __launch_bounds__(PipeShape<R, DIM, M, NE, STAGES>::BS)
    hf_lines_pipe_kernel(const __grid_constant__ Params<R> p) {
    using L = LinesShape<R, DIM, M, NE>;
    using S = PipeShape<R, DIM, M, NE, STAGES>;
    constexpr int ROWS = L::NP * L::NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* computed = full + STAGES;
    R* stage0 = reinterpret_cast<R*>(smem_raw + S::HDR);
    R* acc = stage0 + size_t(STAGES) * L::IN_WORDS;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&computed[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const long long n_chunks = p.n_chunks;
    const long long first = blockIdx.x;
    const long long step = gridDim.x;
    const long long count = first < n_chunks ? (n_chunks - 1 - first) / step + 1 : 0;
    const bool contiguous = (p.group == NE);
    auto chunk_base = [&](long long it) -> long long {
        const long long E0 = (first + it * step) * NE;  // chunk0 == 0 for this kernel
        const long long grp = E0 / p.group;
        return grp * p.group_words + (E0 - grp * p.group);
    };

    if (warp == 0) {
        // ---------------- producer ----------------
        const long long pre = count < STAGES ? count : STAGES;
        for (long long it = 0; it < pre; ++it)
            pipe_load<R, NE, ROWS, L::IN_BYTES, S::PIECE>(stage0 + it * L::IN_WORDS, p.u + chunk_base(it), p.group,
                                                          contiguous, &full[it], lane);
        for (long long it = 0; it < count; ++it) {
            const int s = int(it % STAGES);
            const uint32_t ph = uint32_t((it / STAGES) & 1);
            R* buf = stage0 + size_t(s) * L::IN_WORDS;
            mbar_wait_parity(&computed[s], ph);
            pipe_store<R, NE, ROWS, L::IN_BYTES, S::PIECE>(p.out + chunk_base(it), buf, p.group, contiguous, lane);
            if (it + STAGES < count) {
                bulk_wait_read_all();  // the stage's store has left shared memory
                __syncwarp();
                pipe_load<R, NE, ROWS, L::IN_BYTES, S::PIECE>(buf, p.u + chunk_base(it + STAGES), p.group, contiguous,
                                                              &full[s], lane);
            }
        }
        bulk_wait_read_all();
        return;
    }

    // ---------------- consumers ----------------
    const int ct = tid - 32;
    for (long long it = 0; it < count; ++it) {
        const int s = int(it % STAGES);
        const uint32_t ph = uint32_t((it / STAGES) & 1);
        R* buf = stage0 + size_t(s) * L::IN_WORDS;
        mbar_wait_parity(&full[s], ph);
        if constexpr (DIM == 3) {
            if (ct < L::LINES) lines_sweep<R, 3, M, NE, SRC, 0, 0>(buf, acc, p, ct);
            named_bar_sync(1, S::NCONS);
            if (ct < L::LINES) lines_sweep<R, 3, M, NE, SRC, 1, 1>(buf, acc, p, ct);
            named_bar_sync(1, S::NCONS);
            if (ct < L::LINES) lines_sweep<R, 3, M, NE, SRC, 2, 2>(buf, acc, p, ct);
        } else {
            if (ct < L::LINES) lines_sweep<R, 2, M, NE, SRC, 0, 0>(buf, acc, p, ct);
            named_bar_sync(1, S::NCONS);
            if (ct < L::LINES) lines_sweep<R, 2, M, NE, SRC, 1, 2>(buf, acc, p, ct);
        }
        fence_proxy_async_smem();
        named_bar_sync(1, S::NCONS);
        if (ct == 0) mbar_arrive(&computed[s]);
    }
}

}  // namespace hfb
