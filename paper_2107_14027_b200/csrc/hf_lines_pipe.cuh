// hf_lines_pipe.cuh -- persistent, warp-specialised form of the lines kernel.
//
// Same arithmetic as hf_lines.cuh (three register-line sweeps per chunk), but
// the chunk traffic is decoupled from the compute with a STAGES-deep ring of
// shared-memory chunk buffers fed by cp.async.bulk:
//
//   warp 0 (producer)  : keeps up to STAGES chunks in flight.  For each chunk
//                        it waits for the consumers to finish the stage; then
//                        every lane bulk-stores its 1/32 slice of the finished
//                        divergence, waits for that slice to have left shared
//                        memory, and reloads the slice with the chunk STAGES
//                        ahead (mbarrier complete_tx) -- stores and loads of a
//                        stage overlap slice by slice.
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
    static constexpr size_t STAGE_BYTES = size_t(L::BUF_BYTES);
    static constexpr size_t SMEM = HDR + STAGES * STAGE_BYTES + size_t(L::ACC_WORDS) * sizeof(R);
    static_assert(2 * STAGES * 8 <= HDR, "mbarrier header too small");
};

template <class R, int DIM, int M, int NE, int STAGES, bool SRC>
__global__ void __launch_bounds__(PipeShape<R, DIM, M, NE, STAGES>::BS)
    hf_lines_pipe_kernel(const __grid_constant__ Params<R> p) {
    using L = LinesShape<R, DIM, M, NE>;
    using S = PipeShape<R, DIM, M, NE, STAGES>;
    constexpr int ROWS = L::NP * L::NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* computed = full + STAGES;
    unsigned char* stage0 = smem_raw + S::HDR;
    R* acc = reinterpret_cast<R*>(stage0 + size_t(STAGES) * S::STAGE_BYTES);
    using IO = typename L::IO;

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
        for (long long it = 0; it < pre; ++it) {
            const R* src = p.u + chunk_base(it);
            if (lane == 0) mbar_arrive_expect_tx(&full[it], IO::tx_bytes(src, contiguous));
            __syncwarp();
            IO::load(stage0 + it * S::STAGE_BYTES, src, p.group, contiguous, &full[it], lane);
        }
        for (long long it = 0; it < count; ++it) {
            const int s = int(it % STAGES);
            const uint32_t ph = uint32_t((it / STAGES) & 1);
            unsigned char* buf = stage0 + size_t(s) * S::STAGE_BYTES;
            mbar_wait_parity(&computed[s], ph);
            const bool refill = it + STAGES < count;
            const R* src = p.u + chunk_base(it + STAGES);
            if (refill && lane == 0) mbar_arrive_expect_tx(&full[s], IO::tx_bytes(src, contiguous));
            __syncwarp();
            IO::store(p.out + chunk_base(it), buf, p.group, contiguous, lane);
            if (refill) {
                bulk_wait_read_all();  // this lane's region has left shared memory
                IO::load(buf, src, p.group, contiguous, &full[s], lane);
            }
        }
        bulk_wait_read_all();
        return;
    }

    // ---------------- consumers ----------------
    // The stage loop is unrolled so that each stage's buffer is a compile-time
    // offset into the __shared__ window (see lines_sweeps).
    const int ct = tid - 32;
    for (long long it0 = 0; it0 < count; it0 += STAGES) {
        const uint32_t ph = uint32_t((it0 / STAGES) & 1);
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            const long long it = it0 + s;
            if (it >= count) break;
            const long long cb = chunk_base(it);
            unsigned char* buf = smem_raw + S::HDR + size_t(s) * S::STAGE_BYTES;
            mbar_wait_parity(&full[s], ph);
            lines_sweeps_at<R, DIM, M, NE, SRC, 1, S::NCONS>(buf, IO::head_bytes(p.u + cb, contiguous), acc, p, ct);
            fence_proxy_async_smem();
            named_bar_sync(1, S::NCONS);
            if (ct == 0) mbar_arrive(&computed[s]);
        }
    }
}

}  // namespace hfb
