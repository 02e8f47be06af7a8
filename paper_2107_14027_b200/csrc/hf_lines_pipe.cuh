// hf_lines_pipe.cuh -- persistent, warp-specialised form of the lines kernel.
//
// Same arithmetic as hf_lines.cuh (d register-line sweeps per chunk), but the
// chunk traffic is decoupled from the compute with a STAGES-deep ring of
// shared-memory chunk buffers fed by cp.async.bulk, and the compute is split
// over GROUPS independent consumer groups:
//
//   warp 0 (producer)  : keeps up to STAGES chunks in flight.  For each chunk
//                        it waits for the owning group to finish the stage;
//                        then each lane that owns a piece of the stage (pieces
//                        of >= 64 KB, hf_chunk_io.cuh) bulk-stores it, waits
//                        for it to have left shared memory, and reloads it
//                        with the chunk STAGES ahead (mbarrier complete_tx).
//   consumer group g   : chunks it = g, g+GROUPS, ... on its own SPG =
//   (warps 1+g*W ..)     STAGES/GROUPS stages (s = g*SPG + (it/GROUPS) % SPG):
//                        wait full[s], run the d sweeps (named barrier 1+g
//                        between sweeps, a private accumulator region), fence
//                        the generic-proxy writes for the async proxy, arrive
//                        computed[s].
//
// Why groups: a chunk's compute parallelism is its line count (NE * m^(d-1)),
// so with one group the ring can hold only STAGES = smem / chunk chunks and the
// SM computes one chunk at a time; with GROUPS groups the chunks can be GROUPS
// times smaller for the same number of computing warps, so more of them are in
// flight (STAGES - GROUPS being stored / loaded), and one group's barrier and
// shared-memory latency stalls are covered by the other groups' work.
//
// One CTA per SM slot, chunks assigned round-robin (all chunks cost the same).
// Only whole chunks inside one AoSoA group run here (group % NE == 0, 16-byte
// rows, or group == NE; with TILE also any 16-byte-stride group through one TMA
// tensor copy per chunk); the guarded tail goes through hf_lines_kernel with
// chunk0 = n_chunks.
#pragma once

#include "hf_lines.cuh"

namespace hfb {

// TILE: the ring may run tile mode (p.tile: the caller's AoSoA group is not the chunk; one
// TMA tensor copy per chunk and direction, as hf_lines_kernel's tile mode), so every stage
// starts 128-byte aligned (the tensor copy's shared-memory destination).
template <class R, int DIM, int M, int NE, int STAGES, int GROUPS = 1, bool CS = false, bool TILE = false>
struct PipeShape {
    using L = LinesShape<R, DIM, M, NE>;
    static_assert(STAGES % GROUPS == 0, "every group owns STAGES / GROUPS stages");
    static constexpr int SPG = STAGES / GROUPS;               // stages per group
    static constexpr int NT = ((L::LINES + 31) / 32) * 32;    // line slots per sweep iteration
    static constexpr int NCONS = CS ? DIM * NT : NT;          // consumer threads per group (CS: one per component)
    static constexpr int BS = GROUPS * NCONS + 32;            // + producer warp
    static constexpr int HDR = 256;                           // 2*STAGES mbarriers (<= 32)
    static constexpr size_t STAGE_BYTES = TILE ? (size_t(L::BUF_BYTES) + 127) / 128 * 128 : size_t(L::BUF_BYTES);
    static constexpr size_t ACC_BYTES = ((size_t(L::ACC_WORDS) * sizeof(R) + 127) / 128) * 128;
    static constexpr size_t SMEM = HDR + STAGES * STAGE_BYTES + GROUPS * ACC_BYTES;
    static_assert(2 * STAGES * 8 <= HDR, "mbarrier header too small");
    static_assert(GROUPS <= 15, "one named barrier per group");
};

// Consumer group g: its chunks on its SPG stages.  The stage index inside the
// group is unrolled (compile-time offsets); the group's base (stages and
// accumulator region) is a runtime offset from the __shared__ window, so every
// group runs the same code -- one copy of the sweeps per stage, not per
// (group, stage), which keeps the kernel inside the instruction cache.
template <class R, int DIM, int M, int NE, int STAGES, int GROUPS, bool SRC, bool FACES, bool CS = false,
          bool TILE = false>
__device__ __forceinline__ void pipe_consume(unsigned char* smem_raw, uint64_t* full, uint64_t* computed,
                                             const Params<R>& p, long long count, long long first, long long step,
                                             int g, int ct) {
    using S = PipeShape<R, DIM, M, NE, STAGES, GROUPS, CS, TILE>;
    using L = LinesShape<R, DIM, M, NE>;
    using IO = typename L::IO;
    constexpr int SPG = S::SPG;
    const bool contiguous = (p.group == NE);
    R* acc = reinterpret_cast<R*>(smem_raw + S::HDR + STAGES * S::STAGE_BYTES + size_t(g) * S::ACC_BYTES);
    unsigned char* gbuf = smem_raw + S::HDR + size_t(g) * SPG * S::STAGE_BYTES;
    for (long long q0 = 0; g + q0 * GROUPS < count; q0 += SPG) {
        const uint32_t ph = uint32_t((q0 / SPG) & 1);
#pragma unroll
        for (int j = 0; j < SPG; ++j) {
            const long long it = g + (q0 + j) * GROUPS;
            if (it >= count) break;
            const int s = g * SPG + j;
            long long E0 = (first + it * step) * NE;
            int head = 0;
            if (TILE && p.tile) {  // sub-chunk b % sub of group b / sub: the box lands at offset 0
                const long long b = first + it * step;
                const long long grp = b / p.sub_per_group;
                E0 = grp * p.group + (b - grp * p.sub_per_group) * NE;
            } else {
                const long long grp = E0 / p.group;
                head = IO::head_bytes(p.u + grp * p.group_words + (E0 - grp * p.group), contiguous);
            }
            unsigned char* buf = gbuf + size_t(j) * S::STAGE_BYTES;
            mbar_wait_parity(&full[s], ph);
            if constexpr (GROUPS == 1)
                lines_sweeps_at<R, DIM, M, NE, SRC, 1, S::NT, FACES, NE, CS>(buf, head, acc, p, ct, 0, E0);
            else
                lines_sweeps_at<R, DIM, M, NE, SRC, -1, S::NT, FACES, NE, CS>(buf, head, acc, p, ct, 1 + g, E0);
            fence_proxy_async_smem();
            named_bar_sync(1 + g, S::NCONS);
            if (ct == 0) mbar_arrive(&computed[s]);
        }
    }
}

template <class R, int DIM, int M, int NE, int STAGES, int GROUPS, bool SRC, bool FACES = false, bool CS = false,
          bool TILE = false>
__global__ void __launch_bounds__(PipeShape<R, DIM, M, NE, STAGES, GROUPS, CS, TILE>::BS)
    hf_lines_pipe_kernel(const __grid_constant__ Params<R> p) {
    using L = LinesShape<R, DIM, M, NE>;
    using S = PipeShape<R, DIM, M, NE, STAGES, GROUPS, CS, TILE>;
    constexpr int SPG = S::SPG;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* computed = full + STAGES;
    unsigned char* stage0 = smem_raw + S::HDR;
    using IO = typename L::IO;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    pdl_launch_dependents();
    pdl_wait();
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
    // stage of the CTA's it-th chunk: group it % GROUPS, its (it / GROUPS)-th chunk
    auto stage_of = [&](long long it) -> int { return int(it % GROUPS) * SPG + int((it / GROUPS) % SPG); };

    if (warp == 0) {
        // ---------------- producer ----------------
        if (TILE && p.tile) {
            // tile mode: chunk b = sub-chunk b % sub of group b / sub, one TMA tensor copy per
            // direction issued by lane 0 (the box {NE, m, m^(d-1), n_v, 1}; elements past the
            // group's end zero-filled on load, clipped on store)
            if (lane == 0) {
                tma_prefetch_desc(&p.tm_u);
                tma_prefetch_desc(&p.tm_out);
                auto coords = [&](long long it, int& c0, int& c4) {
                    const long long b = first + it * step;
                    const long long grp = b / p.sub_per_group;
                    c0 = static_cast<int>(b - grp * p.sub_per_group) * NE;
                    c4 = static_cast<int>(grp);
                };
                const long long pre = count < STAGES ? count : STAGES;
                for (long long it = 0; it < pre; ++it) {
                    const int s = stage_of(it);
                    int c0, c4;
                    coords(it, c0, c4);
                    mbar_arrive_expect_tx(&full[s], uint32_t(L::IN_BYTES));
                    tma_load_5d(stage0 + size_t(s) * S::STAGE_BYTES, &p.tm_u, c0, 0, 0, 0, c4, &full[s]);
                }
                for (long long it = 0; it < count; ++it) {
                    const int s = stage_of(it);
                    unsigned char* buf = stage0 + size_t(s) * S::STAGE_BYTES;
                    mbar_wait_parity(&computed[s], uint32_t((it / STAGES) & 1));
                    int c0, c4;
                    coords(it, c0, c4);
                    tma_store_5d(&p.tm_out, c0, 0, 0, 0, c4, buf);
                    bulk_commit();
                    if (it + STAGES < count) {
                        bulk_wait_read_all();  // the box has left shared memory
                        coords(it + STAGES, c0, c4);
                        mbar_arrive_expect_tx(&full[s], uint32_t(L::IN_BYTES));
                        tma_load_5d(buf, &p.tm_u, c0, 0, 0, 0, c4, &full[s]);
                    }
                }
                bulk_wait_read_all();
            }
            return;
        }
        const long long pre = count < STAGES ? count : STAGES;
        for (long long it = 0; it < pre; ++it) {
            const int s = stage_of(it);
            const R* src = p.u + chunk_base(it);
            if (lane == 0) mbar_arrive_expect_tx(&full[s], IO::tx_bytes(src, contiguous));
            __syncwarp();
            IO::load(stage0 + size_t(s) * S::STAGE_BYTES, src, p.group, contiguous, &full[s], lane);
        }
        for (long long it = 0; it < count; ++it) {
            const int s = stage_of(it);
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

    // ---------------- consumer groups ----------------
    const int g = (tid - 32) / S::NCONS;
    const int ct = (tid - 32) - g * S::NCONS;
    pipe_consume<R, DIM, M, NE, STAGES, GROUPS, SRC, FACES, CS, TILE>(smem_raw, full, computed, p, count, first,
                                                                      step, g, ct);
}

}  // namespace hfb
