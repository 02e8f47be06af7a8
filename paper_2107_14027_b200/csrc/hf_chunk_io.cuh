// hf_chunk_io.cuh -- moving one chunk (NE consecutive elements, all m^d points
// and n_v variables) between HBM and shared memory with cp.async.bulk.
//
// Two layouts take the bulk path:
//   * contiguous: the AoSoA group equals NE, so the chunk is ONE byte range of
//     the field (layout.hpp:128-134).  Its start need not be 16-byte aligned
//     (NE * m^d * n_v * w is often 8 mod 16): the load copies the enclosing
//     16-byte-aligned superset into shared memory (the chunk then starts `head`
//     bytes into the buffer), the store bulk-writes the aligned interior and
//     the <= 12-byte head and tail are written with ordinary stores -- so any
//     NE >= 1 works and chunk sizes can be chosen for occupancy alone.
//   * rows: group % NE == 0 with 16-byte rows; one copy per (point, variable)
//     row of NE words at stride `group`.
// The work is split over the lanes of one warp: lane l owns a fixed region (a
// piece of >= 64 KB, so one lane for most chunks) of the stage buffer for both
// directions, so a producer lane can store its region of a finished chunk, wait
// for just that region to leave shared memory, and refill it with the next chunk.
#pragma once

#include "hf_common.cuh"

namespace hfb {

template <class R, int NE, int ROWS, int IN_BYTES>
struct ChunkIO {
#ifdef HF_NO_SLACK
    static constexpr int BUF_BYTES = ((IN_BYTES + 15) / 16) * 16;
#else
    static constexpr int BUF_BYTES = ((IN_BYTES + 15) / 16) * 16 + 32;  // superset capacity
#endif
    static constexpr int ROW_BYTES = NE * int(sizeof(R));

    struct Span {
        uintptr_t a0;  // 16B-aligned start of the superset
        int len;       // superset bytes (multiple of 16)
        int head;      // chunk start - a0 (bytes, multiple of sizeof(R))
    };
    __device__ static Span span(const void* chunk) {
        const uintptr_t c = reinterpret_cast<uintptr_t>(chunk);
        const uintptr_t a0 = c & ~uintptr_t(15);
        const uintptr_t a1 = (c + IN_BYTES + 15) & ~uintptr_t(15);
        return {a0, int(a1 - a0), int(c - a0)};
    }
    // bytes the mbarrier must expect for one chunk load
    __device__ static uint32_t tx_bytes(const R* src, bool contiguous) {
        return contiguous ? uint32_t(span(src).len) : uint32_t(IN_BYTES);
    }
    // byte offset of the chunk's first word inside its stage buffer (callers add
    // it to a pointer derived from the __shared__ array, so that the compiler keeps
    // the shared address space and emits LDS/STS, not generic LD/ST)
    __device__ static int head_bytes(const R* src, bool contiguous) {
        return contiguous ? int(reinterpret_cast<uintptr_t>(src) & 15u) : 0;
    }

    // Lane l owns buffer bytes [l*PIECE, (l+1)*PIECE) for loads AND stores, so a
    // producer lane may refill its region as soon as its own store has read it.
    // PIECE is a multiple of the 128-byte line: when the chunk starts on a line,
    // no two bulk copies share a line or a 32-byte sector (split sectors in the
    // bulk stores cost ~10% of HBM bandwidth, measured).  Few large copies beat
    // many small ones: with pieces of at least 64 KB (one copy per chunk up to
    // 64 KB) the selected kernels gained 0-6 % over 1/32-of-the-chunk pieces
    // (p6: FP32 5.84 -> 6.20, FP64 6.09 -> 6.35 TB/s; profiles/select_r01d.jsonl
    // vs select_r01c.jsonl) -- the bulk-copy engine's per-request cost, not the
    // bytes, limited the small pieces.
#ifndef HF_MIN_PIECE
#define HF_MIN_PIECE 65536
#endif
    static constexpr int PIECE0 = ((BUF_BYTES / 32 + 127) / 128) * 128;
    static constexpr int PIECE = PIECE0 > HF_MIN_PIECE ? PIECE0 : HF_MIN_PIECE;

    __device__ static void load(unsigned char* buf, const R* src, long long group, bool contiguous, uint64_t* bar,
                                int lane) {
        if (contiguous) {
            const Span sp = span(src);
            const int lo = lane * PIECE;
            const int hi = (lo + PIECE) < sp.len ? (lo + PIECE) : sp.len;
            if (hi > lo) bulk_g2s(buf + lo, reinterpret_cast<const void*>(sp.a0 + lo), hi - lo, bar);
        } else {
            R* dst = reinterpret_cast<R*>(buf);
            for (int row = lane; row < ROWS; row += 32) bulk_g2s(dst + NE * row, src + group * row, ROW_BYTES, bar);
        }
    }

    // Store the finished chunk: the <= 12-byte unaligned head and tail with
    // ordinary stores (all lanes' shared-memory reads done before __syncwarp),
    // then each lane bulk-stores the aligned interior inside its own region, and
    // commits.
    __device__ static void store(R* dst, const unsigned char* buf, long long group, bool contiguous, int lane) {
        if (contiguous) {
            const uintptr_t c = reinterpret_cast<uintptr_t>(dst);
            const uintptr_t a0 = c & ~uintptr_t(15);
            const uintptr_t i0 = (c + 15) & ~uintptr_t(15);
            const uintptr_t i1 = (c + IN_BYTES) & ~uintptr_t(15);
            const R* s = reinterpret_cast<const R*>(buf + (c - a0));
            constexpr int W = IN_BYTES / int(sizeof(R));
            if (i1 > i0) {
                const int nh = int(i0 - c) / int(sizeof(R));
                const int t0 = int(i1 - c) / int(sizeof(R));
                if (lane < nh) dst[lane] = s[lane];
                if (t0 + lane < W) dst[t0 + lane] = s[t0 + lane];
                __syncwarp();
                const int b0 = int(i0 - a0), b1 = int(i1 - a0);  // interior in buffer coordinates
                int lo = lane * PIECE, hi = lo + PIECE;
                lo = lo > b0 ? lo : b0;
                hi = hi < b1 ? hi : b1;
                if (hi > lo) bulk_s2g(reinterpret_cast<void*>(a0 + lo), buf + lo, hi - lo);
            } else {  // shorter than one aligned 16-byte block
                for (int w = lane; w < W; w += 32) dst[w] = s[w];
                __syncwarp();
            }
        } else {
            const R* s = reinterpret_cast<const R*>(buf);
            for (int row = lane; row < ROWS; row += 32) bulk_s2g(dst + group * row, s + NE * row, ROW_BYTES);
        }
        bulk_commit();
    }
};

}  // namespace hfb
