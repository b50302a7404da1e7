// border.cuh -- the border pixels of a launch's output rows (filter.cpp:54 /
// parallel.cpp:113): CopyInput copies the input bytes, ZeroFill writes zeros.
// Executed by extra blocks of the launch's first kernel (kernels.cuh
// BorderJob), so it costs no launch of its own and overlaps the pre-pass.
#pragma once
#include <cstdint>

#include "kernels.cuh"

namespace opc {

// Thread t of nt copies its share of n contiguous bytes, 16-byte stores.
__device__ __forceinline__ void border_range(std::uint8_t* d, const std::uint8_t* src, long long n,
                                             long long t, long long nt, bool zero) {
    if (n <= 0) return;
    long long head = (16 - static_cast<long long>(reinterpret_cast<std::uintptr_t>(d) & 15)) & 15;
    if (head > n) head = n;
    if (t < head) d[t] = zero ? 0 : src[t];
    d += head;
    src += head;
    n -= head;
    const long long nv = n >> 4;
    uint4* dv = reinterpret_cast<uint4*>(d);
    if (zero) {
        for (long long i = t; i < nv; i += nt) dv[i] = make_uint4(0, 0, 0, 0);
    } else if ((reinterpret_cast<std::uintptr_t>(src) & 15) == 0) {
        const uint4* sv = reinterpret_cast<const uint4*>(src);
        for (long long i = t; i < nv; i += nt) dv[i] = sv[i];
    } else {
        for (long long i = t; i < nv; i += nt) {
            std::uint32_t w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const std::uint8_t* p = src + 16 * i + 4 * q;
                w[q] = p[0] | (p[1] << 8) | (p[2] << 16) | (static_cast<std::uint32_t>(p[3]) << 24);
            }
            dv[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    for (long long i = 16 * nv + t; i < n; i += nt) d[i] = zero ? 0 : src[i];
}

// Block b (< a.border.nblocks) of the border job for `frame`; tid in [0, 256).
__device__ __forceinline__ void border_block(const BandArgs& a, int b, int frame, int tid) {
    const BorderJob& j = a.border;
    const long long row_bytes = static_cast<long long>(a.width) * 3;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    std::uint8_t* out = a.out + a.out_frame_stride * frame;
    const bool zero = j.policy != 0;
    if (b < j.nfull) {
        const long long t = static_cast<long long>(b) * kBorderThreads + tid;
        const long long nt = static_cast<long long>(j.nfull) * kBorderThreads;
        border_range(out + (j.top_lo - a.out_row0) * row_bytes, in + (j.top_lo - a.in_row0) * row_bytes,
                     j.top_rows * row_bytes, t, nt, zero);
        border_range(out + (j.bot_lo - a.out_row0) * row_bytes, in + (j.bot_lo - a.in_row0) * row_bytes,
                     j.bot_rows * row_bytes, t, nt, zero);
        return;
    }
    const int y = a.y_lo + (b - j.nfull) * (kBorderThreads / 32) + (tid >> 5);
    if (y >= a.y_hi) return;
    const int lane = tid & 31, side = 3 * a.radius;
    const std::uint8_t* srow = in + (y - a.in_row0) * row_bytes;
    std::uint8_t* drow = out + (y - a.out_row0) * row_bytes;
    for (int k = lane; k < 2 * side; k += 32) {
        const long long col = k < side ? k : row_bytes - 2 * side + k;
        drow[col] = zero ? 0 : srow[col];
    }
}

// Extra grid rows a kernel with gridDim.x = gx appends for the border job.
inline unsigned border_grid_rows(const BandArgs& a, unsigned gx) {
    return a.border.nblocks > 0 ? static_cast<unsigned>((a.border.nblocks + gx - 1) / gx) : 0u;
}

}  // namespace opc
