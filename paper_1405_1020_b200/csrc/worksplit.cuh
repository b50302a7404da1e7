// worksplit.cuh -- how the persistent band kernels (skew, slide) divide a launch
// among their resident warps.
//
// Work units are band columns, linearised (frame, 32-row band, column).  Chunk
// i < nstatic is [i*s1, (i+1)*s1) -- one per resident warp, claimed at launch
// and together almost all of the work -- and the remainder is handed out in
// chunks of s2 units by the same atomic counter.  (A segment-major order, which
// keeps vertically adjacent bands of the same columns in flight together so
// that their shared halo rows hit in L2, measured 9% slower on C4 and C5: the
// narrow last segment cuts chunks into many passes.)
//
// The step costs of the skew kernel do not depend on the pixels, so equal
// static shares leave (almost) no tail, and the dynamic remainder absorbs
// per-SM speed differences.  (Equal task counts per warp are not enough: 4.09
// tasks per warp quantise to 5.)  The slide kernel's costs do depend on the
// content, so it keeps a larger dynamic share.  A chunk that crosses a band
// or segment end is processed as two passes.
//
// Launches too small for a static share per warp (< 4 * min_chunk units per
// warp) are cut into equal segments of each band instead (pitch > iw pads the
// linearisation so that a chunk is exactly one segment).
#pragma once

#include <algorithm>
#include <cstdint>

namespace opc {

struct WorkSplit {
    int nbands, iw, pitch;  // pitch >= iw: units per band (segment-aligned chunks)
    int nstatic, nchunks;
    long long units, s1, s2;
};

inline WorkSplit make_split(int frames, int nbands, int iw, long long resident, int static_pct,
                            long long min_chunk) {
    WorkSplit g{};
    g.nbands = nbands;
    g.iw = iw;
    g.pitch = iw;
    g.units = static_cast<long long>(frames) * nbands * iw;
    if (resident < 1) resident = 1;
    if (g.units >= resident * 4 * min_chunk) {
        g.nstatic = static_cast<int>(resident);
        g.s1 = g.units * static_pct / (100 * resident);
        const long long rest = g.units - resident * g.s1;
        g.s2 = std::max(min_chunk, (rest + 2 * resident - 1) / (2 * resident));
        g.nchunks = g.nstatic + static_cast<int>((rest + g.s2 - 1) / g.s2);
    } else {
        // Dynamic only: equal segments of each band, >= 64 columns, about three
        // chunks per resident warp.
        const long long per_band = static_cast<long long>(frames) * nbands;
        const long long want = std::max(64ll, std::min(512ll, g.units / (3 * resident)));
        const int nsegs = static_cast<int>(std::max(1ll, (iw + want - 1) / want));
        g.s2 = (iw + nsegs - 1) / nsegs;
        g.pitch = static_cast<int>(g.s2) * nsegs;
        g.nstatic = 0;
        g.s1 = 0;
        g.units = per_band * g.pitch;
        g.nchunks = static_cast<int>(per_band * nsegs);
    }
    return g;
}

#ifdef __CUDACC__
// Warp-uniform iterator over this warp's passes.  State (u, u_end) starts at
// (0, 0); each call returns the next pass (frame f, band kb, interior columns
// [x0, x1) relative to x_lo) or false when the launch's work is exhausted.
__device__ __forceinline__ bool next_pass(const WorkSplit& g, int* counter, int lane, long long& u,
                                          long long& u_end, int& f, int& kb, int& x0, int& x1) {
    for (;;) {
        if (u >= u_end) {
            int i = 0;
            if (lane == 0) i = atomicAdd(counter, 1);
            i = __shfl_sync(0xFFFFFFFFu, i, 0);
            if (i >= g.nchunks) return false;
            if (i < g.nstatic) {
                u = static_cast<long long>(i) * g.s1;
                u_end = u + g.s1;
            } else {
                u = static_cast<long long>(g.nstatic) * g.s1 +
                    static_cast<long long>(i - g.nstatic) * g.s2;
                u_end = u + g.s2;
            }
            if (u_end > g.units) u_end = g.units;
            continue;
        }
        const long long band = u / g.pitch;
        x0 = static_cast<int>(u - band * g.pitch);
        x1 = static_cast<int>(min(static_cast<long long>(g.iw), x0 + (u_end - u)));
        u = x1 == g.iw ? (band + 1) * g.pitch : u + (x1 - x0);
        f = static_cast<int>(band / g.nbands);
        kb = static_cast<int>(band - static_cast<long long>(f) * g.nbands);
        if (x1 <= x0) continue;
        return true;
    }
}
#endif

}  // namespace opc
