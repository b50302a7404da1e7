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

#ifndef OPC_SPLIT_MIN_SEG
#define OPC_SPLIT_MIN_SEG 32  // narrowest segment of the dynamic-only split
#endif

namespace opc {

struct WorkSplit {
    int nbands, iw, pitch;  // pitch >= iw: units per band (segment-aligned chunks)
    int nstatic, nchunks;
    long long units, s1, s2;
    // Guided mode (guided_div > 0): after the static chunks, the remainder is
    // claimed from a 64-bit unit counter in pieces of max(s2, remaining /
    // guided_div) -- large first, small at the end -- for kernels whose step
    // cost depends on the content (slide), where equal chunks leave a tail.
    long long guided_div;
    // Planned mode (cs != nullptr, device memory): chunk i is the unit range
    // [cs[i] * blk, cs[i + 1] * blk) -- chunk boundaries computed on the device
    // from the content (the slide kernel's equal-cost split), blk units per
    // block, pitch = blocks per band * blk.
    const int* cs;
    int blk;
};

// The planned split (see WorkSplit::cs): nchunks chunks over frames x nbands
// bands of nblk blocks of blk units (the last block of a band may be partial).
inline WorkSplit make_planned_split(int frames, int nbands, int iw, int nblk, int blk, int nchunks,
                                    const int* cs) {
    WorkSplit g{};
    g.nbands = nbands;
    g.iw = iw;
    g.pitch = nblk * blk;
    g.units = static_cast<long long>(frames) * nbands * g.pitch;
    g.nstatic = 0;
    g.nchunks = nchunks;
    g.cs = cs;
    g.blk = blk;
    return g;
}

inline WorkSplit make_split(int frames, int nbands, int iw, long long resident, int static_pct,
                            long long min_chunk, int dyn_per_warp = 2, int guided_k = 0) {
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
        // remainder: about dyn_per_warp chunks per resident warp
        const long long d = static_cast<long long>(dyn_per_warp) * resident;
        g.s2 = std::max(min_chunk, (rest + d - 1) / d);
        g.nchunks = g.nstatic + static_cast<int>((rest + g.s2 - 1) / g.s2);
        if (guided_k > 0) {
            g.s2 = min_chunk;
            g.guided_div = static_cast<long long>(guided_k) * resident;
            g.nchunks = g.nstatic;
        }
    } else {
        // Dynamic only: equal segments of each band, as many as fill ~85% of
        // the resident warps in one round (C2: 48-column segments, 13% faster
        // than 64; narrower segments pay more warm-up and skew fill per
        // output column, more chunks than warps add a round), 32..512 columns.
        const long long per_band = static_cast<long long>(frames) * nbands;
        const long long fit = std::max(1ll, resident * 85 / (100 * per_band));
        const long long want =
            std::max<long long>(OPC_SPLIT_MIN_SEG, std::min(512ll, (iw + fit - 1) / fit));
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

// Band-aligned split: every band cut into the same number of equal segments,
// at most one segment per resident warp, so no chunk crosses a band end and no
// warp takes a second pass.  For launches whose per-warp share is small (the
// bands of a multi-GPU split): there a pass's fixed cost (the skew kernel's
// 2(2r+1) + 32 steps of init lead, warm-up and fill / drain) is a large part of
// a share, and a dynamic remainder chunk is a whole extra pass for the warps
// that take it.  Returns false (g untouched) when the bands outnumber the warps.
inline bool make_aligned_split(int frames, int nbands, int iw, long long resident, int min_seg,
                               WorkSplit& g) {
    const long long per_band = static_cast<long long>(frames) * nbands;
    if (per_band > resident) return false;
    long long nsegs = resident / per_band;
    nsegs = std::max(1ll, std::min(nsegs, static_cast<long long>(iw) / std::max(1, min_seg)));
    WorkSplit w{};
    w.nbands = nbands;
    w.iw = iw;
    w.s2 = (iw + nsegs - 1) / nsegs;
    w.pitch = static_cast<int>(w.s2 * nsegs);
    w.nstatic = 0;
    w.s1 = 0;
    w.units = per_band * w.pitch;
    w.nchunks = static_cast<int>(per_band * nsegs);
    g = w;
    return true;
}

#ifdef __CUDACC__
#define OPC_HD __host__ __device__
#else
#define OPC_HD
#endif

// Units [u, u_end) of chunk i (i < nchunks).  PLANNED (compile time) reads
// the device-side chunk starts g.cs; the other kernels compile without that
// branch (the skew kernel's register allocation changed with it: C4 +14%).
template <bool PLANNED = false>
OPC_HD inline void chunk_range(const WorkSplit& g, int i, long long& u, long long& u_end) {
    if (PLANNED) {
        u = static_cast<long long>(g.cs[i]) * g.blk;
        u_end = static_cast<long long>(g.cs[i + 1]) * g.blk;
    } else if (i < g.nstatic) {
        u = static_cast<long long>(i) * g.s1;
        u_end = u + g.s1;
    } else {
        u = static_cast<long long>(g.nstatic) * g.s1 + static_cast<long long>(i - g.nstatic) * g.s2;
        u_end = u + g.s2;
    }
    if (u_end > g.units) u_end = g.units;
}

// Guided claim: given the units already claimed from the dynamic region
// (approximate is fine), the size of the next piece.
OPC_HD inline long long guided_size(const WorkSplit& g, long long claimed) {
    const long long dyn = g.units - static_cast<long long>(g.nstatic) * g.s1;
    const long long rem = dyn - claimed;
    const long long q = rem / g.guided_div;
    return q > g.s2 ? q : g.s2;
}

// Next pass inside [u, u_end): frame f, band kb, interior columns [x0, x1)
// (relative to x_lo); advances u.  False when the chunk is exhausted.  A pass
// never crosses a band end; the padding of a pitch > iw linearisation is skipped.
OPC_HD inline bool pass_in_chunk(const WorkSplit& g, long long& u, long long u_end, int& f, int& kb,
                                 int& x0, int& x1) {
    while (u < u_end) {
        const long long band = u / g.pitch;
        x0 = static_cast<int>(u - band * g.pitch);
        const long long rest = u_end - u;
        x1 = static_cast<int>(g.iw < x0 + rest ? g.iw : x0 + rest);
        u = x1 == g.iw ? (band + 1) * g.pitch : u + (x1 - x0);
        f = static_cast<int>(band / g.nbands);
        kb = static_cast<int>(band - static_cast<long long>(f) * g.nbands);
        if (x1 > x0) return true;
    }
    return false;
}

#ifdef __CUDACC__
// Warp-uniform iterator over this warp's passes.  State (u, u_end) starts at
// (0, 0); each call returns the next pass or false when the launch's work is
// exhausted.  Chunks are claimed by lane 0 from counter[0] (chunk index) and,
// in guided mode, counter[2..3] (64-bit unit count; 16-byte-aligned counter,
// 16 bytes zeroed by the launcher).
// GUIDED = false compiles the guided claim out (registers: the skew kernel for
// NB = 31 spilled with it).
template <bool GUIDED = false, bool PLANNED = false>
__device__ __forceinline__ bool next_pass(const WorkSplit& g, int* counter, int lane, long long& u,
                                          long long& u_end, int& f, int& kb, int& x0, int& x1) {
    for (;;) {
        if (pass_in_chunk(g, u, u_end, f, kb, x0, x1)) return true;
        if (!GUIDED) {
            int i = 0;
            if (lane == 0) i = atomicAdd(counter, 1);
            i = __shfl_sync(0xFFFFFFFFu, i, 0);
            if (i >= g.nchunks) return false;
            chunk_range<PLANNED>(g, i, u, u_end);
            continue;
        }
        long long a = 0, b = 0;
        int done = 0;
        if (lane == 0) {
            const int i = atomicAdd(counter, 1);
            if (i < g.nchunks) {
                chunk_range<PLANNED>(g, i, a, b);  // (an empty static chunk: claim again)
            } else if (g.guided_div > 0) {
                // counter[2..3]: the 64-bit count of dynamic units claimed
                unsigned long long* uc = reinterpret_cast<unsigned long long*>(counter + 2);
                const long long seen = static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(uc));
                const long long size = guided_size(g, seen);
                const long long base = static_cast<long long>(g.nstatic) * g.s1;
                a = base + static_cast<long long>(atomicAdd(uc, static_cast<unsigned long long>(size)));
                b = a + size < g.units ? a + size : g.units;
                done = a >= b;
            } else {
                done = 1;
            }
        }
        if (__shfl_sync(0xFFFFFFFFu, done, 0)) return false;
        u = __shfl_sync(0xFFFFFFFFu, a, 0);
        u_end = __shfl_sync(0xFFFFFFFFu, b, 0);
    }
}
#endif

}  // namespace opc
