// slide.cu -- kernel family for many bins (L+1 > 32, e.g. config 3's L = 256)
// with r <= 15.
//
// Huang's O(r) sliding histogram per lane (one output row per lane, the 32
// lanes on 32 consecutive rows at the same column):
//  * counts of the lane's window live in shared memory as u16 [bin][lane]
//    (a warp's dynamic-bin accesses touch 32 different lanes' halves: at most
//    2-way bank conflicts);
//  * stepping from x-1 to x adds column x+r and removes column x-r-1 (2(2r+1)
//    updates) -- skipped for the whole warp when every entering pixel equals
//    the leaving pixel of the same row (flat content: C3's rectangles);
//  * the lowest-index maximum (filter.hpp:71-82) is tracked incrementally: a
//    step that increments bins records the best post-increment (count, bin)
//    candidate; if the current winner lost pixels or the candidate was later
//    decremented, the lane rescans all bins;
//  * the winner's channel sums are tracked in registers and recomputed from
//    the window (2r+1)^2 when the winner changes; output = truncating quotient
//    (filter.cpp:41-43) via the exact reciprocal table.
// What the content allows is skipped: runs of flat steps are
// emitted at once and long flat stretches jumped without ring loads; a step
// whose rows form at most two runs of one (entering, leaving) bin pair is two
// weighted count updates; winner changes of several lanes to one bin share
// their row sums; uniform and striped pass starts are set up from 1 or 2r+1
// pixels.  The work plan (slide_plan_kernel) balances the passes by cost.
// Pixels come from a transposed (column-major) entry plane written by the
// shared pre-pass, so a ring column (32+2r rows) is one contiguous run: the
// ring is filled by TMA (one 2D box of 16 columns x the band's rows per
// chunk, completion on an mbarrier), two chunks ahead of the slide.  Finished
// 16-column output blocks leave through a TMA store (the rows' 48 bytes each,
// clipped by the hardware at the interior end and the band end).
#include <cmath>
#include <cstdio>

#include "kernels.cuh"
#include "border.cuh"
#include "tma.cuh"
#include "worksplit.cuh"


namespace opc {

namespace {

#ifndef OPC_SLIDE_TRACE
#define OPC_SLIDE_TRACE 0
#endif
#ifndef OPC_SLIDE_UNROLL_SCAN
#define OPC_SLIDE_UNROLL_SCAN 16
#endif
#ifndef OPC_SLIDE_UNROLL_SUMS
#define OPC_SLIDE_UNROLL_SUMS 16
#endif
#ifndef OPC_SLIDE_GUIDED_K
#define OPC_SLIDE_GUIDED_K 0  // > 0: guided claims of remaining / (k x resident warps); measured no gain on C3
#endif
#ifndef OPC_SLIDE_MIN_CHUNK
#define OPC_SLIDE_MIN_CHUNK 128
#endif
#ifndef OPC_SLIDE_DYN_PER_WARP
#define OPC_SLIDE_DYN_PER_WARP 2
#endif
#ifndef OPC_SLIDE_ATOMICS
#define OPC_SLIDE_ATOMICS 1  // count updates of a step as shared-memory atomics (no RMW chain)
#endif
#ifndef OPC_SLIDE_UNROLL_CHANGE
#define OPC_SLIDE_UNROLL_CHANGE 7  // winner-change column sums: loads in flight per lane
#endif
#ifndef OPC_SLIDE_PACKED_SUMS
#define OPC_SLIDE_PACKED_SUMS 1  // step updates: packed winner-sum differences, PRMT keys, 32-bit shared addresses (C3 slide 252 -> 213 us)
#endif
#ifndef OPC_SLIDE_RUNS
#define OPC_SLIDE_RUNS 1  // steps whose rows form at most two runs of one (entering, leaving) bin pair: two weighted count updates
#endif
#ifndef OPC_SLIDE_BAND_ORDER
#define OPC_SLIDE_BAND_ORDER 1  // the work plan takes the bands costliest first
#endif
#ifndef OPC_SLIDE_ROW_SUMS
#define OPC_SLIDE_ROW_SUMS 1  // winner changes of several lanes to one bin: shared row sums + prefix differences
#endif
#ifndef OPC_SLIDE_STRIPED_START
#define OPC_SLIDE_STRIPED_START 1  // pass starts on horizontal / vertical stripes: 2r + 1 weighted count updates
#endif
#ifndef OPC_SLIDE_COST_COLS
#define OPC_SLIDE_COST_COLS 32  // columns per unit of the work plan (32, 16 or 8; A/B on C3: 137 / 138 / 142 us -- finer chunks start more passes inside busy regions)
#endif
#ifndef OPC_SLIDE_JUMP
#define OPC_SLIDE_JUMP 1  // flat stretches of kJumpMin phases or more: no ring loads, the stretch is emitted at once
#endif
#ifndef OPC_SLIDE_JUMP_MIN
#define OPC_SLIDE_JUMP_MIN 4
#endif
#ifndef OPC_SLIDE_UNROLL_UPDATE
#define OPC_SLIDE_UNROLL_UPDATE 7  // rows of a step's update loop in flight (A/B on C3: 1 / 3 / 7 / 11 / 21 rows -> 235 / 225 / 213 / 221 / 214 us)
#endif
#ifndef OPC_SLIDE_PLAN
#define OPC_SLIDE_PLAN 1  // equal-cost chunks from the column-change masks (0: static + dynamic split)
#endif
#ifndef OPC_SLIDE_PLAN_CPW
#define OPC_SLIDE_PLAN_CPW 4  // planned chunks per resident warp
#endif
#ifndef OPC_SLIDE_PLAN_K
#define OPC_SLIDE_PLAN_K 1  // > 0: decreasing chunk sizes (remaining / (K x warps)), see TGeom
#endif
#ifndef OPC_SLIDE_PLAN_M
#define OPC_SLIDE_PLAN_M 4  // smallest chunk of the decreasing plan: total / (M x warps) (a pass start costs ~10 us: 16 -> 4 with the flat-stretch jumps, C3 -3%)
#endif
#ifndef OPC_SLIDE_COST_K
#define OPC_SLIDE_COST_K 200  // cost of a window-changing step in flat columns (work plan; fitted on per-pass traces: ~1.9 us against ~9 ns once flat stretches are jumped)
#endif
#ifndef OPC_SLIDE_PAR_SUMS
#define OPC_SLIDE_PAR_SUMS 4  // winner changes in one step from which lanes sum their windows in parallel
#endif
#ifndef OPC_SLIDE_STATIC_PCT
#define OPC_SLIDE_STATIC_PCT 50  // content-dependent step costs: 90 measured 20% slower on C3
#endif

constexpr int kWarps = 8;  // upper bound; the launcher fits as many as 227 KB allows
// Ring of entry columns, filled by TMA in chunks of kChunk columns: kSlots
// chunks, i.e. the window (2r+1 <= 31 columns) + the phase being slid + two
// chunks in flight.  Column c of a pass (image column xs - r + c) lives in
// chunk k = (c - B) / kChunk with B = 2r - kChunk * K0, K0 = ceil((2r + 1) / kChunk):
// phase p (output columns 16p .. 16p+15) enters exactly chunk p + K0.
constexpr int kChunk = 16;
constexpr int kSlots = 5;
constexpr int kRingCols = kChunk * kSlots;
constexpr int kUnrollScan = OPC_SLIDE_UNROLL_SCAN;
constexpr int kUnrollSums = OPC_SLIDE_UNROLL_SUMS;
constexpr int kUnrollChange = OPC_SLIDE_UNROLL_CHANGE;
constexpr int kUnrollUpdate = OPC_SLIDE_UNROLL_UPDATE;
constexpr int kJumpMin = OPC_SLIDE_JUMP_MIN;
constexpr int kCostCols = OPC_SLIDE_COST_COLS;
static_assert(kCostCols == 32 || kCostCols == 16 || kCostCols == 8, "cost blocks divide the 32-column nonflat words");
constexpr int kStageCols = 16;   // output columns staged per flush (== kChunk)
constexpr int kStageStride = 17;
constexpr int kRecipBytes = 1024 * 4;
constexpr int kTRows = 32;
constexpr int kTCols = 128;

__host__ __device__ inline int ring_rows(int r) { return (32 + 2 * r + 3) & ~3; }  // 16-B rows
// chunks spanned by a window's 2r + 1 columns (so the column a step removes, x - 1,
// is in chunk p of phase p, never in the slot being refilled)
__host__ __device__ inline int chunk_k0(int r) { return (2 * r + kChunk) / kChunk; }

// Per-warp shared memory, 128-byte aligned pieces (TMA boxes):
//   ring  kRingCols x ring_rows u32 | out tile 32 rows x 48 bytes |
//   counts bins x 32 lanes u16 | stage 32 x kStageStride u32 | kSlots mbarriers
__host__ __device__ inline std::size_t ring_bytes(int r) {
    return static_cast<std::size_t>(kRingCols) * ring_rows(r) * 4;
}
constexpr std::size_t kOutTileBytes = 32 * 3 * kStageCols;
__host__ __device__ inline std::size_t cnt_bytes(int bins) {
    return ((static_cast<std::size_t>(bins) * 32 * 2) + 15) & ~std::size_t(15);
}
__host__ __device__ inline std::size_t per_warp_bytes(int bins, int r) {
    const std::size_t b = ring_bytes(r) + kOutTileBytes + cnt_bytes(bins) + 32 * kStageStride * 4 +
                          kSlots * 8;
    return (b + 127) & ~std::size_t(127);
}

// Geometry of a launch's transposed plane and of the work plan built from it.
// Scratch layout: plane | column-change masks | nonflat bits | block costs |
// chunk starts.
struct TGeom {
    int y_base;
    int Hs;  // rows per column (multiple of 32)
    std::size_t frame_elems;
    int ncols;    // plane columns: W + 64
    int ntr;      // 32-row tiles per column: Hs / 32
    int nbands;   // 32-row bands of the launch
    int nblk;     // 32-column blocks (nonflat words) per band: ceil((x_hi - x_lo) / 32)
    int ncb;      // cost blocks (the plan's units, kCostCols columns) per band: nblk * 32 / kCostCols
    int nch;      // chunks of the cost-balanced split
    std::uint32_t* dmask;  // [frame][ntr][ncols]: bit y of (tile, column c) = plane rows
                           // 32 tile + y of columns c and c - (2r + 1) differ
    std::uint32_t* nf;     // [frame][nband][nblk]: bit x = step at interior column
                           // 32 blk + x changes the window (not flat)
    std::uint32_t* bc;     // [frame][nband][ncb]: cost of the cost block's columns
    int* cs;               // [nch + 1]: first block of each chunk
    int* perm;             // [frames x nbands]: the plan's band order (position -> band), costliest first
    // Decreasing chunk sizes (OPC_SLIDE_PLAN_K > 0): chunk j covers the cost
    // fractions [1 - q^j, 1 - q^(j+1)) with q = 1 - 1 / (K x resident) -- each
    // the remaining cost / (K x resident), guided self-scheduling precomputed --
    // until chunks would shrink below 1 / (M x resident) of the total, then
    // equal chunks of that size (from fraction xJ on, chunk J on).
    float lnq;  // ln q (0: equal-cost chunks)
    float xJ;   // 1 - q^J
    float rm;   // M x resident
    int J;
};

__host__ inline int plan_chunks(long long blocks, long long resident);

__host__ inline TGeom tgeom(const BandArgs& a, void* scratch = nullptr, long long resident = 0) {
    TGeom g{};
    g.y_base = a.y_lo - a.radius;
    g.nbands = (a.y_hi - a.y_lo + 31) / 32;
    g.Hs = 32 * g.nbands + 64;
    g.ncols = a.width + 64;
    g.ntr = g.Hs / 32;
    g.frame_elems = static_cast<std::size_t>(g.ncols) * g.Hs;
    g.nblk = (a.x_hi - a.x_lo + 31) / 32;
    g.ncb = g.nblk * (32 / kCostCols);
    const long long words = static_cast<long long>(a.frames) * g.nbands * g.nblk;
    const long long blocks = static_cast<long long>(a.frames) * g.nbands * g.ncb;
    g.nch = plan_chunks(blocks, resident);
    if (OPC_SLIDE_PLAN_K > 0 && resident > 0) {
        const double R = static_cast<double>(resident), K = OPC_SLIDE_PLAN_K, M = OPC_SLIDE_PLAN_M;
        const double lnq = std::log1p(-1.0 / (K * R));
        const int J = static_cast<int>(std::ceil(std::log(K / M) / lnq));
        const double xJ = 1.0 - std::exp(J * lnq);
        const long long n = J + static_cast<long long>(std::ceil((1.0 - xJ) * M * R)) + 2;
        // (a launch with fewer 32-column blocks than that keeps equal chunks:
        // clamping the guided map would pile its tail onto the last chunk)
        if (n <= blocks) {
            g.lnq = static_cast<float>(lnq);
            g.J = J;
            g.xJ = static_cast<float>(xJ);
            g.rm = static_cast<float>(M * R);
            g.nch = static_cast<int>(n);
        }
    }
    if (scratch) {
        std::uint32_t* p = static_cast<std::uint32_t*>(scratch) + g.frame_elems * a.frames;
        g.dmask = p;
        p += static_cast<std::size_t>(a.frames) * g.ntr * g.ncols;
        g.nf = p;
        p += words;
        g.bc = p;
        p += blocks;
        g.cs = reinterpret_cast<int*>(p);
        g.perm = g.cs + blocks + 2;
    }
    return g;
}

__host__ inline std::size_t tgeom_bytes(const BandArgs& a) {
    const TGeom g = tgeom(a);
    const long long words = static_cast<long long>(a.frames) * g.nbands * g.nblk;
    const long long blocks = static_cast<long long>(a.frames) * g.nbands * g.ncb;
    // plan_chunks never exceeds the block count (+1 for the end marker)
    return (g.frame_elems * a.frames + static_cast<std::size_t>(a.frames) * g.ntr * g.ncols +
            static_cast<std::size_t>(words) + 2 * static_cast<std::size_t>(blocks) + 2 +
            static_cast<std::size_t>(a.frames) * g.nbands) *
           sizeof(std::uint32_t);
}

// Chunks of the cost-balanced split: OPC_SLIDE_PLAN_CPW per resident warp, at
// most one per 32-column block.
__host__ inline int plan_chunks(long long blocks, long long resident) {
    long long n = resident > 0 ? resident * OPC_SLIDE_PLAN_CPW : blocks;
    if (n > blocks) n = blocks;
    if (n < 1) n = 1;
    return static_cast<int>(n);
}

// Column-major plane of raw RGB (R | G << 8 | B << 16), rows [y_base, y_base + Hs);
// rows past the input are zero.  32 x 128 tiles through shared memory, plus
// 32 halo columns on the left; each column's 32 rows are one 128-byte store.
// The same tile gives the column-change masks of the work plan: for plane
// column c, the rows where c and c - (2r + 1) differ (a slide step at output
// column c - r adds column c and removes column c - 2r - 1).  Interior tiles
// load 3 words (4 pixels) per lane and row.
constexpr int kTStride = 32 + kTCols + 1;  // odd: lane-per-row column reads hit distinct banks
__device__ __forceinline__ std::uint32_t brg_word(std::uint32_t t) { return t & 0xFFFFFFu; }

__global__ void __launch_bounds__(256) transpose_kernel(BandArgs a, std::uint32_t* T, TGeom g, int vec_ok) {
    __shared__ std::uint32_t tile[kTRows * kTStride];
    if (static_cast<int>(blockIdx.y) >= g.Hs / kTRows) {  // appended border blocks
        const int b = (blockIdx.y - g.Hs / kTRows) * gridDim.x + blockIdx.x;
        if (b < a.border.nblocks) border_block(a, b, blockIdx.z, threadIdx.x);
        return;
    }
    const int x0 = blockIdx.x * kTCols;
    const int y0 = g.y_base + blockIdx.y * kTRows;
    const int frame = blockIdx.z;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    std::uint32_t* Tf = T + g.frame_elems * frame;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const int in_hi = a.in_row0 + a.in_rows;
    if (vec_ok && x0 >= 32 && x0 + kTCols <= a.width && y0 + kTRows <= in_hi) {
        // words of pixels [x0 - 32, x0 + 128): 120 per row; lane l loads words
        // 3l .. 3l+2 (pixels 4l .. 4l+3) and lanes < 8 also words 96 + 3l ..
#pragma unroll
        for (int k = 0; k < kTRows / 8; ++k) {
            const int row = warp + 8 * k;
            const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(
                in + static_cast<std::size_t>(y0 + row - a.in_row0) * stride +
                static_cast<std::size_t>(x0 - 32) * 3);
            std::uint32_t* trow = tile + row * kTStride;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int l = lane + 32 * h;  // 4-pixel group
                if (l < 40) {
                    const std::uint32_t w0 = __ldg(src + 3 * l), w1 = __ldg(src + 3 * l + 1),
                                        w2_ = __ldg(src + 3 * l + 2);
                    // bytes R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
                    trow[4 * l + 0] = brg_word(w0);
                    trow[4 * l + 1] = __byte_perm(w0, w1, 0x0543) & 0xFFFFFFu;  // (byte 3: zero)
                    trow[4 * l + 2] = __byte_perm(w1, w2_, 0x0432) & 0xFFFFFFu;
                    trow[4 * l + 3] = w2_ >> 8;
                }
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kTRows / 8; ++k) {
            const int row = warp + 8 * k;
            const int y = y0 + row;
#pragma unroll
            for (int j = 0; j < (32 + kTCols) / 32; ++j) {
                const int c = lane + 32 * j;
                const int x = x0 - 32 + c;
                std::uint32_t e = 0;
                if (x >= 0 && x < a.width && y < in_hi) {
                    const std::uint8_t* p = in + static_cast<std::size_t>(y - a.in_row0) * stride +
                                            static_cast<std::size_t>(x) * 3;
                    e = p[0] | (static_cast<std::uint32_t>(p[1]) << 8) |
                        (static_cast<std::uint32_t>(p[2]) << 16);
                }
                tile[row * kTStride + c] = e;
            }
        }
    }
    __syncthreads();
    const int w2 = 2 * a.radius + 1;
    std::uint32_t* dm = g.dmask + (static_cast<std::size_t>(frame) * g.ntr + blockIdx.y) * g.ncols;
    // (pointers stepped per column, the plane's column bound hoisted: the
    // tile rows are all inside the plane -- Hs is a multiple of the tile height)
    const int cmax = min(kTCols, g.ncols - x0);
    const std::uint32_t* tl = tile + lane * kTStride + 32 + warp;
    std::uint32_t* tp = Tf + static_cast<std::size_t>(x0 + warp) * g.Hs + (y0 + lane - g.y_base);
    std::uint32_t* dp = dm + x0 + warp;
    const std::size_t tstep = static_cast<std::size_t>(8) * g.Hs;
    for (int c = warp; c < cmax; c += 8) {
        const std::uint32_t v = tl[0];
        const std::uint32_t m = __ballot_sync(0xFFFFFFFFu, v != tl[-w2]);
        *tp = v;
        if (lane == 0) *dp = m;
        tl += 8;
        tp += tstep;
        dp += 8;
    }
}

// Work plan.  Step 1 (a warp per 4 blocks of 32 interior columns of a band):
// the nonflat bit of every interior column -- a step changes the window iff
// any of the band's 32 + 2r ring rows differs between the entering and the
// leaving column (tile rows kb and the first 2r rows of kb + 1) -- and the
// cost of every block: its columns + OPC_SLIDE_COST_K per nonflat step.
// Step 2, by the last CTA to finish (threadfence + counter): the exclusive
// prefix of the block costs and the first block of each of nch equal-cost
// chunks (a block heavier than a chunk leaves empty chunks behind it; any
// monotone block -> chunk map gives a valid partition, so the float scaling
// is exact enough).
constexpr int kCostBlocksPerWarp = 4;
constexpr int kPlanThreads = 1024;
constexpr long long kPlanSmemCap = 40 * 1024;  // block costs staged in shared memory (160 KB)
__global__ void __launch_bounds__(kPlanThreads) slide_plan_kernel(BandArgs a, TGeom g, long long nblocks,
                                                                  unsigned* done, int smem_cap) {
    extern __shared__ std::uint32_t sbc[];  // the block costs, when they fit (smem_cap entries)
    __shared__ std::uint32_t s_total_;
    __shared__ bool last;
    const int lane = threadIdx.x & 31;
    const int nq = (g.nblk + kCostBlocksPerWarp - 1) / kCostBlocksPerWarp;
    const long long wid = static_cast<long long>(blockIdx.x) * (kPlanThreads / 32) + (threadIdx.x >> 5);
    const int r = a.radius;
    if (wid < static_cast<long long>(a.frames) * g.nbands * nq) {
        const int band = static_cast<int>(wid / nq), q = static_cast<int>(wid - static_cast<long long>(band) * nq);
        const int f = band / g.nbands, kb = band - f * g.nbands;
        const int iw = a.x_hi - a.x_lo;
        const std::uint32_t low = r > 0 ? (0xFFFFFFFFu >> (32 - 2 * r)) : 0u;
        const std::uint32_t* d0 = g.dmask + (static_cast<std::size_t>(f) * g.ntr + kb) * g.ncols;
        const std::uint32_t* d1 = d0 + g.ncols;
        std::uint32_t m[kCostBlocksPerWarp];
#pragma unroll
        for (int i = 0; i < kCostBlocksPerWarp; ++i) {
            const int x = 32 * (kCostBlocksPerWarp * q + i) + lane;
            const int c = a.x_lo + x + r;  // entering plane column of the step at x
            m[i] = x < iw ? (d0[c] | (d1[c] & low)) : 0u;
        }
#pragma unroll
        for (int i = 0; i < kCostBlocksPerWarp; ++i) {
            const int j = kCostBlocksPerWarp * q + i;
            const std::uint32_t word = __ballot_sync(0xFFFFFFFFu, m[i] != 0u);
            if (lane == 0 && j < g.nblk) {
                g.nf[static_cast<std::size_t>(band) * g.nblk + j] = word;
                constexpr int per = 32 / kCostCols;
#pragma unroll
                for (int sb = 0; sb < per; ++sb) {
                    const int cols = max(0, min(kCostCols, iw - 32 * j - kCostCols * sb));
                    const std::uint32_t bits = (word >> (kCostCols * sb)) & (0xFFFFFFFFu >> (32 - kCostCols));
                    g.bc[static_cast<std::size_t>(band) * g.ncb + per * j + sb] =
                        static_cast<std::uint32_t>(cols) + OPC_SLIDE_COST_K * __popc(bits);
                }
            }
        }
    }
    if (!OPC_SLIDE_PLAN) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // ---- step 2: the last CTA ----
#if OPC_PLAN_CLOCK
    long long ck[8];
    ck[0] = clock64();
#define PLAN_TICK(i) ck[i] = clock64()
#else
#define PLAN_TICK(i)
#endif
    // The block costs are staged in shared memory when they fit (one
    // coalesced copy through L2 -- other CTAs wrote them).
    const int t = threadIdx.x;
    if (t == 0) *done = 0u;  // every CTA has arrived: ready for the next launch
    // Band order of the plan: costliest bands first.  The estimates are worst
    // where the content is busiest (rescans, winner changes and non-flat pass
    // starts are not in them), and the guided plan's chunks shrink along the
    // order: the busy bands get the early, large chunks and the tail is flat,
    // predictable work.  (Up to kPlanThreads bands; more keep their order.)
    const int nb = a.frames * g.nbands;
    __shared__ std::uint32_t band_cost[kPlanThreads];
    __shared__ int band_at[kPlanThreads];  // position -> band
    const bool ordered = OPC_SLIDE_BAND_ORDER && nb <= kPlanThreads;
    if (ordered) {
        // (a warp per band: coalesced loads of its block costs, one reduction)
        for (int b = t >> 5; b < nb; b += kPlanThreads / 32) {
            std::uint32_t c = 0;
#pragma unroll 4
            for (int j = lane; j < g.ncb; j += 32) c += __ldcg(g.bc + static_cast<long long>(b) * g.ncb + j);
            c = __reduce_add_sync(0xFFFFFFFFu, c);
            if (lane == 0) band_cost[b] = c;
        }
        __syncthreads();
        if (t < nb) {
            const std::uint32_t c = band_cost[t];
            int rank = 0;
            for (int j = 0; j < nb; ++j) {
                const std::uint32_t o = band_cost[j];
                rank += (o > c || (o == c && j < t)) ? 1 : 0;
            }
            band_at[rank] = t;
            g.perm[rank] = t;
        }
        __syncthreads();
    } else {
        for (int i = t; i < nb; i += kPlanThreads) g.perm[i] = i;
    }
    // block at position i of the plan's order
    auto block_at = [&](long long i) -> long long {
        if (!ordered) return i;
        // (block indices fit 32 bits: the chunk starts are ints)
        const unsigned ii = static_cast<unsigned>(i), ncb = static_cast<unsigned>(g.ncb);
        const unsigned pos = ii / ncb;
        return static_cast<long long>(band_at[pos]) * g.ncb + (ii - pos * ncb);
    };
    PLAN_TICK(4);
    const bool staged = nblocks <= smem_cap;
    if (staged) {
        // (padded: entry b at b + b / 16, so 16 consecutive blocks per lane
        // read conflict-free)
        // (a warp per band position: coalesced loads of the band's costs in
        // batches of 4, no index division)
        const int nbp = a.frames * g.nbands;
        for (int pos = t >> 5; pos < nbp; pos += kPlanThreads / 32) {
            const long long src = static_cast<long long>(ordered ? band_at[pos] : pos) * g.ncb;
            const int dst = pos * g.ncb;
            for (int j0 = lane; j0 < g.ncb; j0 += 4 * 32) {
                std::uint32_t v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = j0 + 32 * k < g.ncb ? __ldcg(g.bc + src + j0 + 32 * k) : 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int i = dst + j0 + 32 * k;
                    if (j0 + 32 * k < g.ncb) sbc[i + (i >> 4)] = v[k];
                }
            }
        }
    }
    for (int i = t; i <= g.nch; i += kPlanThreads) g.cs[i] = static_cast<int>(nblocks);
    __syncthreads();
    PLAN_TICK(1);
    // (32-bit block indices from here on: the chunk starts are ints)
    const int nbl = static_cast<int>(nblocks);
    auto cost = [&](int b) -> std::uint32_t {
        return staged ? sbc[b + (b >> 4)] : __ldcg(g.bc + block_at(b));
    };
    // Thread t owns a contiguous run of blocks [t * per, (t + 1) * per): the
    // run sums, one CTA scan of the 1024 sums (warp shuffles + the 32 warp
    // totals), then each thread walks its run in registers to get every
    // block's exclusive prefix E_b.  32-bit arithmetic (totals past 2^32 are
    // clamped) and the block -> chunk map E_b * nch / total in float: any
    // monotone map gives a valid partition.
    __shared__ std::uint32_t wsum[32];
    const int w = t >> 5;
    const int per = (nbl + kPlanThreads - 1) / kPlanThreads;
    const int b0 = min(nbl, per * t), b1 = min(nbl, b0 + per);
    std::uint32_t mine = 0;
    for (int b = b0; b < b1; ++b) mine += cost(b);
    std::uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const std::uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (t < 32) {
        const std::uint32_t v = wsum[t];
        std::uint32_t wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const std::uint32_t u = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (t >= o) wi += u;
        }
        __syncwarp();
        wsum[t] = wi - v;  // exclusive
        if (t == 31) s_total_ = wi;
    }
    __syncthreads();
    PLAN_TICK(2);
    const std::uint32_t total = static_cast<std::uint32_t>(s_total_);
    if (total == 0) return;
    const float scale = static_cast<float>(g.nch) / static_cast<float>(total);
    const float inv_total = 1.0f / static_cast<float>(total);
    const float inv_lnq = g.lnq != 0.0f ? 1.0f / g.lnq : 0.0f;
    auto chunk_of = [&](std::uint32_t e) {
        if (g.lnq == 0.0f) return static_cast<int>(static_cast<float>(e) * scale);
        const float x = static_cast<float>(e) * inv_total;  // cost fraction before the block
        // (fast logarithm: the walk below keeps the map monotone)
        const int j = x < g.xJ ? static_cast<int>(__logf(1.0f - x) * inv_lnq)
                               : g.J + static_cast<int>((x - g.xJ) * g.rm);
        return min(j, g.nch - 1);
    };
    std::uint32_t e_b = wsum[w] + incl - mine;  // cost before b0
    if (staged) {
        // The staged costs become their exclusive prefixes in place; chunk i
        // then starts at the first block whose prefix reaches the chunk's cost
        // threshold (the inverse of the block -> chunk map: 1 - q^i of the
        // total in the decreasing part, equal steps after it) -- a binary
        // search per chunk instead of a map evaluation per block.  (Should
        // rounding ever order two neighbouring thresholds the wrong way, a few
        // blocks are filtered twice with the same result: every block stays
        // covered.)
        for (int b = b0; b < b1; ++b) {
            const int k = b + (b >> 4);
            const std::uint32_t c = sbc[k];
            sbc[k] = e_b;
            e_b += c;
        }
        __syncthreads();
        for (int i = t; i < g.nch; i += kPlanThreads) {
            float x;  // cost fraction before chunk i
            if (g.lnq == 0.0f) {
                x = static_cast<float>(i) / static_cast<float>(g.nch);
            } else if (i < g.J) {
                x = 1.0f - expf(static_cast<float>(i) * g.lnq);
            } else {
                x = g.xJ + static_cast<float>(i - g.J) / g.rm;
            }
            const float thr_f = x * static_cast<float>(total);
            const std::uint32_t thr = thr_f >= 4294967040.0f ? 0xFFFFFFFFu : static_cast<std::uint32_t>(thr_f);
            int lo = 0, hi = nbl;  // first block with prefix >= thr
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sbc[mid + (mid >> 4)] >= thr) {
                    hi = mid;
                } else {
                    lo = mid + 1;
                }
            }
            g.cs[i] = i == 0 ? 0 : lo;
        }
    } else {
        int prev = b0 == 0 ? -1 : chunk_of(e_b - cost(b0 - 1));
        for (int b = b0; b < b1; ++b) {
            // block b belongs to chunk(E_b), E_b = cost before b; the chunks
            // starting at b are (chunk(E_{b-1}), chunk(E_b)]
            const int cur = max(prev, chunk_of(e_b));
            for (int i = prev + 1; i <= cur && i < g.nch; ++i) g.cs[i] = b;
            prev = cur;
            e_b += cost(b);
        }
    }
    PLAN_TICK(3);
#if OPC_PLAN_CLOCK
    if (t == 0) {
        printf("plan clocks: band order %lld stage %lld sums %lld walk %lld (start %lld)\n", ck[4] - ck[0], ck[1] - ck[4],
               ck[2] - ck[1], ck[3] - ck[2], ck[0]);
    }
#endif
}

// c + sum of (unsigned bytes of a) x (signed bytes of b)
__device__ __forceinline__ std::int32_t dp4a_us(std::uint32_t a, std::uint32_t b, std::int32_t c) {
    std::int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ std::uint32_t bin_of(std::uint32_t e, std::uint32_t bin_mul) {
    const std::uint32_t s = __dp4a(e, 0x00010101u, 0u);  // R + G + B
    return __umulhi(s, bin_mul);                          // filter.hpp:31-35
}

#if !OPC_SLIDE_TRACE
#define SEC_ADD(i, t0) do { } while (0)
#define SEC_NOW() 0ll
#endif
#if OPC_SLIDE_TRACE
// Debug trace of the passes (OPC_SLIDE_TRACE builds only): per pass
// {smid << 48 | kb << 24 | x0, x1, start ns, end ns}.
__device__ unsigned long long g_trace[1 << 16][4];
__device__ int g_trace_n;
// Section clocks (lane 0 of every warp, summed): 0 pass start (claim to first
// output), 1 step walk (bins, sums, change points), 2 count updates, 3 winner
// resolution (rescans), 4 winner-change sums, 5 flat emission, 6 jumps,
// 7 single-column emit + flush, 8 phase top (ring waits / requests).
__device__ unsigned long long g_sec[16];
#define SEC_T0() const long long sec_t0_ = clock64()
#ifndef OPC_TRACE_MAXW
#define OPC_TRACE_MAXW (1 << 30)  // section clocks only in passes at most this wide
#endif
#define SEC_ADD(i, t0) do { if (lane == 0 && sec_on) sec_acc[i] += clock64() - (t0); } while (0)
#define SEC_NOW() clock64()
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// COUNT: the measurement instantiation (OPC_FLAG_COUNT_OPS): the same
// kernel, also counting the primitives it executes (OpCount) per lane and
// adding them to a.op_counts at exit.  TMA_OUT: output blocks leave through
// TMA stores (needs 16-byte aligned rows: width % 16 == 0); otherwise byte
// stores.
template <bool COUNT, bool TMA_OUT>
__global__ void __launch_bounds__(kWarps * 32)
    slide_kernel(BandArgs a, TGeom tg, int* task_counter, WorkSplit g,
                 const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout) {
    unsigned long long opc_n[kOpCountN] = {};
    [[maybe_unused]] long long sec_acc[16] = {};
    [[maybe_unused]] bool sec_on = true;
    auto tally = [&](int k, unsigned long long v) {
        if constexpr (COUNT) opc_n[k] += v;
    };
    extern __shared__ __align__(128) unsigned char smem[];
    std::uint32_t* recip = reinterpret_cast<std::uint32_t*>(smem);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int r = a.radius;
    const int w2 = 2 * r + 1;
    const int kb_ = 16 - (32 - __clz(w2 * w2));  // key bits below the count (>= 6 for r <= 15)
    const unsigned inc = 1u << kb_, gmask = inc - 1;
    const int gsize = 1 << kb_;
    const int bins = a.levels + 1;
    const int RR = ring_rows(r);
    unsigned char* wbase = smem + kRecipBytes + warp * per_warp_bytes(bins, r);
    std::uint32_t* ring = reinterpret_cast<std::uint32_t*>(wbase);
    std::uint32_t* const ring_end = ring + kRingCols * RR;
    std::uint8_t* otile = wbase + ring_bytes(r);
    std::uint16_t* cnt = reinterpret_cast<std::uint16_t*>(otile + kOutTileBytes);
    std::uint32_t* stage = reinterpret_cast<std::uint32_t*>(reinterpret_cast<unsigned char*>(cnt) +
                                                            cnt_bytes(bins));
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(stage + 32 * kStageStride);

    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
    if (lane == 0) {
        for (int k = 0; k < kSlots; ++k) mbar_init(bar + k, 1);
        fence_mbar_init();
        if (warp == 0) {
            prefetch_tensor_map(&tin);
            if constexpr (TMA_OUT) prefetch_tensor_map(&tout);
        }
    }
    __syncthreads();

    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const std::uint32_t bm = a.bin_mul;
    const unsigned FULL = 0xFFFFFFFFu;
    const int K0 = chunk_k0(r);
    const int B = 2 * r - kChunk * K0;  // first column of chunk 0 (<= 0)
    const unsigned box_bytes = static_cast<unsigned>(kChunk * RR * 4);
    unsigned q0 = 0;  // chunks this warp has issued before the current pass (slot = q % kSlots)

    long long u = 0, u_end = 0;
    int f, kb, x0, x1;
    while (next_pass<(OPC_SLIDE_GUIDED_K > 0), (OPC_SLIDE_PLAN != 0)>(g, task_counter, lane, u, u_end, f, kb,
                                                                       x0, x1)) {
        if (OPC_SLIDE_PLAN) {  // the plan's band order (position -> band)
            const int band = __ldg(tg.perm + f * tg.nbands + kb);
            f = band / tg.nbands;
            kb = band - f * tg.nbands;
        }
#if OPC_SLIDE_TRACE
        sec_on = x1 - x0 <= OPC_TRACE_MAXW;
        if (lane == 0 && sec_on) sec_acc[9] += 1;
        int pass_cols = x1 - x0;
        const unsigned long long t_start = gtime();
        struct TraceGuard {
            int kb, x0, &cols, lane, stolen;
            unsigned long long t0;
            __device__ ~TraceGuard() {
                if (lane == 0) {
                    unsigned smid;
                    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                    const int i = atomicAdd(&g_trace_n, 1);
                    if (i < (1 << 16)) {
                        g_trace[i][0] = (static_cast<unsigned long long>(smid) << 48) |
                                        (static_cast<unsigned long long>(kb) << 24) | x0;
                        g_trace[i][1] = static_cast<unsigned long long>(x0 + cols) |
                                        (static_cast<unsigned long long>(stolen) << 30);
                        g_trace[i][2] = t0;
                        g_trace[i][3] = gtime();
                    }
                }
            }
        } trace_guard{kb, x0, pass_cols, lane, 0, t_start};
#endif
        [[maybe_unused]] const long long t_pass = SEC_NOW();
        const int yb = a.y_lo + 32 * kb;
        const int xs = a.x_lo + x0;
        const int xe = a.x_lo + x1;
        const int n = xe - xs;
        const bool row_ok = yb + lane < a.y_hi;
        const int row0 = yb - r - tg.y_base;  // plane row of ring row 0
        std::uint8_t* out = a.out + a.out_frame_stride * f;
        // chunks of this pass: columns up to n - 1 + 2r
        const int kmax = (n - 1 + 2 * r - B) / kChunk;
        // ring position (u32 offset) of pass column c: chunk (c - B) / 16 in
        // slot (q0 + chunk) % kSlots -- i.e. (16 * (q0 % kSlots) + c - B) mod 80
        int pos0 = kChunk * static_cast<int>(q0 % kSlots) - B;  // (re-based by a jump over flat phases)
        auto ringp = [&](int c) { return ring + ((pos0 + c) % kRingCols) * RR + lane; };
        auto issue = [&](int k) {  // lane 0: chunk k of the pass
            const unsigned q = q0 + static_cast<unsigned>(k);
            std::uint64_t* b = bar + q % kSlots;
            mbar_arrive_expect_tx(b, box_bytes);
            tma_load_3d(ring + (q % kSlots) * kChunk * RR, &tin, row0, xs - r + B + kChunk * k, f, b);
        };
        auto wait = [&](int k) {
            const unsigned q = q0 + static_cast<unsigned>(k);
            mbar_wait(bar + q % kSlots, (q / kSlots) & 1u);
        };
        // The ring's previous contents were last read before this point
        // (same warp); order those generic reads before the TMA writes.
        fence_proxy_async_smem();
        __syncwarp();
        const int kfirst = min(kmax, kSlots - 1);
        if (lane == 0) {
            for (int k = 0; k <= kfirst; ++k) issue(k);
        }
        int kissued = kfirst;

        // Counts are kept as keys count << kb_ | (G-1 - b mod G), G = 2^kb_ bins,
        // so within a group of G bins the largest key is the lowest-index
        // maximum and a rescan is a plain packed max.
        // (16-byte stores: one bin row is 64 bytes, 4 lanes per row)
        for (int q = lane; q < bins * 4; q += 32) {
            const std::uint32_t v = gmask - ((q >> 2) & gmask);
            const std::uint32_t v2 = v | (v << 16);
            reinterpret_cast<uint4*>(cnt)[q] = make_uint4(v2, v2, v2, v2);
        }
        // (the first chunks were requested above: their flight covers the reset)
        for (int k = 0; k <= min(K0, kmax); ++k) wait(k);
        int kwaited = min(K0, kmax);
        __syncwarp();
        // Fast path: the first windows of all lanes lie in ring columns
        // [0, 2r] x rows [0, 32 + 2r); when that block is one colour (flat
        // content, config 3) every lane's window is (2r+1)^2 copies of it.
        // Striped starts (an edge through the first windows, no corner): when
        // every column of the block equals column 0 (horizontal stripes) or
        // every column is one colour down the block's rows (vertical stripes)
        // a window is 2r + 1 representative pixels taken 2r + 1 times each.
        const std::uint32_t* const col0 = ringp(0) - lane;  // row 0 of column 0
        const std::uint32_t e0 = col0[0];
        bool uni = true, rows_eq = true, cols_eq = true;
        {
            const bool two = lane < 2 * r;
            const std::uint32_t f0 = col0[lane], f1 = two ? col0[lane + 32] : 0u;
            const std::uint32_t* cb = col0;
            for (int c = 0; c < w2; ++c) {
                const std::uint32_t top = cb[0];
                const std::uint32_t v0 = cb[lane], v1 = two ? cb[lane + 32] : top;
                uni &= v0 == e0 && v1 == e0;
                rows_eq &= v0 == f0 && (!two || v1 == f1);
                cols_eq &= v0 == top && v1 == top;
                cb += RR;
                if (cb >= ring_end) cb -= kRingCols * RR;
            }
        }
        const bool flat0 = __all_sync(FULL, uni);
        const int stripes = flat0 || !OPC_SLIDE_STRIPED_START ? 0
                            : __all_sync(FULL, rows_eq)       ? 1
                            : __all_sync(FULL, cols_eq)       ? 2
                                                              : 0;
        // representative pixel i of a striped start: row lane + i of column 0
        // (horizontal stripes) or row 0 of column i (vertical stripes)
        auto stripe_px = [&](const int i) {
            if (stripes == 1) return col0[lane + i];
            const std::uint32_t* cb = col0 + i * RR;
            if (cb >= ring_end) cb -= kRingCols * RR;
            return cb[0];
        };
        if (flat0) {
            const int b0 = static_cast<int>(bin_of(e0, bm));
            cnt[b0 * 32 + lane] = static_cast<std::uint16_t>(cnt[b0 * 32 + lane] + w2 * w2 * inc);
            tally(kOpUpdates, 1);
        } else if (stripes) {
            tally(kOpUpdates, static_cast<unsigned long long>(w2));
            std::uint32_t* const cw32 = reinterpret_cast<std::uint32_t*>(cnt) + (lane >> 1);
            const unsigned add = (static_cast<unsigned>(w2) * inc) << ((lane & 1) * 16);
#pragma unroll 7
            for (int i = 0; i < w2; ++i) atomicAdd(cw32 + bin_of(stripe_px(i), bm) * 16, add);
            __syncwarp();
        } else {
            // (shared-memory atomics on the word holding this lane's u16 count:
            // no read-modify-write chain through the counts)
            // A column whose rows form at most two runs of one bin in every
            // lane's window (an edge or a corner in the block) is two weighted
            // updates; other columns update row by row.
            std::uint32_t* const cw32 = reinterpret_cast<std::uint32_t*>(cnt) + (lane >> 1);
            const unsigned add = inc << ((lane & 1) * 16);
            const std::uint32_t* col = ringp(0);
            for (int c = 0; c < w2; ++c) {
                const std::uint32_t bfirst = bin_of(col[0], bm);
                std::uint32_t bprev = bfirst;
                int ncp = 0, split = 0;
#pragma unroll 5
                for (int k = 1; k < w2; ++k) {
                    const std::uint32_t b = bin_of(col[k], bm);
                    const bool cp = b != bprev;
                    ncp += cp ? 1 : 0;
                    split = cp ? k : split;
                    bprev = b;
                }
                if (__all_sync(FULL, ncp <= 1)) {
                    const unsigned n1 = static_cast<unsigned>(ncp ? split : w2);
                    tally(kOpUpdates, ncp ? 2 : 1);
                    atomicAdd(cw32 + bfirst * 16, n1 * add);
                    if (__any_sync(FULL, ncp != 0)) atomicAdd(cw32 + bprev * 16, (static_cast<unsigned>(w2) - n1) * add);
                } else {
                    tally(kOpUpdates, static_cast<unsigned long long>(w2));
#pragma unroll 7
                    for (int k = 0; k < w2; ++k) atomicAdd(cw32 + bin_of(col[k], bm) * 16, add);
                }
                col += RR;
                if (col >= ring_end + lane) col -= kRingCols * RR;
            }
            __syncwarp();
        }
        // Full scan for the lowest-index maximum (filter.hpp:71-82), all lanes
        // together: lanes 2k and 2k+1 read the 32-bit words holding both their
        // counts of one bin, the even lane the even bins, the odd lane the odd
        // ones, and swap halves at the end of each group -- half the loads and
        // one packed max per word.  Groups are combined lowest first, strict >.
        // The rescan also returns U, the largest count of any other bin (the
        // top two keys per lane half, packed u16x2 min/max): a later step
        // whose winner lost pixels keeps it without a rescan while its count
        // stays above U (U grows with the other bins' increments).
        auto rescan = [&](int& best, int& bc, int& ub) {
            tally(kOpBinsExamined, static_cast<unsigned long long>(bins));
            if (lane == 0) tally(kOpRescans, 1);
            const std::uint32_t* cw = reinterpret_cast<const std::uint32_t*>(cnt) + (lane >> 1);
            const unsigned sh = (lane & 1) * 16;
            best = 0;
            bc = -1;
            ub = 0;
            for (int g0 = 0; g0 < bins; g0 += gsize) {
                const int gend = min(bins, g0 + gsize);
                std::uint32_t m = 0, m2 = 0;
#pragma unroll kUnrollScan
                for (int b = g0 + (lane & 1); b < gend; b += 2) {
                    const std::uint32_t v = cw[b * 16];
                    m2 = __vmaxu2(m2, __vminu2(m, v));
                    m = __vmaxu2(m, v);
                }
                const std::uint32_t o = __shfl_xor_sync(FULL, m, 1);
                const std::uint32_t o2 = __shfl_xor_sync(FULL, m2, 1);
                const std::uint32_t k1 = (m >> sh) & 0xFFFFu, k1o = (o >> sh) & 0xFFFFu;
                const std::uint32_t key = max(k1, k1o);
                const std::uint32_t key2 = max(min(k1, k1o), max((m2 >> sh) & 0xFFFFu, (o2 >> sh) & 0xFFFFu));
                const int c = static_cast<int>(key >> kb_);
                const int c2 = static_cast<int>(key2 >> kb_);
                if (c > bc) {
                    ub = max(ub, max(bc, c2));
                    bc = c;
                    best = g0 + static_cast<int>(gmask - (key & gmask));
                } else {
                    ub = max(ub, c);
                }
            }
        };
        int best, bc, ub;  // winner, its count, an upper bound of every other bin's count
        std::uint32_t sr, sg, sb;
        // The window sums (sr, sg, sb) of the lanes in `todo`, each for its own
        // bin `best`, the windows at pass column xw (ring columns xw .. xw + 2r).
        auto resum = [&](const int xw, unsigned todo) {
#if OPC_SLIDE_ROW_SUMS
        // Several lanes with one new winner (an edge crossing the
        // band): their windows are rows t .. t + 2r of the same 2r + 1
        // columns, so the warp sums that bin once per ring row (lane t:
        // rows t and 32 + t) and every lane takes the difference of
        // two prefix sums over the rows -- 2(2r + 1) loads per lane
        // instead of (2r + 1)^2.  R, G, B travel as 21-bit fields of
        // one 64-bit word (a prefix is at most 62 rows x 31 x 255).
        // (every bin that four or more of the lanes share; lanes with rarer
        // bins are left for the per-lane forms below)
        unsigned big = 0;  // lanes of `todo` whose bin four or more of them share
        if (__popc(todo) >= OPC_SLIDE_PAR_SUMS) {
            const bool mine = ((todo >> lane) & 1u) != 0u;
            const unsigned same = __match_any_sync(FULL, mine ? best : -1 - lane);
            big = __ballot_sync(FULL, mine && __popc(same) >= OPC_SLIDE_PAR_SUMS);
        }
        todo &= ~big;
        while (big) {
            const int bj = __shfl_sync(FULL, best, __ffs(big) - 1);
            const unsigned grp = __ballot_sync(FULL, ((big >> lane) & 1u) != 0u && best == bj);
            std::uint32_t rb0 = 0, g0 = 0, rb1 = 0, g1 = 0;
            const std::uint32_t* colb = ringp(xw) - lane;  // row 0 of column x
            const bool two = lane < 2 * r;
            tally(kOpSumPixels, static_cast<unsigned long long>(two ? 2 * w2 : w2));
#pragma unroll 3
            for (int c = 0; c < w2; ++c) {
                const std::uint32_t e0 = colb[lane];
                const std::uint32_t e1 = two ? colb[lane + 32] : 0u;
                const std::uint32_t a0 = static_cast<int>(bin_of(e0, bm)) == bj ? e0 : 0u;
                const std::uint32_t a1 = (two && static_cast<int>(bin_of(e1, bm)) == bj) ? e1 : 0u;
                rb0 += a0 & 0x00FF00FFu;
                g0 += a0 & 0x0000FF00u;
                rb1 += a1 & 0x00FF00FFu;
                g1 += a1 & 0x0000FF00u;
                colb += RR;
                if (colb >= ring_end) colb -= kRingCols * RR;
            }
            auto pack = [](std::uint32_t rb, std::uint32_t g) {
                return static_cast<unsigned long long>(rb & 0xFFFFu) |
                       (static_cast<unsigned long long>(g >> 8) << 21) |
                       (static_cast<unsigned long long>(rb >> 16) << 42);
            };
            const unsigned long long v0 = pack(rb0, g0), v1 = pack(rb1, g1);
            unsigned long long s0 = v0, s1 = v1;  // inclusive scans over the lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long u0 = __shfl_up_sync(FULL, s0, o);
                const unsigned long long u1 = __shfl_up_sync(FULL, s1, o);
                if (lane >= o) {
                    s0 += u0;
                    s1 += u1;
                }
            }
            // window of lane t = rows [t, t + 2r]: prefix(t + 2r + 1) - prefix(t)
            const unsigned long long t0 = __shfl_sync(FULL, s0, 31);
            const int jj = lane + w2;
            const unsigned long long pa = __shfl_sync(FULL, s0, (jj - 1) & 31);
            const unsigned long long pb = __shfl_sync(FULL, s1, (jj - 33) & 31);
            const unsigned long long ws = (jj <= 32 ? pa : t0 + pb) - (s0 - v0);
            if ((grp >> lane) & 1u) {
                sr = static_cast<std::uint32_t>(ws) & 0x1FFFFFu;
                sg = static_cast<std::uint32_t>(ws >> 21) & 0x1FFFFFu;
                sb = static_cast<std::uint32_t>(ws >> 42);
            }
            big &= ~grp;
        }
#endif
        const bool own = __popc(todo) >= OPC_SLIDE_PAR_SUMS;
        if (own) {
            // many lanes with different new winners: each sums its own
            // window, in parallel
            if ((todo >> lane) & 1u) {
                tally(kOpSumPixels, static_cast<unsigned long long>(w2) * w2);
                std::uint32_t cr = 0, cg = 0, cbb = 0;
                for (int c = 0; c < w2; ++c) {
                    const std::uint32_t* col = ringp(xw + c);
#pragma unroll kUnrollSums
                    for (int k = 0; k < w2; ++k) {
                        const std::uint32_t e = col[k];
                        if (static_cast<int>(bin_of(e, bm)) == best) {
                            cr += e & 0xFFu;
                            cg += (e >> 8) & 0xFFu;
                            cbb += (e >> 16) & 0xFFu;
                        }
                    }
                }
                sr = cr;
                sg = cg;
                sb = cbb;
            }
            todo = 0u;
        }
        for (; todo; todo &= todo - 1) {
            const int j = __ffs(todo) - 1;
            const int bj = __shfl_sync(FULL, best, j);
            std::uint32_t cr = 0, cg = 0, cbb = 0;
            if (lane < w2) {
                tally(kOpSumPixels, static_cast<unsigned long long>(w2));
                const std::uint32_t* col = ringp(xw + lane) - lane + j;
#pragma unroll kUnrollChange
                for (int k = 0; k < w2; ++k) {
                    const std::uint32_t e = col[k];
                    if (static_cast<int>(bin_of(e, bm)) == bj) {
                        cr += e & 0xFFu;
                        cg += (e >> 8) & 0xFFu;
                        cbb += (e >> 16) & 0xFFu;
                    }
                }
            }
            cr = __reduce_add_sync(FULL, cr);
            cg = __reduce_add_sync(FULL, cg);
            cbb = __reduce_add_sync(FULL, cbb);
            if (lane == j) {
                sr = cr;
                sg = cg;
                sb = cbb;
            }
        }
        };
        if (flat0) {
            const std::uint32_t n0 = static_cast<std::uint32_t>(w2 * w2);
            best = static_cast<int>(bin_of(e0, bm));
            bc = w2 * w2;
            ub = 0;
            sr = n0 * (e0 & 0xFFu);
            sg = n0 * ((e0 >> 8) & 0xFFu);
            sb = n0 * ((e0 >> 16) & 0xFFu);
        } else if (stripes) {
            rescan(best, bc, ub);
            tally(kOpSumPixels, static_cast<unsigned long long>(w2));
            sr = sg = sb = 0;
#pragma unroll 7
            for (int i = 0; i < w2; ++i) {
                const std::uint32_t e = stripe_px(i);
                if (static_cast<int>(bin_of(e, bm)) == best) {
                    sr += e & 0xFFu;
                    sg += (e >> 8) & 0xFFu;
                    sb += (e >> 16) & 0xFFu;
                }
            }
            sr *= static_cast<std::uint32_t>(w2);
            sg *= static_cast<std::uint32_t>(w2);
            sb *= static_cast<std::uint32_t>(w2);
        } else {
            rescan(best, bc, ub);
            sr = sg = sb = 0;
            resum(0, FULL);
        }
        // the output of the current window (recomputed only after a step
        // that changed the window: a flat step repeats the previous pixel)
        auto quotient = [&]() {
            const std::uint32_t m = recip[bc];
            return __umulhi(sr << 1, m) | (__umulhi(sg << 1, m) << 8) | (__umulhi(sb << 1, m) << 16);
        };
        std::uint32_t rgb = quotient();
        SEC_ADD(0, t_pass);

        // entering column x + 2r and leaving column x - 1 of step x, as ring
        // pointers advanced by one column per step (the leaving pointer wraps)
        const std::uint32_t* cin = ringp(2 * r);
        const std::uint32_t* cout = ringp(kRingCols - 1);  // column -1 (unused at x = 0)
        // nonflat bits of this band (work plan): bit x of word j = the step at
        // interior column 32 j + x changes the window
        const std::uint32_t* nfb = tg.nf + (static_cast<std::size_t>(f) * tg.nbands + kb) * tg.nblk;
        int flat_from = xs;  // image column from which every output so far equals rgb
        // A block of 16 columns of one colour (a flat run covering a whole
        // output block): every row of the out tile is the 3-word pattern of
        // rgb repeated -- packed from the register, no staging.
        auto flush_flat = [&](const int xb) {
            if (lane == 0) bulk_wait_read0();  // the previous store has read the tile
            __syncwarp();
            const std::uint32_t w0 = rgb | (rgb << 24), w1 = (rgb >> 8) | (rgb << 16),
                                w2_ = (rgb >> 16) | (rgb << 8);
            uint4* orow = reinterpret_cast<uint4*>(otile + lane * 48);
            orow[0] = make_uint4(w0, w1, w2_, w0);
            orow[1] = make_uint4(w1, w2_, w0, w1);
            orow[2] = make_uint4(w2_, w0, w1, w2_);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
                tma_store_3d(&tout, otile, 3 * xb, yb - a.out_row0, f);
                bulk_commit();
            }
            __syncwarp();
        };
        // Flush of the output block holding image column xa, its last
        // staged column (x = the pass column of xa).  Output blocks are 16
        // image columns [16m, 16m + 15] (a TMA store box must start 16-byte
        // aligned: 48m bytes); the partial blocks at the ends of a pass are
        // written with byte stores.
        auto flush = [&](const int xa) {
            const int xb = xa & ~(kStageCols - 1);      // image column of stage column 0
            if (TMA_OUT && xa - xb == kStageCols - 1 && flat_from <= xb && xb >= xs) {
                flush_flat(xb);  // no step changed the window since the block began
                return;
            }
            __syncwarp();
            const int c_lo = max(xs, xb) - xb;          // valid stage columns [c_lo, c_hi]
            const int c_hi = xa - xb;
            if (TMA_OUT && c_lo == 0 && c_hi == kStageCols - 1) {
                // lane t packs row t's 16 pixels into 48 bytes of the out
                // tile; one TMA store writes the 32 x 48-byte box (rows
                // past the band end are clipped by the tensor map)
                if (lane == 0) bulk_wait_read0();  // the previous store has read the tile
                __syncwarp();
                const std::uint32_t* srow = stage + lane * kStageStride;
                std::uint32_t wv[12];
#pragma unroll
                for (int j = 0; j < 4; ++j) {  // pixels 4j .. 4j+3 -> words 3j .. 3j+2
                    const std::uint32_t p0 = srow[4 * j], p1 = srow[4 * j + 1],
                                        p2 = srow[4 * j + 2], p3 = srow[4 * j + 3];
                    wv[3 * j] = p0 | (p1 << 24);
                    wv[3 * j + 1] = (p1 >> 8) | (p2 << 16);
                    wv[3 * j + 2] = (p2 >> 16) | (p3 << 8);
                }
                uint4* orow = reinterpret_cast<uint4*>(otile + lane * 48);
                orow[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                orow[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
                orow[2] = make_uint4(wv[8], wv[9], wv[10], wv[11]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&tout, otile, 3 * xb, yb - a.out_row0, f);
                    bulk_commit();
                }
            } else {
                const int c = lane & (kStageCols - 1);
                for (int f0 = 0; f0 < 32; f0 += 32 / kStageCols) {  // 2 rows per store
                    const int fr = f0 + lane / kStageCols;
                    if (yb + f0 >= a.y_hi) break;
                    if (c >= c_lo && c <= c_hi && yb + fr < a.y_hi) {
                        const std::uint32_t v = stage[fr * kStageStride + c];
                        std::uint8_t* o = out +
                                          static_cast<std::size_t>(yb + fr - a.out_row0) * stride +
                                          static_cast<std::size_t>(xb + c) * 3;
                        o[0] = static_cast<std::uint8_t>(v);
                        o[1] = static_cast<std::uint8_t>(v >> 8);
                        o[2] = static_cast<std::uint8_t>(v >> 16);
                    }
                }
            }
            __syncwarp();
        };
        // Columns xf .. xf + cnt - 1 of the pass, all equal to rgb (flat steps).
        auto emit_flat = [&](const int xf, const int cnt) {
            tally(kOpSteps, static_cast<unsigned long long>(cnt - (xf == 0 ? 1 : 0)));
            if (row_ok) tally(kOpPixels, static_cast<unsigned long long>(cnt));
            for (int done = 0; done < cnt;) {
                const int xa = xs + xf + done;
                const int c0 = xa & (kStageCols - 1);
                const int seg = min(cnt - done, kStageCols - c0);
                if (TMA_OUT && seg == kStageCols) {
                    flush_flat(xa);
                } else {
                    std::uint32_t* sp = stage + lane * kStageStride + c0;
#pragma unroll
                    for (int i = 0; i < kStageCols; ++i) {
                        if (i < seg) sp[i] = rgb;
                    }
                    if (c0 + seg == kStageCols || xf + done + seg == n) flush(xa + seg - 1);
                }
                done += seg;
            }
        };
        // (the words of the next phase are loaded a phase ahead: an L2 round
        // trip per 16 columns would otherwise be most of a flat phase)
        std::uint32_t nf_lo, nf_hi;
        auto nf_load = [&](const int p) {
            const int j = (x0 + kStageCols * p) >> 5;
            nf_lo = j < tg.nblk ? __ldg(nfb + j) : 0u;
            nf_hi = j + 1 < tg.nblk ? __ldg(nfb + j + 1) : 0u;
        };
        nf_load(0);
        for (int p = 0; kStageCols * p < n; ++p) {
            // bit i: the step at pass column 16p + i is not flat
            const std::uint32_t nfm = __funnelshift_r(nf_lo, nf_hi, (x0 + kStageCols * p) & 31);
            nf_load(p + 1);
#if OPC_SLIDE_JUMP
            // Flat stretches: flat steps read no pixels, so the ring need not
            // follow them.  When this phase and the next hold no window-
            // changing step, look for the next one (one coalesced load of the
            // coming 32 nonflat words); if it is kJumpMin phases or more away,
            // emit the stretch at once and restart the ring at that step's
            // phase (the counts, the winner and its sums are unchanged).
            if (OPC_SLIDE_PLAN && p > 0 && nfm == 0u && kStageCols * (p + kJumpMin) < n + kStageCols) {
                const int xi = x0 + kStageCols * p;
                const int j = xi >> 5, jl = (x0 + n - 1) >> 5;
                std::uint32_t w = j + lane <= jl ? __ldg(nfb + j + lane) : 0u;
                if (lane == 0) w &= 0xFFFFFFFFu << (xi & 31);
                const unsigned any = __ballot_sync(FULL, w != 0u);
                int xn;  // pass column of the next window-changing step (or past the words looked at)
                if (any) {
                    const int l = __ffs(any) - 1;
                    xn = 32 * (j + l) + __ffs(__shfl_sync(FULL, w, l)) - 1 - x0;
                } else {
                    xn = 32 * (j + 32) - x0;
                }
                const int p2 = xn >= n ? (n + kStageCols - 1) / kStageCols : xn / kStageCols;
                if (p2 - p >= kJumpMin) {
                    [[maybe_unused]] const long long t_j = SEC_NOW();
                    if (kStageCols * p2 >= n) {
                        emit_flat(kStageCols * p, n - kStageCols * p);
                        SEC_ADD(6, t_j);
                        break;  // the pass ends flat
                    }
                    // (the ring is restarted first: its loads fly while the
                    // stretch is emitted, which touches no ring column)
                    // every chunk in flight lands before the ring is re-based
                    for (int k = kwaited + 1; k <= kissued; ++k) wait(k);
                    // chunk p2 (the column step 16 p2 removes) takes the next
                    // slot in issue order: q0 + p2 = the next q, up to a multiple
                    // of 2 kSlots (slot and parity of a q repeat with that period)
                    const unsigned qn = q0 + static_cast<unsigned>(kissued + 1);
                    const unsigned per = 2u * kSlots;
                    q0 = qn + (static_cast<unsigned>(p2) + per - 1) / per * per - static_cast<unsigned>(p2);
                    pos0 = kChunk * static_cast<int>(q0 % kSlots) - B;
                    fence_proxy_async_smem();
                    __syncwarp();
                    // (chunks p2 .. p2 + kSlots - 2: phase p2 requests the next one itself)
                    kissued = min(kmax, p2 + kSlots - 2);
                    if (lane == 0) {
                        for (int k = p2; k <= kissued; ++k) issue(k);
                    }
                    emit_flat(kStageCols * p, kStageCols * (p2 - p));
                    kwaited = min(kmax, p2 + K0);
                    for (int k = p2; k <= kwaited; ++k) wait(k);
                    cin = ringp(kStageCols * p2 + 2 * r);
                    cout = ringp(kStageCols * p2 - 1);
                    p = p2 - 1;
                    nf_load(p2);
                    SEC_ADD(6, t_j);
                    continue;
                }
            }
#endif
            [[maybe_unused]] const long long t_top = SEC_NOW();
            if (p > 0) {
                // phase p enters chunk p + K0; the slot of chunk p - 1 is free:
                // request chunk p + kSlots - 1
                if (p + K0 > kwaited) {
                    wait(p + K0);
                    kwaited = p + K0;
                }
                if (p + kSlots - 1 <= kmax) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) issue(p + kSlots - 1);
                    kissued = p + kSlots - 1;
                }
            }
            SEC_ADD(8, t_top);
            const int xend = min(n, kStageCols * p + kStageCols);
            int x = kStageCols * p;
            while (x < xend) {
                // Flat steps ahead of x (the work plan's nonflat bits; step 0
                // of a pass is no step): their outputs repeat rgb, so the run
                // is emitted at once -- stage stores per 16-column output
                // block, no per-step loop.
                int run;
                if (OPC_SLIDE_PLAN) {
                    std::uint32_t bits = nfm >> (x - kStageCols * p);
                    if (x == 0) bits &= ~1u;
                    run = min(bits ? __ffs(bits) - 1 : 32, xend - x);
                } else {
                    bool diff = false;
                    if (x > 0) {
                        const std::uint32_t* cinb = cin - lane;
                        const std::uint32_t* coutb = cout - lane;
                        diff = cinb[lane] != coutb[lane];
                        if (lane < 2 * r) diff |= cinb[lane + 32] != coutb[lane + 32];
                    }
                    run = __any_sync(FULL, diff) ? 0 : 1;
                }
                if (run > 0) {
                    [[maybe_unused]] const long long t_f = SEC_NOW();
                    emit_flat(x, run);
                    SEC_ADD(5, t_f);
                    cin += run * RR;
                    cout += run * RR;
                    if (cout >= ring_end) cout -= kRingCols * RR;
                    if (cin >= ring_end) cin -= kRingCols * RR;
                    x += run;
                    continue;
                }
                // A step that changes the window (x > 0).
                [[maybe_unused]] const long long t_s1 = SEC_NOW();
                // Slide: add ring column x + 2r (image x + r), remove x - 1 (image x - r - 1).
                tally(kOpSteps, 1);
                {
                if (lane == 0) tally(kOpNonFlatSteps, 1);
                const int best0 = best;
                int cand_c = -1;  // the largest post-increment count of another bin
                // Branch-free form: every row pays two count updates (of
                // zero when the pixel does not change bin), so lanes whose
                // changes sit at different rows do not diverge.
                // (atomics: the two updates of a row are shared-memory
                // atomics on the 32-bit word holding this lane's u16 count,
                // so the rows' updates are in flight together instead of
                // one read-modify-write chain; same-address atomics of a
                // thread apply in order, and a count never drops below
                // its key, so no borrow crosses into the other lane's half)
                std::uint32_t* const cw32 = reinterpret_cast<std::uint32_t*>(cnt) + (lane >> 1);
                const unsigned csh = (lane & 1) * 16;
#if OPC_SLIDE_PACKED_SUMS
                // The winner's channel sums change by the masked entering
                // minus leaving pixels.  They are accumulated packed: the
                // whole 24-bit words in one accumulator (one add per row) and
                // G alone in a second (two dot products per row); every
                // channel total is within +-31 * 255, so the packed total
                // decodes exactly after the loop.
                //
                // Count updates: a shared-memory atomic costs ~2 cycles per
                // lane, so 2(2r+1) of them are most of a step.  The rows of a
                // step are first walked without touching the counts (bins,
                // sums, and the rows where the (entering, leaving) bin pair
                // changes); when every lane sees at most one such change --
                // an edge that crosses the window's rows, with at most one
                // corner or horizontal edge in them -- the step is two
                // weighted updates per lane (rows above / below the change)
                // instead of one per row.  Other steps update row by row.
                const unsigned incs = inc << csh;
                // (32-bit shared-window addresses: one multiply-add per
                // count word instead of a 64-bit generic address)
                const std::uint32_t cw_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(cw32));
                const std::uint32_t half = csh ? 0x4432u : 0x4410u;  // PRMT: this lane's u16 half
                std::uint32_t dall = 0;  // R + 256 G + 65536 B differences, summed
                std::int32_t dg = 0;     // the G differences alone
                std::uint32_t cand_k = 0;  // largest post-increment key of another bin
                auto move = [&](const std::uint32_t bi, const std::uint32_t bo, const unsigned d) {
                    std::uint32_t old;
                    asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                                 : "=r"(old)
                                 : "r"(cw_s + bi * 64u), "r"(d)
                                 : "memory");
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cw_s + bo * 64u), "r"(0u - d)
                                 : "memory");
                    // this lane's key of bin bi after the update (a count
                    // never overflows its half -- the pixels leaving are in
                    // other bins -- so there is no carry to drop; keys order
                    // like their counts).  A bin whose count did not move
                    // (d = 0) is already bounded by ub, so it may join the
                    // candidates; so may a count a later update lowers again.
                    const std::uint32_t key = __byte_perm(old + d, 0u, half);
                    cand_k = max(cand_k, bi != static_cast<std::uint32_t>(best0) ? key : 0u);
                };
                std::uint32_t pair0 = 0, prev = 0;  // bi | bo << 16 of row 0 / of the previous row
                int ncp = 0, split = 0;             // rows k >= 1 whose pair differs from row k - 1; the last one
#pragma unroll kUnrollUpdate
                for (int k = 0; k < w2; ++k) {
                    const std::uint32_t ei = cin[k], eo = cout[k];
                    const std::uint32_t bi = bin_of(ei, bm), bo = bin_of(eo, bm);
                    const std::uint32_t pair = bi | (bo << 16);
                    if (k == 0) pair0 = pair;
                    const bool cp = k > 0 && pair != prev;
                    ncp += cp ? 1 : 0;
                    split = cp ? k : split;
                    prev = pair;
                    const std::uint32_t a = bi == static_cast<std::uint32_t>(best0) ? ei : 0u;
                    const std::uint32_t b = bo == static_cast<std::uint32_t>(best0) ? eo : 0u;
                    dall += a - b;                     // (plane words: top byte 0)
                    dg = dp4a_us(a, 0x00000100u, dg);  // + G(a)
                    dg = dp4a_us(b, 0x0000FF00u, dg);  // - G(b): byte 1 of the multiplier = -1
                }
                SEC_ADD(1, t_s1);
                [[maybe_unused]] const long long t_s2 = SEC_NOW();
                if (OPC_SLIDE_RUNS && __all_sync(FULL, ncp <= 1)) {
                    const int n1 = ncp ? split : w2;  // rows of the first run
                    tally(kOpUpdates, ncp ? 4 : 2);
                    {
                        const std::uint32_t bi = pair0 & 0xFFFFu, bo = pair0 >> 16;
                        move(bi, bo, bi != bo ? static_cast<unsigned>(n1) * incs : 0u);
                    }
                    if (__any_sync(FULL, ncp != 0)) {
                        const std::uint32_t bi = prev & 0xFFFFu, bo = prev >> 16;
                        move(bi, bo, bi != bo ? static_cast<unsigned>(w2 - n1) * incs : 0u);
                    }
                } else {
                    // Branch-free form: every row pays two count updates (of
                    // zero when the pixel does not change bin), so lanes whose
                    // changes sit at different rows do not diverge.
                    tally(kOpUpdates, 2ull * w2);
#pragma unroll kUnrollUpdate
                    for (int k = 0; k < w2; ++k) {
                        const std::uint32_t bi = bin_of(cin[k], bm), bo = bin_of(cout[k], bm);
                        move(bi, bo, bi != bo ? incs : 0u);
                    }
                }
                SEC_ADD(2, t_s2);
                [[maybe_unused]] const long long t_s3 = SEC_NOW();
                cand_c = static_cast<int>(cand_k >> kb_);  // (0 when no other bin was touched: ub >= 0)
                {
                    // dall - 256 dg = dR + 65536 dB with |dR|, |dB| <= 31 * 255:
                    // dR is the sign-extended low half, dB what is left.
                    const std::uint32_t drb = dall - (static_cast<std::uint32_t>(dg) << 8);
                    const std::int32_t dr = static_cast<std::int16_t>(drb & 0xFFFFu);
                    sr += static_cast<std::uint32_t>(dr);
                    sb += static_cast<std::uint32_t>(
                        static_cast<std::int32_t>(drb - static_cast<std::uint32_t>(dr)) >> 16);
                    sg += static_cast<std::uint32_t>(dg);
                }
#else
                for (int k = 0; k < w2; ++k) {
                    const std::uint32_t ei = cin[k], eo = cout[k];
                    const int bi = bin_of(ei, bm), bo = bin_of(eo, bm);
                    const bool mv = bi != bo;
                    const unsigned d = mv ? inc : 0u;
                    unsigned ki;
                    if (OPC_SLIDE_ATOMICS) {
                        const unsigned old = atomicAdd(cw32 + bi * 16, d << csh);
                        atomicSub(cw32 + bo * 16, d << csh);
                        ki = ((old >> csh) & 0xFFFFu) + d;
                    } else {
                        ki = cnt[bi * 32 + lane] + d;
                        cnt[bi * 32 + lane] = static_cast<std::uint16_t>(ki);
                        cnt[bo * 32 + lane] = static_cast<std::uint16_t>(cnt[bo * 32 + lane] - d);
                    }
                    const int ci = static_cast<int>(ki >> kb_);
                    cand_c = (mv && bi != best0) ? max(cand_c, ci) : cand_c;
                    const std::uint32_t mi = bi == best0 ? 0xFFFFFFFFu : 0u;
                    const std::uint32_t mo = bo == best0 ? 0xFFFFFFFFu : 0u;
                    sr += (ei & mi & 0xFFu) - (eo & mo & 0xFFu);
                    sg += ((ei & mi) >> 8 & 0xFFu) - ((eo & mo) >> 8 & 0xFFu);
                    sb += ((ei & mi) >> 16 & 0xFFu) - ((eo & mo) >> 16 & 0xFFu);
                }
#endif
                // Resolve the winner (filter.hpp:71-82): it stays while its
                // count is above every other bin's (bounded by ub);
                // otherwise a rescan finds the lowest-index maximum.
                ub = max(ub, cand_c);
                const int bcf = cnt[best0 * 32 + lane] >> kb_;
                bool changed = false;
                const bool need = bcf <= ub;
                if (!need) bc = bcf;
                if (__any_sync(FULL, need)) {
                    int nb, nc, nu;
                    rescan(nb, nc, nu);
                    if (need) {
                        best = nb;
                        bc = nc;
                        ub = nu;
                        changed = best != best0;
                    }
                }
                if (changed) tally(kOpWinnerChanges, 1);
                // Winner changed: the new winner's window sums, one lane's
                // window at a time with lane c < 2r+1 summing its column c
                // (2r+1 loads per lane instead of (2r+1)^2 on one lane
                // while the others wait).
                SEC_ADD(3, t_s3);
                [[maybe_unused]] const long long t_s4 = SEC_NOW();
                const unsigned chg = __ballot_sync(FULL, changed);
                resum(x, chg);
                rgb = quotient();
                SEC_ADD(4, t_s4);
                }
                [[maybe_unused]] const long long t_s7 = SEC_NOW();
                if (row_ok) tally(kOpPixels, 1);
                {
                    const int xa = xs + x;
                    flat_from = xa;
                    stage[lane * kStageStride + (xa & (kStageCols - 1))] = rgb;
                    if ((xa & (kStageCols - 1)) == kStageCols - 1 || x == n - 1) flush(xa);
                }
                cin += RR;
                cout += RR;
                if (cout >= ring_end) cout -= kRingCols * RR;
                if (cin >= ring_end) cin -= kRingCols * RR;
                SEC_ADD(7, t_s7);
                ++x;
            }
        }
        // chunks requested but not consumed: wait, so no TMA write lands in
        // the next pass's ring and the slot parities stay in step
        for (int k = kwaited + 1; k <= kissued; ++k) wait(k);
        q0 += static_cast<unsigned>(kissued + 1);
        __syncwarp();
    }
    if constexpr (TMA_OUT) {
        if (lane == 0) bulk_wait0();
    }
#if OPC_SLIDE_TRACE
    if (lane == 0) {
        for (int k = 0; k < 16; ++k) {
            if (sec_acc[k]) atomicAdd(g_sec + k, static_cast<unsigned long long>(sec_acc[k]));
        }
    }
#endif
    if constexpr (COUNT) {
#pragma unroll
        for (int k = 0; k < kOpCountN; ++k) {
            unsigned long long v = opc_n[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
            if (lane == 0 && v) atomicAdd(a.op_counts + k, v);
        }
    }
}

}  // namespace

bool slide_supported(int levels, int radius) {
    return levels >= 1 && levels <= 256 && radius >= 0 && radius <= 15 &&
           bin_multiplier(levels) != 0 &&
           kRecipBytes + per_warp_bytes(levels + 1, radius) <= 227 * 1024;
}

std::size_t slide_scratch_bytes(const BandArgs& a) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo) return 0;
    return tgeom_bytes(a);
}

cudaError_t launch_slide(const BandArgs& a, int* counter, void* scratch, int num_sms,
                         cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    const int bins = a.levels + 1;
    const std::size_t pw = per_warp_bytes(bins, a.radius);
    const std::size_t limit = 227 * 1024;
    int warps = kWarps;
    while (warps > 1 && kRecipBytes + warps * pw > limit) --warps;
    const std::size_t smem = kRecipBytes + warps * pw;

    const std::size_t row_bytes = static_cast<std::size_t>(a.width) * 3;
    bool tma_out = row_bytes % 16 == 0 && a.out_frame_stride % 16 == 0 &&
                   reinterpret_cast<std::uintptr_t>(a.out) % 16 == 0;
    const bool count = a.op_counts != nullptr;
    // (TMA_OUT decided below; both variants get their attributes set)
    const void* kfn_t = count ? reinterpret_cast<const void*>(slide_kernel<true, true>)
                              : reinterpret_cast<const void*>(slide_kernel<false, true>);
    const void* kfn_b = count ? reinterpret_cast<const void*>(slide_kernel<true, false>)
                              : reinterpret_cast<const void*>(slide_kernel<false, false>);
    cudaError_t e = set_smem_attr(kfn_t, static_cast<int>(smem));
    if (e == cudaSuccess) e = set_smem_attr(kfn_b, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = blocks_per_sm(kfn_t, warps * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const long long resident = static_cast<long long>(num_sms) * per_sm * warps;

    const TGeom tg = tgeom(a, scratch, resident);
    std::uint32_t* T = static_cast<std::uint32_t*>(scratch);
    // TMA maps: the transposed plane (rows, columns, frames) read in boxes of
    // ring_rows x 16 columns; the output (bytes of the interior columns, rows
    // up to the band's interior end, frames) written in 48-byte x 32-row boxes.
    CUtensorMap tin{}, tout{};
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(tg.Hs), static_cast<cuuint64_t>(tg.ncols),
                                    static_cast<cuuint64_t>(a.frames)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(tg.Hs) * 4,
                                       static_cast<cuuint64_t>(tg.frame_elems) * 4};
        const cuuint32_t box[3] = {static_cast<cuuint32_t>(ring_rows(a.radius)),
                                   static_cast<cuuint32_t>(kChunk), 1};
        if (encode_tensor_map(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, T, dims, strides, box) != 0) {
            return cudaErrorInvalidValue;
        }
    }
    if (tma_out) {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.x_hi) * 3,
                                    static_cast<cuuint64_t>(a.y_hi - a.out_row0),
                                    static_cast<cuuint64_t>(a.frames)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_bytes),
                                       static_cast<cuuint64_t>(a.out_frame_stride)};
        const cuuint32_t box[3] = {3 * kStageCols, 32, 1};
        tma_out = encode_tensor_map(&tout, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, a.out, dims, strides,
                                    box) == 0;
    }
    const void* kfn = tma_out ? kfn_t : kfn_b;

    // Pre-pass and work plan: the transposed plane with its column-change
    // masks (border job appended), the nonflat bits and block costs, the
    // equal-cost chunk starts.
    e = cudaMemsetAsync(counter, 0, 4 * sizeof(int), s);
    if (e != cudaSuccess) return e;
    timing_mark(kIdPrePass, 0, s);
    {
        const unsigned gx = static_cast<unsigned>((tg.ncols + kTCols - 1) / kTCols);
        const dim3 grid(gx, static_cast<unsigned>(tg.Hs / kTRows) + border_grid_rows(a, gx),
                        static_cast<unsigned>(a.frames));
        const int vec_ok = (reinterpret_cast<std::uintptr_t>(a.in) % 4 == 0) && (row_bytes % 4 == 0) &&
                           (a.in_frame_stride % 4 == 0);
        transpose_kernel<<<grid, 256, 0, s>>>(a, T, tg, vec_ok);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const long long nblocks = static_cast<long long>(a.frames) * tg.nbands * tg.ncb;  // cost blocks
    {
        const long long nq = (tg.nblk + kCostBlocksPerWarp - 1) / kCostBlocksPerWarp;
        const long long nwarps = static_cast<long long>(a.frames) * tg.nbands * nq;
        const long long ctas = (nwarps + kPlanThreads / 32 - 1) / (kPlanThreads / 32);
        // counter[1]: the plan kernel's done count (zeroed with the task
        // counter before the pre-pass)
        // block costs staged in shared memory by the last CTA when they fit
        const int cap = static_cast<int>(std::min<long long>(nblocks, kPlanSmemCap));
        const int bytes = (cap + cap / 16 + 1) * 4;  // (padded layout)
        e = set_smem_attr(reinterpret_cast<const void*>(slide_plan_kernel), bytes);
        if (e != cudaSuccess) return e;
        slide_plan_kernel<<<static_cast<unsigned>(ctas), kPlanThreads, bytes, s>>>(
            a, tg, nblocks, reinterpret_cast<unsigned*>(counter) + 1, cap);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    timing_mark(kIdPrePass, 1, s);
    const WorkSplit g =
        OPC_SLIDE_PLAN
            ? make_planned_split(a.frames, tg.nbands, a.x_hi - a.x_lo, tg.ncb, kCostCols, tg.nch, tg.cs)
            : make_split(a.frames, tg.nbands, a.x_hi - a.x_lo, resident, OPC_SLIDE_STATIC_PCT,
                         OPC_SLIDE_MIN_CHUNK, OPC_SLIDE_DYN_PER_WARP, OPC_SLIDE_GUIDED_K);
    long long blocks = (g.nchunks + warps - 1) / warps;
    if (blocks > static_cast<long long>(num_sms) * per_sm) blocks = num_sms * per_sm;
    if (blocks < 1) blocks = 1;
    timing_mark(kIdSlide, 0, s);
    const dim3 grid(static_cast<unsigned>(blocks)), block(warps * 32);
    // (through the function pointer: the four instantiations share the launcher)
    BandArgs aa = a;
    TGeom tgg = tg;
    WorkSplit gg = g;
    void* args[] = {&aa, &tgg, &counter, &gg, &tin, &tout};
    e = cudaLaunchKernel(kfn, grid, block, args, smem, s);
    timing_mark(kIdSlide, 1, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace opc

#if OPC_SLIDE_TRACE
extern "C" void opc_debug_slide_sections(unsigned long long* out16) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out16, opc::g_sec, 16 * sizeof(unsigned long long));
    const unsigned long long zero[16] = {};
    cudaMemcpyToSymbol(opc::g_sec, zero, sizeof(zero));
}
extern "C" int opc_debug_slide_trace(unsigned long long* out, int max) {
    int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, opc::g_trace_n, sizeof(int));
    n = n < max ? n : max;
    if (n > (1 << 16)) n = 1 << 16;
    cudaMemcpyFromSymbol(out, opc::g_trace, static_cast<std::size_t>(n) * 32);
    const int zero = 0;
    cudaMemcpyToSymbol(opc::g_trace_n, &zero, sizeof(int));
    return n;
}
#endif
