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
// Pixels come from a transposed (column-major) entry plane written by the
// shared pre-pass, so a ring column (32+2r rows) is one contiguous run that
// cp.async copies 16 bytes at a time, one phase (kPhase columns) ahead.
#include "kernels.cuh"
#include "border.cuh"
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
#ifndef OPC_SLIDE_STATIC_PCT
#define OPC_SLIDE_STATIC_PCT 50  // content-dependent step costs: 90 measured 20% slower on C3
#endif

constexpr int kWarps = 8;  // upper bound; the launcher fits as many as 227 KB allows
// Ring of entry columns: the window (2r+1) + the phase being slid + the phase
// being fetched + the leaving column, a compile-time size so the modulo stays
// cheap; the smaller rings for small radii fit more warps per SM (config 3,
// r = 10: 88 columns and 16-column output staging give 6 warps instead of 5).
#ifndef OPC_SLIDE_PHASE
#define OPC_SLIDE_PHASE 32  // 16 (64-column ring, 7 warps/SM on C3) measured 25% slower:
                            // a 16-column lead no longer hides the fetch latency on flat runs
#endif
constexpr int kPhase = OPC_SLIDE_PHASE;  // columns fetched / slid per phase
__host__ __device__ constexpr int ring_cols(int r) {
    return kPhase == 16 ? 64 : r <= 7 ? 80 : r <= 11 ? 88 : 96;  // >= 2r+1 + 2 kPhase + 1
}
constexpr int kUnrollScan = OPC_SLIDE_UNROLL_SCAN;
constexpr int kUnrollSums = OPC_SLIDE_UNROLL_SUMS;
constexpr int kStageCols = 16;   // output columns staged per flush
constexpr int kStageStride = 17;
constexpr int kRecipBytes = 1024 * 4;
constexpr int kTRows = 32;
constexpr int kTCols = 128;

__host__ __device__ inline int ring_rows(int r) { return (32 + 2 * r + 3) & ~3; }  // 16-B rows

__host__ __device__ inline std::size_t per_warp_bytes(int bins, int r) {
    const std::size_t ring = static_cast<std::size_t>(ring_cols(r)) * ring_rows(r) * 4;
    const std::size_t cnt = ((static_cast<std::size_t>(bins) * 32 * 2) + 15) & ~std::size_t(15);
    return ring + cnt + 32 * kStageStride * 4;
}

struct TGeom {
    int y_base;
    int Hs;  // rows per column (multiple of 32)
    std::size_t frame_elems;
};

__host__ inline TGeom tgeom(const BandArgs& a) {
    TGeom g{};
    g.y_base = a.y_lo - a.radius;
    const int nbands = (a.y_hi - a.y_lo + 31) / 32;
    g.Hs = 32 * nbands + 64;
    g.frame_elems = static_cast<std::size_t>(a.width + 64) * g.Hs;
    return g;
}

// Column-major plane of raw RGB (R | G << 8 | B << 16), rows [y_base, y_base + Hs);
// rows past the input are zero.  32x128 tiles through shared memory: each
// column's 32 rows are one 128-byte store.
__global__ void __launch_bounds__(256) transpose_kernel(BandArgs a, std::uint32_t* T, TGeom g) {
    __shared__ std::uint32_t tile[kTRows * (kTCols + 1)];
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
#pragma unroll
    for (int k = 0; k < kTRows / 8; ++k) {
        const int row = warp + 8 * k;
        const int y = y0 + row;
#pragma unroll
        for (int j = 0; j < kTCols / 32; ++j) {
            const int c = lane + 32 * j;
            const int x = x0 + c;
            std::uint32_t e = 0;
            if (x < a.width && y < in_hi) {
                const std::uint8_t* p = in + static_cast<std::size_t>(y - a.in_row0) * stride +
                                        static_cast<std::size_t>(x) * 3;
                e = p[0] | (static_cast<std::uint32_t>(p[1]) << 8) |
                    (static_cast<std::uint32_t>(p[2]) << 16);
            }
            tile[row * (kTCols + 1) + c] = e;
        }
    }
    __syncthreads();
    const int ymax = g.y_base + g.Hs;
    for (int c = warp; c < kTCols; c += 8) {
        const int x = x0 + c, y = y0 + lane;
        if (x < a.width + 64 && y < ymax) {
            Tf[static_cast<std::size_t>(x) * g.Hs + (y - g.y_base)] = tile[lane * (kTCols + 1) + c];
        }
    }
}

__device__ __forceinline__ std::uint32_t bin_of(std::uint32_t e, std::uint32_t bin_mul) {
    const std::uint32_t s = __dp4a(e, 0x00010101u, 0u);  // R + G + B
    return __umulhi(s, bin_mul);                          // filter.hpp:31-35
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;"); }


#if OPC_SLIDE_TRACE
// Debug trace of the passes (OPC_SLIDE_TRACE builds only): per pass
// {smid << 48 | kb << 24 | x0, x1, start ns, end ns}.
__device__ unsigned long long g_trace[1 << 16][4];
__device__ int g_trace_n;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// COUNT: the measurement instantiation (OPC_FLAG_COUNT_OPS): the same
// kernel, also counting the primitives it executes (OpCount) per lane and
// adding them to a.op_counts at exit.
template <int kRingCols, bool COUNT = false>
__global__ void __launch_bounds__(kWarps * 32)
    slide_kernel(BandArgs a, const std::uint32_t* __restrict__ T, TGeom tg, int* task_counter,
                 WorkSplit g) {
    unsigned long long opc_n[kOpCountN] = {};
    auto tally = [&](int k, unsigned long long v) {
        if constexpr (COUNT) opc_n[k] += v;
    };
    extern __shared__ __align__(16) unsigned char smem[];
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
    std::uint16_t* cnt =
        reinterpret_cast<std::uint16_t*>(wbase + static_cast<std::size_t>(kRingCols) * RR * 4);
    std::uint32_t* stage = reinterpret_cast<std::uint32_t*>(
        wbase + static_cast<std::size_t>(kRingCols) * RR * 4 +
        (((static_cast<std::size_t>(bins) * 64) + 15) & ~std::size_t(15)));

    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
    __syncthreads();

    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const std::uint32_t bm = a.bin_mul;
    const unsigned FULL = 0xFFFFFFFFu;

    long long u = 0, u_end = 0;
    int f, kb, x0, x1;
    while (next_pass<(OPC_SLIDE_GUIDED_K > 0)>(g, task_counter, lane, u, u_end, f, kb, x0, x1)) {
#if OPC_SLIDE_TRACE
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
        const int yb = a.y_lo + 32 * kb;
        const int xs = a.x_lo + x0;
        const int xe = a.x_lo + x1;
        const int ncols = xe - xs + 2 * r;  // ring-relative columns [0, ncols]: image xs-r ..
        const bool row_ok = yb + lane < a.y_hi;
        const std::uint32_t* Tf = T + tg.frame_elems * f +
                                  static_cast<std::size_t>(yb - r - tg.y_base);
        std::uint8_t* out = a.out + a.out_frame_stride * f;

        // Ring column c (relative) <- image column xs - r + c, rows yb - r .. + RR.
        auto load_chunk = [&](int c0, int n) {
            const int pieces = RR / 4;
            for (int i = lane; i < n * pieces; i += 32) {
                const int c = c0 + i / pieces;
                const int q = i - (i / pieces) * pieces;
                if (c > ncols) continue;
                const std::uint32_t* src =
                    Tf + static_cast<std::size_t>(xs - r + c) * tg.Hs + q * 4;
                cp_async16(ring + (c % kRingCols) * RR + q * 4, src);
            }
        };
        auto ringp = [&](int c) { return ring + (c % kRingCols) * RR + lane; };

        // First window: columns [0, w2) plus phase 0's entering columns.
        load_chunk(0, w2 + kPhase);
        cp_async_commit();
        load_chunk(w2 + kPhase, kPhase);
        cp_async_commit();
        cp_async_wait1();
        __syncwarp();

        // Counts are kept as keys count << kb_ | (G-1 - b mod G), G = 2^kb_ bins,
        // so within a group of G bins the largest key is the lowest-index
        // maximum and a rescan is a plain packed max.
        // (16-byte stores: one bin row is 64 bytes, 4 lanes per row)
        for (int q = lane; q < bins * 4; q += 32) {
            const std::uint32_t v = gmask - ((q >> 2) & gmask);
            const std::uint32_t v2 = v | (v << 16);
            reinterpret_cast<uint4*>(cnt)[q] = make_uint4(v2, v2, v2, v2);
        }
        __syncwarp();
        // Fast path: the first windows of all lanes lie in ring columns
        // [0, 2r] x rows [0, 32 + 2r); when that block is one colour (flat
        // content, config 3) every lane's window is (2r+1)^2 copies of it.
        const std::uint32_t e0 = ring[0];
        bool uni = true;
        for (int i = lane; i < w2 * (32 + 2 * r); i += 32) {
            const int c = i / (32 + 2 * r), k = i - c * (32 + 2 * r);
            uni &= ring[c * RR + k] == e0;  // ring columns 0..2r: no wrap
        }
        const bool flat0 = __all_sync(FULL, uni);
        if (flat0) {
            const int b0 = static_cast<int>(bin_of(e0, bm));
            cnt[b0 * 32 + lane] = static_cast<std::uint16_t>(cnt[b0 * 32 + lane] + w2 * w2 * inc);
            tally(kOpUpdates, 1);
        } else {
            tally(kOpUpdates, static_cast<unsigned long long>(w2) * w2);
            for (int c = 0; c < w2; ++c) {
                const std::uint32_t* col = ringp(c);
                for (int k = 0; k < w2; ++k) {
                    const std::uint32_t bn = bin_of(col[k], bm);
                    cnt[bn * 32 + lane] = static_cast<std::uint16_t>(cnt[bn * 32 + lane] + inc);
                }
            }
        }
        // Full scan for the lowest-index maximum (filter.hpp:71-82), all lanes
        // together: lanes 2k and 2k+1 read the 32-bit words holding both their
        // counts of one bin, the even lane the even bins, the odd lane the odd
        // ones, and swap halves at the end of each group -- half the loads and
        // one packed max per word.  Groups are combined lowest first, strict >.
        auto rescan = [&](int& best, int& bc) {
            tally(kOpBinsExamined, static_cast<unsigned long long>(bins));
            if (lane == 0) tally(kOpRescans, 1);
            const std::uint32_t* cw = reinterpret_cast<const std::uint32_t*>(cnt) + (lane >> 1);
            const unsigned sh = (lane & 1) * 16;
            best = 0;
            bc = -1;
            for (int g0 = 0; g0 < bins; g0 += gsize) {
                const int gend = min(bins, g0 + gsize);
                std::uint32_t m = 0;
#pragma unroll kUnrollScan
                for (int b = g0 + (lane & 1); b < gend; b += 2) m = __vmaxu2(m, cw[b * 16]);
                const std::uint32_t o = __shfl_xor_sync(FULL, m, 1);
                const std::uint32_t key = max((m >> sh) & 0xFFFFu, (o >> sh) & 0xFFFFu);
                const int c = static_cast<int>(key >> kb_);
                if (c > bc) {
                    bc = c;
                    best = g0 + static_cast<int>(gmask - (key & gmask));
                }
            }
        };
        auto window_sums = [&](int x_rel, int best, std::uint32_t& sr, std::uint32_t& sg,
                               std::uint32_t& sb) {
            tally(kOpSumPixels, static_cast<unsigned long long>(w2) * w2);
            sr = sg = sb = 0;
            for (int c = x_rel - r; c <= x_rel + r; ++c) {
                const std::uint32_t* col = ringp(c + r);
#pragma unroll kUnrollSums
                for (int k = 0; k < w2; ++k) {
                    const std::uint32_t e = col[k];
                    if (static_cast<int>(bin_of(e, bm)) == best) {
                        sr += e & 0xFFu;
                        sg += (e >> 8) & 0xFFu;
                        sb += (e >> 16) & 0xFFu;
                    }
                }
            }
        };
        int best, bc;
        std::uint32_t sr, sg, sb;
        if (flat0) {
            const std::uint32_t n0 = static_cast<std::uint32_t>(w2 * w2);
            best = static_cast<int>(bin_of(e0, bm));
            bc = w2 * w2;
            sr = n0 * (e0 & 0xFFu);
            sg = n0 * ((e0 >> 8) & 0xFFu);
            sb = n0 * ((e0 >> 16) & 0xFFu);
        } else {
            rescan(best, bc);
            window_sums(0, best, sr, sg, sb);
        }

        int n = xe - xs;
        for (int p = 0; kPhase * p < n; ++p) {
            if (p > 0) {
                // Phase p's entering columns were requested a phase ago; request p+1's.
                load_chunk(w2 + kPhase * (p + 1), kPhase);
                cp_async_commit();
                cp_async_wait1();
                __syncwarp();
            }
            const int xend = min(n, kPhase * p + kPhase);
            for (int x = kPhase * p; x < xend; ++x) {
                if (x > 0) {
                    tally(kOpSteps, 1);
                    // Slide: add ring column x + 2r (image x + r), remove x - 1 (image x - r - 1).
                    const std::uint32_t* cin = ringp(x + 2 * r);
                    const std::uint32_t* cout = ringp(x - 1);
                    // Warp-wide flat check: the lanes' windows cover ring rows
                    // 0 .. 31 + 2r, two rows per lane (was 2r+1 per lane: 23% of
                    // the kernel's stall samples on C3).
                    const std::uint32_t* cinb = cin - lane;
                    const std::uint32_t* coutb = cout - lane;
                    bool diff = cinb[lane] != coutb[lane];
                    if (lane < 2 * r) diff |= cinb[lane + 32] != coutb[lane + 32];
                    if (__any_sync(FULL, diff)) {
                        tally(kOpUpdates, 2ull * w2);
                        if (lane == 0) tally(kOpNonFlatSteps, 1);
                        const int best0 = best;
                        bool lost = false, cand = false;
                        int cand_b = 0, cand_c = 0;
                        // Branch-free form: every row pays two count updates (of
                        // zero when the pixel does not change bin), so lanes whose
                        // changes sit at different rows do not diverge.
                        for (int k = 0; k < w2; ++k) {
                            const std::uint32_t ei = cin[k], eo = cout[k];
                            const int bi = bin_of(ei, bm), bo = bin_of(eo, bm);
                            const bool mv = bi != bo;
                            const unsigned d = mv ? inc : 0u;
                            const unsigned ki = cnt[bi * 32 + lane] + d;
                            cnt[bi * 32 + lane] = static_cast<std::uint16_t>(ki);
                            cnt[bo * 32 + lane] = static_cast<std::uint16_t>(cnt[bo * 32 + lane] - d);
                            const int ci = static_cast<int>(ki >> kb_);
                            lost |= mv && bo == best0;
                            const bool better = mv && (ci > cand_c || (ci == cand_c && bi < cand_b));
                            cand_b = better ? bi : cand_b;
                            cand_c = better ? ci : cand_c;
                            cand |= better;
                            const std::uint32_t mi = bi == best0 ? 0xFFFFFFFFu : 0u;
                            const std::uint32_t mo = bo == best0 ? 0xFFFFFFFFu : 0u;
                            sr += (ei & mi & 0xFFu) - (eo & mo & 0xFFu);
                            sg += ((ei & mi) >> 8 & 0xFFu) - ((eo & mo) >> 8 & 0xFFu);
                            sb += ((ei & mi) >> 16 & 0xFFu) - ((eo & mo) >> 16 & 0xFFu);
                        }
                        // Resolve the winner (filter.hpp:71-82).
                        const int bcf = cnt[best0 * 32 + lane] >> kb_;
                        bool changed = false, need = false;
                        if (lost && bcf < bc) {
                            need = true;
                        } else {
                            bc = bcf;
                            if (cand) {
                                const int cf = cnt[cand_b * 32 + lane] >> kb_;
                                if (cf < cand_c) {
                                    need = true;
                                } else if (cf > bc || (cf == bc && cand_b < best)) {
                                    best = cand_b;
                                    bc = cf;
                                    changed = true;
                                }
                            }
                        }
                        if (__any_sync(FULL, need)) {
                            int nb, nc;
                            rescan(nb, nc);
                            if (need) {
                                best = nb;
                                bc = nc;
                                changed = best != best0;
                            }
                        }
                        // Winner changed: the new winner's window sums, one lane's
                        // window at a time with lane c < 2r+1 summing its column c
                        // (2r+1 loads per lane instead of (2r+1)^2 on one lane
                        // while the others wait).
                        if (changed) {
                            tally(kOpSumPixels, static_cast<unsigned long long>(w2) * w2);
                            tally(kOpWinnerChanges, 1);
                        }
                        for (unsigned todo = __ballot_sync(FULL, changed); todo; todo &= todo - 1) {
                            const int j = __ffs(todo) - 1;
                            const int bj = __shfl_sync(FULL, best, j);
                            std::uint32_t cr = 0, cg = 0, cbb = 0;
                            if (lane < w2) {
                                const std::uint32_t* col = ring + ((x + lane) % kRingCols) * RR + j;
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
                    }
                }
                if (row_ok) {
                    tally(kOpPixels, 1);
                    const std::uint32_t m = recip[bc];
                    const std::uint32_t rgb = __umulhi(sr << 1, m) | (__umulhi(sg << 1, m) << 8) |
                                              (__umulhi(sb << 1, m) << 16);
                    stage[lane * kStageStride + (x & (kStageCols - 1))] = rgb;
                }
                if ((x & (kStageCols - 1)) == kStageCols - 1 || x == n - 1) {  // flush the block
                    __syncwarp();
                    const int xb = x & ~(kStageCols - 1);
                    const int cols = x - xb + 1;
                    const int c = lane & (kStageCols - 1);
                    for (int f0 = 0; f0 < 32; f0 += 32 / kStageCols) {  // 2 rows per store
                        const int fr = f0 + lane / kStageCols;
                        if (yb + f0 >= a.y_hi) break;
                        if (c < cols && yb + fr < a.y_hi) {
                            const std::uint32_t rgb = stage[fr * kStageStride + c];
                            std::uint8_t* o = out +
                                              static_cast<std::size_t>(yb + fr - a.out_row0) * stride +
                                              static_cast<std::size_t>(xs + xb + c) * 3;
                            o[0] = static_cast<std::uint8_t>(rgb);
                            o[1] = static_cast<std::uint8_t>(rgb >> 8);
                            o[2] = static_cast<std::uint8_t>(rgb >> 16);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        cp_async_wait0();
        __syncwarp();
    }
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
    return tgeom(a).frame_elems * a.frames * sizeof(std::uint32_t);
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
    const int rc = ring_cols(a.radius);
    const bool count = a.op_counts != nullptr;
    const void* kfn =
        count ? (rc == 64   ? reinterpret_cast<const void*>(slide_kernel<64, true>)
                 : rc == 80 ? reinterpret_cast<const void*>(slide_kernel<80, true>)
                 : rc == 88 ? reinterpret_cast<const void*>(slide_kernel<88, true>)
                            : reinterpret_cast<const void*>(slide_kernel<96, true>))
              : (rc == 64   ? reinterpret_cast<const void*>(slide_kernel<64>)
                 : rc == 80 ? reinterpret_cast<const void*>(slide_kernel<80>)
                 : rc == 88 ? reinterpret_cast<const void*>(slide_kernel<88>)
                            : reinterpret_cast<const void*>(slide_kernel<96>));
    cudaError_t e = set_smem_attr(kfn, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = blocks_per_sm(kfn, warps * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;

    const TGeom tg = tgeom(a);
    std::uint32_t* T = static_cast<std::uint32_t*>(scratch);
    {
        const unsigned gx = static_cast<unsigned>((a.width + 64 + kTCols - 1) / kTCols);
        const dim3 grid(gx, static_cast<unsigned>(tg.Hs / kTRows) + border_grid_rows(a, gx),
                        static_cast<unsigned>(a.frames));
        timing_mark(kIdPrePass, 0, s);
        transpose_kernel<<<grid, 256, 0, s>>>(a, T, tg);
        timing_mark(kIdPrePass, 1, s);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const long long resident = static_cast<long long>(num_sms) * per_sm * warps;
    // Each pass pays a full window build, rescan and window sums (~3(2r+1)^2 +
    // L updates per lane): keep chunks >= 128 columns.
    const WorkSplit g = make_split(a.frames, (a.y_hi - a.y_lo + 31) / 32, a.x_hi - a.x_lo, resident,
                                   OPC_SLIDE_STATIC_PCT, OPC_SLIDE_MIN_CHUNK, OPC_SLIDE_DYN_PER_WARP,
                                   OPC_SLIDE_GUIDED_K);
    long long blocks = (g.nchunks + warps - 1) / warps;
    if (blocks > static_cast<long long>(num_sms) * per_sm) blocks = num_sms * per_sm;
    if (blocks < 1) blocks = 1;
    e = cudaMemsetAsync(counter, 0, 4 * sizeof(int), s);
    if (e != cudaSuccess) return e;
    timing_mark(kIdSlide, 0, s);
    const dim3 grid(static_cast<unsigned>(blocks)), block(warps * 32);
    // (the launch goes through the function pointer: the counting and the
    // timed instantiations share the launcher)
    void* args[] = {const_cast<BandArgs*>(&a), &T, const_cast<TGeom*>(&tg), &counter,
                    const_cast<WorkSplit*>(&g)};
    e = cudaLaunchKernel(kfn, grid, block, args, smem, s);
    timing_mark(kIdSlide, 1, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace opc

#if OPC_SLIDE_TRACE
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
