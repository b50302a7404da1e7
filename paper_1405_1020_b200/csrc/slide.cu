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
// cp.async copies 16 bytes at a time, one 32-column phase ahead.
#include "kernels.cuh"
#include "worksplit.cuh"

namespace opc {

namespace {

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
constexpr int kRingCols = 96;
constexpr int kStageStride = 33;
constexpr int kRecipBytes = 1024 * 4;
constexpr int kTRows = 32;
constexpr int kTCols = 128;

__host__ __device__ inline int ring_rows(int r) { return (32 + 2 * r + 3) & ~3; }  // 16-B rows

__host__ __device__ inline std::size_t per_warp_bytes(int bins, int r) {
    const std::size_t ring = static_cast<std::size_t>(kRingCols) * ring_rows(r) * 4;
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

__global__ void __launch_bounds__(kWarps * 32)
    slide_kernel(BandArgs a, const std::uint32_t* __restrict__ T, TGeom tg, int* task_counter,
                 WorkSplit g) {
    extern __shared__ __align__(16) unsigned char smem[];
    std::uint32_t* recip = reinterpret_cast<std::uint32_t*>(smem);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int r = a.radius;
    const int w2 = 2 * r + 1;
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
        load_chunk(0, w2 + 32);
        cp_async_commit();
        load_chunk(w2 + 32, 32);
        cp_async_commit();
        cp_async_wait1();
        __syncwarp();

        for (int b = 0; b < bins; ++b) cnt[b * 32 + lane] = 0;
        for (int c = 0; c < w2; ++c) {
            const std::uint32_t* col = ringp(c);
            for (int k = 0; k < w2; ++k) {
                const std::uint32_t bn = bin_of(col[k], bm);
                cnt[bn * 32 + lane] = static_cast<std::uint16_t>(cnt[bn * 32 + lane] + 1);
            }
        }
        // Full scan for the lowest-index maximum, then the winner's sums.
        auto rescan = [&](int& best, int& bc) {
            best = 0;
            bc = cnt[lane];
            for (int b = 1; b < bins; ++b) {
                const int c = cnt[b * 32 + lane];
                if (c > bc) {
                    bc = c;
                    best = b;
                }
            }
        };
        auto window_sums = [&](int x_rel, int best, std::uint32_t& sr, std::uint32_t& sg,
                               std::uint32_t& sb) {
            sr = sg = sb = 0;
            for (int c = x_rel - r; c <= x_rel + r; ++c) {
                const std::uint32_t* col = ringp(c + r);
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
        rescan(best, bc);
        std::uint32_t sr, sg, sb;
        window_sums(0, best, sr, sg, sb);

        const int n = xe - xs;
        for (int p = 0; 32 * p < n; ++p) {
            if (p > 0) {
                // Phase p's entering columns were requested a phase ago; request p+1's.
                load_chunk(w2 + 32 * (p + 1), 32);
                cp_async_commit();
                cp_async_wait1();
                __syncwarp();
            }
            const int xend = min(n, 32 * p + 32);
            for (int x = 32 * p; x < xend; ++x) {
                if (x > 0) {
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
                        const int best0 = best;
                        bool lost = false, cand = false;
                        int cand_b = 0, cand_c = 0;
                        for (int k = 0; k < w2; ++k) {
                            const std::uint32_t ei = cin[k], eo = cout[k];
                            if (ei == eo) continue;
                            const int bi = bin_of(ei, bm), bo = bin_of(eo, bm);
                            if (bi != bo) {
                                const int ci = cnt[bi * 32 + lane] + 1;
                                cnt[bi * 32 + lane] = static_cast<std::uint16_t>(ci);
                                cnt[bo * 32 + lane] = static_cast<std::uint16_t>(cnt[bo * 32 + lane] - 1);
                                if (bo == best0) lost = true;
                                if (ci > cand_c || (ci == cand_c && bi < cand_b)) {
                                    cand_b = bi;
                                    cand_c = ci;
                                    cand = true;
                                }
                            }
                            if (bi == best0) {
                                sr += ei & 0xFFu;
                                sg += (ei >> 8) & 0xFFu;
                                sb += (ei >> 16) & 0xFFu;
                            }
                            if (bo == best0) {
                                sr -= eo & 0xFFu;
                                sg -= (eo >> 8) & 0xFFu;
                                sb -= (eo >> 16) & 0xFFu;
                            }
                        }
                        // Resolve the winner (filter.hpp:71-82).
                        const int bcf = cnt[best0 * 32 + lane];
                        bool changed = false;
                        if (lost && bcf < bc) {
                            rescan(best, bc);
                            changed = best != best0;
                        } else {
                            bc = bcf;
                            if (cand) {
                                const int cf = cnt[cand_b * 32 + lane];
                                if (cf < cand_c) {
                                    rescan(best, bc);
                                    changed = best != best0;
                                } else if (cf > bc || (cf == bc && cand_b < best)) {
                                    best = cand_b;
                                    bc = cf;
                                    changed = true;
                                }
                            }
                        }
                        if (changed) window_sums(x, best, sr, sg, sb);
                    }
                }
                if (row_ok) {
                    const std::uint32_t m = recip[bc];
                    const std::uint32_t rgb = __umulhi(sr << 1, m) | (__umulhi(sg << 1, m) << 8) |
                                              (__umulhi(sb << 1, m) << 16);
                    stage[lane * kStageStride + (x & 31)] = rgb;
                }
                if ((x & 31) == 31 || x == n - 1) {  // flush the 32-column block
                    __syncwarp();
                    const int xb = x & ~31;
                    const int cols = x - xb + 1;
                    for (int fr = 0; fr < 32; ++fr) {
                        if (yb + fr >= a.y_hi) break;
                        if (lane < cols) {
                            const std::uint32_t rgb = stage[fr * kStageStride + lane];
                            std::uint8_t* o = out +
                                              static_cast<std::size_t>(yb + fr - a.out_row0) * stride +
                                              static_cast<std::size_t>(xs + xb + lane) * 3;
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
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(slide_kernel), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = blocks_per_sm(reinterpret_cast<const void*>(slide_kernel), warps * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;

    const TGeom tg = tgeom(a);
    std::uint32_t* T = static_cast<std::uint32_t*>(scratch);
    {
        const dim3 grid(static_cast<unsigned>((a.width + 64 + kTCols - 1) / kTCols),
                        static_cast<unsigned>(tg.Hs / kTRows), static_cast<unsigned>(a.frames));
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
    slide_kernel<<<static_cast<unsigned>(blocks), warps * 32, smem, s>>>(a, T, tg, counter, g);
    timing_mark(kIdSlide, 1, s);
    return cudaGetLastError();
}

}  // namespace opc
