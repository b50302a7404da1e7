// planes.cu -- the bit-plane column family (L+1 <= 32, r <= 7): window counts
// as bit planes in registers, the winner's channel sums from column-sum
// histograms in shared memory.  DESIGN.md section 3.0.
//
// The column family (column.cu) keeps every thread's window histogram in
// shared memory and pays two 32-bit read-modify-writes per updated pixel
// (2(2r+1) per output row): ~166 shared-memory wavefronts per 32 pixels on
// config 2, which bounds it at the L1 data pipe (profiles/r01_c2_column_ncu.md).
// Here a 128-thread block owns 128 output columns x TH rows, each lane one
// column, and the vertical slide is split in two:
//
//  * COUNTS, bit-sliced in registers (bitplanes.cuh).  Bit b of plane word
//    Wk holds bit k of bin b's window count (<= 32 bins, one bit each).  The
//    row histogram of the entering window row (2r+1 one-hot masks 1 << bin)
//    is a carry-save adder tree (XOR3 / MAJ, one LOP3 each: 16 for 11 masks);
//    the window counts advance by W += RH(y+r+1) - RH(y-r) with the leaving
//    row's planes kept in a register ring of 2r+1 slots (the row loop is
//    unrolled by 2r+1).  The lowest-index bin with the largest count
//    (filter.hpp:71-82) falls out of a walk down the planes from the top:
//    keep the candidates that have bit k set if any does -- the survivors are
//    the bins with the maximum count, the lowest one is __ffs.  No shared
//    memory, no dynamic indexing.
//
//  * SUMS of the winning bin only, from column histograms.  For every tile
//    column, CS[bin][column] = (R | count << 16, G << 16 | B) over the
//    current 2r+1 window rows (r <= 7: column sums < 2^12, window sums and
//    counts fit their 16-bit fields).  Per output row each lane subtracts
//    the leaving and adds the entering pixel of its column (lanes < 2r also
//    of one halo column), then sums CS[best][x .. x+2r] -- 2r+1 LDS.64 with a
//    bin pitch that is a multiple of 32 words, so lane l reads bank (l + j)
//    mod 32 whatever the lanes' bins -- and the hi-word sum carries the
//    winner's count.  One-round launches keep one CS array per warp ([warp]
//    [nb][48], warp barriers); multi-round launches one per block ([nb][144],
//    block barriers, three blocks per SM).
//
//  * Tile by TMA: one box of raw RGB rows per block, converted in shared
//    memory to entries bin | R << 8 | G << 16 | B << 24 (byte loads where
//    the rows are not 16-byte aligned).
//
// Per row step (r = 5): ~177 SASS instructions, ~45 shared-memory wavefronts
// per 32 pixels.
//
// Truncating quotient per channel (filter.cpp:41-43): umulhi(2*sum, m_c),
// m_c = floor(2^31/c) + 1 (exact for c <= 1023, sum <= 255c; checked
// exhaustively by tests/test_oracle.py::test_reciprocal_division_exact).
// The launch's border pixels are shared out over the filter blocks (border.cuh).
#include "kernels.cuh"
#include "border.cuh"
#include "tma.cuh"
#include "bitplanes.cuh"

#include <algorithm>

#ifndef OPC_PLANES_PITCH_W
#define OPC_PLANES_PITCH_W 48  // uint2 entries per bin row of a warp's column sums (>= 32 + 2r, multiple of 16)
#endif
#ifndef OPC_PLANES_PITCH_B
#define OPC_PLANES_PITCH_B 144  // ... of a block's (>= 128 + 2r, multiple of 16)
#endif
#ifndef OPC_PLANES_HALO_BRANCHLESS
#define OPC_PLANES_HALO_BRANCHLESS 1  // per-warp sums: halo column updates without a divergent block
#endif
#ifndef OPC_PLANES_TMA
#define OPC_PLANES_TMA 1  // TMA tile loads (raw RGB rows) where the row layout allows
#endif
#ifndef OPC_PLANES_BCS
#define OPC_PLANES_BCS 2  // column sums: 0 per warp, 1 block-shared (block barriers), 2 by launch size
#endif
#ifndef OPC_PLANES_THMAX_BCS
#define OPC_PLANES_THMAX_BCS 48  // rows per block of multi-round launches with block-shared sums
#endif
#ifndef OPC_PLANES_BPS_MAX
#define OPC_PLANES_BPS_MAX 4  // most blocks per SM the row planning aims for
#endif
#ifndef OPC_PLANES_THMAX
#define OPC_PLANES_THMAX 64  // rows per block when the image needs several rounds of blocks
#endif

namespace opc {

namespace {

constexpr int kPlWarps = 4;
constexpr int kPlThreads = 32 * kPlWarps;
constexpr int kPlCols = 32 * kPlWarps;  // output columns per block
constexpr int kPlMaxR = 7;
constexpr int kPlPitch = OPC_PLANES_PITCH_W;  // per-warp CS: uint2 per bin row, >= 32 + 2r, a multiple of 16 (2 words each)
constexpr int kPlBPitch = OPC_PLANES_PITCH_B;  // block-shared CS: >= 128 + 2r, a multiple of 16

struct PlGeom {
    int th;  // output rows per block
    int nb;  // bins (L + 1)
};

template <int R>
__host__ __device__ constexpr int pl_planes() {
    // bits of the largest window count (2R+1)^2
    int n = (2 * R + 1) * (2 * R + 1), p = 0;
    while (n) {
        ++p;
        n >>= 1;
    }
    return p;
}

template <int R>
__host__ __device__ constexpr int pl_tile_cols() {
    return kPlCols + 2 * R;
}


// Tile entry of one pixel: bin | R << 8 | G << 16 | B << 24.
// hi word R | 1 << 16: the column sums count their pixels in bits 16..23
// (window counts <= 225; R sums < 2^16 never carry into them), so the
// winner's count comes with its sums (A/B against spelling it from the plane
// walk: C2 -6%, C5 -3%, profiles/r02_notes.md)
__device__ __forceinline__ std::uint32_t pl_hi(std::uint32_t e) { return __byte_perm(e, 1u, 0x5451); }
__device__ __forceinline__ std::uint32_t pl_lo(std::uint32_t e) { return __byte_perm(e, 0u, 0x4243); }  // G << 16 | B

// Row histogram (4 planes: counts <= 15) of the 2R+1 entries at row[0 .. 2R].
template <int R>
__device__ __forceinline__ void row_planes(const std::uint32_t* row, std::uint32_t (&q)[4]) {
    constexpr int W2 = 2 * R + 1;
    std::uint32_t m[W2];
#pragma unroll
    for (int j = 0; j < W2; ++j) m[j] = bin_mask(row[j]);
    Csa<W2, 0, 4>::run(m, q);
}

// Raw RGB rows staged by TMA (the TMA variant): one box of 112 u32 words (448
// bytes >= 3 (128 + 2r) + 15) x TR rows, starting at the 16-byte-aligned
// word at or left of the tile's first byte; row pitch 448 bytes.
constexpr int kPlRawWords = 112;

template <int R>
__host__ inline std::size_t pl_region_bytes(const PlGeom& g, bool tma, bool bcs) {
    const std::size_t cs = bcs ? static_cast<std::size_t>(g.nb) * kPlBPitch * 8
                               : static_cast<std::size_t>(kPlWarps) * g.nb * kPlPitch * 8;
    const std::size_t raw = tma ? static_cast<std::size_t>(kPlRawWords) * 4 * (g.th + 2 * R) : 0;
    return cs > raw ? cs : raw;
}

template <int R>
__host__ inline std::size_t pl_smem_total(const PlGeom& g, bool tma, bool bcs) {
    const std::size_t tile = static_cast<std::size_t>(pl_tile_cols<R>()) * (g.th + 2 * R) * 4;
    const std::size_t recip = static_cast<std::size_t>((2 * R + 1) * (2 * R + 1) + 1) * 4;
    return pl_region_bytes<R>(g, tma, bcs) + tile + ((recip + 15) & ~std::size_t(15)) + 16;
}

// The launch's border pixels (border.cuh: 256-thread job blocks of the
// frame) are shared out over the filter blocks of that frame, so no extra
// blocks queue behind the filter blocks; each filter block runs its share
// while its tile loads.
__device__ __forceinline__ void border_share(const BandArgs& a, int tid) {
    const int per_frame = gridDim.x * gridDim.y;
    for (int b = blockIdx.y * gridDim.x + blockIdx.x; b < a.border.nblocks; b += per_frame) {
        border_block(a, b, blockIdx.z, tid);
        border_block(a, b, blockIdx.z, tid + kPlThreads);
    }
}

// BCS: one block-shared column-sum array ([nb][144]: every tile column once,
// the block's 4 warps step in lockstep with block barriers) instead of one
// per warp ([warp][nb][48]: 2r halo columns per warp, warp barriers only).
template <int R, bool TMA, bool BCS>
__global__ void __launch_bounds__(kPlThreads)
    planes_kernel(BandArgs a, PlGeom g, unsigned region_bytes, const __grid_constant__ CUtensorMap tin) {
    constexpr int W2 = 2 * R + 1;
    constexpr int P = pl_planes<R>();
    constexpr int TW = pl_tile_cols<R>();
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = g.nb;
    const int TR = g.th + 2 * R;
    constexpr int PITCH = BCS ? kPlBPitch : kPlPitch;
    uint2* cs_all = reinterpret_cast<uint2*>(smem);  // [warp][nb][48] or [nb][144]: (R | count << 16, G << 16 | B)
    std::uint32_t* tile = reinterpret_cast<std::uint32_t*>(smem + region_bytes);  // [TR][TW]
    std::uint32_t* recip = tile + TR * TW;
    recip = reinterpret_cast<std::uint32_t*>((reinterpret_cast<std::uintptr_t>(recip) + 15) & ~std::uintptr_t(15));
    constexpr int nrec = W2 * W2 + 1;
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(recip + ((nrec + 3) & ~3));

    const int x0 = a.x_lo + blockIdx.x * kPlCols;  // first output column of the block
    const int y0 = a.y_lo + blockIdx.y * g.th;     // first output row of the block
    const int frame = blockIdx.z;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;

    // ---- tile: (TR rows) x (TW columns) entries bin | R << 8 | G << 16 |
    // B << 24 of input rows y0-R .., columns x0-R ..  Columns past the image
    // and rows past the band only feed outputs that are not stored: the LDG
    // path clamps them, TMA zero-fills them ----
    if constexpr (TMA) {
        const int xb = 3 * (x0 - R);
        const int xw = (xb >> 4) << 2;  // 16-byte-aligned start word
        const int delta = xb - 4 * xw;  // 0 .. 15
        if (tid == 0) {
            prefetch_tensor_map(&tin);
            mbar_init(bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(bar, static_cast<unsigned>(kPlRawWords * 4 * TR));
            tma_load_3d(smem, &tin, xw, y0 - R - a.in_row0, frame, bar);
        }
        for (int i = tid; i < nrec; i += kPlThreads) recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
        border_share(a, tid);  // while the tile is in flight
        __syncthreads();  // (barrier initialised before anyone waits on it)
        mbar_wait(bar, 0);
        const std::uint32_t* raw = reinterpret_cast<const std::uint32_t*>(smem);
        const int n = TR * TW;
        for (int i = tid; i < n; i += kPlThreads) {
            const int ty = i / TW, tx = i - ty * TW;
            const int bo = delta + 3 * tx;
            const std::uint32_t* q = raw + ty * kPlRawWords + (bo >> 2);
            const std::uint32_t v = __funnelshift_r(q[0], q[1], (bo & 3) * 8);  // R | G << 8 | B << 16 | x
            tile[i] = __umulhi(__dp4a(v, 0x00010101u, 0u), a.bin_mul) | (v << 8);
        }
        __syncthreads();  // raw rows consumed: the region becomes the column sums
    } else {
        border_share(a, tid);
        const std::uint8_t* in = a.in + a.in_frame_stride * frame;
        const int in_last = a.in_row0 + a.in_rows - 1;
        constexpr int kBatch = 8;
        const int n = TR * TW;
        for (int i0 = tid; i0 < n; i0 += kBatch * kPlThreads) {
            std::uint32_t R_[kBatch], G_[kBatch], B_[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = min(i0 + j * kPlThreads, n - 1);
                const int ty = i / TW, tx = i - ty * TW;
                const int x = min(x0 - R + tx, a.width - 1);
                const int y = min(y0 - R + ty, in_last);
                const std::uint8_t* q = in + static_cast<std::size_t>(y - a.in_row0) * stride + static_cast<std::size_t>(x) * 3;
                R_[j] = q[0];
                G_[j] = q[1];
                B_[j] = q[2];
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j * kPlThreads;
                if (i < n) {
                    tile[i] = __umulhi(R_[j] + G_[j] + B_[j], a.bin_mul) | (R_[j] << 8) | (G_[j] << 16) |
                              (B_[j] << 24);
                }
            }
        }
        for (int i = tid; i < nrec; i += kPlThreads) recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
    uint2* cs = BCS ? cs_all : cs_all + warp * nb * kPlPitch;
    // zero the column sums of the columns in use only (the block's TW = 128 +
    // 2R or the warp's 32 + 2R of each bin row; the pitch pads them to a bank
    // multiple): thread (or lane) c zeroes column c and the halo thread its
    // halo column, of every bin
    {
        const int c = BCS ? tid : lane;
        const bool zh = BCS ? tid < 2 * R : lane < 2 * R;
        constexpr int ZH = BCS ? kPlCols : 32;
        for (int b = 0; b < nb; ++b) {
            cs[b * PITCH + c] = make_uint2(0u, 0u);
            if (zh) cs[b * PITCH + c + ZH] = make_uint2(0u, 0u);
        }
    }
    __syncthreads();

    const int nrows = min(g.th, a.y_hi - y0);  // warp-uniform
    if (nrows <= 0) return;
    // lane's window: tile columns c0 .. c0 + 2R; its own CS column (c0 in
    // the block's array, lane in the warp's) and its halo column, tile column
    // c0 + HOFF (per-warp arrays: lanes < 2R, column lane + 32; block array:
    // warp 0's lanes < 2R, column 128 + lane)
    const int c0 = warp * 32 + lane;
    const bool halo = BCS ? (warp == 0 && lane < 2 * R) : lane < 2 * R;
    constexpr int HOFF = BCS ? kPlCols : 32;
    const int own = BCS ? c0 : lane;
    const std::uint32_t* trow = tile + c0;  // tile row 0, the lane's window start

    // ---- first window: tile rows 0 .. 2R ----
    std::uint32_t ring[W2][4];
    std::uint32_t w[P];
#pragma unroll
    for (int k = 0; k < P; ++k) w[k] = 0u;
#pragma unroll
    for (int i = 0; i < W2; ++i) {
        row_planes<R>(trow + i * TW, ring[i]);
        planes_add<P>(w, ring[i]);
    }
#pragma unroll 1
    for (int i = 0; i < W2; ++i) {
        const std::uint32_t e = trow[i * TW];
        uint2& v = cs[(e & 31u) * PITCH + own];
        v.x += pl_hi(e);
        v.y += pl_lo(e);
        if (halo) {
            const std::uint32_t eh = trow[i * TW + HOFF];
            uint2& vh = cs[(eh & 31u) * PITCH + own + HOFF];
            vh.x += pl_hi(eh);
            vh.y += pl_lo(eh);
        }
    }
    if (BCS) {
        __syncthreads();
    } else {
        __syncwarp();
    }

    const int x = x0 + lane + warp * 32;
    const bool store = x < a.x_hi;
    std::uint8_t* o = a.out + a.out_frame_stride * frame +
                      static_cast<std::size_t>(y0 - a.out_row0) * stride + static_cast<std::size_t>(x) * 3;
    const uint2* csl = cs + own;

    // Entries the next slide needs (entering row e = k + 1 + 2R: the lane's
    // 2R+1 window columns and its halo column; leaving row k: its own and halo
    // column), loaded one row ahead.  Rows past the tile are clamped: the
    // slide they feed is never emitted.
    std::uint32_t ent[W2], eh, el, elh;
    auto fetch = [&](int k) {
        const std::uint32_t* erow = trow + min(k + 1 + 2 * R, TR - 1) * TW;
        const std::uint32_t* lrow = trow + min(k, TR - 1) * TW;
#pragma unroll
        for (int j = 0; j < W2; ++j) ent[j] = erow[j];
        eh = halo ? erow[HOFF] : 0u;  // (column c0 + HOFF exists for halo lanes only)
        el = lrow[0];
        elh = halo ? lrow[HOFF] : 0u;
    };
    fetch(0);

    // ---- row loop.  Iteration k emits output row k (window = tile rows k ..
    // k + 2R, column sums of those rows) and slides the planes and column sums
    // to row k + 1.  The next window's counts are computed between issuing the
    // winner's column-sum loads and using them.  Ring slot s holds the planes
    // of tile row k (k == s mod W2), the row that leaves next. ----
    int k = 0;
    for (;;) {
#pragma unroll
        for (int s = 0; s < W2; ++s) {
            // argmax of window k (filter.hpp:71-82): the lowest of the bins
            // holding the largest count (plane walk, bitplanes.cuh)
            const uint2* pb = csl + (__ffs(plane_max_bins<P>(w)) - 1) * PITCH;
            uint2 v[W2];
#pragma unroll
            for (int j = 0; j < W2; ++j) v[j] = pb[j];
            // counts of window k + 1
            {
                std::uint32_t rin[4], mk[W2];
#pragma unroll
                for (int j = 0; j < W2; ++j) mk[j] = bin_mask(ent[j]);
                Csa<W2, 0, 4>::run(mk, rin);
                planes_update<P>(w, rin, ring[s]);
#pragma unroll
                for (int p = 0; p < 4; ++p) ring[s][p] = rin[p];
            }
            const std::uint32_t ee = ent[0], ehe = eh, el0 = el, elh0 = elh;
            fetch(k + 1);
            // output row k (filter.cpp:41-43)
            std::uint32_t sr = 0u, sgb = 0u;
#pragma unroll
            for (int j = 0; j < W2; ++j) {
                sr += v[j].x;
                sgb += v[j].y;
            }
            const std::uint32_t m = recip[sr >> 16];  // the winner's count rides in the hi words
            sr &= 0xFFFFu;
            if (store) {
                o[0] = static_cast<std::uint8_t>(__umulhi(sr << 1, m));
                o[1] = static_cast<std::uint8_t>(__umulhi((sgb >> 16) << 1, m));
                o[2] = static_cast<std::uint8_t>(__umulhi((sgb & 0xFFFFu) << 1, m));
            }
            o += stride;
            if (++k >= nrows) return;
            // every lane has read row k - 1's column sums
            if (BCS) {
                __syncthreads();
            } else {
                __syncwarp();
            }
            {
                uint2& vl = cs[(el0 & 31u) * PITCH + own];
                vl.x -= pl_hi(el0);
                vl.y -= pl_lo(el0);
                uint2& ve = cs[(ee & 31u) * PITCH + own];
                ve.x += pl_hi(ee);
                ve.y += pl_lo(ee);
#if OPC_PLANES_HALO_BRANCHLESS
                if (!BCS) {
                    // Branch-free halo update (per-warp sums, where every warp
                    // has halo lanes): the other lanes add zero to bin 0 of
                    // their own column (elh0 = ehe = 0 for them), which only
                    // they write -- conflict-free, no divergent block.
                    const int hc = halo ? own + HOFF : own;
                    const std::uint32_t hm = halo ? 0xFFFFFFFFu : 0u;
                    uint2& hl = cs[(elh0 & 31u) * PITCH + hc];
                    hl.x -= pl_hi(elh0) & hm;
                    hl.y -= pl_lo(elh0);
                    uint2& he = cs[(ehe & 31u) * PITCH + hc];
                    he.x += pl_hi(ehe) & hm;
                    he.y += pl_lo(ehe);
                } else
#endif
                if (halo) {
                    uint2& hl = cs[(elh0 & 31u) * PITCH + own + HOFF];
                    hl.x -= pl_hi(elh0);
                    hl.y -= pl_lo(elh0);
                    uint2& he = cs[(ehe & 31u) * PITCH + own + HOFF];
                    he.x += pl_hi(ehe);
                    he.y += pl_lo(ehe);
                }
            }
            // column sums of row k complete
            if (BCS) {
                __syncthreads();
            } else {
                __syncwarp();
            }
        }
    }
}

template <int R, bool TMA, bool BCS>
cudaError_t launch_rt(const BandArgs& a, const PlGeom& g, const CUtensorMap& tin, cudaStream_t s) {
    const std::size_t region = pl_region_bytes<R>(g, TMA, BCS);
    const std::size_t smem = pl_smem_total<R>(g, TMA, BCS);
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(planes_kernel<R, TMA, BCS>), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const unsigned gx = static_cast<unsigned>((a.x_hi - a.x_lo + kPlCols - 1) / kPlCols);
    const dim3 grid(gx, static_cast<unsigned>((a.y_hi - a.y_lo + g.th - 1) / g.th), static_cast<unsigned>(a.frames));
    timing_mark(kIdPlanes, 0, s);
    planes_kernel<R, TMA, BCS><<<grid, kPlThreads, smem, s>>>(a, g, static_cast<unsigned>(region), tin);
    timing_mark(kIdPlanes, 1, s);
    return cudaGetLastError();
}

// Rows per block: one round of resident blocks when the image allows (the
// first window's 2r+1 rows are amortised over as many rows as possible),
// capped at thmax rows otherwise.  Returns true when the cap was hit (the
// launch needs several rounds of blocks).
template <int R>
bool plan_rows(const BandArgs& a, int num_sms, bool tma, bool bcs, int thmax, PlGeom& g) {
    const long long iw = a.x_hi - a.x_lo, ih = a.y_hi - a.y_lo;
    const long long units = (iw + kPlCols - 1) / kPlCols * ih * a.frames;  // block-columns x rows
    for (int bps = OPC_PLANES_BPS_MAX; bps >= 1; --bps) {
        const long long want = static_cast<long long>(num_sms) * bps;
        const long long th = (units + want - 1) / want;
        g.th = static_cast<int>(std::max(4ll, std::min<long long>(thmax, th)));
        if (bps == 1 || pl_smem_total<R>(g, tma, bcs) * bps + bps * 1024 <= 228u * 1024) return th > thmax;
    }
    return false;
}

template <int R>
cudaError_t launch_r(const BandArgs& a, int num_sms, cudaStream_t s) {
    PlGeom g{};
    g.nb = a.levels + 1;
    // TMA tile loads when the rows are 16-byte-aligned word arrays
    const std::size_t row_bytes = static_cast<std::size_t>(a.width) * 3;
    bool tma = OPC_PLANES_TMA && row_bytes % 16 == 0 && a.in_frame_stride % 16 == 0 &&
               reinterpret_cast<std::uintptr_t>(a.in) % 16 == 0;
    // Column sums: per warp for a launch that fits one round of blocks (no
    // block barriers; C2 -6%), block-shared for launches of several rounds
    // (smaller blocks, more of them resident: C5 -10%; measured, profiles/r02_notes.md)
    bool bcs = OPC_PLANES_BCS == 1;
    if (OPC_PLANES_BCS == 2) {
        bcs = plan_rows<R>(a, num_sms, tma, false, OPC_PLANES_THMAX, g);
    }
    plan_rows<R>(a, num_sms, tma, bcs, bcs ? OPC_PLANES_THMAX_BCS : OPC_PLANES_THMAX, g);
    CUtensorMap tin{};
    if (tma) {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(row_bytes / 4), static_cast<cuuint64_t>(a.in_rows),
                                    static_cast<cuuint64_t>(a.frames)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_bytes),
                                       static_cast<cuuint64_t>(a.in_frame_stride)};
        const cuuint32_t box[3] = {static_cast<cuuint32_t>(kPlRawWords),
                                   static_cast<cuuint32_t>(g.th + 2 * R), 1};
        tma = encode_tensor_map(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<std::uint8_t*>(a.in), dims,
                                strides, box) == 0;
    }
    if (tma) return bcs ? launch_rt<R, true, true>(a, g, tin, s) : launch_rt<R, true, false>(a, g, tin, s);
    return bcs ? launch_rt<R, false, true>(a, g, tin, s) : launch_rt<R, false, false>(a, g, tin, s);
}

}  // namespace

bool planes_supported(int levels, int radius) {
    return levels >= 1 && levels + 1 <= 32 && radius >= 1 && radius <= kPlMaxR && bin_multiplier(levels) != 0;
}

cudaError_t launch_planes(const BandArgs& a, int num_sms, cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    switch (a.radius) {
        case 1: return launch_r<1>(a, num_sms, s);
        case 2: return launch_r<2>(a, num_sms, s);
        case 3: return launch_r<3>(a, num_sms, s);
        case 4: return launch_r<4>(a, num_sms, s);
        case 5: return launch_r<5>(a, num_sms, s);
        case 6: return launch_r<6>(a, num_sms, s);
        case 7: return launch_r<7>(a, num_sms, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace opc
