// column.cu -- the small-image kernel family (L+1 <= 32, r <= 7): one thread per
// output column segment, sliding its window histogram DOWN the segment.
//
// The skew family pays a fixed 2(2r+1) + 32-step fill/drain per pass, which is
// most of the work when an image has only a few thousand band columns per SM
// (config 2: 1920x1080 -> 48-column passes, 47% of the steps produce output).
// Here a block of 256 threads owns a tile of TWC columns x (256/TWC) row
// groups; thread (cx, gy) produces column x0 + cx, rows y0 + gy*TH .. + TH - 1:
//
//  * the tile's input pixels (plus the r-pixel halo) are loaded once into
//    shared memory as entries B | R << 8 | G << 16 | bin << 24
//    (bin = (R+G+B)*L/765, filter.hpp:31-35);
//  * the thread's window histogram lives in shared memory as two 32-bit words
//    per bin, hi = count << 22 | (31 - bin) << 16 | sumR, lo = sumG << 16 | sumB
//    (r <= 7: sums < 2^16), in [bin][thread] arrays (a warp's dynamic-bin
//    accesses hit 32 consecutive words: conflict-free);
//  * the first window is built with (2r+1)^2 updates, every next row with
//    2(2r+1): the leaving row's pixels subtracted, the entering row's added
//    (modular packed arithmetic is exact while every window total fits its
//    field);
//  * lowest-index bin with the largest count (filter.hpp:71-82): the largest
//    hi word -- count first, then the constant (31 - bin) field;
//  * truncating quotient per channel (filter.cpp:41-43): umulhi(2*sum, m_c),
//    m_c = floor(2^31/c) + 1 from a shared table (exact for c <= 1023).
//
// The border pixels of the launch ride on extra blocks (border.cuh), as in the
// direct tile kernel.
#include "kernels.cuh"
#include "border.cuh"

#include <algorithm>

#ifndef OPC_COLUMN_TWC
#define OPC_COLUMN_TWC 64
#endif
#ifndef OPC_COLUMN_THREADS_PER_SM
#define OPC_COLUMN_THREADS_PER_SM 768
#endif
#ifndef OPC_COLUMN_TH
#define OPC_COLUMN_TH 0  // rows per thread; 0 = sized to the launch
#endif

namespace opc {

namespace {

constexpr int kColThreads = 256;
constexpr int kColMaxR = 7;
constexpr int kColMaxBins = 32;

struct ColGeom {
    int twc;  // columns per tile (32, 64, 128, 256)
    int th;   // rows per thread
};

__host__ __device__ inline int col_tile_rows(const ColGeom& g) { return (kColThreads / g.twc) * g.th; }

__host__ inline std::size_t col_smem_bytes(const ColGeom& g, int bins, int r) {
    const std::size_t hist = static_cast<std::size_t>(bins) * kColThreads * 8;
    const std::size_t tile = static_cast<std::size_t>(g.twc + 2 * r) * (col_tile_rows(g) + 2 * r) * 4;
    const std::size_t recip = static_cast<std::size_t>((2 * r + 1) * (2 * r + 1) + 1) * 4;
    return hist + tile + 16 + ((recip + 15) & ~std::size_t(15));
}

// Histogram words of one bin (r <= 7: window totals count <= 225, channel sums
// <= 225 * 255 < 2^16), two independent 32-bit words:
//   hi = count << 22 | (31 - bin) << 16 | sumR      lo = sumG << 16 | sumB
// The constant (31 - bin) field makes the largest hi word the largest count at
// the lowest bin, so the argmax is a plain max.  Adds and subtracts are modular
// 32-bit arithmetic, exact whenever the window totals fit their fields (no
// carry ever needs to cross from lo to hi).  Separate [bin][thread] arrays of
// 32-bit words: the argmax reads of the hi words are conflict-free (as the
// high halves of 64-bit words, lanes t and t+16 shared a bank).
// Tile entry of one pixel: B | R << 8 | G << 16 | bin << 24.
__device__ __forceinline__ std::uint32_t col_lo(std::uint32_t e) { return __byte_perm(e, 0u, 0x4240); }  // B | G << 16
__device__ __forceinline__ std::uint32_t col_hi(std::uint32_t e) {
    return __byte_perm(e, 0x00400000u, 0x7641);  // R | 1 << 22
}

template <int NB>
__global__ void __launch_bounds__(kColThreads)
    column_kernel(BandArgs a, ColGeom g) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    const int rg = kColThreads / g.twc;
    const int trows = rg * g.th;
    const int main_rows = (a.y_hi - a.y_lo + trows - 1) / trows;
    if (static_cast<int>(blockIdx.y) >= main_rows) {  // appended border blocks
        const int b = (blockIdx.y - main_rows) * gridDim.x + blockIdx.x;
        if (b < a.border.nblocks) border_block(a, b, blockIdx.z, tid);
        return;
    }
    const int r = a.radius;
    const int w2 = 2 * r + 1;
    const int tw = g.twc + 2 * r, tht = trows + 2 * r;
    std::uint32_t* hist_hi = reinterpret_cast<std::uint32_t*>(smem);  // [NB][256]
    std::uint32_t* hist_lo = hist_hi + NB * kColThreads;               // [NB][256]
    std::uint32_t* tile = reinterpret_cast<std::uint32_t*>(smem + std::size_t(NB) * kColThreads * 8);
    std::uint32_t* recip = tile + tw * tht;
    recip = reinterpret_cast<std::uint32_t*>((reinterpret_cast<std::uintptr_t>(recip) + 15) & ~std::uintptr_t(15));

    const int x0 = a.x_lo + blockIdx.x * g.twc;
    const int y0 = a.y_lo + blockIdx.y * trows;
    const int frame = blockIdx.z;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    const int in_last = a.in_row0 + a.in_rows - 1;
    {
        // rows_per_pass rows of the tile per pass of the block (tw <= 256 + 2r)
        const int rows_per_pass = max(1, kColThreads / tw);
        const int ty0 = tid / tw, tx = tid - ty0 * tw;
        if (ty0 < rows_per_pass) {
            const int x = min(x0 - r + tx, a.width - 1);
            const std::uint8_t* p = in + static_cast<std::size_t>(x) * 3;
            // kLoadBatch rows' loads in flight before the first store: the
            // launch is one round of blocks, so this phase is pure latency
            constexpr int kLoadBatch = 8;
            for (int ty = ty0; ty < tht; ty += kLoadBatch * rows_per_pass) {
                std::uint32_t R[kLoadBatch], G[kLoadBatch], B[kLoadBatch];
#pragma unroll
                for (int j = 0; j < kLoadBatch; ++j) {
                    const int y = min(y0 - r + min(ty + j * rows_per_pass, tht - 1), in_last);
                    const std::uint8_t* q = p + static_cast<std::size_t>(y - a.in_row0) * stride;
                    R[j] = q[0];
                    G[j] = q[1];
                    B[j] = q[2];
                }
#pragma unroll
                for (int j = 0; j < kLoadBatch; ++j) {
                    const int yy = ty + j * rows_per_pass;
                    if (yy < tht) {
                        tile[yy * tw + tx] = B[j] | (R[j] << 8) | (G[j] << 16) |
                                             (__umulhi(R[j] + G[j] + B[j], a.bin_mul) << 24);
                    }
                }
            }
        }
    }
    const int nrec = w2 * w2 + 1;
    for (int i = tid; i < nrec; i += kColThreads) {
        recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        hist_hi[b * kColThreads + tid] = static_cast<std::uint32_t>(31 - b) << 16;
        hist_lo[b * kColThreads + tid] = 0u;
    }
    __syncthreads();

    const int cx = tid % g.twc, gy = tid / g.twc;
    const int x = x0 + cx;
    const int ybeg = y0 + gy * g.th;
    if (x >= a.x_hi || ybeg >= a.y_hi) return;
    const int yend = min(ybeg + g.th, a.y_hi);
    std::uint32_t* hh = hist_hi + tid;
    std::uint32_t* hl = hist_lo + tid;
    const std::uint32_t* col = tile + (gy * g.th) * tw + cx;  // window top-left of row ybeg

    for (int dy = 0; dy < w2; ++dy) {
        const std::uint32_t* row = col + dy * tw;
        for (int dx = 0; dx < w2; ++dx) {
            const std::uint32_t e = row[dx];
            const int b = static_cast<int>(e >> 24) * kColThreads;
            hh[b] += col_hi(e);
            hl[b] += col_lo(e);
        }
    }
    std::uint8_t* o = a.out + a.out_frame_stride * frame +
                      static_cast<std::size_t>(ybeg - a.out_row0) * stride + static_cast<std::size_t>(x) * 3;
    for (int y = ybeg;; ++y) {
        // argmax: max count over the bins, then the lowest bin holding it
        // argmax (filter.hpp:71-82): the largest hi word
        std::uint32_t hw[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) hw[b] = hh[b * kColThreads];
#pragma unroll
        for (int step = 1; step < NB; step *= 3) {
#pragma unroll
            for (int i = 0; i + step < NB; i += 3 * step) {
                hw[i] = max(hw[i], hw[i + step]);
                if (i + 2 * step < NB) hw[i] = max(hw[i], hw[i + 2 * step]);
            }
        }
        const std::uint32_t hi32 = hw[0];
        const int best = 31 - static_cast<int>((hi32 >> 16) & 31u);
        const std::uint32_t lo32 = hl[best * kColThreads];
        const std::uint32_t m = recip[hi32 >> 22];  // filter.cpp:41-43
        o[0] = static_cast<std::uint8_t>(__umulhi((hi32 & 0xFFFFu) << 1, m));
        o[1] = static_cast<std::uint8_t>(__umulhi((lo32 >> 16) << 1, m));
        o[2] = static_cast<std::uint8_t>(__umulhi((lo32 & 0xFFFFu) << 1, m));
        if (y + 1 >= yend) break;
        o += stride;
        // slide down one row: remove window row 0, add row w2
        const std::uint32_t* leave = col;
        const std::uint32_t* enter = col + w2 * tw;
        for (int dx = 0; dx < w2; ++dx) {
            const std::uint32_t el = leave[dx], ee = enter[dx];
            const int bl = static_cast<int>(el >> 24) * kColThreads;
            hh[bl] -= col_hi(el);
            hl[bl] -= col_lo(el);
            const int be = static_cast<int>(ee >> 24) * kColThreads;
            hh[be] += col_hi(ee);
            hl[be] += col_lo(ee);
        }
        col += tw;
    }
}

template <int NB>
cudaError_t launch_nb(const BandArgs& a, const ColGeom& g, cudaStream_t s) {
    const std::size_t smem = col_smem_bytes(g, NB, a.radius);
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(column_kernel<NB>), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const unsigned gx = static_cast<unsigned>((a.x_hi - a.x_lo + g.twc - 1) / g.twc);
    const int trows = col_tile_rows(g);
    const dim3 grid(gx, static_cast<unsigned>((a.y_hi - a.y_lo + trows - 1) / trows) + border_grid_rows(a, gx),
                    static_cast<unsigned>(a.frames));
    timing_mark(kIdColumn, 0, s);
    column_kernel<NB><<<grid, kColThreads, smem, s>>>(a, g);
    timing_mark(kIdColumn, 1, s);
    return cudaGetLastError();
}

}  // namespace

bool column_supported(int levels, int radius) {
    return levels >= 1 && levels + 1 <= kColMaxBins && radius >= 0 && radius <= kColMaxR &&
           bin_multiplier(levels) != 0;
}

// Tile shape: rows per thread sized so that the launch is about one round of
// resident blocks (the work per thread then amortises the first window's
// (2r+1)^2 updates over as many rows as the image allows).
cudaError_t launch_column(const BandArgs& a, int num_sms, cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    ColGeom g{};
    g.twc = OPC_COLUMN_TWC;
    const long long iw = a.x_hi - a.x_lo, ih = a.y_hi - a.y_lo;
    const long long threads_per_row = (iw + g.twc - 1) / g.twc * g.twc;
    // target ~ num_sms * OPC_COLUMN_THREADS_PER_SM threads in flight
    const long long want = static_cast<long long>(num_sms) * OPC_COLUMN_THREADS_PER_SM;
    long long th = (threads_per_row * ih * a.frames * 1ll + want - 1) / want;  // rows per thread
    if (OPC_COLUMN_TH > 0) th = OPC_COLUMN_TH;
    g.th = static_cast<int>(std::max(1ll, std::min(64ll, th)));
    const int bins = a.levels + 1;
    if (bins <= 16) return launch_nb<16>(a, g, s);
    if (bins <= 21) return launch_nb<21>(a, g, s);
    if (bins <= 24) return launch_nb<24>(a, g, s);
    return launch_nb<32>(a, g, s);
}

}  // namespace opc
