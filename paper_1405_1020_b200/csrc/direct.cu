// direct.cu -- the generic kernel family (any radius, any L <= 256) and the
// border kernel.
//
// DIRECT: one thread per interior output pixel, the reference's O((2r+1)^2)
// scan restated for the GPU (proj/src/filter.cpp:28-44):
//   pass 1  per-bin counts in shared memory ([bin][thread] layout, so the
//           dynamic-bin increments of a warp hit 32 distinct banks);
//   argmax  lowest index with the strictly largest count (filter.hpp:71-82);
//   pass 2  channel sums of the winning bin only, in registers (u64), then the
//           truncating quotient (filter.cpp:41-43).
// It is the correctness backstop for shapes the fast families do not cover
// (r > 15, or L+1 > 32 at r > 15) and the kernel the tests force to cross-check
// the fast families.
#include "kernels.cuh"
#include "border.cuh"

namespace opc {

namespace {

constexpr int kDirectThreads = 64;

__device__ __forceinline__ unsigned bin_of(unsigned s, int levels, std::uint32_t bin_mul) {
    // filter.hpp:31-35: (r+g+b) * L / 765 in unsigned arithmetic.
    return bin_mul ? __umulhi(s, bin_mul) : (s * static_cast<unsigned>(levels)) / 765u;
}

__global__ void __launch_bounds__(kDirectThreads)
    direct_kernel(BandArgs a, long long pixels_per_frame) {
    extern __shared__ std::uint32_t counts[];  // [bins][kDirectThreads]
    const int tid = threadIdx.x;
    const long long idx = static_cast<long long>(blockIdx.x) * kDirectThreads + tid;
    const int frame = blockIdx.y;
    if (idx >= pixels_per_frame) return;
    const int iw = a.x_hi - a.x_lo;
    const int y = a.y_lo + static_cast<int>(idx / iw);
    const int x = a.x_lo + static_cast<int>(idx % iw);
    const int r = a.radius;
    const int bins = a.levels + 1;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    std::uint8_t* out = a.out + a.out_frame_stride * frame;

    for (int b = 0; b < bins; ++b) counts[b * kDirectThreads + tid] = 0;
    for (int ny = y - r; ny <= y + r; ++ny) {
        const std::uint8_t* p = in + static_cast<std::size_t>(ny - a.in_row0) * stride +
                                static_cast<std::size_t>(x - r) * 3;
        for (int i = 0; i <= 2 * r; ++i, p += 3) {
            const unsigned b = bin_of(unsigned(p[0]) + p[1] + p[2], a.levels, a.bin_mul);
            counts[b * kDirectThreads + tid] += 1;
        }
    }
    int best = 0;
    std::uint32_t best_count = counts[tid];
    for (int b = 1; b < bins; ++b) {
        const std::uint32_t c = counts[b * kDirectThreads + tid];
        if (c > best_count) {  // strict '>' keeps the lowest index on ties
            best_count = c;
            best = b;
        }
    }
    unsigned long long sr = 0, sg = 0, sb = 0;
    for (int ny = y - r; ny <= y + r; ++ny) {
        const std::uint8_t* p = in + static_cast<std::size_t>(ny - a.in_row0) * stride +
                                static_cast<std::size_t>(x - r) * 3;
        for (int i = 0; i <= 2 * r; ++i, p += 3) {
            const unsigned b = bin_of(unsigned(p[0]) + p[1] + p[2], a.levels, a.bin_mul);
            if (b == static_cast<unsigned>(best)) {
                sr += p[0];
                sg += p[1];
                sb += p[2];
            }
        }
    }
    std::uint8_t* o = out + static_cast<std::size_t>(y - a.out_row0) * stride +
                      static_cast<std::size_t>(x) * 3;
    o[0] = static_cast<std::uint8_t>(sr / best_count);
    o[1] = static_cast<std::uint8_t>(sg / best_count);
    o[2] = static_cast<std::uint8_t>(sb / best_count);
}

// Small windows (r <= 3) with few bins (L+1 <= 64): a 32x8 output tile per
// block, its (32+2r) x (8+2r) input pixels loaded once into shared memory as
// entries R | G << 8 | B << 16 | bin << 24 (bin computed once per pixel instead
// of twice per window position), then the same two passes from shared memory.
constexpr int kTileW = 32, kTileH = 8, kTileMaxR = 3, kTileMaxBins = 64;

__global__ void __launch_bounds__(kTileW * kTileH)
    direct_tile_kernel(BandArgs a) {
    __shared__ std::uint32_t tile[(kTileH + 2 * kTileMaxR) * (kTileW + 2 * kTileMaxR)];
    extern __shared__ std::uint32_t counts[];  // [bins][256]
    const int main_rows = (a.y_hi - a.y_lo + kTileH - 1) / kTileH;
    if (static_cast<int>(blockIdx.y) >= main_rows) {  // appended border blocks
        const int b = (blockIdx.y - main_rows) * gridDim.x + blockIdx.x;
        if (b < a.border.nblocks) border_block(a, b, blockIdx.z, threadIdx.y * kTileW + threadIdx.x);
        return;
    }
    const int r = a.radius;
    const int tw = kTileW + 2 * r, th = kTileH + 2 * r;
    const int x0 = a.x_lo + blockIdx.x * kTileW;  // first output column of the tile
    const int y0 = a.y_lo + blockIdx.y * kTileH;
    const int frame = blockIdx.z;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    const int tid = threadIdx.y * kTileW + threadIdx.x;
    for (int i = tid; i < tw * th; i += kTileW * kTileH) {
        const int ty = i / tw, tx = i - ty * tw;
        const int x = min(x0 - r + tx, a.width - 1), y = min(y0 - r + ty, a.in_row0 + a.in_rows - 1);
        const std::uint8_t* p = in + static_cast<std::size_t>(y - a.in_row0) * stride +
                                static_cast<std::size_t>(x) * 3;
        const unsigned R = p[0], G = p[1], B = p[2];
        tile[i] = R | G << 8 | B << 16 | bin_of(R + G + B, a.levels, a.bin_mul) << 24;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= a.x_hi || y >= a.y_hi) return;
    const int bins = a.levels + 1;
    constexpr int T = kTileW * kTileH;
    for (int b = 0; b < bins; ++b) counts[b * T + tid] = 0;
    const int w2 = 2 * r + 1;
    const std::uint32_t* base = tile + threadIdx.y * tw + threadIdx.x;
    for (int dy = 0; dy < w2; ++dy) {
        for (int dx = 0; dx < w2; ++dx) counts[(base[dy * tw + dx] >> 24) * T + tid] += 1;
    }
    unsigned best = 0, best_count = counts[tid];
    for (int b = 1; b < bins; ++b) {
        const unsigned c = counts[b * T + tid];
        if (c > best_count) {  // strict '>' keeps the lowest index on ties (filter.hpp:71-82)
            best_count = c;
            best = b;
        }
    }
    unsigned sr = 0, sg = 0, sb = 0;
    for (int dy = 0; dy < w2; ++dy) {
        for (int dx = 0; dx < w2; ++dx) {
            const std::uint32_t e = base[dy * tw + dx];
            if ((e >> 24) == best) {
                sr += e & 0xFFu;
                sg += (e >> 8) & 0xFFu;
                sb += (e >> 16) & 0xFFu;
            }
        }
    }
    std::uint8_t* o = a.out + a.out_frame_stride * frame +
                      static_cast<std::size_t>(y - a.out_row0) * stride + static_cast<std::size_t>(x) * 3;
    o[0] = static_cast<std::uint8_t>(sr / best_count);  // filter.cpp:41-43
    o[1] = static_cast<std::uint8_t>(sg / best_count);
    o[2] = static_cast<std::uint8_t>(sb / best_count);
}

// Standalone border launch: all blocks on the border job.
__global__ void __launch_bounds__(kBorderThreads) border_kernel(BandArgs a) {
    border_block(a, blockIdx.x, blockIdx.y, threadIdx.x);
}

}  // namespace

std::uint32_t bin_multiplier(int levels) {
    // Smallest-error magic for floor(s*L/765) over s in [0, 765]; verified
    // exhaustively, else 0 (kernels then divide).
    if (levels < 1 || levels > 256) return 0;
    const unsigned long long base =
        ((static_cast<unsigned long long>(levels) << 32) + 764ull) / 765ull;
    for (unsigned long long c = base; c < base + 4 && c <= 0xFFFFFFFFull; ++c) {
        bool ok = true;
        for (unsigned s = 0; s <= 765 && ok; ++s) {
            const unsigned want = s * static_cast<unsigned>(levels) / 765u;
            const unsigned got = static_cast<unsigned>((s * c) >> 32);
            ok = want == got;
        }
        if (ok) return static_cast<std::uint32_t>(c);
    }
    return 0;
}

bool direct_fuses_border(const BandArgs& a) {
    return a.radius <= kTileMaxR && a.levels + 1 <= kTileMaxBins && a.levels <= 255;
}

cudaError_t launch_direct(const BandArgs& a, cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    if (direct_fuses_border(a)) {
        const std::size_t smem = static_cast<std::size_t>(a.levels + 1) * kTileW * kTileH * 4;
        cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(direct_tile_kernel), static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const unsigned gx = static_cast<unsigned>((a.x_hi - a.x_lo + kTileW - 1) / kTileW);
        const dim3 grid(gx, static_cast<unsigned>((a.y_hi - a.y_lo + kTileH - 1) / kTileH) +
                                border_grid_rows(a, gx),
                        static_cast<unsigned>(a.frames));
        timing_mark(kIdDirect, 0, s);
        direct_tile_kernel<<<grid, dim3(kTileW, kTileH), smem, s>>>(a);
        timing_mark(kIdDirect, 1, s);
        return cudaGetLastError();
    }
    const long long pixels = static_cast<long long>(a.y_hi - a.y_lo) * (a.x_hi - a.x_lo);
    const std::size_t smem =
        static_cast<std::size_t>(a.levels + 1) * kDirectThreads * sizeof(std::uint32_t);
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(direct_kernel), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const dim3 grid(static_cast<unsigned>((pixels + kDirectThreads - 1) / kDirectThreads),
                    static_cast<unsigned>(a.frames));
    timing_mark(kIdDirect, 0, s);
    direct_kernel<<<grid, kDirectThreads, smem, s>>>(a, pixels);
    timing_mark(kIdDirect, 1, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_border(a, s);  // 64-thread blocks: the border job runs on its own
}

BorderJob make_border_job(const BandArgs& a, int policy) {
    BorderJob j{};
    j.policy = policy;
    // Full border rows inside this band's output rows.
    const int out_lo = a.y_begin, out_hi = a.y_end;
    j.top_lo = out_lo;
    const int top_hi = out_hi < a.radius ? out_hi : a.radius;
    j.top_rows = top_hi > j.top_lo ? top_hi - j.top_lo : 0;
    j.bot_lo = out_lo > a.height - a.radius ? out_lo : a.height - a.radius;
    j.bot_rows = out_hi > j.bot_lo ? out_hi - j.bot_lo : 0;
    const long long full_bytes = static_cast<long long>(j.top_rows + j.bot_rows) * a.width * 3;
    const int mid_rows = a.y_hi > a.y_lo && a.radius > 0 ? a.y_hi - a.y_lo : 0;
    if (full_bytes <= 0 && mid_rows <= 0) return j;
    long long nfull = (full_bytes + 16 * kBorderThreads - 1) / (16 * kBorderThreads);
    if (nfull > 1184) nfull = 1184;
    j.nfull = static_cast<int>(nfull);
    j.nblocks = j.nfull + (mid_rows + kBorderThreads / 32 - 1) / (kBorderThreads / 32);
    return j;
}

cudaError_t launch_border(const BandArgs& a, cudaStream_t s) {
    if (a.border.nblocks <= 0 || a.frames <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(a.border.nblocks), static_cast<unsigned>(a.frames));
    timing_mark(kIdBorder, 0, s);
    border_kernel<<<grid, kBorderThreads, 0, s>>>(a);
    timing_mark(kIdBorder, 1, s);
    return cudaGetLastError();
}

}  // namespace opc
