// skew.cu -- the performance kernel family for L+1 <= 32 bins and r <= 15.
//
// Algorithm: column-difference sliding window, one output ROW per lane, the 32
// lanes of a warp skewed by one column each (lane t works on virtual column
// v = s - t at step s).  DESIGN.md section 3 has the derivation; in short:
//
//  * The window histogram of lane t (row y) lives in registers as NB packed
//    64-bit words  [count:10 | sumR:18 | sumG:18 | sumB:18]  (exact for
//    (2r+1)^2 <= 1023, i.e. r <= 15; modular packed arithmetic is exact because
//    every window total fits its field).
//  * Sliding right:  W(x+1,y) = W(x,y) + E(x,y),
//        E(x,y) = Col(x+r+1,y) - Col(x-r,y)   (Col = 2r+1-row column histogram).
//    E slots live in shared memory, [bin][slot] layout (conflict-free: lanes
//    always touch distinct slots, the dynamic bin only selects the row).
//  * E(x,y+1) = E(x,y) + f(x+r+1,y+r+1) - f(x+r+1,y-r) - f(x-r,y+r+1) + f(x-r,y-r)
//    -- four dynamic-bin updates.  Lane t reads E(x,y) at step s and advances it
//    to row y+1; lane t+1 consumes it at step s+1.  The skew turns the vertical
//    recurrence into a pipeline across the lanes.
//  * E(x, band top) is built from scratch (2(2r+1) updates per column): at step
//    s lane t < 2r+1 adds row t of column s - t + 2r+1 (one diagonal, one
//    coalesced load; the pixel it removes is the E update's own load b), which
//    finishes each column exactly one step before lane 0 first reads it.
//  * Pixels come from a SHEARED entry plane S[d = x + y][y] written by
//    shear_kernel (u32 = B | R<<8 | G<<18 | bin<<26): every pixel a warp needs
//    at step s lies on one of six anti-diagonals, 32 consecutive rows each, so
//    every access is a single coalesced 128-byte load.
//  * Argmax ("max-scan"): the largest hi word carries the largest count; a scan
//    from the top bin down keeps the last (lowest-index) bin whose count equals
//    it, filter.hpp:71-82.  The conditional copies are predicated IMADs (FMA
//    pipe), the max a tree of 3-input integer max ops (ALU pipe).
//  * Work split: persistent CTAs, equal static shares per warp plus a small
//    dynamic remainder (worksplit.cuh).
//  * Quotient: q = umulhi(2*sum, floor(2^31/c)+1), exact for c <= 1023,
//    sum <= 255c (tests/test_oracle.py checks it exhaustively); filter.cpp:41-43.
//  * Output: a 32x32 staging tile; each step one row completes a 32-pixel
//    block, written as one coalesced 96-byte run.
#include "kernels.cuh"
#include "border.cuh"
#include "tma.cuh"
#include "worksplit.cuh"

#ifndef OPC_SHEAR_TMA
#define OPC_SHEAR_TMA 1  // TMA interior tiles in the shear pre-pass (A/B: profiles/r02_notes.md)
#endif

namespace opc {

namespace {

// == 2 (mod 32): skewed (row t, column s-t) writes hit distinct banks (stride 32 is conflict-free
// too -- bank (s - t) & 31 -- and measured the same: profiles/r02_notes.md)
constexpr int kStageStride = 34;
constexpr int kRecipBytes = 1024 * 4;
constexpr int kShearRows = 32;
constexpr int kShearCols = 128;
// Row stride 132 words: multiple of 4 (16-byte tile stores) and the diagonal
// read address lane * 131 + dd hits 32 distinct banks (131 is odd).
constexpr int kShearStride = kShearCols + 4;
// Zero entries are written for columns [W, W + kShearPad): E columns past the
// last output column (unused values) read up to column W + 32, and a zero
// entry keeps their bin index in range.
constexpr int kShearPad = 64;

// Geometry of the sheared plane for a launch: rows [y_base, y_base + Hs) of
// the image, diagonal d = x + (y - y_base), element (d, y) at d * Hs + (y - y_base).
struct ShearGeom {
    int y_base;
    int Hs;       // multiple of 32
    int ndiag;    // W + kShearPad + Hs
    std::size_t frame_elems;
};

__host__ inline ShearGeom shear_geom(const BandArgs& a) {
    ShearGeom g{};
    g.y_base = a.y_lo - a.radius;
    const int nbands = (a.y_hi - a.y_lo + 63) / 64;  // 64-row bands cover 32-row ones too
    g.Hs = 64 * nbands + 64;
    g.ndiag = a.width + kShearPad + g.Hs;
    g.frame_elems = static_cast<std::size_t>(g.ndiag) * g.Hs;
    return g;
}

// Sheared-plane entry of one pixel: B | R << 8 | G << 18 | bin << 26.  The
// layout is chosen so that the packed 64-bit contribution (count 1, R, G, B)
// costs two ALU ops: lo = e & 0x03FC00FF (B | G << 18) and the byte permute
// R + 2^18, whose x16 is the hi word R << 4 | 1 << 22.
// With `key` (r <= 7, the KEY layout below) the entry is B | R << 8 | G << 16 |
// bin << 24 instead.
__device__ __forceinline__ std::uint32_t make_entry(std::uint32_t r, std::uint32_t g,
                                                    std::uint32_t b, std::uint32_t bin_mul, int key) {
    const std::uint32_t bin = __umulhi(r + g + b, bin_mul);  // filter.hpp:31-35
    return key ? b | (r << 8) | (g << 16) | (bin << 24) : b | (r << 8) | (g << 18) | (bin << 26);
}

// Entry from t = B | R << 8 | G << 16 (byte 3 ignored).
__device__ __forceinline__ std::uint32_t entry_from_brg(std::uint32_t t, std::uint32_t bin_mul, int key) {
    const std::uint32_t bin = __umulhi(__dp4a(t, 0x00010101u, 0u), bin_mul);
    return key ? (t & 0xFFFFFFu) | (bin << 24) : (t & 0xFFFFu) | ((t & 0x00FF0000u) << 2) | (bin << 26);
}

// Sheared entry plane.  Block: 32 rows x 128 columns staged through shared
// memory, then written diagonal by diagonal (lane = row -> contiguous).
// Interior tiles: each thread loads 3 words (4 pixels) per row straight from
// global memory and splits them with byte permutes; row stride 132 words keeps
// both the 16-byte tile stores and the diagonal reads conflict-free.
// TMA (OPC_SHEAR_TMA, A/B in profiles/r02_notes.md): interior tiles arrive as
// one cp.async.bulk.tensor box of 96 words x 32 rows and are split from shared
// memory instead of by 12 __ldg per thread.
template <bool TMA>
__global__ void __launch_bounds__(256)
    shear_kernel(BandArgs a, std::uint32_t* S, ShearGeom g, int vec_ok, int key, std::uint32_t* bmask,
                 const __grid_constant__ CUtensorMap tin) {
    __shared__ __align__(16) std::uint32_t tile[kShearRows * kShearStride];
    if (static_cast<int>(blockIdx.y) >= g.Hs / kShearRows) {  // appended border blocks
        const int b = (blockIdx.y - g.Hs / kShearRows) * gridDim.x + blockIdx.x;
        if (b < a.border.nblocks) border_block(a, b, blockIdx.z, threadIdx.x);
        return;
    }
    const int x0 = blockIdx.x * kShearCols;
    const int y0 = g.y_base + blockIdx.y * kShearRows;
    const int frame = blockIdx.z;
    const std::uint8_t* in = a.in + a.in_frame_stride * frame;
    std::uint32_t* Sf = S + g.frame_elems * frame;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const std::size_t stride = static_cast<std::size_t>(a.width) * 3;
    const int in_hi = a.in_row0 + a.in_rows;
    if (vec_ok && x0 + kShearCols <= a.width && y0 + kShearRows <= in_hi) {
        std::uint32_t w[kShearRows / 8][3];
        if constexpr (TMA) {
            __shared__ __align__(128) std::uint32_t raw[kShearRows * kShearCols * 3 / 4];
            __shared__ std::uint64_t bar;
            if (threadIdx.x == 0) {
                mbar_init(&bar, 1);
                fence_mbar_init();
                mbar_arrive_expect_tx(&bar, sizeof(raw));
                tma_load_3d(raw, &tin, x0 * 3 / 4, y0 - a.in_row0, frame, &bar);
            }
            __syncthreads();
            mbar_wait(&bar, 0);
#pragma unroll
            for (int k = 0; k < kShearRows / 8; ++k) {
#pragma unroll
                for (int q = 0; q < 3; ++q) w[k][q] = raw[(warp + 8 * k) * (kShearCols * 3 / 4) + 3 * lane + q];
            }
        } else {
#pragma unroll
            for (int k = 0; k < kShearRows / 8; ++k) {
                const std::uint32_t* src = reinterpret_cast<const std::uint32_t*>(
                    in + static_cast<std::size_t>(y0 + warp + 8 * k - a.in_row0) * stride +
                    static_cast<std::size_t>(x0) * 3) + 3 * lane;
#pragma unroll
                for (int q = 0; q < 3; ++q) w[k][q] = __ldg(src + q);
            }
        }
#pragma unroll
        for (int k = 0; k < kShearRows / 8; ++k) {
            // bytes R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
            uint4 e;
            e.x = entry_from_brg(__byte_perm(w[k][0], w[k][1], 0x0102), a.bin_mul, key);
            e.y = entry_from_brg(__byte_perm(w[k][0], w[k][1], 0x0435), a.bin_mul, key);
            e.z = entry_from_brg(__byte_perm(w[k][1], w[k][2], 0x0324), a.bin_mul, key);
            e.w = entry_from_brg(__byte_perm(w[k][2], w[k][2], 0x0213), a.bin_mul, key);
            *reinterpret_cast<uint4*>(&tile[(warp + 8 * k) * kShearStride + 4 * lane]) = e;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kShearRows / 8; ++k) {
            const int row = warp + 8 * k;
            const int y = y0 + row;
#pragma unroll
            for (int j = 0; j < kShearCols / 32; ++j) {
                const int c = lane + 32 * j;
                const int x = x0 + c;
                std::uint32_t e = 0;
                if (x < a.width && y < in_hi) {
                    const std::uint8_t* p = in + static_cast<std::size_t>(y - a.in_row0) * stride +
                                            static_cast<std::size_t>(x) * 3;
                    e = make_entry(p[0], p[1], p[2], a.bin_mul, key);
                }
                tile[row * kShearStride + c] = e;
            }
        }
    }
    __syncthreads();
    if (bmask) {
        // Bin masks of the tile's four 32-column blocks (bit b: some pixel of
        // the block has bin b), for the skew kernel's per-phase bin groups:
        // warp w covers block w / 2, rows (w & 1) * 16 .. + 15.
        __shared__ std::uint32_t wm[8];
        const int j = warp >> 1;
        std::uint32_t m = 0;
        // (pixels of the pad columns and of rows past the input are not in
        // any output window: left out)
        const bool col_ok = x0 + 32 * j + lane < a.width;
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const int row = (warp & 1) * 16 + rr;
            const std::uint32_t e = tile[row * kShearStride + 32 * j + lane];
            if (col_ok && y0 + row < in_hi) m |= 1u << (key ? e >> 24 : e >> 26);
        }
        m = __reduce_or_sync(0xFFFFFFFFu, m);
        if (lane == 0) wm[warp] = m;
        __syncthreads();
        if (threadIdx.x < kShearCols / 32) {
            const std::size_t nbx = static_cast<std::size_t>(gridDim.x) * (kShearCols / 32);
            bmask[(static_cast<std::size_t>(frame) * (g.Hs / kShearRows) + blockIdx.y) * nbx +
                  blockIdx.x * (kShearCols / 32) + threadIdx.x] = wm[2 * threadIdx.x] | wm[2 * threadIdx.x + 1];
        }
    }
    // Element (x, y) -> (x + yo) * Hs + yo with yo = y - y_base; for row lane of
    // the tile and diagonal dd = c + lane that is base + dd * Hs.  The grid
    // covers exactly Hs rows, so only the column range needs a check.
    // (32-bit element offsets: skew_fits() bounds the plane of a frame.)
    const int yoff = y0 - g.y_base;
    const std::uint32_t Hs = static_cast<std::uint32_t>(g.Hs);
    std::uint32_t off = static_cast<std::uint32_t>(x0 + yoff + warp) * Hs + yoff + lane;
    const std::uint32_t* src = tile + lane * (kShearStride - 1) + warp;
    const unsigned cmax = static_cast<unsigned>(min(kShearCols, a.width + kShearPad - x0));
    const int c0 = warp - lane;
#pragma unroll
    for (int i = 0; i < (kShearCols + kShearRows + 6) / 8; ++i) {  // dd = warp + 8i <= 158
        const std::uint32_t v = src[8 * i];
        asm volatile(
            "{\n\t.reg .pred p;\n\t.reg .u64 a;\n\tsetp.lt.u32 p, %0, %1;\n\t"
            "mad.wide.u32 a, %2, 4, %3;\n\t@p st.global.u32 [a], %4;\n\t}"
            ::"r"(static_cast<unsigned>(c0 + 8 * i)), "r"(cmax), "r"(off), "l"(Sf), "r"(v)
            : "memory");
        off += 8 * Hs;
    }
}

// ---- packed 64-bit updates ----
// Multipliers come from a kernel argument (Mul) so that ptxas keeps the
// "r1 * 16 + hi (+ carry)" as one IMAD.X on the FMA pipe instead of folding it
// into shifts on the ALU pipe, which is the kernel's binding resource.
struct Mul {
    std::uint32_t m16, negm16, four, one;  // 16, -16, 4, 1
    std::uint32_t r1k;  // entry_r1's constant operand (0x00040000; KEY: 0x01000000)
};

// Packed histogram words.  Default layout (any r <= 15):
//   hi = count << 22 | sumR << 4 | sumG >> 14      lo = sumG << 18 | sumB
// KEY layout (r <= 7: count <= 225, sums < 2^16), the multiplier M.m16 = 1:
//   hi = count << 24 | (31 - bin) << 16 | sumR      lo = sumG << 16 | sumB
// where the window words start at (31 - bin) << 48 (E words carry no key), so
// the largest hi word is the largest count at the lowest bin.
template <bool KEY = false>
__device__ __forceinline__ std::uint32_t entry_lo(std::uint32_t e) {
    return KEY ? __byte_perm(e, 0u, 0x4240) : e & 0x03FC00FFu;  // KEY: B | G << 16
}
#ifndef OPC_SKEW_R1K_ARG
#define OPC_SKEW_R1K_ARG 1
#endif
// (the constant operand comes from the kernel argument M.r1k: the selector is
// then PRMT's immediate and no per-use register copy of a constant is needed)
template <bool KEY = false>
__device__ __forceinline__ std::uint32_t entry_r1(std::uint32_t e, std::uint32_t r1k) {
    // default: R + 2^18 (x16 = R << 4 | 1 << 22); KEY: R | 1 << 24 (x1)
    if (!OPC_SKEW_R1K_ARG) r1k = KEY ? 0x01000000u : 0x00040000u;
    return KEY ? __byte_perm(e, r1k, 0x7541) : __byte_perm(e, r1k, 0x7641);
}
template <bool KEY = false>
__device__ __forceinline__ std::uint32_t entry_bin(std::uint32_t e) { return KEY ? e >> 24 : e >> 26; }

// w + (r1 * mul) << 32 | lo   (64-bit, carry from the low word)
__device__ __forceinline__ unsigned long long packed_plus(unsigned long long w, std::uint32_t lo,
                                                          std::uint32_t r1, std::uint32_t mul) {
    std::uint32_t wl, wh;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(wl), "=r"(wh) : "l"(w));
    asm("add.cc.u32 %0, %0, %2;\n\tmadc.lo.u32 %1, %3, %4, %1;"
        : "+r"(wl), "+r"(wh) : "r"(lo), "r"(r1), "r"(mul));
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(wl), "r"(wh));
    return r;
}
// w - (r1 * 16) << 32 | lo
__device__ __forceinline__ unsigned long long packed_minus(unsigned long long w, std::uint32_t lo,
                                                           std::uint32_t r1, std::uint32_t negmul) {
    std::uint32_t wl, wh;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(wl), "=r"(wh) : "l"(w));
    // wl - lo with borrow; hi - 16*r1 - borrow == hi + (-16)*r1 - borrow
    asm("sub.cc.u32 %0, %0, %2;\n\tsubc.u32 %1, %1, 0;\n\tmad.lo.u32 %1, %3, %4, %1;"
        : "+r"(wl), "+r"(wh) : "r"(lo), "r"(r1), "r"(negmul));
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(wl), "r"(wh));
    return r;
}
__device__ __forceinline__ void packed_add(unsigned long long* p, std::uint32_t lo, std::uint32_t r1,
                                           std::uint32_t mul) {
    *p = packed_plus(*p, lo, r1, mul);
}
__device__ __forceinline__ void packed_sub(unsigned long long* p, std::uint32_t lo, std::uint32_t r1,
                                           std::uint32_t negmul) {
    *p = packed_minus(*p, lo, r1, negmul);
}

// E[bin(e)][slot] += / -= packed(e).  Es = E + slot, SL slots per bin row.
template <int SL, bool KEY = false>
__device__ __forceinline__ void rmw_add(unsigned long long* Es, std::uint32_t e, const Mul& M) {
    packed_add(Es + entry_bin<KEY>(e) * SL, entry_lo<KEY>(e), entry_r1<KEY>(e, M.r1k), M.m16);
}
template <int SL, bool KEY = false>
__device__ __forceinline__ void rmw_sub(unsigned long long* Es, std::uint32_t e, const Mul& M) {
    packed_sub(Es + entry_bin<KEY>(e) * SL, entry_lo<KEY>(e), entry_r1<KEY>(e, M.r1k), M.negm16);
}

// Masked forms (all lanes execute; lanes with mask 0 add zero): lo & mask,
// multiplier m16 = 16 & mask or nm16 = -16 & mask.
template <int SL, bool KEY = false>
__device__ __forceinline__ void rmw_add_m(unsigned long long* Es, std::uint32_t e, std::uint32_t mask,
                                          std::uint32_t m16, const Mul& M) {
    packed_add(Es + entry_bin<KEY>(e) * SL, entry_lo<KEY>(e) & mask, entry_r1<KEY>(e, M.r1k), m16);
}
template <int SL, bool KEY = false>
__device__ __forceinline__ void rmw_sub_m(unsigned long long* Es, std::uint32_t e, std::uint32_t mask,
                                          std::uint32_t nm16, const Mul& M) {
    packed_sub(Es + entry_bin<KEY>(e) * SL, entry_lo<KEY>(e) & mask, entry_r1<KEY>(e, M.r1k), nm16);
}

// Lowest-index bin with the largest count (filter.hpp:71-82) and its truncated
// channel averages (filter.cpp:41-43), packed R | G << 8 | B << 16.
// (A static tournament, FMA-pipe selects in its first level, and 3/4/7
// parallel scan groups were measured slower than the max-scan below:
// profiles/r01_notes.md.)

// Conditional copy on the FMA pipe: if (p) d = a * one (one = 1 at run time,
// so ptxas cannot turn the predicated IMAD into an ALU select).
__device__ __forceinline__ void pick_if_ge(std::uint32_t& lo, std::uint32_t& hi, std::uint32_t bl,
                                           std::uint32_t bh, std::uint32_t T, std::uint32_t one) {
    asm("{\n\t.reg .pred p;\n\tsetp.ge.u32 p, %3, %4;\n\t"
        "@p mad.lo.u32 %0, %2, %5, 0;\n\t@p mad.lo.u32 %1, %3, %5, 0;\n\t}"
        : "+r"(lo), "+r"(hi)
        : "r"(bl), "r"(bh), "r"(T), "r"(one));
}

// KEY layout: the largest hi word (a max tree) is the winner's hi word; its
// (31 - bin) field selects the lo word through a 5-level multiplexer.
template <int NB>
__device__ __forceinline__ std::uint32_t winner_rgb_key(const unsigned long long (&w)[NB],
                                                        const std::uint32_t* recip, int base = 0) {
    std::uint32_t mx[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) mx[b] = static_cast<std::uint32_t>(w[b] >> 32);
#pragma unroll
    for (int step = 1; step < NB; step *= 3) {
#pragma unroll
        for (int i = 0; i + step < NB; i += 3 * step) {
            mx[i] = max(mx[i], mx[i + step]);
            if (i + 2 * step < NB) mx[i] = max(mx[i], mx[i + 2 * step]);
        }
    }
    const std::uint32_t hi = mx[0];
    const std::uint32_t best = 31u - ((hi >> 16) & 31u) - static_cast<std::uint32_t>(base);
    std::uint32_t v[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) v[b] = static_cast<std::uint32_t>(w[b]);
#pragma unroll
    for (int k = 0; (1 << k) < NB; ++k) {
        const bool bit = (best >> k) & 1u;
#pragma unroll
        for (int i = 0; i + (1 << k) < NB; i += 2 << k) v[i] = bit ? v[i + (1 << k)] : v[i];
    }
    const std::uint32_t lo = v[0];
    const std::uint32_t m = recip[hi >> 24];
    const std::uint32_t qr = __umulhi((hi & 0xFFFFu) << 1, m);
    const std::uint32_t qg = __umulhi((lo >> 16) << 1, m);
    const std::uint32_t qb = __umulhi((lo & 0xFFFFu) << 1, m);
    return qr | (qg << 8) | (qb << 16);
}

template <int NB>
__device__ __forceinline__ std::uint32_t winner_rgb(const unsigned long long (&w)[NB],
                                                    const std::uint32_t* recip, std::uint32_t one) {
    // Max-scan: the largest hi word carries the largest count c* (its low 22
    // bits are sums, irrelevant to the count).  T = c* << 22; then a scan from
    // the top bin down keeps the last (= lowest-index) bin with hi >= T, i.e.
    // count == c*.  The max is an ALU min/max tree (balanced: short dependency
    // chains); the conditional copies are predicated IMADs on the FMA pipe,
    // which has the spare issue slots.
    std::uint32_t mx[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) mx[b] = static_cast<std::uint32_t>(w[b] >> 32);
#pragma unroll
    for (int step = 1; step < NB; step *= 3) {
#pragma unroll
        for (int i = 0; i + step < NB; i += 3 * step) {
            mx[i] = max(mx[i], mx[i + step]);
            if (i + 2 * step < NB) mx[i] = max(mx[i], mx[i + 2 * step]);
        }
    }
    const std::uint32_t T = mx[0] & 0xFFC00000u;
    std::uint32_t lo = static_cast<std::uint32_t>(w[NB - 1]);
    std::uint32_t hi = static_cast<std::uint32_t>(w[NB - 1] >> 32);
#pragma unroll
    for (int b = NB - 2; b >= 0; --b) {
        pick_if_ge(lo, hi, static_cast<std::uint32_t>(w[b]), static_cast<std::uint32_t>(w[b] >> 32), T, one);
    }
    const std::uint32_t count = hi >> 22;
    const std::uint32_t m = recip[count];
    const std::uint32_t sr = (hi >> 4) & 0x3FFFFu;
    const std::uint32_t sg = (lo >> 18) | ((hi & 0xFu) << 14);
    const std::uint32_t sb = lo & 0x3FFFFu;
    const std::uint32_t qr = __umulhi(sr << 1, m);
    const std::uint32_t qg = __umulhi(sg << 1, m);
    const std::uint32_t qb = __umulhi(sb << 1, m);
    return qr | (qg << 8) | (qb << 16);
}


// E ring.  The init of column c adds its rows k < w2 at steps c - w2 .. c - 1
// (lane t adds row t of column s - t + w2 at step s), and
// lane 31 reads it last at step c + 31: a column lives 32 + w2 steps.  Slots
// are cleared kBatch at a time (conflict-free) at the end of every step
// s = -1 mod kBatch: columns s + 1 + w2 .. s + kBatch + w2, whose previous
// occupants (c - SL) were last read by step s - 1 when SL >= kBatch + w2 + 32.
//   r <= 7  (w2 <= 16): 64 slots, batches of 16 (used for NB >= 24: config 5 fits 11 warps/SM)
//   r <= 15 (w2 <= 31): 96 slots, batches of 32
#ifndef OPC_SKEW_SL_LARGE
#define OPC_SKEW_SL_LARGE 96  // ring for w2 > 16; 80 (batches of 16, 12 warps/SM) measured 2.6% slower on C4
#endif
template <int SL>
struct Ring {
    static constexpr int kBatch = (SL == 64 || SL == 80) ? 16 : 32;
    static constexpr int kLanes = 32 / kBatch;  // bins cleared per column per store
};
#ifndef OPC_SKEW_LOOKAHEAD
#define OPC_SKEW_LOOKAHEAD 3  // steps between a step's global loads and their use (NB <= 21)
#endif
#ifndef OPC_SKEW_LOOK3_MAXNB
#define OPC_SKEW_LOOK3_MAXNB 21  // bins up to which loads run 3 steps ahead (registers)
#endif
#ifndef OPC_SKEW_HOIST_INIT
#define OPC_SKEW_HOIST_INIT 1
#endif
#ifndef OPC_SKEW_PF_DIST
#define OPC_SKEW_PF_DIST 8  // L2 prefetch distance (steps) of the init diagonal; 0 = off
#endif
#ifndef OPC_SKEW_STATIC_PCT
#define OPC_SKEW_STATIC_PCT 98  // 90-100 within 2% on C4; C5 best at 97-100
#endif
#ifndef OPC_SKEW_STATIC_PCT_SMALL
#define OPC_SKEW_STATIC_PCT_SMALL 99
#endif
#ifndef OPC_SKEW_SMALL_SHARE
#define OPC_SKEW_SMALL_SHARE 4000  // band columns per resident warp below which the small-share split applies
#endif
#ifndef OPC_SKEW_ALIGNED
#define OPC_SKEW_ALIGNED 1  // band-aligned one-pass-per-warp split for small shares
#endif
#ifndef OPC_SKEW_MIN_CHUNK
#define OPC_SKEW_MIN_CHUNK 128
#endif
#ifndef OPC_SKEW_KEY
#define OPC_SKEW_KEY 1  // KEY histogram layout for r <= 7 (the SPARSE launches)
#endif
#ifndef OPC_SKEW_MAX_WARPS
#define OPC_SKEW_MAX_WARPS 12
#endif
constexpr int kMaxWarps = OPC_SKEW_MAX_WARPS;  // 12: <= 170 registers per thread

template <int NB, int SL>
__host__ __device__ inline std::size_t per_warp_bytes() {
    return static_cast<std::size_t>(NB) * SL * 8 + 32 * kStageStride * 4;
}

struct Loads {
    std::uint32_t a, b, c, d;  // E update: entering / leaving rows of the two columns
    std::uint32_t i1;          // init: row t of column s - t + w2 (its leaving pixel is b)
};

struct Task {
    Mul M;
    std::uint32_t imask, im16, inm16;  // per lane: t < w2 ? (~0, 16, -16) : 0 (masked init)
    const std::uint32_t* Sf;  // sheared plane of this frame
    std::uint32_t o0;         // element offset of diagonal D0 (ring column 0), ring row 0
    std::uint32_t Hs;         // elements per diagonal
    std::uint32_t dA, dD, dI;  // w2*Hs + w2, w2*Hs, w2*Hs
    std::uint8_t* out_row0;   // output row yb (band row 0), column 0
    int NV, X0, w2, lane;
    int y_rows;               // valid rows in the band (<= 32)
    std::size_t stride;
    std::uint32_t stride32;   // row stride in bytes (32 rows of it fit 32 bits)
    std::uint32_t gm;         // bin groups (8 bins each) the current phase touches (GROUPED steps)
    int base;                 // windowed passes: bin of win[0]
};
#ifndef OPC_SKEW_WINDOW
#define OPC_SKEW_WINDOW 16  // KEY launches with NB >= 24: window of bins kept per pass when every phase fits (0 = off)
#endif
#ifndef OPC_SKEW_GROUPS
#define OPC_SKEW_GROUPS 1  // KEY launches with NB >= 24: skip the E rows of bin groups a phase never sees
#endif
#ifndef OPC_SKEW_GROUPS_MIN_NB
#define OPC_SKEW_GROUPS_MIN_NB 24
#endif
#ifndef OPC_SKEW_WINDOW_MIN_NB
#define OPC_SKEW_WINDOW_MIN_NB 24
#endif
#ifndef OPC_SKEW_GROUP_BINS
#define OPC_SKEW_GROUP_BINS 8  // bins per group (4, 8 or 16)
#endif

#ifndef OPC_SKEW_LDOFF_IMM
#define OPC_SKEW_LDOFF_IMM 1  // r > 7 launches (C4 -1.1%); the SPARSE launches keep the runtime multiplier (C5 +0.8% with it)
#endif
// 32-bit element offset from a 64-bit base.  IMM: immediate multiplier 4
// (ptxas emits LEA + LEA.HI.X); otherwise the runtime multiplier four = 4
// (IMAD.WIDE + IADD3 + IADD3.X: one op more, but one of them on the FMA pipe).
template <bool IMM>
__device__ __forceinline__ std::uint32_t ld_off(const std::uint32_t* base, std::uint32_t off,
                                                std::uint32_t four) {
    std::uint32_t v;
    if constexpr (IMM) {
        asm volatile(
            "{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %1, 4, %2;\n\tld.global.nc.u32 %0, [a];\n\t}"
            : "=r"(v)
            : "r"(off), "l"(base));
    } else {
        asm volatile(
            "{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %1, %2, %3;\n\tld.global.nc.u32 %0, [a];\n\t}"
            : "=r"(v)
            : "r"(off), "r"(four), "l"(base));
    }
    return v;
}

// Loads of step s.  Ring column c, ring row rho live at offset
// o0 + (c + rho) * Hs + rho, so every access of a step is on diagonal D0 + s
// (+ a step-independent shift), 32 consecutive rows per access.
template <bool EDGE, bool SPARSE>
__device__ __forceinline__ Loads fetch(const Task& T, int s) {
    constexpr bool IMM = OPC_SKEW_LDOFF_IMM && !SPARSE;
    Loads L;
    const int t = T.lane;
    const int w2 = T.w2;
    const std::uint32_t ob = T.o0 + static_cast<std::uint32_t>(s) * T.Hs + t;  // diag D0+s, row t
    const std::uint32_t four = T.M.four;
    const int v = s - t;
    L.a = L.b = L.c = L.d = 0;
    if (!EDGE || (v >= 0 && v < T.NV)) {
        L.a = ld_off<IMM>(T.Sf, ob + T.dA, four);  // new row t+w2, entering column
        L.b = ld_off<IMM>(T.Sf, ob, four);         // old row t, entering column
        if (!EDGE || v >= w2) {
            L.c = ld_off<IMM>(T.Sf, ob + w2, four);     // new row, leaving column
            L.d = ld_off<IMM>(T.Sf, ob - T.dD, four);   // old row, leaving column
        }
    }
    // Init (lanes t < w2): row t of column vi = s - t + w2, i.e. diagonal
    // s + w2, row t; its leaving pixel (column vi - w2 = v, row t) is b.
    const int vi = s - t + w2;
    L.i1 = 0;
    if (!EDGE || (t < w2 && vi >= 0 && vi < T.NV)) L.i1 = ld_off<IMM>(T.Sf, ob + T.dI, four);
    return L;
}

// L2 prefetch of the band rows of the diagonal the init reads at step s.
__device__ __forceinline__ void prefetch_l2(const Task& T, int s) {
    const std::uint32_t o = T.o0 + static_cast<std::uint32_t>(s) * T.Hs + T.dI + T.lane;
    const std::uint32_t* p = T.Sf + o;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + 32));
}

// SPARSE: lanes t >= w2 skip the init (a branch; small windows, where the
// active lanes fit one half-warp and the init accesses take half the
// shared-memory wavefronts); otherwise all lanes run it masked (no divergence;
// measured 13% faster for r = 15).
template <int NB, int SL, bool SPARSE, bool EDGE, int NW = NB>
__device__ __forceinline__ void step(const Task& T, int s, const Loads& cur,
                                     unsigned long long (&win)[NW], unsigned long long* E,
                                     std::uint32_t* stage, const std::uint32_t* recip) {
    constexpr bool KEY = SPARSE && OPC_SKEW_KEY;
    const int t = T.lane;
    const int w2 = T.w2;
    const int v = s - t;
    // Steady steps: the two init targets (slot of column v + w2, never the E
    // update's slot) are read before the E update chain and written after it,
    // so the two read-modify-write chains overlap instead of queueing.
    const int vi = s - t + w2;
    const int islot = static_cast<unsigned>(vi) % SL;
    unsigned long long* ip1 = E + islot + entry_bin<KEY>(cur.i1) * SL;
    unsigned long long* ip2 = E + islot + entry_bin<KEY>(cur.b) * SL;
    unsigned long long iold1 = 0, iold2 = 0;
    // (Only lanes t < w2 touch them: a lane t >= w2 would address the slot of
    // column s - t + w2 >= s - 31 + w2, which another lane updates in between.)
    constexpr bool kHoist = !EDGE && SPARSE && OPC_SKEW_HOIST_INIT;  // (r = 15: 1.8% slower)
    if (kHoist && t < w2) {
        iold1 = *ip1;
        iold2 = *ip2;
    }
    if (!EDGE || (v >= 0 && v < T.NV)) {
        const int slot = static_cast<unsigned>(v) % SL;
        // GROUPED: E rows of bin groups the phase's pixels never reach are
        // zero for every column of the phase: neither read nor added (the
        // winner first, then each active group's rows loaded and added).
        constexpr bool WIN = NW < NB;  // windowed pass: win[k] is bin T.base + k
        constexpr bool GROUPED = KEY && NB >= OPC_SKEW_GROUPS_MIN_NB && OPC_SKEW_GROUPS && !EDGE && !WIN;
        if constexpr (WIN) {
            unsigned long long e[NW];
            const unsigned long long* Eb = E + T.base * SL + slot;
#pragma unroll
            for (int k = 0; k < NW; ++k) e[k] = Eb[k * SL];
            if (!EDGE || (v >= w2 && t < T.y_rows)) {
                stage[t * kStageStride + (v & 31)] = winner_rgb_key<NW>(win, recip, T.base);
            }
#pragma unroll
            for (int k = 0; k < NW; ++k) win[k] += e[k];
        } else if constexpr (GROUPED) {
            stage[t * kStageStride + (v & 31)] = winner_rgb_key<NB>(win, recip);
            constexpr int GS = OPC_SKEW_GROUP_BINS;
#pragma unroll
            for (int g8 = 0; g8 < (NB + GS - 1) / GS; ++g8) {
                if ((T.gm >> g8) & 1u) {
                    unsigned long long e[GS];
#pragma unroll
                    for (int b = GS * g8; b < NB && b < GS * g8 + GS; ++b) e[b - GS * g8] = E[b * SL + slot];
#pragma unroll
                    for (int b = GS * g8; b < NB && b < GS * g8 + GS; ++b) win[b] += e[b - GS * g8];
                }
            }
        } else {
            unsigned long long e[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) e[b] = E[b * SL + slot];
            if (!EDGE || (v >= w2 && t < T.y_rows)) {
                stage[t * kStageStride + (v & 31)] =
                    KEY ? winner_rgb_key<NB>(win, recip) : winner_rgb<NB>(win, recip, T.M.one);
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) win[b] += e[b];
        }
        // Advance E(v) from row t to row t + 1 (lane t + 1 reads it next step).
        unsigned long long* Es = E + slot;
        rmw_add<SL, KEY>(Es, cur.a, T.M);
        rmw_sub<SL, KEY>(Es, cur.b, T.M);
        if (!EDGE || v >= w2) {
            rmw_sub<SL, KEY>(Es, cur.c, T.M);
            rmw_add<SL, KEY>(Es, cur.d, T.M);
        }
    }
    {  // one row of the from-scratch build of E(vi, band top): lane t adds row t
        if (kHoist) {
            const unsigned long long n1 =
                packed_plus(iold1, entry_lo<KEY>(cur.i1), entry_r1<KEY>(cur.i1, T.M.r1k), T.M.m16);
            // (both in one bin: one word, the second update applies to n1)
            const unsigned long long n2 =
                packed_minus(ip1 == ip2 ? n1 : iold2, entry_lo<KEY>(cur.b), entry_r1<KEY>(cur.b, T.M.r1k), T.M.negm16);
            if (t < w2) {
                *ip1 = n1;
                *ip2 = n2;
            }
        } else if (EDGE) {
            if (t < w2 && vi >= 0 && vi < T.NV) {
                rmw_add<SL, KEY>(E + islot, cur.i1, T.M);
                if (vi >= w2) rmw_sub<SL, KEY>(E + islot, cur.b, T.M);
            }
        } else if (SPARSE) {
            if (t < w2) {  // (a per-lane constant)
                rmw_add<SL, KEY>(E + islot, cur.i1, T.M);
                rmw_sub<SL, KEY>(E + islot, cur.b, T.M);
            }
        } else {
            rmw_add_m<SL, KEY>(E + islot, cur.i1, T.imask, T.im16, T.M);
            rmw_sub_m<SL, KEY>(E + islot, cur.b, T.imask, T.inm16, T.M);
        }
    }
    __syncwarp();
    // Row fr just completed the 32-column block ending at v = s - fr.
    const int fr = (s + 1) & 31;
    const int vv = s - fr - 31 + t;
    if (fr < T.y_rows && (!EDGE || (vv >= w2 && vv < T.NV))) {
        const std::uint32_t rgb = stage[fr * kStageStride + t];
        // 32-bit byte offset within the band's 32 rows (skew_fits(): W < 2^25,
        // so 32 rows x 3W bytes < 2^32)
        const std::uint32_t ob = static_cast<std::uint32_t>(fr) * T.stride32 +
                                 static_cast<std::uint32_t>(T.X0 + vv) * 3u;
        std::uint8_t* o = T.out_row0 + ob;
        o[0] = static_cast<std::uint8_t>(rgb);
        o[1] = static_cast<std::uint8_t>(rgb >> 8);
        o[2] = static_cast<std::uint8_t>(rgb >> 16);
    }
    constexpr int B = Ring<SL>::kBatch;
    if ((s & (B - 1)) == B - 1) {  // clear the slots of columns s + 1 + w2 .. s + B + w2
        const int zs = static_cast<unsigned>(s + 1 + w2 + (t & (B - 1))) % SL;
#pragma unroll
        for (int j = 0; j < (NB + Ring<SL>::kLanes - 1) / Ring<SL>::kLanes; ++j) {
            const int b = Ring<SL>::kLanes * j + t / B;
            if (b < NB) E[b * SL + zs] = 0ull;
        }
    }
    __syncwarp();
}

// Bin groups (8 bins each) the pixels of a steady phase can contribute to:
// the lanes' E columns v in [s0 - 31, s0 + 31] hold column histograms of image
// columns [xs - r + v - w2, xs - r + v], rows [yb - r, yb + 31 + r]; the OR of
// the shear pre-pass's 32 x 32 block bin masks over that region.
__device__ __forceinline__ std::uint32_t phase_bins(const BandArgs& a, const ShearGeom& sg,
                                                    const std::uint32_t* bmask, int f, int yb, int xs,
                                                    int s0, int w2, int lane) {
    const int r = a.radius;
    const int nty = sg.Hs / kShearRows;
    const int nbx = (a.width + kShearPad + kShearCols - 1) / kShearCols * (kShearCols / 32);
    const int ty0 = (yb - r - sg.y_base) >> 5;
    const int ty1 = min(nty - 1, (yb + 31 + r - sg.y_base) >> 5);
    const int c0 = max(0, xs - r + s0 - 31 - w2);
    const int c1 = min(a.width - 1, xs - r + s0 + 31);
    if (c1 < c0) return 0u;  // no image column in the phase yet
    const int bx0 = c0 >> 5, bx1 = max(bx0, c1 >> 5);
    const int nx = bx1 - bx0 + 1;
    std::uint32_t m = 0;
    if (lane < (ty1 - ty0 + 1) * nx) {
        const int ty = ty0 + lane / nx, bx = bx0 + lane % nx;
        m = bmask[(static_cast<std::size_t>(f) * nty + ty) * nbx + bx];
    }
    return __reduce_or_sync(0xFFFFFFFFu, m);
}
__device__ __forceinline__ std::uint32_t phase_groups(const BandArgs& a, const ShearGeom& sg,
                                                      const std::uint32_t* bmask, int f, int yb, int xs,
                                                      int s0, int w2, int lane) {
    const std::uint32_t m = phase_bins(a, sg, bmask, f, yb, xs, s0, w2, lane);
    constexpr int GS = OPC_SKEW_GROUP_BINS;
    constexpr std::uint32_t gmask = (1u << GS) - 1u;
    std::uint32_t gm = 0;
#pragma unroll
    for (int g8 = 0; g8 < 32 / GS; ++g8) gm |= ((m >> (GS * g8)) & gmask) ? 1u << g8 : 0u;
    return gm;
}

// One pass (band kb of frame f, columns [0, NV)) of a warp; Task set up by the
// caller.  NW < NB: windowed pass (KEY layout) -- win[k] holds bin T.base + k.
template <int NB, int SL, bool SPARSE, int NW>
__device__ __forceinline__ void run_pass(Task& T, const BandArgs& a, const ShearGeom& sg,
                                         const std::uint32_t* bmask, int f, int yb, int xs,
                                         unsigned long long* E, std::uint32_t* stage,
                                         const std::uint32_t* recip, int base0) {
    constexpr bool WIN = NW < NB;
    unsigned long long win[NW];
    if constexpr (WIN) T.base = base0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const int b = (WIN ? base0 : 0) + k;
        win[k] = (SPARSE && OPC_SKEW_KEY) ? static_cast<unsigned long long>(31 - b) << 48 : 0ull;
    }
    for (int i = T.lane; i < NB * SL; i += 32) E[i] = 0ull;
    __syncwarp();

    const int nphases = ((T.NV - 1) >> 5) + 2;
    // steady: every lane past warm-up and every flushed column valid
    // From phase p on every step is steady: all lanes past warm-up
    // (s - 31 >= w2 from s = 32p) and every flushed column valid
    // (32p - 32 >= w2): 32p >= w2 + 32.
    const int p_steady_lo = (T.w2 + 32 + 31) >> 5;
    // The first init row (column 0, lane 0) is added at step -w2: phase -1
    // starts there.  (Slots the skipped steps would clear are still zero.)
    Loads cur = fetch<true, SPARSE>(T, -T.w2);
    for (int p = -1; p < nphases; ++p) {
        if constexpr (WIN) {
            // keep the phase's bins inside the window [base, base + NW): the
            // pass was admitted because every phase's range fits; words
            // shifted out hold no pixel (the phase region contains every
            // lane's window)
            const std::uint32_t m = phase_bins(a, sg, bmask, f, yb, xs, 32 * p, T.w2, T.lane);
            if (m) {
                const int lo = __ffs(m) - 1, hi = 31 - __clz(m);
                if (lo < T.base || hi >= T.base + NW) {
                    int nb = lo - (NW - (hi - lo + 1)) / 2;
                    nb = max(0, min(nb, NB - NW));
                    while (T.base < nb) {
#pragma unroll
                        for (int k = 0; k + 1 < NW; ++k) win[k] = win[k + 1];
                        win[NW - 1] = static_cast<unsigned long long>(31 - (T.base + NW)) << 48;
                        ++T.base;
                    }
                    while (T.base > nb) {
#pragma unroll
                        for (int k = NW - 1; k > 0; --k) win[k] = win[k - 1];
                        win[0] = static_cast<unsigned long long>(31 - (T.base - 1)) << 48;
                        --T.base;
                    }
                }
            }
        }
        // (A partial last band runs the steady path too: its rows past
        // y_rows read valid plane rows and are never flushed.)
        const bool steady = p >= p_steady_lo && 32 * p + 31 < T.NV;
        if (steady) {
            if constexpr (!WIN && SPARSE && OPC_SKEW_KEY && NB >= OPC_SKEW_GROUPS_MIN_NB && OPC_SKEW_GROUPS) {
                T.gm = phase_groups(a, sg, bmask, f, yb, xs, 32 * p, T.w2, T.lane);
            }
            // Loads run two steps ahead; the diagonal first touched eight
            // steps ahead (the init column's) is pulled into L2 now.
            // Global loads run kLook steps ahead of their use (3 for NB <= 21:
            // 1% faster on C4; 2 for more bins, where the registers run out).
            constexpr int kLook = NB <= OPC_SKEW_LOOK3_MAXNB ? OPC_SKEW_LOOKAHEAD : 2;
            Loads n1 = fetch<false, SPARSE>(T, 32 * p + 1);
            Loads n2{};
            if constexpr (kLook >= 3) n2 = fetch<false, SPARSE>(T, 32 * p + 2);
#pragma unroll 1
            for (int ss = 0; ss < 32; ss += 2) {
                const int s = 32 * p + ss;
                if (OPC_SKEW_PF_DIST > 0) prefetch_l2(T, s + OPC_SKEW_PF_DIST);
                if constexpr (kLook >= 3) {
                    const Loads n3 = fetch<false, SPARSE>(T, s + 3);
                    step<NB, SL, SPARSE, false, NW>(T, s, cur, win, E, stage, recip);
                    if (OPC_SKEW_PF_DIST > 0) prefetch_l2(T, s + OPC_SKEW_PF_DIST + 1);
                    const Loads n4 = fetch<false, SPARSE>(T, s + 4);
                    step<NB, SL, SPARSE, false, NW>(T, s + 1, n1, win, E, stage, recip);
                    cur = n2;
                    n1 = n3;
                    n2 = n4;
                } else {
                    const Loads m2 = fetch<false, SPARSE>(T, s + 2);
                    step<NB, SL, SPARSE, false, NW>(T, s, cur, win, E, stage, recip);
                    if (OPC_SKEW_PF_DIST > 0) prefetch_l2(T, s + OPC_SKEW_PF_DIST + 1);
                    const Loads m3 = fetch<false, SPARSE>(T, s + 3);
                    step<NB, SL, SPARSE, false, NW>(T, s + 1, n1, win, E, stage, recip);
                    cur = m2;
                    n1 = m3;
                }
            }
        } else {
#pragma unroll 1
            for (int ss = p < 0 ? 32 - T.w2 : 0; ss < 32; ++ss) {
                const int s = 32 * p + ss;
                const Loads nxt = fetch<true, SPARSE>(T, s + 1);
                step<NB, SL, SPARSE, true, NW>(T, s, cur, win, E, stage, recip);
                cur = nxt;
            }
        }
    }
}

template <int NB, int SL, bool SPARSE>
__global__ void __launch_bounds__(kMaxWarps * 32)
    skew_kernel(BandArgs a, const std::uint32_t* __restrict__ S, ShearGeom sg, int* task_counter,
                WorkSplit g, Mul M, const std::uint32_t* __restrict__ bmask) {
    extern __shared__ __align__(16) unsigned char smem[];
    std::uint32_t* recip = reinterpret_cast<std::uint32_t*>(smem);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int r = a.radius;
    unsigned char* wbase = smem + kRecipBytes + warp * per_warp_bytes<NB, SL>();
    unsigned long long* E = reinterpret_cast<unsigned long long*>(wbase);
    std::uint32_t* stage = reinterpret_cast<std::uint32_t*>(wbase + std::size_t(NB) * SL * 8);

    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
    __syncthreads();

    Task T;
    T.M = M;
    T.Hs = static_cast<std::uint32_t>(sg.Hs);
    T.w2 = 2 * r + 1;
    T.dA = T.w2 * T.Hs + T.w2;
    T.dD = T.w2 * T.Hs;
    T.dI = T.w2 * T.Hs;
    T.lane = lane;
    T.stride = static_cast<std::size_t>(a.width) * 3;
    T.stride32 = static_cast<std::uint32_t>(T.stride);
    T.imask = lane < T.w2 ? ~0u : 0u;
    T.im16 = T.imask & M.m16;
    T.inm16 = T.imask & M.negm16;

    long long u = 0, u_end = 0;  // unprocessed units of the current chunk
    int f, kb, x0, x1;
    while (next_pass(g, task_counter, lane, u, u_end, f, kb, x0, x1)) {
        const int yb = a.y_lo + 32 * kb;
        const int xs = a.x_lo + x0;
        const int xe = a.x_lo + x1;
        T.NV = T.w2 + (xe - xs);  // virtual columns: w2 warm-up + outputs
        T.X0 = xs - T.w2;         // image column of virtual column 0
        T.y_rows = min(32, a.y_hi - yb);
        T.out_row0 = a.out + a.out_frame_stride * f +
                     static_cast<std::size_t>(yb - a.out_row0) * T.stride;
        // ring column c = image column xs - r + c, ring row rho = image row yb - r + rho;
        // element (d, y) of the plane at d * Hs + (y - y_base), d = x + (y - y_base).
        const int R0 = yb - r - sg.y_base;
        const std::uint32_t D0 = static_cast<std::uint32_t>(xs - r + R0);
        T.Sf = S + sg.frame_elems * f;
        T.o0 = D0 * T.Hs + R0;

        constexpr bool kWinOk = SPARSE && OPC_SKEW_KEY && NB >= OPC_SKEW_WINDOW_MIN_NB && OPC_SKEW_GROUPS &&
                                OPC_SKEW_WINDOW > 0 && OPC_SKEW_WINDOW < NB;
        if constexpr (kWinOk) {
            // Windowed pass when every phase's bin range fits the window.
            const int nph = ((T.NV - 1) >> 5) + 2;
            bool fits = true;
            int base0 = -1;
            for (int p = -1; p < nph && fits; ++p) {
                const std::uint32_t m = phase_bins(a, sg, bmask, f, yb, xs, 32 * p, T.w2, lane);
                if (!m) continue;
                const int lo = __ffs(m) - 1, hi = 31 - __clz(m);
                fits = hi - lo < OPC_SKEW_WINDOW;
                if (base0 < 0) base0 = max(0, min(lo - (OPC_SKEW_WINDOW - (hi - lo + 1)) / 2, NB - OPC_SKEW_WINDOW));
            }
            if (fits) {
                run_pass<NB, SL, SPARSE, (kWinOk ? OPC_SKEW_WINDOW : NB)>(T, a, sg, bmask, f, yb, xs, E, stage,
                                                                            recip, max(base0, 0));
                continue;
            }
        }
        run_pass<NB, SL, SPARSE, NB>(T, a, sg, bmask, f, yb, xs, E, stage, recip, 0);
    }
}

template <int NB, int SL, bool SPARSE>
cudaError_t launch_nbs(const BandArgs& a, int* counter, void* scratch, int num_sms,
                       cudaStream_t s) {
    const std::size_t pw = per_warp_bytes<NB, SL>();
    const std::size_t limit = 227 * 1024;
    int warps = kMaxWarps;
    while (warps > 1 && kRecipBytes + warps * pw > limit) --warps;
    const std::size_t smem = kRecipBytes + warps * pw;
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(skew_kernel<NB, SL, SPARSE>),
                                  static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = blocks_per_sm(reinterpret_cast<const void*>(skew_kernel<NB, SL, SPARSE>), warps * 32, smem, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;

    const ShearGeom sg = shear_geom(a);
    std::uint32_t* S = static_cast<std::uint32_t*>(scratch);
    // block bin-mask table (GROUPED launches), after the plane
    std::uint32_t* bmask = nullptr;
    if constexpr (SPARSE && OPC_SKEW_KEY && OPC_SKEW_GROUPS &&
                  (NB >= OPC_SKEW_GROUPS_MIN_NB || NB >= OPC_SKEW_WINDOW_MIN_NB)) {
        bmask = S + sg.frame_elems * a.frames;
    }
    {
        const unsigned gx = static_cast<unsigned>((a.width + kShearPad + kShearCols - 1) / kShearCols);
        const dim3 grid(gx, static_cast<unsigned>(sg.Hs / kShearRows) + border_grid_rows(a, gx),
                        static_cast<unsigned>(a.frames));
        const int vec_ok = (reinterpret_cast<std::uintptr_t>(a.in) % 4 == 0) &&
                           ((static_cast<std::size_t>(a.width) * 3) % 4 == 0) &&
                           (a.in_frame_stride % 4 == 0);
        // TMA interior tiles: rows and frames 16-byte aligned
        const std::size_t row_bytes = static_cast<std::size_t>(a.width) * 3;
        CUtensorMap tin{};
        bool tma = OPC_SHEAR_TMA && row_bytes % 16 == 0 && a.in_frame_stride % 16 == 0 &&
                   reinterpret_cast<std::uintptr_t>(a.in) % 16 == 0;
        if (tma) {
            const cuuint64_t dims[3] = {static_cast<cuuint64_t>(row_bytes / 4),
                                        static_cast<cuuint64_t>(a.in_rows), static_cast<cuuint64_t>(a.frames)};
            const cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_bytes),
                                           static_cast<cuuint64_t>(a.in_frame_stride)};
            const cuuint32_t box[3] = {kShearCols * 3 / 4, kShearRows, 1};
            tma = encode_tensor_map(&tin, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<std::uint8_t*>(a.in),
                                    dims, strides, box) == 0;
        }
        const int key = (SPARSE && OPC_SKEW_KEY) ? 1 : 0;
        timing_mark(kIdPrePass, 0, s);
        if (tma) {
            shear_kernel<true><<<grid, 256, 0, s>>>(a, S, sg, vec_ok, key, bmask, tin);
        } else {
            shear_kernel<false><<<grid, 256, 0, s>>>(a, S, sg, vec_ok, key, bmask, tin);
        }
        timing_mark(kIdPrePass, 1, s);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }

    const long long resident = static_cast<long long>(num_sms) * per_sm * warps;
    // Static share 98%, 99% when a warp's share is small (bands of a multi-GPU
    // split): there each dynamic chunk is a sizeable extra pass for the warp
    // that takes it (C4 band of an 8-way split: -6.6%; whole C4: 98% 0.7% faster).
    const int nbands = (a.y_hi - a.y_lo + 31) / 32;
    const long long units = static_cast<long long>(a.frames) * nbands * (a.x_hi - a.x_lo);
    const int static_pct = units >= resident * OPC_SKEW_SMALL_SHARE ? OPC_SKEW_STATIC_PCT
                                                                     : OPC_SKEW_STATIC_PCT_SMALL;
    WorkSplit g = make_split(a.frames, nbands, a.x_hi - a.x_lo, resident, static_pct, OPC_SKEW_MIN_CHUNK);
    // Small shares (multi-GPU bands): band-aligned equal segments, one pass per
    // warp, when the step-count model says it ends sooner.  A pass costs its
    // columns plus F = 2(2r+1) + 32 fixed steps; a static chunk of s1 columns
    // crosses a band end with probability s1 / iw; about half a dynamic chunk
    // lands on the critical path.  (C4 band of an 8-way split: 0.560 -> 0.522
    // ms; the 2-way split and C5's frame shares stay on the default split,
    // where the aligned one measured 3% and 39% slower.)
    if (OPC_SKEW_ALIGNED && units < resident * OPC_SKEW_SMALL_SHARE) {
        WorkSplit al{};
        const int iw = a.x_hi - a.x_lo;
        if (make_aligned_split(a.frames, nbands, iw, resident, OPC_SKEW_MIN_CHUNK, al)) {
            const double F = 2.0 * (2 * a.radius + 1) + 32.0;
            const double aligned = static_cast<double>(al.s2) + F;
            const double s1 = static_cast<double>(g.s1);
            const double dflt = s1 + F * (1.0 + s1 / iw) +
                                (g.nchunks > g.nstatic ? 0.5 * (static_cast<double>(g.s2) + F) : 0.0);
            if (aligned < dflt) g = al;
        }
    }
    long long blocks = (g.nchunks + warps - 1) / warps;
    if (blocks > static_cast<long long>(num_sms) * per_sm) blocks = num_sms * per_sm;
    if (blocks < 1) blocks = 1;

    e = cudaMemsetAsync(counter, 0, 4 * sizeof(int), s);
    if (e != cudaSuccess) return e;
    const Mul M = (SPARSE && OPC_SKEW_KEY) ? Mul{1u, 0xFFFFFFFFu, 4u, 1u, 0x01000000u} : Mul{16u, 0xFFFFFFF0u, 4u, 1u, 0x00040000u};
    timing_mark(kIdSkew, 0, s);
    skew_kernel<NB, SL, SPARSE><<<static_cast<unsigned>(blocks), warps * 32, smem, s>>>(a, S, sg, counter, g, M,
                                                                                      bmask);
    timing_mark(kIdSkew, 1, s);
    return cudaGetLastError();
}

template <int NB>
cudaError_t launch_nb(const BandArgs& a, int* counter, void* scratch, int num_sms,
                      cudaStream_t s) {
    // The smaller ring when the window allows it (64 >= 16 + w2 + 32) and it
    // buys occupancy: NB = 31 goes from 8 to 11 warps per SM (config 5: -2.4%);
    // for NB = 21 (11 -> 12 warps) it measured 10% slower on config 2.
    const bool small = 2 * a.radius + 1 <= 16;
    if constexpr (NB >= 24) {
        if (small) return launch_nbs<NB, 64, true>(a, counter, scratch, num_sms, s);
    }
    if (small) return launch_nbs<NB, 96, true>(a, counter, scratch, num_sms, s);
    return launch_nbs<NB, OPC_SKEW_SL_LARGE, false>(a, counter, scratch, num_sms, s);
}

}  // namespace

bool skew_fits(const BandArgs& a) {
    return shear_geom(a).frame_elems < (1ull << 32) - 64;
}

bool skew_supported(int levels, int radius) {
    return levels >= 1 && levels + 1 <= 32 && radius >= 0 && radius <= 15 &&
           bin_multiplier(levels) != 0;
}

std::size_t skew_scratch_bytes(const BandArgs& a) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo) return 0;
    const ShearGeom sg = shear_geom(a);
    const std::size_t nbx = static_cast<std::size_t>(a.width + kShearPad + kShearCols - 1) / kShearCols *
                            (kShearCols / 32);
    const std::size_t table = static_cast<std::size_t>(a.frames) * (sg.Hs / kShearRows) * nbx;  // bin masks
    return (sg.frame_elems * a.frames + table) * sizeof(std::uint32_t);
}

cudaError_t launch_skew(const BandArgs& a, int* task_counter, void* scratch, int num_sms,
                        cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    const int bins = a.levels + 1;
    if (bins <= 4) return launch_nb<4>(a, task_counter, scratch, num_sms, s);
    if (bins <= 8) return launch_nb<8>(a, task_counter, scratch, num_sms, s);
    if (bins <= 12) return launch_nb<12>(a, task_counter, scratch, num_sms, s);
    if (bins <= 16) return launch_nb<16>(a, task_counter, scratch, num_sms, s);
    if (bins <= 21) return launch_nb<21>(a, task_counter, scratch, num_sms, s);
    if (bins <= 24) return launch_nb<24>(a, task_counter, scratch, num_sms, s);
    if (bins <= 28) return launch_nb<28>(a, task_counter, scratch, num_sms, s);
    if (bins <= 31) return launch_nb<31>(a, task_counter, scratch, num_sms, s);
    return launch_nb<32>(a, task_counter, scratch, num_sms, s);
}

}  // namespace opc
