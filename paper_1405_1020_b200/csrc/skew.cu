// skew.cu -- the performance kernel family for L+1 <= 32 bins and r <= 15.
//
// Algorithm: column-difference sliding window, one output ROW per lane, the 32
// lanes of a warp skewed by one column each (lane t works on virtual column
// v = s - t at step s).  See DESIGN.md section 3 for the derivation; in short:
//
//  * The window histogram of lane t (row y) lives in registers as NB packed
//    64-bit words  [count:10 | sumR:18 | sumG:18 | sumB:18]  (exact for
//    (2r+1)^2 <= 1023, i.e. r <= 15; modular packed arithmetic is exact because
//    every window total fits its field).
//  * Sliding right:  W(x+1,y) = W(x,y) + E(x,y),
//        E(x,y) = Col(x+r+1,y) - Col(x-r,y)   (Col = 2r+1-row column histogram).
//    E slots live in shared memory, [bin][slot] layout.
//  * E(x,y+1) = E(x,y) + f(x+r+1,y+r+1) - f(x+r+1,y-r) - f(x-r,y+r+1) + f(x-r,y-r)
//    -- four dynamic-bin updates.  Lane t reads E(x,y) at step s and advances it
//    to row y+1; lane t+1 consumes it at step s+1 (same column, next row).  The
//    skew is what turns the vertical recurrence into a conflict-free pipeline.
//  * E(x, band top) is built from scratch (2(2r+1) updates per column) one
//    phase (32 steps) ahead, one column per lane.
//  * Argmax: a static tournament over the NB words comparing counts only
//    (hi word > other.hi | 0x3FFFFF <=> strictly larger count), left (lower
//    bin) operand kept on ties -> lowest-index maximum, filter.hpp:71-82.
//  * Quotient: q = umulhi(2*sum, floor(2^31/c)+1), exact for c <= 1023,
//    sum <= 255c (tests/test_oracle.py checks it exhaustively); filter.cpp:41-43.
//
// Memory: per warp a pixel ring (33+2r rows x 128 columns, 4 B per pixel:
// R,G,B,bin), the E ring (96 slots x NB x 8 B) and a 32x32 output staging tile
// that is flushed one completed row-block per step as coalesced 96-byte runs.
#include "kernels.cuh"

namespace opc {

namespace {

constexpr int kMaxWarps = 4;
constexpr int kRing = 128;
constexpr int kRingStride = kRing + 2;  // == 2 (mod 32): skewed accesses hit distinct banks
constexpr int kSlots = 96;
constexpr int kStageStride = 33;
constexpr int kRecipBytes = 1024 * 4;

__host__ __device__ inline int ring_rows(int r) { return 33 + 2 * r; }

__host__ __device__ inline std::size_t ring_bytes(int r) {
    return static_cast<std::size_t>(ring_rows(r)) * kRingStride * 4;
}

__host__ __device__ inline std::size_t per_warp_bytes(int nb, int r) {
    return ring_bytes(r) + static_cast<std::size_t>(nb) * kSlots * 8 + 32 * kStageStride * 4;
}

__device__ __forceinline__ std::uint32_t make_entry(std::uint32_t r, std::uint32_t g,
                                                    std::uint32_t b, std::uint32_t bin_mul) {
    const std::uint32_t bin = __umulhi(r + g + b, bin_mul);  // filter.hpp:31-35
    return r | (g << 8) | (b << 16) | (bin << 24);
}

// Packed single-pixel contribution (count 1, R, G, B) of a ring entry.
__device__ __forceinline__ unsigned long long packed_of(std::uint32_t e) {
    const std::uint32_t lo = ((e >> 16) & 0xFFu) | ((e & 0xFF00u) << 10);  // B | G << 18
    const std::uint32_t hi = ((e & 0xFFu) << 4) | 0x400000u;                // R << 36, 1 << 54
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

__device__ __forceinline__ void rmw_add(unsigned long long* E, int slot, std::uint32_t e) {
    unsigned long long* p = E + (e >> 24) * kSlots + slot;
    *p += packed_of(e);
}

__device__ __forceinline__ void rmw_sub(unsigned long long* E, int slot, std::uint32_t e) {
    unsigned long long* p = E + (e >> 24) * kSlots + slot;
    *p -= packed_of(e);
}

template <int NB>
__device__ __forceinline__ std::uint32_t winner_rgb(const unsigned long long (&w)[NB],
                                                    const std::uint32_t* recip) {
    unsigned long long t[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) t[b] = w[b];
#pragma unroll
    for (int step = 1; step < NB; step <<= 1) {
#pragma unroll
        for (int i = 0; i + step < NB; i += 2 * step) {
            const std::uint32_t ah = static_cast<std::uint32_t>(t[i] >> 32);
            const std::uint32_t bh = static_cast<std::uint32_t>(t[i + step] >> 32);
            t[i] = bh > (ah | 0x3FFFFFu) ? t[i + step] : t[i];
        }
    }
    const std::uint32_t lo = static_cast<std::uint32_t>(t[0]);
    const std::uint32_t hi = static_cast<std::uint32_t>(t[0] >> 32);
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

struct TaskGeom {
    int nbands, nsegs, segw, ntasks;
};

template <int NB>
__global__ void __launch_bounds__(kMaxWarps * 32, 1)
    skew_kernel(BandArgs a, int* task_counter, TaskGeom g) {
    extern __shared__ __align__(16) unsigned char smem[];
    std::uint32_t* recip = reinterpret_cast<std::uint32_t*>(smem);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int r = a.radius;
    const int w2 = 2 * r + 1;
    const int rows = ring_rows(r);
    unsigned char* wbase = smem + kRecipBytes + warp * per_warp_bytes(NB, r);
    std::uint32_t* ring = reinterpret_cast<std::uint32_t*>(wbase);
    unsigned long long* E = reinterpret_cast<unsigned long long*>(wbase + ring_bytes(r));
    std::uint32_t* stage =
        reinterpret_cast<std::uint32_t*>(wbase + ring_bytes(r) + std::size_t(NB) * kSlots * 8);

    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        recip[i] = i ? 0x80000000u / static_cast<std::uint32_t>(i) + 1u : 0u;
    }
    __syncthreads();

    const int W = a.width;
    const std::size_t stride = static_cast<std::size_t>(W) * 3;
    const int per_frame = g.nbands * g.nsegs;

    for (;;) {
        int task = 0;
        if (lane == 0) task = atomicAdd(task_counter, 1);
        task = __shfl_sync(0xFFFFFFFFu, task, 0);
        if (task >= g.ntasks) break;
        const int f = task / per_frame;
        const int rem = task - f * per_frame;
        const int kb = rem / g.nsegs;
        const int js = rem - kb * g.nsegs;
        const int yb = a.y_lo + 32 * kb;
        const int xs = a.x_lo + js * g.segw;
        const int xe = min(xs + g.segw, a.x_hi);
        const int NV = w2 + (xe - xs);  // virtual columns: w2 warm-up + outputs
        const int base_col = xs - r;    // image column of ring-relative column 0
        const int X0 = xs - w2;         // image column of virtual column 0
        const int row0 = yb - r;        // image row of ring row 0
        const std::uint8_t* in = a.in + a.in_frame_stride * f;
        std::uint8_t* out = a.out + a.out_frame_stride * f;
        const bool row_ok = yb + lane < a.y_hi;

        // Pixel ring loader: ring-relative columns [32c, 32c+32), all ring rows.
        auto load_chunk = [&](int c) {
            const int col = base_col + 32 * c + lane;
            const int ridx = (32 * c + lane) & (kRing - 1);
            const bool col_ok = col < W;
#pragma unroll 4
            for (int rho = 0; rho < rows; ++rho) {
                const int y = row0 + rho;
                std::uint32_t e = 0;
                if (col_ok && y < a.in_row0 + a.in_rows) {
                    const std::uint8_t* p = in + static_cast<std::size_t>(y - a.in_row0) * stride +
                                            static_cast<std::size_t>(col) * 3;
                    e = make_entry(p[0], p[1], p[2], a.bin_mul);
                }
                ring[rho * kRingStride + ridx] = e;
            }
        };
        auto zero_slot = [&](int slot) {
#pragma unroll
            for (int b = 0; b < NB; ++b) E[b * kSlots + slot] = 0ull;
        };
        // One row (k) of the from-scratch build of E(vi, yb).
        auto init_step = [&](int vi, int k) {
            const int slot = vi % kSlots;
            rmw_add(E, slot, ring[k * kRingStride + (vi & (kRing - 1))]);
            if (vi >= w2) rmw_sub(E, slot, ring[k * kRingStride + ((vi - w2) & (kRing - 1))]);
        };

        unsigned long long win[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) win[b] = 0ull;

        // Prologue: chunk 0 and E(v, yb) for v in [0, 32).
        load_chunk(0);
        zero_slot(lane);
        __syncwarp();
        for (int k = 0; k < w2; ++k) init_step(lane, k);
        __syncwarp();

        const int nphases = ((NV - 1) >> 5) + 2;
        for (int p = 0; p < nphases; ++p) {
            load_chunk(p + 1);
            const int vi = 32 * (p + 1) + lane;
            zero_slot(vi % kSlots);
            __syncwarp();
            for (int ss = 0; ss < 32; ++ss) {
                const int s = 32 * p + ss;
                const int v = s - lane;
                if (v >= 0 && v < NV) {
                    const int slot = v % kSlots;
                    unsigned long long e[NB];
#pragma unroll
                    for (int b = 0; b < NB; ++b) e[b] = E[b * kSlots + slot];
                    if (v >= w2 && row_ok) {
                        stage[lane * kStageStride + (v & 31)] = winner_rgb<NB>(win, recip);
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b) win[b] += e[b];
                    // Advance E(v) from row yb+lane to yb+lane+1 for lane+1.
                    const int ce = v & (kRing - 1);
                    const std::uint32_t* rn = ring + (lane + w2) * kRingStride;  // row y+r+1
                    const std::uint32_t* ro = ring + lane * kRingStride;         // row y-r
                    rmw_add(E, slot, rn[ce]);
                    rmw_sub(E, slot, ro[ce]);
                    if (v >= w2) {
                        const int cl = (v - w2) & (kRing - 1);
                        rmw_sub(E, slot, rn[cl]);
                        rmw_add(E, slot, ro[cl]);
                    }
                }
                if (ss < w2) init_step(vi, ss);
                __syncwarp();
                // Row fr just completed the 32-column block ending at v = s - fr.
                const int fr = (s + 1) & 31;
                const int vend = s - fr;
                if (vend >= 0) {
                    const int vv = vend - 31 + lane;
                    if (vv >= w2 && vv < NV && yb + fr < a.y_hi) {
                        const std::uint32_t rgb = stage[fr * kStageStride + lane];
                        std::uint8_t* o = out +
                                          static_cast<std::size_t>(yb + fr - a.out_row0) * stride +
                                          static_cast<std::size_t>(X0 + vv) * 3;
                        o[0] = static_cast<std::uint8_t>(rgb);
                        o[1] = static_cast<std::uint8_t>(rgb >> 8);
                        o[2] = static_cast<std::uint8_t>(rgb >> 16);
                    }
                }
                __syncwarp();
            }
        }
    }
}

template <int NB>
cudaError_t launch_nb(const BandArgs& a, int* counter, int num_sms, cudaStream_t s) {
    const std::size_t pw = per_warp_bytes(NB, a.radius);
    int warps = kMaxWarps;
    const std::size_t limit = 227 * 1024;
    while (warps > 1 && kRecipBytes + warps * pw > limit) --warps;
    const std::size_t smem = kRecipBytes + warps * pw;
    if (smem > limit) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(skew_kernel<NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;

    TaskGeom g{};
    const int rows = a.y_hi - a.y_lo;
    const int iw = a.x_hi - a.x_lo;
    g.nbands = (rows + 31) / 32;
    const long long total_warps = static_cast<long long>(num_sms) * warps;
    // Aim for >= 4 tasks per resident warp, segments no narrower than 128.
    long long want = 4 * total_warps;
    long long per_seg = static_cast<long long>(g.nbands) * a.frames;
    int nsegs = static_cast<int>((want + per_seg - 1) / per_seg);
    const int max_segs = (iw + 127) / 128;
    if (nsegs > max_segs) nsegs = max_segs;
    if (nsegs < 1) nsegs = 1;
    g.segw = (iw + nsegs - 1) / nsegs;
    g.nsegs = (iw + g.segw - 1) / g.segw;
    g.ntasks = a.frames * g.nbands * g.nsegs;
    int blocks = static_cast<int>((g.ntasks + warps - 1) / warps);
    if (blocks > num_sms) blocks = num_sms;
    if (blocks < 1) blocks = 1;

    e = cudaMemsetAsync(counter, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    skew_kernel<NB><<<blocks, warps * 32, smem, s>>>(a, counter, g);
    return cudaGetLastError();
}

}  // namespace

bool skew_supported(int levels, int radius) {
    return levels >= 1 && levels + 1 <= 32 && radius >= 0 && radius <= 15 &&
           bin_multiplier(levels) != 0;
}

std::size_t skew_smem_bytes(int levels, int radius) {
    return kRecipBytes + per_warp_bytes(levels + 1, radius);
}

cudaError_t launch_skew(const BandArgs& a, int* task_counter, int num_sms, cudaStream_t s) {
    if (a.y_hi <= a.y_lo || a.x_hi <= a.x_lo || a.frames <= 0) return cudaSuccess;
    const int bins = a.levels + 1;
    if (bins <= 4) return launch_nb<4>(a, task_counter, num_sms, s);
    if (bins <= 8) return launch_nb<8>(a, task_counter, num_sms, s);
    if (bins <= 12) return launch_nb<12>(a, task_counter, num_sms, s);
    if (bins <= 16) return launch_nb<16>(a, task_counter, num_sms, s);
    if (bins <= 21) return launch_nb<21>(a, task_counter, num_sms, s);
    if (bins <= 24) return launch_nb<24>(a, task_counter, num_sms, s);
    if (bins <= 28) return launch_nb<28>(a, task_counter, num_sms, s);
    if (bins <= 31) return launch_nb<31>(a, task_counter, num_sms, s);
    return launch_nb<32>(a, task_counter, num_sms, s);
}

}  // namespace opc
