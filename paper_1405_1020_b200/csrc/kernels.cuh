// kernels.cuh -- device-side declarations shared by the kernel families and
// the C-ABI host code.  All kernels follow the reference semantics of
// proj/include/oilpaint/filter.hpp:31-105 and proj/src/filter.cpp:28-68.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include <cuda_runtime.h>

namespace opc {

// Per-device caches of kernel attributes (the launchers run on every call;
// cudaFuncSetAttribute / occupancy queries are a few microseconds each, which
// small images feel).
inline cudaError_t set_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    int& have = done[{dev, func}];
    if (have >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

inline cudaError_t blocks_per_sm(const void* func, int threads, std::size_t smem, int* out) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, std::size_t>, int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find({dev, func, threads, smem});
    if (it != done.end()) {
        *out = it->second;
        return cudaSuccess;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, func, threads, smem);
    if (e == cudaSuccess) done[{dev, func, threads, smem}] = *out;
    return e;
}

// Live kernel timing (opc_kernel_timing in the C-ABI): when a hook is set, the
// launchers call it right before (phase 0) and after (phase 1) each kernel
// launch, on the launch's stream, and the C-ABI records CUDA events there.
enum KernelId {
    kIdDirect = 1, kIdSkew = 2, kIdSlide = 3, kIdPrePass = 4, kIdBorder = 5, kIdColumn = 6, kIdPlanes = 7
};
using TimingHook = void (*)(int id, int phase, cudaStream_t s);
extern TimingHook g_timing_hook;
inline void timing_mark(int id, int phase, cudaStream_t s) {
    if (g_timing_hook) g_timing_hook(id, phase, s);
}

// One launch produces output rows [y_begin, y_end) of `frames` frames of a
// width x height image.  Input buffer row 0 is image row in_row0 and holds
// in_rows rows; output buffer row 0 is image row out_row0.  Interior rows
// [y_lo, y_hi) (= [y_begin, y_end) clipped to [r, H-r)) and columns
// [x_lo, x_hi) are computed by the filter kernels; the border pixels of rows
// [y_begin, y_end) are written by the border kernel.
// The border pixels of a launch's output rows, written by extra blocks of the
// launch's first kernel (pre-pass or direct), or by border_kernel when the
// band has no interior.  Blocks [0, nfull) copy the full border rows, the
// rest one interior row's left and right r-pixel strips per warp.
struct BorderJob {
    int policy;  // 0 CopyInput, 1 ZeroFill
    int top_lo, top_rows, bot_lo, bot_rows;
    int nfull;    // blocks on the full rows
    int nblocks;  // nfull + strip blocks; 0 = nothing to write
};
constexpr int kBorderThreads = 256;

struct BandArgs {
    const std::uint8_t* in;
    std::uint8_t* out;
    std::size_t in_frame_stride;   // bytes between frames in `in`
    std::size_t out_frame_stride;  // bytes between frames in `out`
    int frames;
    int width;
    int height;  // full image height (global border rows)
    int in_row0;
    int in_rows;
    int out_row0;
    int y_begin, y_end;  // output rows this launch produces
    int y_lo, y_hi;  // interior rows of this band (may be empty)
    int x_lo, x_hi;  // interior columns [r, W - r)
    int radius;
    int levels;
    std::uint32_t bin_mul;  // bin = umulhi(r+g+b, bin_mul) == (r+g+b)*L/765
    BorderJob border;       // fused into the first kernel of the launch
    // Non-null (OPC_FLAG_COUNT_OPS): the content-dependent families (slide)
    // launch their counting instantiation, which adds its executed primitive
    // counts (OpCount indices) here -- a measurement run, never the timed one.
    unsigned long long* op_counts;
};

// Primitive counts of a counted launch (SURVEY.md 8(d) primitives).
enum OpCount {
    kOpPixels = 0,       // output pixels written by the filter kernel (12 lane-ops each)
    kOpSteps = 1,        // lane-steps of the slide (the per-step flat check, 3 lane-ops)
    kOpUpdates = 2,      // histogram count updates executed (7 lane-ops each)
    kOpBinsExamined = 3, // bins examined by argmax rescans (3 lane-ops each)
    kOpSumPixels = 4,    // window pixels examined to rebuild a winner's channel sums (7 each)
    kOpRescans = 5,      // warp-wide rescans (diagnostic)
    kOpWinnerChanges = 6,// lanes whose winner changed (diagnostic)
    kOpNonFlatSteps = 7, // warp-steps that applied updates (diagnostic)
    kOpCountN = 8
};

// Exact magic multiplier for floor(s * L / 765), s in [0, 765], L in [1, 256];
// 0 if none exists (host falls back to the generic division path).
std::uint32_t bin_multiplier(int levels);

// ---- kernel families (each returns cudaError_t of the launch) ----
cudaError_t launch_direct(const BandArgs& a, cudaStream_t s);
bool direct_fuses_border(const BandArgs& a);  // tile kernel: border blocks appended
BorderJob make_border_job(const BandArgs& a, int border_policy);
// Standalone border launch (a band without interior rows): a.border's blocks.
cudaError_t launch_border(const BandArgs& a, cudaStream_t s);

// Column family (small images): L + 1 <= 32, radius <= 7; border fused.
bool column_supported(int levels, int radius);
cudaError_t launch_column(const BandArgs& a, int num_sms, cudaStream_t s);

// Bit-plane column family: L + 1 <= 32, 1 <= radius <= 7; border fused.
bool planes_supported(int levels, int radius);
cudaError_t launch_planes(const BandArgs& a, int num_sms, cudaStream_t s);

// Skew family: L + 1 <= 32, radius <= 15.  `task_counter` is a device int
// (zeroed by the launcher on the stream).
// Skew family also needs device scratch (the sheared entry plane) of
// skew_scratch_bytes(a) bytes.
bool skew_supported(int levels, int radius);
bool skew_fits(const BandArgs& a);  // sheared plane addressable with 32-bit offsets
std::size_t skew_scratch_bytes(const BandArgs& a);
cudaError_t launch_skew(const BandArgs& a, int* task_counter, void* scratch, int num_sms,
                        cudaStream_t s);

// Slide family (any L <= 256, r <= 15; the default for L+1 > 32): needs a
// transposed entry plane of slide_scratch_bytes(a) bytes.
bool slide_supported(int levels, int radius);
std::size_t slide_scratch_bytes(const BandArgs& a);
cudaError_t launch_slide(const BandArgs& a, int* task_counter, void* scratch, int num_sms,
                         cudaStream_t s);

// On-device pattern generation (gen.cu): 0 launched (*err = launch status),
// 1 invalid argument, -1 no device generator for `kind`.
int launch_generate(int kind, std::uint64_t seed, int w, int h, std::uint8_t* out, cudaStream_t s,
                    cudaError_t* err);

}  // namespace opc
