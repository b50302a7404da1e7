/*
 * oilpaint_b200.h -- C-ABI of the B200-native histogram oil-paint filter.
 *
 * Drop-in boundary for the reference engines of arxiv/paper_1405_1020
 * ("oilbench", /root/reference/proj):
 *
 *   Image apply_sequential(const Image&, const FilterParams&)
 *       -- proj/include/oilpaint/filter.hpp:109, proj/src/filter.cpp:51-68
 *   Image apply_parallel(const Image&, const FilterParams&, const ParallelConfig&)
 *       -- proj/include/oilpaint/parallel.hpp:33, proj/src/parallel.cpp:110-132
 *   void validate(const Image&, const FilterParams&)
 *       -- proj/include/oilpaint/filter.hpp:25, proj/src/filter.cpp:8-26
 *
 * Buffer layout is the reference Image layout (proj/include/oilpaint/image.hpp:
 * 17-19, 27): interleaved 8-bit R,G,B, row-major, stride 3*W bytes, no padding,
 * exactly 3*W*H bytes per image.  Semantics are the reference's bit for bit:
 * bin = (R+G+B)*L/765 in unsigned integer arithmetic (filter.hpp:31-35), L+1
 * bins, lowest-index strict-> maximum (filter.hpp:71-82), truncating channel
 * quotient (filter.cpp:41-43), interior x in [r, W-r), y in [r, H-r), border
 * copied (CopyInput, default) or zeroed (ZeroFill) (filter.hpp:13-22).
 *
 * Status codes (errors are codes here; include/oilpaint_b200.hpp maps them to
 * the reference's exception types):
 *   OPC_OK      0
 *   OPC_EINVAL  1  parameter/shape error   -> std::invalid_argument
 *   OPC_ECUDA   2  CUDA/runtime failure     -> std::runtime_error
 *   OPC_ENOMEM  3  device/host allocation   -> std::system_error / bad_alloc
 * opc_last_error() returns a thread-local message for the last failing call.
 *
 * Threading: every entry point is blocking (host-pointer calls) and
 * thread-safe; calls on one device are serialised by the library (the
 * reference allows "serialized or interleaved at the engine's discretion",
 * SPEC.md concurrency model).  Device-pointer calls (OPC_FLAG_DEVICE_POINTERS)
 * are asynchronous on cfg->stream.
 */
#ifndef OILPAINT_B200_H
#define OILPAINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPC_OK 0
#define OPC_EINVAL 1
#define OPC_ECUDA 2
#define OPC_ENOMEM 3

/* BorderPolicy, proj/include/oilpaint/filter.hpp:13-16 */
#define OPC_BORDER_COPY_INPUT 0
#define OPC_BORDER_ZERO_FILL 1

/* cfg->flags */
#define OPC_FLAG_DEVICE_POINTERS 0x1u /* in/out are device pointers on cfg->device  */
#define OPC_FLAG_ALLOW_LEVELS_256 0x2u /* documented extension: accept L = 256 (257 bins, config 3) */
#define OPC_FLAG_COUNT_OPS 0x4u /* measurement run: the content-dependent kernel family (slide)
                                   counts the primitives it executes (opc_op_counts) */

/* cfg->kernel: 0 = automatic choice; the others force one kernel family
 * (test hooks, every family is bit-exact on every input it accepts). */
#define OPC_KERNEL_AUTO 0
#define OPC_KERNEL_DIRECT 1 /* one thread per output pixel, O(r^2), any r and L  */
#define OPC_KERNEL_SKEW 2   /* warp-skewed column-difference sliding, L+1 <= 32, r <= 15 */
#define OPC_KERNEL_SLIDE 3  /* per-lane O(r) sliding histogram, any L, r <= 15 (L+1 > 32 default) */
#define OPC_KERNEL_COLUMN 4 /* per-thread column-segment sliding, L+1 <= 32, r <= 7 (small images) */
#define OPC_KERNEL_PLANES 5 /* bit-plane counts + column-sum histograms per warp, L+1 <= 32, 1 <= r <= 7 */

typedef struct opc_config {
    int32_t device;  /* CUDA device ordinal; -1 = current device              */
    uint32_t flags;  /* OPC_FLAG_*                                            */
    void* stream;    /* cudaStream_t for device-pointer calls; NULL = default */
    int32_t kernel;  /* OPC_KERNEL_*                                          */
    int32_t reserved;
} opc_config;

/* Reference validate (proj/src/filter.cpp:8-26): 0 or OPC_EINVAL with a
 * message in opc_last_error().  Pure host logic, needs no GPU.  `flags` may
 * carry OPC_FLAG_ALLOW_LEVELS_256. */
int opc_validate(int32_t width, int32_t height, uint64_t nbytes, int32_t radius, int32_t levels,
                 uint32_t flags);

/* Whole-image filter: the apply_sequential / apply_parallel replacement.
 * in, out: 3*width*height bytes each, must not alias.  cfg may be NULL. */
int opc_filter_rgb8(const uint8_t* in, uint8_t* out, int32_t width, int32_t height,
                    int32_t radius, int32_t levels, int32_t border, const opc_config* cfg);

/* Frame batch (config 5): `frames` images of width x height stored back to
 * back (frame f at byte offset f*3*width*height) in in and out. */
int opc_filter_rgb8_batch(const uint8_t* in, uint8_t* out, int32_t frames, int32_t width,
                          int32_t height, int32_t radius, int32_t levels, int32_t border,
                          const opc_config* cfg);

/* Row band of a height-row image (multi-GPU row partition):
 * in_rows holds image rows [max(0, y_begin - radius), min(height, y_end + radius))
 * and out_rows receives output rows [y_begin, y_end); the border policy applies
 * to the global border only.  Bands [0,a),[a,b),...,[z,height) reassemble the
 * whole-image result byte for byte. */
int opc_filter_rgb8_band(const uint8_t* in_rows, uint8_t* out_rows, int32_t width,
                         int32_t height, int32_t y_begin, int32_t y_end, int32_t radius,
                         int32_t levels, int32_t border, const opc_config* cfg);

/* Multi-GPU host path.  frames == 1: the output rows are split
 * into ndevices contiguous bands [opc_band_begin(h,n,k), opc_band_begin(h,n,k+1))
 * and each device filters its band from its halo'd input rows; frames > 1: the
 * frames are split the same way.  One host thread per device, each with its
 * own device buffers and streams; no collective (the gather is the disjoint
 * writes into `out`).  Output is byte-identical to opc_filter_rgb8 / _batch.
 * devices: ndevices CUDA ordinals (repeats allowed, e.g. {0,0} on one GPU). */
int opc_filter_rgb8_multi(const uint8_t* in, uint8_t* out, int32_t frames, int32_t width,
                          int32_t height, int32_t radius, int32_t levels, int32_t border,
                          const int32_t* devices, int32_t ndevices, const opc_config* cfg);

/* First row (or frame) of part k of n equal contiguous parts of [0, total). */
int32_t opc_band_begin(int32_t total, int32_t parts, int32_t k);

/* Helpers for the band protocol: first input row and input row count. */
int32_t opc_band_in_row0(int32_t height, int32_t y_begin, int32_t radius);
int32_t opc_band_in_rows(int32_t height, int32_t y_begin, int32_t y_end, int32_t radius);

const char* opc_last_error(void);
const char* opc_version(void);

/* Number of CUDA kernels this library has launched in this process (the
 * bench's gpu_launches evidence). */
uint64_t opc_kernel_launches(void);

/* Number of visible CUDA devices (0 without a GPU; never fails). */
int32_t opc_device_count(void);

/* Blocks until all work the library queued on cfg's device/stream is done. */
int opc_synchronize(const opc_config* cfg);

/* Live kernel timing for benchmarks: with timing enabled every kernel launch
 * of the library is bracketed by CUDA events on its stream.
 * opc_kernel_timing(1) starts (and clears), opc_kernel_timing(0) stops;
 * opc_kernel_timing_read sums the recorded launches of one kernel
 * (synchronizing on their events).  Ids: 1 direct, 2 skew, 3 slide, 4 the
 * pre-pass (shear / transpose), 5 border, 6 column, 7 planes. */
#define OPC_KID_DIRECT 1
#define OPC_KID_SKEW 2
#define OPC_KID_SLIDE 3
#define OPC_KID_PREPASS 4
#define OPC_KID_BORDER 5
#define OPC_KID_COLUMN 6
#define OPC_KID_PLANES 7
int opc_kernel_timing(int32_t enable);
int opc_kernel_timing_read(int32_t kernel_id, double* ms_total, int64_t* launches);

/* Primitive counts accumulated on `device` by calls made with
 * OPC_FLAG_COUNT_OPS (synchronizes the device): out[0] output pixels, [1]
 * lane-steps, [2] histogram updates, [3] bins examined by argmax rescans,
 * [4] window pixels examined to rebuild winner sums, [5] warp rescans,
 * [6] winner changes, [7] warp-steps with updates.  n <= 8 entries are
 * written; reset != 0 zeroes the counters afterwards.  The slide kernel's
 * work depends on the content; bench.py turns these counts into the
 * algorithmic lane-op count of its roofline (SURVEY.md 8(d) primitives). */
#define OPC_OPCOUNT_N 8
int opc_op_counts(int32_t device, uint64_t* out, int32_t n, int32_t reset);

/* Which kernel family OPC_KERNEL_AUTO would use for these parameters
 * (OPC_KERNEL_*), or -1 if invalid.  Host logic only.  _batch: for a call
 * of `frames` frames (opc_filter_rgb8_batch; video batches may plan another
 * family than single images). */
int32_t opc_plan_kernel(int32_t width, int32_t height, int32_t radius, int32_t levels);
int32_t opc_plan_kernel_batch(int32_t width, int32_t height, int32_t radius, int32_t levels,
                              int32_t frames);

/* Releases cached device buffers and streams. */
void opc_release(void);

#ifdef __cplusplus
}
#endif

#endif /* OILPAINT_B200_H */
