/*
 * oilpaint_b200_patterns.h -- deterministic synthetic inputs (harness code,
 * not on the measured path).
 *
 * Kinds 0-3 restate the reference's pattern generator (proj/src/pattern.cpp:
 * 19-88): Noise{seed} is byte i = byte (i mod 8) of splitmix64 word i/8 of a
 * generator seeded with `seed` (pattern.cpp:11-17, 64-76) -- configs 1 and 4.
 * Kinds 10-12 are new harness generators for configs 2, 3 and 5 (BASELINE.json
 * "configs"), specified in DESIGN.md section 6.  They use integer arithmetic
 * after table set-up, so the bytes do not depend on the thread count.
 */
#ifndef OILPAINT_B200_PATTERNS_H
#define OILPAINT_B200_PATTERNS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPC_PATTERN_NOISE 0    /* reference Noise{seed}                         */
#define OPC_PATTERN_GRADIENT 1 /* reference Gradient                            */
#define OPC_PATTERN_UNIFORM 2  /* reference Uniform{r,g,b = seed bytes 0,1,2}   */
#define OPC_PATTERN_CHECKER 3  /* reference Checker{cell = seed, white/black}   */
#define OPC_PATTERN_SMOOTH 10  /* config 2: 4 low-frequency sinusoids/channel + U{-8..8} */
#define OPC_PATTERN_RECTS 11   /* config 3: 64 random rectangles over a background */
#define OPC_PATTERN_VIDEO 12   /* config 5: smooth field seeded seed+frame + N(0, 12^2) */

/* Writes 3*width*height bytes.  threads <= 0: hardware concurrency.
 * Returns 0 or 1 (invalid argument). */
int opc_generate(int32_t kind, uint64_t seed, int32_t width, int32_t height, int32_t frame,
                 uint8_t* out, int32_t threads);

/* Rows [row0, row0 + nrows) of the same image (3*width*nrows bytes, the bytes
 * opc_generate writes there): a rank of a row-band split generates only its
 * band and halo rows.  Returns 0 or 1 (invalid argument / rows outside the
 * image). */
int opc_generate_rows(int32_t kind, uint64_t seed, int32_t width, int32_t height, int32_t frame,
                      int32_t row0, int32_t nrows, uint8_t* out, int32_t threads);

/* The same bytes written into DEVICE memory `d_out` (3*width*height bytes) on
 * `stream` (NULL: the library's stream of `device`; device < 0: current), for
 * every kind; OPC_PATTERN_VIDEO takes the frame folded into the seed (seed +
 * frame, as opc_generate does internally).  Asynchronous, except that the first
 * call of kinds 10/12 on a device copies the sine / Gaussian tables and waits
 * for them.  Returns 0, 1 (invalid argument) or 2 (CUDA error);
 * opc_last_error() has the message. */
int opc_generate_device(int32_t kind, uint64_t seed, int32_t width, int32_t height,
                        uint8_t* d_out, int32_t device, void* stream);

#ifdef __cplusplus
}
#endif

#endif
