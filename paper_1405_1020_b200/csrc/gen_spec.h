// gen_spec.h -- parameters of the config 2/3/5 generators (patterns.cpp),
// derived once on the host and shared by the host generator and the device
// generator (gen.cu), so both write the same bytes.
#pragma once

#include <cstdint>

namespace opc {

struct GenWave {
    std::uint32_t px, py, ph;  // phase increments / offset in 2^-32 turns
    std::int32_t amp;          // weight; the 4 waves of a channel sum to ~2^14
};

// OPC_PATTERN_SMOOTH / OPC_PATTERN_VIDEO: per channel c, waves[4c .. 4c+3].
struct SmoothSpec {
    GenWave waves[12];
    std::uint64_t noise_seed;  // per-pixel noise: word pix*3+c of this stream
};

struct GenRect {
    std::int32_t x0, x1, y0, y1;  // inclusive
    std::uint32_t rgb;            // R | G << 8 | B << 16
};

// OPC_PATTERN_RECTS: background, then the rectangles painted in order.
struct RectsSpec {
    std::uint32_t bg;
    GenRect rects[64];
};

void smooth_spec(std::uint64_t seed, int w, int h, SmoothSpec* out);
void rects_spec(std::uint64_t seed, int w, int h, RectsSpec* out);
const std::int32_t* sine_table_data();   // 4096 entries: round(sin(2 pi i / 4096) * 32767)
const std::int32_t* gauss_table_data();  // 65536 entries: N(0, 12^2) quantiles in 1/256 units

}  // namespace opc
