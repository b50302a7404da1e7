// patterns.cpp -- deterministic benchmark/test inputs (harness, not on the
// measured path).  Kinds 0-3 restate proj/src/pattern.cpp:19-88; kinds 10-12
// are the config 2/3/5 generators.  Every byte is a
// function of (kind, seed, width, height, frame) only: the random streams are
// counter-based splitmix64 (word k of seed s = mix(s + (k+1)*gamma), the same
// values pattern.cpp:11-17 produces sequentially), and per-pixel arithmetic is
// integer after the sine / Gaussian-quantile tables are built.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/oilpaint_b200_patterns.h"
#include "gen_spec.h"

namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

inline std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Word k (0-based) of the stream seeded with s (pattern.cpp:11-17).
inline std::uint64_t stream_word(std::uint64_t s, std::uint64_t k) {
    return mix64(s + (k + 1) * kGamma);
}

struct Stream {
    std::uint64_t state;
    std::uint64_t next() {
        state += kGamma;
        return mix64(state);
    }
    double unit() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// body(y0, y1) over the rows [row0, row1), split across threads.
template <class F>
void parallel_rows(int row0, int row1, int threads, F&& body) {
    const int rows = row1 - row0;
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    threads = std::min(threads, 64);
    threads = std::min(threads, rows);
    if (threads <= 1) {
        body(row0, row1);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        const int b = row0 + static_cast<int>(static_cast<long long>(rows) * t / threads);
        const int e = row0 + static_cast<int>(static_cast<long long>(rows) * (t + 1) / threads);
        pool.emplace_back([&body, b, e] { body(b, e); });
    }
    for (auto& th : pool) th.join();
}

const std::vector<std::int32_t>& sine_table() {
    static const std::vector<std::int32_t> t = [] {
        std::vector<std::int32_t> v(4096);
        for (int i = 0; i < 4096; ++i) {
            v[i] = static_cast<std::int32_t>(
                std::lround(std::sin(6.283185307179586 * i / 4096.0) * 32767.0));
        }
        return v;
    }();
    return t;
}

// Acklam's rational approximation of the standard normal quantile.
double normal_quantile(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                               -2.759285104469687e+02, 1.383577518672690e+02,
                               -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                               -1.556989798598866e+02, 6.680131188771972e+01,
                               -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                               -2.400758277161838e+00, -2.549732539343734e+00,
                               4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                               2.445134137142996e+00, 3.754408661907416e+00};
    const double plow = 0.02425;
    if (p < plow) {
        const double q = std::sqrt(-2 * std::log(p));
        return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    }
    if (p > 1 - plow) {
        const double q = std::sqrt(-2 * std::log(1 - p));
        return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    }
    const double q = p - 0.5;
    const double r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
}

// Gaussian N(0, 12^2) noise in 1/256 units, indexed by a 16-bit uniform.
const std::vector<std::int32_t>& gauss_table() {
    static const std::vector<std::int32_t> t = [] {
        std::vector<std::int32_t> v(65536);
        for (int i = 0; i < 65536; ++i) {
            v[i] = static_cast<std::int32_t>(
                std::lround(12.0 * 256.0 * normal_quantile((i + 0.5) / 65536.0)));
        }
        return v;
    }();
    return t;
}

// Config 2 / 5 field: per channel, 4 sinusoids with 0.5-4 cycles across the
// frame in x and y, random phase, amplitude in [0.5, 1).
// `out` holds rows [row0, row1) of the frame.
void smooth_field(std::uint64_t seed, int w, int h, bool gaussian, int row0, int row1,
                  std::uint8_t* out, int threads) {
    opc::SmoothSpec sp;
    opc::smooth_spec(seed, w, h, &sp);
    const std::int32_t* sine = opc::sine_table_data();
    const std::int32_t* gauss = gaussian ? opc::gauss_table_data() : nullptr;
    parallel_rows(row0, row1, threads, [&](int y0, int y1) {
        for (int y = y0; y < y1; ++y) {
            std::uint8_t* row = out + static_cast<std::size_t>(y - row0) * w * 3;
            for (int x = 0; x < w; ++x) {
                const std::uint64_t pix = static_cast<std::uint64_t>(y) * w + x;
                for (int c = 0; c < 3; ++c) {
                    std::int64_t s = 0;
                    for (int k = 0; k < 4; ++k) {
                        const opc::GenWave& wv = sp.waves[4 * c + k];
                        const std::uint32_t phase = wv.px * static_cast<std::uint32_t>(x) +
                                                    wv.py * static_cast<std::uint32_t>(y) + wv.ph;
                        s += static_cast<std::int64_t>(wv.amp) * sine[phase >> 20];
                    }
                    int v = 128 + static_cast<int>((s * 255) >> 30);
                    const std::uint64_t word = stream_word(sp.noise_seed, pix * 3 + c);
                    if (gauss) {
                        v += (gauss[word & 0xFFFFu] + 128) >> 8;
                    } else {
                        v += static_cast<int>(word % 17) - 8;
                    }
                    row[3 * x + c] = static_cast<std::uint8_t>(std::clamp(v, 0, 255));
                }
            }
        }
    });
}

// Config 3: background colour plus 64 axis-aligned rectangles with random
// inclusive corners and colours, painted in order (later on top).
void rects(std::uint64_t seed, int w, int h, int row0, int row1, std::uint8_t* out, int threads) {
    opc::RectsSpec sp;
    opc::rects_spec(seed, w, h, &sp);
    parallel_rows(row0, row1, threads, [&](int y0, int y1) {
        for (int y = y0; y < y1; ++y) {
            std::uint8_t* row = out + static_cast<std::size_t>(y - row0) * w * 3;
            for (int x = 0; x < w; ++x) {
                row[3 * x] = static_cast<std::uint8_t>(sp.bg);
                row[3 * x + 1] = static_cast<std::uint8_t>(sp.bg >> 8);
                row[3 * x + 2] = static_cast<std::uint8_t>(sp.bg >> 16);
            }
            for (const opc::GenRect& q : sp.rects) {
                if (y < q.y0 || y > q.y1) continue;
                for (int x = q.x0; x <= q.x1; ++x) {
                    row[3 * x] = static_cast<std::uint8_t>(q.rgb);
                    row[3 * x + 1] = static_cast<std::uint8_t>(q.rgb >> 8);
                    row[3 * x + 2] = static_cast<std::uint8_t>(q.rgb >> 16);
                }
            }
        }
    });
}

}  // namespace

namespace opc {

void smooth_spec(std::uint64_t seed, int w, int h, SmoothSpec* out) {
    Stream rng{seed};
    for (int c = 0; c < 3; ++c) {
        double amp[4], sum = 0;
        for (int k = 0; k < 4; ++k) {
            amp[k] = 0.5 + 0.5 * rng.unit();
            const double fx = (0.5 + 3.5 * rng.unit()) / w;
            const double fy = (0.5 + 3.5 * rng.unit()) / h;
            const double ph = rng.unit();
            GenWave& wv = out->waves[4 * c + k];
            wv.px = static_cast<std::uint32_t>(std::llround(fx * 4294967296.0));
            wv.py = static_cast<std::uint32_t>(std::llround(fy * 4294967296.0));
            wv.ph = static_cast<std::uint32_t>(std::llround(ph * 4294967296.0) & 0xFFFFFFFFll);
            sum += amp[k];
        }
        for (int k = 0; k < 4; ++k) {
            out->waves[4 * c + k].amp = static_cast<std::int32_t>(std::lround(amp[k] / sum * 16384.0));
        }
    }
    out->noise_seed = rng.next();
}

void rects_spec(std::uint64_t seed, int w, int h, RectsSpec* out) {
    Stream rng{seed};
    out->bg = static_cast<std::uint32_t>(rng.next() & 0xFFFFFFu);
    for (GenRect& q : out->rects) {
        const int xa = static_cast<int>(rng.next() % static_cast<std::uint64_t>(w));
        const int xb = static_cast<int>(rng.next() % static_cast<std::uint64_t>(w));
        const int ya = static_cast<int>(rng.next() % static_cast<std::uint64_t>(h));
        const int yb = static_cast<int>(rng.next() % static_cast<std::uint64_t>(h));
        const std::uint64_t col = rng.next();
        q.x0 = std::min(xa, xb);
        q.x1 = std::max(xa, xb);
        q.y0 = std::min(ya, yb);
        q.y1 = std::max(ya, yb);
        q.rgb = static_cast<std::uint32_t>(col & 0xFFFFFFu);
    }
}

const std::int32_t* sine_table_data() { return sine_table().data(); }
const std::int32_t* gauss_table_data() { return gauss_table().data(); }

}  // namespace opc

extern "C" int opc_generate_rows(int32_t kind, uint64_t seed, int32_t w, int32_t h,
                                 int32_t frame, int32_t row0, int32_t nrows, uint8_t* out,
                                 int32_t threads) {
    if (w < 1 || h < 1 || !out || row0 < 0 || nrows < 1 || row0 > h - nrows) return 1;
    const int row1 = row0 + nrows;
    const std::size_t row_bytes = static_cast<std::size_t>(w) * 3;
    switch (kind) {
        case OPC_PATTERN_NOISE:
            // byte i of the image = byte (i mod 8) of stream word i / 8
            parallel_rows(row0, row1, threads, [&](int y0, int y1) {
                const std::size_t b = static_cast<std::size_t>(y0) * row_bytes;
                const std::size_t e = static_cast<std::size_t>(y1) * row_bytes;
                std::uint8_t* o = out + (b - static_cast<std::size_t>(row0) * row_bytes);
                std::uint64_t k = ~0ull, word = 0;
                for (std::size_t i = b; i < e; ++i, ++o) {
                    if ((i >> 3) != k) {
                        k = i >> 3;
                        word = stream_word(seed, k);
                    }
                    *o = static_cast<std::uint8_t>(word >> (8 * (i & 7)));
                }
            });
            return 0;
        case OPC_PATTERN_GRADIENT: {
            const int dx = w > 1 ? w - 1 : 1, dy = h > 1 ? h - 1 : 1;
            const int dd = w + h > 2 ? w + h - 2 : 1;
            for (int y = row0; y < row1; ++y) {
                std::uint8_t* p = out + static_cast<std::size_t>(y - row0) * row_bytes;
                for (int x = 0; x < w; ++x, p += 3) {
                    p[0] = static_cast<std::uint8_t>(x * 255 / dx);
                    p[1] = static_cast<std::uint8_t>(y * 255 / dy);
                    p[2] = static_cast<std::uint8_t>((x + y) * 255 / dd);
                }
            }
            return 0;
        }
        case OPC_PATTERN_UNIFORM: {
            const std::size_t n = row_bytes * static_cast<std::size_t>(nrows);
            for (std::size_t i = 0; i < n; i += 3) {
                out[i] = static_cast<std::uint8_t>(seed);
                out[i + 1] = static_cast<std::uint8_t>(seed >> 8);
                out[i + 2] = static_cast<std::uint8_t>(seed >> 16);
            }
            return 0;
        }
        case OPC_PATTERN_CHECKER: {
            const int cell = static_cast<int>(seed);
            if (cell < 1) return 1;
            for (int y = row0; y < row1; ++y) {
                std::uint8_t* p = out + static_cast<std::size_t>(y - row0) * row_bytes;
                for (int x = 0; x < w; ++x, p += 3) {
                    const std::uint8_t v = ((x / cell) + (y / cell)) % 2 == 0 ? 255 : 0;
                    p[0] = p[1] = p[2] = v;
                }
            }
            return 0;
        }
        case OPC_PATTERN_SMOOTH:
            smooth_field(seed, w, h, false, row0, row1, out, threads);
            return 0;
        case OPC_PATTERN_RECTS:
            rects(seed, w, h, row0, row1, out, threads);
            return 0;
        case OPC_PATTERN_VIDEO:
            smooth_field(seed + static_cast<std::uint64_t>(frame), w, h, true, row0, row1, out,
                         threads);
            return 0;
        default:
            return 1;
    }
}

extern "C" int opc_generate(int32_t kind, uint64_t seed, int32_t w, int32_t h, int32_t frame,
                            uint8_t* out, int32_t threads) {
    return opc_generate_rows(kind, seed, w, h, frame, 0, h, out, threads);
}
