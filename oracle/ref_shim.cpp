// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp + proj/tests/support/oracle.cpp), compiled by
// oracle/Makefile into oracle/_ref/libref_oilpaint.so.  This file is ours; the
// reference sources are compiled where they lie and never copied into the repo.
//
// Used by: tests (to pin oracle/oilpaint_oracle.c and to generate the golden
// fixtures) and bench.py (the cpu_baseline leg and `--impl reference`, which
// time the reference's own apply_parallel on the box's host cores).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oilpaint/filter.hpp"
#include "oilpaint/parallel.hpp"
#include "oilpaint/pattern.hpp"
#include "oilpaint/ppm.hpp"
#include "support/oracle.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

oilpaint::BorderPolicy border_of(int b) {
    return b == 0 ? oilpaint::BorderPolicy::CopyInput : oilpaint::BorderPolicy::ZeroFill;
}

oilpaint::Image image_of(const std::uint8_t* in, int w, int h) {
    std::vector<std::uint8_t> data(in, in + static_cast<std::size_t>(w) * h * 3);
    return oilpaint::Image(w, h, std::move(data));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

unsigned ref_hardware_concurrency(void) { return std::thread::hardware_concurrency(); }

// engine 0 = apply_sequential (proj/src/filter.cpp:51), 1 = apply_parallel
// (proj/src/parallel.cpp:110) with `workers` threads (0 = Auto).
// Returns 0 ok, 1 std::invalid_argument (reference validate), 2 other.
int ref_apply(const std::uint8_t* in, std::uint8_t* out, int w, int h, int radius, int levels,
              int border, int engine, int workers) {
    try {
        const oilpaint::Image img = image_of(in, w, h);
        const oilpaint::FilterParams params{radius, levels, border_of(border)};
        oilpaint::Image res = [&] {
            if (engine == 0) return oilpaint::apply_sequential(img, params);
            oilpaint::ParallelConfig cfg;
            if (workers > 0) cfg.worker_count = workers;
            return oilpaint::apply_parallel(img, params, cfg);
        }();
        std::memcpy(out, res.data().data(), res.data().size());
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// The test-suite brute-force oracle, proj/tests/support/oracle.cpp:7-57.  It
// has no L bound, so it is the reference oracle for config 3 (L = 256).
int ref_oracle_filter(const std::uint8_t* in, std::uint8_t* out, int w, int h, int radius,
                      int levels, int border) {
    try {
        const oilpaint::Image res = oracle::filter(image_of(in, w, h), radius, levels,
                                                   border_of(border));
        std::memcpy(out, res.data().data(), res.data().size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// The reference's own row-parallel engine body (proj/src/parallel.cpp:117-130:
// parallel_for_rows + private HistogramAccumulator + filter_pixel) without the
// L <= 255 validate gate, for config 3's L = 256 (built with -DNDEBUG, so the
// filter.hpp:32,51 asserts are compiled out).  Interior rows only; border per
// policy exactly as apply_parallel does it (parallel.cpp:113).
int ref_filter_rows_any_levels(const std::uint8_t* in, std::uint8_t* out, int w, int h,
                               int radius, int levels, int border, int workers) {
    try {
        const oilpaint::Image img = image_of(in, w, h);
        oilpaint::Image res = border == 0 ? img : oilpaint::Image(w, h);
        oilpaint::ParallelConfig cfg;
        if (workers > 0) cfg.worker_count = workers;
        oilpaint::parallel_for_rows(radius, h - radius, cfg, [&](int b, int e) {
            oilpaint::HistogramAccumulator hist(levels);
            for (int y = b; y < e; ++y) {
                std::uint8_t* o = res.pixel(radius, y);
                for (int x = radius; x < w - radius; ++x, o += 3) {
                    const oilpaint::Rgb c = oilpaint::filter_pixel(img, x, y, radius, hist);
                    o[0] = c.r;
                    o[1] = c.g;
                    o[2] = c.b;
                }
            }
        });
        std::memcpy(out, res.data().data(), res.data().size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// Same body restricted to interior rows [row_begin, row_end): the bounded
// CPU-baseline sample used by bench.py (a band of the benchmark image).  Only
// the band's rows plus their r-row halos are wrapped in the reference Image
// (the caller already holds the image; wrapping the whole 805 MB config 4
// image would time a copy the reference engine never makes).  `in` is the
// whole image; output rows land at their image offsets in `out`.
int ref_filter_band(const std::uint8_t* in, std::uint8_t* out, int w, int h, int radius,
                    int levels, int row_begin, int row_end, int workers) {
    try {
        const int lo = row_begin - radius > 0 ? row_begin - radius : 0;
        const int hi = row_end + radius < h ? row_end + radius : h;
        const oilpaint::Image img = image_of(in + static_cast<std::size_t>(lo) * w * 3, w, hi - lo);
        oilpaint::ParallelConfig cfg;
        if (workers > 0) cfg.worker_count = workers;
        oilpaint::parallel_for_rows(row_begin, row_end, cfg, [&](int b, int e) {
            oilpaint::HistogramAccumulator hist(levels);
            for (int y = b; y < e; ++y) {
                std::uint8_t* o = out + (static_cast<std::size_t>(y) * w + radius) * 3;
                for (int x = radius; x < w - radius; ++x, o += 3) {
                    const oilpaint::Rgb c = oilpaint::filter_pixel(img, x, y - lo, radius, hist);
                    o[0] = c.r;
                    o[1] = c.g;
                    o[2] = c.b;
                }
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// proj/src/pattern.cpp:81-88 generate(): kind 0 Noise{seed}, 1 Gradient,
// 2 Uniform{r,g,b = seed bytes 0..2}, 3 Checker{cell = seed}.
int ref_generate(int kind, std::uint64_t seed, int w, int h, std::uint8_t* out) {
    try {
        oilpaint::PatternSpec spec;
        spec.width = w;
        spec.height = h;
        switch (kind) {
            case 0: spec.kind = oilpaint::patterns::Noise{seed}; break;
            case 1: spec.kind = oilpaint::patterns::Gradient{}; break;
            case 2:
                spec.kind = oilpaint::patterns::Uniform{
                    {static_cast<std::uint8_t>(seed), static_cast<std::uint8_t>(seed >> 8),
                     static_cast<std::uint8_t>(seed >> 16)}};
                break;
            default: spec.kind = oilpaint::patterns::Checker{static_cast<int>(seed)}; break;
        }
        const oilpaint::Image img = oilpaint::generate(spec);
        std::memcpy(out, img.data().data(), img.data().size());
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// proj/src/ppm.cpp:108-117 write_ppm; returns the byte count written into
// out (capacity cap) or -1.
long ref_write_ppm(const std::uint8_t* in, int w, int h, std::uint8_t* out, long cap) {
    try {
        const std::vector<std::uint8_t> bytes = oilpaint::write_ppm(image_of(in, w, h));
        if (static_cast<long>(bytes.size()) > cap) return -1;
        std::memcpy(out, bytes.data(), bytes.size());
        return static_cast<long>(bytes.size());
    } catch (const std::exception& e) {
        fail(e, 2);
        return -1;
    }
}

}  // extern "C"
