// oilpaint_b200.hpp -- C++ host API over the C-ABI, mirroring the reference
// engine interface of arxiv/paper_1405_1020 ("oilbench", /root/reference/proj)
// so that a caller of apply_sequential / apply_parallel switches by renaming
// the call:
//
//   reference                                            here
//   oilpaint::Rgb, oilpaint::Image (image.hpp:9-59)      oilpaint_b200::Rgb, Image
//   oilpaint::BorderPolicy, FilterParams (filter.hpp:13-22)  same names, same defaults
//   void validate(const Image&, const FilterParams&)     validate(...)   (filter.cpp:8-26)
//   Image apply_sequential(const Image&, const FilterParams&)   apply_cuda(img, params)
//   Image apply_parallel(const Image&, const FilterParams&,
//                        const ParallelConfig& = {})      apply_cuda(img, params, CudaConfig)
//
// Error behaviour is the reference's: parameter errors throw
// std::invalid_argument with the reference's messages, runtime/CUDA failures
// throw std::runtime_error, allocation failures std::bad_alloc.  The call is
// pure, blocking and thread-safe (SPEC.md concurrency model).
//
// CudaConfig::devices with more than one entry splits the interior rows into
// contiguous bands (r-row halos) across those GPUs, like
// ParallelConfig::worker_count splits rows across threads (parallel.cpp:55-108);
// the output is byte-identical for every configuration.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "oilpaint_b200.h"

namespace oilpaint_b200 {

struct Rgb {
    std::uint8_t r = 0;
    std::uint8_t g = 0;
    std::uint8_t b = 0;
    friend bool operator==(const Rgb&, const Rgb&) = default;
};

// Owned 8-bit RGB raster, channels interleaved R,G,B, rows top to bottom,
// stride == width * 3, data().size() == width * height * 3.
class Image {
  public:
    Image(int width, int height) : width_(width), height_(height), data_(checked(width, height), 0) {}
    Image(int width, int height, std::vector<std::uint8_t> data)
        : width_(width), height_(height), data_(std::move(data)) {
        if (data_.size() != checked(width, height)) {
            throw std::invalid_argument("image data length " + std::to_string(data_.size()) +
                                        " does not match " + std::to_string(width) + "x" +
                                        std::to_string(height));
        }
    }
    int width() const { return width_; }
    int height() const { return height_; }
    std::size_t stride() const { return static_cast<std::size_t>(width_) * 3; }
    std::uint8_t* row(int y) { return data_.data() + static_cast<std::size_t>(y) * stride(); }
    const std::uint8_t* row(int y) const {
        return data_.data() + static_cast<std::size_t>(y) * stride();
    }
    std::uint8_t* pixel(int x, int y) { return row(y) + static_cast<std::size_t>(x) * 3; }
    const std::uint8_t* pixel(int x, int y) const {
        return row(y) + static_cast<std::size_t>(x) * 3;
    }
    Rgb at(int x, int y) const {
        const std::uint8_t* p = pixel(x, y);
        return Rgb{p[0], p[1], p[2]};
    }
    void set(int x, int y, Rgb c) {
        std::uint8_t* p = pixel(x, y);
        p[0] = c.r;
        p[1] = c.g;
        p[2] = c.b;
    }
    std::vector<std::uint8_t>& data() { return data_; }
    const std::vector<std::uint8_t>& data() const { return data_; }
    friend bool operator==(const Image&, const Image&) = default;

  private:
    static std::size_t checked(int w, int h) {
        if (w < 1 || h < 1) {
            throw std::invalid_argument("image dimensions must be positive, got " +
                                        std::to_string(w) + "x" + std::to_string(h));
        }
        return static_cast<std::size_t>(w) * static_cast<std::size_t>(h) * 3;
    }
    int width_ = 0;
    int height_ = 0;
    std::vector<std::uint8_t> data_;
};

enum class BorderPolicy {
    CopyInput,  // border pixels copied verbatim from the input
    ZeroFill,   // border pixels left at channel value 0
};

struct FilterParams {
    int radius = 2;
    int intensity_levels = 20;
    BorderPolicy border = BorderPolicy::CopyInput;
};

struct CudaConfig {
    std::vector<int> devices;        // empty: current device; >1: row bands / frames split
    bool allow_levels_256 = false;   // documented C-ABI extension (config 3); off = reference contract
    int kernel = OPC_KERNEL_AUTO;    // test hook: force a kernel family
};

namespace detail {

inline void raise(int status) {
    if (status == OPC_OK) return;
    const std::string msg = opc_last_error();
    if (status == OPC_EINVAL) throw std::invalid_argument(msg);
    if (status == OPC_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}

inline opc_config to_c(const CudaConfig& cfg, int device) {
    opc_config c{};
    c.device = device;
    c.flags = cfg.allow_levels_256 ? OPC_FLAG_ALLOW_LEVELS_256 : 0u;
    c.stream = nullptr;
    c.kernel = cfg.kernel;
    return c;
}

inline int border_code(BorderPolicy b) {
    return b == BorderPolicy::CopyInput ? OPC_BORDER_COPY_INPUT : OPC_BORDER_ZERO_FILL;
}

}  // namespace detail

// Reference validate (proj/src/filter.cpp:8-26).
inline void validate(const Image& img, const FilterParams& params, bool allow_levels_256 = false) {
    detail::raise(opc_validate(img.width(), img.height(), img.data().size(), params.radius,
                               params.intensity_levels,
                               allow_levels_256 ? OPC_FLAG_ALLOW_LEVELS_256 : 0u));
}

// The CUDA engine: drop-in for apply_sequential / apply_parallel.
inline Image apply_cuda(const Image& img, const FilterParams& params, const CudaConfig& cfg = {}) {
    validate(img, params, cfg.allow_levels_256);
    Image out(img.width(), img.height());
    const int border = detail::border_code(params.border);
    if (cfg.devices.size() <= 1) {
        const opc_config c = detail::to_c(cfg, cfg.devices.empty() ? -1 : cfg.devices[0]);
        detail::raise(opc_filter_rgb8(img.data().data(), out.data().data(), img.width(),
                                      img.height(), params.radius, params.intensity_levels, border,
                                      &c));
        return out;
    }
    const opc_config c = detail::to_c(cfg, -1);
    detail::raise(opc_filter_rgb8_multi(img.data().data(), out.data().data(), 1, img.width(),
                                        img.height(), params.radius, params.intensity_levels,
                                        border, cfg.devices.data(),
                                        static_cast<int32_t>(cfg.devices.size()), &c));
    return out;
}

// Frame batch (config 5): frames of one size, split by frame across devices.
inline std::vector<Image> apply_cuda_batch(const std::vector<Image>& frames,
                                           const FilterParams& params,
                                           const CudaConfig& cfg = {}) {
    std::vector<Image> outs;
    if (frames.empty()) return outs;
    const int w = frames[0].width(), h = frames[0].height();
    std::vector<std::uint8_t> in;
    in.reserve(frames.size() * frames[0].data().size());
    for (const Image& f : frames) {
        if (f.width() != w || f.height() != h) {
            throw std::invalid_argument("all frames of a batch must have the same size");
        }
        validate(f, params, cfg.allow_levels_256);
        in.insert(in.end(), f.data().begin(), f.data().end());
    }
    std::vector<std::uint8_t> out(in.size());
    const int border = detail::border_code(params.border);
    const opc_config c = detail::to_c(cfg, cfg.devices.size() == 1 ? cfg.devices[0] : -1);
    if (cfg.devices.size() > 1) {
        detail::raise(opc_filter_rgb8_multi(in.data(), out.data(), static_cast<int32_t>(frames.size()),
                                            w, h, params.radius, params.intensity_levels, border,
                                            cfg.devices.data(),
                                            static_cast<int32_t>(cfg.devices.size()), &c));
    } else {
        detail::raise(opc_filter_rgb8_batch(in.data(), out.data(),
                                            static_cast<int32_t>(frames.size()), w, h,
                                            params.radius, params.intensity_levels, border, &c));
    }
    const std::size_t n = frames[0].data().size();
    for (std::size_t f = 0; f < frames.size(); ++f) {
        outs.emplace_back(w, h, std::vector<std::uint8_t>(out.begin() + f * n, out.begin() + (f + 1) * n));
    }
    return outs;
}

}  // namespace oilpaint_b200
