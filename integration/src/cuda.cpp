// cuda.cpp -- oilpaint::apply_cuda over the C-ABI (include/oilpaint_b200.h).
//
// Reference contract followed (proj/include/oilpaint/filter.hpp:107-109,
// proj/src/filter.cpp:51-68):
//   1. validate(img, params) -- the reference's own function, so every
//      rejection (radius < 0, L outside [1, 255], 2r >= min(W, H)) throws the
//      reference's std::invalid_argument with the reference's message;
//   2. the output Image is allocated here and returned by value; the engine
//      keeps no reference to either image after return;
//   3. C status codes map to the reference's exception types: OPC_EINVAL ->
//      std::invalid_argument, OPC_ENOMEM -> std::bad_alloc, OPC_ECUDA ->
//      std::system_error (parallel.hpp:24-25: resource failures).
#include "oilpaint/cuda.hpp"

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <system_error>

#include "oilpaint_b200.h"

namespace oilpaint {

namespace {

void check(int status, const char* what) {
    if (status == OPC_OK) return;
    const std::string msg = std::string(what) + ": " + opc_last_error();
    if (status == OPC_EINVAL) throw std::invalid_argument(msg);
    if (status == OPC_ENOMEM) throw std::bad_alloc();
    throw std::system_error(std::make_error_code(std::errc::io_error), msg);
}

}  // namespace

Image apply_cuda(const Image& img, const FilterParams& params, const CudaConfig& cfg) {
    validate(img, params);
    Image out(img.width(), img.height());
    const int border = params.border == BorderPolicy::CopyInput ? OPC_BORDER_COPY_INPUT
                                                                : OPC_BORDER_ZERO_FILL;
    opc_config c{};
    c.device = cfg.device;
    if (cfg.devices.size() > 1) {
        const std::vector<std::int32_t> devs(cfg.devices.begin(), cfg.devices.end());
        check(opc_filter_rgb8_multi(img.data().data(), out.data().data(), 1, img.width(),
                                    img.height(), params.radius, params.intensity_levels, border,
                                    devs.data(), static_cast<std::int32_t>(devs.size()), &c),
              "apply_cuda");
    } else {
        if (cfg.devices.size() == 1) c.device = cfg.devices[0];
        check(opc_filter_rgb8(img.data().data(), out.data().data(), img.width(), img.height(),
                              params.radius, params.intensity_levels, border, &c),
              "apply_cuda");
    }
    return out;
}

}  // namespace oilpaint
