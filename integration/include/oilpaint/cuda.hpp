// oilpaint/cuda.hpp -- the B200 engine as a reference-native component.
//
// Drops into the reference library next to apply_sequential
// (proj/include/oilpaint/filter.hpp:109) and apply_parallel
// (proj/include/oilpaint/parallel.hpp:33): same Image and FilterParams types,
// same ownership (input by const&, new Image returned by value), same error
// behaviour (the reference validate runs first and throws
// std::invalid_argument; resource failures throw std::system_error /
// std::bad_alloc like parallel.hpp:24-25).  Compiled against the reference
// headers and linked with liboilpaint_b200.so (the C-ABI in
// include/oilpaint_b200.h); see INTEGRATION.md.
#pragma once

#include <vector>

#include "oilpaint/filter.hpp"
#include "oilpaint/image.hpp"

namespace oilpaint {

// The CUDA analogue of ParallelConfig (parallel.hpp:10-17).
struct CudaConfig {
    // CUDA device for a single-device call; -1 = the current device.
    int device = -1;
    // Two or more entries: the interior rows are split into that many
    // contiguous bands with r-row halos, one per entry (ordinals may repeat:
    // {0, 0, 0} runs three bands on device 0).  The output is byte-identical
    // to the single-device call, as apply_parallel's is for every worker count.
    std::vector<int> devices;
};

// Output byte-identical to apply_sequential(img, params) for every cfg.
Image apply_cuda(const Image& img, const FilterParams& params, const CudaConfig& cfg = {});

}  // namespace oilpaint
