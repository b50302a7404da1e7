// Acceptance suite for the CUDA engine, in the style of the reference's own
// proj/tests/acceptance.cpp: one PASS/FAIL line per criterion, nonzero exit on
// failure.  It drives the C++ host API (include/oilpaint_b200.hpp) exactly as a
// reference caller would drive apply_sequential / apply_parallel, and checks
// against the CPU oracle (oracle/oilpaint_oracle.c, the checker -- linked only
// into this test binary).
//
//   1  apply_cuda == oracle on 1000 random images, w,h <= 16, r <= 3,
//      L in {1,10,20,255}, both borders           (acceptance.cpp:44-67)
//   2  apply_cuda identical across device-band splits {1,2,4,8 bands on this
//      GPU} and forced kernel families, 200 images up to 128x128, r <= 5
//                                                  (acceptance.cpp:71-101)
//   6  golden 8x8 gradient, r=2, L=20, ZeroFill reproduces the committed PPM
//                                                  (acceptance.cpp:196-218)
//   V  validate: reference exceptions for bad parameters (test_filter.cpp:293-304)
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iterator>
#include <random>
#include <string>
#include <vector>

#include "oilpaint_b200.hpp"

extern "C" int oracle_filter(const uint8_t* in, uint8_t* out, int w, int h, int radius, int levels,
                             int border);

using namespace oilpaint_b200;

namespace {

struct Outcome {
    bool ok;
    std::string detail;
};

Image random_image(std::mt19937_64& rng, int w, int h) {
    std::vector<std::uint8_t> data(static_cast<std::size_t>(w) * h * 3);
    for (auto& b : data) b = static_cast<std::uint8_t>(rng());
    return Image(w, h, std::move(data));
}

Image oracle(const Image& img, const FilterParams& p) {
    Image out(img.width(), img.height());
    oracle_filter(img.data().data(), out.data().data(), img.width(), img.height(), p.radius,
                  p.intensity_levels, p.border == BorderPolicy::CopyInput ? 0 : 1);
    return out;
}

Outcome criterion1() {
    std::mt19937_64 rng(101);
    const int levels_pool[] = {1, 10, 20, 255};
    for (int i = 0; i < 1000; ++i) {
        const int w = 1 + static_cast<int>(rng() % 16), h = 1 + static_cast<int>(rng() % 16);
        const int max_r = std::min(3, (std::min(w, h) - 1) / 2);
        const FilterParams p{static_cast<int>(rng() % (max_r + 1)), levels_pool[rng() % 4],
                             rng() % 2 ? BorderPolicy::ZeroFill : BorderPolicy::CopyInput};
        const Image img = random_image(rng, w, h);
        if (!(apply_cuda(img, p) == oracle(img, p))) {
            return {false, "mismatch at case " + std::to_string(i)};
        }
    }
    return {true, "1000 randomized cases byte-exact vs the oracle"};
}

Outcome criterion2() {
    std::mt19937_64 rng(202);
    const int levels_pool[] = {1, 20, 255};
    for (int i = 0; i < 200; ++i) {
        const int w = 1 + static_cast<int>(rng() % 128), h = 1 + static_cast<int>(rng() % 128);
        const int max_r = std::min(5, (std::min(w, h) - 1) / 2);
        const FilterParams p{static_cast<int>(rng() % (max_r + 1)), levels_pool[rng() % 3],
                             rng() % 2 ? BorderPolicy::ZeroFill : BorderPolicy::CopyInput};
        const Image img = random_image(rng, w, h);
        const Image want = oracle(img, p);
        for (const int bands : {1, 2, 4, 8}) {
            CudaConfig cfg;
            cfg.devices.assign(static_cast<std::size_t>(bands), 0);  // bands on this one GPU
            if (!(apply_cuda(img, p, cfg) == want)) {
                return {false, "divergence at case " + std::to_string(i) + " bands=" +
                                   std::to_string(bands)};
            }
        }
        CudaConfig direct;
        direct.kernel = OPC_KERNEL_DIRECT;
        if (!(apply_cuda(img, p, direct) == want)) {
            return {false, "direct kernel divergence at case " + std::to_string(i)};
        }
    }
    return {true, "200 randomized cases identical across band splits {1,2,4,8} and kernels"};
}

Outcome criterion6(const std::string& golden_path) {
    std::ifstream in(golden_path, std::ios::binary);
    if (!in) return {false, "cannot open " + golden_path};
    const std::vector<std::uint8_t> golden{std::istreambuf_iterator<char>(in),
                                           std::istreambuf_iterator<char>()};
    Image grad(8, 8);
    for (int y = 0; y < 8; ++y) {
        for (int x = 0; x < 8; ++x) {  // proj/src/pattern.cpp:33-47 Gradient
            grad.set(x, y, Rgb{static_cast<std::uint8_t>(x * 255 / 7),
                               static_cast<std::uint8_t>(y * 255 / 7),
                               static_cast<std::uint8_t>((x + y) * 255 / 14)});
        }
    }
    const Image out = apply_cuda(grad, FilterParams{2, 20, BorderPolicy::ZeroFill});
    const std::string header = "P6\n8 8\n255\n";
    std::vector<std::uint8_t> ppm(header.begin(), header.end());
    ppm.insert(ppm.end(), out.data().begin(), out.data().end());
    if (ppm != golden) return {false, "output differs from the golden bytes"};
    return {true, "reproduces the " + std::to_string(golden.size()) + " golden bytes"};
}

Outcome criterion_validate() {
    const Image img(8, 8);
    const FilterParams bad[] = {{4, 20, BorderPolicy::CopyInput},
                                {-1, 20, BorderPolicy::CopyInput},
                                {1, 0, BorderPolicy::CopyInput},
                                {1, 256, BorderPolicy::CopyInput}};
    for (const FilterParams& p : bad) {
        try {
            apply_cuda(img, p);
            return {false, "no exception for r=" + std::to_string(p.radius) + " L=" +
                               std::to_string(p.intensity_levels)};
        } catch (const std::invalid_argument&) {
        }
    }
    apply_cuda(Image(1, 1), FilterParams{0, 20, BorderPolicy::CopyInput});
    apply_cuda(img, FilterParams{3, 20, BorderPolicy::CopyInput});
    return {true, "invalid_argument for the four reference rejections"};
}

}  // namespace

int main(int argc, char** argv) {
    const std::string golden = argc > 1 ? argv[1] : "tests/golden/gradient8_r2_l20_zero.ppm";
    struct C {
        const char* id;
        const char* name;
        std::function<Outcome()> run;
    };
    const std::vector<C> criteria = {
        {"1", "oracle equivalence", criterion1},
        {"2", "band/kernel equivalence", criterion2},
        {"6", "golden file", [&] { return criterion6(golden); }},
        {"V", "validation", criterion_validate},
    };
    int failures = 0;
    for (const C& c : criteria) {
        const auto t0 = std::chrono::steady_clock::now();
        Outcome o{false, ""};
        try {
            o = c.run();
        } catch (const std::exception& e) {
            o = {false, std::string("exception: ") + e.what()};
        }
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("%s  criterion %s  %s: %s (%.1fs)\n", o.ok ? "PASS" : "FAIL", c.id, c.name,
                    o.detail.c_str(), s);
        failures += o.ok ? 0 : 1;
    }
    return failures ? 1 : 0;
}
