// sweep_cuda -- the reference's size x radius sweep (run_sweep + write_csv,
// proj/src/bench.cpp:78-166) with the CUDA engine as the contender of the
// sequential engine: the reference harness itself, built from the staged
// reference sources with integration/patches/engine-cuda.patch applied
// (EngineKind::Cuda, proj/include/oilpaint/bench.hpp:12).  Prints the
// reference CSV (records, blank line, pairs with improvement_pct).
//
//   sweep_cuda [--sizes vga,xga,...] [--radii 2,4,...] [--levels 20] [--reps 5]
//              [--engine cuda|par]
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "oilpaint/bench.hpp"

namespace {

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream in(s);
    std::string item;
    while (std::getline(in, item, ',')) {
        if (!item.empty()) out.push_back(item);
    }
    return out;
}

int to_int(const std::string& s) {
    std::size_t used = 0;
    const int v = std::stoi(s, &used);
    if (used != s.size()) throw std::invalid_argument("not an integer: " + s);
    return v;
}

}  // namespace

int main(int argc, char** argv) {
    std::string sizes_arg = "vga,svga,xga,fhd,wqxga", radii_arg = "2,4,6,8", engine = "cuda";
    int levels = 20, reps = 5;
    try {
        for (int i = 1; i + 1 < argc; i += 2) {
            const std::string k = argv[i], v = argv[i + 1];
            if (k == "--sizes") sizes_arg = v;
            else if (k == "--radii") radii_arg = v;
            else if (k == "--levels") levels = to_int(v);
            else if (k == "--reps") reps = to_int(v);
            else if (k == "--engine") engine = v;
            else throw std::invalid_argument("unknown option " + k);
        }
        if (argc % 2 == 0) throw std::invalid_argument("options take one value each");
        std::vector<oilpaint::SizeSpec> sizes;
        for (const std::string& label : split(sizes_arg)) {
            const auto size = oilpaint::find_standard_size(label);
            if (!size) throw std::invalid_argument("unknown size " + label);
            sizes.push_back(*size);
        }
        std::vector<int> radii;
        for (const std::string& r : split(radii_arg)) radii.push_back(to_int(r));
        if (engine != "cuda" && engine != "par") throw std::invalid_argument("engine cuda|par");
        const oilpaint::EngineKind contender =
            engine == "cuda" ? oilpaint::EngineKind::Cuda : oilpaint::EngineKind::Parallel;
        const oilpaint::BenchReport report =
            oilpaint::run_sweep(sizes, radii, levels, reps, {}, contender);
        std::fputs(oilpaint::write_csv(report).c_str(), stdout);
        return 0;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
