// oilbench_cuda -- command-line front end of the CUDA engine, mirroring the
// reference CLI `oilbench` (proj/tools/oilbench.cpp): subcommands apply, gen
// and bench over binary PPM files, and the reference's exit codes
// (oilbench.cpp:3-4): 0 success, 1 usage error, 2 I/O, parse or runtime error,
// 3 filter parameter error (std::invalid_argument).
//
//   apply --input IN --output OUT [--radius 2] [--levels 20] [--engine cuda]
//         [--border copy|zero] [--devices 0,1,...]
//   gen   --pattern uniform|gradient|checker|noise --width W --height H
//         [--seed S] --output OUT
//   bench [--sizes vga,svga,xga,fhd,wqxga,WxH] [--radii 2,4,6,8] [--levels 20]
//         [--reps 5] [--out FILE|-] [--baseline REF.csv] [--devices 0,1,...]
//
// `bench` is the reference sweep (bench.cpp:78-132: Noise{1} workload per size,
// one untimed warm-up, `reps` timed calls of the host-to-host engine call,
// lower median) for the CUDA engine, written in the reference CSV layout
// (bench.hpp:71-75) with engine "cuda".  With --baseline (a CSV written by the
// reference's `oilbench bench`), the pair rows give the reference sequential
// median as t1, the CUDA median as t2 and improvement_pct = 100 (t1 - t2) / t1
// (bench.cpp:67-72) -- the paper's size x radius tables with a GPU column.
// The CPU engines themselves live in the reference; this tool only runs CUDA.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "oilpaint_b200.hpp"
#include "oilpaint_b200_patterns.h"
#include "oilpaint_b200_ppm.hpp"

namespace {

using oilpaint_b200::Image;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// --name value / --name=value options of one subcommand.
class Options {
  public:
    Options(int argc, char** argv, int first, const std::vector<std::string>& known) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
            std::string name = a.substr(2), value;
            const auto eq = name.find('=');
            if (eq != std::string::npos) {
                value = name.substr(eq + 1);
                name = name.substr(0, eq);
            } else {
                if (i + 1 >= argc) throw UsageError("--" + name + " needs a value");
                value = argv[++i];
            }
            if (std::find(known.begin(), known.end(), name) == known.end()) {
                throw UsageError("unknown option --" + name);
            }
            if (values_.count(name)) throw UsageError("--" + name + " given twice");
            values_[name] = value;
        }
    }
    bool has(const std::string& n) const { return values_.count(n) != 0; }
    std::string str(const std::string& n, const std::string& def = "") const {
        auto it = values_.find(n);
        return it == values_.end() ? def : it->second;
    }
    std::string required(const std::string& n) const {
        if (!has(n)) throw UsageError("--" + n + " is required");
        return str(n);
    }
    long long integer(const std::string& n, long long def, long long lo, long long hi) const {
        if (!has(n)) return def;
        return parse_int(str(n), n, lo, hi);
    }
    static long long parse_int(const std::string& s, const std::string& n, long long lo,
                               long long hi) {
        char* end = nullptr;
        const long long v = std::strtoll(s.c_str(), &end, 10);
        if (s.empty() || *end != '\0') throw UsageError("--" + n + ": '" + s + "' is not an integer");
        if (v < lo || v > hi) {
            throw UsageError("--" + n + ": " + s + " not in [" + std::to_string(lo) + ", " +
                             std::to_string(hi) + "]");
        }
        return v;
    }
    std::vector<std::string> list(const std::string& n) const {
        std::vector<std::string> out;
        std::stringstream ss(str(n));
        std::string tok;
        while (std::getline(ss, tok, ',')) {
            if (!tok.empty()) out.push_back(tok);
        }
        return out;
    }

  private:
    std::map<std::string, std::string> values_;
};

oilpaint_b200::CudaConfig make_config(const Options& o) {
    oilpaint_b200::CudaConfig cfg;
    for (const std::string& d : o.list("devices")) {
        cfg.devices.push_back(static_cast<int>(Options::parse_int(d, "devices", 0, 1 << 16)));
    }
    return cfg;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

int run_apply(const Options& o) {
    const std::string in = o.required("input"), out = o.required("output");
    oilpaint_b200::FilterParams p;
    p.radius = static_cast<int>(o.integer("radius", 2, 0, 1 << 20));
    p.intensity_levels = static_cast<int>(o.integer("levels", 20, 1, 255));
    const std::string engine = o.str("engine", "cuda");
    if (engine != "cuda") {
        throw UsageError("--engine: '" + engine +
                         "' is a reference CPU engine (seq, par); this tool runs cuda");
    }
    const std::string border = o.str("border", "copy");
    if (border != "copy" && border != "zero") throw UsageError("--border: want copy or zero");
    p.border = border == "zero" ? oilpaint_b200::BorderPolicy::ZeroFill
                                : oilpaint_b200::BorderPolicy::CopyInput;
    const Image img = oilpaint_b200::load_ppm(in);
    const double t0 = now_ms();
    const Image res = oilpaint_b200::apply_cuda(img, p, make_config(o));
    const double ms = now_ms() - t0;
    oilpaint_b200::save_ppm(res, out);
    std::fprintf(stderr, "width=%d height=%d time_process_ms=%.3f\n", img.width(), img.height(), ms);
    return 0;
}

Image generate(int kind, std::uint64_t seed, int w, int h) {
    Image img(w, h);
    if (opc_generate(kind, seed, w, h, 0, img.data().data(), 0) != 0) {
        throw std::invalid_argument("pattern generator rejected its arguments");
    }
    return img;
}

int run_gen(const Options& o) {
    const std::string pattern = o.required("pattern");
    const int w = static_cast<int>(Options::parse_int(o.required("width"), "width", 1, 1 << 20));
    const int h = static_cast<int>(Options::parse_int(o.required("height"), "height", 1, 1 << 20));
    const std::string out = o.required("output");
    const std::uint64_t seed = static_cast<std::uint64_t>(o.integer("seed", 0, 0, LLONG_MAX));
    int kind;
    std::uint64_t arg = seed;
    if (pattern == "uniform") {
        kind = OPC_PATTERN_UNIFORM;
        arg = 0x808080;  // oilbench gen: Uniform{{128, 128, 128}}
    } else if (pattern == "gradient") {
        kind = OPC_PATTERN_GRADIENT;
    } else if (pattern == "checker") {
        kind = OPC_PATTERN_CHECKER;
        arg = 8;  // Checker{} defaults: 8-pixel cells, white / black
    } else if (pattern == "noise") {
        kind = OPC_PATTERN_NOISE;
    } else {
        throw UsageError("--pattern: want uniform, gradient, checker or noise");
    }
    oilpaint_b200::save_ppm(generate(kind, arg, w, h), out);
    return 0;
}

struct Size {
    std::string label;
    int w, h;
};

const std::vector<Size>& standard_sizes() {  // bench.cpp:37-44
    static const std::vector<Size> s = {{"VGA", 640, 480},   {"SVGA", 800, 600}, {"XGA", 1024, 768},
                                        {"FHD", 1920, 1080}, {"WQXGA", 2560, 1600}};
    return s;
}

Size parse_size(const std::string& tok) {
    std::string low = tok;
    for (char& c : low) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    for (const Size& s : standard_sizes()) {
        std::string l = s.label;
        for (char& c : l) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
        if (l == low) return s;
    }
    const auto x = low.find('x');
    if (x != std::string::npos && x > 0 && x + 1 < low.size()) {
        char* e1 = nullptr;
        char* e2 = nullptr;
        const long w = std::strtol(low.substr(0, x).c_str(), &e1, 10);
        const std::string hs = low.substr(x + 1);
        const long h = std::strtol(hs.c_str(), &e2, 10);
        if (*e1 == '\0' && *e2 == '\0' && w >= 1 && h >= 1) return {tok, static_cast<int>(w), static_cast<int>(h)};
    }
    throw UsageError("--sizes: unknown size '" + tok + "' (want vga/svga/xga/fhd/wqxga or WxH)");
}

double lower_median(std::vector<double> v) {  // bench.cpp:74-78
    std::sort(v.begin(), v.end());
    return v[(v.size() - 1) / 2];
}

std::string fixed6(double v) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.6f", v);
    return b;
}

// (label, radius) -> sequential median of a reference `oilbench bench` CSV.
std::map<std::pair<std::string, int>, double> read_baseline(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::map<std::pair<std::string, int>, double> t1;
    std::string line;
    std::getline(in, line);  // record header
    while (std::getline(in, line) && !line.empty()) {
        std::vector<std::string> f;
        std::stringstream ss(line);
        std::string tok;
        while (std::getline(ss, tok, ',')) f.push_back(tok);
        if (f.size() != 10) throw std::runtime_error(path + ": bad record row '" + line + "'");
        if (f[5] == "seq") t1[{f[0], std::atoi(f[3].c_str())}] = std::atof(f[7].c_str());
    }
    return t1;
}

int run_bench(const Options& o) {
    std::vector<Size> sizes;
    if (o.has("sizes")) {
        for (const std::string& t : o.list("sizes")) sizes.push_back(parse_size(t));
    } else {
        sizes = standard_sizes();
    }
    std::vector<int> radii = {2, 4, 6, 8};
    if (o.has("radii")) {
        radii.clear();
        for (const std::string& t : o.list("radii")) {
            radii.push_back(static_cast<int>(Options::parse_int(t, "radii", 0, 1 << 20)));
        }
    }
    const int levels = static_cast<int>(o.integer("levels", 20, 1, 255));
    const int reps = static_cast<int>(o.integer("reps", 5, 1, 1000));
    std::map<std::pair<std::string, int>, double> base;
    if (o.has("baseline")) base = read_baseline(o.str("baseline"));
    const oilpaint_b200::CudaConfig cfg = make_config(o);

    std::string csv = "label,width,height,radius,levels,engine,reps,median_ms,min_ms,max_ms\n";
    std::string pairs = "label,radius,t1_ms,t2_ms,improvement_pct\n";
    for (const Size& s : sizes) {
        const Image work = generate(OPC_PATTERN_NOISE, 1, s.w, s.h);  // bench.cpp:16, 86-89
        for (const int r : radii) {
            oilpaint_b200::FilterParams p;
            p.radius = r;
            p.intensity_levels = levels;
            oilpaint_b200::validate(work, p);
            oilpaint_b200::apply_cuda(work, p, cfg);  // warm-up, untimed
            std::vector<double> t;
            for (int i = 0; i < reps; ++i) {
                const double t0 = now_ms();
                oilpaint_b200::apply_cuda(work, p, cfg);
                t.push_back(now_ms() - t0);
            }
            const double med = lower_median(t);
            csv += s.label + "," + std::to_string(s.w) + "," + std::to_string(s.h) + "," +
                   std::to_string(r) + "," + std::to_string(levels) + ",cuda," + std::to_string(reps) +
                   "," + fixed6(med) + "," + fixed6(*std::min_element(t.begin(), t.end())) + "," +
                   fixed6(*std::max_element(t.begin(), t.end())) + "\n";
            auto it = base.find({s.label, r});
            if (it != base.end() && it->second > 0) {
                const double imp = 100.0 * (it->second - med) / it->second;
                pairs += s.label + "," + std::to_string(r) + "," + fixed6(it->second) + "," +
                         fixed6(med) + "," + fixed6(imp) + "\n";
                std::fprintf(stderr, "label=%s radius=%d t1_ms=%.3f t2_ms=%.3f improvement_pct=%.2f\n",
                             s.label.c_str(), r, it->second, med, imp);
            } else {
                std::fprintf(stderr, "label=%s radius=%d cuda_median_ms=%.3f\n", s.label.c_str(), r, med);
            }
        }
    }
    const std::string text = csv + "\n" + pairs;
    const std::string out = o.str("out");
    if (out.empty() || out == "-") {
        std::cout << text;
        return 0;
    }
    std::ofstream f(out, std::ios::binary | std::ios::trunc);
    if (!f) throw std::runtime_error("cannot open " + out + " for writing");
    f << text;
    if (!f) throw std::runtime_error("write failed on " + out);
    return 0;
}

const char* kUsage =
    "usage: oilbench_cuda <apply|gen|bench> [options]\n"
    "  apply --input IN --output OUT [--radius 2] [--levels 20] [--engine cuda]\n"
    "        [--border copy|zero] [--devices 0,1,...]\n"
    "  gen   --pattern uniform|gradient|checker|noise --width W --height H [--seed S] --output OUT\n"
    "  bench [--sizes vga,svga,xga,fhd,wqxga,WxH] [--radii 2,4,6,8] [--levels 20] [--reps 5]\n"
    "        [--out FILE|-] [--baseline REF.csv] [--devices 0,1,...]\n";

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && (std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h")) {
        std::cout << kUsage;
        return 0;
    }
    try {
        if (argc < 2) throw UsageError("a subcommand is required");
        const std::string cmd = argv[1];
        for (int i = 2; i < argc; ++i) {
            const std::string a = argv[i];
            if (a == "--threads" || a.rfind("--threads=", 0) == 0) {
                // the reference CLI's worker count belongs to its CPU engines
                // (oilbench.cpp --engine par); the GPU engine has no thread knob
                throw UsageError("--threads selects CPU workers of the reference engines; the "
                                 "cuda engine does not take it (use --devices)");
            }
        }
        if (cmd == "apply") {
            return run_apply(Options(argc, argv, 2, {"input", "output", "radius", "levels", "engine",
                                                     "border", "devices"}));
        }
        if (cmd == "gen") {
            return run_gen(Options(argc, argv, 2, {"pattern", "width", "height", "seed", "output"}));
        }
        if (cmd == "bench") {
            return run_bench(Options(argc, argv, 2, {"sizes", "radii", "levels", "reps", "out",
                                                     "baseline", "devices"}));
        }
        throw UsageError("unknown subcommand '" + cmd + "'");
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n\n" << kUsage << std::flush;
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
