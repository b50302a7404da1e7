// gen.cu -- on-device input generation: the reference
// patterns of proj/src/pattern.cpp:19-88 and the config 2/3/5 generators
// written straight into device memory, byte-identical to opc_generate
// (patterns.cpp) on the host (the generator parameters come from the same host
// functions, gen_spec.h).  Harness code, not
// on the measured path; it saves the host generation and the H2D copy of large
// synthetic inputs (config 4: 805 MB).
#include <cstdint>
#include <mutex>

#include "../../include/oilpaint_b200_patterns.h"
#include "gen_spec.h"
#include "kernels.cuh"

namespace opc {

namespace {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Noise{seed}: byte i = byte (i mod 8) of word i / 8 of the splitmix64 stream
// seeded with `seed` (pattern.cpp:11-17, 64-76); word k = mix(seed + (k+1) gamma).
// One thread per 8-byte word.
__global__ void noise_kernel(std::uint64_t seed, std::uint8_t* out, std::size_t n) {
    const std::size_t k = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x;
    const std::size_t i0 = k * 8;
    if (i0 >= n) return;
    const std::uint64_t word = mix64(seed + (k + 1) * kGamma);
    if (i0 + 8 <= n && (reinterpret_cast<std::uintptr_t>(out + i0) & 7) == 0) {
        *reinterpret_cast<std::uint64_t*>(out + i0) = word;  // little-endian byte order
        return;
    }
    for (std::size_t i = i0; i < n && i < i0 + 8; ++i) {
        out[i] = static_cast<std::uint8_t>(word >> (8 * (i - i0)));
    }
}

// Gradient, Uniform{rgb}, Checker{cell, white, black}: one thread per pixel,
// the formulas of patterns.cpp (pattern.cpp:19-62).
__global__ void pixel_kernel(int kind, std::uint64_t seed, int w, int h, std::uint8_t* out) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= static_cast<long long>(w) * h) return;
    const int y = static_cast<int>(p / w), x = static_cast<int>(p - static_cast<long long>(y) * w);
    std::uint8_t r, g, b;
    if (kind == OPC_PATTERN_GRADIENT) {
        const int dx = w > 1 ? w - 1 : 1, dy = h > 1 ? h - 1 : 1;
        const int dd = w + h > 2 ? w + h - 2 : 1;
        r = static_cast<std::uint8_t>(x * 255 / dx);
        g = static_cast<std::uint8_t>(y * 255 / dy);
        b = static_cast<std::uint8_t>((x + y) * 255 / dd);
    } else if (kind == OPC_PATTERN_UNIFORM) {
        r = static_cast<std::uint8_t>(seed);
        g = static_cast<std::uint8_t>(seed >> 8);
        b = static_cast<std::uint8_t>(seed >> 16);
    } else {  // checker, cell = seed
        const int cell = static_cast<int>(seed);
        r = g = b = ((x / cell) + (y / cell)) % 2 == 0 ? 255 : 0;
    }
    std::uint8_t* o = out + p * 3;
    o[0] = r;
    o[1] = g;
    o[2] = b;
}

// Config 2 / 5 fields (patterns.cpp smooth_field): one thread per pixel.
__device__ std::int32_t g_sine[4096];
__device__ std::int32_t g_gauss[65536];

__global__ void smooth_kernel(SmoothSpec sp, int w, int h, int gaussian, std::uint8_t* out) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= static_cast<long long>(w) * h) return;
    const int y = static_cast<int>(p / w), x = static_cast<int>(p - static_cast<long long>(y) * w);
    const std::uint64_t pix = static_cast<std::uint64_t>(p);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        long long s = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const GenWave& wv = sp.waves[4 * c + k];
            const std::uint32_t phase = wv.px * static_cast<std::uint32_t>(x) +
                                        wv.py * static_cast<std::uint32_t>(y) + wv.ph;
            s += static_cast<long long>(wv.amp) * g_sine[phase >> 20];
        }
        int v = 128 + static_cast<int>((s * 255) >> 30);
        const std::uint64_t word = mix64(sp.noise_seed + (pix * 3 + c + 1) * kGamma);
        v += gaussian ? (g_gauss[word & 0xFFFFu] + 128) >> 8 : static_cast<int>(word % 17) - 8;
        out[pix * 3 + c] = static_cast<std::uint8_t>(min(max(v, 0), 255));
    }
}

// Config 3 (patterns.cpp rects): one thread per pixel, the last rectangle
// covering it wins.
__global__ void rects_kernel(RectsSpec sp, int w, int h, std::uint8_t* out) {
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= static_cast<long long>(w) * h) return;
    const int y = static_cast<int>(p / w), x = static_cast<int>(p - static_cast<long long>(y) * w);
    std::uint32_t rgb = sp.bg;
    for (int i = 0; i < 64; ++i) {
        const GenRect& q = sp.rects[i];
        if (x >= q.x0 && x <= q.x1 && y >= q.y0 && y <= q.y1) rgb = q.rgb;
    }
    std::uint8_t* o = out + p * 3;
    o[0] = static_cast<std::uint8_t>(rgb);
    o[1] = static_cast<std::uint8_t>(rgb >> 8);
    o[2] = static_cast<std::uint8_t>(rgb >> 16);
}

// The sine / Gaussian tables are copied once per device (the host tables are
// the patterns.cpp ones, so both generators index identical values).
cudaError_t ensure_tables(cudaStream_t s) {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
    e = cudaMemcpyToSymbolAsync(g_sine, sine_table_data(), sizeof(g_sine), 0, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        e = cudaMemcpyToSymbolAsync(g_gauss, gauss_table_data(), sizeof(g_gauss), 0,
                                    cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
    return e;
}

}  // namespace

// -1: kind not available on the device; 1: invalid argument.
int launch_generate(int kind, std::uint64_t seed, int w, int h, std::uint8_t* out, cudaStream_t s,
                    cudaError_t* err) {
    *err = cudaSuccess;
    if (w < 1 || h < 1 || !out) return 1;
    const std::size_t n = static_cast<std::size_t>(w) * h * 3;
    if (kind == OPC_PATTERN_NOISE) {
        const std::size_t words = (n + 7) / 8;
        noise_kernel<<<static_cast<unsigned>((words + 255) / 256), 256, 0, s>>>(seed, out, n);
    } else if (kind == OPC_PATTERN_GRADIENT || kind == OPC_PATTERN_UNIFORM ||
               kind == OPC_PATTERN_CHECKER) {
        if (kind == OPC_PATTERN_CHECKER && static_cast<long long>(seed) < 1) return 1;
        const long long px = static_cast<long long>(w) * h;
        pixel_kernel<<<static_cast<unsigned>((px + 255) / 256), 256, 0, s>>>(kind, seed, w, h, out);
    } else if (kind == OPC_PATTERN_SMOOTH || kind == OPC_PATTERN_VIDEO) {
        // (VIDEO: the frame is folded into the seed by the caller, seed + frame)
        *err = ensure_tables(s);
        if (*err != cudaSuccess) return 0;
        SmoothSpec sp;
        smooth_spec(seed, w, h, &sp);
        const long long px = static_cast<long long>(w) * h;
        smooth_kernel<<<static_cast<unsigned>((px + 255) / 256), 256, 0, s>>>(
            sp, w, h, kind == OPC_PATTERN_VIDEO ? 1 : 0, out);
    } else if (kind == OPC_PATTERN_RECTS) {
        RectsSpec sp;
        rects_spec(seed, w, h, &sp);
        const long long px = static_cast<long long>(w) * h;
        rects_kernel<<<static_cast<unsigned>((px + 255) / 256), 256, 0, s>>>(sp, w, h, out);
    } else {
        return -1;
    }
    *err = cudaGetLastError();
    return 0;
}

}  // namespace opc
