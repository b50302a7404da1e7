// bitplanes.cuh -- bit-sliced per-bin counters (the bit-plane family,
// planes.cu), host + device so that tests/cpp/bitplanes_test.cpp checks them
// on the CPU.
//
// A "plane" word holds one bit of up to 32 per-bin counters: bit b of plane
// k is bit k of bin b's count.  Every operation below is a few 3-input logic
// ops (one LOP3 each on the GPU) per plane, for all 32 bins at once.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define OPC_BP_HD __host__ __device__ __forceinline__
#else
#define OPC_BP_HD inline
#endif

namespace opc {

// One-hot mask of a tile entry's bin (the bin in the entry's low 5 bits).
OPC_BP_HD std::uint32_t bin_mask(std::uint32_t e) { return 1u << (e & 31u); }

OPC_BP_HD std::uint32_t maj3(std::uint32_t a, std::uint32_t b, std::uint32_t c) {
    return (a & b) | (a & c) | (b & c);
}

// Carry-save adder tree: N signals of weight 2^K (bit-sliced one-hot masks or
// carries) reduced into plane K of q and N/2 carries of weight 2^(K+1).  For
// one-hot masks the result is each bin's count of the N masks.
template <int N, int K, int NP>
struct Csa {
    OPC_BP_HD static void run(const std::uint32_t* in, std::uint32_t (&q)[NP]) {
        constexpr int NC = N / 2;
        std::uint32_t c[NC];
        std::uint32_t s = in[0];
#pragma unroll
        for (int i = 1, k = 0; i < N; i += 2, ++k) {
            if (i + 1 < N) {  // full adder
                const std::uint32_t x = in[i], y = in[i + 1];
                c[k] = maj3(s, x, y);
                s = s ^ x ^ y;
            } else {  // half adder
                c[k] = s & in[i];
                s ^= in[i];
            }
        }
        q[K] = s;
        Csa<NC, K + 1, NP>::run(c, q);
    }
};
template <int K, int NP>
struct Csa<1, K, NP> {
    OPC_BP_HD static void run(const std::uint32_t* in, std::uint32_t (&q)[NP]) {
        q[K] = in[0];
#pragma unroll
        for (int k = K + 1; k < NP; ++k) q[k] = 0u;
    }
};
template <int K, int NP>
struct Csa<0, K, NP> {
    OPC_BP_HD static void run(const std::uint32_t*, std::uint32_t (&q)[NP]) {
#pragma unroll
        for (int k = K; k < NP; ++k) q[k] = 0u;
    }
};

// w += d (d: 4 planes), modulo 2^P per bin.
template <int P>
OPC_BP_HD void planes_add(std::uint32_t (&w)[P], const std::uint32_t (&d)[4]) {
    std::uint32_t c = 0u;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const std::uint32_t x = k < 4 ? d[k] : 0u, a = w[k];
        w[k] = a ^ x ^ c;
        c = maj3(a, x, c);
    }
}

// w += a - d in one pass, modulo 2^P per bin: w + a + ~d + 1 -- a carry-save
// layer (planes >= 4 of a are 0 and of ~d are 1) and one ripple with carry-in 1.
template <int P>
OPC_BP_HD void planes_update(std::uint32_t (&w)[P], const std::uint32_t (&a)[4], const std::uint32_t (&d)[4]) {
    std::uint32_t s[P], c[P + 1];
    c[0] = 0u;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const std::uint32_t x = w[k], y = k < 4 ? a[k] : 0u, z = k < 4 ? ~d[k] : 0xFFFFFFFFu;
        s[k] = x ^ y ^ z;
        c[k + 1] = maj3(x, y, z);
    }
    std::uint32_t cin = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const std::uint32_t x = s[k], y = c[k];
        w[k] = x ^ y ^ cin;
        cin = maj3(x, y, cin);
    }
}

// The bins holding the largest count (filter.hpp:71-82 takes the lowest of
// them): walk the planes from the top, keeping the candidates that have bit
// k set whenever any does.  (All-zero counts leave every bin a candidate.)
template <int P>
OPC_BP_HD std::uint32_t plane_max_bins(const std::uint32_t (&w)[P]) {
    std::uint32_t cand = 0xFFFFFFFFu;
#pragma unroll
    for (int p = P - 1; p >= 0; --p) {
        const std::uint32_t t = cand & w[p];
        cand = t != 0u ? t : cand;
    }
    return cand;
}

}  // namespace opc
