// Host check of csrc/bitplanes.cuh, the bit-sliced per-bin counters of the
// bit-plane kernel family (planes.cu), against plain per-bin integers:
//  * Csa: 1..15 one-hot masks -> 4 planes == each bin's count of the masks;
//  * planes_update: w + a - d (a, d row histograms <= 15 per bin) == the
//    integer update, for every plane count the kernel instantiates (4..8);
//  * plane_max_bins: the bins holding the largest count, whose lowest is the
//    reference's argmax (filter.hpp:71-82: strict > from bin 0 upwards).
// Build: g++ -std=c++17 -O2 -I paper_1405_1020_b200/csrc tests/cpp/bitplanes_test.cpp
#include <cstdio>
#include <cstdint>
#include <random>

#include "bitplanes.cuh"

using u32 = std::uint32_t;

template <int NP>
static void to_planes(const int (&cnt)[32], u32 (&w)[NP]) {
    for (int k = 0; k < NP; ++k) {
        w[k] = 0;
        for (int b = 0; b < 32; ++b) w[k] |= static_cast<u32>((cnt[b] >> k) & 1) << b;
    }
}

template <int NP>
static int plane_count(const u32 (&w)[NP], int b) {
    int c = 0;
    for (int k = 0; k < NP; ++k) c |= static_cast<int>((w[k] >> b) & 1u) << k;
    return c;
}

template <int N>
static int check_csa(std::mt19937& rng) {
    std::uniform_int_distribution<int> bin(0, 31);
    for (int it = 0; it < 2000; ++it) {
        u32 m[N];
        int cnt[32] = {};
        for (int j = 0; j < N; ++j) {
            const int b = bin(rng);
            m[j] = opc::bin_mask(static_cast<u32>(b) | 0xABCDE00u);  // (only the low 5 bits pick the bin)
            ++cnt[b];
        }
        u32 q[4];
        opc::Csa<N, 0, 4>::run(m, q);
        for (int b = 0; b < 32; ++b) {
            if (plane_count(q, b) != cnt[b]) {
                std::printf("Csa<%d>: bin %d count %d, planes say %d\n", N, b, cnt[b], plane_count(q, b));
                return 1;
            }
        }
    }
    return 0;
}

template <int P>
static int check_update(std::mt19937& rng, int max_count) {
    for (int it = 0; it < 5000; ++it) {
        int w[32], a[32], d[32], want[32];
        for (int b = 0; b < 32; ++b) {
            // a row leaves (d <= w) and a row enters (a), the result stays a count
            w[b] = static_cast<int>(rng() % (max_count + 1));
            d[b] = static_cast<int>(rng() % 16);
            if (d[b] > w[b]) d[b] = w[b];
            a[b] = static_cast<int>(rng() % 16);
            if (w[b] - d[b] + a[b] > max_count) a[b] = max_count - (w[b] - d[b]);
            want[b] = w[b] - d[b] + a[b];
        }
        u32 W[P], A[4], D[4];
        to_planes(w, W);
        to_planes(a, A);
        to_planes(d, D);
        opc::planes_update<P>(W, A, D);
        for (int b = 0; b < 32; ++b) {
            if (plane_count(W, b) != want[b]) {
                std::printf("planes_update<%d>: bin %d want %d got %d\n", P, b, want[b], plane_count(W, b));
                return 1;
            }
        }
        u32 W2[P];
        to_planes(w, W2);
        opc::planes_add<P>(W2, A);
        for (int b = 0; b < 32; ++b) {
            if (plane_count(W2, b) != ((w[b] + a[b]) & ((1 << P) - 1))) {
                std::printf("planes_add<%d>: bin %d\n", P, b);
                return 1;
            }
        }
    }
    return 0;
}

template <int P>
static int check_max(std::mt19937& rng, int max_count) {
    for (int it = 0; it < 5000; ++it) {
        int cnt[32] = {};
        const int nbins = 1 + static_cast<int>(rng() % 32);
        // ties are common in the filter's windows: draw from a narrow range
        const int span = 1 + static_cast<int>(rng() % (max_count + 1));
        for (int b = 0; b < nbins; ++b) cnt[b] = static_cast<int>(rng() % span) + (it & 1 ? 0 : 1);
        u32 W[P];
        to_planes(cnt, W);
        const u32 cand = opc::plane_max_bins<P>(W);
        int best = 0;  // the reference's scan: strict > keeps the lowest bin
        for (int b = 1; b < 32; ++b) {
            if (cnt[b] > cnt[best]) best = b;
        }
        u32 want = 0;
        for (int b = 0; b < 32; ++b) {
            if (cnt[b] == cnt[best]) want |= 1u << b;
        }
        if (cand != want || __builtin_ctz(cand) != best) {
            std::printf("plane_max_bins<%d>: want %08x (lowest %d), got %08x\n", P, want, best, cand);
            return 1;
        }
    }
    return 0;
}

int main() {
    std::mt19937 rng(12345);
    int fails = 0;
    fails += check_csa<1>(rng) + check_csa<3>(rng) + check_csa<5>(rng) + check_csa<7>(rng) +
             check_csa<9>(rng) + check_csa<11>(rng) + check_csa<13>(rng) + check_csa<15>(rng) +
             check_csa<2>(rng) + check_csa<4>(rng) + check_csa<8>(rng) + check_csa<14>(rng);
    // plane counts of r = 1..7: (2r+1)^2 = 9, 25, 49, 81, 121, 169, 225
    fails += check_update<4>(rng, 9) + check_update<5>(rng, 25) + check_update<6>(rng, 49) +
             check_update<7>(rng, 81) + check_update<7>(rng, 121) + check_update<8>(rng, 169) +
             check_update<8>(rng, 225);
    fails += check_max<4>(rng, 9) + check_max<5>(rng, 25) + check_max<7>(rng, 121) + check_max<8>(rng, 225);
    std::printf("%d failures\n", fails);
    return fails ? 1 : 0;
}
