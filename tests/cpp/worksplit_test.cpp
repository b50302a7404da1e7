// Host check of csrc/worksplit.cuh: for many launch shapes, the chunks of a
// WorkSplit cover every (frame, band, interior column) exactly once, passes
// never cross a band end, and chunk counts stay within int range.
// Build: g++ -std=c++17 -O2 -I paper_1405_1020_b200/csrc tests/cpp/worksplit_test.cpp
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "worksplit.cuh"

static int check_split(const opc::WorkSplit& g, int frames, int nbands, int iw, long long max_chunks,
                       bool one_pass);

static int check(int frames, int nbands, int iw, long long blocks, int wpb, int pct, long long minc,
                 int dyn, int guided) {
    const opc::WorkSplit g = opc::make_split(frames, nbands, iw, blocks * wpb, pct, minc, dyn, guided);
    int fails = check_split(g, frames, nbands, iw, -1, false);
    // the band-aligned split of small shares: every unit once, at most one
    // chunk per resident warp, every chunk a single pass
    opc::WorkSplit a = g;
    if (opc::make_aligned_split(frames, nbands, iw, blocks * wpb, static_cast<int>(minc), a)) {
        fails += check_split(a, frames, nbands, iw, blocks * wpb, true);
    }
    return fails;
}

static int check_split(const opc::WorkSplit& g, int frames, int nbands, int iw, long long max_chunks,
                       bool one_pass) {
    if (max_chunks >= 0 && g.nchunks > max_chunks) {
        std::printf("aligned split: %d chunks for %lld warps\n", g.nchunks, max_chunks);
        return 1;
    }
    std::vector<unsigned char> seen(static_cast<std::size_t>(frames) * nbands * iw, 0);
    long long passes = 0;
    // chunks as the kernels claim them: indexed chunks, then (guided mode)
    // pieces of the unit counter, claimed one after another here
    std::vector<std::pair<long long, long long>> chunks;
    for (int i = 0; i < g.nchunks; ++i) {
        long long u, u_end;
        opc::chunk_range(g, i, u, u_end);
        chunks.push_back({u, u_end});
    }
    if (g.guided_div > 0) {
        const long long base = static_cast<long long>(g.nstatic) * g.s1;
        for (long long claimed = 0;;) {
            const long long size = opc::guided_size(g, claimed);
            const long long a = base + claimed, b = a + size < g.units ? a + size : g.units;
            if (a >= b) break;
            chunks.push_back({a, b});
            claimed += size;
        }
    }
    for (auto [u, u_end] : chunks) {
        int f, kb, x0, x1;
        int chunk_passes = 0;
        while (opc::pass_in_chunk(g, u, u_end, f, kb, x0, x1)) {
            ++passes;
            if (one_pass && ++chunk_passes > 1) {
                std::printf("aligned split: a chunk of two passes, shape %d/%d/%d\n", frames, nbands, iw);
                return 1;
            }
            if (f < 0 || f >= frames || kb < 0 || kb >= nbands || x0 < 0 || x1 > iw || x0 >= x1) {
                std::printf("bad pass f=%d kb=%d [%d,%d) shape %d/%d/%d\n", f, kb, x0, x1, frames,
                            nbands, iw);
                return 1;
            }
            for (int x = x0; x < x1; ++x) {
                unsigned char& c = seen[(static_cast<std::size_t>(f) * nbands + kb) * iw + x];
                if (c) {
                    std::printf("unit covered twice: f=%d kb=%d x=%d\n", f, kb, x);
                    return 1;
                }
                c = 1;
            }
        }
    }
    for (std::size_t k = 0; k < seen.size(); ++k) {
        if (!seen[k]) {
            std::printf("unit never covered: %zu of shape %d/%d/%d (nchunks %d)\n", k, frames,
                        nbands, iw, g.nchunks);
            return 1;
        }
    }
    return 0;
}

int main() {
    int fails = 0, n = 0;
    const int frames_[] = {1, 2, 8, 64};
    const int nbands_[] = {1, 3, 34, 128, 512};
    const int iw_[] = {1, 7, 63, 64, 65, 1000, 1910, 4076, 16354};
    const int wpb_[] = {1, 5, 11};
    const long long blocks_[] = {1, 148};
    for (int frames : frames_)
        for (int nbands : nbands_)
            for (int iw : iw_)
                for (int wpb : wpb_)
                    for (long long blocks : blocks_)
                        for (int pct : {0, 50, 98, 100})
                            for (int guided : {0, 4}) {
                                if (static_cast<long long>(frames) * nbands * iw > 20000000) continue;
                                fails += check(frames, nbands, iw, blocks, wpb, pct, 128,
                                               pct == 50 ? 2 : 3, guided);
                                ++n;
                            }
    std::printf("%d shapes, %d failures\n", n, fails);
    return fails ? 1 : 0;
}
