/*
 * oilpaint_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU hot path of the histogram
 * oil-paint filter (arxiv/paper_1405_1020, "oilbench" C++ reimplementation
 * under /root/reference/proj).  It is the parity CHECKER for the CUDA product
 * path, never the product: only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load it.  The product library
 * (paper_1405_1020_b200/liboilpaint_b200.so) does not link or call it.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares this file
 * with the reference build in oracle/_ref (apply_sequential, oracle::filter)
 * through committed fixtures in tests/golden/ and the golden 8x8 PPM produced
 * by the reference's own tests/golden/make_golden.py.
 *
 * Every function cites the reference lines it restates.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENOMEM 3

/* proj/include/oilpaint/filter.hpp:31-35 -- intensity_bin:
 * (unsigned(r)+g+b) * unsigned(L) / 765u, a value in [0, L]. */
int oracle_intensity_bin(uint8_t r, uint8_t g, uint8_t b, int levels) {
    return (int)(((unsigned)r + g + b) * (unsigned)levels / 765u);
}

/* proj/src/filter.cpp:8-26 -- validate.  Returns 0 or ORACLE_EINVAL.
 * max_levels is 255 for the reference contract (filter.cpp:12); the
 * documented L=256 extension of the C-ABI passes 256. */
int oracle_validate(int w, int h, uint64_t nbytes, int radius, int levels, int max_levels) {
    if (w < 1 || h < 1) return ORACLE_EINVAL; /* proj/src/image.cpp:10-16 */
    if (radius < 0) return ORACLE_EINVAL;     /* filter.cpp:9-11 */
    if (levels < 1 || levels > max_levels) return ORACLE_EINVAL; /* filter.cpp:12-15 */
    int min_dim = w < h ? w : h;
    if (2 * radius >= min_dim) return ORACLE_EINVAL; /* filter.cpp:16-22 */
    if (nbytes != (uint64_t)w * (uint64_t)h * 3u) return ORACLE_EINVAL; /* filter.cpp:23-25 */
    return ORACLE_OK;
}

/* Scratch of HistogramAccumulator, proj/include/oilpaint/filter.hpp:38-97:
 * uint32 counts + uint64 channel sums over L+1 bins. */
typedef struct {
    int bins;
    uint32_t* count;
    uint64_t* sum_r;
    uint64_t* sum_g;
    uint64_t* sum_b;
} oracle_hist;

static int hist_init(oracle_hist* h, int levels) {
    h->bins = levels + 1;
    h->count = (uint32_t*)calloc((size_t)h->bins, sizeof(uint32_t));
    h->sum_r = (uint64_t*)calloc((size_t)h->bins, sizeof(uint64_t));
    h->sum_g = (uint64_t*)calloc((size_t)h->bins, sizeof(uint64_t));
    h->sum_b = (uint64_t*)calloc((size_t)h->bins, sizeof(uint64_t));
    return (h->count && h->sum_r && h->sum_g && h->sum_b) ? 0 : -1;
}

static void hist_free(oracle_hist* h) {
    free(h->count);
    free(h->sum_r);
    free(h->sum_g);
    free(h->sum_b);
}

/* proj/src/filter.cpp:28-44 -- filter_pixel: reset (filter.hpp:54-59), add
 * every window pixel (filter.hpp:61-67), lowest-index strict-> max bin
 * (filter.hpp:71-82), truncating quotient (filter.cpp:41-43). */
static void filter_pixel(const uint8_t* in, int w, int x, int y, int radius, int levels,
                         oracle_hist* h, uint8_t* out_px) {
    memset(h->count, 0, sizeof(uint32_t) * (size_t)h->bins);
    memset(h->sum_r, 0, sizeof(uint64_t) * (size_t)h->bins);
    memset(h->sum_g, 0, sizeof(uint64_t) * (size_t)h->bins);
    memset(h->sum_b, 0, sizeof(uint64_t) * (size_t)h->bins);
    for (int ny = y - radius; ny <= y + radius; ++ny) {
        const uint8_t* p = in + ((size_t)ny * (size_t)w + (size_t)(x - radius)) * 3u;
        for (int i = 0; i < 2 * radius + 1; ++i, p += 3) {
            int bin = oracle_intensity_bin(p[0], p[1], p[2], levels);
            h->count[bin] += 1;
            h->sum_r[bin] += p[0];
            h->sum_g[bin] += p[1];
            h->sum_b[bin] += p[2];
        }
    }
    int best = 0;
    uint32_t best_count = h->count[0];
    for (int i = 1; i < h->bins; ++i) {
        if (h->count[i] > best_count) {
            best_count = h->count[i];
            best = i;
        }
    }
    out_px[0] = (uint8_t)(h->sum_r[best] / best_count);
    out_px[1] = (uint8_t)(h->sum_g[best] / best_count);
    out_px[2] = (uint8_t)(h->sum_b[best] / best_count);
}

/* Border initialisation, proj/src/filter.cpp:54 / proj/src/parallel.cpp:113:
 * CopyInput (0) copies the input, ZeroFill (1) zero-fills. */
static void init_output(const uint8_t* in, uint8_t* out, size_t nbytes, int border) {
    if (border == 0) {
        memcpy(out, in, nbytes);
    } else {
        memset(out, 0, nbytes);
    }
}

static int filter_rows(const uint8_t* in, uint8_t* out, int w, int radius, int levels,
                       int row_begin, int row_end) {
    oracle_hist h;
    if (hist_init(&h, levels) != 0) {
        hist_free(&h);
        return ORACLE_ENOMEM;
    }
    for (int y = row_begin; y < row_end; ++y) {
        uint8_t* out_px = out + ((size_t)y * (size_t)w + (size_t)radius) * 3u;
        for (int x = radius; x < w - radius; ++x, out_px += 3) {
            filter_pixel(in, w, x, y, radius, levels, &h, out_px);
        }
    }
    hist_free(&h);
    return ORACLE_OK;
}

/* proj/src/filter.cpp:51-68 -- apply_sequential, without the L<=255 bound
 * (the bound lives in oracle_validate; proj/tests/support/oracle.cpp:7-57 has
 * no bound either, which is what config 3's L=256 relies on). */
int oracle_filter(const uint8_t* in, uint8_t* out, int w, int h, int radius, int levels,
                  int border) {
    if (oracle_validate(w, h, (uint64_t)w * (uint64_t)h * 3u, radius, levels, 256) != 0) {
        return ORACLE_EINVAL;
    }
    init_output(in, out, (size_t)w * (size_t)h * 3u, border);
    return filter_rows(in, out, w, radius, levels, radius, h - radius);
}

typedef struct {
    const uint8_t* in;
    uint8_t* out;
    int w, radius, levels, row_begin, row_end, status;
} band_job;

static void* band_main(void* arg) {
    band_job* j = (band_job*)arg;
    j->status = filter_rows(j->in, j->out, j->w, j->radius, j->levels, j->row_begin, j->row_end);
    return NULL;
}

/* Row-band data parallelism as in proj/src/parallel.cpp:55-132: interior rows
 * split into disjoint contiguous bands, one private histogram per band. */
int oracle_filter_mt(const uint8_t* in, uint8_t* out, int w, int h, int radius, int levels,
                     int border, int threads) {
    if (oracle_validate(w, h, (uint64_t)w * (uint64_t)h * 3u, radius, levels, 256) != 0) {
        return ORACLE_EINVAL;
    }
    init_output(in, out, (size_t)w * (size_t)h * 3u, border);
    int rows = h - 2 * radius;
    if (threads < 1) threads = 1;
    if (threads > rows) threads = rows;
    if (threads <= 1) return filter_rows(in, out, w, radius, levels, radius, h - radius);
    band_job* jobs = (band_job*)calloc((size_t)threads, sizeof(band_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !tids) {
        free(jobs);
        free(tids);
        return ORACLE_ENOMEM;
    }
    int status = ORACLE_OK;
    for (int t = 0; t < threads; ++t) {
        jobs[t].in = in;
        jobs[t].out = out;
        jobs[t].w = w;
        jobs[t].radius = radius;
        jobs[t].levels = levels;
        jobs[t].row_begin = radius + (int)((int64_t)rows * t / threads);
        jobs[t].row_end = radius + (int)((int64_t)rows * (t + 1) / threads);
        if (pthread_create(&tids[t], NULL, band_main, &jobs[t]) != 0) {
            jobs[t].status = filter_rows(in, out, w, radius, levels, jobs[t].row_begin,
                                         jobs[t].row_end);
            tids[t] = 0;
        }
    }
    for (int t = 0; t < threads; ++t) {
        if (tids[t]) pthread_join(tids[t], NULL);
        if (jobs[t].status != ORACLE_OK) status = jobs[t].status;
    }
    free(jobs);
    free(tids);
    return status;
}

/* proj/src/pattern.cpp:11-17 -- splitmix64 step. */
static uint64_t splitmix64(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* proj/src/pattern.cpp:64-76 -- Noise: byte i is byte (i mod 8) of the
 * (i/8)-th splitmix64 word of a generator seeded with seed. */
void oracle_noise(uint64_t seed, uint8_t* out, uint64_t nbytes) {
    uint64_t state = seed;
    uint64_t i = 0;
    while (i < nbytes) {
        uint64_t word = splitmix64(&state);
        for (int k = 0; k < 8 && i < nbytes; ++k, ++i) {
            out[i] = (uint8_t)(word >> (8 * k));
        }
    }
}

/* proj/src/pattern.cpp:33-47 -- Gradient with truncating division. */
void oracle_gradient(int w, int h, uint8_t* out) {
    int dx = w > 1 ? w - 1 : 1;
    int dy = h > 1 ? h - 1 : 1;
    int dd = w + h > 2 ? w + h - 2 : 1;
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            uint8_t* p = out + ((size_t)y * (size_t)w + (size_t)x) * 3u;
            p[0] = (uint8_t)(x * 255 / dx);
            p[1] = (uint8_t)(y * 255 / dy);
            p[2] = (uint8_t)((x + y) * 255 / dd);
        }
    }
}
