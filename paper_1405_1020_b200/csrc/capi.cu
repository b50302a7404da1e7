// capi.cu -- the C-ABI (include/oilpaint_b200.h): validation with the
// reference's rules and messages, per-device contexts (stream + cached device
// buffers behind a mutex), host<->device staging, kernel-family dispatch and
// status/error mapping.
#include <algorithm>
#include <immintrin.h>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/oilpaint_b200.h"
#include "../../include/oilpaint_b200_patterns.h"
#include "kernels.cuh"

#ifndef OPC_HOST_CHUNK_MB
#define OPC_HOST_CHUNK_MB 48  // row chunks of the host-pointer pipeline (single images)
#endif
#ifndef OPC_HOST_SMALL_CHUNKS
#define OPC_HOST_SMALL_CHUNKS 16  // most chunks of a host-pointer image below four 48 MB chunks
#endif
#ifndef OPC_HOST_SMALL_MIN_KB
#define OPC_HOST_SMALL_MIN_KB 6144  // smallest such chunk (per-chunk launch gaps: 2-4 MB chunks measured slower)
#endif

namespace {

thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_error(cudaError_t e, const char* what) {
    const int code = (e == cudaErrorMemoryAllocation) ? OPC_ENOMEM : OPC_ECUDA;
    return set_error(code, std::string(what) + ": " + cudaGetErrorString(e));
}

// proj/src/filter.cpp:8-26 (messages restated) and proj/src/image.cpp:10-16.
int validate_params(int w, int h, unsigned long long nbytes, int radius, int levels,
                    unsigned flags) {
    if (w < 1 || h < 1) {
        return set_error(OPC_EINVAL, "image dimensions must be positive, got " +
                                         std::to_string(w) + "x" + std::to_string(h));
    }
    if (radius < 0) {
        return set_error(OPC_EINVAL, "radius must be >= 0, got " + std::to_string(radius));
    }
    const int max_levels = (flags & OPC_FLAG_ALLOW_LEVELS_256) ? 256 : 255;
    if (levels < 1 || levels > max_levels) {
        return set_error(OPC_EINVAL, "intensity_levels must be in [1, " +
                                         std::to_string(max_levels) + "], got " +
                                         std::to_string(levels));
    }
    const int min_dim = w < h ? w : h;
    if (2LL * radius >= min_dim) {
        return set_error(OPC_EINVAL, "radius " + std::to_string(radius) +
                                         " leaves no interior for a " + std::to_string(w) + "x" +
                                         std::to_string(h) +
                                         " image (need 2*radius < min dimension)");
    }
    if (nbytes != 3ull * static_cast<unsigned long long>(w) * static_cast<unsigned long long>(h)) {
        return set_error(OPC_EINVAL, "image data length does not match its dimensions");
    }
    return OPC_OK;
}

struct DevCtx {
    std::mutex mu;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    void* d_in = nullptr;
    std::size_t in_cap = 0;
    void* d_out = nullptr;
    std::size_t out_cap = 0;
    void* d_scratch = nullptr;  // skew family: sheared entry plane
    std::size_t scratch_cap = 0;
    // The scratch plane is shared by every launch on the device, whatever its
    // stream: a launch on stream s waits for the event recorded after the
    // previous scratch user when that ran on another stream, so two calls in
    // flight on different user streams never overwrite each other's plane.
    cudaEvent_t scratch_ev = nullptr;
    cudaStream_t scratch_stream = nullptr;
    bool scratch_busy = false;
    int* d_counter = nullptr;
    unsigned counter_idx = 0;
    unsigned long long* d_opcounts = nullptr;  // OPC_FLAG_COUNT_OPS accumulators (kOpCountN)
    cudaStream_t s_in = nullptr;   // H2D copies
    cudaStream_t s_out = nullptr;  // D2H copies
    std::vector<cudaEvent_t> ev_in, ev_out, ev_d2h;
    // pinned staging ring for pageable host buffers (only the slots a call
    // uses are allocated: pin_slots of them, pin_cap bytes each)
    static constexpr int kSlots = 3;
    void* pin_in[kSlots] = {};
    void* pin_out[kSlots] = {};
    std::size_t pin_cap = 0;
    int pin_slots = 0;
    cudaEvent_t ev_slot[kSlots] = {};
};

void free_staging(DevCtx* c) {
    for (int k = 0; k < DevCtx::kSlots; ++k) {
        if (c->pin_in[k]) cudaFreeHost(c->pin_in[k]);
        if (c->pin_out[k]) cudaFreeHost(c->pin_out[k]);
        c->pin_in[k] = c->pin_out[k] = nullptr;
    }
    c->pin_cap = 0;
    c->pin_slots = 0;
}

// Orders a scratch-plane launch on stream s after the previous one (see DevCtx).
int scratch_acquire(DevCtx* c, cudaStream_t s) {
    if (!c->scratch_ev) {
        const cudaError_t e = cudaEventCreateWithFlags(&c->scratch_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            g_last_error = std::string("cudaEventCreate(scratch): ") + cudaGetErrorString(e);
            return OPC_ECUDA;
        }
    }
    if (c->scratch_busy && c->scratch_stream != s) {
        const cudaError_t e = cudaStreamWaitEvent(s, c->scratch_ev, 0);
        if (e != cudaSuccess) {
            g_last_error = std::string("cudaStreamWaitEvent(scratch): ") + cudaGetErrorString(e);
            return OPC_ECUDA;
        }
    }
    return OPC_OK;
}

int scratch_release(DevCtx* c, cudaStream_t s) {
    const cudaError_t e = cudaEventRecord(c->scratch_ev, s);
    if (e != cudaSuccess) {
        g_last_error = std::string("cudaEventRecord(scratch): ") + cudaGetErrorString(e);
        return OPC_ECUDA;
    }
    c->scratch_stream = s;
    c->scratch_busy = true;
    return OPC_OK;
}

int ensure_streams(DevCtx* c, std::size_t units) {
    cudaError_t e = cudaSuccess;
    if (!c->s_in) {
        e = cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            g_last_error = std::string("cudaStreamCreate: ") + cudaGetErrorString(e);
            return OPC_ECUDA;
        }
    }
    while (c->ev_in.size() < units) {
        cudaEvent_t a = nullptr, b = nullptr, d = nullptr;
        e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            g_last_error = std::string("cudaEventCreate: ") + cudaGetErrorString(e);
            return OPC_ECUDA;
        }
        c->ev_in.push_back(a);
        c->ev_out.push_back(b);
        c->ev_d2h.push_back(d);
    }
    for (int k = 0; k < DevCtx::kSlots; ++k) {
        if (!c->ev_slot[k]) {
            e = cudaEventCreateWithFlags(&c->ev_slot[k], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                g_last_error = std::string("cudaEventCreate: ") + cudaGetErrorString(e);
                return OPC_ECUDA;
            }
        }
    }
    return OPC_OK;
}

// Streaming (non-temporal) copy: the staging copies touch each byte once, so
// the stores bypass the caches and skip the read-for-ownership of the
// destination (one third of the copy's memory traffic).
__attribute__((target("avx2"))) void copy_stream_avx2(std::uint8_t* dst, const std::uint8_t* src,
                                                     std::size_t n) {
    std::size_t i = 0;
    const std::size_t head = (32 - (reinterpret_cast<std::uintptr_t>(dst) & 31)) & 31;
    if (head) {
        const std::size_t h = std::min(head, n);
        std::memcpy(dst, src, h);
        i = h;
    }
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    _mm_sfence();
    if (i < n) std::memcpy(dst + i, src + i, n - i);
}

#ifndef OPC_COPY_NT
#define OPC_COPY_NT 1
#endif

void copy_bytes(std::uint8_t* dst, const std::uint8_t* src, std::size_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (OPC_COPY_NT && avx2 && n >= 4096) {
        copy_stream_avx2(dst, src, n);
    } else {
        std::memcpy(dst, src, n);
    }
}

// Host memcpy on a pool of worker threads (the pageable-buffer staging copies
// must keep up with PCIe: one thread copies ~10 GB/s, a PCIe direction moves
// ~50 GB/s).  The caller works on the copy too; jobs are shared_ptr-owned so a
// worker that picks a finished job never touches freed memory.
class CopyPool {
  public:
    // One pool per device, so the staging copies of devices filtering
    // concurrently (opc_filter_rgb8_multi from pageable buffers) do not queue
    // behind each other; the host threads are split between the devices.
    static CopyPool& get(int device) {
        static std::mutex mu;
        static std::vector<CopyPool*> pools;  // never destroyed: workers sleep until exit
        std::lock_guard<std::mutex> lk(mu);
        int ndev = 1;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            ndev = 1;
        }
        if (device < 0) device = 0;
        if (pools.size() <= static_cast<std::size_t>(device)) pools.resize(device + 1, nullptr);
        if (!pools[device]) {
            const unsigned hc = std::max(2u, std::thread::hardware_concurrency());
            const unsigned share = (hc - 1) / static_cast<unsigned>(ndev);
            pools[device] = new CopyPool(std::max(1u, std::min(15u, share)));
        }
        return *pools[device];
    }
    void copy(void* dst, const void* src, std::size_t n) {
        constexpr std::size_t kPiece = 2u << 20;
        const std::size_t pieces = std::min<std::size_t>(workers_ + 1, (n + kPiece - 1) / kPiece);
        if (pieces <= 1) {
            copy_bytes(static_cast<std::uint8_t*>(dst), static_cast<const std::uint8_t*>(src), n);
            return;
        }
        auto job = std::make_shared<Job>();
        job->dst = static_cast<std::uint8_t*>(dst);
        job->src = static_cast<const std::uint8_t*>(src);
        job->n = n;
        job->pieces = pieces;
        {
            std::lock_guard<std::mutex> lk(mu_);
            for (std::size_t i = 1; i < pieces; ++i) queue_.push_back(job);
        }
        cv_.notify_all();
        run(*job);
        std::unique_lock<std::mutex> lk(job->mu);
        job->cv.wait(lk, [&] { return job->done == job->pieces; });
    }

  private:
    struct Job {
        std::uint8_t* dst;
        const std::uint8_t* src;
        std::size_t n, pieces;
        std::atomic<std::size_t> next{0};
        std::size_t done = 0;
        std::mutex mu;
        std::condition_variable cv;
    };
    static void run(Job& j) {
        for (;;) {
            const std::size_t i = j.next.fetch_add(1);
            if (i >= j.pieces) return;
            const std::size_t b = j.n * i / j.pieces & ~std::size_t(63);
            const std::size_t e = i + 1 == j.pieces ? j.n : (j.n * (i + 1) / j.pieces & ~std::size_t(63));
            copy_bytes(j.dst + b, j.src + b, e - b);
            std::lock_guard<std::mutex> lk(j.mu);
            if (++j.done == j.pieces) j.cv.notify_all();
        }
    }
    explicit CopyPool(unsigned workers) : workers_(workers) {
        for (unsigned t = 0; t < workers_; ++t) {
            std::thread([this] {
                for (;;) {
                    std::shared_ptr<Job> j;
                    {
                        std::unique_lock<std::mutex> lk(mu_);
                        cv_.wait(lk, [&] { return !queue_.empty(); });
                        j = std::move(queue_.front());
                        queue_.pop_front();
                    }
                    run(*j);
                }
            }).detach();
        }
    }
    unsigned workers_ = 0;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::shared_ptr<Job>> queue_;
};

bool is_pinned_or_device(const void* p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();  // clear
        return false;
    }
    return attr.type != cudaMemoryTypeUnregistered;
}

// ---- live kernel timing (opc_kernel_timing) ----
// Each launch is bracketed by a start and a stop event recorded on the launch
// stream; the open start is keyed by (device, stream, kernel id), so launches
// in flight on different streams or devices never pair up, and events come
// from a per-device pool (an event must live on its stream's device).
struct TimedLaunch {
    int id;
    int device;
    cudaEvent_t start, stop;
};
std::mutex g_timing_mu;
std::vector<TimedLaunch> g_timed;                                    // recorded launches
std::map<int, std::vector<cudaEvent_t>> g_ev_pool;                   // spare events per device
std::map<std::tuple<int, cudaStream_t, int>, cudaEvent_t> g_open;    // start recorded, stop pending

cudaEvent_t take_event(int device) {
    std::vector<cudaEvent_t>& pool = g_ev_pool[device];
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return e;
}

void timing_hook(int id, int phase, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    int device = 0;
    if (cudaGetDevice(&device) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    const auto key = std::make_tuple(device, s, id);
    if (phase == 0) {
        cudaEvent_t ev = take_event(device);
        if (!ev) return;
        if (cudaEventRecord(ev, s) != cudaSuccess) {
            cudaGetLastError();
            g_ev_pool[device].push_back(ev);
            return;
        }
        auto it = g_open.find(key);
        if (it != g_open.end()) g_ev_pool[device].push_back(it->second);  // unmatched start
        g_open[key] = ev;
        return;
    }
    auto it = g_open.find(key);
    if (it == g_open.end()) return;
    cudaEvent_t start = it->second;
    g_open.erase(it);
    cudaEvent_t stop = take_event(device);
    if (!stop || cudaEventRecord(stop, s) != cudaSuccess) {
        cudaGetLastError();
        g_ev_pool[device].push_back(start);
        if (stop) g_ev_pool[device].push_back(stop);
        return;
    }
    g_timed.push_back({id, device, start, stop});
}

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevCtx>> g_ctx;

int get_ctx(int device, DevCtx** out) {
    static std::atomic<int> known_count{0};  // device count once one was seen
    int count = known_count.load();
    cudaError_t e = cudaSuccess;
    if (count == 0) {
        e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            return set_error(OPC_ECUDA, std::string("no CUDA device available: ") +
                                            (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)));
        }
        known_count.store(count);
    }
    if (device < 0) {
        e = cudaGetDevice(&device);
        if (e != cudaSuccess) return cuda_error(e, "cudaGetDevice");
    }
    if (device >= count) {
        return set_error(OPC_EINVAL, "device " + std::to_string(device) + " out of range (" +
                                         std::to_string(count) + " devices)");
    }
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (g_ctx.size() < static_cast<std::size_t>(count)) g_ctx.resize(count);
    if (!g_ctx[device]) {
        auto c = std::make_unique<DevCtx>();
        c->device = device;
        e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
        cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_error(e, "cudaStreamCreate");
        e = cudaMalloc(&c->d_counter, 64 * sizeof(int));
        if (e != cudaSuccess) return cuda_error(e, "cudaMalloc(counter)");
        e = cudaMalloc(&c->d_opcounts, opc::kOpCountN * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemset(c->d_opcounts, 0, opc::kOpCountN * sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_error(e, "cudaMalloc(op counts)");
        g_ctx[device] = std::move(c);
    }
    *out = g_ctx[device].get();
    return OPC_OK;
}

int ensure(void** p, std::size_t* cap, std::size_t need) {
    if (*cap >= need) return OPC_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) return cuda_error(e, "cudaMalloc");
    *cap = need;
    return OPC_OK;
}

// Kernel family for a call.  Auto: the bit-plane
// family for r <= 7 and L+1 <= 32 (video batches with >= 24 bins: skew);
// r = 0 (identity) the column family on small images; direct for r <= 3 with
// many bins on small images, where the O(r^2) scan is cheap and the sliding
// families cannot fill the GPU; then skew for L+1 <= 32, slide for more bins
// (both r <= 15), direct otherwise.  interior_px is per frame.
int plan(int levels, int radius, int forced, long long interior_px, int frames) {
    if (forced == OPC_KERNEL_DIRECT) return OPC_KERNEL_DIRECT;
    if (forced == OPC_KERNEL_SKEW) return opc::skew_supported(levels, radius) ? OPC_KERNEL_SKEW : -1;
    if (forced == OPC_KERNEL_COLUMN) {
        return opc::column_supported(levels, radius) ? OPC_KERNEL_COLUMN : -1;
    }
    if (forced == OPC_KERNEL_SLIDE) {
        return opc::slide_supported(levels, radius) ? OPC_KERNEL_SLIDE : -1;
    }
    if (forced == OPC_KERNEL_PLANES) {
        return opc::planes_supported(levels, radius) ? OPC_KERNEL_PLANES : -1;
    }
    // r <= 7, L+1 <= 32: the bit-plane family, at every size (scripts/size_sweep.py
    // on one B200, noise, L = 20 / 30, 640x480 .. 7680x4320: faster than the
    // column and skew families everywhere).
    // Exception: batches of >= 8 frames with >= 24 bins, i.e. video, go to the
    // skew family, whose per-pass 16-bin window pays on smooth frames
    // (scripts/batch_families.py, 64 x 3840x2160, r = 7, L = 30: smooth skew
    // 6.37 ms / planes 7.01; uniform noise skew 8.48 / planes 7.01).
    if (forced == OPC_KERNEL_AUTO && opc::planes_supported(levels, radius)) {
        if (levels + 1 >= 24 && frames >= 8 && opc::skew_supported(levels, radius)) return OPC_KERNEL_SKEW;
        return OPC_KERNEL_PLANES;
    }
    // (only r = 0 is left here) small images: the column family, while its
    // per-pixel cost stays below the skew family's fill-bound launch
    // (round 1, scripts/size_sweep.py: interior * (2r+1) ~ 50M).
    if (forced == OPC_KERNEL_AUTO && opc::column_supported(levels, radius) &&
        interior_px * (2 * radius + 1) <= 50ll * 1000 * 1000) {
        return OPC_KERNEL_COLUMN;
    }
    if (forced == OPC_KERNEL_AUTO && radius <= 3 && interior_px <= (4ll << 20)) {
        return OPC_KERNEL_DIRECT;
    }
    if (opc::skew_supported(levels, radius)) return OPC_KERNEL_SKEW;
    if (opc::slide_supported(levels, radius)) return OPC_KERNEL_SLIDE;
    return OPC_KERNEL_DIRECT;
}

// Runs the filter on device buffers already holding the band input.
int run_device(const opc::BandArgs& band, int border, int kernel, DevCtx* ctx, cudaStream_t s) {
    // Frames ride on gridDim.z (<= 65535) in the per-frame kernels: larger
    // batches run as consecutive launches of at most that many frames.
    constexpr int kMaxFrames = 65535;
    if (band.frames > kMaxFrames) {
        for (int f0 = 0; f0 < band.frames; f0 += kMaxFrames) {
            opc::BandArgs b = band;
            b.frames = std::min(kMaxFrames, band.frames - f0);
            b.in = band.in + band.in_frame_stride * static_cast<std::size_t>(f0);
            b.out = band.out + band.out_frame_stride * static_cast<std::size_t>(f0);
            const int rc = run_device(b, border, kernel, ctx, s);
            if (rc != OPC_OK) return rc;
        }
        return OPC_OK;
    }
    // (a frame too large for the skew family's 32-bit plane offsets takes the direct family)
    cudaError_t e = cudaSuccess;
    opc::BandArgs a = band;
    a.border = opc::make_border_job(a, border);
    const bool interior = a.y_hi > a.y_lo && a.x_hi > a.x_lo;
    if (kernel == OPC_KERNEL_SKEW && !opc::skew_fits(a)) kernel = OPC_KERNEL_DIRECT;
    if (kernel == OPC_KERNEL_SKEW) {
        // Rotate over 16 task counters (16 bytes each: chunk index + 64-bit
        // unit count) so kernels in flight on different streams never share one.
        int* counter = ctx->d_counter + 4 * (ctx->counter_idx++ & 15u);
        int rc = ensure(&ctx->d_scratch, &ctx->scratch_cap, opc::skew_scratch_bytes(a));
        if (rc == OPC_OK) rc = scratch_acquire(ctx, s);
        if (rc != OPC_OK) return rc;
        e = opc::launch_skew(a, counter, ctx->d_scratch, ctx->num_sms, s);
        if (e != cudaSuccess) return cuda_error(e, "skew kernel launch");
        rc = scratch_release(ctx, s);
        if (rc != OPC_OK) return rc;
    } else if (kernel == OPC_KERNEL_SLIDE) {
        int* counter = ctx->d_counter + 4 * (ctx->counter_idx++ & 15u);
        int rc = ensure(&ctx->d_scratch, &ctx->scratch_cap, opc::slide_scratch_bytes(a));
        if (rc == OPC_OK) rc = scratch_acquire(ctx, s);
        if (rc != OPC_OK) return rc;
        e = opc::launch_slide(a, counter, ctx->d_scratch, ctx->num_sms, s);
        if (e != cudaSuccess) return cuda_error(e, "slide kernel launch");
        rc = scratch_release(ctx, s);
        if (rc != OPC_OK) return rc;
    } else if (kernel == OPC_KERNEL_COLUMN) {
        e = opc::launch_column(a, ctx->num_sms, s);
        if (e != cudaSuccess) return cuda_error(e, "column kernel launch");
    } else if (kernel == OPC_KERNEL_PLANES) {
        e = opc::launch_planes(a, ctx->num_sms, s);
        if (e != cudaSuccess) return cuda_error(e, "planes kernel launch");
    } else {
        e = opc::launch_direct(a, s);
        if (e != cudaSuccess) return cuda_error(e, "direct kernel launch");
    }
    // The border job rides on the first kernel of the family (direct tile,
    // shear or transpose pre-pass); a band without interior launches it alone,
    // and so does the generic direct kernel.
    if (interior) {
        const bool own_border = kernel == OPC_KERNEL_DIRECT && !opc::direct_fuses_border(a);
        // direct / column: one kernel; skew: shear + skew; slide: transpose,
        // plan + slide
        const int n = kernel == OPC_KERNEL_DIRECT || kernel == OPC_KERNEL_COLUMN ||
                              kernel == OPC_KERNEL_PLANES
                          ? 1
                      : kernel == OPC_KERNEL_SLIDE                                ? 3
                                                                                  : 2;
        g_launches.fetch_add(n + (own_border && a.border.nblocks > 0 ? 1 : 0));
    } else {
        e = opc::launch_border(a, s);
        if (e != cudaSuccess) return cuda_error(e, "border kernel launch");
        if (a.border.nblocks > 0) g_launches.fetch_add(1);
    }
    return OPC_OK;
}

int filter_core(const std::uint8_t* in, std::uint8_t* out, int frames, int w, int h, int y_begin,
                int y_end, int radius, int levels, int border, const opc_config* cfg) {
    const unsigned flags = cfg ? cfg->flags : 0u;
    int rc = validate_params(w, h, 3ull * w * h, radius, levels, flags);
    if (rc != OPC_OK) return rc;
    if (frames < 1) return set_error(OPC_EINVAL, "frames must be >= 1, got " + std::to_string(frames));
    if (y_begin < 0 || y_end > h || y_begin >= y_end) {
        return set_error(OPC_EINVAL, "row band [" + std::to_string(y_begin) + ", " +
                                         std::to_string(y_end) + ") is not inside [0, " +
                                         std::to_string(h) + ")");
    }
    if (border != OPC_BORDER_COPY_INPUT && border != OPC_BORDER_ZERO_FILL) {
        return set_error(OPC_EINVAL, "border must be 0 (CopyInput) or 1 (ZeroFill), got " +
                                         std::to_string(border));
    }
    if (!in || !out) return set_error(OPC_EINVAL, "null image buffer");
    const long long iy = std::max(0, std::min(y_end, h - radius) - std::max(y_begin, radius));
    const long long interior = std::max(0, w - 2 * radius) * iy * frames;
    int kernel = plan(levels, radius, cfg ? cfg->kernel : 0, interior / std::max(1, frames), frames);
    if (kernel < 0) {
        return set_error(OPC_EINVAL, "requested kernel family does not support L=" +
                                         std::to_string(levels) + " r=" + std::to_string(radius));
    }

    DevCtx* ctx = nullptr;
    rc = get_ctx(cfg ? cfg->device : -1, &ctx);
    if (rc != OPC_OK) return rc;

    // Buffer geometry: per frame, `in` holds image rows [in_row0, in_row0 +
    // in_rows) and `out` holds output rows [y_begin, y_end).
    opc::BandArgs a{};
    a.width = w;
    a.height = h;
    a.in_row0 = opc_band_in_row0(h, y_begin, radius);
    a.in_rows = opc_band_in_rows(h, y_begin, y_end, radius);
    a.out_row0 = y_begin;
    a.x_lo = radius;
    a.x_hi = w - radius;
    a.radius = radius;
    a.levels = levels;
    a.bin_mul = opc::bin_multiplier(levels);
    a.op_counts = (flags & OPC_FLAG_COUNT_OPS) ? ctx->d_opcounts : nullptr;
    const std::size_t row_bytes = static_cast<std::size_t>(w) * 3;
    const std::size_t in_bytes = row_bytes * a.in_rows;
    const std::size_t out_bytes = row_bytes * (y_end - y_begin);
    a.in_frame_stride = in_bytes;
    a.out_frame_stride = out_bytes;
    auto set_rows = [&](int y0, int y1) {
        a.y_begin = y0;
        a.y_end = y1;
        a.y_lo = y0 > radius ? y0 : radius;
        a.y_hi = y1 < h - radius ? y1 : h - radius;
        if (a.y_hi < a.y_lo) a.y_hi = a.y_lo;
    };

    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");

    if (flags & OPC_FLAG_DEVICE_POINTERS) {
        cudaStream_t s = cfg && cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : ctx->stream;
        a.in = in;
        a.out = out;
        a.frames = frames;
        set_rows(y_begin, y_end);
        return run_device(a, border, kernel, ctx, s);
    }

    // Host pointers: H2D / kernels / D2H pipelined over units (row chunks of
    // a large image, or frames of a batch) on three streams, so PCIe traffic
    // in both directions overlaps the filter.
    const std::size_t tot_in = in_bytes * frames, tot_out = out_bytes * frames;
    rc = ensure(&ctx->d_in, &ctx->in_cap, tot_in);
    if (rc != OPC_OK) return rc;
    rc = ensure(&ctx->d_out, &ctx->out_cap, tot_out);
    if (rc != OPC_OK) return rc;
    struct Unit {
        int frame, nframes, y0, y1;
    };
    std::vector<Unit> units;
    const int rows = y_end - y_begin;
    if (frames == 1) {
        // Row chunks of ~48 MB, with a geometric ramp (1/16, 1/8, ... of a chunk)
        // at both ends: only the first chunk's H2D and the last chunk's kernels
        // and D2H are not overlapped with transfers in the other direction.
        const long long chunk_rows =
            std::max<long long>(1, static_cast<long long>((static_cast<unsigned long long>(OPC_HOST_CHUNK_MB) << 20) / row_bytes));
        std::vector<int> sizes;
        if (rows > 4 * chunk_rows) {
            std::vector<int> ramp;
            for (long long q = std::max<long long>(8, chunk_rows / 16); q < chunk_rows; q *= 2) {
                ramp.push_back(static_cast<int>(q));
            }
            long long ramp_rows = 0;
            for (int q : ramp) ramp_rows += 2 * q;
            const long long mid = rows - ramp_rows;
            const int nmid = static_cast<int>((mid + chunk_rows - 1) / chunk_rows);
            sizes = ramp;
            for (int k = 0; k < nmid; ++k) {
                sizes.push_back(static_cast<int>(mid * (k + 1) / nmid - mid * k / nmid));
            }
            sizes.insert(sizes.end(), ramp.rbegin(), ramp.rend());
        } else {
            // Smaller images: up to OPC_HOST_SMALL_CHUNKS chunks of >= 6 MB, so
            // the H2D of chunk k+1 and the D2H of chunk k overlap even when the
            // image is below one 48 MB chunk (C2: one 6 MB transfer each way
            // plus the kernel, end to end, was fully serial).
            int n = static_cast<int>((rows + chunk_rows - 1) / chunk_rows);
            const long long bytes = static_cast<long long>(rows) * static_cast<long long>(row_bytes);
            const int small = static_cast<int>(std::min<long long>(
                OPC_HOST_SMALL_CHUNKS, bytes / static_cast<long long>(OPC_HOST_SMALL_MIN_KB * 1024)));
            n = std::max(n, small);
            n = std::min(n, std::max(1, rows / std::max(1, 2 * radius + 1)));  // chunks >= 2r+1 rows
            n = n < 1 ? 1 : n;
            for (int k = 0; k < n; ++k) {
                sizes.push_back(static_cast<int>(static_cast<long long>(rows) * (k + 1) / n -
                                                 static_cast<long long>(rows) * k / n));
            }
        }
        int y = y_begin;
        for (int q : sizes) {
            units.push_back({0, 1, y, y + q});
            y += q;
        }
    } else {
        // Frames of >= 4 MB one per unit; smaller frames grouped into units of
        // about 48 MB (one launch each), so the staging slots stay bounded
        // whatever the batch length.
        const std::size_t fb = std::max(in_bytes, out_bytes);
        const int per = fb >= (4ull << 20)
                            ? 1
                            : static_cast<int>(std::max<std::size_t>(1, (48ull << 20) / fb));
        for (int f = 0; f < frames; f += per) {
            units.push_back({f, std::min(per, frames - f), y_begin, y_end});
        }
    }
    rc = ensure_streams(ctx, units.size());
    if (rc != OPC_OK) return rc;
    // Per unit: the new input bytes (rows beyond what earlier units loaded; the
    // host and device buffers share offsets) and the output bytes.
    struct Xfer {
        std::size_t in_off, in_n, out_off, out_n;
        int f0, nf, y0, y1;
    };
    std::vector<Xfer> xs;
    std::vector<int> loaded_hi(frames > 0 ? frames : 1, a.in_row0);
    for (const Unit& un : units) {
        Xfer x{};
        x.f0 = un.frame;
        x.nf = un.nframes;
        x.y0 = un.y0;
        x.y1 = un.y1;
        if (un.nframes > 1) {
            x.in_off = in_bytes * x.f0;
            x.in_n = in_bytes * x.nf;
            x.out_off = out_bytes * x.f0;
            x.out_n = out_bytes * x.nf;
        } else {
            const int need_hi = opc_band_in_row0(h, un.y0, radius) +
                                opc_band_in_rows(h, un.y0, un.y1, radius);
            if (need_hi > loaded_hi[x.f0]) {
                const int lo = loaded_hi[x.f0];
                x.in_off = in_bytes * x.f0 + static_cast<std::size_t>(lo - a.in_row0) * row_bytes;
                x.in_n = static_cast<std::size_t>(need_hi - lo) * row_bytes;
                loaded_hi[x.f0] = need_hi;
            }
            x.out_off = out_bytes * x.f0 + static_cast<std::size_t>(un.y0 - y_begin) * row_bytes;
            x.out_n = static_cast<std::size_t>(un.y1 - un.y0) * row_bytes;
        }
        xs.push_back(x);
    }
    std::uint8_t* d_in = static_cast<std::uint8_t*>(ctx->d_in);
    std::uint8_t* d_out = static_cast<std::uint8_t*>(ctx->d_out);
    // Kernels of unit u after its H2D; its D2H after the kernels.
    auto compute = [&](std::size_t u) -> int {
        const Xfer& x = xs[u];
        cudaError_t e2 = cudaEventRecord(ctx->ev_in[u], ctx->s_in);
        if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(ctx->stream, ctx->ev_in[u], 0);
        if (e2 != cudaSuccess) return cuda_error(e2, "cudaEventRecord / cudaStreamWaitEvent");
        a.in = d_in + in_bytes * x.f0;
        a.out = d_out + out_bytes * x.f0;
        a.frames = x.nf;
        set_rows(x.y0, x.y1);
        const int rc2 = run_device(a, border, kernel, ctx, ctx->stream);
        if (rc2 != OPC_OK) return rc2;
        e2 = cudaEventRecord(ctx->ev_out[u], ctx->stream);
        if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(ctx->s_out, ctx->ev_out[u], 0);
        if (e2 != cudaSuccess) return cuda_error(e2, "cudaEventRecord / cudaStreamWaitEvent");
        return OPC_OK;
    };
    auto finish = [&]() -> int {
        cudaError_t e2 = cudaStreamSynchronize(ctx->s_out);
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(ctx->stream);
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(ctx->s_in);
        return e2 == cudaSuccess ? OPC_OK : cuda_error(e2, "cudaStreamSynchronize");
    };

    const bool staged = (tot_in + tot_out >= (16ull << 20)) &&
                        !(is_pinned_or_device(in) && is_pinned_or_device(out));
    if (!staged) {
        // Pinned (or small) host buffers: DMA straight from / to them.
        for (std::size_t u = 0; u < xs.size(); ++u) {
            const Xfer& x = xs[u];
            if (x.in_n) {
                e = cudaMemcpyAsync(d_in + x.in_off, in + x.in_off, x.in_n, cudaMemcpyHostToDevice,
                                    ctx->s_in);
                if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync(H2D)");
            }
            rc = compute(u);
            if (rc != OPC_OK) return rc;
            e = cudaMemcpyAsync(out + x.out_off, d_out + x.out_off, x.out_n, cudaMemcpyDeviceToHost,
                                ctx->s_out);
            if (e != cudaSuccess) return cuda_error(e, "cudaMemcpyAsync(D2H)");
        }
        return finish();
    }

    // Pageable host buffers (a std::vector Image, a numpy array): staged through
    // a ring of kSlots pinned buffers per direction.  This thread copies unit
    // u's input rows into an input slot (CopyPool) and enqueues H2D / kernels /
    // D2H into an output slot; a second thread copies finished output slots
    // back.  Slot reuse waits on the H2D that read the slot (event) and on the
    // copy-out of the unit that last used the output slot (counter).  The driver's
    // own pageable path ran C4 end to end at 2.2 GP/s against 15 GP/s pinned.
    std::size_t slot_need = 0;
    for (const Xfer& x : xs) slot_need = std::max(slot_need, std::max(x.in_n, x.out_n));
    const int slots_need = static_cast<int>(std::min<std::size_t>(DevCtx::kSlots, xs.size()));
    if (ctx->pin_cap < slot_need || ctx->pin_slots < slots_need) {
        const std::size_t cap = std::max(slot_need, ctx->pin_cap);
        const int nslots = std::max(slots_need, ctx->pin_slots);
        free_staging(ctx);
        for (int k = 0; k < nslots; ++k) {
            e = cudaHostAlloc(&ctx->pin_in[k], cap, cudaHostAllocPortable);
            if (e == cudaSuccess) e = cudaHostAlloc(&ctx->pin_out[k], cap, cudaHostAllocPortable);
            if (e != cudaSuccess) {
                free_staging(ctx);
                return cuda_error(e, "cudaHostAlloc(staging)");
            }
        }
        ctx->pin_cap = cap;
        ctx->pin_slots = nslots;
    }
    CopyPool& pool = CopyPool::get(ctx->device);
    std::mutex m;
    std::condition_variable cv;
    std::size_t enqueued = 0, drained = 0;  // units whose D2H is enqueued / copied out
    bool abort = false;
    int consumer_rc = OPC_OK;
    const int dev = ctx->device;
    std::thread consumer([&] {
        cudaSetDevice(dev);
        for (std::size_t u = 0; u < xs.size(); ++u) {
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return enqueued > u || abort; });
                if (abort) return;
            }
            const cudaError_t e2 = cudaEventSynchronize(ctx->ev_d2h[u]);
            if (e2 != cudaSuccess) {
                consumer_rc = cuda_error(e2, "cudaEventSynchronize(D2H)");
                std::lock_guard<std::mutex> lk(m);
                abort = true;
                cv.notify_all();
                return;
            }
            pool.copy(out + xs[u].out_off, ctx->pin_out[u % DevCtx::kSlots], xs[u].out_n);
            std::lock_guard<std::mutex> lk(m);
            drained = u + 1;
            cv.notify_all();
        }
    });
    auto fail = [&](int code) {
        {
            std::lock_guard<std::mutex> lk(m);
            abort = true;
        }
        cv.notify_all();
        consumer.join();
        cudaStreamSynchronize(ctx->s_out);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamSynchronize(ctx->s_in);
        return code;
    };
    for (std::size_t u = 0; u < xs.size(); ++u) {
        const Xfer& x = xs[u];
        const int k = static_cast<int>(u % DevCtx::kSlots);
        if (x.in_n) {
            e = cudaEventSynchronize(ctx->ev_slot[k]);  // the H2D that last read slot k
            if (e != cudaSuccess) return fail(cuda_error(e, "cudaEventSynchronize(slot)"));
            pool.copy(ctx->pin_in[k], in + x.in_off, x.in_n);
            e = cudaMemcpyAsync(d_in + x.in_off, ctx->pin_in[k], x.in_n, cudaMemcpyHostToDevice,
                                ctx->s_in);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_slot[k], ctx->s_in);
            if (e != cudaSuccess) return fail(cuda_error(e, "cudaMemcpyAsync(H2D)"));
        }
        rc = compute(u);
        if (rc != OPC_OK) return fail(rc);
        {  // output slot k is free once unit u - kSlots has been copied out
            std::unique_lock<std::mutex> lk(m);
            cv.wait(lk, [&] { return drained + DevCtx::kSlots > u || abort; });
            if (abort) {
                lk.unlock();
                return fail(consumer_rc);
            }
        }
        e = cudaMemcpyAsync(ctx->pin_out[k], d_out + x.out_off, x.out_n, cudaMemcpyDeviceToHost,
                            ctx->s_out);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_d2h[u], ctx->s_out);
        if (e != cudaSuccess) return fail(cuda_error(e, "cudaMemcpyAsync(D2H)"));
        {
            std::lock_guard<std::mutex> lk(m);
            enqueued = u + 1;
        }
        cv.notify_all();
    }
    consumer.join();
    if (consumer_rc != OPC_OK) return consumer_rc;
    return finish();
}

}  // namespace

namespace opc {
TimingHook g_timing_hook = nullptr;
}  // namespace opc

extern "C" {

int opc_kernel_timing(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    for (const TimedLaunch& t : g_timed) {
        g_ev_pool[t.device].push_back(t.start);
        g_ev_pool[t.device].push_back(t.stop);
    }
    g_timed.clear();
    for (const auto& kv : g_open) g_ev_pool[std::get<0>(kv.first)].push_back(kv.second);
    g_open.clear();
    opc::g_timing_hook = enable ? timing_hook : nullptr;
    return OPC_OK;
}

int opc_kernel_timing_read(int32_t kernel_id, double* ms_total, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    double total = 0;
    long long n = 0;
    for (const TimedLaunch& t : g_timed) {
        if (t.id != kernel_id) continue;
        cudaError_t e = cudaEventSynchronize(t.stop);
        float ms = 0;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, t.start, t.stop);
        if (e != cudaSuccess) return cuda_error(e, "cudaEventElapsedTime");
        total += ms;
        ++n;
    }
    if (ms_total) *ms_total = total;
    if (launches) *launches = n;
    return OPC_OK;
}

int opc_validate(int32_t width, int32_t height, uint64_t nbytes, int32_t radius, int32_t levels,
                 uint32_t flags) {
    return validate_params(width, height, nbytes, radius, levels, flags);
}

int opc_filter_rgb8(const uint8_t* in, uint8_t* out, int32_t width, int32_t height,
                    int32_t radius, int32_t levels, int32_t border, const opc_config* cfg) {
    return filter_core(in, out, 1, width, height, 0, height, radius, levels, border, cfg);
}

int opc_filter_rgb8_batch(const uint8_t* in, uint8_t* out, int32_t frames, int32_t width,
                          int32_t height, int32_t radius, int32_t levels, int32_t border,
                          const opc_config* cfg) {
    return filter_core(in, out, frames, width, height, 0, height, radius, levels, border, cfg);
}

int opc_filter_rgb8_band(const uint8_t* in_rows, uint8_t* out_rows, int32_t width,
                         int32_t height, int32_t y_begin, int32_t y_end, int32_t radius,
                         int32_t levels, int32_t border, const opc_config* cfg) {
    return filter_core(in_rows, out_rows, 1, width, height, y_begin, y_end, radius, levels, border,
                       cfg);
}

int32_t opc_band_begin(int32_t total, int32_t parts, int32_t k) {
    if (parts < 1) return 0;
    return static_cast<int32_t>(static_cast<long long>(total) * k / parts);
}

int opc_filter_rgb8_multi(const uint8_t* in, uint8_t* out, int32_t frames, int32_t width,
                          int32_t height, int32_t radius, int32_t levels, int32_t border,
                          const int32_t* devices, int32_t ndevices, const opc_config* cfg) {
    const unsigned flags = cfg ? cfg->flags : 0u;
    int rc = validate_params(width, height, 3ull * width * height, radius, levels, flags);
    if (rc != OPC_OK) return rc;
    if (flags & OPC_FLAG_DEVICE_POINTERS) {
        return set_error(OPC_EINVAL, "opc_filter_rgb8_multi takes host buffers only");
    }
    if (!devices || ndevices < 1) return set_error(OPC_EINVAL, "ndevices must be >= 1");
    if (frames < 1) return set_error(OPC_EINVAL, "frames must be >= 1, got " + std::to_string(frames));
    const std::size_t row_bytes = static_cast<std::size_t>(width) * 3;
    const std::size_t frame_bytes = row_bytes * height;
    const int total = frames == 1 ? height : frames;
    int parts = ndevices < total ? ndevices : total;
    std::vector<int> status(parts, OPC_OK);
    std::vector<std::string> msg(parts);
    std::vector<std::thread> pool;
    for (int k = 0; k < parts; ++k) {
        pool.emplace_back([&, k] {
            opc_config c = cfg ? *cfg : opc_config{};
            c.device = devices[k];
            c.stream = nullptr;
            const int b = opc_band_begin(total, parts, k), e = opc_band_begin(total, parts, k + 1);
            if (frames == 1) {
                const int lo = opc_band_in_row0(height, b, radius);
                status[k] = filter_core(in + row_bytes * lo, out + row_bytes * b, 1, width, height,
                                        b, e, radius, levels, border, &c);
            } else {
                status[k] = filter_core(in + frame_bytes * b, out + frame_bytes * b, e - b, width,
                                        height, 0, height, radius, levels, border, &c);
            }
            if (status[k] != OPC_OK) msg[k] = g_last_error;
        });
    }
    for (auto& t : pool) t.join();
    for (int k = 0; k < parts; ++k) {
        if (status[k] != OPC_OK) {
            return set_error(status[k], "device " + std::to_string(devices[k]) + ": " + msg[k]);
        }
    }
    return OPC_OK;
}

int32_t opc_band_in_row0(int32_t height, int32_t y_begin, int32_t radius) {
    (void)height;
    const int32_t v = y_begin - radius;
    return v > 0 ? v : 0;
}

int32_t opc_band_in_rows(int32_t height, int32_t y_begin, int32_t y_end, int32_t radius) {
    const int32_t lo = opc_band_in_row0(height, y_begin, radius);
    const int32_t hi = y_end + radius < height ? y_end + radius : height;
    return hi - lo;
}

const char* opc_last_error(void) { return g_last_error.c_str(); }

const char* opc_version(void) { return "oilpaint-b200 0.1.0 (sm_100a)"; }

uint64_t opc_kernel_launches(void) { return g_launches.load(); }

int32_t opc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int opc_synchronize(const opc_config* cfg) {
    DevCtx* ctx = nullptr;
    int rc = get_ctx(cfg ? cfg->device : -1, &ctx);
    if (rc != OPC_OK) return rc;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    cudaStream_t s = cfg && cfg->stream ? static_cast<cudaStream_t>(cfg->stream) : ctx->stream;
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "cudaStreamSynchronize");
    return OPC_OK;
}

int opc_generate_device(int32_t kind, uint64_t seed, int32_t width, int32_t height, uint8_t* d_out,
                        int32_t device, void* stream) {
    DevCtx* ctx = nullptr;
    int rc = get_ctx(device, &ctx);
    if (rc != OPC_OK) return rc;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    rc = opc::launch_generate(kind, seed, width, height, d_out, s, &e);
    if (rc == -1) {
        return set_error(OPC_EINVAL, "pattern kind " + std::to_string(kind) +
                                         " has no device generator");
    }
    if (rc != 0) return set_error(OPC_EINVAL, "invalid pattern spec");
    if (e != cudaSuccess) return cuda_error(e, "generator launch");
    return OPC_OK;
}

int opc_op_counts(int32_t device, uint64_t* out, int32_t n, int32_t reset) {
    DevCtx* ctx = nullptr;
    int rc = get_ctx(device, &ctx);
    if (rc != OPC_OK) return rc;
    if (n < 0 || n > opc::kOpCountN || (n > 0 && !out)) {
        return set_error(OPC_EINVAL, "opc_op_counts: n must be in [0, " +
                                         std::to_string(opc::kOpCountN) + "]");
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long tmp[opc::kOpCountN] = {};
    if (e == cudaSuccess) {
        e = cudaMemcpy(tmp, ctx->d_opcounts, sizeof(tmp), cudaMemcpyDeviceToHost);
    }
    if (e == cudaSuccess && reset) e = cudaMemset(ctx->d_opcounts, 0, sizeof(tmp));
    if (e != cudaSuccess) return cuda_error(e, "opc_op_counts");
    for (int i = 0; i < n; ++i) out[i] = tmp[i];
    return OPC_OK;
}

int32_t opc_plan_kernel(int32_t width, int32_t height, int32_t radius, int32_t levels) {
    if (validate_params(width, height, 3ull * width * height, radius, levels,
                        OPC_FLAG_ALLOW_LEVELS_256) != OPC_OK) {
        return -1;
    }
    return plan(levels, radius, 0,
                static_cast<long long>(width - 2 * radius) * (height - 2 * radius), 1);
}

int32_t opc_plan_kernel_batch(int32_t width, int32_t height, int32_t radius, int32_t levels,
                              int32_t frames) {
    if (frames < 1 || validate_params(width, height, 3ull * width * height, radius, levels,
                                      OPC_FLAG_ALLOW_LEVELS_256) != OPC_OK) {
        return -1;
    }
    return plan(levels, radius, 0,
                static_cast<long long>(width - 2 * radius) * (height - 2 * radius), frames);
}

void opc_release(void) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto& c : g_ctx) {
        if (!c) continue;
        std::lock_guard<std::mutex> lk2(c->mu);
        cudaSetDevice(c->device);
        if (c->d_in) cudaFree(c->d_in);
        if (c->d_out) cudaFree(c->d_out);
        if (c->d_scratch) cudaFree(c->d_scratch);
        if (c->d_counter) cudaFree(c->d_counter);
        if (c->d_opcounts) cudaFree(c->d_opcounts);
        if (c->stream) cudaStreamDestroy(c->stream);
        if (c->s_in) cudaStreamDestroy(c->s_in);
        if (c->s_out) cudaStreamDestroy(c->s_out);
        for (cudaEvent_t ev : c->ev_in) cudaEventDestroy(ev);
        for (cudaEvent_t ev : c->ev_out) cudaEventDestroy(ev);
        for (cudaEvent_t ev : c->ev_d2h) cudaEventDestroy(ev);
        for (cudaEvent_t ev : c->ev_slot) {
            if (ev) cudaEventDestroy(ev);
        }
        if (c->scratch_ev) cudaEventDestroy(c->scratch_ev);
        free_staging(c.get());
        c.reset();
    }
    g_ctx.clear();
}

}  // extern "C"
