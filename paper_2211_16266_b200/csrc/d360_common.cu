// Error reporting, parameter validation and the FMA-peak microbenchmark.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "d360_device.cuh"

namespace d360 {

static thread_local char g_error[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

// ---------------------------------------------------------------------------------------
// Launch accounting and optional per-launch device timing (the reference's only
// instrumentation is a perf_counter per stage; here every kernel launch is
// counted, and with tracing on it is bracketed by CUDA events on its own stream).
// ---------------------------------------------------------------------------------------
static std::atomic<unsigned long long> g_launches{0};
static std::atomic<int> g_trace_on{0};
struct TraceRec {
    const char* kind;
    cudaEvent_t e0, e1;
    int device;
    bool closed;  // e1 recorded
};
static std::mutex g_trace_mu;
static std::vector<TraceRec> g_trace;
static unsigned g_trace_generation = 0;  // bumped whenever g_trace is cleared
// An event belongs to the device it was created on, so the pool of spare events is per device.
struct PooledEvent {
    cudaEvent_t e;
    int device;
};
static std::vector<PooledEvent> g_event_pool;

static cudaEvent_t take_event(int device) {
    for (size_t i = 0; i < g_event_pool.size(); ++i) {
        if (g_event_pool[i].device == device) {
            cudaEvent_t e = g_event_pool[i].e;
            g_event_pool[i] = g_event_pool.back();
            g_event_pool.pop_back();
            return e;
        }
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    return e;
}

TraceScope::TraceScope(const char* kind, cudaStream_t s) : idx_(-1), gen_(0), s_(s) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_trace_on.load(std::memory_order_relaxed)) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    TraceRec r{kind, take_event(dev), take_event(dev), dev, false};
    if (r.e0 == nullptr || r.e1 == nullptr || cudaEventRecord(r.e0, s_) != cudaSuccess) {
        (void)cudaGetLastError();  // the launch itself is not affected; this record is dropped
        if (r.e0) g_event_pool.push_back(PooledEvent{r.e0, dev});
        if (r.e1) g_event_pool.push_back(PooledEvent{r.e1, dev});
        return;
    }
    g_trace.push_back(r);
    idx_ = (int)g_trace.size() - 1;
    gen_ = g_trace_generation;
}

TraceScope::~TraceScope() {
    if (idx_ < 0) return;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    // the trace may have been cleared (d360_trace_enable) while this scope was open: its slot is gone
    if (gen_ != g_trace_generation || idx_ >= (int)g_trace.size()) return;
    if (cudaEventRecord(g_trace[idx_].e1, s_) == cudaSuccess) g_trace[idx_].closed = true;
    else (void)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Generic-kernel fallbacks.  The throughput kernels (d360_fast_*.cu) cover the MIXED policy on
// regular sample grids with padded f64 planes; anything else runs on the generic kernels of
// d360_patchmatch.cu, about 2x slower.  That is never silent: every such launch is counted
// (d360_generic_fallbacks) and the first one of each reason is reported on stderr.
// ---------------------------------------------------------------------------------------
static std::atomic<unsigned long long> g_fallbacks{0};
static thread_local const char* g_fast_reject = "not applicable";
static std::mutex g_fallback_mu;
static std::vector<const char*> g_fallback_seen;

int fast_reject(const char* why) {
    g_fast_reject = why;
    return -1;
}

void note_generic_fallback(const char* kernel, const GroupDev& gd) {
    g_fallbacks.fetch_add(1, std::memory_order_relaxed);
    const char* why = g_fast_reject;
    std::lock_guard<std::mutex> lk(g_fallback_mu);
    for (const char* seen : g_fallback_seen)
        if (seen == why) return;
    g_fallback_seen.push_back(why);
    if (getenv("D360_QUIET_FALLBACK") == nullptr)
        fprintf(stderr,
                "libd360: %s runs on the generic kernels (about 2x slower) for this group (%dx%d, %d views, %d "
                "samples): %s\n",
                kernel, gd.W, gd.H, gd.V, gd.S, why);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
        return 2;
    }
    return 0;
}

int make_group_dev(const d360_group* g, GroupDev* out) {
    if (g == nullptr) { set_error("group is NULL"); return 1; }
    if (g->width < 2 || g->height < 2) {
        set_error("camera size must be at least 2x2, got %dx%d", g->width, g->height);
        return 1;
    }
    if (g->n_views < 1 || g->n_views > D360_MAX_VIEWS) {
        set_error("n_views %d outside [1, %d]", g->n_views, D360_MAX_VIEWS);
        return 1;
    }
    if (g->n_samples < 1 || g->n_samples > D360_MAX_SAMPLES) {
        set_error("n_samples %d outside [1, %d]", g->n_samples, D360_MAX_SAMPLES);
        return 1;
    }
    if (g->top_k < 1 || g->top_k > g->n_views) {
        set_error("top_k %d outside [1, n_views=%d]", g->top_k, g->n_views);
        return 1;
    }
    if (g->precision != D360_PREC_EXACT && g->precision != D360_PREC_MIXED) {
        set_error("unsupported precision policy %d", g->precision);
        return 1;
    }
    if (!(g->trunc > 0.0)) { set_error("cost_truncation must be > 0, got %g", g->trunc); return 1; }
    if (!g->rays || !g->ref_gray || !g->nb || !g->rel_r || !g->rel_t || !g->offsets) {
        set_error("group has a NULL array pointer");
        return 1;
    }
    GroupDev& d = *out;
    d.W = g->width; d.H = g->height; d.V = g->n_views; d.S = g->n_samples; d.top_k = g->top_k;
    d.rays = g->rays; d.ref_gray = g->ref_gray; d.nb = g->nb; d.trunc = g->trunc;
    if (g->nb_pad_x < 0 || g->nb_pad_y < 0 || g->nb_pad_x > 64 || g->nb_pad_y > 64) {
        set_error("neighbour plane pads (%d, %d) outside [0, 64]", g->nb_pad_x, g->nb_pad_y);
        return 1;
    }
    d.nb_pad_x = g->nb_pad_x; d.nb_pad_y = g->nb_pad_y;
    d.nb64 = g->nb64;
    d.ref_ctx = g->ref_ctx;
    d.ref_ctx_pad = g->ref_ctx_pad;
    if (d.ref_ctx != nullptr && (d.ref_ctx_pad < 0 || d.ref_ctx_pad > 64)) {
        set_error("reference context pad %d outside [0, 64]", d.ref_ctx_pad);
        return 1;
    }
    int reach = 0;
    for (int k = 0; k < g->n_samples; ++k) {
        const int dx = g->offsets[2 * k], dy = g->offsets[2 * k + 1];
        if (abs(dx) > D360_MAX_REACH || abs(dy) > D360_MAX_REACH) {
            set_error("sample offset (%d,%d) exceeds the supported reach %d", dx, dy, D360_MAX_REACH);
            return 1;
        }
        if (abs(dx) >= g->width) {
            set_error("sample offset dx=%d does not fit width %d (single wrap, K:169-172)", dx, g->width);
            return 1;
        }
        reach = abs(dx) > reach ? abs(dx) : reach;
        reach = abs(dy) > reach ? abs(dy) : reach;
        d.dx[k] = (signed char)dx;
        d.dy[k] = (signed char)dy;
    }
    d.reach = reach;
    for (int v = 0; v < g->n_views; ++v) {
        for (int i = 0; i < 9; ++i) d.rel_r[v][i] = g->rel_r[9 * v + i];
        for (int i = 0; i < 3; ++i) d.rel_t[v][i] = g->rel_t[3 * v + i];
    }
    return 0;
}

// ---------------------------------------------------------------------------------------
// FMA-pipe peak: 16 independent accumulator chains per thread, 8 CTAs of 256 per SM.
// ---------------------------------------------------------------------------------------
template <typename T>
__global__ void k_fma_peak(T* out, int iters, T a, T b) {
    T acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = (T)(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = acc[i] * a + b;
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == (T)123456789) out[0] = s;  // never true; keeps the chains alive
}

}  // namespace d360

extern "C" const char* d360_last_error(void) { return d360::g_error; }

extern "C" unsigned long long d360_launch_count(void) { return d360::g_launches.load(); }

extern "C" unsigned long long d360_generic_fallbacks(void) { return d360::g_fallbacks.load(); }

extern "C" int d360_trace_enable(int on) {
    using namespace d360;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    for (auto& r : g_trace) {
        g_event_pool.push_back(PooledEvent{r.e0, r.device});
        g_event_pool.push_back(PooledEvent{r.e1, r.device});
    }
    g_trace.clear();
    ++g_trace_generation;
    g_trace_on.store(on ? 1 : 0);
    return 0;
}

extern "C" int d360_trace_summary(char* buf, int cap) {
    using namespace d360;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    struct Agg { const char* kind; int n; double ms; };
    std::vector<Agg> aggs;
    for (auto& r : g_trace) {
        if (!r.closed) continue;  // scope still open, or its end could not be recorded
        if (cudaEventSynchronize(r.e1) != cudaSuccess) {
            set_error("trace: event synchronize failed: %s", cudaGetErrorString(cudaGetLastError()));
            return -1;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.e0, r.e1);
        Agg* a = nullptr;
        for (auto& x : aggs)
            if (strcmp(x.kind, r.kind) == 0) a = &x;
        if (!a) {
            aggs.push_back(Agg{r.kind, 0, 0.0});
            a = &aggs.back();
        }
        a->n += 1;
        a->ms += ms;
    }
    int off = 0;
    for (auto& a : aggs) {
        int w = snprintf(buf + off, off < cap ? cap - off : 0, "%s %d %.6f\n", a.kind, a.n, a.ms);
        if (w < 0 || off + w >= cap) {
            set_error("trace: summary buffer of %d bytes is too small", cap);
            return -1;
        }
        off += w;
    }
    return off;
}
extern "C" int d360_version(void) { return 100; }

extern "C" double d360_measure_fma_peak(int fp64, int iters) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* out = nullptr;
    if (cudaMalloc(&out, 64) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    float best_ms = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (fp64) d360::k_fma_peak<double><<<blocks, threads>>>((double*)out, iters, 1.0000001, 1e-9);
        else d360::k_fma_peak<float><<<blocks, threads>>>((float*)out, iters, 1.0000001f, 1e-9f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best_ms) best_ms = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 16.0 * (double)iters * (double)blocks * threads;
    return flops / (best_ms * 1e-3) / 1e12;
}
