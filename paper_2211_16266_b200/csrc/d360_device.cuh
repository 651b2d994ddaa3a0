// Shared device-side definitions for the densify360 B200 kernels.
//
// Reference shorthand (see include/d360.h): K = kernels.py, E = engine.py.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/d360.h"

#define D360_PI 3.141592653589793
#define D360_HALF_PI 1.5707963267948966

// Penalty guards, K:34-37.
#define D360_FACING_EPS 1e-6
#define D360_PARALLEL_EPS 1e-9
#define D360_SIGMA_EPS 1e-4
#define D360_VAR_EPS 1e-8

namespace d360 {

// Kernel parameter block (passed by value; small arrays live in the constant bank).
struct GroupDev {
    int W, H, V, S, top_k, reach;
    int nb_pad_x, nb_pad_y;  // neighbour planes are (H + 2 pad_y, W + 2 pad_x), see d360.h
    const float* rays;
    const float* ref_gray;
    const float* nb;
    const double* nb64;  // optional f64 copy of the padded neighbour planes (d360.h)
    const float* ref_ctx;  // optional padded (ray, luma) plane of the reference (d360.h)
    int ref_ctx_pad;
    float rel_r[D360_MAX_VIEWS][9];
    float rel_t[D360_MAX_VIEWS][3];
    signed char dx[D360_MAX_SAMPLES];
    signed char dy[D360_MAX_SAMPLES];
    double trunc;
};

// Counts one kernel launch; when tracing is enabled (d360_trace_enable) also brackets it
// with CUDA events on `s`.  Construct right before the <<<>>> launch, in its own scope.
class TraceScope {
public:
    TraceScope(const char* kind, cudaStream_t s);
    ~TraceScope();
    TraceScope(const TraceScope&) = delete;
    TraceScope& operator=(const TraceScope&) = delete;
private:
    int idx_;
    unsigned gen_;
    cudaStream_t s_;
};

// Shared refinement schedule of one pass (E:495-526), passed to the kernels by value.
struct RefineTable {
    float dd[D360_MAX_REFINE], sa[D360_MAX_REFINE], ca[D360_MAX_REFINE], caz[D360_MAX_REFINE],
        saz[D360_MAX_REFINE];
    int n;
    double depth_min, depth_max;
};

// Throughput kernels (d360_fast.cu): policy MIXED on a regular sample grid.  Each returns -1
// when it does not apply (irregular offsets, unsupported view count) and the caller falls
// back to the generic kernels of d360_patchmatch.cu.
int fast_eval(const struct GroupDev& gd, const float* depth, const float* normal, float* cost_out, cudaStream_t s);
int fast_red_black(const struct GroupDev& gd, int parity, const float* di, const float* ni, const float* ci,
                   float* dout, float* nout, float* cout, const unsigned char* changed_in,
                   unsigned char* changed_out, unsigned char* memo_valid, double* memo_cost,
                   unsigned long long* n_evals, cudaStream_t s);
int fast_refine(const struct GroupDev& gd, const RefineTable& tab, float* depth, float* normal, float* cost,
                unsigned char* changed, unsigned long long* n_evals, cudaStream_t s);

// A throughput kernel that does not apply records why and returns -1 (fast_reject); the caller
// then counts and reports the generic-kernel launch (note_generic_fallback), d360_common.cu.
int fast_reject(const char* why);
void note_generic_fallback(const char* kernel, const struct GroupDev& gd);

void set_error(const char* fmt, ...);
int check_launch(const char* what);
int make_group_dev(const d360_group* g, GroupDev* out);

// ---------------------------------------------------------------------------------------
// f64 helpers.  EXACT uses one IEEE operation per reference statement (no contraction),
// MIXED contracts to DFMA and replaces div/sqrt by MUFU seeds + Newton steps that are
// accurate to < 1e-13 relative, far below the f32 rounding of the projected (u, v).
// ---------------------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ double madd(double a, double b, double c) {
    if constexpr (MODE == D360_PREC_EXACT) return __dadd_rn(__dmul_rn(a, b), c);
    else return fma(a, b, c);
}

__device__ __forceinline__ double rcp_seed(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
// 1/x for normal positive or negative x, two Newton steps (seed ~2^-20 -> 2^-80).
__device__ __forceinline__ double fast_rcp(double x) {
    double y = rcp_seed(x);
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
// 1/sqrt(x), x > 0 normal.  One third-order step: error ~ e^3.
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y = rsqrt_seed(x);
    double t = x * y;
    double e = fma(-t, y, 1.0);
    double p = fma(e, 0.375, 0.5) * e;
    y = fma(y, p, y);
    // second (cheap, quadratic) step guards a coarse seed
    t = x * y;
    e = fma(-t, y, 1.0);
    return fma(0.5 * y, e, y);
}

template <int MODE>
__device__ __forceinline__ double div_(double a, double b) {
    if constexpr (MODE == D360_PREC_EXACT) return a / b;
    else return a * fast_rcp(b);
}

// K:59-99
template <int MODE>
__device__ __forceinline__ double fast_atan2(double y_, double x_) {
    const double ax = fabs(x_), ay = fabs(y_);
    const bool swap = ay > ax;
    const double hi = swap ? ay : ax;
    const double lo = swap ? ax : ay;
    double r;
    if constexpr (MODE == D360_PREC_EXACT) r = lo / (hi + 1e-300);
    else r = lo * fast_rcp(hi + 1e-300);
    const double s = r * r;
    double p = -5.021063913876e-03;
    p = madd<MODE>(s, p, 2.533170107199e-02);
    p = madd<MODE>(s, p, -6.087448223083e-02);
    p = madd<MODE>(s, p, 1.000220525649e-01);
    p = madd<MODE>(s, p, -1.404782123164e-01);
    p = madd<MODE>(s, p, 1.997402857787e-01);
    p = madd<MODE>(s, p, -3.333223261885e-01);
    p = madd<MODE>(s, p, 9.999999227776e-01);
    p = r * p;
    p = swap ? D360_HALF_PI - p : p;
    p = x_ < 0.0 ? D360_PI - p : p;
    return y_ < 0.0 ? -p : p;
}

// K:102-131
template <int MODE>
__device__ __forceinline__ double fast_acos(double x_) {
    double a = fabs(x_);
    a = a > 1.0 ? 1.0 : a;
    double p = -1.223553911532e-03;
    p = madd<MODE>(a, p, 6.510368059701e-03);
    p = madd<MODE>(a, p, -1.682974898800e-02);
    p = madd<MODE>(a, p, 3.068214201158e-02);
    p = madd<MODE>(a, p, -5.008467775423e-02);
    p = madd<MODE>(a, p, 8.895977933699e-02);
    p = madd<MODE>(a, p, -2.145970563340e-01);
    p = madd<MODE>(a, p, 1.570796263346e00);
    double w = 1.0 - a;
    double sq;
    if constexpr (MODE == D360_PREC_EXACT) {
        sq = sqrt(w);
    } else {
        w = fmax(w, 1e-280);
        sq = w * fast_rsqrt(w);
    }
    p = p * sq;
    return x_ < 0.0 ? D360_PI - p : p;
}

// Non-contracted f32 dot product, left to right: the oracle's (and numba's nominal)
// a0*b0 + a1*b1 + a2*b2 in float32.
__device__ __forceinline__ float dot3_f32(float a0, float a1, float a2, float b0, float b1,
                                          float b2) {
    return __fadd_rn(__fadd_rn(__fmul_rn(a0, b0), __fmul_rn(a1, b1)), __fmul_rn(a2, b2));
}
__device__ __forceinline__ double dot3_f64(double a0, double a1, double a2, double b0, double b1,
                                           double b2) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

__device__ __forceinline__ int wrap_once(int x, int w) {
    x = x < 0 ? x + w : x;
    return x >= w ? x - w : x;
}
__device__ __forceinline__ int pos_mod(int x, int w) {
    int r = x % w;
    return r < 0 ? r + w : r;
}

}  // namespace d360
