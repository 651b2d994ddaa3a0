// Throughput build of the PatchMatch cost kernels (precision policy D360_PREC_MIXED on a
// regular sample grid) for sm_100a.
//
// Same algorithm and same decision rules as d360_patchmatch.cu (K:156-297, K:300-610), with
// the per-sample-view instruction stream cut to what the B200's pipes need:
//   * FP64 pipe (64 lanes/clk/SM, the binding resource): 47 operations per sample-view —
//     t = lam * Rq + t_v, |t|^2, one third-order rsqrt / rcp refinement of the MUFU.64H
//     seeds (error ~1e-18, no IEEE div/sqrt), the two degree-7 Horner chains of the
//     reference's atan2 / acos polynomials, and the three NCC sums;
//   * octant / hemisphere fix-ups of K:90-99 and K:129-131 are folded into one DFMA whose
//     multiplier and addend come from 8- and 2-entry constant tables indexed by sign bits;
//   * XU pipe (16 lanes/clk/SM): 3 MUFU.64H seeds + 3 F2F (u, v -> f32 as the reference's
//     f32 scratch K:250-258, bilinear value -> f64); floor / frac of (u, v) use the
//     1.5 * 2^23 magic-add on the FP32 pipe instead of F2I / I2F;
//   * sample offsets come from loop counters (regular grid), all parameters from the
//     constant bank, nothing is converted twice.
// (u, v) are therefore the reference's f64 values to ~1e-12 px before the f32 rounding, which
// is what holds the 1e-4 relative cost parity.
#include <math.h>

#include "d360_device.cuh"

namespace d360 {
namespace fast {

constexpr int TW = 32;        // tile width (pixels)
constexpr int TH_FULL = 8;    // tile height for eval / refine: 256 threads, one per pixel
constexpr int TH_RB = 16;     // tile height for red-black: 256 threads, one per same-colour pixel
constexpr int THREADS = 256;
#ifndef D360_FAST_MINB
#define D360_FAST_MINB 2
#endif

struct FastGroup {
    int W, H, ns, stride, reach, top_k;
    int pitch;            // neighbour plane row pitch (W + 2 pad_x), elements
    unsigned max_idx;     // last index of a plane from which a 2x2 footprint may start
    size_t plane;         // elements per neighbour plane
    const float* rays;
    const float* ref_gray;
    const double* nb64;   // padded planes widened to f64, two doubles per texel, see d360.h
    float rel_r[D360_MAX_VIEWS][9];
    double rel_t[D360_MAX_VIEWS][3];
    double mu[8], cu[8];  // longitude: u = p * mu[oct] + cu[oct]
    double mv[2], cv[2];  // latitude:  v = p * mv[hem] + cv[hem]
    double ca[8], cq[8];  // atan / acos polynomial coefficients, highest degree first (K:75-85, K:112-122)
    double trunc, inv_s;
    double neg_par_eps, tiny, c0375;  // -PARALLEL_EPS, 1e-30 (K:246), 3/8: 64-bit literals live in the constant bank
    unsigned plane32;     // plane as a 32-bit element count
    float pitch_f;        // pitch as float
    float idx_bias;       // 2^23 + pad_y * pitch + pad_x: float -> index by mantissa extraction
    float den_lim;        // largest f32 below -PARALLEL_EPS
};

// Patch context of a CTA tile in shared memory.  Window entry (i, j) <-> pixel
// ((x0 - R + i) mod W, clamp(y0 - R + j, 0, H-1)), K:168-177.  With `compress` (red-black pass
// on an even sample stride: every sample of an updated pixel has the pixel's colour) only the
// entries of that colour are kept, two window columns per slot — half the shared memory, and
// neighbouring lanes read neighbouring slots.
struct Tile {
    const float4* qg;  // (qx, qy, qz, reference luma) per entry
    const double* rq;  // [(v*3 + c) * ne + entry]  R_v q as f64 (exact widening of the f32 dot, K:184-189)
    int wwc;           // entries per window row
    int ne;            // entries per plane
    int sx, sy;        // entry step of one sample column / row
};

__host__ __device__ inline int window_entries(int tw, int th, int reach, bool compress) {
    const int ww = tw + 2 * reach;
    return (compress ? ww / 2 : ww) * (th + 2 * reach);
}
__host__ __device__ inline size_t tile_bytes(int tw, int th, int reach, bool compress, int n_views) {
    const size_t ne = (size_t)window_entries(tw, th, reach, compress);
    return ne * sizeof(float4) + ne * sizeof(double) * 3 * n_views;
}

template <int VT>
__device__ __forceinline__ Tile tile_setup(const FastGroup& g, unsigned char* smem, int x0, int y0, int th,
                                           bool compress, int keep) {
    const int R = g.reach;
    const int ww = TW + 2 * R, hh = th + 2 * R;
    const int wwc = compress ? ww / 2 : ww;
    const int ne = wwc * hh;
    float4* qg = reinterpret_cast<float4*>(smem);
    double* rq = reinterpret_cast<double*>(smem + (size_t)ne * sizeof(float4));
    for (int e = threadIdx.x; e < ne; e += THREADS) {
        const int j = e / wwc, ic = e - j * wwc;
        const int i = compress ? 2 * ic + ((keep + j) & 1) : ic;
        const int gx = pos_mod(x0 - R + i, g.W);
        const int gy = min(max(y0 - R + j, 0), g.H - 1);
        const size_t gi = (size_t)gy * g.W + gx;
        const float bx = __ldg(g.rays + 3 * gi), by = __ldg(g.rays + 3 * gi + 1), bz = __ldg(g.rays + 3 * gi + 2);
        qg[e] = make_float4(bx, by, bz, __ldg(g.ref_gray + gi));
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            const float* r = g.rel_r[v];
            rq[(v * 3 + 0) * ne + e] = (double)dot3_f32(r[0], r[1], r[2], bx, by, bz);
            rq[(v * 3 + 1) * ne + e] = (double)dot3_f32(r[3], r[4], r[5], bx, by, bz);
            rq[(v * 3 + 2) * ne + e] = (double)dot3_f32(r[6], r[7], r[8], bx, by, bz);
        }
    }
    Tile t;
    t.qg = qg;
    t.rq = rq;
    t.wwc = wwc;
    t.ne = ne;
    t.sx = compress ? g.stride / 2 : g.stride;
    t.sy = g.stride * wwc;
    return t;
}

// K:190-198 (f64 accumulation of the f32 luma and of its f32 square)
__device__ __forceinline__ void pixel_stats(const FastGroup& g, const Tile& t, int ce, double& mr, double& sr) {
    double acc = 0.0, acc2 = 0.0;
    const int half = (g.ns - 1) / 2;
    int e_row = ce - half * (t.sx + t.sy);
    for (int j = 0; j < g.ns; ++j) {
        int e = e_row;
        for (int i = 0; i < g.ns; ++i) {
            const float v = t.qg[e].w;
            acc = __dadd_rn(acc, (double)v);
            acc2 = __dadd_rn(acc2, (double)__fmul_rn(v, v));
            e += t.sx;
        }
        e_row += t.sy;
    }
    const double m = acc * g.inv_s;  // S is a small integer: acc / S to <= 1 ulp, see note below
    // the reference divides (acc / S); multiply-by-reciprocal differs by <= 1 ulp of f64,
    // 12 orders below the parity tolerance.
    double var = __dsub_rn(acc2 * g.inv_s, __dmul_rn(m, m));
    var = var < 0.0 ? 0.0 : var;
    mr = m;
    sr = sqrt(var);
}

// 1/x, third-order refinement of the MUFU.RCP64H seed (2^-20 -> ~2^-60)
__device__ __forceinline__ double rcp3(double x) {
    const double y = rcp_seed(x);
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}
// 1/sqrt(x), third-order refinement of the MUFU.RSQ64H seed
__device__ __forceinline__ double rsqrt3(double x, double c0375) {
    const double y = rsqrt_seed(x);
    const double e = fma(-(x * y), y, 1.0);
    return fma(y * e, fma(e, c0375, 0.5), y);
}

// (u, v) of K:244-258 for the VT neighbour-frame points of one sample, rounded to f32 like the
// reference's scratch, then the f64 bilinear taps of K:134-153.  Written stage by stage over
// the views so that the VT independent dependency chains sit next to each other in program
// order (measured: -8 % on refine_pass versus one view after the other).
//
// No guards on the two measure-zero singularities (t on the neighbour's polar axis:
// max(|tx|,|tz|) = 0, or 1 - |ty|/|t| <= 0); they yield NaN, which cand_cost maps to `trunc`.
//
// Bilinear: the planes are padded (wrapped columns, replicated rows), so floor(u), floor(u)+1,
// floor(v), floor(v)+1 are all in-plane and the reference's wrap / clamp rules are data, not
// code; they are stored widened to f64 as { value, value(x+1) - value }, so a footprint is two
// 16-byte loads with no conversion and no subtraction (an f32 lerp costs up to
// 1e-2 relative on the cost of low-texture patches, measured).  floor by the 1.5 * 2^23 magic
// add; the element index is formed in f32 (exact below 2^23) and read out of the mantissa, so
// no F2I / I2F conversions are issued; all offsets are 32-bit element indices from one base.
#define D360_FORV for (int v = 0; v < VT; ++v)
template <int VT>
__device__ __forceinline__ void project_bilinear_all(const FastGroup& g, int v0, const double (&tx)[VT],
                                                     const double (&ty)[VT], const double (&tz)[VT],
                                                     double (&val)[VT]) {
    double r2[VT], y1[VT], e1[VT], a[VT], q[VT], w[VT], y2[VT], e2[VT], sq[VT];
#pragma unroll
    D360_FORV r2[v] = fma(tz[v], tz[v], fma(ty[v], ty[v], fma(tx[v], tx[v], g.tiny)));
#pragma unroll
    D360_FORV y1[v] = rsqrt_seed(r2[v]);
    double hi[VT], lo[VT], y3[VT];
    bool swap[VT];
#pragma unroll
    D360_FORV {
        swap[v] = fabs(tx[v]) > fabs(tz[v]);
        hi[v] = swap[v] ? tx[v] : tz[v];
        lo[v] = swap[v] ? tz[v] : tx[v];
    }
#pragma unroll
    D360_FORV y3[v] = rcp_seed(hi[v]);
#pragma unroll
    D360_FORV e1[v] = fma(-(r2[v] * y1[v]), y1[v], 1.0);
    double e3[VT];
#pragma unroll
    D360_FORV e3[v] = fma(-hi[v], y3[v], 1.0);
#pragma unroll
    D360_FORV y1[v] = fma(y1[v] * e1[v], fma(e1[v], g.c0375, 0.5), y1[v]);
#pragma unroll
    D360_FORV y3[v] = fma(y3[v], fma(e3[v], e3[v], e3[v]), y3[v]);
#pragma unroll
    D360_FORV a[v] = fabs(ty[v]) * y1[v];
    double r[VT], s[VT], p[VT];
#pragma unroll
    D360_FORV { r[v] = lo[v] * y3[v]; s[v] = r[v] * r[v]; }
#pragma unroll
    D360_FORV { w[v] = 1.0 - a[v]; y2[v] = rsqrt_seed(w[v]); }
#pragma unroll
    D360_FORV { q[v] = g.cq[0]; p[v] = g.ca[0]; }
#pragma unroll
    for (int i = 1; i < 8; ++i) {
#pragma unroll
        D360_FORV { q[v] = fma(a[v], q[v], g.cq[i]); p[v] = fma(s[v], p[v], g.ca[i]); }
    }
#pragma unroll
    D360_FORV e2[v] = fma(-(w[v] * y2[v]), y2[v], 1.0);  // (the compiler shares w y2 with s0 below)
#pragma unroll
    D360_FORV {  // sqrt(w) = s0 (1 + e/2 + 3e^2/8), s0 = w y2
        const double s0 = w[v] * y2[v];
        sq[v] = fma(s0 * e2[v], fma(e2[v], g.c0375, 0.5), s0);
    }
    float pu[VT], pv[VT];
#pragma unroll
    D360_FORV {
        const int hem = (unsigned)__double2hiint(ty[v]) >> 31 ^ 1;
        pv[v] = (float)fma(q[v] * sq[v], g.mv[hem], g.cv[hem]);
        const unsigned hx = (unsigned)__double2hiint(tx[v]), hz = (unsigned)__double2hiint(tz[v]);
        const int oct = (swap[v] ? 1 : 0) + 2 * (hz >> 31) + 4 * (hx >> 31);
        pu[v] = (float)fma(fabs(r[v]) * p[v], g.mu[oct], g.cu[oct]);
    }
    const float MAGIC = 12582912.0f;
    float fl_u[VT], fl_v[VT];
#pragma unroll
    D360_FORV { fl_u[v] = __fadd_rn(__fadd_rn(pu[v], MAGIC), -MAGIC); fl_v[v] = __fadd_rn(__fadd_rn(pv[v], MAGIC), -MAGIC); }
#pragma unroll
    D360_FORV { if (fl_u[v] > pu[v]) fl_u[v] -= 1.0f; if (fl_v[v] > pv[v]) fl_v[v] -= 1.0f; }
    unsigned idx[VT];
#pragma unroll
    D360_FORV {
        const float off = __fadd_rn(fmaf(fl_v[v], g.pitch_f, fl_u[v]), g.idx_bias);
        idx[v] = min((unsigned)__float_as_int(off) & 0x7fffffu, g.max_idx) + (unsigned)(v0 + v) * g.plane32;
    }
    const double2* __restrict__ nb = reinterpret_cast<const double2*>(g.nb64);  // { value, value(x+1) - value }
    double2 r0[VT], r1[VT];
#pragma unroll
    D360_FORV {
        r0[v] = __ldg(nb + idx[v]);
        r1[v] = __ldg(nb + (idx[v] + (unsigned)g.pitch));
    }
#pragma unroll
    D360_FORV {
        const double fu = (double)(pu[v] - fl_u[v]), fv = (double)(pv[v] - fl_v[v]);
        const double top = fma(r0[v].y, fu, r0[v].x);
        const double bot = fma(r1[v].y, fu, r1[v].x);
        val[v] = fma(bot - top, fv, top);
    }
}

template <int VT>
__device__ __forceinline__ double aggregate(double (&cv)[VT], int top_k) {
#pragma unroll
    for (int i = 1; i < VT; ++i) {
#pragma unroll
        for (int j = i; j > 0; --j) {
            const double lo = cv[j - 1] < cv[j] ? cv[j - 1] : cv[j];
            const double hi = cv[j - 1] < cv[j] ? cv[j] : cv[j - 1];
            cv[j - 1] = lo;
            cv[j] = hi;
        }
    }
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < VT; ++i)
        if (i < top_k) total = __dadd_rn(total, cv[i]);
    return __dmul_rn(1.0 / top_k, total);
}

// Cost of one hypothesis at the pixel whose window entry is `ce` (K:201-297).
template <int VT, typename HT>
__device__ __forceinline__ double cand_cost(const FastGroup& g, const Tile& t, int ce, double mr, double sr, HT d,
                                            HT nx, HT ny, HT nz) {
    const double trunc = g.trunc;
    const float4 a = t.qg[ce];
    double num;
    if constexpr (sizeof(HT) == 4) {
        const float ndota = dot3_f32(nx, ny, nz, a.x, a.y, a.z);
        if ((double)ndota >= -D360_FACING_EPS || sr < D360_SIGMA_EPS) return trunc;
        num = (double)__fmul_rn(d, ndota);
    } else {
        const double ndota = dot3_f64(nx, ny, nz, (double)a.x, (double)a.y, (double)a.z);
        if (ndota >= -D360_FACING_EPS || sr < D360_SIGMA_EPS) return trunc;
        num = __dmul_rn(d, ndota);
    }
    double s0[VT], ss0[VT], rs0[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) s0[v] = ss0[v] = rs0[v] = 0.0;
    bool bad = false;

    // lam_k = num / dn_k of sample k (K:240-247) and the f64 luma of that sample
    auto plane_depth = [&](int e, double& lam, double& rv) {
        const float4 q = t.qg[e];
        double dn;
        if constexpr (sizeof(HT) == 4) {
            const float den = dot3_f32(nx, ny, nz, q.x, q.y, q.z);
            bad = bad || (den > g.den_lim);
            dn = (double)fminf(den, g.den_lim);
        } else {
            const double den = fma(nz, (double)q.z, fma(ny, (double)q.y, nx * (double)q.x));
            const bool par = den > g.neg_par_eps;
            bad = bad || par;
            dn = par ? g.neg_par_eps : den;
        }
        lam = num * rcp3(dn);
        rv = (double)q.w;
    };

    // One flat loop over the S = ns * ns samples (dy outer, dx inner, E:60-65), software-pipelined
    // by hand: the serial lam chain of sample k+1 (LDS, dot, rcp seed, Newton) is issued next to
    // the VT projection chains of sample k instead of in front of them.
    const int half = (g.ns - 1) / 2;
    const int n_samples = g.ns * g.ns;
    const int row_wrap = t.sy - g.ns * t.sx;
    int e = ce - half * (t.sx + t.sy), col = 0;
    double lam, rv;
    plane_depth(e, lam, rv);
    for (int k = 0; k < n_samples; ++k) {
        int e_next = e + t.sx;
        if (++col == g.ns) { col = 0; e_next += row_wrap; }
        double lam_next = 0.0, rv_next = 0.0;
        if (k + 1 < n_samples) plane_depth(e_next, lam_next, rv_next);
        const double* rqe = t.rq + e;
        // views in chunks of at most 4 staged chains (more would not fit the register file)
        constexpr int VC = VT <= 4 ? VT : (VT + 1) / 2;
#pragma unroll
        for (int v0 = 0; v0 < VT; v0 += VC) {
            if (v0 == 0) {
                double tx[VC], ty[VC], tz[VC], val[VC];
#pragma unroll
                for (int v = 0; v < VC; ++v) {
                    tx[v] = fma(lam, rqe[(v * 3 + 0) * t.ne], g.rel_t[v][0]);
                    ty[v] = fma(lam, rqe[(v * 3 + 1) * t.ne], g.rel_t[v][1]);
                    tz[v] = fma(lam, rqe[(v * 3 + 2) * t.ne], g.rel_t[v][2]);
                }
                project_bilinear_all<VC>(g, 0, tx, ty, tz, val);
#pragma unroll
                for (int v = 0; v < VC; ++v) {
                    s0[v] += val[v];
                    ss0[v] = fma(val[v], val[v], ss0[v]);
                    rs0[v] = fma(rv, val[v], rs0[v]);
                }
            } else {
                constexpr int VR = VT - VC > 0 ? VT - VC : 1;  // second (last) chunk
                double tx[VR], ty[VR], tz[VR], val[VR];
#pragma unroll
                for (int v = 0; v < VR; ++v) {
                    tx[v] = fma(lam, rqe[((VC + v) * 3 + 0) * t.ne], g.rel_t[VC + v][0]);
                    ty[v] = fma(lam, rqe[((VC + v) * 3 + 1) * t.ne], g.rel_t[VC + v][1]);
                    tz[v] = fma(lam, rqe[((VC + v) * 3 + 2) * t.ne], g.rel_t[VC + v][2]);
                }
                project_bilinear_all<VR>(g, VC, tx, ty, tz, val);
#pragma unroll
                for (int v = 0; v < VR; ++v) {
                    s0[VC + v] += val[v];
                    ss0[VC + v] = fma(val[v], val[v], ss0[VC + v]);
                    rs0[VC + v] = fma(rv, val[v], rs0[VC + v]);
                }
            }
        }
        e = e_next;
        lam = lam_next;
        rv = rv_next;
    }
    if (bad) return trunc;

    const double inv_s = g.inv_s;
    double cv[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        cv[v] = trunc;
        const double m0 = s0[v] * inv_s;
        const double v0 = ss0[v] * inv_s - m0 * m0;
        if (!(v0 < D360_VAR_EPS)) {
            const double cov = rs0[v] * inv_s - mr * m0;
            double c = 1.0 - cov / (sr * sqrt(v0));
            c = c < 0.0 ? 0.0 : c;
            c = c > trunc ? trunc : c;
            cv[v] = c;
        }
    }
    const double total = aggregate<VT>(cv, g.top_k);
    return total == total ? total : trunc;  // NaN only from the unguarded polar singularities
}

// ---------------------------------------------------------------------------------------
// eval_costs, K:300-349
// ---------------------------------------------------------------------------------------
template <int VT>
__global__ void __launch_bounds__(THREADS, D360_FAST_MINB)
    k_eval(const __grid_constant__ FastGroup g, const float* __restrict__ depth, const float* __restrict__ normal,
           float* __restrict__ cost_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH_FULL;
    const Tile t = tile_setup<VT>(g, smem, x0, y0, TH_FULL, false, 0);
    __syncthreads();
    const int lx = threadIdx.x % TW, ly = threadIdx.x / TW;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= g.W || y >= g.H) return;
    const int ce = (ly + g.reach) * t.wwc + lx + g.reach;
    double mr, sr;
    pixel_stats(g, t, ce, mr, sr);
    const size_t i = (size_t)y * g.W + x;
    cost_out[i] = (float)cand_cost<VT, float>(g, t, ce, mr, sr, depth[i], normal[3 * i], normal[3 * i + 1],
                                              normal[3 * i + 2]);
}

// ---------------------------------------------------------------------------------------
// red_black_pass, K:352-473.  A CTA covers TW x TH_RB pixels, 256 of them of the requested
// colour.  The number of candidates a pixel has to evaluate varies (0..8 after the duplicate
// skipping of K:418-432), so the work is levelled through a CTA-wide queue:
//   phase 1  one thread per pixel: in-range, non-duplicate neighbours -> candidate mask;
//            patch statistics; exclusive scan of the counts; (pixel, neighbour) items queued;
//   phase 2  warps pull 32 items at a time and evaluate them (any lane, any pixel of the tile);
//   phase 3  one thread per pixel: strict-< arg-min over its candidates in neighbour order
//            (K:463; the cost of a hypothesis does not depend on evaluation order, so this is
//            the reference's sequential accept).
// ---------------------------------------------------------------------------------------
__constant__ int c_nbr2[8][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}, {0, -2}, {0, 2}, {-2, 0}, {2, 0}};

struct RbQueue {
    double2 stats[THREADS];            // (mr, sr) per pixel
    double costs[THREADS * 8];         // cost of neighbour j's hypothesis at pixel p
    unsigned short items[THREADS * 8]; // p * 8 + j
    int warp_totals[THREADS / 32];
    int total, next;
};

__host__ __device__ inline size_t rb_queue_offset(size_t tile) { return (tile + 15) & ~(size_t)15; }

template <int VT>
__global__ void __launch_bounds__(THREADS, D360_FAST_MINB)
    k_red_black(const __grid_constant__ FastGroup g, int parity, const float* __restrict__ depth_in,
                const float* __restrict__ normal_in, const float* __restrict__ cost_in, float* __restrict__ depth_out,
                float* __restrict__ normal_out, float* __restrict__ cost_out, unsigned long long* n_evals) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH_RB;  // x0 is even
    const bool compress = (g.stride & 1) == 0;
    RbQueue& q = *reinterpret_cast<RbQueue*>(smem + rb_queue_offset(tile_bytes(TW, TH_RB, g.reach, compress, VT)));
    if (threadIdx.x == 0) q.next = 0;
    const Tile t = tile_setup<VT>(g, smem, x0, y0, TH_RB, compress, (parity + y0) & 1);
    __syncthreads();

    // ---- phase 1
    const int tid = threadIdx.x;
    const int ly = tid / (TW / 2);
    const int y = y0 + ly;
    const int lx = 2 * (tid % (TW / 2)) + ((parity + y) & 1);
    const int x = x0 + lx;
    const bool live = x < g.W && y < g.H;
    if (y < g.H) {
        // carry the off-colour pixel of this pair over unchanged (E:575-577)
        const int xo = x0 + (lx ^ 1);
        if (xo < g.W) {
            const size_t o = (size_t)y * g.W + xo;
            depth_out[o] = depth_in[o];
            normal_out[3 * o] = normal_in[3 * o];
            normal_out[3 * o + 1] = normal_in[3 * o + 1];
            normal_out[3 * o + 2] = normal_in[3 * o + 2];
            cost_out[o] = cost_in[o];
        }
    }
    const size_t i = live ? (size_t)y * g.W + x : 0;
    unsigned mask = 0;
    if (live) {
        // K:418-432 skips exact duplicates of the best-so-far and of already evaluated
        // candidates.  Every earlier in-range neighbour was either evaluated or itself such a
        // duplicate, so comparing with the pixel's original hypothesis and with the earlier
        // neighbours selects the same set, except that it also skips re-evaluating the original
        // hypothesis once it has been displaced, which strict < would reject anyway.
        const float od = depth_in[i];
        const float onx = normal_in[3 * i], ony = normal_in[3 * i + 1], onz = normal_in[3 * i + 2];
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            const int qy = y + c_nbr2[j][1];
            if (qy < 0 || qy >= g.H) continue;  // K:407 rows skipped
            const size_t qi = (size_t)qy * g.W + wrap_once(x + c_nbr2[j][0], g.W);  // K:410-413 columns wrap
            const float d = depth_in[qi];
            const float nx = normal_in[3 * qi], ny = normal_in[3 * qi + 1], nz = normal_in[3 * qi + 2];
            bool dup = d == od && nx == onx && ny == ony && nz == onz;
            for (int m = 0; m < j; ++m) {
                const int my = y + c_nbr2[m][1];
                if (my < 0 || my >= g.H) continue;
                const size_t mi = (size_t)my * g.W + wrap_once(x + c_nbr2[m][0], g.W);
                if (depth_in[mi] == d)
                    dup = dup || (normal_in[3 * mi] == nx && normal_in[3 * mi + 1] == ny &&
                                  normal_in[3 * mi + 2] == nz);
            }
            if (!dup) mask |= 1u << j;
        }
    }
    const int n_mine = __popc(mask);
    if (n_mine) {
        const int ce = (ly + g.reach) * t.wwc + (compress ? (lx + g.reach) >> 1 : lx + g.reach);
        double mr, sr;
        pixel_stats(g, t, ce, mr, sr);
        q.stats[tid] = make_double2(mr, sr);
    }
    int incl = n_mine;  // CTA-wide exclusive scan of the counts
    for (int o = 1; o < 32; o <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= o) incl += up;
    }
    if ((tid & 31) == 31) q.warp_totals[tid >> 5] = incl;
    __syncthreads();
    int off = incl - n_mine;
    for (int w = 0; w < (tid >> 5); ++w) off += q.warp_totals[w];
    if (tid == THREADS - 1) q.total = off + n_mine;
    for (unsigned m = mask; m; m &= m - 1) q.items[off++] = (unsigned short)(tid * 8 + (__ffs(m) - 1));
    __syncthreads();

    // ---- phase 2
    const int total = q.total;
    for (;;) {
        int base = 0;
        if ((tid & 31) == 0) base = atomicAdd(&q.next, 32);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= total) break;
        const int it = base + (tid & 31);
        if (it < total) {
            const int item = q.items[it];
            const int p = item >> 3, j = item & 7;
            const int ply = p / (TW / 2);
            const int py = y0 + ply;
            const int plx = 2 * (p % (TW / 2)) + ((parity + py) & 1);
            const int px = x0 + plx;
            const size_t qi = (size_t)(py + c_nbr2[j][1]) * g.W + wrap_once(px + c_nbr2[j][0], g.W);
            const int ce = (ply + g.reach) * t.wwc + (compress ? (plx + g.reach) >> 1 : plx + g.reach);
            const double2 st = q.stats[p];
            q.costs[item] = cand_cost<VT, float>(g, t, ce, st.x, st.y, depth_in[qi], normal_in[3 * qi],
                                                 normal_in[3 * qi + 1], normal_in[3 * qi + 2]);
        }
    }
    __syncthreads();

    // ---- phase 3
    if (live) {
        double bc = (double)cost_in[i];
        int bj = -1;
        for (unsigned m = mask; m; m &= m - 1) {
            const int j = __ffs(m) - 1;
            const double c = q.costs[tid * 8 + j];
            if (c < bc) {  // K:463
                bc = c;
                bj = j;
            }
        }
        size_t bi = i;
        if (bj >= 0) bi = (size_t)(y + c_nbr2[bj][1]) * g.W + wrap_once(x + c_nbr2[bj][0], g.W);
        depth_out[i] = depth_in[bi];
        normal_out[3 * i] = normal_in[3 * bi];
        normal_out[3 * i + 1] = normal_in[3 * bi + 1];
        normal_out[3 * i + 2] = normal_in[3 * bi + 2];
        cost_out[i] = (float)bc;
    }
    if (n_evals != nullptr && tid == 0 && total) atomicAdd(n_evals, (unsigned long long)total);
}

// ---------------------------------------------------------------------------------------
// refine_pass, K:476-610.  Loop-carried d, n, c are f64 as in the reference.
// ---------------------------------------------------------------------------------------
template <int VT>
__global__ void __launch_bounds__(THREADS, D360_FAST_MINB)
    k_refine(const __grid_constant__ FastGroup g, const __grid_constant__ RefineTable tab, float* __restrict__ depth,
             float* __restrict__ normal, float* __restrict__ cost, unsigned long long* n_evals) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH_FULL;
    const Tile t = tile_setup<VT>(g, smem, x0, y0, TH_FULL, false, 0);
    __syncthreads();
    const int lx = threadIdx.x % TW, ly = threadIdx.x / TW;
    const int x = x0 + lx, y = y0 + ly;
    unsigned int evals = 0;
    if (x < g.W && y < g.H) {
        const int ce = (ly + g.reach) * t.wwc + lx + g.reach;
        const size_t i = (size_t)y * g.W + x;
        double d = depth[i];
        double nx = normal[3 * i], ny = normal[3 * i + 1], nz = normal[3 * i + 2];
        double c = cost[i];
        const float4 a4 = t.qg[ce];
        const double ax = a4.x, ay = a4.y, az = a4.z;
        double mr, sr;
        pixel_stats(g, t, ce, mr, sr);
        bool stale = true;
        double e1x = 0, e1y = 0, e1z = 0, e2x = 0, e2y = 0, e2z = 0;
#pragma unroll 1
        for (int k = 0; k < tab.n; ++k) {
            double nd = __dadd_rn(d, (double)tab.dd[k]);
            if (nd < tab.depth_min) nd = tab.depth_min;
            else if (nd > tab.depth_max) nd = tab.depth_max;
            if (stale) {
                e1x = __dsub_rn(__dmul_rn(ny, az), __dmul_rn(nz, ay));
                e1y = __dsub_rn(__dmul_rn(nz, ax), __dmul_rn(nx, az));
                e1z = __dsub_rn(__dmul_rn(nx, ay), __dmul_rn(ny, ax));
                double m2 = dot3_f64(e1x, e1y, e1z, e1x, e1y, e1z);
                if (m2 < 1e-12) {
                    e1x = -nz; e1y = 0.0; e1z = nx;
                    m2 = __dadd_rn(__dmul_rn(e1x, e1x), __dmul_rn(e1z, e1z));
                    if (m2 < 1e-12) { e1x = 1.0; e1z = 0.0; m2 = 1.0; }
                }
                const double inv = 1.0 / sqrt(m2);
                e1x = __dmul_rn(e1x, inv); e1y = __dmul_rn(e1y, inv); e1z = __dmul_rn(e1z, inv);
                e2x = __dsub_rn(__dmul_rn(ny, e1z), __dmul_rn(nz, e1y));
                e2y = __dsub_rn(__dmul_rn(nz, e1x), __dmul_rn(nx, e1z));
                e2z = __dsub_rn(__dmul_rn(nx, e1y), __dmul_rn(ny, e1x));
                stale = false;
            }
            const double sa = tab.sa[k], ca = tab.ca[k], caz = tab.caz[k], saz = tab.saz[k];
            double cnx = __dadd_rn(__dmul_rn(nx, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1x, caz), __dmul_rn(e2x, saz)), sa));
            double cny = __dadd_rn(__dmul_rn(ny, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1y, caz), __dmul_rn(e2y, saz)), sa));
            double cnz = __dadd_rn(__dmul_rn(nz, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1z, caz), __dmul_rn(e2z, saz)), sa));
            const double nrm = sqrt(dot3_f64(cnx, cny, cnz, cnx, cny, cnz));
            if (nrm < 1e-12) continue;
            const double inv = 1.0 / nrm;
            cnx = __dmul_rn(cnx, inv); cny = __dmul_rn(cny, inv); cnz = __dmul_rn(cnz, inv);
            const double ev = cand_cost<VT, double>(g, t, ce, mr, sr, nd, cnx, cny, cnz);
            ++evals;
            if (ev < c) {
                c = ev; d = nd; nx = cnx; ny = cny; nz = cnz;
                stale = true;
            }
        }
        depth[i] = (float)d;
        normal[3 * i] = (float)nx;
        normal[3 * i + 1] = (float)ny;
        normal[3 * i + 2] = (float)nz;
        cost[i] = (float)c;
    }
    if (n_evals != nullptr) {
        for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
        if ((threadIdx.x & 31) == 0 && evals) atomicAdd(n_evals, (unsigned long long)evals);
    }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
static bool make_fast_group(const GroupDev& gd, FastGroup* out) {
    // regular grid?  S = ns^2, offsets (dx, dy) = stride * (i - half, j - half), dy outer (E:60-65)
    int ns = 1;
    while (ns * ns < gd.S) ++ns;
    if (ns * ns != gd.S || (ns & 1) == 0) return false;
    const int half = (ns - 1) / 2;
    const int stride = ns > 1 ? gd.dx[1] - gd.dx[0] : 1;
    if (stride < 1) return false;
    for (int k = 0; k < gd.S; ++k) {
        if (gd.dx[k] != (k % ns - half) * stride || gd.dy[k] != (k / ns - half) * stride) return false;
    }
    if (gd.nb_pad_x < 1 || gd.nb_pad_y < 1 || gd.nb64 == nullptr) return false;  // needs padded f64 planes
    const long long pitch = gd.W + 2 * gd.nb_pad_x, rows = gd.H + 2 * gd.nb_pad_y;
    if (pitch * rows >= (1ll << 23)) return false;  // f32 index arithmetic must stay exact
    FastGroup& g = *out;
    g.W = gd.W; g.H = gd.H; g.ns = ns; g.stride = stride; g.reach = half * stride; g.top_k = gd.top_k;
    g.pitch = (int)pitch;
    g.plane = (size_t)(pitch * rows);
    g.max_idx = (unsigned)(pitch * rows - pitch - 2);
    g.pitch_f = (float)pitch;
    g.idx_bias = 8388608.0f + (float)(gd.nb_pad_y * pitch + gd.nb_pad_x);
    g.rays = gd.rays; g.ref_gray = gd.ref_gray; g.nb64 = gd.nb64;
    for (int v = 0; v < gd.V; ++v) {
        for (int i = 0; i < 9; ++i) g.rel_r[v][i] = gd.rel_r[v][i];
        for (int i = 0; i < 3; ++i) g.rel_t[v][i] = (double)gd.rel_t[v][i];
    }
    const double hw = gd.W * (0.5 / D360_PI), ls = gd.H / D360_PI;
    for (int oct = 0; oct < 8; ++oct) {
        const bool swap = oct & 1, xneg = oct & 2, yneg = oct & 4;
        // theta = sy * (cx + sx * (cs + ss * p)), K:96-99
        const double ss = swap ? -1.0 : 1.0, cs = swap ? D360_HALF_PI : 0.0;
        const double sx = xneg ? -1.0 : 1.0, cx = xneg ? D360_PI : 0.0;
        const double sy = yneg ? -1.0 : 1.0;
        g.mu[oct] = sy * sx * ss * hw;
        g.cu[oct] = (sy * (cx + sx * cs) + D360_PI) * hw - 0.5;
    }
    g.mv[0] = ls;  g.cv[0] = -0.5;                  // ty < 0: sphi > 0
    g.mv[1] = -ls; g.cv[1] = D360_PI * ls - 0.5;    // ty > 0: sphi < 0, acos = pi - p (K:131)
    static const double CA[8] = {-5.021063913876e-03, 2.533170107199e-02, -6.087448223083e-02, 1.000220525649e-01,
                                 -1.404782123164e-01, 1.997402857787e-01, -3.333223261885e-01, 9.999999227776e-01};
    static const double CQ[8] = {-1.223553911532e-03, 6.510368059701e-03, -1.682974898800e-02, 3.068214201158e-02,
                                 -5.008467775423e-02, 8.895977933699e-02, -2.145970563340e-01, 1.570796263346e00};
    for (int i = 0; i < 8; ++i) { g.ca[i] = CA[i]; g.cq[i] = CQ[i]; }
    if ((unsigned long long)(pitch * rows) * (unsigned long long)gd.V >= (1ull << 32)) return false;
    g.plane32 = (unsigned)(pitch * rows);
    g.neg_par_eps = -D360_PARALLEL_EPS;
    g.tiny = 1e-30;
    g.c0375 = 0.375;
    g.trunc = gd.trunc;
    g.inv_s = 1.0 / gd.S;
    g.den_lim = nextafterf((float)(-D360_PARALLEL_EPS), -1.0f);
    if ((double)g.den_lim >= -D360_PARALLEL_EPS) g.den_lim = nextafterf(g.den_lim, -1.0f);
    return true;
}

template <typename K>
static int prepare(K kernel, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(%zu B smem): %s", smem, cudaGetErrorString(e));
        return 1;
    }
    return 0;
}

#define D360_FAST_DISPATCH(V, ...)                             \
    switch (V) {                                                \
        case 1: { constexpr int VT = 1; __VA_ARGS__; } break;   \
        case 2: { constexpr int VT = 2; __VA_ARGS__; } break;   \
        case 3: { constexpr int VT = 3; __VA_ARGS__; } break;   \
        case 4: { constexpr int VT = 4; __VA_ARGS__; } break;   \
        case 6: { constexpr int VT = 6; __VA_ARGS__; } break;   \
        default: return -1;                                     \
    }

}  // namespace fast

using namespace fast;

// Each returns -1 when the fast path does not apply (caller falls back to the generic kernel).
int fast_eval(const GroupDev& gd, const float* depth, const float* normal, float* cost_out, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    const size_t smem = tile_bytes(TW, TH_FULL, g.reach, false, gd.V);
    if (smem > 200 * 1024) return -1;
    dim3 grid((gd.W + TW - 1) / TW, (gd.H + TH_FULL - 1) / TH_FULL);
    D360_FAST_DISPATCH(gd.V, {
        auto k = k_eval<VT>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("eval_costs", s);
        k<<<grid, THREADS, smem, s>>>(g, depth, normal, cost_out);
    })
    return check_launch("eval_costs");
}

int fast_red_black(const GroupDev& gd, int parity, const float* di, const float* ni, const float* ci, float* dout,
                   float* nout, float* cout, unsigned long long* n_evals, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    const size_t smem = rb_queue_offset(tile_bytes(TW, TH_RB, g.reach, (g.stride & 1) == 0, gd.V)) + sizeof(RbQueue);
    if (smem > 200 * 1024) return -1;
    dim3 grid((gd.W + TW - 1) / TW, (gd.H + TH_RB - 1) / TH_RB);
    D360_FAST_DISPATCH(gd.V, {
        auto k = k_red_black<VT>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("red_black", s);
        k<<<grid, THREADS, smem, s>>>(g, parity, di, ni, ci, dout, nout, cout, n_evals);
    })
    return check_launch("red_black_pass");
}

int fast_refine(const GroupDev& gd, const RefineTable& tab, float* depth, float* normal, float* cost,
                unsigned long long* n_evals, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    const size_t smem = tile_bytes(TW, TH_FULL, g.reach, false, gd.V);
    if (smem > 200 * 1024) return -1;
    dim3 grid((gd.W + TW - 1) / TW, (gd.H + TH_FULL - 1) / TH_FULL);
    D360_FAST_DISPATCH(gd.V, {
        auto k = k_refine<VT>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("refine", s);
        k<<<grid, THREADS, smem, s>>>(g, tab, depth, normal, cost, n_evals);
    })
    return check_launch("refine_pass");
}

}  // namespace d360
