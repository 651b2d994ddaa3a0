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
    const double* nb64;   // padded planes widened to f64, see d360.h
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
#ifdef D360_NEWTON2
    return fma(y, e, y);
#else
    return fma(y, fma(e, e, e), y);
#endif
}
// 1/sqrt(x), third-order refinement of the MUFU.RSQ64H seed
__device__ __forceinline__ double rsqrt3(double x, double c0375) {
    const double y = rsqrt_seed(x);
    const double e = fma(-(x * y), y, 1.0);
#ifdef D360_NEWTON2
    return fma(y * e, 0.5, y);
#else
    return fma(y * e, fma(e, c0375, 0.5), y);
#endif
}

// (u, v) of K:244-258 for one neighbour-frame point t, rounded to f32 like the reference's
// scratch.  No guards on the two measure-zero singularities (t on the neighbour's polar axis:
// max(|tx|,|tz|) = 0 or 1 - |ty|/|t| <= 0); they yield NaN, which cand_cost maps to `trunc`.
__device__ __forceinline__ void project(const FastGroup& g, double tx, double ty, double tz, float& pu, float& pv) {
    // latitude: v = acos_poly(-ty / |t|) * H/pi - 0.5  (K:102-131)
    const double r2 = fma(tz, tz, fma(ty, ty, fma(tx, tx, g.tiny)));
    const double a = fabs(ty) * rsqrt3(r2, g.c0375);
#ifdef D360_ESTRIN
    double q;
    {
        const double a2 = a * a, a4 = a2 * a2;
        const double b3 = fma(g.cq[0], a, g.cq[1]), b2 = fma(g.cq[2], a, g.cq[3]);
        const double b1 = fma(g.cq[4], a, g.cq[5]), b0 = fma(g.cq[6], a, g.cq[7]);
        q = fma(fma(b3, a2, b2), a4, fma(b1, a2, b0));
    }
#else
    double q = g.cq[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) q = fma(a, q, g.cq[i]);
#endif
    const double w = 1.0 - a;
    const double sq = w * rsqrt3(w, g.c0375);
    const int hem = (unsigned)__double2hiint(ty) >> 31 ^ 1;  // 1 when ty >= +0: sphi <= -0 (K:131)
    pv = (float)fma(q * sq, g.mv[hem], g.cv[hem]);

    // longitude: u = (atan2_poly(tx, tz) + pi) * W/2pi - 0.5  (K:59-99)
    const unsigned hx = (unsigned)__double2hiint(tx), hz = (unsigned)__double2hiint(tz);
    const bool swap = fabs(tx) > fabs(tz);
    const double hi = swap ? tx : tz, lo = swap ? tz : tx;
    const double r = lo * rcp3(hi);  // signed; only |r| is used (abs is a free operand modifier)
    const double s = r * r;
#ifdef D360_ESTRIN
    double p;
    {
        const double s2 = s * s, s4 = s2 * s2;
        const double b3 = fma(g.ca[0], s, g.ca[1]), b2 = fma(g.ca[2], s, g.ca[3]);
        const double b1 = fma(g.ca[4], s, g.ca[5]), b0 = fma(g.ca[6], s, g.ca[7]);
        p = fma(fma(b3, s2, b2), s4, fma(b1, s2, b0));
    }
#else
    double p = g.ca[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) p = fma(s, p, g.ca[i]);
#endif
    const int oct = (swap ? 1 : 0) + 2 * (hz >> 31) + 4 * (hx >> 31);
    pu = (float)fma(fabs(r) * p, g.mu[oct], g.cu[oct]);
}

// K:134-153 on the f32 (u, v), interpolated in f64 like the reference (the planes are stored
// widened, so the taps need no conversion; an f32 lerp costs up to 1e-2 relative on the cost of
// low-texture patches, measured).  The plane is padded
// (wrapped columns, replicated rows), so floor(u), floor(u)+1, floor(v), floor(v)+1 are all
// in-plane and the reference's wrap / clamp rules are data, not code.  floor by the
// 1.5 * 2^23 magic add; the element index is formed in f32 (exact below 2^23) and read out of
// the mantissa, so no F2I / I2F conversions are issued.
__device__ __forceinline__ double bilinear(const FastGroup& g, unsigned view_off, float u, float v) {
    const float MAGIC = 12582912.0f;
    float fl_u = __fadd_rn(__fadd_rn(u, MAGIC), -MAGIC);
    if (fl_u > u) fl_u -= 1.0f;
    float fl_v = __fadd_rn(__fadd_rn(v, MAGIC), -MAGIC);
    if (fl_v > v) fl_v -= 1.0f;
    const double fu = (double)(u - fl_u), fv = (double)(v - fl_v);  // the f32 differences are exact
    const float off = __fadd_rn(fmaf(fl_v, g.pitch_f, fl_u), g.idx_bias);
    // min: only non-finite (u, v) can exceed it.  All offsets are 32-bit element indices from
    // one 64-bit base, so each tap costs one IMAD.WIDE.
    const unsigned idx = min((unsigned)__float_as_int(off) & 0x7fffffu, g.max_idx) + view_off;
    const double* __restrict__ nb = g.nb64;
    const double a = __ldg(nb + idx), b = __ldg(nb + idx + 1u);
    const unsigned idx1 = idx + (unsigned)g.pitch;
    const double c = __ldg(nb + idx1), d = __ldg(nb + idx1 + 1u);
    const double top = fma(b - a, fu, a);
    const double bot = fma(d - c, fu, c);
    return fma(bot - top, fv, top);
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
#ifdef D360_ACC32
    // mean-shifted f32 sums: a = val - mr, b = ref - mr
    const float mrf = (float)mr;
    float a0[VT], a1[VT], a2[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) a0[v] = a1[v] = a2[v] = 0.0f;
#else
    double s0[VT], ss0[VT], rs0[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) s0[v] = ss0[v] = rs0[v] = 0.0;
#endif
    bool bad = false;

    const int half = (g.ns - 1) / 2;
    int e_row = ce - half * (t.sx + t.sy);
    for (int j = 0; j < g.ns; ++j) {
        int e = e_row;
        for (int i = 0; i < g.ns; ++i) {
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
            const double lam = num * rcp3(dn);
#ifndef D360_ACC32
            const double rv = (double)q.w;
#endif
            const double* rqe = t.rq + e;
#pragma unroll
            for (int v = 0; v < VT; ++v) {
                const double tx = fma(lam, rqe[(v * 3 + 0) * t.ne], g.rel_t[v][0]);
                const double ty = fma(lam, rqe[(v * 3 + 1) * t.ne], g.rel_t[v][1]);
                const double tz = fma(lam, rqe[(v * 3 + 2) * t.ne], g.rel_t[v][2]);
                float pu, pv;
                project(g, tx, ty, tz, pu, pv);
#ifdef D360_ACC32
                const float valf = bilinear(g, v * g.plane32, pu, pv) - mrf;
                a0[v] += valf;
                a1[v] = fmaf(valf, valf, a1[v]);
                a2[v] = fmaf(q.w - mrf, valf, a2[v]);
#else
                const double val = bilinear(g, v * g.plane32, pu, pv);
                s0[v] += val;
                ss0[v] = fma(val, val, ss0[v]);
                rs0[v] = fma(rv, val, rs0[v]);
#endif
            }
            e += t.sx;
        }
        e_row += t.sy;
    }
    if (bad) return trunc;

    const double inv_s = g.inv_s;
    double cv[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        cv[v] = trunc;
#ifdef D360_ACC32
        // sums of shifted values: mean(b) = mr - mrf (tiny), so cov = E[ab] - E[a] E[b]
        const double ma = (double)a0[v] * inv_s;
        const double m0 = ma + (double)mrf;
        const double v0 = (double)a1[v] * inv_s - ma * ma;
        (void)m0;
        if (!(v0 < D360_VAR_EPS)) {
            const double cov = (double)a2[v] * inv_s - ma * (mr - (double)mrf);
#else
        const double m0 = s0[v] * inv_s;
        const double v0 = ss0[v] * inv_s - m0 * m0;
        if (!(v0 < D360_VAR_EPS)) {
            const double cov = rs0[v] * inv_s - mr * m0;
#endif
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
// red_black_pass, K:352-473.  A CTA covers TW x TH_RB pixels; each of its 256 threads owns one
// pixel of the requested colour and carries its off-colour neighbour over unchanged.
// ---------------------------------------------------------------------------------------
__constant__ int c_nbr2[8][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}, {0, -2}, {0, 2}, {-2, 0}, {2, 0}};

template <int VT>
__global__ void __launch_bounds__(THREADS, D360_FAST_MINB)
    k_red_black(const __grid_constant__ FastGroup g, int parity, const float* __restrict__ depth_in,
                const float* __restrict__ normal_in, const float* __restrict__ cost_in, float* __restrict__ depth_out,
                float* __restrict__ normal_out, float* __restrict__ cost_out, unsigned long long* n_evals) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH_RB;  // x0 is even
    const bool compress = (g.stride & 1) == 0;
    const Tile t = tile_setup<VT>(g, smem, x0, y0, TH_RB, compress, (parity + y0) & 1);
    __syncthreads();
    const int ly = threadIdx.x / (TW / 2);
    const int y = y0 + ly;
    const int lx = 2 * (threadIdx.x % (TW / 2)) + ((parity + y) & 1);
    const int x = x0 + lx;
    unsigned int evals = 0;
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
    if (x < g.W && y < g.H) {
        const size_t i = (size_t)y * g.W + x;
        // original hypothesis of the pixel: a neighbour equal to it is a duplicate for the whole
        // pass (its cost is cost_in, which can never beat the running best under strict <)
        const float od = depth_in[i];
        const float onx = normal_in[3 * i], ony = normal_in[3 * i + 1], onz = normal_in[3 * i + 2];
        float bd = od, bnx = onx, bny = ony, bnz = onz;
        double bc = (double)cost_in[i];
        const int ce = (ly + g.reach) * t.wwc + (compress ? (lx + g.reach) >> 1 : lx + g.reach);
        double mr = 0.0, sr = 0.0;
        bool gathered = false;
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            const int qy = y + c_nbr2[j][1];
            if (qy < 0 || qy >= g.H) continue;  // K:407 rows skipped
            const int qx = wrap_once(x + c_nbr2[j][0], g.W);  // K:410-413 columns wrap
            const size_t qi = (size_t)qy * g.W + qx;
            const float d = depth_in[qi];
            const float nx = normal_in[3 * qi], ny = normal_in[3 * qi + 1], nz = normal_in[3 * qi + 2];
            // K:418-432: skip exact duplicates of the best-so-far / of an already evaluated
            // candidate.  Every earlier in-range neighbour was either evaluated or itself such a
            // duplicate, so comparing with the original hypothesis and with the earlier
            // neighbours (re-read through L1 instead of being kept in 32 registers) selects the
            // same set, except that it also skips re-evaluating the original hypothesis once it
            // has been displaced, which the strict < would reject anyway.
            bool dup = d == od && nx == onx && ny == ony && nz == onz;
            for (int m = 0; m < j; ++m) {
                const int my = y + c_nbr2[m][1];
                if (my < 0 || my >= g.H) continue;
                const size_t mi = (size_t)my * g.W + wrap_once(x + c_nbr2[m][0], g.W);
                if (depth_in[mi] == d)
                    dup = dup || (normal_in[3 * mi] == nx && normal_in[3 * mi + 1] == ny &&
                                  normal_in[3 * mi + 2] == nz);
            }
            if (dup) continue;
            if (!gathered) {
                pixel_stats(g, t, ce, mr, sr);
                gathered = true;
            }
            const double c = cand_cost<VT, float>(g, t, ce, mr, sr, d, nx, ny, nz);
            ++evals;
            if (c < bc) {  // K:463
                bc = c;
                bd = d; bnx = nx; bny = ny; bnz = nz;
            }
        }
        depth_out[i] = bd;
        normal_out[3 * i] = bnx;
        normal_out[3 * i + 1] = bny;
        normal_out[3 * i + 2] = bnz;
        cost_out[i] = (float)bc;
    }
    if (n_evals != nullptr) {
        for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
        if ((threadIdx.x & 31) == 0 && evals) atomicAdd(n_evals, (unsigned long long)evals);
    }
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
    const size_t smem = tile_bytes(TW, TH_RB, g.reach, (g.stride & 1) == 0, gd.V);
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
