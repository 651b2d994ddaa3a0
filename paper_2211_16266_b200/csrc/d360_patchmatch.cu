// PatchMatch cost / propagation / refinement kernels for sm_100a.
//
// One thread evaluates one plane hypothesis for one pixel: S patch samples x V views of
//   bearing -> plane intersection -> neighbour sphere -> (lon, lat) -> bilinear -> NCC sums
// (K:201-297).  A CTA owns a TILE_W x TILE_H pixel tile; the per-sample context the
// reference gathers per pixel (K:156-198: sample ray q, R_v q, reference luma) depends only
// on the sample pixel, so it is built once per tile (with a `reach` halo, columns wrapped,
// rows clamped) in shared memory and shared by every pixel and every candidate of the tile.
//
// Arithmetic follows the reference's numba type inference: f32 hypothesis
// dot products in eval_costs / red_black_pass, f64 hypotheses in refine_pass, f64
// projection, (u, v) rounded to f32, NCC sums in f64.  The f64 work runs on the B200's
// half-rate FP64 pipe concurrently with the FP32/ALU/LSU work of the bilinear taps.
#include <math.h>

#include "d360_device.cuh"

namespace d360 {

constexpr int TILE_W = 32;
constexpr int TILE_H = 8;
constexpr int RB_THREADS = (TILE_W / 2) * TILE_H;

struct Tile {
    const float4* qg;   // (qx, qy, qz, reference luma) per window entry
    const double* rq;   // [(v*3 + c) * ne + entry]  R_v q as f64 (exact widening of f32)
    int ww, ne;
};

__host__ __device__ inline size_t tile_smem_bytes(int tw, int th, int reach, int n_views) {
    size_t ne = (size_t)(tw + 2 * reach) * (th + 2 * reach);
    return ne * sizeof(float4) + ne * sizeof(double) * 3 * n_views;
}

// Build the tile context.  Window entry (i, j) <-> pixel ((x0 - R + i) mod W,
// clamp(y0 - R + j, 0, H-1)), matching K:168-177 for every pixel of the tile.
__device__ __forceinline__ Tile tile_setup(const GroupDev& g, unsigned char* smem, int x0, int y0,
                                           int tw, int th) {
    const int R = g.reach;
    const int ww = tw + 2 * R, hh = th + 2 * R, ne = ww * hh;
    float4* qg = reinterpret_cast<float4*>(smem);
    double* rq = reinterpret_cast<double*>(smem + (size_t)ne * sizeof(float4));
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const int j = e / ww, i = e - j * ww;
        const int gx = pos_mod(x0 - R + i, g.W);
        const int gy = min(max(y0 - R + j, 0), g.H - 1);
        const size_t gi = (size_t)gy * g.W + gx;
        const float bx = __ldg(g.rays + 3 * gi), by = __ldg(g.rays + 3 * gi + 1),
                    bz = __ldg(g.rays + 3 * gi + 2);
        qg[e] = make_float4(bx, by, bz, __ldg(g.ref_gray + gi));
        for (int v = 0; v < g.V; ++v) {
            const float* r = g.rel_r[v];
            rq[(size_t)(v * 3 + 0) * ne + e] = (double)dot3_f32(r[0], r[1], r[2], bx, by, bz);
            rq[(size_t)(v * 3 + 1) * ne + e] = (double)dot3_f32(r[3], r[4], r[5], bx, by, bz);
            rq[(size_t)(v * 3 + 2) * ne + e] = (double)dot3_f32(r[6], r[7], r[8], bx, by, bz);
        }
    }
    Tile t;
    t.qg = qg;
    t.rq = rq;
    t.ww = ww;
    t.ne = ne;
    return t;
}

// Patch mean / population sigma of the reference samples, K:190-198 (f64 accumulation of
// f32 values, f32 squares).
__device__ __forceinline__ void pixel_stats(const GroupDev& g, const Tile& t, int ce, double& mr,
                                            double& sr) {
    double acc = 0.0, acc2 = 0.0;
    for (int k = 0; k < g.S; ++k) {
        const float v = t.qg[ce + g.dy[k] * t.ww + g.dx[k]].w;
        acc = __dadd_rn(acc, (double)v);
        acc2 = __dadd_rn(acc2, (double)__fmul_rn(v, v));
    }
    const double m = acc / g.S;
    double var = __dsub_rn(acc2 / g.S, __dmul_rn(m, m));
    var = var < 0.0 ? 0.0 : var;
    mr = m;
    sr = sqrt(var);
}

// K:134-153 on the f32-rounded projection.  EXACT: f64 weights like the reference.
template <int MODE>
__device__ __forceinline__ double bilinear(const float* __restrict__ img, int H, int W, int pitch, float u,
                                           float v) {
    const float fl = floorf(u);
    int u0 = (int)fl;
    u0 = u0 < 0 ? u0 + W : u0;
    u0 = u0 >= W ? u0 - W : u0;
    u0 = min(max(u0, 0), W - 1);  // memory safety on non-finite input only
    int u1 = u0 + 1;
    u1 = u1 == W ? 0 : u1;
    float vc = v < 0.0f ? 0.0f : v;
    const float vm = (float)(H - 1);
    vc = vc > vm ? vm : vc;
    int v0 = (int)vc;
    v0 = v0 > H - 2 ? H - 2 : v0;
    v0 = max(v0, 0);
    const float* r0 = img + (size_t)v0 * pitch;
    const float* r1 = r0 + pitch;
    const float a = __ldg(r0 + u0), b = __ldg(r0 + u1), c = __ldg(r1 + u0), d = __ldg(r1 + u1);
    if constexpr (MODE == D360_PREC_EXACT) {
        const double fu = (double)u - (double)fl;
        const double fv = (double)vc - (double)v0;
        const double top = __dadd_rn(__dmul_rn(a, 1.0 - fu), __dmul_rn(b, fu));
        const double bot = __dadd_rn(__dmul_rn(c, 1.0 - fu), __dmul_rn(d, fu));
        return __dadd_rn(__dmul_rn(top, 1.0 - fv), __dmul_rn(bot, fv));
    } else {
        const float fu = u - fl;               // exact
        const float fv = vc - (float)v0;       // exact
        const float top = fmaf(b - a, fu, a);
        const float bot = fmaf(d - c, fu, c);
        return (double)fmaf(bot - top, fv, top);
    }
}

// Top-k aggregation: mean of the k smallest per-view costs, summed ascending.
template <int VT>
__device__ __forceinline__ double aggregate(double* cv, int V, int top_k) {
    constexpr int N = VT > 0 ? VT : D360_MAX_VIEWS;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        if (i < V) {
#pragma unroll
            for (int j = i; j > 0; --j) {
                const double lo = fmin(cv[j - 1], cv[j]), hi = fmax(cv[j - 1], cv[j]);
                cv[j - 1] = lo;
                cv[j] = hi;
            }
        }
    }
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (i < top_k) total = __dadd_rn(total, cv[i]);
    return __dmul_rn(1.0 / top_k, total);
}

// Cost of one hypothesis at the pixel whose window entry is `ce` (K:201-297).
// HT = float for f32 hypotheses (eval_costs, red_black_pass), double inside refine_pass.
template <int MODE, int VT, typename HT>
__device__ __forceinline__ double cand_cost(const GroupDev& g, const Tile& t, int ce, double mr,
                                            double sr, HT d, HT nx, HT ny, HT nz) {
    constexpr int NV = VT > 0 ? VT : D360_MAX_VIEWS;
    const int V = VT > 0 ? VT : g.V;
    const double trunc = g.trunc;
    const float4 a = t.qg[ce];
    HT ndota;
    if constexpr (sizeof(HT) == 4) ndota = dot3_f32(nx, ny, nz, a.x, a.y, a.z);
    else ndota = dot3_f64(nx, ny, nz, (double)a.x, (double)a.y, (double)a.z);
    if ((double)ndota >= -D360_FACING_EPS || sr < D360_SIGMA_EPS) return trunc;
    HT num_h;
    if constexpr (sizeof(HT) == 4) num_h = __fmul_rn(d, ndota);
    else num_h = __dmul_rn(d, ndota);
    const double num = (double)num_h;

    const double half_w = g.W * (0.5 / D360_PI);
    const double lat_scale = g.H / D360_PI;
    const int H = g.H, W = g.W;
    const int pitch = W + 2 * g.nb_pad_x;
    const size_t plane = (size_t)(H + 2 * g.nb_pad_y) * pitch;
    const float* nb0 = g.nb + (size_t)g.nb_pad_y * pitch + g.nb_pad_x;  // pixel (0, 0) of view 0

    double s0[NV], ss0[NV], rs0[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) s0[v] = ss0[v] = rs0[v] = 0.0;
    bool bad = false;

    for (int k = 0; k < g.S; ++k) {
        const int e = ce + g.dy[k] * t.ww + g.dx[k];
        const float4 q = t.qg[e];
        double den;
        if constexpr (sizeof(HT) == 4) den = (double)dot3_f32(nx, ny, nz, q.x, q.y, q.z);
        else den = dot3_f64(nx, ny, nz, (double)q.x, (double)q.y, (double)q.z);
        bad = bad || (den > -D360_PARALLEL_EPS);
        const double dn = den < -D360_PARALLEL_EPS ? den : -D360_PARALLEL_EPS;
        const double lam = div_<MODE>(num, dn);
        const double rv = (double)q.w;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if (v < V) {
                const double* rqv = t.rq + (size_t)(v * 3) * t.ne + e;
                const double tx = madd<MODE>(lam, rqv[0], (double)g.rel_t[v][0]);
                const double ty = madd<MODE>(lam, rqv[t.ne], (double)g.rel_t[v][1]);
                const double tz = madd<MODE>(lam, rqv[2 * t.ne], (double)g.rel_t[v][2]);
                double r2 = madd<MODE>(tz, tz, madd<MODE>(ty, ty, __dmul_rn(tx, tx)));
                r2 = __dadd_rn(r2, 1e-30);
                double inv_r;
                if constexpr (MODE == D360_PREC_EXACT) inv_r = 1.0 / sqrt(r2);
                else inv_r = fast_rsqrt(r2);
                const double sphi = -ty * inv_r;
                const float pu =
                    (float)madd<MODE>(__dadd_rn(fast_atan2<MODE>(tx, tz), D360_PI), half_w, -0.5);
                const float pv = (float)madd<MODE>(fast_acos<MODE>(sphi), lat_scale, -0.5);
                const double val = bilinear<MODE>(nb0 + v * plane, H, W, pitch, pu, pv);
                s0[v] = __dadd_rn(s0[v], val);
                ss0[v] = madd<MODE>(val, val, ss0[v]);
                rs0[v] = madd<MODE>(rv, val, rs0[v]);
            }
        }
    }
    if (bad) return trunc;

    const double inv_s = 1.0 / g.S;
    double cv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        cv[v] = trunc;
        if (v < V) {
            const double m0 = s0[v] * inv_s;
            const double v0 = __dsub_rn(__dmul_rn(ss0[v], inv_s), __dmul_rn(m0, m0));
            if (!(v0 < D360_VAR_EPS)) {
                const double cov = __dsub_rn(__dmul_rn(rs0[v], inv_s), __dmul_rn(mr, m0));
                double c = 1.0 - cov / (sr * sqrt(v0));
                c = c < 0.0 ? 0.0 : c;
                c = c > trunc ? trunc : c;
                cv[v] = c;
            }
        }
    }
    return aggregate<VT>(cv, V, g.top_k);
}

// ---------------------------------------------------------------------------------------
// eval_costs, K:300-349
// ---------------------------------------------------------------------------------------
template <int MODE, int VT>
__global__ void __launch_bounds__(TILE_W* TILE_H)
    k_eval_costs(const __grid_constant__ GroupDev g, const float* __restrict__ depth,
                 const float* __restrict__ normal, float* __restrict__ cost_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TILE_W, y0 = blockIdx.y * TILE_H;
    const Tile t = tile_setup(g, smem, x0, y0, TILE_W, TILE_H);
    __syncthreads();
    const int lx = threadIdx.x % TILE_W, ly = threadIdx.x / TILE_W;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= g.W || y >= g.H) return;
    const int ce = (ly + g.reach) * t.ww + lx + g.reach;
    double mr, sr;
    pixel_stats(g, t, ce, mr, sr);
    const size_t i = (size_t)y * g.W + x;
    const double c = cand_cost<MODE, VT, float>(g, t, ce, mr, sr, depth[i], normal[3 * i],
                                                normal[3 * i + 1], normal[3 * i + 2]);
    cost_out[i] = (float)c;
}

// ---------------------------------------------------------------------------------------
// red_black_pass, K:352-473.  A CTA covers a TILE_W x TILE_H region; its RB_THREADS threads
// own the pixels of the requested colour and also carry the other colour over unchanged.
// ---------------------------------------------------------------------------------------
__constant__ int c_nbr[8][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}, {0, -2}, {0, 2}, {-2, 0}, {2, 0}};

template <int MODE, int VT>
__global__ void __launch_bounds__(RB_THREADS)
    k_red_black(const __grid_constant__ GroupDev g, int parity, const float* __restrict__ depth_in,
                const float* __restrict__ normal_in, const float* __restrict__ cost_in,
                float* __restrict__ depth_out, float* __restrict__ normal_out,
                float* __restrict__ cost_out, unsigned long long* n_evals) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TILE_W, y0 = blockIdx.y * TILE_H;
    const Tile t = tile_setup(g, smem, x0, y0, TILE_W, TILE_H);
    __syncthreads();
    const int ly = threadIdx.x / (TILE_W / 2);
    const int y = y0 + ly;
    const int lx = 2 * (threadIdx.x % (TILE_W / 2)) + ((parity + y) & 1);  // x0 is even
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
        float bd = depth_in[i];
        float bnx = normal_in[3 * i], bny = normal_in[3 * i + 1], bnz = normal_in[3 * i + 2];
        double bc = (double)cost_in[i];
        const int ce = (ly + g.reach) * t.ww + lx + g.reach;
        double mr = 0.0, sr = 0.0;
        bool gathered = false;
        float cd[8], cx[8], cy[8], cz[8];
        int n_seen = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int qy = y + c_nbr[j][1];
            if (qy < 0 || qy >= g.H) continue;
            const int qx = wrap_once(x + c_nbr[j][0], g.W);
            const size_t qi = (size_t)qy * g.W + qx;
            const float d = depth_in[qi];
            const float nx = normal_in[3 * qi], ny = normal_in[3 * qi + 1], nz = normal_in[3 * qi + 2];
            bool dup = d == bd && nx == bnx && ny == bny && nz == bnz;
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m < j && m < n_seen)
                    dup = dup || (d == cd[m] && nx == cx[m] && ny == cy[m] && nz == cz[m]);
            if (dup) continue;
            // n_seen <= j, so the static-index store below keeps cd[] in registers
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m == n_seen) { cd[m] = d; cx[m] = nx; cy[m] = ny; cz[m] = nz; }
            ++n_seen;
            if (!gathered) {
                pixel_stats(g, t, ce, mr, sr);
                gathered = true;
            }
            const double c = cand_cost<MODE, VT, float>(g, t, ce, mr, sr, d, nx, ny, nz);
            ++evals;
            if (c < bc) {
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
template <int MODE, int VT>
__global__ void __launch_bounds__(TILE_W* TILE_H)
    k_refine(const __grid_constant__ GroupDev g, const __grid_constant__ RefineTable tab,
             float* __restrict__ depth, float* __restrict__ normal, float* __restrict__ cost,
             unsigned long long* n_evals) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int x0 = blockIdx.x * TILE_W, y0 = blockIdx.y * TILE_H;
    const Tile t = tile_setup(g, smem, x0, y0, TILE_W, TILE_H);
    __syncthreads();
    const int lx = threadIdx.x % TILE_W, ly = threadIdx.x / TILE_W;
    const int x = x0 + lx, y = y0 + ly;
    unsigned int evals = 0;
    if (x < g.W && y < g.H) {
        const int ce = (ly + g.reach) * t.ww + lx + g.reach;
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
            const double ev = cand_cost<MODE, VT, double>(g, t, ce, mr, sr, nd, cnx, cny, cnz);
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

__global__ void k_valid_from_cost(const float* __restrict__ cost, float trunc, uint8_t* valid,
                                  size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) valid[i] = cost[i] < trunc;  // E:629 (f32 compare, NumPy weak scalar)
}

// ---------------------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------------------
template <typename K>
static int prepare_kernel(K kernel, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(%zu B smem): %s", smem, cudaGetErrorString(e));
            return 1;
        }
    }
    return 0;
}

#define D360_DISPATCH_V(V, ...)                               \
    switch (V) {                                               \
        case 1: { constexpr int VT = 1; __VA_ARGS__; } break;  \
        case 2: { constexpr int VT = 2; __VA_ARGS__; } break;  \
        case 4: { constexpr int VT = 4; __VA_ARGS__; } break;  \
        case 6: { constexpr int VT = 6; __VA_ARGS__; } break;  \
        default: { constexpr int VT = 0; __VA_ARGS__; } break; \
    }

#define D360_DISPATCH(PREC, V, ...)                                                         \
    if ((PREC) == D360_PREC_EXACT) { constexpr int MODE = D360_PREC_EXACT; D360_DISPATCH_V(V, __VA_ARGS__) } \
    else { constexpr int MODE = D360_PREC_MIXED; D360_DISPATCH_V(V, __VA_ARGS__) }

static int launch_eval(const GroupDev& gd, int prec, const float* depth, const float* normal,
                       float* cost_out, cudaStream_t s) {
    if (prec == D360_PREC_MIXED) {
        const int frc = fast_eval(gd, depth, normal, cost_out, s);
        if (frc >= 0) return frc;
        note_generic_fallback("eval_costs", gd);
    }
    const size_t smem = tile_smem_bytes(TILE_W, TILE_H, gd.reach, gd.V);
    dim3 grid((gd.W + TILE_W - 1) / TILE_W, (gd.H + TILE_H - 1) / TILE_H);
    int rc = 0;
    D360_DISPATCH(prec, gd.V, {
        auto k = k_eval_costs<MODE, VT>;
        rc = prepare_kernel(k, smem);
        if (!rc) {
            TraceScope ts_("eval_costs", s);
            k<<<grid, TILE_W * TILE_H, smem, s>>>(gd, depth, normal, cost_out);
        }
    })
    return rc ? rc : check_launch("eval_costs");
}

// changed_in / changed_out, memo_valid / memo_cost (optional): memoised candidate costs of the
// throughput kernels (d360_fast_rb.cu).  The generic kernels do not use them; they mark every
// pixel changed and drop every memo entry, which is always safe.
static int launch_red_black(const GroupDev& gd, int prec, int parity, const float* di,
                            const float* ni, const float* ci, float* dout, float* nout, float* cout,
                            const unsigned char* changed_in, unsigned char* changed_out,
                            unsigned char* memo_valid, double* memo_cost, unsigned long long* n_evals,
                            cudaStream_t s) {
    if (prec == D360_PREC_MIXED) {
        const int frc = fast_red_black(gd, parity, di, ni, ci, dout, nout, cout, changed_in, changed_out, memo_valid,
                                       memo_cost, n_evals, s);
        if (frc >= 0) return frc;
        note_generic_fallback("red_black_pass", gd);
    }
    if (memo_valid != nullptr && cudaMemsetAsync(memo_valid, 0, (size_t)gd.W * gd.H, s) != cudaSuccess) {
        set_error("cudaMemsetAsync(memo validity) failed");
        return 1;
    }
    if (changed_out != nullptr && cudaMemsetAsync(changed_out, 1, (size_t)gd.W * gd.H, s) != cudaSuccess) {
        set_error("cudaMemsetAsync(changed flags) failed");
        return 1;
    }
    const size_t smem = tile_smem_bytes(TILE_W, TILE_H, gd.reach, gd.V);
    dim3 grid((gd.W + TILE_W - 1) / TILE_W, (gd.H + TILE_H - 1) / TILE_H);
    int rc = 0;
    D360_DISPATCH(prec, gd.V, {
        auto k = k_red_black<MODE, VT>;
        rc = prepare_kernel(k, smem);
        if (!rc) {
            TraceScope ts_("red_black", s);
            k<<<grid, RB_THREADS, smem, s>>>(gd, parity, di, ni, ci, dout, nout, cout, n_evals);
        }
    })
    return rc ? rc : check_launch("red_black_pass");
}

static int launch_refine(const GroupDev& gd, int prec, const RefineTable& tab, float* depth,
                         float* normal, float* cost, unsigned char* changed, unsigned long long* n_evals,
                         cudaStream_t s) {
    if (prec == D360_PREC_MIXED) {
        const int frc = fast_refine(gd, tab, depth, normal, cost, changed, n_evals, s);
        if (frc >= 0) return frc;
        note_generic_fallback("refine_pass", gd);
    }
    if (changed != nullptr && cudaMemsetAsync(changed, 1, (size_t)gd.W * gd.H, s) != cudaSuccess) {
        set_error("cudaMemsetAsync(changed flags) failed");
        return 1;
    }
    const size_t smem = tile_smem_bytes(TILE_W, TILE_H, gd.reach, gd.V);
    dim3 grid((gd.W + TILE_W - 1) / TILE_W, (gd.H + TILE_H - 1) / TILE_H);
    int rc = 0;
    D360_DISPATCH(prec, gd.V, {
        auto k = k_refine<MODE, VT>;
        rc = prepare_kernel(k, smem);
        if (!rc) {
            TraceScope ts_("refine", s);
            k<<<grid, TILE_W * TILE_H, smem, s>>>(gd, tab, depth, normal, cost, n_evals);
        }
    })
    return rc ? rc : check_launch("refine_pass");
}

static int fill_table(RefineTable* tab, const float* dd, const float* sa, const float* ca,
                      const float* caz, const float* saz, int n, double dmin, double dmax) {
    if (n < 0 || n > D360_MAX_REFINE) {
        set_error("n_cand %d outside [0, %d]", n, D360_MAX_REFINE);
        return 1;
    }
    if (!(dmin > 0.0 && dmax > dmin)) {
        set_error("depth range must satisfy 0 < min < max, got [%g, %g]", dmin, dmax);
        return 1;
    }
    tab->n = n;
    tab->depth_min = dmin;
    tab->depth_max = dmax;
    for (int i = 0; i < n; ++i) {
        tab->dd[i] = dd[i]; tab->sa[i] = sa[i]; tab->ca[i] = ca[i]; tab->caz[i] = caz[i]; tab->saz[i] = saz[i];
    }
    return 0;
}

}  // namespace d360

using namespace d360;

extern "C" int d360_eval_costs(const d360_group* g, const float* depth, const float* normal,
                               float* cost_out, void* stream) {
    GroupDev gd;
    if (make_group_dev(g, &gd)) return 1;
    return launch_eval(gd, g->precision, depth, normal, cost_out, (cudaStream_t)stream);
}

extern "C" int d360_red_black_pass(const d360_group* g, int parity, const float* depth_in,
                                   const float* normal_in, const float* cost_in, float* depth_out,
                                   float* normal_out, float* cost_out, unsigned long long* n_evals,
                                   void* stream) {
    GroupDev gd;
    if (make_group_dev(g, &gd)) return 1;
    if (parity != 0 && parity != 1) {
        set_error("parity must be 0 or 1, got %d", parity);
        return 1;
    }
    if (depth_in == depth_out || normal_in == normal_out || cost_in == cost_out) {
        set_error("red_black_pass must be double-buffered (K:371-377): in/out alias");
        return 1;
    }
    return launch_red_black(gd, g->precision, parity, depth_in, normal_in, cost_in, depth_out,
                            normal_out, cost_out, nullptr, nullptr, nullptr, nullptr, n_evals, (cudaStream_t)stream);
}

extern "C" int d360_refine_pass(const d360_group* g, float* depth, float* normal, float* cost,
                                const float* cand_dd, const float* cand_sa, const float* cand_ca,
                                const float* cand_caz, const float* cand_saz, int n_cand,
                                double depth_min, double depth_max, void* stream) {
    GroupDev gd;
    if (make_group_dev(g, &gd)) return 1;
    RefineTable tab;
    if (fill_table(&tab, cand_dd, cand_sa, cand_ca, cand_caz, cand_saz, n_cand, depth_min, depth_max))
        return 1;
    return launch_refine(gd, g->precision, tab, depth, normal, cost, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int d360_run_patchmatch(const d360_group* g, float* depth, float* normal, float* cost,
                                   float* scratch_depth, float* scratch_normal, float* scratch_cost,
                                   uint8_t* scratch_flags, double* scratch_memo, const float* tables, int iterations,
                                   int n_cand, double depth_min,
                                   double depth_max, uint8_t* valid_out, unsigned long long* n_evals,
                                   void* stream) {
    GroupDev gd;
    if (make_group_dev(g, &gd)) return 1;
    if (iterations < 1) {
        set_error("patchmatch.iterations must be >= 1, got %d", iterations);
        return 1;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int prec = g->precision;
    if (launch_eval(gd, prec, depth, normal, cost, s)) return 1;
    float *cd = depth, *cn = normal, *cc = cost;
    float *nd = scratch_depth, *nn = scratch_normal, *nc = scratch_cost;
    // memoised candidate costs: two "changed" flag planes (read one / write the other, swapped per
    // iteration), one validity plane, eight f64 costs per pixel
    const size_t n_px = (size_t)gd.W * gd.H;
    const bool memo = scratch_flags != nullptr && scratch_memo != nullptr;
    unsigned char* chg_in = memo ? scratch_flags : nullptr;
    unsigned char* chg_out = memo ? scratch_flags + n_px : nullptr;
    unsigned char* memo_valid = memo ? scratch_flags + 2 * n_px : nullptr;
    double* memo_cost = memo ? scratch_memo : nullptr;
    if (memo && (cudaMemsetAsync(chg_in, 1, n_px, s) != cudaSuccess ||
                 cudaMemsetAsync(memo_valid, 0, n_px, s) != cudaSuccess)) {
        set_error("cudaMemsetAsync(memo flags) failed");
        return 1;
    }
    for (int it = 0; it < iterations; ++it) {
        // The two colours never read each other (every neighbour offset of K:44-56 keeps x + y even or
        // odd), so the throughput kernel takes both passes in one launch; the generic kernels run them
        // one after the other as the reference does.
        int frc = -1;
        if (prec == D360_PREC_MIXED)
            frc = fast_red_black(gd, 2, cd, cn, cc, nd, nn, nc, chg_in, chg_out, memo_valid, memo_cost, n_evals, s);
        if (frc > 0) return 1;
        const int n_pass = frc == 0 ? 1 : 2;
        for (int parity = 0; parity < n_pass; ++parity) {
            if (frc != 0 &&
                launch_red_black(gd, prec, parity, cd, cn, cc, nd, nn, nc, chg_in, chg_out, memo_valid, memo_cost, n_evals, s))
                return 1;
            float* tmp;
            tmp = cd; cd = nd; nd = tmp;
            tmp = cn; cn = nn; nn = tmp;
            tmp = cc; cc = nc; nc = tmp;
        }
        RefineTable tab;
        const float* tb = tables + (size_t)it * 5 * n_cand;
        if (fill_table(&tab, tb, tb + n_cand, tb + 2 * n_cand, tb + 3 * n_cand, tb + 4 * n_cand, n_cand,
                       depth_min, depth_max))
            return 1;
        if (launch_refine(gd, prec, tab, cd, cn, cc, chg_out, n_evals, s)) return 1;
        unsigned char* tmpc = chg_in; chg_in = chg_out; chg_out = tmpc;
    }
    if (cd != depth) {  // an odd number of buffer swaps: the result goes back to the caller's buffers
        if (cudaMemcpyAsync(depth, cd, n_px * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(normal, cn, 3 * n_px * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(cost, cc, n_px * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
            set_error("cudaMemcpyAsync(result) failed");
            return 1;
        }
        cc = cost;
    }
    if (valid_out != nullptr) {
        const size_t n = n_px;
        {
            TraceScope ts_("valid_from_cost", s);
            k_valid_from_cost<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cc, (float)gd.trunc, valid_out, n);
        }
        if (check_launch("valid_from_cost")) return 1;
    }
    return 0;
}
