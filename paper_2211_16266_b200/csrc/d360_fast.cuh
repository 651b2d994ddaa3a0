// Throughput build of the PatchMatch cost evaluation (precision policy D360_PREC_MIXED on a
// regular sample grid) for sm_100a: shared device code of d360_fast_{eval,rb,refine}.cu.
//
// Same algorithm and same decision rules as d360_patchmatch.cu (K:156-297, K:300-610), with
// the per-sample-view instruction stream cut to what the B200's pipes need:
//   * FP64 pipe (64 lanes/clk/SM, DFMA latency 8 clk, the binding resource): ~50 operations
//     per sample-view — t = lam * Rq + t_v, |t|^2, one third-order rsqrt / rcp refinement of
//     the MUFU.64H seeds (error ~1e-18, no IEEE div/sqrt), the two degree-7 Horner chains of
//     the reference's atan2 / acos polynomials, the f64 bilinear and the three NCC sums;
//   * octant / hemisphere fix-ups of K:90-99 and K:129-131 are folded into one DFMA whose
//     multiplier and addend come from 8- and 2-entry constant tables indexed by sign bits;
//   * XU pipe (16 lanes/clk/SM): 3 MUFU.64H seeds + 4 F2F (u, v -> f32 as the reference's
//     f32 scratch K:250-258, the exact f32 fractions -> f64); floor / frac of (u, v) use the
//     1.5 * 2^23 magic-add on the FP32 pipe instead of F2I / I2F;
//   * the patch geometry (samples per side, stride) is a template parameter for the
//     reference's default patch, so every shared-memory offset is an immediate.
// (u, v) are therefore the reference's f64 values to ~1e-12 px before the f32 rounding, which
// is what holds the 1e-4 relative cost parity.
//
// One lane evaluates one hypothesis over all V views.  (Splitting an evaluation over a lane
// pair, V / 2 views each, was built and measured: 80 registers and 3 CTAs per SM, but +25 %
// instructions for the duplicated plane-depth chain and the per-lane view addressing, and the
// smaller L1 next to 3 x 72 KB of shared memory: 20 % slower.  See DESIGN.md.)
#pragma once
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched through the runtime, no -lcuda)
#include <math.h>

#include "d360_device.cuh"

namespace d360 {
namespace fast {

constexpr int TW = 32;  // tile width (pixels)
// octant table slots, in 16-byte entries (FastGroup::uo)
constexpr int OCT_SX = 1, OCT_SZ = 16, OCT_SW = 4, OCT_SLOTS = OCT_SX + OCT_SZ + OCT_SW + 1;

#ifndef D360_W_FUSED
#define D360_W_FUSED 1
#endif
#ifndef D360_PIN_C38
#define D360_PIN_C38 1
#endif
#ifndef D360_NT
#define D360_NT 256  // threads per CTA
#endif
#ifndef D360_MINB
#define D360_MINB 2  // CTAs per SM the register budget is sized for (128 registers)
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
    // longitude: u = p * uo[k].x + uo[k].y, k = OCT_SX * (tx < 0) + OCT_SZ * (tz < 0) + OCT_SW * (|tx| > |tz|):
    // the slots a byte permute of the two sign bytes plus one predicated OR can address (see project_uv)
    double2 uo[OCT_SLOTS];
    double2 vo[2];        // latitude: v = p * vo[ty >= 0].x + vo[ty >= 0].y  (index 1: ty < 0)
    double ca[8], cq[8];  // atan polynomial in s = (lo / hi)^2 (K:75-85) and acos polynomial re-expanded in
                          // w = 1 - |sphi| (K:112-122), highest degree first, divided by the leading
                          // coefficient ([0] unused; it is folded into uo / vo)
    double trunc, inv_s;
    double neg_par_eps, tiny, c0375;  // -PARALLEL_EPS, 1e-30 (K:246), 3/8: 64-bit literals live in the constant bank
    unsigned plane32;     // plane as a 32-bit element count
    float pitch_f;        // pitch as float
    float idx_bias;       // 2^23 + pad_y * pitch + pad_x: float -> index by mantissa extraction (big planes: 2^23 + pad_x)
    float den_lim;        // largest f32 below -PARALLEL_EPS
    int big;              // a plane holds 2^23 texels or more: row and column are combined in integer arithmetic
    unsigned big_const;   // (pad_y - 2^22) * pitch, mod 2^32: the row bias of the 1.5 * 2^23 floor, see gather_bilinear
};

// V views, NS x NS samples at stride ST (NS = 0: taken from the FastGroup at run time).  BIG: padded planes of
// 2^23 texels or more (beyond 3840x1920, e.g. the paper's 5760x2880 quality mode), see gather_bilinear.
template <int V_, int NS_, int ST_, bool BIG_ = false>
struct Cfg {
    static constexpr int VT = V_, V = V_;
    static constexpr bool BIG = BIG_;
    static constexpr int NT = D360_NT;
    static constexpr int MINB = D360_MINB;
    static constexpr int TH_FULL = NT / TW;    // eval / refine: NT pixels per CTA
    static constexpr int TH_RB = 2 * NT / TW;  // red-black: NT pixels of the updated colour per CTA
    static constexpr int NS = NS_, ST = ST_;
    __host__ __device__ static int ns(const FastGroup& g) { return NS_ > 0 ? NS_ : g.ns; }
    __host__ __device__ static int stride(const FastGroup& g) { return NS_ > 0 ? ST_ : g.stride; }
    __host__ __device__ static int reach(const FastGroup& g) { return NS_ > 0 ? (NS_ - 1) / 2 * ST_ : g.reach; }
};

// Patch context of a CTA tile in shared memory.  Window entry (i, j) <-> pixel
// ((x0 - R + i) mod W, clamp(y0 - R + j, 0, H-1)), K:168-177.  With `compress` (red-black pass
// on an even sample stride: every sample of an updated pixel has the pixel's colour) only the
// entries of that colour are kept, two window columns per slot — half the shared memory, and
// neighbouring lanes read neighbouring slots.
struct Tile {
    const float4* qg;  // (qx, qy, qz, reference luma) per entry
    // R_v q as f64 (exact widening of the f32 dot, K:184-189), laid out for 16-byte loads:
    // rxy[v * ne + entry] = (x, y) of view v;  rz[(v / 2) * ne + entry] = z of views (v & ~1, v | 1)
    const double2* rxy;
    const double2* rz;
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
    return ne * sizeof(float4) + ne * sizeof(double2) * (n_views + (n_views + 1) / 2);
}

// R_v q of window entry e for all views, from its ray q
template <class C>
__device__ __forceinline__ void store_rq(const FastGroup& g, double2* rxy, double2* rz, int ne, int e, float qx,
                                         float qy, float qz) {
#pragma unroll
    for (int v = 0; v < C::V; v += 2) {
        double z[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2 && v + h < C::V; ++h) {
            const float* r = g.rel_r[v + h];
            rxy[(v + h) * ne + e] = make_double2((double)dot3_f32(r[0], r[1], r[2], qx, qy, qz),
                                                 (double)dot3_f32(r[3], r[4], r[5], qx, qy, qz));
            z[h] = (double)dot3_f32(r[6], r[7], r[8], qx, qy, qz);
        }
        rz[(v >> 1) * ne + e] = make_double2(z[0], z[1]);
    }
}

__host__ __device__ inline size_t mbar_offset(size_t tile) { return (tile + 15) & ~(size_t)15; }

template <class C>
__device__ __forceinline__ Tile tile_setup(const FastGroup& g, unsigned char* smem, int x0, int y0, int th,
                                           bool compress, int keep) {
    const int R = C::reach(g);
    const int ww = TW + 2 * R, hh = th + 2 * R;
    const int wwc = compress ? ww / 2 : ww;
    const int ne = wwc * hh;
    float4* qg = reinterpret_cast<float4*>(smem);
    double2* rxy = reinterpret_cast<double2*>(smem + (size_t)ne * sizeof(float4));
    double2* rz = rxy + (size_t)C::V * ne;
    for (int e = threadIdx.x; e < ne; e += C::NT) {
        const int j = e / wwc, ic = e - j * wwc;
        const int i = compress ? 2 * ic + ((keep + j) & 1) : ic;
        const int gx = pos_mod(x0 - R + i, g.W);
        const int gy = min(max(y0 - R + j, 0), g.H - 1);
        const size_t gi = (size_t)gy * g.W + gx;
        const float bx = __ldg(g.rays + 3 * gi), by = __ldg(g.rays + 3 * gi + 1), bz = __ldg(g.rays + 3 * gi + 2);
        qg[e] = make_float4(bx, by, bz, __ldg(g.ref_gray + gi));
        store_rq<C>(g, rxy, rz, ne, e, bx, by, bz);
    }
    Tile t;
    t.qg = qg;
    t.rxy = rxy;
    t.rz = rz;
    t.wwc = wwc;
    t.ne = ne;
    t.sx = compress ? C::stride(g) / 2 : C::stride(g);
    t.sy = C::stride(g) * wwc;
    return t;
}

// The same window staged by TMA (eval / refine, no colour compression): the reference's (ray, luma)
// context lives in one padded float4 plane (d360_group.ref_ctx: wrapped columns, replicated rows,
// so K:168-177's wrap / clamp is data), and the window of a CTA is exactly one box of it.  One
// thread arms an mbarrier with the box's byte count and issues cp.async.bulk.tensor.2d; the TMA
// unit writes the ww x hh float4 entries row-major to the start of shared memory, which is the
// layout tile_setup produces, while the CTA's other warps are already through their index
// arithmetic.  Then every thread derives R_v q of its entries from shared memory.
struct WindowMap {
    CUtensorMap map;  // 2-D f32 tensor (H + 2p rows, 4 (W + 2p) floats per row), box = (4 ww, hh)
    int pad;          // p; < 0: no map, use tile_setup
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <class C>
__device__ __forceinline__ Tile tile_setup_tma(const FastGroup& g, const WindowMap& wm, unsigned char* smem,
                                               unsigned long long* mbar, int x0, int y0, int th) {
    const int R = C::reach(g);
    const int ww = TW + 2 * R, hh = th + 2 * R;
    const int ne = ww * hh;
    float4* qg = reinterpret_cast<float4*>(smem);
    double2* rxy = reinterpret_cast<double2*>(smem + (size_t)ne * sizeof(float4));
    double2* rz = rxy + (size_t)C::V * ne;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                     "r"((unsigned)(ne * sizeof(float4)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(qg)),
            "l"(reinterpret_cast<unsigned long long>(&wm.map)), "r"(4 * (x0 - R + wm.pad)), "r"(y0 - R + wm.pad),
            "r"(smem_u32(mbar))
            : "memory");
    }
    __syncthreads();  // the barrier is initialised for everyone
    {
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(mbar))
                : "memory");
        }
    }
    for (int e = threadIdx.x; e < ne; e += C::NT) {
        const float4 q = qg[e];
        store_rq<C>(g, rxy, rz, ne, e, q.x, q.y, q.z);
    }
    Tile t;
    t.qg = qg;
    t.rxy = rxy;
    t.rz = rz;
    t.wwc = ww;
    t.ne = ne;
    t.sx = C::stride(g);
    t.sy = C::stride(g) * ww;
    return t;
}

// K:190-198 (f64 accumulation of the f32 luma and of its f32 square)
template <class C>
__device__ __forceinline__ void pixel_stats(const FastGroup& g, const Tile& t, int ce, double& mr, double& sr) {
    double acc = 0.0, acc2 = 0.0;
    const int ns = C::ns(g);
    const int half = (ns - 1) / 2;
    int e_row = ce - half * (t.sx + t.sy);
#pragma unroll 1
    for (int j = 0; j < ns; ++j) {
        int e = e_row;
#pragma unroll
        for (int i = 0; i < ns; ++i) {
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

// Stage A of one sample: (u, v) of K:244-258 for the VT neighbour-frame points, rounded to f32
// like the reference's scratch.  Written stage by stage over the views so that the VT
// independent dependency chains sit next to each other in program order.
//
// No guards on the two measure-zero singularities (t on the neighbour's polar axis:
// max(|tx|,|tz|) = 0, or 1 - |ty|/|t| <= 0); they yield NaN, which the caller maps to `trunc`.
#define D360_FORV for (int v = 0; v < VT; ++v)
template <int VT>
__device__ __forceinline__ void project_uv(const FastGroup& g, double c38, const double (&tx)[VT],
                                           const double (&ty)[VT], const double (&tz)[VT], float (&pu)[VT],
                                           float (&pv)[VT]) {
    double r2[VT], y1[VT], e1[VT], q[VT], w[VT], y2[VT], e2[VT], sq[VT];
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
    D360_FORV y1[v] = fma(y1[v] * e1[v], fma(e1[v], c38, 0.5), y1[v]);
#pragma unroll
    D360_FORV y3[v] = fma(y3[v], fma(e3[v], e3[v], e3[v]), y3[v]);
    double r[VT], s[VT], p[VT];
#pragma unroll
    D360_FORV { r[v] = lo[v] * y3[v]; s[v] = r[v] * r[v]; }
    // w = 1 - |sphi| = 1 - |ty| / |t| in one rounding; the acos polynomial is expanded in w
#pragma unroll
#if D360_W_FUSED
    D360_FORV { w[v] = fma(-fabs(ty[v]), y1[v], 1.0); y2[v] = rsqrt_seed(w[v]); }
#else
    double a[VT];
    D360_FORV { a[v] = fabs(ty[v]) * y1[v]; w[v] = 1.0 - a[v]; y2[v] = rsqrt_seed(w[v]); }
#define w a
#endif
    // Horner on the monic polynomials (coefficients divided by the leading one, which is folded
    // into the uo / vo tables): the first step is an add with one constant operand instead of an
    // FMA with two, which would cost two register moves per polynomial.
#pragma unroll
    D360_FORV { q[v] = w[v] + g.cq[1]; p[v] = s[v] + g.ca[1]; }
#pragma unroll
    for (int i = 2; i < 8; ++i) {
#pragma unroll
        D360_FORV { q[v] = fma(w[v], q[v], g.cq[i]); p[v] = fma(s[v], p[v], g.ca[i]); }
    }
#if !D360_W_FUSED
#undef w
#endif
    double s0[VT];
#pragma unroll
    D360_FORV { s0[v] = w[v] * y2[v]; e2[v] = fma(-s0[v], y2[v], 1.0); }
#pragma unroll
    D360_FORV sq[v] = fma(s0[v] * e2[v], fma(e2[v], c38, 0.5), s0[v]);  // sqrt(w) = s0 (1 + e/2 + 3e^2/8)
#pragma unroll
    D360_FORV {
        // table slots straight from the sign bytes: a byte permute with sign replication puts
        // (tx < 0) into byte 0 and (tz < 0) into byte 1, one AND keeps bit 4 of each (byte offsets
        // 16 OCT_SX and 16 OCT_SZ), the swap adds 16 OCT_SW
        const unsigned hx = (unsigned)__double2hiint(tx[v]), hz = (unsigned)__double2hiint(tz[v]);
        unsigned ko;
        asm("prmt.b32 %0, %1, %2, 0x44fb;" : "=r"(ko) : "r"(hx), "r"(hz));
        ko &= 16u * OCT_SX + 16u * OCT_SZ;
        if (swap[v]) ko |= 16u * OCT_SW;
        const double2 ut = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(g.uo) + ko);
        const unsigned kv = (unsigned)(__double2hiint(ty[v]) >> 31) & 16u;  // 16: ty < 0 (sphi > 0)
        const double2 vt = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(g.vo) + kv);
        pv[v] = (float)fma(q[v] * sq[v], vt.x, vt.y);
        pu[v] = (float)fma(fabs(r[v]) * p[v], ut.x, ut.y);
    }
}

// Stage B of one sample: the f64 bilinear taps of K:134-153 at the f32 (u, v) and the NCC sums.
//
// The planes are padded (wrapped columns, replicated rows), so floor(u), floor(u)+1, floor(v),
// floor(v)+1 are all in-plane and the reference's wrap / clamp rules are data, not code; they
// are stored widened to f64 as { value, value(x+1) - value }, so a footprint is two 16-byte
// loads with no conversion and no subtraction (an f32 lerp costs up to 1e-2 relative on the
// cost of low-texture patches, measured).  floor by the 1.5 * 2^23 magic add; the element index
// is formed in f32 (exact below 2^23) and read out of the mantissa, so no F2I / I2F conversions
// are issued; all offsets are 32-bit element indices from one base.
template <int VT, int PERIOD = VT, bool BIG = false>
__device__ __forceinline__ void gather_bilinear(const FastGroup& g, const double2* __restrict__ nb,
                                                unsigned plane_stride, const float (&pu)[VT], const float (&pv)[VT],
                                                double (&val)[VT]) {
    // floor by a round-down add of a magic constant: (x + M) rounded towards -inf is floor(x) + M for
    // an integer M in [2^23, 2^24) (ulp 1).  For u the constant is idx_bias = 2^23 + pad_y * pitch +
    // pad_x, so the biased floor is already the low part of the texel index.
    const float MAGIC = 12582912.0f;  // 1.5 * 2^23
    float fl_u[VT], fl_v[VT], bu[VT], bv[VT];
#pragma unroll
    D360_FORV {
        bu[v] = __fadd_rd(pu[v], g.idx_bias);
        fl_u[v] = __fadd_rn(bu[v], -g.idx_bias);
        bv[v] = __fadd_rd(pv[v], MAGIC);
        fl_v[v] = __fadd_rn(bv[v], -MAGIC);
    }
    unsigned idx[VT];
#pragma unroll
    D360_FORV {
        if constexpr (BIG) {
            // 2^23 texels or more per plane: row * pitch + column no longer fits f32 arithmetic, so the two biased
            // floors are read out of their mantissas separately (column + pad_x; row + 2^22) and combined by one IMAD
            const unsigned iu = (unsigned)__float_as_int(bu[v]) & 0x7fffffu;
            const unsigned iv = (unsigned)__float_as_int(bv[v]) & 0x7fffffu;
            idx[v] = min(iv * (unsigned)g.pitch + iu + g.big_const, g.max_idx);
        } else {
            const float off = fmaf(fl_v[v], g.pitch_f, bu[v]);  // exact: < 2^24
            idx[v] = min((unsigned)__float_as_int(off) & 0x7fffffu, g.max_idx);
        }
    }
    double2 r0[VT], r1[VT];  // { value, value(x+1) - value }
#pragma unroll
    D360_FORV {
        // 32-bit element indices from one base (all planes together hold < 2^32 texels): one integer
        // add and one IMAD.WIDE per load; 64-bit per-view bases cost four instructions per load
        const unsigned i0 = idx[v] + (unsigned)(v % PERIOD) * plane_stride;
        r0[v] = __ldg(nb + i0);
        r1[v] = __ldg(nb + (i0 + (unsigned)g.pitch));
    }
#pragma unroll
    D360_FORV {
        const double fu = (double)(pu[v] - fl_u[v]), fv = (double)(pv[v] - fl_v[v]);
        const double top = fma(r0[v].y, fu, r0[v].x);
        const double bot = fma(r1[v].y, fu, r1[v].x);
        val[v] = fma(bot - top, fv, top);
    }
}

template <int NV>
__device__ __forceinline__ double aggregate(double (&cv)[NV], int top_k) {
#pragma unroll
    for (int i = 1; i < NV; ++i) {
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
    for (int i = 0; i < NV; ++i)
        if (i < top_k) total = __dadd_rn(total, cv[i]);
    return __dmul_rn(1.0 / top_k, total);
}

// NCC sums (K:240-276) of one hypothesis over the views V0 .. V0 + NV - 1 at the pixel whose
// window entry is `ce`.  `bad` is set when a sample is poisoned (K:242); it does not depend on
// the views.  One flat loop over the S = ns * ns samples (dy outer, dx inner, E:60-65), SPT
// samples per trip: consecutive samples are staged side by side, which gives ptxas SPT * NV
// independent projection chains to interleave (measured at V = 4 against one sample per trip:
// -4 % on refine_pass with its three first-pass views, -12 % on its single-view second pass,
// -2 % on red_black_pass).  The sums take the samples in reference order.
template <class C, typename HT, int V0, int NV, int SPT>
__device__ __forceinline__ void accumulate_views_multi(const FastGroup& g, const Tile& t, int ce, double num, HT nx,
                                                       HT ny, HT nz, bool& bad, double (&s0)[NV], double (&ss0)[NV],
                                                       double (&rs0)[NV], int vbase = 0) {
    // vbase: run-time view offset added to V0 (only the sparse-tile path of red_black_pass, where
    // the lanes of a warp work on different views, passes anything but 0)
#pragma unroll
    for (int v = 0; v < NV; ++v) s0[v] = ss0[v] = rs0[v] = 0.0;
    const double2* __restrict__ nb = reinterpret_cast<const double2*>(g.nb64) + (size_t)(V0 + vbase) * g.plane32;
    double rel[NV][3];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int c = 0; c < 3; ++c) rel[v][c] = g.rel_t[V0 + vbase + v][c];
    // plane depth along the sample's ray (K:241-247): lam, the reference luma, and whether the sample is
    // poisoned (K:242; the caller ORs it into `bad` when it consumes the sample)
    auto plane_depth = [&](int es, double& lam, float& rv, bool& par) {
        const float4 q = t.qg[es];
        double dn;
        if constexpr (sizeof(HT) == 4) {
            const float den = dot3_f32(nx, ny, nz, q.x, q.y, q.z);
            par = den > g.den_lim;
            dn = (double)fminf(den, g.den_lim);
        } else {
            const double den = fma(nz, (double)q.z, fma(ny, (double)q.y, nx * (double)q.x));
            par = den > g.neg_par_eps;
            dn = par ? g.neg_par_eps : den;
        }
        lam = num * rcp3(dn);
        rv = q.w;
    };
    // 3/8 of the third-order rsqrt steps: fma(e, 3/8, 1/2) has two literal operands, one of which has to
    // sit in a register pair; an opaque move keeps it there for the whole loop instead of two moves per use
    double c38;
#if D360_PIN_C38
    asm volatile("mov.f64 %0, %1;" : "=d"(c38) : "d"(g.c0375));
#else
    c38 = g.c0375;
#endif
    const int ns = C::ns(g);
    const int half = (ns - 1) / 2;
    const int n_samples = ns * ns;
    const int row_wrap = t.sy - ns * t.sx;
    // views come in (even, odd) pairs that share a z load; a lone view may start anywhere
    static_assert(NV == 1 || (V0 & 1) == 0, "multi-view passes start at an even view");
    const double2* rxy0 = t.rxy + (V0 + vbase) * t.ne;
    const double* rz0 = reinterpret_cast<const double*>(t.rz + ((V0 + vbase) >> 1) * t.ne) + ((V0 + vbase) & 1);
    auto load_t = [&](int es, double lam, double* tx, double* ty, double* tz) {
#pragma unroll
        for (int v = 0; v < NV; v += 2) {
            if (v + 1 < NV) {
                const double2 z = *reinterpret_cast<const double2*>(rz0 + 2 * ((v >> 1) * t.ne + es));
                tz[v] = fma(lam, z.x, rel[v][2]);
                tz[v + 1] = fma(lam, z.y, rel[v + 1][2]);
            } else {
                tz[v] = fma(lam, rz0[2 * ((v >> 1) * t.ne + es)], rel[v][2]);
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const double2 xy = rxy0[v * t.ne + es];
            tx[v] = fma(lam, xy.x, rel[v][0]);
            ty[v] = fma(lam, xy.y, rel[v][1]);
        }
    };
    int e = ce - half * (t.sx + t.sy), col = 0;
    auto next_entry = [&](int cur) {
        int nxt = cur + t.sx;
        if (++col == ns) { col = 0; nxt += row_wrap; }
        return nxt;
    };
    // The plane-depth chain of a sample (ray load, dot product, reciprocal: a dozen dependent steps with
    // only SPT-way parallelism) is computed one trip ahead, so that it overlaps the projection and
    // gather of the samples before it instead of heading every trip.  The last trip prefetches past
    // the patch: entries inside the CTA's shared memory, values never used.
    int es[SPT];
    double lam[SPT];
    float rvf[SPT];
    bool par[SPT];
#pragma unroll
    for (int j = 0; j < SPT; ++j) {
        es[j] = e;
        e = next_entry(e);
        plane_depth(es[j], lam[j], rvf[j], par[j]);
    }
    int k = 0;
#pragma unroll 1
    for (; k + SPT <= n_samples; k += SPT) {
        double rv[SPT], tx[SPT * NV], ty[SPT * NV], tz[SPT * NV], val[SPT * NV];
        float pu[SPT * NV], pv[SPT * NV];
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            load_t(es[j], lam[j], tx + j * NV, ty + j * NV, tz + j * NV);
            rv[j] = (double)rvf[j];
            bad = bad || par[j];
        }
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            es[j] = e;
            e = next_entry(e);
            plane_depth(es[j], lam[j], rvf[j], par[j]);
        }
        project_uv<SPT * NV>(g, c38, tx, ty, tz, pu, pv);
        gather_bilinear<SPT * NV, NV, C::BIG>(g, nb, g.plane32, pu, pv, val);
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                s0[v] += val[j * NV + v];
                ss0[v] = fma(val[j * NV + v], val[j * NV + v], ss0[v]);
                rs0[v] = fma(rv[j], val[j * NV + v], rs0[v]);
            }
        }
    }
    // remainder (S not a multiple of SPT): the prefetched samples, one at a time
#pragma unroll
    for (int j = 0; j < SPT - 1; ++j) {
        if (k + j < n_samples) {
            double tx[NV], ty[NV], tz[NV], val[NV];
            float pu[NV], pv[NV];
            load_t(es[j], lam[j], tx, ty, tz);
            const double rv = (double)rvf[j];
            bad = bad || par[j];
            project_uv<NV>(g, c38, tx, ty, tz, pu, pv);
            gather_bilinear<NV, NV, C::BIG>(g, nb, g.plane32, pu, pv, val);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                s0[v] += val[v];
                ss0[v] = fma(val[v], val[v], ss0[v]);
                rs0[v] = fma(rv, val[v], rs0[v]);
            }
        }
    }
}

#ifndef D360_SPT
#define D360_SPT 2  // samples per trip (3 and 4 were measured: no further gain, more registers)
#endif

// 1/sqrt(x), third-order refinement of the MUFU.RSQ64H seed (2^-20 -> ~2^-60)
__device__ __forceinline__ double rsqrt3(double x, double c0375) {
    const double y = rsqrt_seed(x);
    const double e = fma(-(x * y), y, 1.0);
    return fma(y * e, fma(e, c0375, 0.5), y);
}

// K:277-296 for one view: truncated 1 - NCC from the sums.  FAST: cov / (sr * sqrt(var)) as
// cov * rsqrt(var) / sr with the Newton-refined seeds (~1e-18) instead of IEEE sqrt + div, ~15
// instructions instead of ~70 per view (-1 % on red_black_pass).  refine_pass keeps the IEEE
// form: there the two extra live values push the sample loop into a register spill (+24 %).
template <bool FAST>
__device__ __forceinline__ double view_cost(const FastGroup& g, double s0, double ss0, double rs0, double mr,
                                            double sr) {
    const double trunc = g.trunc, inv_s = g.inv_s;
    const double m0 = s0 * inv_s;
    const double v0 = ss0 * inv_s - m0 * m0;
    if (v0 < D360_VAR_EPS) return trunc;
    const double cov = rs0 * inv_s - mr * m0;
    double c;
    if constexpr (FAST) c = fma(-(cov * rcp3(sr)), rsqrt3(v0, g.c0375), 1.0);  // sr >= SIGMA_EPS here
    else c = 1.0 - cov / (sr * sqrt(v0));
    c = c < 0.0 ? 0.0 : c;
    return c > trunc ? trunc : c;  // NaN (unguarded polar singularities) passes through, see cand_cost
}

// Per-view costs of views V0 .. V0 + NV - 1 into cv[V0 ...].  Up to four views go through one
// pass over the samples; more are split into two passes (each repeats the shared plane-depth
// chain, but keeps its NCC sums and projection chains inside the register budget; V = 6 at
// 3840x1920: -1 % against one six-view pass).
template <class C, typename HT, bool FAST, int V0, int NV, int NCV>
__device__ __forceinline__ void accumulate_costs(const FastGroup& g, const Tile& t, int ce, double num, HT nx, HT ny,
                                                 HT nz, double mr, double sr, bool& bad, double (&cv)[NCV]) {
    if constexpr (NV <= 4) {
        double s0[NV], ss0[NV], rs0[NV];
        accumulate_views_multi<C, HT, V0, NV, D360_SPT>(g, t, ce, num, nx, ny, nz, bad, s0, ss0, rs0);
#pragma unroll
        for (int v = 0; v < NV; ++v) cv[V0 + v] = view_cost<FAST>(g, s0[v], ss0[v], rs0[v], mr, sr);
    } else {
        constexpr int NA = 4;  // an even number of views first: the second pass starts at an even view
        accumulate_costs<C, HT, FAST, V0, NA>(g, t, ce, num, nx, ny, nz, mr, sr, bad, cv);
        if (bad) return;
        accumulate_costs<C, HT, FAST, V0 + NA, NV - NA>(g, t, ce, num, nx, ny, nz, mr, sr, bad, cv);
    }
}

// Cost of one hypothesis at the pixel whose window entry is `ce` (K:201-297).
//
// EARLY (refine_pass): the caller only asks "is the cost below `bound`" (K:600 `ev < c`) and
// discards the value otherwise.  The cost is the mean of the top_k smallest per-view costs and
// every per-view cost is >= 0, so after V - 1 views the mean of { 0, and the top_k - 1 smallest
// of those } is a lower bound; when it is already >= bound the last view cannot change the
// decision and is not evaluated (the bound itself is returned, which the caller rejects).
// Measured on the benchmark sequence: 76-95 % of the refinement candidates, 52-84 % of the warps.
// Otherwise the last view is evaluated in a second pass over the samples and the result is the
// single-pass one bit for bit (per-view sums do not interact).
template <class C, typename HT, bool EARLY = false>
__device__ __forceinline__ double cand_cost(const FastGroup& g, const Tile& t, int ce, double mr, double sr, HT d,
                                            HT nx, HT ny, HT nz, double bound = 0.0, unsigned* cuts = nullptr) {
    constexpr int VT = C::VT;
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
    bool bad = false;
    double cv[VT];
    if constexpr (EARLY && VT >= 2) {
        constexpr int VA = VT - 1;
        {
            accumulate_costs<C, HT, false, 0, VA>(g, t, ce, num, nx, ny, nz, mr, sr, bad, cv);
            if (bad) return trunc;
        }
        {
            double known[VA];
#pragma unroll
            for (int v = 0; v < VA; ++v) known[v] = cv[v];
            // top_k - 1 smallest known costs plus one unknown cost >= 0.  top_k = 2: half the
            // smallest known cost, exact, and fl(a1 + a2) >= it for any two of the costs.  Otherwise
            // the sum is rounded differently from the final one: shave 1e-12 off (any smaller
            // number is still a lower bound).
            double lower = 0.0;
            if (g.top_k >= 2) lower = aggregate<VA>(known, g.top_k - 1) * ((double)(g.top_k - 1) / g.top_k);
            if (g.top_k > 2) lower *= 1.0 - 1e-12;
            if (lower >= bound) {  // false for NaN: falls through to the full evaluation
                if (cuts != nullptr) ++*cuts;
                return lower;
            }
        }
        {
            double s0[1], ss0[1], rs0[1];
            bool bad_again = false;  // same samples as the first pass: nothing new
            accumulate_views_multi<C, HT, VA, 1, D360_SPT>(g, t, ce, num, nx, ny, nz, bad_again, s0, ss0, rs0);
            cv[VA] = view_cost<false>(g, s0[0], ss0[0], rs0[0], mr, sr);
        }
    } else {
        {
            accumulate_costs<C, HT, true, 0, VT>(g, t, ce, num, nx, ny, nz, mr, sr, bad, cv);
            if (bad) return trunc;
        }
    }
    const double total = aggregate<VT>(cv, g.top_k);
    return total == total ? total : trunc;  // NaN only from the unguarded polar singularities
}

// NVL consecutive views (from the run-time view `view0`) of the same evaluation (f32 hypothesis):
// the per-view costs cand_cost would compute for them, bit for bit (a view's sums see the samples
// in the same order whether its chains run next to other views' chains or alone).  `whole` is
// cleared when the evaluation as a whole scores `trunc` (facing / sigma guard, poisoned sample):
// that decision does not depend on the views.
template <class C, int NVL>
__device__ __forceinline__ void cand_views_cost(const FastGroup& g, const Tile& t, int ce, int view0, double mr,
                                                double sr, float d, float nx, float ny, float nz, bool& whole,
                                                double (&cv)[NVL]) {
#pragma unroll
    for (int v = 0; v < NVL; ++v) cv[v] = g.trunc;
    const float4 a = t.qg[ce];
    const float ndota = dot3_f32(nx, ny, nz, a.x, a.y, a.z);
    if ((double)ndota >= -D360_FACING_EPS || sr < D360_SIGMA_EPS) {
        whole = false;
        return;
    }
    const double num = (double)__fmul_rn(d, ndota);
    bool bad = false;
    double s0[NVL], ss0[NVL], rs0[NVL];
    accumulate_views_multi<C, float, 0, NVL, D360_SPT>(g, t, ce, num, nx, ny, nz, bad, s0, ss0, rs0, view0);
    if (bad) whole = false;
#pragma unroll
    for (int v = 0; v < NVL; ++v) cv[v] = view_cost<true>(g, s0[v], ss0[v], rs0[v], mr, sr);
}

// host side, d360_fast.cu
bool make_fast_group(const GroupDev& gd, FastGroup* out);
// Tensor map of gd.ref_ctx with a (tile_w + 2 reach) x (tile_h + 2 reach) entry box; wm->pad = -1
// when the group carries no context plane, its pad is smaller than the reach, or the driver has
// no encoder (the kernels then fill the window with plain loads).
void make_window_map(const GroupDev& gd, int reach, int tile_w, int tile_h, WindowMap* wm);

// Opt a kernel into `smem` bytes of dynamic shared memory.  The attribute is per (kernel, device) and
// only ever has to grow, so it is set when it first has to and remembered (d360_fast.cu), not before
// each of the 13 launches of a map.
bool smem_already_granted(const void* kernel, size_t smem);
void remember_smem_grant(const void* kernel, size_t smem);

template <typename K>
static int prepare(K kernel, size_t smem) {
    const void* key = reinterpret_cast<const void*>(kernel);
    if (smem_already_granted(key, smem)) return 0;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(%zu B smem): %s", smem, cudaGetErrorString(e));
        return 1;
    }
    remember_smem_grant(key, smem);
    return 0;
}

#define D360_FAST_GEO(V, ...)                                                         \
    if (g.ns == 5 && g.stride == 2 && g.big) { using C = Cfg<V, 5, 2, true>; __VA_ARGS__; } \
    else if (g.big) return fast_reject("planes of 2^23 texels or more are covered for the default 5x5 stride-2 patch only"); \
    else if (g.ns == 5 && g.stride == 2) { using C = Cfg<V, 5, 2>; __VA_ARGS__; }     \
    else { using C = Cfg<V, 0, 0>; __VA_ARGS__; }

#define D360_FAST_DISPATCH(V, ...)                                                    \
    switch (V) {                                                                      \
        case 1: D360_FAST_GEO(1, __VA_ARGS__) break;                                  \
        case 2: D360_FAST_GEO(2, __VA_ARGS__) break;                                  \
        case 3: D360_FAST_GEO(3, __VA_ARGS__) break;                                  \
        case 4: D360_FAST_GEO(4, __VA_ARGS__) break;                                  \
        case 5: D360_FAST_GEO(5, __VA_ARGS__) break;                                  \
        case 6: D360_FAST_GEO(6, __VA_ARGS__) break;                                  \
        case 7: D360_FAST_GEO(7, __VA_ARGS__) break;                                  \
        case 8: D360_FAST_GEO(8, __VA_ARGS__) break;                                  \
        default: return fast_reject("view count outside 1..8");                       \
    }

}  // namespace fast
}  // namespace d360
