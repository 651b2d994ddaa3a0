// Per-keyframe support kernels around PatchMatch: luma, camera rays, random / warped
// initialisation, median and pole masks, geometric-consistency filter, fusion with
// order-preserving stream compaction, and the synthetic box-scene renderer.
//
// These follow the reference's float64 numpy code (E = engine.py, P = pipeline.py,
// G = geometry.py, SY = synth.py) operation by operation; _rn intrinsics keep nvcc from
// contracting a*b+c into FMA where numpy executes two rounded operations.
#include <math.h>

#include "d360_device.cuh"

namespace d360 {

// ---------------------------------------------------------------------------------------
// to_gray, keyframes.py:64-72 (float32 arithmetic, NumPy weak Python scalars)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float luma_of(const uint8_t* __restrict__ img, int channels, size_t i) {
    if (channels == 1) return __fdiv_rn((float)img[i], 255.0f);
    const float r = img[3 * i], g = img[3 * i + 1], b = img[3 * i + 2];
    float acc = __fmul_rn(0.299f, r);
    acc = __fadd_rn(acc, __fmul_rn(0.587f, g));
    acc = __fadd_rn(acc, __fmul_rn(0.114f, b));
    return __fdiv_rn(acc, 255.0f);
}

// Output raster (H + 2 pad_y, W + 2 pad_x): columns wrap, rows replicate (pads may be 0).
__global__ void k_to_gray(const uint8_t* __restrict__ img, int channels, float* __restrict__ gray,
                          double* __restrict__ gray64, int H, int W, int pad_x, int pad_y) {
    const int pw = W + 2 * pad_x, ph = H + 2 * pad_y;
    const int px = blockIdx.x * blockDim.x + threadIdx.x, py = blockIdx.y;
    if (px >= pw || py >= ph) return;
    const int x = pos_mod(px - pad_x, W);
    const int y = min(max(py - pad_y, 0), H - 1);
    const float l = luma_of(img, channels, (size_t)y * W + x);
    if (gray != nullptr) gray[(size_t)py * pw + px] = l;
    if (gray64 != nullptr) {  // { value, value(x+1) - value }
        const float ln = luma_of(img, channels, (size_t)y * W + pos_mod(px + 1 - pad_x, W));
        reinterpret_cast<double2*>(gray64)[(size_t)py * pw + px] = make_double2((double)l, (double)ln - (double)l);
    }
}

// ---------------------------------------------------------------------------------------
// camera_rays, G:117-122 with the row / column tables of G:81-86
// ---------------------------------------------------------------------------------------
__global__ void k_camera_rays(const double* __restrict__ sin_lam, const double* __restrict__ cos_lam,
                              const double* __restrict__ sin_phi, const double* __restrict__ cos_phi,
                              float* rays32, double* rays64, int H, int W) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= W || y >= H) return;
    const double cp = cos_phi[y];
    const double rx = __dmul_rn(cp, sin_lam[x]), ry = -sin_phi[y], rz = __dmul_rn(cp, cos_lam[x]);
    const size_t i = ((size_t)y * W + x) * 3;
    if (rays32) { rays32[i] = (float)rx; rays32[i + 1] = (float)ry; rays32[i + 2] = (float)rz; }
    if (rays64) { rays64[i] = rx; rays64[i + 1] = ry; rays64[i + 2] = rz; }
}

// ---------------------------------------------------------------------------------------
// random_init, E:244-283
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c0), l0 = 0xD2511F53u * c0;
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c2), l1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = h1 ^ c1 ^ k0, n2 = h0 ^ c3 ^ k1;
        c0 = n0; c1 = l1; c2 = n2; c3 = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__device__ __forceinline__ double u01_from32(uint32_t x) { return ((double)x + 0.5) * 2.3283064365386963e-10; }

__global__ void k_random_init(float* depth, float* normal, float* cost, uint8_t* valid,
                              const double* __restrict__ inv_draws, const double* __restrict__ g_draws,
                              uint64_t seed, double inv_lo, double inv_hi,
                              const double* __restrict__ rays64, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (valid[i]) return;  // pass-through of already-filled pixels (E:276-281)
    double inv, gx, gy, gz;
    if (inv_draws != nullptr) {
        inv = inv_draws[i];
        gx = g_draws[3 * i]; gy = g_draws[3 * i + 1]; gz = g_draws[3 * i + 2];
    } else {
        // Philox4x32-10: key = seed, counter = (pixel index, block id)
        uint32_t a[4], b[4];
        const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
        philox4x32_10((uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0u, k0, k1, a);
        philox4x32_10((uint32_t)i, (uint32_t)((uint64_t)i >> 32), 1u, 0u, k0, k1, b);
        const double u = ((double)(((uint64_t)a[0] << 21) ^ (uint64_t)(a[1] >> 11)) + 0.5) *
                         1.1102230246251565e-16;  // 53 random bits -> (0, 1)
        inv = inv_lo + (inv_hi - inv_lo) * u;
        const double r0 = sqrt(-2.0 * log(u01_from32(a[2]))), t0 = 2.0 * D360_PI * u01_from32(a[3]);
        const double r1 = sqrt(-2.0 * log(u01_from32(b[0]))), t1 = 2.0 * D360_PI * u01_from32(b[1]);
        gx = r0 * cos(t0); gy = r0 * sin(t0); gz = r1 * cos(t1);
    }
    double nrm = sqrt(dot3_f64(gx, gy, gz, gx, gy, gz));
    nrm = nrm < 1e-12 ? 1e-12 : nrm;
    gx /= nrm; gy /= nrm; gz /= nrm;
    const double rx = rays64[3 * i], ry = rays64[3 * i + 1], rz = rays64[3 * i + 2];
    double dot = dot3_f64(gx, gy, gz, rx, ry, rz);
    if (dot > 0.0) {  // reflect across the tangent plane (E:270-272)
        const double two_dot = __dmul_rn(2.0, dot);
        gx = __dsub_rn(gx, __dmul_rn(two_dot, rx));
        gy = __dsub_rn(gy, __dmul_rn(two_dot, ry));
        gz = __dsub_rn(gz, __dmul_rn(two_dot, rz));
    }
    dot = dot3_f64(gx, gy, gz, rx, ry, rz);
    if (dot >= -1e-6) { gx = -rx; gy = -ry; gz = -rz; }
    depth[i] = (float)(1.0 / inv);
    normal[3 * i] = (float)gx; normal[3 * i + 1] = (float)gy; normal[3 * i + 2] = (float)gz;
    cost[i] = INFINITY;
}

// d360_group.ref_ctx: (ray, luma) per pixel with `pad` wrapped columns and replicated rows
__global__ void k_build_ref_ctx(const float* __restrict__ rays, const float* __restrict__ gray, float4* __restrict__ ctx,
                                int H, int W, int pad) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    const int PW = W + 2 * pad;
    if (c >= PW) return;
    const int x = pos_mod(c - pad, W), y = min(max(r - pad, 0), H - 1);
    const size_t i = (size_t)y * W + x;
    ctx[(size_t)r * PW + c] = make_float4(rays[3 * i], rays[3 * i + 1], rays[3 * i + 2], gray[i]);
}

__global__ void k_fill_u8(uint8_t* p, uint8_t v, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------------------
// warp_plane_map, E:286-355: scatter with a packed (cost, source index) atomicMin, then a
// gather pass that re-derives the winning hypothesis.
// ---------------------------------------------------------------------------------------
struct Rigid {
    double r[9];
    double t[3];
};

struct WarpHit {
    bool keep;
    long long target;
    double depth, nx, ny, nz;
};

__device__ __forceinline__ WarpHit warp_one(size_t i, const float* depth, const float* normal,
                                            const double* rays64, const Rigid& rel, double dmin,
                                            double dmax, int H, int W) {
    WarpHit hit;
    const double d = depth[i];
    const double nx = normal[3 * i], ny = normal[3 * i + 1], nz = normal[3 * i + 2];
    const double px = __dmul_rn(d, rays64[3 * i]), py = __dmul_rn(d, rays64[3 * i + 1]),
                 pz = __dmul_rn(d, rays64[3 * i + 2]);
    const double* r = rel.r;
    const double cx = __dadd_rn(dot3_f64(px, py, pz, r[0], r[1], r[2]), rel.t[0]);
    const double cy = __dadd_rn(dot3_f64(px, py, pz, r[3], r[4], r[5]), rel.t[1]);
    const double cz = __dadd_rn(dot3_f64(px, py, pz, r[6], r[7], r[8]), rel.t[2]);
    const double mx = dot3_f64(nx, ny, nz, r[0], r[1], r[2]);
    const double my = dot3_f64(nx, ny, nz, r[3], r[4], r[5]);
    const double mz = dot3_f64(nx, ny, nz, r[6], r[7], r[8]);
    const double rr = sqrt(dot3_f64(cx, cy, cz, cx, cy, cz));
    bool keep = rr > 1e-9;
    const double lon = atan2(cx, cz);
    double sphi = -cy / fmax(rr, 1e-15);
    sphi = fmin(fmax(sphi, -1.0), 1.0);
    const double fx = __dsub_rn(__dmul_rn(__dadd_rn(lon, D360_PI), W / (2 * D360_PI)), 0.5);
    const double fy = __dsub_rn(__dmul_rn(__dsub_rn(D360_PI / 2, asin(sphi)), H / D360_PI), 0.5);
    long long tx = (long long)rint(fx) % W;
    tx = tx < 0 ? tx + W : tx;
    long long ty = (long long)rint(fy);
    ty = ty < 0 ? 0 : (ty > H - 1 ? H - 1 : ty);
    const double* tr = rays64 + ((size_t)ty * W + tx) * 3;
    const double num = dot3_f64(cx, cy, cz, mx, my, mz);
    const double den = dot3_f64(tr[0], tr[1], tr[2], mx, my, mz);
    keep = keep && den < -D360_FACING_EPS;
    const double nd = den != 0.0 ? num / den : -1.0;
    keep = keep && nd >= dmin && nd <= dmax;
    hit.keep = keep;
    hit.target = ty * W + tx;
    hit.depth = nd; hit.nx = mx; hit.ny = my; hit.nz = mz;
    return hit;
}

__device__ __forceinline__ uint32_t ordered_bits(float c) {
    const uint32_t b = __float_as_uint(c);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void k_warp_scatter(const float* __restrict__ depth, const float* __restrict__ normal,
                               const float* __restrict__ cost, const uint8_t* __restrict__ valid,
                               const double* __restrict__ rays64, const __grid_constant__ Rigid rel,
                               double dmin, double dmax, unsigned long long* winner, int H, int W) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)H * W) return;
    const float c = cost[i];
    if (!valid[i] || !isfinite(c)) return;
    const WarpHit hit = warp_one(i, depth, normal, rays64, rel, dmin, dmax, H, W);
    if (!hit.keep) return;
    // smallest cost wins; ties -> earliest source in scan order (E:342-348)
    const unsigned long long key = ((unsigned long long)ordered_bits(c) << 32) | (unsigned long long)i;
    atomicMin(winner + hit.target, key);
}

__global__ void k_warp_gather(const float* __restrict__ depth, const float* __restrict__ normal,
                              const float* __restrict__ cost, const double* __restrict__ rays64,
                              const __grid_constant__ Rigid rel, double dmin, double dmax,
                              const unsigned long long* __restrict__ winner, float* out_depth,
                              float* out_normal, float* out_cost, uint8_t* out_valid, int H, int W) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (size_t)H * W) return;
    const unsigned long long key = winner[t];
    if (key == ~0ull) {  // PlaneMap.empty (E:86-95)
        out_depth[t] = 0.0f;
        out_normal[3 * t] = 0.0f; out_normal[3 * t + 1] = 0.0f; out_normal[3 * t + 2] = 0.0f;
        out_cost[t] = INFINITY;
        out_valid[t] = 0;
        return;
    }
    const size_t src = (size_t)(key & 0xffffffffull);
    const WarpHit hit = warp_one(src, depth, normal, rays64, rel, dmin, dmax, H, W);
    out_depth[t] = (float)hit.depth;
    out_normal[3 * t] = (float)hit.nx; out_normal[3 * t + 1] = (float)hit.ny; out_normal[3 * t + 2] = (float)hit.nz;
    out_cost[t] = cost[src];
    out_valid[t] = 1;
}

// ---------------------------------------------------------------------------------------
// median_support_mask, K:613-647.  Tile + halo in shared memory (NaN = not a sample),
// median by rank counting (no sort, no dynamic register indexing).
// ---------------------------------------------------------------------------------------
constexpr int MED_TW = 32, MED_TH = 8;

__global__ void __launch_bounds__(MED_TW* MED_TH)
    k_median(const float* __restrict__ depth, const uint8_t* __restrict__ valid, int half,
             double rel_threshold, uint8_t* __restrict__ out_valid, int H, int W) {
    extern __shared__ float tile[];
    const int ww = MED_TW + 2 * half, hh = MED_TH + 2 * half;
    const int x0 = blockIdx.x * MED_TW, y0 = blockIdx.y * MED_TH;
    for (int e = threadIdx.x; e < ww * hh; e += blockDim.x) {
        const int j = e / ww, i = e - j * ww;
        const int gy = y0 - half + j;
        float v = __int_as_float(0x7fc00000);
        if (gy >= 0 && gy < H) {  // rows outside the raster are skipped (K:631)
            const int gx = pos_mod(x0 - half + i, W);  // columns wrap (K:635-638)
            const size_t gi = (size_t)gy * W + gx;
            if (valid[gi]) v = depth[gi];
        }
        tile[e] = v;
    }
    __syncthreads();
    const int lx = threadIdx.x % MED_TW, ly = threadIdx.x / MED_TW;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= W || y >= H) return;
    const size_t gi = (size_t)y * W + x;
    if (!valid[gi]) { out_valid[gi] = 0; return; }
    const int win = 2 * half + 1;
    // a window wider than the image would revisit columns; the reference does the same
    int n = 0;
    float v_hi = 0.0f, v_lo = 0.0f;
    if (half == 2) {
        // the default 5x5 window: 25 values in registers (invalid -> +inf, sorted last), odd-even
        // transposition network, then the two middle ranks of the n valid ones picked by position
        float w[25];
        const float inf = __int_as_float(0x7f800000);
#pragma unroll
        for (int j = 0; j < 5; ++j)
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const float v = tile[(ly + j) * ww + lx + i];
                const bool ok = !isnan(v);
                n += ok;
                w[j * 5 + i] = ok ? v : inf;
            }
#pragma unroll
        for (int round = 0; round < 25; ++round)
#pragma unroll
            for (int a = round & 1; a + 1 < 25; a += 2) {
                const float lo = fminf(w[a], w[a + 1]), hi = fmaxf(w[a], w[a + 1]);
                w[a] = lo;
                w[a + 1] = hi;
            }
        const int k_hi = n / 2, k_lo = (n % 2 == 1) ? n / 2 : n / 2 - 1;
#pragma unroll
        for (int a = 0; a < 25; ++a) {
            v_hi = a == k_hi ? w[a] : v_hi;
            v_lo = a == k_lo ? w[a] : v_lo;
        }
    } else {
        for (int j = 0; j < win; ++j)
            for (int i = 0; i < win; ++i) n += !isnan(tile[(ly + j) * ww + lx + i]);
        const int k_hi = n / 2, k_lo = (n % 2 == 1) ? n / 2 : n / 2 - 1;
        for (int j = 0; j < win; ++j)
            for (int i = 0; i < win; ++i) {
                const int ei = (ly + j) * ww + lx + i;
                const float vi = tile[ei];
                if (isnan(vi)) continue;
                int rank = 0;  // elements strictly smaller, ties broken by window position
                for (int jj = 0; jj < win; ++jj)
                    for (int ii = 0; ii < win; ++ii) {
                        const int ej = (ly + jj) * ww + lx + ii;
                        const float vj = tile[ej];
                        rank += (vj < vi) || (vj == vi && ej < ei);
                    }
                if (rank == k_hi) v_hi = vi;
                if (rank == k_lo) v_lo = vi;
            }
    }
    const double med = (n % 2 == 1) ? (double)v_hi : 0.5 * (double)__fadd_rn(v_lo, v_hi);
    out_valid[gi] = fabs((double)depth[gi] - med) <= rel_threshold * med;
}

// ---------------------------------------------------------------------------------------
// pole mask, P:48 / P:214 / P:236 with G:125-128
// ---------------------------------------------------------------------------------------
__global__ void k_pole_mask(uint8_t* valid, double limit_deg, int H, int W) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= W || y >= H) return;
    const double ys = (double)y + 0.5;
    const double lat = __dsub_rn(D360_PI / 2.0, __dmul_rn(D360_PI, ys / H));
    const double deg = __dmul_rn(lat, 180.0 / D360_PI);
    if (fabs(deg) > limit_deg) valid[(size_t)y * W + x] = 0;
}

// ---------------------------------------------------------------------------------------
// consistency_filter and fusion share lift / project
// ---------------------------------------------------------------------------------------
struct Frames {
    const float* depth[D360_MAX_FRAMES];
    const uint8_t* valid[D360_MAX_FRAMES];
    double rot[D360_MAX_FRAMES][9];
    double trans[D360_MAX_FRAMES][3];
    int n;
};

__device__ __forceinline__ void lift_point(const double* rays64, size_t i, double depth, const Rigid& pose,
                                           double& wx, double& wy, double& wz) {
    const double px = __dmul_rn(depth, rays64[3 * i]), py = __dmul_rn(depth, rays64[3 * i + 1]),
                 pz = __dmul_rn(depth, rays64[3 * i + 2]);
    const double* r = pose.r;
    wx = __dadd_rn(dot3_f64(px, py, pz, r[0], r[1], r[2]), pose.t[0]);
    wy = __dadd_rn(dot3_f64(px, py, pz, r[3], r[4], r[5]), pose.t[1]);
    wz = __dadd_rn(dot3_f64(px, py, pz, r[6], r[7], r[8]), pose.t[2]);
}

__device__ __forceinline__ void project_point(const double* rot, const double* trans, double wx, double wy,
                                              double wz, int H, int W, double& u, double& v, double& r) {
    const double dx = __dsub_rn(wx, trans[0]), dy = __dsub_rn(wy, trans[1]), dz = __dsub_rn(wz, trans[2]);
    const double lx = dot3_f64(dx, dy, dz, rot[0], rot[3], rot[6]);
    const double ly = dot3_f64(dx, dy, dz, rot[1], rot[4], rot[7]);
    const double lz = dot3_f64(dx, dy, dz, rot[2], rot[5], rot[8]);
    const double rr = sqrt(dot3_f64(lx, ly, lz, lx, ly, lz));
    double lon = atan2(lx, lz);
    if (lon >= D360_PI) lon -= 2.0 * D360_PI;
    u = __dsub_rn(__dmul_rn(__dadd_rn(lon, D360_PI), W / (2.0 * D360_PI)), 0.5);
    double s = -ly / fmax(rr, 1e-300);
    s = fmin(fmax(s, -1.0), 1.0);
    v = __dsub_rn(__dmul_rn(acos(s), H / D360_PI), 0.5);
    r = rr;
}

__global__ void k_consistency(const float* __restrict__ depth, const uint8_t* __restrict__ valid,
                              const __grid_constant__ Rigid pose, const __grid_constant__ Frames win,
                              const double* __restrict__ rays64, int min_support, double rel_tol,
                              uint8_t* __restrict__ out_valid, int H, int W) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)H * W) return;
    if (!valid[i]) { out_valid[i] = 0; return; }
    double wx, wy, wz;
    lift_point(rays64, i, (double)depth[i], pose, wx, wy, wz);
    int support = 0;
    for (int f = 0; f < win.n; ++f) {
        double u, v, r;
        project_point(win.rot[f], win.trans[f], wx, wy, wz, H, W, u, v, r);
        long long px = (long long)rint(u) % W;
        px = px < 0 ? px + W : px;
        long long py = (long long)rint(v);
        py = py < 0 ? 0 : (py > H - 1 ? H - 1 : py);
        const size_t t = (size_t)py * W + px;
        const double stored = win.depth[f][t];
        support += win.valid[f][t] && (fabs(__dsub_rn(r, stored)) <= __dmul_rn(rel_tol, fabs(stored)));
    }
    out_valid[i] = support >= min_support;
}

constexpr int FUSE_BLOCK = 256;

__global__ void __launch_bounds__(FUSE_BLOCK)
    k_fuse_mark(const float* __restrict__ depth, const uint8_t* __restrict__ valid,
                const __grid_constant__ Rigid pose, const __grid_constant__ Frames newer,
                const double* __restrict__ rays64, double reproj_px, double rel_tol,
                uint8_t* __restrict__ keep, uint32_t* __restrict__ block_counts, int H, int W) {
    const size_t i = (size_t)blockIdx.x * FUSE_BLOCK + threadIdx.x;
    bool k = false;
    if (i < (size_t)H * W && valid[i]) {
        double wx, wy, wz;
        lift_point(rays64, i, (double)depth[i], pose, wx, wy, wz);
        bool duplicate = false;
        const double rad2 = __dmul_rn(reproj_px, reproj_px);
        for (int f = 0; f < newer.n && !duplicate; ++f) {
            double u, v, r;
            project_point(newer.rot[f], newer.trans[f], wx, wy, wz, H, W, u, v, r);
            const long long bx = (long long)rint(u), by = (long long)rint(v);
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const long long px = bx + dx, py = by + dy;
                    const double ddx = __dsub_rn((double)px, u), ddy = __dsub_rn((double)py, v);
                    const double dist2 = __dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy));
                    const bool inside = py >= 0 && py < H && dist2 <= rad2;
                    long long pxm = px % W;
                    pxm = pxm < 0 ? pxm + W : pxm;
                    const long long pyc = py < 0 ? 0 : (py > H - 1 ? H - 1 : py);
                    const size_t t = (size_t)pyc * W + pxm;
                    const double stored = newer.depth[f][t];
                    duplicate = duplicate || (inside && newer.valid[f][t] &&
                                              fabs(__dsub_rn(r, stored)) <= __dmul_rn(rel_tol, fabs(stored)));
                }
        }
        k = !duplicate;
    }
    if (i < (size_t)H * W) keep[i] = k;
    const int cnt = __syncthreads_count(k);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = (uint32_t)cnt;
}

// Exclusive scan of block_counts[0..n) in place by one CTA; total lands in [n].
__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* counts, int n) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < n ? counts[i] : 0u;
        uint32_t s = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
            if ((threadIdx.x & 31) >= o) s += t;
        }
        if ((threadIdx.x & 31) == 31) warp_sums[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t w = warp_sums[threadIdx.x];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += t;
            }
            warp_sums[threadIdx.x] = w;
        }
        __syncthreads();
        const uint32_t warp_off = (threadIdx.x >> 5) ? warp_sums[(threadIdx.x >> 5) - 1] : 0u;
        const uint32_t incl = s + warp_off + carry;
        if (i < n) counts[i] = incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[n] = carry;
}

__global__ void __launch_bounds__(FUSE_BLOCK)
    k_fuse_emit(const float* __restrict__ depth, const uint8_t* __restrict__ keep,
                const __grid_constant__ Rigid pose, const uint8_t* __restrict__ image_rgb,
                const double* __restrict__ rays64, const uint32_t* __restrict__ block_offsets,
                double* __restrict__ points, uint8_t* __restrict__ colors, int H, int W) {
    __shared__ uint32_t warp_cnt[FUSE_BLOCK / 32];
    const size_t i = (size_t)blockIdx.x * FUSE_BLOCK + threadIdx.x;
    const bool k = i < (size_t)H * W && keep[i];
    const unsigned ballot = __ballot_sync(0xffffffffu, k);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_cnt[warp] = __popc(ballot);
    __syncthreads();
    if (!k) return;
    uint32_t off = block_offsets[blockIdx.x];
    for (int w = 0; w < warp; ++w) off += warp_cnt[w];
    off += __popc(ballot & ((1u << lane) - 1u));
    double wx, wy, wz;
    lift_point(rays64, i, (double)depth[i], pose, wx, wy, wz);
    points[3 * (size_t)off] = wx; points[3 * (size_t)off + 1] = wy; points[3 * (size_t)off + 2] = wz;
    colors[3 * (size_t)off] = image_rgb[3 * i];
    colors[3 * (size_t)off + 1] = image_rgb[3 * i + 1];
    colors[3 * (size_t)off + 2] = image_rgb[3 * i + 2];
}

// ---------------------------------------------------------------------------------------
// Synthetic box / corridor renderer, SY:66-84 (cast), SY:101-151 (value noise), SY:154-169
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t h) {
    h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
    h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
    return h ^ (h >> 31);
}

__device__ __forceinline__ double lattice_value(long long ix, long long iy, long long iz, uint64_t salt) {
    const uint64_t h = (uint64_t)ix * 0x9E3779B97F4A7C15ull + (uint64_t)iy * 0xC2B2AE3D27D4EB4Full +
                       (uint64_t)iz * 0x165667B19E3779F9ull + salt;
    return (double)(mix64(h) >> 11) * 1.1102230246251565e-16;
}

__device__ double value_noise(double px, double py, double pz, double scale, int seed, int octaves) {
    double out = 0.0, amp_total = 0.0, amp = 1.0, freq = 1.0 / scale;
    for (int o = 0; o < octaves; ++o) {
        const double qx = __dmul_rn(px, freq), qy = __dmul_rn(py, freq), qz = __dmul_rn(pz, freq);
        const double q0x = floor(qx), q0y = floor(qy), q0z = floor(qz);
        double fx = __dsub_rn(qx, q0x), fy = __dsub_rn(qy, q0y), fz = __dsub_rn(qz, q0z);
        fx = __dmul_rn(__dmul_rn(fx, fx), __dsub_rn(3.0, __dmul_rn(2.0, fx)));
        fy = __dmul_rn(__dmul_rn(fy, fy), __dsub_rn(3.0, __dmul_rn(2.0, fy)));
        fz = __dmul_rn(__dmul_rn(fz, fz), __dsub_rn(3.0, __dmul_rn(2.0, fz)));
        const long long ix = (long long)q0x, iy = (long long)q0y, iz = (long long)q0z;
        const uint64_t salt = (uint64_t)(long long)(seed + o) * 0x27D4EB2F165667C5ull;
        double acc = 0.0;
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy) {
                const double wz = dz ? fz : __dsub_rn(1.0, fz);
                const double wy = dy ? fy : __dsub_rn(1.0, fy);
                for (int dx = 0; dx < 2; ++dx) {
                    const double wx = dx ? fx : __dsub_rn(1.0, fx);
                    const double v = lattice_value(ix + dx, iy + dy, iz + dz, salt);
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(wx, wy), wz), v));
                }
            }
        out = __dadd_rn(out, __dmul_rn(amp, acc));
        amp_total = __dadd_rn(amp_total, amp);
        amp = __dmul_rn(amp, 0.6);
        freq = __dmul_rn(freq, 2.0);
    }
    out = out / amp_total;
    const double s = __dadd_rn(0.5, __dmul_rn(__dsub_rn(out, 0.5), 2.4));
    return fmin(fmax(s, 0.0), 1.0);
}

struct SceneDev {
    double half[3];
    int texture_seed, octaves;
    double noise_scale;
    int kind;             // 0: axis-aligned box / corridor (SY:76-84), 1: sphere shell (SY:70-74)
    int checker;          // SY:88-92
    double oo_minus_r2;   // sphere: o @ o - radius^2, evaluated by the caller with numpy like the reference
};

// render_scene, SY:154-169, statement by statement in f64.  Two of the reference's statements are BLAS
// calls whose rounding numpy does not define; they are restated the way the reference's numpy evaluates
// them on the build host (OpenBLAS FMA kernels; checked with exact rational arithmetic, all elements):
//   camera_rays(camera) @ pose.rotation.T   (dgemm, k = 3)  ->  fma(a2, b2, fma(a1, b1, a0 * b0))
//   d @ o                                   (dgemv, n = 3)  ->  fma(a2, b2, fma(a0, b0, a1 * b1))
// With those the images are bit-identical to the reference's under any rotation and for the sphere scene
// (goldens render_64x32.npz); on a host whose BLAS rounds differently the reference itself changes by the
// same last bit.
__global__ void k_render_scene(const __grid_constant__ SceneDev sc, const __grid_constant__ Rigid pose,
                               const double* __restrict__ rays64, uint8_t* __restrict__ image,
                               float* __restrict__ depth, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rx = rays64[3 * i], ry = rays64[3 * i + 1], rz = rays64[3 * i + 2];
    const double* r = pose.r;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = fma(rz, r[3 * a + 2], fma(ry, r[3 * a + 1], __dmul_rn(rx, r[3 * a])));
    double t;
    if (sc.kind == 1) {
        const double od = fma(d[2], pose.t[2], fma(d[0], pose.t[0], __dmul_rn(d[1], pose.t[1])));
        const double disc = __dsub_rn(__dmul_rn(od, od), sc.oo_minus_r2);
        t = __dadd_rn(-od, sqrt(fmax(disc, 0.0)));
    } else {
        t = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double bound = d[a] > 0 ? sc.half[a] : -sc.half[a];
            const double ta = d[a] != 0.0 ? __dsub_rn(bound, pose.t[a]) / d[a] : INFINITY;
            t = fmin(t, ta > 0 ? ta : INFINITY);
        }
    }
    const double px = __dadd_rn(pose.t[0], __dmul_rn(t, d[0]));
    const double py = __dadd_rn(pose.t[1], __dmul_rn(t, d[1]));
    const double pz = __dadd_rn(pose.t[2], __dmul_rn(t, d[2]));
    if (sc.checker) {
        const long long cells = (long long)floor(px / sc.noise_scale) + (long long)floor(py / sc.noise_scale) +
                                (long long)floor(pz / sc.noise_scale);
        const uint8_t v = (cells & 1) == 0 ? 40 : 215;
        image[3 * i] = image[3 * i + 1] = image[3 * i + 2] = v;
    } else {
#pragma unroll 1
        for (int c = 0; c < 3; ++c) {
            const double v = value_noise(px, py, pz, sc.noise_scale, sc.texture_seed + 101 * c, sc.octaves);
            const double s = fmin(fmax(__dmul_rn(v, 255.0), 0.0), 255.0);
            image[3 * i + c] = (uint8_t)s;  // astype(uint8) truncates
        }
    }
    depth[i] = (float)t;
}

static inline unsigned blocks_for(size_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

static void fill_rigid(Rigid* r, const double* rot, const double* trans) {
    for (int i = 0; i < 9; ++i) r->r[i] = rot[i];
    for (int i = 0; i < 3; ++i) r->t[i] = trans[i];
}

static int fill_frames(Frames* f, const float* const* depth, const uint8_t* const* valid, const double* rot,
                       const double* trans, int n) {
    if (n < 0 || n > D360_MAX_FRAMES) {
        set_error("frame count %d outside [0, %d]", n, D360_MAX_FRAMES);
        return 1;
    }
    f->n = n;
    for (int k = 0; k < n; ++k) {
        f->depth[k] = depth[k];
        f->valid[k] = valid[k];
        for (int i = 0; i < 9; ++i) f->rot[k][i] = rot[9 * k + i];
        for (int i = 0; i < 3; ++i) f->trans[k][i] = trans[3 * k + i];
    }
    return 0;
}

}  // namespace d360

using namespace d360;

extern "C" int d360_to_gray_padded(const uint8_t* image, int channels, float* gray, double* gray64, int height,
                                   int width, int pad_x, int pad_y, void* stream) {
    if (channels != 1 && channels != 3) {
        set_error("expected (H, W) or (H, W, 3) image, got %d channels", channels);
        return 1;
    }
    if (pad_x < 0 || pad_y < 0 || pad_x > width) {
        set_error("to_gray: pads must satisfy 0 <= pad_x <= width, 0 <= pad_y; got (%d, %d)", pad_x, pad_y);
        return 1;
    }
    dim3 grid((width + 2 * pad_x + 255) / 256, height + 2 * pad_y);
    {
        TraceScope ts_("to_gray", (cudaStream_t)stream);
        k_to_gray<<<grid, 256, 0, (cudaStream_t)stream>>>(image, channels, gray, gray64, height, width, pad_x,
                                                          pad_y);
    }
    return check_launch("to_gray");
}

extern "C" int d360_to_gray(const uint8_t* image, int channels, float* gray, int height, int width,
                            void* stream) {
    return d360_to_gray_padded(image, channels, gray, nullptr, height, width, 0, 0, stream);
}

extern "C" int d360_camera_rays(const double* sin_lam, const double* cos_lam, const double* sin_phi,
                                const double* cos_phi, float* rays32, double* rays64, int height,
                                int width, void* stream) {
    dim3 grid((width + 127) / 128, height);
    {
        TraceScope ts_("camera_rays", (cudaStream_t)stream);
        k_camera_rays<<<grid, 128, 0, (cudaStream_t)stream>>>(sin_lam, cos_lam, sin_phi, cos_phi, rays32, rays64,
                                                             height, width);
    }
    return check_launch("camera_rays");
}

extern "C" int d360_random_init(float* depth, float* normal, float* cost, uint8_t* valid,
                                const double* inv_draws, const double* normal_draws, uint64_t seed,
                                double depth_min, double depth_max, const double* rays64, int height,
                                int width, void* stream) {
    if (!(depth_min > 0.0 && depth_max > depth_min)) {
        set_error("patchmatch.depth_range must satisfy 0 < min < max, got [%g, %g]", depth_min, depth_max);
        return 1;
    }
    if ((inv_draws == nullptr) != (normal_draws == nullptr)) {
        set_error("inv_draws and normal_draws must be injected together");
        return 1;
    }
    const size_t n = (size_t)height * width;
    cudaStream_t s = (cudaStream_t)stream;
    {
        TraceScope ts_("random_init", s);
        k_random_init<<<blocks_for(n, 256), 256, 0, s>>>(depth, normal, cost, valid, inv_draws, normal_draws, seed,
                                                        1.0 / depth_max, 1.0 / depth_min, rays64, n);
    }
    if (check_launch("random_init")) return 2;
    {
        TraceScope ts_("fill_u8", s);
        k_fill_u8<<<blocks_for(n, 256), 256, 0, s>>>(valid, 1, n);
    }
    return check_launch("random_init/valid");
}

extern "C" int d360_warp_plane_map(const float* src_depth, const float* src_normal, const float* src_cost,
                                   const uint8_t* src_valid, const double* rays64, const double* r_rel,
                                   const double* t_rel, double depth_min, double depth_max, float* out_depth,
                                   float* out_normal, float* out_cost, uint8_t* out_valid,
                                   unsigned long long* winner, int height, int width, void* stream) {
    if ((size_t)height * width > 0xffffffffull) {
        set_error("raster too large for 32-bit source indices");
        return 1;
    }
    Rigid rel;
    fill_rigid(&rel, r_rel, t_rel);
    const size_t n = (size_t)height * width;
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(winner, 0xff, n * sizeof(unsigned long long), s) != cudaSuccess) {
        set_error("warp_plane_map: memset failed");
        return 2;
    }
    {
        TraceScope ts_("warp_scatter", s);
        k_warp_scatter<<<blocks_for(n, 256), 256, 0, s>>>(src_depth, src_normal, src_cost, src_valid, rays64, rel,
                                                         depth_min, depth_max, winner, height, width);
    }
    if (check_launch("warp_plane_map/scatter")) return 2;
    {
        TraceScope ts_("warp_gather", s);
        k_warp_gather<<<blocks_for(n, 256), 256, 0, s>>>(src_depth, src_normal, src_cost, rays64, rel, depth_min,
                                                        depth_max, winner, out_depth, out_normal, out_cost,
                                                        out_valid, height, width);
    }
    return check_launch("warp_plane_map/gather");
}

extern "C" int d360_median_support_mask(const float* depth, const uint8_t* valid, int half,
                                        double rel_threshold, uint8_t* out_valid, int height, int width,
                                        void* stream) {
    if (half < 1 || half > 16) {
        set_error("median filter window must be odd and >= 3 (half in [1,16]), got half=%d", half);
        return 1;
    }
    const size_t smem = (size_t)(MED_TW + 2 * half) * (MED_TH + 2 * half) * sizeof(float);
    dim3 grid((width + MED_TW - 1) / MED_TW, (height + MED_TH - 1) / MED_TH);
    {
        TraceScope ts_("median", (cudaStream_t)stream);
        k_median<<<grid, MED_TW * MED_TH, smem, (cudaStream_t)stream>>>(depth, valid, half, rel_threshold, out_valid,
                                                                       height, width);
    }
    return check_launch("median_support_mask");
}

extern "C" int d360_build_ref_context(const float* rays, const float* ref_gray, float* ctx, int height, int width,
                                      int pad, void* stream) {
    if (pad < 0 || pad > 64 || height < 1 || width < 1) {
        set_error("build_ref_context: bad size %dx%d pad %d", width, height, pad);
        return 1;
    }
    dim3 grid((width + 2 * pad + 127) / 128, height + 2 * pad);
    {
        TraceScope ts_("build_ref_ctx", (cudaStream_t)stream);
        k_build_ref_ctx<<<grid, 128, 0, (cudaStream_t)stream>>>(rays, ref_gray, reinterpret_cast<float4*>(ctx), height,
                                                                width, pad);
    }
    return check_launch("build_ref_context");
}

extern "C" int d360_pole_mask(uint8_t* valid, double limit_deg, int height, int width, void* stream) {
    dim3 grid((width + 127) / 128, height);
    {
        TraceScope ts_("pole_mask", (cudaStream_t)stream);
        k_pole_mask<<<grid, 128, 0, (cudaStream_t)stream>>>(valid, limit_deg, height, width);
    }
    return check_launch("pole_mask");
}

extern "C" int d360_consistency_filter(const float* depth, const uint8_t* valid, const double* rot,
                                       const double* trans, const float* const* win_depth,
                                       const uint8_t* const* win_valid, const double* win_rot,
                                       const double* win_trans, int n_frames, const double* rays64,
                                       int min_support, double rel_tol, uint8_t* out_valid, int height,
                                       int width, void* stream) {
    Rigid pose;
    fill_rigid(&pose, rot, trans);
    Frames win;
    if (fill_frames(&win, win_depth, win_valid, win_rot, win_trans, n_frames)) return 1;
    const size_t n = (size_t)height * width;
    {
        TraceScope ts_("consistency", (cudaStream_t)stream);
        k_consistency<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(depth, valid, pose, win, rays64,
                                                                           min_support, rel_tol, out_valid, height,
                                                                           width);
    }
    return check_launch("consistency_filter");
}

extern "C" int d360_fuse_blocks(int height, int width) {
    return (int)blocks_for((size_t)height * width, FUSE_BLOCK);
}

extern "C" int d360_fuse_oldest(const float* depth, const uint8_t* valid, const double* rot,
                                const double* trans, const uint8_t* image_rgb,
                                const float* const* newer_depth, const uint8_t* const* newer_valid,
                                const double* newer_rot, const double* newer_trans, int n_newer,
                                const double* rays64, double reproj_px, double rel_tol, uint8_t* keep,
                                uint32_t* block_counts, double* points, uint8_t* colors,
                                int64_t* n_points_host, int height, int width, void* stream) {
    Rigid pose;
    fill_rigid(&pose, rot, trans);
    Frames newer;
    if (fill_frames(&newer, newer_depth, newer_valid, newer_rot, newer_trans, n_newer)) return 1;
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = d360_fuse_blocks(height, width);
    {
        TraceScope ts_("fuse_mark", s);
        k_fuse_mark<<<nb, FUSE_BLOCK, 0, s>>>(depth, valid, pose, newer, rays64, reproj_px, rel_tol, keep,
                                             block_counts, height, width);
    }
    if (check_launch("fuse/mark")) return 2;
    {
        TraceScope ts_("scan_blocks", s);
        k_scan_blocks<<<1, 1024, 0, s>>>(block_counts, nb);
    }
    if (check_launch("fuse/scan")) return 2;
    {
        TraceScope ts_("fuse_emit", s);
        k_fuse_emit<<<nb, FUSE_BLOCK, 0, s>>>(depth, keep, pose, image_rgb, rays64, block_counts, points, colors,
                                             height, width);
    }
    if (check_launch("fuse/emit")) return 2;
    uint32_t total = 0;
    cudaError_t e = cudaMemcpyAsync(&total, block_counts + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error("fuse_oldest: %s", cudaGetErrorString(e));
        return 2;
    }
    *n_points_host = (int64_t)total;
    return 0;
}

extern "C" int d360_render_scene(int kind, int checker, const double* size_xyz, double oo_minus_r2, int texture_seed,
                                 double noise_scale, int octaves, const double* rot, const double* trans,
                                 const double* rays64, uint8_t* image, float* depth, int height, int width,
                                 void* stream) {
    if (kind != 0 && kind != 1) {
        set_error("scene kind %d is neither 0 (box / corridor) nor 1 (sphere)", kind);
        return 1;
    }
    if (octaves < 1 || !(noise_scale > 0.0)) {
        set_error("texture octaves must be >= 1 and noise_scale > 0, got %d, %g", octaves, noise_scale);
        return 1;
    }
    SceneDev sc;
    for (int a = 0; a < 3; ++a) sc.half[a] = size_xyz[a] / 2.0;
    sc.texture_seed = texture_seed;
    sc.octaves = octaves;
    sc.noise_scale = noise_scale;
    sc.kind = kind;
    sc.checker = checker != 0;
    sc.oo_minus_r2 = oo_minus_r2;
    Rigid pose;
    fill_rigid(&pose, rot, trans);
    const size_t n = (size_t)height * width;
    {
        TraceScope ts_("render_scene", (cudaStream_t)stream);
        k_render_scene<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(sc, pose, rays64, image, depth, n);
    }
    return check_launch("render_scene");
}

extern "C" int d360_render_box_scene(const double* size_xyz, int texture_seed, double noise_scale, int octaves,
                                     const double* rot, const double* trans, const double* rays64,
                                     uint8_t* image, float* depth, int height, int width, void* stream) {
    return d360_render_scene(0, 0, size_xyz, 0.0, texture_seed, noise_scale, octaves, rot, trans, rays64, image, depth,
                             height, width, stream);
}
