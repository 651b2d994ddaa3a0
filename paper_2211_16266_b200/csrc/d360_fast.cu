// Host side shared by the throughput kernels (d360_fast_{eval,rb,refine}.cu): the FastGroup
// parameter block.
#include <string.h>

#include <mutex>

#include "d360_fast.cuh"

namespace d360 {
namespace fast {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        (void)cudaGetLastError();
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

namespace {
struct SmemGrant {
    const void* kernel;
    int device;
    size_t bytes;
};
std::mutex g_grant_mutex;
SmemGrant g_grants[256];
int g_n_grants = 0;
}  // namespace

bool smem_already_granted(const void* kernel, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    std::lock_guard<std::mutex> lock(g_grant_mutex);
    for (int i = 0; i < g_n_grants; ++i)
        if (g_grants[i].kernel == kernel && g_grants[i].device == dev) return g_grants[i].bytes >= smem;
    return false;
}

void remember_smem_grant(const void* kernel, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lock(g_grant_mutex);
    for (int i = 0; i < g_n_grants; ++i)
        if (g_grants[i].kernel == kernel && g_grants[i].device == dev) {
            if (g_grants[i].bytes < smem) g_grants[i].bytes = smem;
            return;
        }
    if (g_n_grants < 256) g_grants[g_n_grants++] = SmemGrant{kernel, dev, smem};
}

void make_window_map(const GroupDev& gd, int reach, int tile_w, int tile_h, WindowMap* wm) {
    wm->pad = -1;
    memset(&wm->map, 0, sizeof(wm->map));
    if (gd.ref_ctx == nullptr || gd.ref_ctx_pad < reach) return;
    EncodeTiledFn enc = encode_tiled();
    if (enc == nullptr) return;
    const int p = gd.ref_ctx_pad;
    const cuuint64_t dims[2] = {(cuuint64_t)4 * (gd.W + 2 * p), (cuuint64_t)(gd.H + 2 * p)};
    const cuuint64_t strides[1] = {(cuuint64_t)4 * (gd.W + 2 * p) * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)(4 * (tile_w + 2 * reach)), (cuuint32_t)(tile_h + 2 * reach)};
    const cuuint32_t estr[2] = {1, 1};
    if (box[0] > 256 || box[1] > 256 || (reinterpret_cast<uintptr_t>(gd.ref_ctx) & 15) != 0) return;
    const CUresult rc = enc(&wm->map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gd.ref_ctx), dims, strides,
                            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc == CUDA_SUCCESS) wm->pad = p;
}

static bool no(const char* why) {
    fast_reject(why);
    return false;
}

bool make_fast_group(const GroupDev& gd, FastGroup* out) {
    // regular grid?  S = ns^2, offsets (dx, dy) = stride * (i - half, j - half), dy outer (E:60-65)
    int ns = 1;
    while (ns * ns < gd.S) ++ns;
    if (ns * ns != gd.S || (ns & 1) == 0) return no("the sample pattern is not a square odd grid");
    const int half = (ns - 1) / 2;
    const int stride = ns > 1 ? gd.dx[1] - gd.dx[0] : 1;
    if (stride < 1) return no("the sample pattern is not a regular grid (E:60-65 order)");
    for (int k = 0; k < gd.S; ++k) {
        if (gd.dx[k] != (k % ns - half) * stride || gd.dy[k] != (k / ns - half) * stride)
            return no("the sample pattern is not a regular grid (E:60-65 order)");
    }
    if (gd.nb_pad_x < 1 || gd.nb_pad_y < 1 || gd.nb64 == nullptr)  // needs padded f64 planes
        return no("the group carries no padded f64 {value, dx} neighbour planes (d360_group.nb64, pads >= 1)");
    const long long pitch = gd.W + 2 * gd.nb_pad_x, rows = gd.H + 2 * gd.nb_pad_y;
    // up to 2^23 texels per plane the texel index is formed in f32 (exact); beyond that (3840x1920 is the last size
    // below) row and column are combined in integer arithmetic, Cfg::BIG
    const bool big = pitch * rows >= (1ll << 23);
    if (pitch >= (1ll << 22) || rows >= (1ll << 22)) return no("a neighbour plane side of 2^22 texels or more");
    FastGroup& g = *out;
    g.W = gd.W; g.H = gd.H; g.ns = ns; g.stride = stride; g.reach = half * stride; g.top_k = gd.top_k;
    g.pitch = (int)pitch;
    g.plane = (size_t)(pitch * rows);
    g.max_idx = (unsigned)(pitch * rows - pitch - 2);
    g.pitch_f = (float)pitch;
    g.big = big ? 1 : 0;
    g.idx_bias = big ? 8388608.0f + (float)gd.nb_pad_x : 8388608.0f + (float)(gd.nb_pad_y * pitch + gd.nb_pad_x);
    g.big_const = (unsigned)(((long long)gd.nb_pad_y - (1ll << 22)) * pitch);
    g.rays = gd.rays; g.ref_gray = gd.ref_gray; g.nb64 = gd.nb64;
    for (int v = 0; v < gd.V; ++v) {
        for (int i = 0; i < 9; ++i) g.rel_r[v][i] = gd.rel_r[v][i];
        for (int i = 0; i < 3; ++i) g.rel_t[v][i] = (double)gd.rel_t[v][i];
    }
    const double hw = gd.W * (0.5 / D360_PI), ls = gd.H / D360_PI;
    static const double CA[8] = {-5.021063913876e-03, 2.533170107199e-02, -6.087448223083e-02, 1.000220525649e-01,
                                 -1.404782123164e-01, 1.997402857787e-01, -3.333223261885e-01, 9.999999227776e-01};
    static const double CQ[8] = {-1.223553911532e-03, 6.510368059701e-03, -1.682974898800e-02, 3.068214201158e-02,
                                 -5.008467775423e-02, 8.895977933699e-02, -2.145970563340e-01, 1.570796263346e00};
    // acos polynomial (K:112-122) re-expanded in w = 1 - x: q(1 - w) by repeated synthetic division at
    // x = 1 (Taylor shift) in extended precision, then the sign of the odd powers of (x - 1) = -w
    long double cw[8];  // ascending powers
    for (int i = 0; i < 8; ++i) cw[i] = (long double)CQ[7 - i];
    for (int i = 0; i < 7; ++i)
        for (int j = 6; j >= i; --j) cw[j] += cw[j + 1];
    for (int i = 1; i < 8; i += 2) cw[i] = -cw[i];
#if !D360_W_FUSED
    for (int i = 0; i < 8; ++i) cw[i] = (long double)CQ[7 - i];
#endif
    for (int i = 0; i < 8; ++i) {  // monic, highest degree first, see project_uv
        g.ca[i] = CA[i] / CA[0];
        g.cq[i] = (double)(cw[7 - i] / cw[7]);
    }
    for (int k = 0; k < fast::OCT_SLOTS; ++k) g.uo[k] = make_double2(0.0, 0.0);
    for (int oct = 0; oct < 8; ++oct) {
        const bool swap = oct & 1, xneg = oct & 2, yneg = oct & 4;
        // theta = sy * (cx + sx * (cs + ss * p)), K:96-99 with y = tx, x = tz
        const double ss = swap ? -1.0 : 1.0, cs = swap ? D360_HALF_PI : 0.0;
        const double sx = xneg ? -1.0 : 1.0, cx = xneg ? D360_PI : 0.0;
        const double sy = yneg ? -1.0 : 1.0;
        const int slot = (yneg ? fast::OCT_SX : 0) + (xneg ? fast::OCT_SZ : 0) + (swap ? fast::OCT_SW : 0);
        g.uo[slot] = make_double2(sy * sx * ss * hw * CA[0], (sy * (cx + sx * cs) + D360_PI) * hw - 0.5);
    }
    g.vo[1] = make_double2(ls * (double)cw[7], -0.5);                   // ty < 0: sphi > 0
    g.vo[0] = make_double2(-ls * (double)cw[7], D360_PI * ls - 0.5);    // ty > 0: sphi < 0, acos = pi - p (K:131)
    if ((unsigned long long)(pitch * rows) * (unsigned long long)gd.V >= (1ull << 32))
        return no("the neighbour planes together hold 2^32 texels or more");
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

}  // namespace fast
}  // namespace d360
