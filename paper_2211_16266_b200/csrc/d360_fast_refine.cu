// refine_pass, K:476-610 (throughput build; see d360_fast.cuh).  Loop-carried d, n, c are f64 as
// in the reference.
#include "d360_fast.cuh"

namespace d360 {
namespace fast {

// A CTA covers TW x TH_FULL pixels, one thread per pixel.  `flags` (optional, u8 per pixel):
// set to 1 where a candidate was accepted, see d360_fast_rb.cu.
__host__ __device__ inline size_t park_offset(size_t tile) { return (tile + 15) & ~(size_t)15; }

#ifdef D360_REFINE_STATS
// Experiment only (tools/refine_stats.py): how many refinement evaluations a conservative
// approximate filter with sample-value error bound delta could reject.  [0] evaluations,
// [1] accepted, [2] not cut by the V-1 view bound, [3 + i] unresolved at delta_i,
// [8 + k] evaluations of candidate k, [16 + k] accepts of candidate k.
__device__ unsigned long long g_refine_stats[96];
template <class C>
__device__ __forceinline__ void refine_stats(const FastGroup& g, const Tile& t, int ce, double mr, double sr, double d,
                                             double nx, double ny, double nz, double bound, int k) {
    constexpr int VT = C::VT;
    const float4 a = t.qg[ce];
    const double ndota = dot3_f64(nx, ny, nz, (double)a.x, (double)a.y, (double)a.z);
    atomicAdd(&g_refine_stats[0], 1ull);
    atomicAdd(&g_refine_stats[8 + k], 1ull);
    if (ndota >= -D360_FACING_EPS || sr < D360_SIGMA_EPS) return;
    const double num = __dmul_rn(d, ndota);
    bool bad = false;
    double s0[VT], ss0[VT], rs0[VT];
    accumulate_views_multi<C, double, 0, VT, 1>(g, t, ce, num, nx, ny, nz, bad, s0, ss0, rs0);
    if (bad) return;
    double cv[VT], sg[VT];
    for (int v = 0; v < VT; ++v) {
        cv[v] = view_cost<false>(g, s0[v], ss0[v], rs0[v], mr, sr);
        const double m0 = s0[v] * g.inv_s;
        const double v0 = ss0[v] * g.inv_s - m0 * m0;
        sg[v] = v0 > 0 ? sqrt(v0) : 0.0;
    }
    double tmp[VT];
    for (int v = 0; v < VT; ++v) tmp[v] = cv[v];
    const double c = aggregate<VT>(tmp, g.top_k);
    if (c < bound) { atomicAdd(&g_refine_stats[1], 1ull); atomicAdd(&g_refine_stats[16 + k], 1ull); }
    {
        const double edges[8] = {0.01, 0.02, 0.05, 0.1, 0.2, 0.5, 1.0, 10.0};
        int b = 0;
        while (bound >= edges[b]) ++b;
        atomicAdd(&g_refine_stats[64 + b], 1ull);
        double smin = 1e30;
        for (int v = 0; v < VT; ++v) smin = sg[v] < smin ? sg[v] : smin;
        const double se[8] = {1e-3, 2e-3, 5e-3, 1e-2, 2e-2, 5e-2, 1e-1, 10.0};
        b = 0;
        while (smin >= se[b]) ++b;
        atomicAdd(&g_refine_stats[72 + b], 1ull);
    }
    double mn = 1e30;
    for (int v = 0; v < VT - 1; ++v) mn = cv[v] < mn ? cv[v] : mn;
    if (!(0.5 * mn >= bound)) atomicAdd(&g_refine_stats[2], 1ull);
    const double deltas[5] = {0.0, 1e-5, 3e-5, 1e-4, 3e-4};
    for (int i = 0; i < 5; ++i) {
        const double dl = deltas[i];
        double lb[VT];
        for (int v = 0; v < VT; ++v) {
            if (sg[v] > 2 * dl && cv[v] < g.trunc) {
                const double rho = 1.0 - cv[v];
                double l = 1.0 - (rho * sg[v] + dl) / (sg[v] - dl);
                l = l < 0 ? 0 : l;
                lb[v] = l > g.trunc ? g.trunc : l;
            } else lb[v] = cv[v] >= g.trunc && dl == 0.0 ? g.trunc : 0.0;
        }
        const double L = aggregate<VT>(lb, g.top_k);
        if (!(L >= bound)) { atomicAdd(&g_refine_stats[3 + i], 1ull); atomicAdd(&g_refine_stats[32 + k * 5 + i], 1ull); }
    }
}
#endif

template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
    k_refine(const __grid_constant__ FastGroup g, const __grid_constant__ WindowMap wm,
             const __grid_constant__ RefineTable tab, float* __restrict__ depth,
             float* __restrict__ normal, float* __restrict__ cost, unsigned char* __restrict__ flags,
             unsigned long long* n_evals) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * C::TH_FULL;
    const size_t park_at = park_offset(tile_bytes(TW, C::TH_FULL, C::reach(g), false, C::V));
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem + park_at + 5 * sizeof(double) * C::NT);
    const Tile t = wm.pad >= 0 ? tile_setup_tma<C>(g, wm, smem, mbar, x0, y0, C::TH_FULL)
                               : tile_setup<C>(g, smem, x0, y0, C::TH_FULL, false, 0);
    // loop-carried hypothesis (d, n) and cost of each thread, parked here while a candidate is
    // evaluated: ten registers the evaluation's dependency chains can use instead
    double* park = reinterpret_cast<double*>(smem + park_at) + threadIdx.x;
    __syncthreads();
    const int lx = threadIdx.x % TW, ly = threadIdx.x / TW;
    const int x = x0 + lx, y = y0 + ly;
    unsigned int evals = 0, cuts = 0;  // evaluations started; evaluations that stopped before the last view
    if (x < g.W && y < g.H) {
        const int R = C::reach(g);
        const int ce = (ly + R) * t.wwc + lx + R;
        const size_t i = (size_t)y * g.W + x;
        park[0 * C::NT] = depth[i];
        park[1 * C::NT] = normal[3 * i];
        park[2 * C::NT] = normal[3 * i + 1];
        park[3 * C::NT] = normal[3 * i + 2];
        park[4 * C::NT] = cost[i];
        double mr, sr;
        pixel_stats<C>(g, t, ce, mr, sr);
        bool accepted = false;
#pragma unroll 1
        for (int k = 0; k < tab.n; ++k) {
            const double d = park[0 * C::NT], nx = park[1 * C::NT], ny = park[2 * C::NT], nz = park[3 * C::NT];
            double nd = __dadd_rn(d, (double)tab.dd[k]);
            if (nd < tab.depth_min) nd = tab.depth_min;
            else if (nd > tab.depth_max) nd = tab.depth_max;
            // Tangent basis of the current normal (K:540-560).  The reference refreshes it only
            // after an accept; recomputing it from the same (n, a) gives the same values and keeps
            // twelve registers free during the evaluation (-5 % on the pass, measured).
            double e1x, e1y, e1z, e2x, e2y, e2z;
            {
                const float4 a4 = t.qg[ce];
                const double ax = a4.x, ay = a4.y, az = a4.z;
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
            }
            const double sa = tab.sa[k], ca = tab.ca[k], caz = tab.caz[k], saz = tab.saz[k];
            double cnx = __dadd_rn(__dmul_rn(nx, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1x, caz), __dmul_rn(e2x, saz)), sa));
            double cny = __dadd_rn(__dmul_rn(ny, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1y, caz), __dmul_rn(e2y, saz)), sa));
            double cnz = __dadd_rn(__dmul_rn(nz, ca), __dmul_rn(__dadd_rn(__dmul_rn(e1z, caz), __dmul_rn(e2z, saz)), sa));
            const double nrm = sqrt(dot3_f64(cnx, cny, cnz, cnx, cny, cnz));
            if (nrm < 1e-12) continue;
            const double inv = 1.0 / nrm;
            cnx = __dmul_rn(cnx, inv); cny = __dmul_rn(cny, inv); cnz = __dmul_rn(cnz, inv);
#ifdef D360_REFINE_STATS
            refine_stats<C>(g, t, ce, mr, sr, nd, cnx, cny, cnz, park[4 * C::NT], k);
#endif
            const double ev = cand_cost<C, double, true>(g, t, ce, mr, sr, nd, cnx, cny, cnz, park[4 * C::NT], &cuts);
            ++evals;
            if (ev < park[4 * C::NT]) {
                park[0 * C::NT] = nd; park[1 * C::NT] = cnx; park[2 * C::NT] = cny; park[3 * C::NT] = cnz;
                park[4 * C::NT] = ev;
                accepted = true;
            }
        }
        depth[i] = (float)park[0 * C::NT];
        normal[3 * i] = (float)park[1 * C::NT];
        normal[3 * i + 1] = (float)park[2 * C::NT];
        normal[3 * i + 2] = (float)park[3 * C::NT];
        cost[i] = (float)park[4 * C::NT];
        if (flags != nullptr && accepted) flags[i] = 1;
    }
    if (n_evals != nullptr) {
        for (int o = 16; o > 0; o >>= 1) {
            evals += __shfl_xor_sync(0xffffffffu, evals, o);
            cuts += __shfl_xor_sync(0xffffffffu, cuts, o);
        }
        if ((threadIdx.x & 31) == 0 && evals) {
            atomicAdd(n_evals, (unsigned long long)evals);
            if (cuts) atomicAdd(n_evals + 1, (unsigned long long)cuts);
        }
    }
}

}  // namespace fast

using namespace fast;

int fast_refine(const GroupDev& gd, const RefineTable& tab, float* depth, float* normal, float* cost,
                unsigned char* flags, unsigned long long* n_evals, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    D360_FAST_DISPATCH(gd.V, {
        const size_t smem = park_offset(tile_bytes(TW, C::TH_FULL, g.reach, false, gd.V)) + 5 * sizeof(double) * C::NT + 16;
        if (smem > 200 * 1024) return -1;
        dim3 grid((gd.W + TW - 1) / TW, (gd.H + C::TH_FULL - 1) / C::TH_FULL);
        WindowMap wm;
        make_window_map(gd, g.reach, TW, C::TH_FULL, &wm);
        auto k = k_refine<C>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("refine", s);
        k<<<grid, C::NT, smem, s>>>(g, wm, tab, depth, normal, cost, flags, n_evals);
    })
    return check_launch("refine_pass");
}

#ifdef D360_REFINE_STATS
extern "C" int d360_debug_refine_stats(unsigned long long* out, int reset) {
    cudaMemcpyFromSymbol(out, d360::fast::g_refine_stats, sizeof(unsigned long long) * 96);
    if (reset) {
        unsigned long long z[96] = {0};
        cudaMemcpyToSymbol(d360::fast::g_refine_stats, z, sizeof(z));
    }
    return 0;
}
#endif

}  // namespace d360
