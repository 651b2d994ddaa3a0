// refine_pass, K:476-610 (throughput build; see d360_fast.cuh).  Loop-carried d, n, c are f64 as
// in the reference.
#include "d360_fast.cuh"

namespace d360 {
namespace fast {

// A CTA covers TW x TH_FULL pixels, one thread per pixel.  `flags` (optional, u8 per pixel):
// set to 1 where a candidate was accepted, see d360_fast_rb.cu.
__host__ __device__ inline size_t park_offset(size_t tile) { return (tile + 15) & ~(size_t)15; }


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
        if (smem > 200 * 1024) return fast_reject("the patch window of a tile needs more than 200 KB of shared memory");
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

}  // namespace d360
