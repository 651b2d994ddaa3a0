// eval_costs, K:300-349 (throughput build; see d360_fast.cuh).
#include "d360_fast.cuh"

namespace d360 {
namespace fast {

// A CTA covers TW x TH_FULL pixels, one thread per pixel.
template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
    k_eval(const __grid_constant__ FastGroup g, const __grid_constant__ WindowMap wm, const float* __restrict__ depth,
           const float* __restrict__ normal, float* __restrict__ cost_out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * C::TH_FULL;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(
        smem + mbar_offset(tile_bytes(TW, C::TH_FULL, C::reach(g), false, C::V)));
    const Tile t = wm.pad >= 0 ? tile_setup_tma<C>(g, wm, smem, mbar, x0, y0, C::TH_FULL)
                               : tile_setup<C>(g, smem, x0, y0, C::TH_FULL, false, 0);
    __syncthreads();
    const int lx = threadIdx.x % TW, ly = threadIdx.x / TW;
    const int x = x0 + lx, y = y0 + ly;
    if (x >= g.W || y >= g.H) return;
    const int R = C::reach(g);
    const int ce = (ly + R) * t.wwc + lx + R;
    double mr, sr;
    pixel_stats<C>(g, t, ce, mr, sr);
    const size_t i = (size_t)y * g.W + x;
    cost_out[i] = (float)cand_cost<C, float>(g, t, ce, mr, sr, depth[i], normal[3 * i], normal[3 * i + 1],
                                             normal[3 * i + 2]);
}

}  // namespace fast

using namespace fast;

// Returns -1 when the fast path does not apply (caller falls back to the generic kernel).
int fast_eval(const GroupDev& gd, const float* depth, const float* normal, float* cost_out, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    D360_FAST_DISPATCH(gd.V, {
        const size_t smem = mbar_offset(tile_bytes(TW, C::TH_FULL, g.reach, false, gd.V)) + 16;
        if (smem > 200 * 1024) return fast_reject("the patch window of a tile needs more than 200 KB of shared memory");
        dim3 grid((gd.W + TW - 1) / TW, (gd.H + C::TH_FULL - 1) / C::TH_FULL);
        WindowMap wm;
        make_window_map(gd, g.reach, TW, C::TH_FULL, &wm);
        auto k = k_eval<C>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("eval_costs", s);
        k<<<grid, C::NT, smem, s>>>(g, wm, depth, normal, cost_out);
    })
    return check_launch("eval_costs");
}

}  // namespace d360
