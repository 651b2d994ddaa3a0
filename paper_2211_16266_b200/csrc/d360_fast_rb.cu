// red_black_pass, K:352-473 (throughput build; see d360_fast.cuh).
//
// A CTA covers TW x TH_RB pixels, NT of them of the requested colour.  The number of candidates
// a pixel has to evaluate varies (0..8 after the duplicate skipping of K:418-432), so the work
// is levelled through a CTA-wide queue:
//   phase 1  one thread per pixel: in-range, non-duplicate neighbours -> candidate mask;
//            exclusive scan of the counts; (pixel, neighbour) items queued.  The patch window
//            is being loaded meanwhile and is only unpacked if the CTA has any item at all;
//   phase 2  warps pull 32 items at a time and evaluate them (any lane, any pixel of the tile);
//   phase 3  one thread per pixel: strict-< arg-min over its candidates in neighbour order
//            (K:463; the cost of a hypothesis does not depend on evaluation order, so this is
//            the reference's sequential accept).
//
// Memoised candidate costs (optional: `flags_in` / `flags_out`, `memo_valid`, `memo_cost`).  The
// cost of hypothesis h at pixel p is a pure function of (p, h) — p's own hypothesis does not
// enter it — so c_p(h_q) stays what it was for as long as the neighbour q keeps its hypothesis.
// Per pixel the pass keeps the eight costs it last computed (f64, exactly the values phase 2
// produced) and a validity byte; at the next pass it drops the entries of neighbours whose
// "changed" flag is set, evaluates only the in-range, non-duplicate candidates without a valid
// entry, and takes the arg-min over fresh and remembered costs alike.  Duplicates (K:418-432)
// stay excluded exactly as before, so the result is bit-identical to evaluating everything; on a
// warp-initialised sequence 40-45 % of the propagation evaluations of the later iterations are
// remembered ones.
//   flags: 1 = the pixel's hypothesis changed during its own red-black pass or the refinement
//   of the previous iteration.  The first iteration starts from all ones.  A pass writes
//   flags_out for the pixels it updates and refine_pass sets it where it accepts.  All eight
//   neighbours have the pixel's colour, so a pass reads only flags that no pass of the same
//   iteration writes, and only pixel p touches p's memo entries.
#include "d360_fast.cuh"

namespace d360 {
namespace fast {

__constant__ int c_nbr2[8][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1}, {0, -2}, {0, 2}, {-2, 0}, {2, 0}};

template <int NT>
struct RbQueue {
    double2 stats[NT];            // (mr, sr) per pixel
    double costs[NT * 8];         // cost of neighbour j's hypothesis at pixel p
    unsigned short items[NT * 8]; // p * 8 + j
    int warp_totals[NT / 32];
    int total, next;
    unsigned long long mbar;      // TMA completion barrier of the window load
};

// 128-byte aligned: the cost array doubles as the TMA landing area of the uncompressed window
__host__ __device__ inline size_t rb_queue_offset(size_t tile) { return (tile + 127) & ~(size_t)127; }

// Colour-compressed window from one TMA box: the full (TW + 2R) x (TH_RB + 2R) float4 window lands
// in `stage` (the queue's cost array, not needed before phase 2), then every thread copies the
// entries of the pass's colour to their compressed slots and derives R_v q for them.  Issue and
// completion are separate so that the load is in flight during phase 1.
template <class C>
__device__ __forceinline__ void window_tma_issue(const FastGroup& g, const WindowMap& wm, float4* stage,
                                                 unsigned long long* mbar, int x0, int y0) {
    const int R = C::reach(g);
    const int ww = TW + 2 * R, hh = C::TH_RB + 2 * R;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                 "r"((unsigned)(ww * hh * sizeof(float4)))
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(stage)),
        "l"(reinterpret_cast<unsigned long long>(&wm.map)), "r"(4 * (x0 - R + wm.pad)), "r"(y0 - R + wm.pad),
        "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void window_tma_wait(unsigned long long* mbar) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(mbar))
            : "memory");
    }
}

template <class C>
__device__ __forceinline__ Tile window_from_stage(const FastGroup& g, unsigned char* smem, const float4* stage,
                                                  int keep) {
    const int R = C::reach(g);
    const int ww = TW + 2 * R, hh = C::TH_RB + 2 * R;
    const int wwc = ww / 2;
    const int ne = wwc * hh;
    float4* qg = reinterpret_cast<float4*>(smem);
    double2* rxy = reinterpret_cast<double2*>(smem + (size_t)ne * sizeof(float4));
    double2* rz = rxy + (size_t)C::V * ne;
    for (int e = threadIdx.x; e < ne; e += C::NT) {
        const int j = e / wwc, ic = e - j * wwc;
        const int i = 2 * ic + ((keep + j) & 1);
        const float4 q = stage[j * ww + i];
        qg[e] = q;
        store_rq<C>(g, rxy, rz, ne, e, q.x, q.y, q.z);
    }
    Tile t;
    t.qg = qg;
    t.rxy = rxy;
    t.rz = rz;
    t.wwc = wwc;
    t.ne = ne;
    t.sx = C::stride(g) / 2;
    t.sy = C::stride(g) * wwc;
    return t;
}

template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
    k_red_black(const __grid_constant__ FastGroup g, const __grid_constant__ WindowMap wm, int parity_arg,
                const float* __restrict__ depth_in,
                const float* __restrict__ normal_in, const float* __restrict__ cost_in, float* __restrict__ depth_out,
                float* __restrict__ normal_out, float* __restrict__ cost_out,
                const unsigned char* __restrict__ flags_in, unsigned char* __restrict__ flags_out,
                unsigned char* __restrict__ memo_valid, double* __restrict__ memo_cost, unsigned long long* n_evals) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NT = C::NT;
    // parity_arg 2: both colours in one launch, one per grid z-slice.  The eight neighbours of a pixel all
    // have its colour (K:44-56), so the two passes of an iteration read and write disjoint pixels: running
    // them side by side gives what running them one after the other gives, and the off-colour pixels need
    // no carrying over (the other slice writes them).
    const bool both = parity_arg == 2;
    const int parity = both ? (int)blockIdx.z : parity_arg;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * C::TH_RB;  // x0 is even
    const int R = C::reach(g);
    const bool compress = (C::stride(g) & 1) == 0;
    RbQueue<NT>& q = *reinterpret_cast<RbQueue<NT>*>(smem + rb_queue_offset(tile_bytes(TW, C::TH_RB, R, compress, C::V)));
    if (threadIdx.x == 0) q.next = 0;
    // the uncompressed window must fit the landing area (TW + 2R) (TH_RB + 2R) float4 <= NT * 8 doubles
    const bool by_tma = wm.pad >= 0 && compress &&
                        (size_t)(TW + 2 * R) * (C::TH_RB + 2 * R) * sizeof(float4) <= sizeof(q.costs);
    if (by_tma && threadIdx.x == 0) window_tma_issue<C>(g, wm, reinterpret_cast<float4*>(q.costs), &q.mbar, x0, y0);
    __syncthreads();  // queue head and barrier initialised; the window load is in flight during phase 1

    // ---- phase 1
    const int tid = threadIdx.x;
    const int ly = tid / (TW / 2);
    const int y = y0 + ly;
    const int lx = 2 * (tid % (TW / 2)) + ((parity + y) & 1);
    const int x = x0 + lx;
    const bool live = x < g.W && y < g.H;
    if (y < g.H && !both) {
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
    unsigned mask = 0, considered = 0, kept = 0;  // to evaluate now; all candidates of the arg-min; valid memo entries
    if (live) {
        // K:418-432 skips exact duplicates of the best-so-far and of already evaluated
        // candidates.  Every earlier in-range neighbour was either evaluated or itself such a
        // duplicate, so comparing with the pixel's original hypothesis and with the earlier
        // neighbours selects the same set, except that it also skips re-evaluating the original
        // hypothesis once it has been displaced, which strict < would reject anyway.
        //
        // The eight neighbour hypotheses are fetched first, as 40 independent loads, and compared
        // in registers: this phase is pure memory latency and sits in front of every CTA's work
        // (a loop of dependent loads here cost ~0.3 ms per launch, 7 % of a step).
        constexpr int NDX[8] = {-1, 1, -1, 1, 0, 0, -2, 2}, NDY[8] = {-1, -1, 1, 1, -2, 2, 0, 0};
        float hd[8], hx[8], hy[8], hz[8];
        unsigned char changed[8];
        bool in_range[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int qy = y + NDY[j];
            in_range[j] = qy >= 0 && qy < g.H;                                          // K:407 rows skipped
            const size_t qi = in_range[j] ? (size_t)qy * g.W + wrap_once(x + NDX[j], g.W) : i;  // K:410-413 columns wrap
            hd[j] = depth_in[qi];
            hx[j] = normal_in[3 * qi];
            hy[j] = normal_in[3 * qi + 1];
            hz[j] = normal_in[3 * qi + 2];
            changed[j] = flags_in != nullptr ? flags_in[qi] : (unsigned char)1;
        }
        const float od = depth_in[i];
        const float onx = normal_in[3 * i], ony = normal_in[3 * i + 1], onz = normal_in[3 * i + 2];
        unsigned remembered = memo_valid != nullptr && flags_in != nullptr ? memo_valid[i] : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            bool dup = hd[j] == od && hx[j] == onx && hy[j] == ony && hz[j] == onz;
#pragma unroll
            for (int m = 0; m < j; ++m)
                dup = dup || (in_range[m] && hd[m] == hd[j] && hx[m] == hx[j] && hy[m] == hy[j] && hz[m] == hz[j]);
            if (in_range[j] && !dup) considered |= 1u << j;
            if (changed[j]) remembered &= ~(1u << j);
        }
        kept = remembered;
        mask = considered & ~remembered;
    }
    const int n_mine = __popc(mask);
    int incl = n_mine;  // CTA-wide exclusive scan of the counts
    for (int o = 1; o < 32; o <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, incl, o);
        if ((tid & 31) >= o) incl += up;
    }
    if ((tid & 31) == 31) q.warp_totals[tid >> 5] = incl;
    __syncthreads();
    int off = incl - n_mine;
    for (int w = 0; w < (tid >> 5); ++w) off += q.warp_totals[w];
    if (tid == NT - 1) q.total = off + n_mine;
    for (unsigned m = mask; m; m &= m - 1) q.items[off++] = (unsigned short)(tid * 8 + (__ffs(m) - 1));
    __syncthreads();
    const int total = q.total;
    if (by_tma) window_tma_wait(&q.mbar);  // also with nothing to do: never leave with a copy in flight

    // ---- phase 2 (skipped, with the whole patch window, by a CTA that has no candidate left)
    if (total > 0) {
        const Tile t = by_tma ? window_from_stage<C>(g, smem, reinterpret_cast<const float4*>(q.costs), (parity + y0) & 1)
                              : tile_setup<C>(g, smem, x0, y0, C::TH_RB, compress, (parity + y0) & 1);
        __syncthreads();
        if (n_mine) {
            const int ce = (ly + R) * t.wwc + (compress ? (lx + R) >> 1 : lx + R);
            double mr, sr;
            pixel_stats<C>(g, t, ce, mr, sr);
            q.stats[tid] = make_double2(mr, sr);
        }
        __syncthreads();
        // Sparse tile (late iterations: a handful of candidates per CTA): the pass is then bound by
        // the latency of one evaluation per CTA, so an item is spread over 4 lanes (one view each)
        // or 2 lanes (two views each) as far as the CTA's lanes go round.  The per-view costs are
        // the ones the joint evaluation computes, bit for bit, so memoised and fresh costs stay
        // interchangeable.
        int lanes_per_item = 1;
        if constexpr (C::V == 4) lanes_per_item = total <= NT / 4 ? 4 : (total <= NT / 2 ? 2 : 1);
        if (lanes_per_item > 1) {
            if constexpr (C::V == 4) {
                const int slot = lanes_per_item == 4 ? tid >> 2 : tid >> 1;
                const int part = lanes_per_item == 4 ? tid & 3 : tid & 1;
                if (slot < total) {  // uniform within the lane group
                    const int item = q.items[slot];
                    const int p = item >> 3, j = item & 7;
                    const int ply = p / (TW / 2);
                    const int py = y0 + ply;
                    const int plx = 2 * (p % (TW / 2)) + ((parity + py) & 1);
                    const int px = x0 + plx;
                    const size_t qi = (size_t)(py + c_nbr2[j][1]) * g.W + wrap_once(px + c_nbr2[j][0], g.W);
                    const int ce = (ply + R) * t.wwc + (compress ? (plx + R) >> 1 : plx + R);
                    const double2 st = q.stats[p];
                    const float hd0 = depth_in[qi], hx0 = normal_in[3 * qi], hy0 = normal_in[3 * qi + 1],
                                hz0 = normal_in[3 * qi + 2];
                    bool whole = true;
                    double cv[4];
                    if (lanes_per_item == 4) {
                        double mine[1];
                        cand_views_cost<C, 1>(g, t, ce, part, st.x, st.y, hd0, hx0, hy0, hz0, whole, mine);
                        const unsigned group = 0xfu << (tid & 28);
#pragma unroll
                        for (int v = 0; v < 4; ++v) cv[v] = __shfl_sync(group, mine[0], (tid & 28) + v);
                    } else {
                        double mine[2];
                        cand_views_cost<C, 2>(g, t, ce, 2 * part, st.x, st.y, hd0, hx0, hy0, hz0, whole, mine);
                        const unsigned group = 0x3u << (tid & 30);
#pragma unroll
                        for (int v = 0; v < 4; ++v) cv[v] = __shfl_sync(group, mine[v & 1], (tid & 30) + (v >> 1));
                    }
                    if (part == 0) {
                        double c = g.trunc;
                        if (whole) {
                            const double agg = aggregate<4>(cv, g.top_k);
                            c = agg == agg ? agg : g.trunc;
                        }
                        q.costs[item] = c;
                    }
                }
            }
        } else {
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
                    const int ce = (ply + R) * t.wwc + (compress ? (plx + R) >> 1 : plx + R);
                    const double2 st = q.stats[p];
                    q.costs[item] = cand_cost<C, float>(g, t, ce, st.x, st.y, depth_in[qi], normal_in[3 * qi],
                                                        normal_in[3 * qi + 1], normal_in[3 * qi + 2]);
                }
            }
        }
        __syncthreads();
    }

    // ---- phase 3
    if (live) {
        // Remembered costs (computed by an earlier pass for the same (pixel, hypothesis)) are fetched first, as up to
        // eight independent loads: taken one by one inside the arg-min loop they were eight dependent memory
        // latencies per pixel, which is most of what a launch costs once the propagation has gone sparse.
        const unsigned from_memo = considered & ~mask;
        double remembered_cost[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            remembered_cost[j] = (from_memo >> j & 1u) ? __ldcs(memo_cost + 8 * i + j) : 0.0;
        double bc = (double)cost_in[i];
        int bj = -1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (!(considered >> j & 1u)) continue;
            double c;
            if (mask >> j & 1u) {
                c = q.costs[tid * 8 + j];
                if (memo_cost != nullptr) __stcs(memo_cost + 8 * i + j, c);
            } else {
                c = remembered_cost[j];
            }
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
        if (flags_out != nullptr) flags_out[i] = bj >= 0;
        if (memo_valid != nullptr) memo_valid[i] = (unsigned char)(kept | mask);
    }
    if (n_evals != nullptr && tid == 0 && total) atomicAdd(n_evals, (unsigned long long)total);
}

}  // namespace fast

using namespace fast;

int fast_red_black(const GroupDev& gd, int parity, const float* di, const float* ni, const float* ci, float* dout,
                   float* nout, float* cout, const unsigned char* flags_in, unsigned char* flags_out,
                   unsigned char* memo_valid, double* memo_cost, unsigned long long* n_evals, cudaStream_t s) {
    FastGroup g;
    if (!make_fast_group(gd, &g)) return -1;
    D360_FAST_DISPATCH(gd.V, {
        const size_t smem = rb_queue_offset(tile_bytes(TW, C::TH_RB, g.reach, (g.stride & 1) == 0, gd.V)) +
                            sizeof(RbQueue<C::NT>);
        if (smem > 200 * 1024) return fast_reject("the patch window of a tile needs more than 200 KB of shared memory");
        dim3 grid((gd.W + TW - 1) / TW, (gd.H + C::TH_RB - 1) / C::TH_RB, parity == 2 ? 2 : 1);
        WindowMap wm;
        make_window_map(gd, g.reach, TW, C::TH_RB, &wm);
        auto k = k_red_black<C>;
        if (prepare(k, smem)) return 1;
        TraceScope ts_("red_black", s);
        k<<<grid, C::NT, smem, s>>>(g, wm, parity, di, ni, ci, dout, nout, cout, flags_in, flags_out, memo_valid, memo_cost, n_evals);
    })
    return check_launch("red_black_pass");
}

}  // namespace d360
