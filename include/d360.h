/*
 * d360.h — C ABI of the B200-native densify360 hot path (libd360.so).
 *
 * The reference has no FFI: its operator boundary is the Python module
 * densify360.kernels (four numba functions over C-contiguous arrays), called only by
 * densify360.engine, plus two numpy routines in densify360.pipeline.  Every entry point
 * below replaces one of those call targets; "replaces" cites the reference file:line
 * (K = pkg/src/densify360/kernels.py, E = engine.py, P = pipeline.py, G = geometry.py,
 * KF = keyframes.py, SY = synth.py).
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / numpy types.
 *  - pointers documented "device" are CUDA device pointers owned by the caller;
 *    "host" pointers are small parameter blocks read before the call returns.
 *  - `stream` is a cudaStream_t passed as void*; calls are asynchronous on it unless
 *    stated otherwise.  The library allocates nothing persistent.
 *  - return 0 on success, nonzero on error; d360_last_error() describes the failure
 *    (thread-local).  Kernels never "raise": unusable hypotheses score `trunc`
 *    exactly as the reference does (K:32-37).
 *  - images / state use the reference's array layouts: depth (H,W) f32, normal (H,W,3)
 *    f32, cost (H,W) f32, masks (H,W) u8 (numpy bool), rays (H,W,3) f32.
 */
#ifndef D360_H
#define D360_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define D360_MAX_VIEWS 8
#define D360_MAX_SAMPLES 128
#define D360_MAX_REACH 8      /* max |dx|,|dy| of a patch sample offset */
#define D360_MAX_REFINE 16    /* max refinement candidates per pass (reference: 6) */
#define D360_MAX_FRAMES 8     /* max frames in a consistency window / fusion buffer */

/* Arithmetic policy of the cost kernels. */
enum {
    D360_PREC_EXACT = 0, /* literal f64 restatement (IEEE div/sqrt, f64 bilinear + sums) */
    D360_PREC_MIXED = 1, /* f64 projection with DFMA contraction and Newton-refined rcp/rsqrt
                            seeds (~1e-18), f64 bilinear + sums: the throughput policy      */
    D360_PREC_FAST = 2   /* reserved, rejected by every entry point: an all-f32 projection
                            cannot hold the 1e-4 cost parity        */
};

/* One stereo group in kernel layout == densify360.engine.PreparedGroup (E:137-156),
 * generalised from 2 to n_views neighbours. */
typedef struct d360_group {
    int32_t width, height;      /* W == 2H (G:40) */
    int32_t n_views;            /* 1..D360_MAX_VIEWS */
    int32_t n_samples;          /* 1..D360_MAX_SAMPLES */
    int32_t top_k;              /* 1..n_views; cost = mean of the k smallest per-view costs.
                                   n_views=2, top_k=2 is the reference's 0.5*(c0+c1) (K:297) */
    int32_t precision;          /* D360_PREC_* */
    const float *rays;          /* device (H,W,3) */
    const float *ref_gray;      /* device (H,W) */
    const float *nb;            /* device neighbour luma, V planes of (H + 2*nb_pad_y, W + 2*nb_pad_x):
                                   the image with nb_pad_x wrapped columns on each side (the
                                   panorama is periodic in x, K:141-150) and nb_pad_y replicated
                                   rows above/below (v is clamped, K:143-147).  Pads 0 = dense
                                   (V,H,W).  d360_to_gray_padded writes this layout; pads >= 1
                                   enable the branch-free bilinear taps of the throughput kernels */
    int32_t nb_pad_x, nb_pad_y;
    const double *nb64;         /* device, optional: the same padded planes widened to f64 (exact), two
                                   doubles per texel: { value, value(x+1) - value }.  The reference
                                   interpolates in f64 (K:134-153); with these planes a bilinear
                                   footprint is two 16-byte loads and no per-tap conversion.
                                   NULL: the generic kernels run */
    const float *rel_r;         /* host (V,3,3) x_nb = R x_ref + t (G:182-188), f32 (E:152) */
    const float *rel_t;         /* host (V,3) */
    const int32_t *offsets;     /* host (S,2) as (dx,dy) (E:60-65) */
    double trunc;               /* PatchSpec.cost_truncation */
    const float *ref_ctx;       /* device, optional: reference patch context as one padded plane
                                   (H + 2p, W + 2p, 4) f32 = (ray.x, ray.y, ray.z, luma) with
                                   p = ref_ctx_pad wrapped columns / replicated rows (the sample
                                   wrap / clamp rules of K:168-177 as data).  Written by
                                   d360_build_ref_context.  With it (and p >= the patch reach) the
                                   throughput kernels stage a CTA's patch window in
                                   shared memory with one TMA tile load (cp.async.bulk.tensor.2d)
                                   instead of four scattered loads per window entry.  NULL: plain loads */
    int32_t ref_ctx_pad;
} d360_group;

const char *d360_last_error(void);
int d360_version(void);

/* Instrumentation (the reference has only perf_counter stage clocks).
 * d360_launch_count: kernels launched by this library since it was loaded.
 * d360_trace_enable(1) clears the trace and starts bracketing every launch with CUDA
 * events on its stream; d360_trace_summary synchronises them and writes one line per
 * kernel kind, "<kind> <launches> <total_ms>\n", returning the byte count (-1 on error). */
unsigned long long d360_launch_count(void);
/* Launches that ran on the generic kernels (csrc/d360_patchmatch.cu, about 2x slower) although the
 * MIXED policy was requested, because the throughput kernels do not cover the group: irregular sample
 * pattern, no padded f64 planes (nb64 / pads), a padded plane of 2^23 texels or more together with a patch other
 * than the default 5x5 stride-2 one (with the default patch such planes stay on the throughput kernels), or a patch window
 * above 200 KB of shared memory.  The first launch of each reason is also reported on stderr (silenced by
 * the environment variable D360_QUIET_FALLBACK).  The reference has no such split (one numba path). */
unsigned long long d360_generic_fallbacks(void);
int d360_trace_enable(int on);
int d360_trace_summary(char *buf, int cap);

/* replaces kernels.eval_costs (K:300-349; caller E:366-379) */
int d360_eval_costs(const d360_group *g, const float *depth, const float *normal,
                    float *cost_out, void *stream);

/* replaces kernels.red_black_pass (K:352-473; callers E:403-420, E:578-595).
 * Unlike the reference the caller need NOT pre-copy in->out: off-parity pixels are
 * copied by the kernel.  n_evals (device, optional, uint64) is incremented by the number
 * of cost evaluations executed (duplicate candidates skipped, K:418-432).
 * Contract on cost_in: it must be the cost of the stored hypothesis (what d360_eval_costs or an
 * earlier pass wrote), as it always is inside run_patchmatch (E:564).  Under D360_PREC_MIXED the
 * throughput kernel skips a neighbour equal to the pixel's ORIGINAL hypothesis even after that
 * hypothesis has been displaced; the reference re-evaluates it and strict `<` rejects it exactly
 * when cost_in is its true cost.  With stale finite costs the two rules can differ, and n_evals
 * then counts fewer evaluations than the reference executes.  D360_PREC_EXACT follows K:418-432
 * to the letter. */
int d360_red_black_pass(const d360_group *g, int parity, const float *depth_in,
                        const float *normal_in, const float *cost_in, float *depth_out,
                        float *normal_out, float *cost_out, unsigned long long *n_evals,
                        void *stream);

/* replaces kernels.refine_pass (K:476-610; caller E:602-621).  cand_* are host arrays of
 * n_cand floats (E:495-526).  In place. */
int d360_refine_pass(const d360_group *g, float *depth, float *normal, float *cost,
                     const float *cand_dd, const float *cand_sa, const float *cand_ca,
                     const float *cand_caz, const float *cand_saz, int n_cand,
                     double depth_min, double depth_max, void *stream);

/* replaces the loop of engine.run_patchmatch (E:563-631): eval_costs, then `iterations`
 * x (red, black, refine) with state resident on the device.  tables: host
 * (iterations,5,n_cand) f32 in the order (dd, sin ang, cos ang, cos az, sin az).
 * depth/normal in/out, cost out; scratch_* are caller-owned ping-pong buffers of the same
 * shapes.  scratch_flags (u8, 3*H*W bytes) and scratch_memo (f64, 8*H*W) — optional, both or
 * neither — are the work area of memoised candidate costs: the cost of a neighbour's
 * hypothesis at a pixel is a pure function of the two, so a propagation pass re-evaluates a
 * candidate only when that neighbour's hypothesis changed since the pixel last evaluated it
 * and otherwise reuses the f64 cost it computed then; results are bit-identical with and
 * without it, only fewer evaluations run (csrc/d360_fast_rb.cu).
 * valid_out (optional, u8) = cost < trunc (E:629).
 * n_evals (device, optional, uint64[2]): [0] += cost evaluations started (propagation +
 * refinement), [1] += refinement evaluations that were decided after V - 1 views (the last
 * view cannot lift a candidate over the acceptance threshold of K:600, csrc/d360_fast.cuh)
 * and so did 1/V less work. */
int d360_run_patchmatch(const d360_group *g, float *depth, float *normal, float *cost,
                        float *scratch_depth, float *scratch_normal, float *scratch_cost,
                        uint8_t *scratch_flags, double *scratch_memo, const float *tables,
                        int iterations, int n_cand, double depth_min,
                        double depth_max, uint8_t *valid_out, unsigned long long *n_evals,
                        void *stream);

/* writes d360_group.ref_ctx from the (H,W,3) rays and the (H,W) reference luma */
int d360_build_ref_context(const float *rays, const float *ref_gray, float *ctx, int height,
                           int width, int pad, void *stream);

/* replaces kernels.median_support_mask (K:613-647; caller E:634-648) */
int d360_median_support_mask(const float *depth, const uint8_t *valid, int half,
                             double rel_threshold, uint8_t *out_valid, int height, int width,
                             void *stream);

/* replaces keyframes.to_gray (KF:64-72).  channels = 1 or 3, image device u8. */
int d360_to_gray(const uint8_t *image, int channels, float *gray, int height, int width,
                 void *stream);
/* same, written into the padded plane layout of d360_group.nb / nb64: gray is
 * (height + 2*pad_y, width + 2*pad_x) f32, gray64 the same raster with two doubles per texel
 * { value, value(x+1) - value }; either may be NULL */
int d360_to_gray_padded(const uint8_t *image, int channels, float *gray, double *gray64,
                        int height, int width, int pad_x, int pad_y, void *stream);

/* replaces geometry.camera_rays (G:117-122).  Tables are device f64 arrays computed by the
 * host exactly as G:81-86; rays32 (H,W,3) f32 and/or rays64 (H,W,3) f64 may be NULL. */
int d360_camera_rays(const double *sin_lam, const double *cos_lam, const double *sin_phi,
                     const double *cos_phi, float *rays32, double *rays64, int height,
                     int width, void *stream);

/* replaces engine.random_init (E:244-283).
 * Injected mode (inv_draws/normal_draws non-NULL, device f64 (H,W) / (H,W,3)): applies the
 * reference transform to host-generated NumPy PCG64 draws -> identical hypotheses.
 * Native mode (both NULL): counter-based Philox4x32-10 keyed by `seed`, counter = pixel
 * index; same distributions (uniform inverse depth, uniform facing hemisphere).
 * Fills only pixels with valid==0, sets their cost to +inf, then marks all valid. */
int d360_random_init(float *depth, float *normal, float *cost, uint8_t *valid,
                     const double *inv_draws, const double *normal_draws, uint64_t seed,
                     double depth_min, double depth_max, const double *rays64, int height,
                     int width, void *stream);

/* replaces engine.warp_plane_map (E:286-355).  r_rel/t_rel host f64 from
 * relative_transform(pose_prev, pose_cur).  Outputs are fully overwritten (unfilled pixels
 * get depth 0, normal 0, cost +inf, valid 0).  winner: device scratch (H,W) uint64. */
int d360_warp_plane_map(const float *src_depth, const float *src_normal,
                        const float *src_cost, const uint8_t *src_valid, const double *rays64,
                        const double *r_rel, const double *t_rel, double depth_min,
                        double depth_max, float *out_depth, float *out_normal, float *out_cost,
                        uint8_t *out_valid, unsigned long long *winner, int height, int width,
                        void *stream);

/* rows with |latitude| > limit_deg are invalidated in place */
int d360_pole_mask(uint8_t *valid, double limit_deg, int height, int width, void *stream);

/* replaces pipeline.consistency_filter.  Window frames: device depth/valid
 * pointers per frame (host arrays of n_frames pointers), poses host f64 (n_frames,9)/(n_frames,3)
 * camera->world. */
int d360_consistency_filter(const float *depth, const uint8_t *valid, const double *rot,
                            const double *trans, const float *const *win_depth,
                            const uint8_t *const *win_valid, const double *win_rot,
                            const double *win_trans, int n_frames, const double *rays64,
                            int min_support, double rel_tol, uint8_t *out_valid, int height,
                            int width, void *stream);

/* replaces FusionBuffer._fuse_oldest.  Emits surviving points in row-major
 * order of the oldest frame (np.nonzero order): points (N,3) f64, colors (N,3) u8.
 * keep (H,W) u8 and block_counts (device uint32, >= d360_fuse_blocks(H,W)+1 entries) are
 * scratch; *n_points_host receives N (this call synchronises the stream once). */
int d360_fuse_blocks(int height, int width);
int d360_fuse_oldest(const float *depth, const uint8_t *valid, const double *rot,
                     const double *trans, const uint8_t *image_rgb,
                     const float *const *newer_depth, const uint8_t *const *newer_valid,
                     const double *newer_rot, const double *newer_trans, int n_newer,
                     const double *rays64, double reproj_px, double rel_tol, uint8_t *keep,
                     uint32_t *block_counts, double *points, uint8_t *colors,
                     int64_t *n_points_host, int height, int width, void *stream);

/* replaces synth.render_scene (SY:154-169) with SyntheticScene.cast (SY:66-84) and .shade (SY:86-98):
 * analytic ray cast of a closed scene seen from inside - kind 0: axis-aligned box / corridor of full extents
 * size_xyz, kind 1: sphere shell of radius size_xyz[0] / 2 with oo_minus_r2 = o @ o - radius^2 evaluated by
 * the caller - and its texture: multi-octave splitmix value noise (SY:101-151), or with checker != 0 the
 * 40 / 215 checkerboard of SY:88-92 with noise_scale-sized cells.  f64 throughout; image (H,W,3) u8,
 * depth (H,W) f32.  Bit-identical to the reference's images, rotations included (see the kernel's note on
 * the two BLAS statements). */
int d360_render_scene(int kind, int checker, const double *size_xyz, double oo_minus_r2,
                      int texture_seed, double noise_scale, int octaves, const double *rot,
                      const double *trans, const double *rays64, uint8_t *image, float *depth,
                      int height, int width, void *stream);
/* the same for kind 0 without checker (kept for callers of the first release) */
int d360_render_box_scene(const double *size_xyz, int texture_seed, double noise_scale,
                          int octaves, const double *rot, const double *trans,
                          const double *rays64, uint8_t *image, float *depth, int height,
                          int width, void *stream);

/* replaces dataset.resample_keyframe (dataset.py:146-157) = Pillow Image.resize(size, LANCZOS) on an 8-bit
 * (H,W) or (H,W,3) image (Pillow 12.2.0, src/libImaging/Resample.c: horizontal pass into a uint8 intermediate,
 * then vertical pass; 22-bit fixed-point coefficients).  bounds_* (n_out, 2) = (first source index, tap count),
 * kk_* (n_out, ksize_*) = integer coefficients, both on the device, computed by the caller as Pillow's
 * precompute_coeffs + normalize_coeffs_8bpc do (paper_2211_16266_b200/ingest.py).  bounds_y must already be
 * relative to row0; tmp holds (rows, dst_w, channels) bytes for source rows [row0, row0 + rows).  When only one
 * axis changes Pillow skips the other pass; the caller then passes identity windows (one tap of 1 << 22). */
int d360_resample_u8(const uint8_t *src, int src_h, int src_w, int channels, uint8_t *tmp, uint8_t *dst,
                     int dst_h, int dst_w, const int32_t *bounds_x, const int32_t *kk_x, int ksize_x,
                     const int32_t *bounds_y, const int32_t *kk_y, int ksize_y, int row0, int rows,
                     void *stream);

/* FP32-FMA peak microbenchmark used as the roofline denominator for the cost kernels
 * (MEASURED_PEAKS.json carries no FP32 figure).  Returns achieved TFLOP/s (FMA = 2),
 * fp64 != 0 measures the DFMA pipe instead.  Synchronous. */
double d360_measure_fma_peak(int fp64, int iters);

/* ---- output packing and metrics --------------------- */

/* replaces the record packing of outputs.write_ply (outputs.py:30-54): n records of 15 bytes,
 * (x, y, z) = astype(float32) of the f64 world points, little endian, then r, g, b. */
int d360_pack_ply_records(const double *points, const uint8_t *colors, uint8_t *records,
                          int64_t n, void *stream);

/* replaces the quantisation of outputs.write_depth_png (outputs.py:81-97):
 * mm = clip(rint(depth * 1000), 0, 65535) in f64 as u16, 0 where invalid.  stats (device,
 * 3 x uint32, written): valid count, and the min / max valid depth as order-preserving keys
 * (key = bits ^ (sign ? 0xffffffff : 0x80000000)) for the JSON sidecar. */
int d360_depth_to_mm16(const float *depth, const uint8_t *valid, uint16_t *mm, uint32_t *stats,
                       int height, int width, void *stream);

/* replaces the per-pose splat of metrics.completeness (metrics.py:31-45): marks
 * raster[py, px] = 1 (u8 (height, width), zeroed by the caller) for every point. */
int d360_completeness_splat(const double *points, int64_t n, const double *rot,
                            const double *trans, uint8_t *raster, int height, int width,
                            void *stream);
/* *count (device) += number of nonzero bytes */
int d360_count_nonzero(const uint8_t *a, int64_t n, unsigned long long *count, void *stream);

/* replaces metrics.accuracy (metrics.py:52-78): out (device, 4 doubles) = { sum |p-g|/g,
 * sum (p-g)^2, #(|p-g|/g <= 0.02), #jointly valid }; scratch: device,
 * d360_accuracy_scratch_doubles() doubles.  Fixed reduction order (run-to-run identical). */
int d360_accuracy_scratch_doubles(void);
int d360_depth_accuracy(const float *pred_depth, const uint8_t *pred_valid, const float *gt_depth,
                        const uint8_t *gt_valid, int64_t n, double *scratch, double *out,
                        void *stream);

/* metrics.voxel_occupancy (metrics.py:81-87): keys[i] = floor(p / voxel) per axis packed
 * 3 x 21 bits; *overflow (device int) set if a cell index leaves [-2^20, 2^20). */
int d360_voxel_keys(const double *points, int64_t n, double voxel, long long *keys, int *overflow,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* D360_H */
