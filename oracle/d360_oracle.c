/*
 * d360_oracle.c — CPU restatement of the densify360 hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity ORACLE for the CUDA path in paper_2211_16266_b200/csrc.
 * It is a from-scratch plain-C restatement of the reference's algorithm; it is not
 * shipped, never imported by the product package, and may only be used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
 *
 * Parity status: PINNED at V=2 against the reference itself (numba 0.65 build of
 * /root/reference/pkg/src/densify360 run in the build container; vectors under
 * tests/golden/, generator oracle/gen_golden.py).  UNPINNED for V>2 / top-k (the
 * reference rejects len(neighbors) != 2, keyframes.py:47-49) — there the oracle is
 * the direct per-view generalisation of K:201-297 and is asserted equal at V=2,k=2.
 *
 * Reference shorthand: K = pkg/src/densify360/kernels.py, E = engine.py,
 * P = pipeline.py, G = geometry.py.
 *
 * Mixed precision follows numba's type inference of the reference (verified with
 * inspect_types): hypothesis dot products are f32 when the caller
 * passes f32 hypotheses (eval_costs, red_black_pass) and f64 inside refine_pass,
 * whose loop-carried d/n/c unify to float64; everything after lam = num/dn is f64;
 * projected (u, v) are rounded to f32 (the reference's `scr` scratch array);
 * bilinear and the NCC sums are f64; stored costs are rounded to f32.
 * Built with -ffp-contract=off so every statement below is one IEEE operation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

/* Row-parallel driver (pthreads; the image's default gcc has no usable libgomp spec
 * and the host process already carries torch's OpenMP runtime).  Rows are handed out
 * dynamically; results do not depend on the thread count because every row writes
 * only its own outputs (same argument as K:3-5). */
static int g_threads = 0;
void d360o_set_threads(int n) { g_threads = n; }
int d360o_get_threads(void) {
    if (g_threads > 0) return g_threads;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}
typedef void (*row_fn)(int y, void *arg, void *scratch);
typedef struct { row_fn fn; void *arg; int h; atomic_int next; size_t scratch_bytes; } job_t;
static void *worker(void *p) {
    job_t *j = (job_t *)p;
    void *scratch = j->scratch_bytes ? malloc(j->scratch_bytes) : NULL;
    for (;;) {
        int y = atomic_fetch_add(&j->next, 1);
        if (y >= j->h) break;
        j->fn(y, j->arg, scratch);
    }
    free(scratch);
    return NULL;
}
static void parallel_rows(int h, row_fn fn, void *arg, size_t scratch_bytes) {
    job_t j = {fn, arg, h, 0, scratch_bytes};
    int nt = d360o_get_threads();
    if (nt > h) nt = h;
    if (nt <= 1) { worker(&j); return; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nt);
    int started = 0;
    for (int i = 0; i < nt - 1; ++i)
        if (pthread_create(&th[started], NULL, worker, &j) == 0) ++started;
    worker(&j);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th);
}

#define FACING_EPS 1e-6   /* K:34 */
#define PARALLEL_EPS 1e-9 /* K:35 */
#define SIGMA_EPS 1e-4    /* K:36 */
#define VAR_EPS 1e-8      /* K:37 */
#define D360_PI 3.141592653589793
#define MAX_VIEWS 8
#define MAX_SAMPLES 256

/* K:44-56 */
static const int NEIGHBOR_OFFSETS[8][2] = {{-1, -1}, {1, -1}, {-1, 1}, {1, 1},
                                           {0, -2},  {0, 2},  {-2, 0}, {2, 0}};

typedef struct {
    int h, w, n_views, n_samples, top_k;
    const float *rays;     /* (H, W, 3) */
    const float *ref_gray; /* (H, W) */
    const float *nb;       /* (V, H, W) */
    const float *rel_r;    /* (V, 3, 3) */
    const float *rel_t;    /* (V, 3) */
    const int32_t *offsets; /* (S, 2) as (dx, dy) */
    double trunc;
} group_t;

/* K:59-99 */
static inline double fast_atan2(double y_, double x_) {
    double ax = fabs(x_), ay = fabs(y_);
    double hi = ax > ay ? ax : ay;
    double lo = ax > ay ? ay : ax;
    double r = lo / (hi + 1e-300);
    double s = r * r;
    double p =
        r *
        (9.999999227776e-01 +
         s * (-3.333223261885e-01 +
              s * (1.997402857787e-01 +
                   s * (-1.404782123164e-01 +
                        s * (1.000220525649e-01 +
                             s * (-6.087448223083e-02 +
                                  s * (2.533170107199e-02 + s * -5.021063913876e-03)))))));
    p = ay > ax ? 1.5707963267948966 - p : p;
    p = x_ < 0.0 ? 3.141592653589793 - p : p;
    return y_ < 0.0 ? -p : p;
}

/* K:102-131 */
static inline double fast_acos(double x_) {
    double a = fabs(x_);
    a = a > 1.0 ? 1.0 : a;
    double p =
        (1.570796263346e00 +
         a * (-2.145970563340e-01 +
              a * (8.895977933699e-02 +
                   a * (-5.008467775423e-02 +
                        a * (3.068214201158e-02 +
                             a * (-1.682974898800e-02 +
                                  a * (6.510368059701e-03 + a * -1.223553911532e-03))))))) *
        sqrt(1.0 - a);
    return x_ < 0.0 ? 3.141592653589793 - p : p;
}

#ifdef D360O_F32_PROJECTION
/* Experiment build only (tools/f32_projection.py): the same projection with every
 * operation after lam in float32.  Never the checker: the default build does not define the macro. */
static inline float fast_atan2_f32(float y_, float x_) {
    float ax = fabsf(x_), ay = fabsf(y_);
    float hi = ax > ay ? ax : ay;
    float lo = ax > ay ? ay : ax;
    float r = lo / (hi + 1e-30f);
    float s = r * r;
    float p = r * (9.999999227776e-01f +
                   s * (-3.333223261885e-01f +
                        s * (1.997402857787e-01f +
                             s * (-1.404782123164e-01f +
                                  s * (1.000220525649e-01f +
                                       s * (-6.087448223083e-02f +
                                            s * (2.533170107199e-02f + s * -5.021063913876e-03f)))))));
    p = ay > ax ? 1.5707963267948966f - p : p;
    p = x_ < 0.0f ? 3.141592653589793f - p : p;
    return y_ < 0.0f ? -p : p;
}
static inline float fast_acos_f32(float x_) {
    float a = fabsf(x_);
    a = a > 1.0f ? 1.0f : a;
    float p = (1.570796263346e00f +
               a * (-2.145970563340e-01f +
                    a * (8.895977933699e-02f +
                         a * (-5.008467775423e-02f +
                              a * (3.068214201158e-02f +
                                   a * (-1.682974898800e-02f +
                                        a * (6.510368059701e-03f + a * -1.223553911532e-03f))))))) *
              sqrtf(1.0f - a);
    return x_ < 0.0f ? 3.141592653589793f - p : p;
}
#endif

/* K:134-153 */
static inline double bilinear(const float *img, int h, int w, float u, float v) {
    long u0 = (long)floorf(u);
    double fu = (double)u - (double)u0;
    u0 = u0 < 0 ? u0 + w : u0;
    u0 = u0 >= w ? u0 - w : u0;
    long u1 = u0 + 1;
    u1 = u1 == w ? 0 : u1;
    double vc = v < 0.0f ? 0.0 : (double)v;
    double vm = h - 1.0;
    vc = vc > vm ? vm : vc;
    long v0 = (long)vc;
    v0 = v0 > h - 2 ? h - 2 : v0;
    double fv = vc - (double)v0;
    long v1 = v0 + 1;
    double top = img[v0 * w + u0] * (1.0 - fu) + img[v0 * w + u1] * fu;
    double bot = img[v1 * w + u0] * (1.0 - fu) + img[v1 * w + u1] * fu;
    return top * (1.0 - fv) + bot * fv;
}

/* Per-pixel context block, K:156-198.  buf rows: 0..2 sample ray, 3+3v..5+3v ray
 * rotated into neighbour v, last row reference intensity. */
typedef struct {
    float q[3][MAX_SAMPLES];
    float rq[MAX_VIEWS][3][MAX_SAMPLES];
    float ref[MAX_SAMPLES];
    double mr, sr;
} ctx_t;

static void gather_ctx(const group_t *g, int x, int y, ctx_t *c) {
    const int h = g->h, w = g->w, s = g->n_samples;
    double acc = 0.0, acc2 = 0.0;
    for (int k = 0; k < s; ++k) {
        int qx = x + g->offsets[2 * k];
        if (qx < 0) qx += w; else if (qx >= w) qx -= w;
        int qy = y + g->offsets[2 * k + 1];
        if (qy < 0) qy = 0; else if (qy >= h) qy = h - 1;
        const float *ray = g->rays + ((size_t)qy * w + qx) * 3;
        float bx = ray[0], by = ray[1], bz = ray[2];
        c->q[0][k] = bx; c->q[1][k] = by; c->q[2][k] = bz;
        for (int v = 0; v < g->n_views; ++v) {
            const float *r = g->rel_r + 9 * v;
            c->rq[v][0][k] = r[0] * bx + r[1] * by + r[2] * bz;
            c->rq[v][1][k] = r[3] * bx + r[4] * by + r[5] * bz;
            c->rq[v][2][k] = r[6] * bx + r[7] * by + r[8] * bz;
        }
        float val = g->ref_gray[(size_t)qy * w + qx];
        c->ref[k] = val;
        acc += val;
        acc2 += (double)(val * val); /* f32 product, f64 accumulate (K:193) */
    }
    double m = acc / s;
    double var = acc2 / s - m * m;
    if (var < 0.0) var = 0.0;
    c->mr = m;
    c->sr = sqrt(var);
}

/* Top-k aggregation of per-view truncated costs: mean of the k smallest, summed in
 * ascending order.  V=2,k=2 is the reference's 0.5*(c0+c1) (K:297). */
static inline double aggregate(double *cv, int n_views, int top_k) {
    for (int i = 1; i < n_views; ++i) { /* insertion sort, stable */
        double t = cv[i];
        int j = i - 1;
        while (j >= 0 && cv[j] > t) { cv[j + 1] = cv[j]; --j; }
        cv[j + 1] = t;
    }
    double total = 0.0;
    for (int i = 0; i < top_k; ++i) total += cv[i];
    return (1.0 / top_k) * total;
}

/* Phase A+B of K:201-297 given num (f64 value of the caller-precision product) and
 * a per-sample denominator callback result array. */
static double cand_cost_core(const group_t *g, const ctx_t *c, double num,
                             const double *dn, int bad) {
    const int s = g->n_samples, h = g->h, w = g->w, nv = g->n_views;
    const double trunc = g->trunc;
    if (bad) return trunc; /* K:259-260 (projection has no side effects) */
    const double half_w = w * (0.5 / D360_PI);
    const double lat_scale = h / D360_PI;
    double cv[MAX_VIEWS];
    const double inv_s = 1.0 / s;
    for (int v = 0; v < nv; ++v) {
        const double t0x = g->rel_t[3 * v], t0y = g->rel_t[3 * v + 1], t0z = g->rel_t[3 * v + 2];
        const float *img = g->nb + (size_t)v * h * w;
        double s0 = 0.0, ss0 = 0.0, rs0 = 0.0;
        for (int k = 0; k < s; ++k) {
#ifdef D360O_F32_PROJECTION
            float lam = (float)num / (float)dn[k];
            float tx = lam * (float)c->rq[v][0][k] + (float)t0x;
            float ty = lam * (float)c->rq[v][1][k] + (float)t0y;
            float tz = lam * (float)c->rq[v][2][k] + (float)t0z;
            float inv_r = 1.0f / sqrtf(tx * tx + ty * ty + tz * tz + 1e-30f);
            float sphi = -ty * inv_r;
            float pu = (fast_atan2_f32(tx, tz) + (float)D360_PI) * (float)half_w - 0.5f;
            float pv = fast_acos_f32(sphi) * (float)lat_scale - 0.5f;
#else
            double lam = num / dn[k];
            double tx = lam * c->rq[v][0][k] + t0x;
            double ty = lam * c->rq[v][1][k] + t0y;
            double tz = lam * c->rq[v][2][k] + t0z;
            double inv_r = 1.0 / sqrt(tx * tx + ty * ty + tz * tz + 1e-30);
            double sphi = -ty * inv_r;
            float pu = (float)((fast_atan2(tx, tz) + D360_PI) * half_w - 0.5);
            float pv = (float)(fast_acos(sphi) * lat_scale - 0.5);
#endif
            double val = bilinear(img, h, w, pu, pv);
            s0 += val;
            ss0 += val * val;
            rs0 += c->ref[k] * val;
        }
        double m0 = s0 * inv_s;
        double v0 = ss0 * inv_s - m0 * m0;
        if (v0 < VAR_EPS) {
            cv[v] = trunc;
        } else {
            double cc = 1.0 - (rs0 * inv_s - c->mr * m0) / (c->sr * sqrt(v0));
            cc = cc < 0.0 ? 0.0 : cc;
            cc = cc > trunc ? trunc : cc;
            cv[v] = cc;
        }
    }
    return aggregate(cv, nv, g->top_k);
}

/* f32-hypothesis specialisation (callers: eval_costs K:328, red_black_pass K:441). */
static double cand_cost_f32(const group_t *g, const ctx_t *c, float d, float nx, float ny,
                            float nz, float ax, float ay, float az) {
    float ndota = nx * ax + ny * ay + nz * az;
    if ((double)ndota >= -FACING_EPS || c->sr < SIGMA_EPS) return g->trunc;
    float num = d * ndota;
    double dn[MAX_SAMPLES];
    int bad = 0;
    for (int k = 0; k < g->n_samples; ++k) {
        float den = nx * c->q[0][k] + ny * c->q[1][k] + nz * c->q[2][k];
        if ((double)den > -PARALLEL_EPS) bad = 1;
        dn[k] = (double)den < -PARALLEL_EPS ? (double)den : -PARALLEL_EPS;
    }
    return cand_cost_core(g, c, (double)num, dn, bad);
}

/* f64-hypothesis specialisation (caller: refine_pass K:577, whose d/n unify to f64). */
static double cand_cost_f64(const group_t *g, const ctx_t *c, double d, double nx, double ny,
                            double nz, float ax, float ay, float az) {
    double ndota = nx * ax + ny * ay + nz * az;
    if (ndota >= -FACING_EPS || c->sr < SIGMA_EPS) return g->trunc;
    double num = d * ndota;
    double dn[MAX_SAMPLES];
    int bad = 0;
    for (int k = 0; k < g->n_samples; ++k) {
        double den = nx * c->q[0][k] + ny * c->q[1][k] + nz * c->q[2][k];
        if (den > -PARALLEL_EPS) bad = 1;
        dn[k] = den < -PARALLEL_EPS ? den : -PARALLEL_EPS;
    }
    return cand_cost_core(g, c, num, dn, bad);
}

static group_t make_group(int h, int w, int n_views, int n_samples, int top_k,
                          const float *rays, const float *ref_gray, const float *nb,
                          const float *rel_r, const float *rel_t, const int32_t *offsets,
                          double trunc) {
    group_t g = {h, w, n_views, n_samples, top_k, rays, ref_gray, nb, rel_r, rel_t, offsets, trunc};
    return g;
}

int d360o_max_views(void) { return MAX_VIEWS; }
int d360o_max_samples(void) { return MAX_SAMPLES; }

static int check_dims(int n_views, int n_samples, int top_k) {
    return n_views < 1 || n_views > MAX_VIEWS || n_samples < 1 || n_samples > MAX_SAMPLES ||
           top_k < 1 || top_k > n_views;
}

/* ---- eval_costs, K:300-349 ---- */
typedef struct {
    group_t g;
    const float *depth, *normal;
    float *cost_out;
} eval_args;

static void eval_row(int y, void *arg, void *scratch) {
    eval_args *a = (eval_args *)arg;
    ctx_t *c = (ctx_t *)scratch;
    const group_t *g = &a->g;
    const int w = g->w;
    for (int x = 0; x < w; ++x) {
        size_t i = (size_t)y * w + x;
        gather_ctx(g, x, y, c);
        a->cost_out[i] = (float)cand_cost_f32(g, c, a->depth[i], a->normal[3 * i],
                                              a->normal[3 * i + 1], a->normal[3 * i + 2],
                                              g->rays[3 * i], g->rays[3 * i + 1], g->rays[3 * i + 2]);
    }
}

int d360o_eval_costs(const float *depth, const float *normal, float *cost_out,
                     const float *rays, const float *ref_gray, const float *nb, int n_views,
                     const float *rel_r, const float *rel_t, const int32_t *offsets,
                     int n_samples, int h, int w, double trunc, int top_k) {
    if (check_dims(n_views, n_samples, top_k)) return 1;
    eval_args a = {make_group(h, w, n_views, n_samples, top_k, rays, ref_gray, nb, rel_r, rel_t,
                              offsets, trunc),
                   depth, normal, cost_out};
    parallel_rows(h, eval_row, &a, sizeof(ctx_t));
    return 0;
}

/* ---- red_black_pass, K:352-473.  Caller pre-copies in -> out (E:575-577). ---- */
typedef struct {
    group_t g;
    int parity;
    const float *depth_in, *normal_in, *cost_in;
    float *depth_out, *normal_out, *cost_out;
    _Atomic int64_t evals;
} rb_args;

static void rb_row(int y, void *arg, void *scratch) {
    rb_args *a = (rb_args *)arg;
    ctx_t *c = (ctx_t *)scratch;
    const group_t *g = &a->g;
    const int h = g->h, w = g->w;
    const float *depth_in = a->depth_in, *normal_in = a->normal_in;
    float cand_d[8], cand_nx[8], cand_ny[8], cand_nz[8];
    int64_t evals = 0;
    int x0 = (a->parity + y) & 1;
    for (int x = x0; x < w; x += 2) {
        size_t i = (size_t)y * w + x;
        float bd = depth_in[i];
        float bnx = normal_in[3 * i], bny = normal_in[3 * i + 1], bnz = normal_in[3 * i + 2];
        double bc = a->cost_in[i]; /* unifies to float64 once a candidate wins */
        int gathered = 0, n_seen = 0;
        for (int j = 0; j < 8; ++j) {
            int qy = y + NEIGHBOR_OFFSETS[j][1];
            if (qy < 0 || qy >= h) continue; /* K:407 rows skipped */
            int qx = x + NEIGHBOR_OFFSETS[j][0];
            if (qx < 0) qx += w; else if (qx >= w) qx -= w; /* K:410-413 columns wrap */
            size_t qi = (size_t)qy * w + qx;
            float d = depth_in[qi];
            float nx = normal_in[3 * qi], ny = normal_in[3 * qi + 1], nz = normal_in[3 * qi + 2];
            int dup = d == bd && nx == bnx && ny == bny && nz == bnz;
            if (!dup) {
                for (int m = 0; m < n_seen; ++m) {
                    if (d == cand_d[m] && nx == cand_nx[m] && ny == cand_ny[m] && nz == cand_nz[m]) {
                        dup = 1;
                        break;
                    }
                }
            }
            if (dup) continue;
            cand_d[n_seen] = d; cand_nx[n_seen] = nx; cand_ny[n_seen] = ny; cand_nz[n_seen] = nz;
            ++n_seen;
            if (!gathered) { gather_ctx(g, x, y, c); gathered = 1; }
            double cc = cand_cost_f32(g, c, d, nx, ny, nz, g->rays[3 * i], g->rays[3 * i + 1],
                                      g->rays[3 * i + 2]);
            ++evals;
            if (cc < bc) { /* K:463 */
                bc = cc;
                bd = d; bnx = nx; bny = ny; bnz = nz;
            }
        }
        a->depth_out[i] = bd;
        a->normal_out[3 * i] = bnx; a->normal_out[3 * i + 1] = bny; a->normal_out[3 * i + 2] = bnz;
        a->cost_out[i] = (float)bc;
    }
    atomic_fetch_add(&a->evals, evals);
}

/* n_evals (optional) receives the number of cost evaluations actually executed. */
int d360o_red_black_pass(int parity, const float *depth_in, const float *normal_in,
                         const float *cost_in, float *depth_out, float *normal_out,
                         float *cost_out, const float *rays, const float *ref_gray,
                         const float *nb, int n_views, const float *rel_r, const float *rel_t,
                         const int32_t *offsets, int n_samples, int h, int w, double trunc,
                         int top_k, int64_t *n_evals) {
    if (check_dims(n_views, n_samples, top_k)) return 1;
    rb_args a = {make_group(h, w, n_views, n_samples, top_k, rays, ref_gray, nb, rel_r, rel_t,
                            offsets, trunc),
                 parity, depth_in, normal_in, cost_in, depth_out, normal_out, cost_out, 0};
    parallel_rows(h, rb_row, &a, sizeof(ctx_t));
    if (n_evals) *n_evals = a.evals;
    return 0;
}

/* ---- refine_pass, K:476-610.  In place.  Loop-carried d, n, c are float64. ---- */
typedef struct {
    group_t g;
    float *depth, *normal, *cost;
    const float *cand_dd, *cand_sa, *cand_ca, *cand_caz, *cand_saz;
    int n_cand;
    double depth_min, depth_max;
} refine_args;

static void refine_row(int y, void *arg, void *scratch) {
    refine_args *a = (refine_args *)arg;
    ctx_t *cx = (ctx_t *)scratch;
    const group_t *g = &a->g;
    const int w = g->w;
    for (int x = 0; x < w; ++x) {
        size_t i = (size_t)y * w + x;
        double d = a->depth[i];
        double nx = a->normal[3 * i], ny = a->normal[3 * i + 1], nz = a->normal[3 * i + 2];
        double c = a->cost[i];
        float ax = g->rays[3 * i], ay = g->rays[3 * i + 1], az = g->rays[3 * i + 2];
        gather_ctx(g, x, y, cx);
        int basis_stale = 1;
        double e1x = 0, e1y = 0, e1z = 0, e2x = 0, e2y = 0, e2z = 0;
        for (int k = 0; k < a->n_cand; ++k) {
            double nd = d + (double)a->cand_dd[k];
            if (nd < a->depth_min) nd = a->depth_min;
            else if (nd > a->depth_max) nd = a->depth_max;
            if (basis_stale) {
                e1x = ny * az - nz * ay;
                e1y = nz * ax - nx * az;
                e1z = nx * ay - ny * ax;
                double m2 = e1x * e1x + e1y * e1y + e1z * e1z;
                if (m2 < 1e-12) {
                    e1x = -nz; e1y = 0.0; e1z = nx;
                    m2 = e1x * e1x + e1z * e1z;
                    if (m2 < 1e-12) { e1x = 1.0; e1z = 0.0; m2 = 1.0; }
                }
                double inv = 1.0 / sqrt(m2);
                e1x *= inv; e1y *= inv; e1z *= inv;
                e2x = ny * e1z - nz * e1y;
                e2y = nz * e1x - nx * e1z;
                e2z = nx * e1y - ny * e1x;
                basis_stale = 0;
            }
            double sa = a->cand_sa[k], ca = a->cand_ca[k], caz = a->cand_caz[k], saz = a->cand_saz[k];
            double cnx = nx * ca + (e1x * caz + e2x * saz) * sa;
            double cny = ny * ca + (e1y * caz + e2y * saz) * sa;
            double cnz = nz * ca + (e1z * caz + e2z * saz) * sa;
            double nrm = sqrt(cnx * cnx + cny * cny + cnz * cnz);
            if (nrm < 1e-12) continue;
            double inv = 1.0 / nrm;
            cnx *= inv; cny *= inv; cnz *= inv;
            double ev = cand_cost_f64(g, cx, nd, cnx, cny, cnz, ax, ay, az);
            if (ev < c) {
                c = ev; d = nd; nx = cnx; ny = cny; nz = cnz;
                basis_stale = 1;
            }
        }
        a->depth[i] = (float)d;
        a->normal[3 * i] = (float)nx; a->normal[3 * i + 1] = (float)ny; a->normal[3 * i + 2] = (float)nz;
        a->cost[i] = (float)c;
    }
}

int d360o_refine_pass(float *depth, float *normal, float *cost, const float *cand_dd,
                      const float *cand_sa, const float *cand_ca, const float *cand_caz,
                      const float *cand_saz, int n_cand, double depth_min, double depth_max,
                      const float *rays, const float *ref_gray, const float *nb, int n_views,
                      const float *rel_r, const float *rel_t, const int32_t *offsets,
                      int n_samples, int h, int w, double trunc, int top_k) {
    if (check_dims(n_views, n_samples, top_k)) return 1;
    refine_args a = {make_group(h, w, n_views, n_samples, top_k, rays, ref_gray, nb, rel_r,
                                rel_t, offsets, trunc),
                     depth, normal, cost, cand_dd, cand_sa, cand_ca, cand_caz, cand_saz,
                     n_cand, depth_min, depth_max};
    parallel_rows(h, refine_row, &a, sizeof(ctx_t));
    return 0;
}

static int cmp_f32(const void *a, const void *b) {
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

/* ---- median_support_mask, K:613-647 (not fastmath); masks are 1 byte/pixel ---- */
typedef struct {
    const float *depth;
    const uint8_t *valid;
    uint8_t *out_valid;
    int half, h, w;
    double rel_threshold;
} median_args;

static void median_row(int y, void *arg, void *scratch) {
    median_args *a = (median_args *)arg;
    float *buf = (float *)scratch;
    const int h = a->h, w = a->w, half = a->half;
    for (int x = 0; x < w; ++x) {
        size_t i = (size_t)y * w + x;
        if (!a->valid[i]) { a->out_valid[i] = 0; continue; }
        int n = 0;
        for (int dy = -half; dy <= half; ++dy) {
            int qy = y + dy;
            if (qy < 0 || qy >= h) continue;
            for (int dx = -half; dx <= half; ++dx) {
                int qx = x + dx;
                if (qx < 0) qx += w; else if (qx >= w) qx -= w;
                if (a->valid[(size_t)qy * w + qx]) buf[n++] = a->depth[(size_t)qy * w + qx];
            }
        }
        qsort(buf, n, sizeof(float), cmp_f32);
        double med;
        if (n % 2 == 1) med = buf[n / 2];
        else med = 0.5 * (double)(buf[n / 2 - 1] + buf[n / 2]); /* f32 add, K:646 */
        a->out_valid[i] = fabs((double)a->depth[i] - med) <= a->rel_threshold * med;
    }
}

int d360o_median_support_mask(const float *depth, const uint8_t *valid, int half,
                              double rel_threshold, uint8_t *out_valid, int h, int w) {
    const int win = 2 * half + 1;
    median_args a = {depth, valid, out_valid, half, h, w, rel_threshold};
    parallel_rows(h, median_row, &a, sizeof(float) * win * win);
    return 0;
}

/* keyframes.py:64-72, RGB branch: float32 arithmetic throughout (NumPy weak scalars). */
int d360o_to_gray_rgb(const uint8_t *rgb, float *gray, int h, int w) {
    for (size_t i = 0; i < (size_t)h * w; ++i) {
        float r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
        float acc = 0.299f * r;
        acc = acc + 0.587f * g;
        acc = acc + 0.114f * b;
        gray[i] = acc / 255.0f;
    }
    return 0;
}

/* G:117-122 via row/column tables computed by the caller exactly as G:81-86 does:
 * ray = (cos_phi[y]*sin_lam[x], -sin_phi[y], cos_phi[y]*cos_lam[x]) in f64 -> f32. */
int d360o_camera_rays(const double *sin_lam, const double *cos_lam, const double *sin_phi,
                      const double *cos_phi, float *rays, int h, int w) {
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            float *r = rays + ((size_t)y * w + x) * 3;
            r[0] = (float)(cos_phi[y] * sin_lam[x]);
            r[1] = (float)(-sin_phi[y]);
            r[2] = (float)(cos_phi[y] * cos_lam[x]);
        }
    return 0;
}

/* E:262-283 given the host RNG draws: inv (H,W) f64 uniform inverse depths and
 * g (H,W,3) f64 standard normals.  Fills only ~valid pixels; marks all valid. */
int d360o_random_init_apply(const double *inv, const double *gdraw, const double *rays64,
                            float *depth, float *normal, float *cost, uint8_t *valid, int h,
                            int w) {
    for (size_t i = 0; i < (size_t)h * w; ++i) {
        if (!valid[i]) {
            double gx = gdraw[3 * i], gy = gdraw[3 * i + 1], gz = gdraw[3 * i + 2];
            double nrm = sqrt(gx * gx + gy * gy + gz * gz);
            if (nrm < 1e-12) nrm = 1e-12;
            gx /= nrm; gy /= nrm; gz /= nrm;
            double rx = rays64[3 * i], ry = rays64[3 * i + 1], rz = rays64[3 * i + 2];
            double dot = gx * rx + gy * ry + gz * rz;
            if (dot > 0.0) {
                gx = gx - 2.0 * dot * rx; gy = gy - 2.0 * dot * ry; gz = gz - 2.0 * dot * rz;
            }
            dot = gx * rx + gy * ry + gz * rz;
            if (dot >= -1e-6) { gx = -rx; gy = -ry; gz = -rz; }
            depth[i] = (float)(1.0 / inv[i]);
            normal[3 * i] = (float)gx; normal[3 * i + 1] = (float)gy; normal[3 * i + 2] = (float)gz;
            cost[i] = INFINITY;
        }
        valid[i] = 1;
    }
    return 0;
}

static inline long py_mod(long a, long m) { long r = a % m; return r < 0 ? r + m : r; }
static inline long clipl(long a, long lo, long hi) { return a < lo ? lo : (a > hi ? hi : a); }

/* E:286-355.  rays64 = camera_rays(camera) f64 (H,W,3).  r_rel/t_rel from
 * relative_transform(pose_prev, pose_cur).  Outputs must be PlaneMap.empty(). */
int d360o_warp_plane_map(const float *src_depth, const float *src_normal, const float *src_cost,
                         const uint8_t *src_valid, const double *rays64, const double *r_rel,
                         const double *t_rel, double dmin, double dmax, float *out_depth,
                         float *out_normal, float *out_cost, uint8_t *out_valid, int h, int w) {
    const size_t n = (size_t)h * w;
    for (size_t i = 0; i < n; ++i) { /* scan order = np.nonzero order */
        if (!(src_valid[i] && isfinite(src_cost[i]))) continue;
        double d = src_depth[i];
        double nx = src_normal[3 * i], ny = src_normal[3 * i + 1], nz = src_normal[3 * i + 2];
        double px = d * rays64[3 * i], py = d * rays64[3 * i + 1], pz = d * rays64[3 * i + 2];
        double cx = px * r_rel[0] + py * r_rel[1] + pz * r_rel[2] + t_rel[0];
        double cy = px * r_rel[3] + py * r_rel[4] + pz * r_rel[5] + t_rel[1];
        double cz = px * r_rel[6] + py * r_rel[7] + pz * r_rel[8] + t_rel[2];
        double mx = nx * r_rel[0] + ny * r_rel[1] + nz * r_rel[2];
        double my = nx * r_rel[3] + ny * r_rel[4] + nz * r_rel[5];
        double mz = nx * r_rel[6] + ny * r_rel[7] + nz * r_rel[8];
        double rr = sqrt(cx * cx + cy * cy + cz * cz);
        int keep = rr > 1e-9;
        double lon = atan2(cx, cz);
        double sphi = -cy / (rr > 1e-15 ? rr : 1e-15);
        sphi = sphi < -1.0 ? -1.0 : (sphi > 1.0 ? 1.0 : sphi);
        double fx = (lon + D360_PI) * (w / (2 * D360_PI)) - 0.5;
        double fy = (D360_PI / 2 - asin(sphi)) * (h / D360_PI) - 0.5;
        long tx = py_mod((long)rint(fx), w);
        long ty = clipl((long)rint(fy), 0, h - 1);
        const double *tr = rays64 + ((size_t)ty * w + tx) * 3;
        double num = cx * mx + cy * my + cz * mz;
        double den = tr[0] * mx + tr[1] * my + tr[2] * mz;
        keep = keep && (den < -FACING_EPS);
        double nd = den != 0.0 ? num / den : -1.0;
        keep = keep && nd >= dmin && nd <= dmax;
        if (!keep) continue;
        size_t t = (size_t)ty * w + tx;
        float c = src_cost[i];
        /* smallest source cost wins, ties -> earliest source in scan order (E:342-348) */
        if (!out_valid[t] || c < out_cost[t]) {
            out_depth[t] = (float)nd;
            out_normal[3 * t] = (float)mx; out_normal[3 * t + 1] = (float)my; out_normal[3 * t + 2] = (float)mz;
            out_cost[t] = c;
            out_valid[t] = 1;
        }
    }
    return 0;
}

/* P:118-129 for one world point */
static inline void project_point(const double *rot, const double *trans, double wx, double wy,
                                 double wz, int h, int w, double *u, double *v, double *r) {
    double dx = wx - trans[0], dy = wy - trans[1], dz = wz - trans[2];
    /* local = (X - t) @ R  -> local_j = sum_i d_i R[i][j] */
    double lx = dx * rot[0] + dy * rot[3] + dz * rot[6];
    double ly = dx * rot[1] + dy * rot[4] + dz * rot[7];
    double lz = dx * rot[2] + dy * rot[5] + dz * rot[8];
    double rr = sqrt(lx * lx + ly * ly + lz * lz);
    double lon = atan2(lx, lz);
    if (lon >= D360_PI) lon -= 2.0 * D360_PI;
    *u = (lon + D360_PI) * (w / (2.0 * D360_PI)) - 0.5;
    double safe_r = rr > 1e-300 ? rr : 1e-300;
    double s = -ly / safe_r;
    s = s < -1.0 ? -1.0 : (s > 1.0 ? 1.0 : s);
    *v = acos(s) * (h / D360_PI) - 0.5;
    *r = rr;
}

static inline void lift_point(const double *rays64, size_t i, double depth, const double *rot,
                              const double *trans, double *wx, double *wy, double *wz) {
    double px = depth * rays64[3 * i], py = depth * rays64[3 * i + 1], pz = depth * rays64[3 * i + 2];
    /* world = p @ R.T + t -> world_i = sum_j p_j R[i][j] + t_i */
    *wx = px * rot[0] + py * rot[1] + pz * rot[2] + trans[0];
    *wy = px * rot[3] + py * rot[4] + pz * rot[5] + trans[1];
    *wz = px * rot[6] + py * rot[7] + pz * rot[8] + trans[2];
}

/* P:246-281.  win_* hold n_win frames: depth (n_win,H,W) f32, valid (n_win,H,W) u8,
 * rot (n_win,9), trans (n_win,3). */
int d360o_consistency_filter(const float *depth, const uint8_t *valid, const double *rot,
                             const double *trans, const float *win_depth,
                             const uint8_t *win_valid, const double *win_rot,
                             const double *win_trans, int n_win, const double *rays64,
                             int min_support, double rel_tol, uint8_t *out_valid, int h, int w) {
    const size_t n = (size_t)h * w;
    for (size_t i = 0; i < n; ++i) {
        if (!valid[i]) { out_valid[i] = 0; continue; }
        double wx, wy, wz;
        lift_point(rays64, i, (double)depth[i], rot, trans, &wx, &wy, &wz);
        int support = 0;
        for (int f = 0; f < n_win; ++f) {
            double u, v, r;
            project_point(win_rot + 9 * f, win_trans + 3 * f, wx, wy, wz, h, w, &u, &v, &r);
            long px = py_mod((long)rint(u), w);
            long py = clipl((long)rint(v), 0, h - 1);
            size_t t = (size_t)f * n + (size_t)py * w + px;
            double stored = win_depth[t];
            if (win_valid[t] && fabs(r - stored) <= rel_tol * fabs(stored)) ++support;
        }
        out_valid[i] = support >= min_support;
    }
    return 0;
}

/* P:310-348.  Emits surviving points in row-major order of the oldest frame.
 * Returns the number of points via *n_out; buffers must hold H*W entries. */
int d360o_fuse_oldest(const float *depth, const uint8_t *valid, const double *rot,
                      const double *trans, const uint8_t *image_rgb, const float *newer_depth,
                      const uint8_t *newer_valid, const double *newer_rot,
                      const double *newer_trans, int n_newer, const double *rays64,
                      double reproj_px, double rel_tol, double *points, uint8_t *colors,
                      int64_t *n_out, int h, int w) {
    const size_t n = (size_t)h * w;
    int64_t count = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!valid[i]) continue;
        double wx, wy, wz;
        lift_point(rays64, i, (double)depth[i], rot, trans, &wx, &wy, &wz);
        int duplicate = 0;
        for (int f = 0; f < n_newer && !duplicate; ++f) {
            double u, v, r;
            project_point(newer_rot + 9 * f, newer_trans + 3 * f, wx, wy, wz, h, w, &u, &v, &r);
            long bx = (long)rint(u), by = (long)rint(v);
            for (int dy = -1; dy <= 1 && !duplicate; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    long px = bx + dx, py = by + dy;
                    double ddx = (double)px - u, ddy = (double)py - v;
                    double dist2 = ddx * ddx + ddy * ddy;
                    int inside = py >= 0 && py < h && dist2 <= reproj_px * reproj_px;
                    long pxm = py_mod(px, w);
                    long pyc = clipl(py, 0, h - 1);
                    size_t t = (size_t)f * n + (size_t)pyc * w + pxm;
                    double stored = newer_depth[t];
                    if (inside && newer_valid[t] && fabs(r - stored) <= rel_tol * fabs(stored)) {
                        duplicate = 1;
                        break;
                    }
                }
        }
        if (duplicate) continue;
        points[3 * count] = wx; points[3 * count + 1] = wy; points[3 * count + 2] = wz;
        colors[3 * count] = image_rgb[3 * i]; colors[3 * count + 1] = image_rgb[3 * i + 1];
        colors[3 * count + 2] = image_rgb[3 * i + 2];
        ++count;
    }
    *n_out = count;
    return 0;
}

/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator the CUDA
 * random_init kernel uses in production mode.  Not part of the reference (which
 * draws from NumPy PCG64, E:262); restated here so the device stream can be
 * checked bit-for-bit. */
void d360o_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
