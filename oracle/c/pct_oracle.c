/* pct_oracle.c -- multi-threaded C restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the CPU checker for the
 * full-size parity tests and the CPU baseline / reference arm of bench.py.
 * The product package never loads this library.
 *
 * It restates, operation for operation, the reference `tomoplan` package:
 *
 *   orc_bounds        cloud_io.py:47-50          exact min/max
 *   orc_scatter       tomogram.py:147-194        float64 rasterisation, plane
 *                                                split with ties to ground,
 *                                                per-(plane bin, cell) max/min
 *   orc_finalize      tomogram.py:179-204        cumulative max (ground, bottom
 *                                                up) / min (ceiling, top down),
 *                                                NaN (0x7FC00000) where empty
 *   orc_evaluate      traversability.py:59-236   interval cost, axis gradients,
 *                                                hypot, gentle window, terrain
 *                                                branches, fuse, inflation
 *   orc_simplify      simplify.py:18-73          unique-cell test, forward
 *                                                sweep to a fixpoint
 *
 * Numerics: compiled with -ffp-contract=off and without fast-math, so every
 * float64 expression rounds exactly as numpy's elementwise ufuncs do; hypot
 * is the C library's (numpy's np.hypot calls the same glibc routine); float32
 * products and casts are IEEE round-to-nearest.  The reference z-sorts and
 * uses ufunc.at; max/min are order independent, so per-point atomic max/min
 * on order-preserving integer keys give the same values (only the sign of a
 * zero can differ, where +0.0 and -0.0 meet in one cell -- the reference
 * keeps the first one it sees).
 *
 * Parallelism: a plain pthread task pool (no OpenMP runtime, which could
 * clash with the one torch loads).
 */

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* task pool                                                                 */

typedef void (*task_fn)(void *ctx, int64_t task);

typedef struct {
    task_fn fn;
    void *ctx;
    int64_t ntasks;
    int64_t next;
} pool_t;

static void *pool_worker(void *arg) {
    pool_t *pl = (pool_t *)arg;
    for (;;) {
        int64_t t = __atomic_fetch_add(&pl->next, 1, __ATOMIC_RELAXED);
        if (t >= pl->ntasks) break;
        pl->fn(pl->ctx, t);
    }
    return NULL;
}

#define MAX_THREADS 512

static void parallel_for(int threads, int64_t ntasks, task_fn fn, void *ctx) {
    pool_t pl = {fn, ctx, ntasks, 0};
    if (threads > MAX_THREADS) threads = MAX_THREADS;
    if (threads > ntasks) threads = (int)ntasks;
    if (threads <= 1) {
        pool_worker(&pl);
        return;
    }
    pthread_t th[MAX_THREADS];
    int started = 0;
    for (int i = 0; i < threads - 1; i++)
        if (pthread_create(&th[started], NULL, pool_worker, &pl) == 0) started++;
    pool_worker(&pl);
    for (int i = 0; i < started; i++) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------------ */
/* bounds (cloud_io.py:47-50)                                                */

#define PTS_PER_TASK (1 << 20)

typedef struct {
    const void *xyz;
    int64_t n;
    int is_f64;
    double *part; /* ntasks x 6 */
} bounds_ctx;

static inline double pt(const void *xyz, int is_f64, int64_t i, int a) {
    return is_f64 ? ((const double *)xyz)[3 * i + a] : (double)((const float *)xyz)[3 * i + a];
}

static void bounds_task(void *c, int64_t t) {
    bounds_ctx *b = (bounds_ctx *)c;
    int64_t i0 = t * PTS_PER_TASK, i1 = i0 + PTS_PER_TASK;
    if (i1 > b->n) i1 = b->n;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = i0; i < i1; i++)
        for (int a = 0; a < 3; a++) {
            double v = pt(b->xyz, b->is_f64, i, a);
            lo[a] = v < lo[a] ? v : lo[a];
            hi[a] = v > hi[a] ? v : hi[a];
        }
    for (int a = 0; a < 3; a++) {
        b->part[6 * t + a] = lo[a];
        b->part[6 * t + 3 + a] = hi[a];
    }
}

/* min/max of each coordinate in the input precision, widened to float64
 * (exact).  Inputs are finite (PointCloud rejects anything else). */
int orc_bounds(const void *xyz, int64_t n, int is_f64, int threads, double lo[3], double hi[3]) {
    if (n <= 0) return -1;
    int64_t nt = (n + PTS_PER_TASK - 1) / PTS_PER_TASK;
    double *part = (double *)malloc(sizeof(double) * 6 * nt);
    if (!part) return -2;
    bounds_ctx b = {xyz, n, is_f64, part};
    parallel_for(threads, nt, bounds_task, &b);
    for (int a = 0; a < 3; a++) {
        lo[a] = INFINITY;
        hi[a] = -INFINITY;
    }
    for (int64_t t = 0; t < nt; t++)
        for (int a = 0; a < 3; a++) {
            double l = part[6 * t + a], h = part[6 * t + 3 + a];
            lo[a] = l < lo[a] ? l : lo[a];
            hi[a] = h > hi[a] ? h : hi[a];
        }
    free(part);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* build (tomogram.py:147-213)                                               */

static inline uint32_t f2key(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

static inline float key2f(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
    memcpy(&f, &b, 4);
    return f;
}

#define GKEY_EMPTY 0u          /* below every float key */
#define CKEY_EMPTY 0xFFFFFFFFu /* above every float key */
#define NAN_BITS 0x7FC00000u   /* numpy's NaN */

typedef struct {
    uint32_t *g, *c;
    int64_t total;
} fill_ctx;

#define CELLS_PER_TASK (1 << 16)

static void fill_task(void *p, int64_t t) {
    fill_ctx *f = (fill_ctx *)p;
    int64_t a = t * CELLS_PER_TASK, e = a + CELLS_PER_TASK;
    if (e > f->total) e = f->total;
    for (int64_t i = a; i < e; i++) {
        f->g[i] = GKEY_EMPTY;
        f->c[i] = CKEY_EMPTY;
    }
}

typedef struct {
    const void *xyz;
    int64_t n;
    int is_f64;
    double x0, y0, r_g;
    int64_t rows, cols;
    const double *heights;
    int S;
    uint32_t *g, *c;
    int64_t bad; /* points outside the grid (cannot happen with the true bounds) */
} scatter_ctx;

static inline void atomic_max_u32(uint32_t *p, uint32_t v) {
    uint32_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
    while (v > cur && !__atomic_compare_exchange_n(p, &cur, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
}

static inline void atomic_min_u32(uint32_t *p, uint32_t v) {
    uint32_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
    while (v < cur && !__atomic_compare_exchange_n(p, &cur, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
}

static void scatter_task(void *p, int64_t t) {
    scatter_ctx *s = (scatter_ctx *)p;
    int64_t i0 = t * PTS_PER_TASK, i1 = i0 + PTS_PER_TASK;
    if (i1 > s->n) i1 = s->n;
    const int64_t ncells = s->rows * s->cols;
    int64_t bad = 0;
    for (int64_t q = i0; q < i1; q++) {
        double x = pt(s->xyz, s->is_f64, q, 0);
        double y = pt(s->xyz, s->is_f64, q, 1);
        double z = pt(s->xyz, s->is_f64, q, 2);
        /* tomogram.py:147-150: floor((y - y_min) / r_g + 0.5) in float64 */
        int64_t i = (int64_t)floor((y - s->y0) / s->r_g + 0.5);
        int64_t j = (int64_t)floor((x - s->x0) / s->r_g + 0.5);
        if (i < 0 || i >= s->rows || j < 0 || j >= s->cols) {
            bad++;
            continue;
        }
        int64_t cell = i * s->cols + j;
        /* tomogram.py:152-157: bin b = #{k : h_k < z} (z == h_k stays ground) */
        int lo = 0, hi = s->S;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (s->heights[mid] < z) lo = mid + 1;
            else hi = mid;
        }
        uint32_t key = f2key((float)z);
        if (lo < s->S) atomic_max_u32(&s->g[(int64_t)lo * ncells + cell], key);
        if (lo >= 1) atomic_min_u32(&s->c[(int64_t)(lo - 1) * ncells + cell], key);
    }
    if (bad) __atomic_fetch_add(&s->bad, bad, __ATOMIC_RELAXED);
}

typedef struct {
    uint32_t *g, *c;
    int S;
    int64_t ncells;
} fin_ctx;

#define FIN_CELLS 4096

static void finalize_task(void *p, int64_t t) {
    fin_ctx *f = (fin_ctx *)p;
    int64_t a = t * FIN_CELLS, e = a + FIN_CELLS;
    if (e > f->ncells) e = f->ncells;
    int64_t w = e - a;
    uint32_t run[FIN_CELLS];
    /* ground[k] = max over bins 0..k (reduce_pass over ground_chunks) */
    for (int64_t x = 0; x < w; x++) run[x] = GKEY_EMPTY;
    for (int k = 0; k < f->S; k++) {
        uint32_t *row = f->g + (int64_t)k * f->ncells + a;
        for (int64_t x = 0; x < w; x++) {
            uint32_t v = row[x] > run[x] ? row[x] : run[x];
            run[x] = v;
            float fv = key2f(v);
            uint32_t bits;
            memcpy(&bits, &fv, 4);
            row[x] = (v == GKEY_EMPTY || !isfinite(fv)) ? NAN_BITS : bits;
        }
    }
    /* ceiling[k] = min over bins k+1..S (ceiling_chunks, top down) */
    for (int64_t x = 0; x < w; x++) run[x] = CKEY_EMPTY;
    for (int k = f->S - 1; k >= 0; k--) {
        uint32_t *row = f->c + (int64_t)k * f->ncells + a;
        for (int64_t x = 0; x < w; x++) {
            uint32_t v = row[x] < run[x] ? row[x] : run[x];
            run[x] = v;
            float fv = key2f(v);
            uint32_t bits;
            memcpy(&bits, &fv, 4);
            row[x] = (v == CKEY_EMPTY || !isfinite(fv)) ? NAN_BITS : bits;
        }
    }
}

/* ground / ceiling stacks (S, rows, cols) float32 for the points, given the
 * frame computed on the host exactly as tomogram.py:134-145.  Returns the
 * number of points that fell outside the grid (0 for the true bounds). */
int64_t orc_build(const void *xyz, int64_t n, int is_f64, double x0, double y0, double r_g,
                  int64_t rows, int64_t cols, const double *heights, int S, float *ground,
                  float *ceiling, int threads) {
    int64_t ncells = rows * cols;
    int64_t total = ncells * (int64_t)S;
    fill_ctx fc = {(uint32_t *)ground, (uint32_t *)ceiling, total};
    parallel_for(threads, (total + CELLS_PER_TASK - 1) / CELLS_PER_TASK, fill_task, &fc);
    scatter_ctx sc = {xyz, n, is_f64, x0, y0, r_g, rows, cols, heights, S,
                      (uint32_t *)ground, (uint32_t *)ceiling, 0};
    parallel_for(threads, (n + PTS_PER_TASK - 1) / PTS_PER_TASK, scatter_task, &sc);
    fin_ctx fn = {(uint32_t *)ground, (uint32_t *)ceiling, S, ncells};
    parallel_for(threads, (ncells + FIN_CELLS - 1) / FIN_CELLS, finalize_task, &fn);
    return sc.bad;
}

/* ------------------------------------------------------------------------ */
/* evaluate (traversability.py:59-236)                                       */

typedef struct {
    double d_min, d_ref, theta_b, theta_s, theta_p, c_barrier, alpha_d, alpha_b, alpha_s;
    int32_t patch_radius;
    int32_t pad_;
} orc_params;

#define F_GENTLE 1u
#define F_PENDING 2u /* foothold branch: cost depends on the gentle window */

typedef struct {
    const float *g, *c;
    int S;
    int64_t rows, cols;
    double r_g;
    const orc_params *p;
    const float *w;
    int kside;
    float *cost;
    float *cg;      /* phase 1: ground cost / step value; phase 2: c_init */
    uint8_t *flags; /* F_GENTLE | F_PENDING per cell-slice */
    int64_t nblk;   /* row blocks per slice */
} eval_ctx;

#define ROW_BLOCK 32

static inline int fin(float v) { return isfinite(v); }

/* phase 1: slope_magnitudes (:106-114 with _axis_gradient :76-103), the
 * gentle mask (:154) and terrain_cost_values / ground_cost (:131-159) for
 * every cell whose branch does not depend on the gentle window. */
static void eval_phase1(void *q, int64_t t) {
    eval_ctx *E = (eval_ctx *)q;
    int k = (int)(t / E->nblk);
    int64_t r0 = (t % E->nblk) * ROW_BLOCK, r1 = r0 + ROW_BLOCK;
    if (r1 > E->rows) r1 = E->rows;
    const int64_t R = E->rows, Cc = E->cols, ncells = R * Cc;
    const float *g = E->g + (int64_t)k * ncells;
    float *cg = E->cg + (int64_t)k * ncells;
    uint8_t *fl = E->flags + (int64_t)k * ncells;
    const orc_params *P = E->p;
    const double r_g = E->r_g, two_rg = 2.0 * E->r_g;
    for (int64_t i = r0; i < r1; i++) {
        for (int64_t j = 0; j < Cc; j++) {
            int64_t x = i * Cc + j;
            float e = g[x];
            if (!fin(e)) { /* invalid: cost 0, not gentle (ground_cost :157-158) */
                cg[x] = 0.0f;
                fl[x] = 0;
                continue;
            }
            double ec = (double)e;
            /* axis 1 (x): neighbours j+1 / j-1, borders count as invalid */
            int vn = j + 1 < Cc && fin(g[x + 1]);
            int vp = j >= 1 && fin(g[x - 1]);
            double en = vn ? (double)g[x + 1] : 0.0, ep = vp ? (double)g[x - 1] : 0.0;
            double gx = (vn && vp) ? (en - ep) / two_rg
                      : vn         ? (en - ec) / r_g
                      : vp         ? (ec - ep) / r_g
                                   : 0.0;
            int hx = vn || vp;
            /* axis 0 (y): rows i+1 / i-1 */
            vn = i + 1 < R && fin(g[x + Cc]);
            vp = i >= 1 && fin(g[x - Cc]);
            en = vn ? (double)g[x + Cc] : 0.0;
            ep = vp ? (double)g[x - Cc] : 0.0;
            double gy = (vn && vp) ? (en - ep) / two_rg
                      : vn         ? (en - ec) / r_g
                      : vp         ? (ec - ep) / r_g
                                   : 0.0;
            int hy = vn || vp;
            double ax = fabs(gx), ay = fabs(gy);
            double m_xy = ax >= ay ? ax : ay;
            double m_grad = hypot(gx, gy);
            uint8_t f = (m_grad < P->theta_s) ? F_GENTLE : 0;
            double v;
            if (!(hx || hy)) {
                v = P->c_barrier; /* isolated (:157) */
            } else if (m_xy > P->theta_b) {
                v = P->c_barrier;
            } else if (m_grad < P->theta_s) {
                double qq = m_grad / P->theta_s;
                v = P->alpha_s * (qq * qq);
            } else {
                double qq = m_xy / P->theta_b;
                v = P->alpha_b * (qq * qq); /* kept if p_s > theta_p (phase 2) */
                f |= F_PENDING;
            }
            cg[x] = (float)v;
            fl[x] = f;
        }
    }
}

/* phase 2: gentle_fraction (:117-128) for pending cells, interval_cost
 * (:59-73) and fuse_costs (:162-170) -> c_init, in place of cg. */
static void eval_phase2(void *q, int64_t t) {
    eval_ctx *E = (eval_ctx *)q;
    int k = (int)(t / E->nblk);
    int64_t r0 = (t % E->nblk) * ROW_BLOCK, r1 = r0 + ROW_BLOCK;
    if (r1 > E->rows) r1 = E->rows;
    const int64_t R = E->rows, Cc = E->cols, ncells = R * Cc;
    const float *g = E->g + (int64_t)k * ncells;
    const float *c = E->c + (int64_t)k * ncells;
    float *cg = E->cg + (int64_t)k * ncells;
    const uint8_t *fl = E->flags + (int64_t)k * ncells;
    const orc_params *P = E->p;
    const int64_t rad = P->patch_radius;
    const double side2 = (double)((2 * rad + 1) * (2 * rad + 1));
    for (int64_t i = r0; i < r1; i++) {
        for (int64_t j = 0; j < Cc; j++) {
            int64_t x = i * Cc + j;
            float gv32 = g[x], cv32 = c[x];
            int gv = fin(gv32), cv = fin(cv32);
            float cgv = cg[x];
            if (fl[x] & F_PENDING) {
                int64_t a0 = i - rad < 0 ? 0 : i - rad, a1 = i + rad + 1 > R ? R : i + rad + 1;
                int64_t b0 = j - rad < 0 ? 0 : j - rad, b1 = j + rad + 1 > Cc ? Cc : j + rad + 1;
                int64_t cnt = 0;
                for (int64_t ii = a0; ii < a1; ii++)
                    for (int64_t jj = b0; jj < b1; jj++) cnt += fl[ii * Cc + jj] & F_GENTLE;
                double p_s = (double)cnt / side2;
                if (!(p_s > P->theta_p)) cgv = (float)P->c_barrier;
            }
            /* interval_cost */
            double d = (gv && cv) ? (double)cv32 - (double)gv32 : INFINITY;
            double adapt = P->alpha_d * (P->d_ref - d);
            if (!(adapt > 0.0)) adapt = 0.0;
            double ci = d < P->d_min ? P->c_barrier : adapt;
            if (!cv) ci = 0.0;
            if (!gv) ci = P->c_barrier;
            float ci32 = (float)ci;
            /* fuse_costs: min(c_B, f64(c_i) + f64(c_g)), invalid ground -> c_B */
            double tot = (double)ci32 + (double)cgv;
            if (P->c_barrier < tot) tot = P->c_barrier;
            if (!gv) tot = P->c_barrier;
            cg[x] = (float)tot;
        }
    }
}

/* phase 3: inflate (:205-213) = max over taps of fl32(w * c_init), zero
 * outside the map. */
static void eval_phase3(void *q, int64_t t) {
    eval_ctx *E = (eval_ctx *)q;
    int k = (int)(t / E->nblk);
    int64_t r0 = (t % E->nblk) * ROW_BLOCK, r1 = r0 + ROW_BLOCK;
    if (r1 > E->rows) r1 = E->rows;
    const int64_t R = E->rows, Cc = E->cols, ncells = R * Cc;
    const float *src = E->cg + (int64_t)k * ncells;
    float *dst = E->cost + (int64_t)k * ncells;
    const int rad = E->kside / 2;
    for (int64_t i = r0; i < r1; i++) {
        float *o = dst + i * Cc;
        for (int64_t j = 0; j < Cc; j++) o[j] = 0.0f;
        for (int dm = -rad; dm <= rad; dm++) {
            int64_t si = i + dm;
            if (si < 0 || si >= R) continue;
            const float *s = src + si * Cc;
            for (int dn = -rad; dn <= rad; dn++) {
                float wv = E->w[(dm + rad) * E->kside + (dn + rad)];
                if (!(wv > 0.0f)) continue;
                int64_t ja = dn < 0 ? -dn : 0, jb = dn > 0 ? Cc - dn : Cc;
                const float *sp = s + dn;
                for (int64_t j = ja; j < jb; j++) {
                    float v = wv * sp[j];
                    o[j] = v > o[j] ? v : o[j];
                }
            }
        }
    }
}

/* cost stack (S, rows, cols) float32 for ground / ceiling stacks. */
int orc_evaluate(const float *ground, const float *ceiling, int S, int64_t rows, int64_t cols,
                 double r_g, const orc_params *p, const float *w, int kside, float *cost,
                 int threads) {
    if (S <= 0 || rows <= 0 || cols <= 0) return 0;
    int64_t total = (int64_t)S * rows * cols;
    float *cg = (float *)malloc(sizeof(float) * total);
    uint8_t *flags = (uint8_t *)malloc(total);
    if (!cg || !flags) {
        free(cg);
        free(flags);
        return -2;
    }
    eval_ctx E = {ground, ceiling, S, rows, cols, r_g, p, w, kside, cost, cg, flags,
                  (rows + ROW_BLOCK - 1) / ROW_BLOCK};
    int64_t ntasks = (int64_t)S * E.nblk;
    parallel_for(threads, ntasks, eval_phase1, &E);
    parallel_for(threads, ntasks, eval_phase2, &E);
    parallel_for(threads, ntasks, eval_phase3, &E);
    free(cg);
    free(flags);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* simplify (simplify.py:18-73)                                              */

typedef struct {
    const float *g, *cost;
    int64_t ncells;
    int k, below, above;
    double eps;
    float cb;
    int found;
} uniq_ctx;

static void uniq_task(void *q, int64_t t) {
    uniq_ctx *U = (uniq_ctx *)q;
    if (__atomic_load_n(&U->found, __ATOMIC_RELAXED)) return;
    int64_t a = t * CELLS_PER_TASK, e = a + CELLS_PER_TASK;
    if (e > U->ncells) e = U->ncells;
    const float *g = U->g + (int64_t)U->k * U->ncells, *c = U->cost + (int64_t)U->k * U->ncells;
    const float *gb = U->below >= 0 ? U->g + (int64_t)U->below * U->ncells : NULL;
    const float *cb = U->below >= 0 ? U->cost + (int64_t)U->below * U->ncells : NULL;
    const float *ga = U->above >= 0 ? U->g + (int64_t)U->above * U->ncells : NULL;
    const float *ca = U->above >= 0 ? U->cost + (int64_t)U->above * U->ncells : NULL;
    for (int64_t x = a; x < e; x++) {
        float gv = g[x], cv = c[x];
        int valid = fin(gv);
        if (!(valid && cv < U->cb)) continue; /* trav (:36) */
        double ev = valid ? (double)gv : 0.0;
        if (gb && fin(gb[x])) { /* _side_condition(lower=True) */
            double enb = (double)gb[x];
            if (!((ev - enb > U->eps) || (cv < cb[x]))) continue;
        }
        if (ga && fin(ga[x])) { /* _side_condition(lower=False) */
            double enb = (double)ga[x];
            if (!((enb - ev > U->eps) || (cv < ca[x]))) continue;
        }
        __atomic_store_n(&U->found, 1, __ATOMIC_RELAXED);
        return;
    }
}

/* any() of _unique_mask for slice k with neighbours below / above (-1 = none) */
int orc_unique_any(const float *ground, const float *cost, int64_t ncells, int k, int below,
                   int above, double eps_e, double c_barrier, int threads) {
    uniq_ctx U = {ground, cost, ncells, k, below, above, eps_e, (float)c_barrier, 0};
    parallel_for(threads, (ncells + CELLS_PER_TASK - 1) / CELLS_PER_TASK, uniq_task, &U);
    return U.found;
}

/* the forward sweep of simplify_tomogram (:59-70): keep_out receives the
 * surviving original slice indices; returns their number. */
int orc_simplify(const float *ground, const float *cost, int S, int64_t ncells, double eps_e,
                 double c_barrier, int32_t *keep_out, int threads) {
    int n = S;
    for (int k = 0; k < S; k++) keep_out[k] = k;
    for (;;) {
        int removed = 0, pos = 0;
        while (pos < n) {
            if (n > 1) {
                int below = pos > 0 ? keep_out[pos - 1] : -1;
                int above = pos + 1 < n ? keep_out[pos + 1] : -1;
                if (!orc_unique_any(ground, cost, ncells, keep_out[pos], below, above, eps_e,
                                    c_barrier, threads)) {
                    memmove(keep_out + pos, keep_out + pos + 1, sizeof(int32_t) * (n - pos - 1));
                    n--;
                    removed = 1;
                    continue;
                }
            }
            pos++;
        }
        if (!removed) break;
    }
    return n;
}
