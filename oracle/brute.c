/*
 * oracle/brute.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 brute-force X-ray transform of a unit-basis image: every ray is
 * clipped against EVERY unit box (Liang-Barsky / slab test).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code with paper_2006_00686_b200/ (the product).
 *
 * What it computes (the plain definition the paper's method reaches exactly):
 *   * Eq. (1.4):   (A f)(ray) = sum_I f_I * l_I(ray)
 *   * l_I = the length of the ray inside the unit Omega_I, eq:intersection_length
 *     P:153-156 (2D) and eq:intersection_length_3D P:429-432 (3D), i.e. the length of
 *     the t-range satisfying eq:condition_nonzero P:157-164 / eq:condition_nonzero_3D
 *     per axis one slab inequality, intersected over the axes
 *     (C_low = max of the lower ends, C_up = min of the upper ends, l = C_up - C_low,
 *     eq:conditions_2D_1 P:180-187, eq:range_length P:217-220).
 *   * The row of the projection matrix = {(I, l_I) : l_I > tau}, in ascending
 *     flat index I = (k*N_y + j)*N_x + i (reading 1).
 *   * adjoint = transpose product.
 *
 * Frame (readings 2-4): the caller hands rays in PHYSICAL coordinates
 * (point p, unit direction theta, already snapped |theta_a| <= 1e-12 -> 0).  Per axis
 * the index-space coordinate is u_x = (x - x_lo)/d_x, u_y = (y_hi - y)/d_y,
 * u_z = (z_hi - z)/d_z, so that unit (i,j,k) = [i,i+1] x [j,j+1] x [k,k+1]
 * (the paper's Omega_ji P:151 / Omega_kji P:427 with j running down y and k down z).
 *   * axis with theta_a != 0: slab t-interval [(c - u0)/w, (c + 1 - u0)/w], ordered;
 *   * axis with theta_a == 0: the ray is inside slab c iff c <= u0 < c + 1 (half-open:
 *     the paper's "bigger 1D index" tie-break, reading 2);
 *   * emit iff l > tau (strict condition C_low < C_up, reading 4).
 * t is the physical arc length along theta, so l is in physical units (reading 14).
 *
 * mode 0 = full brute force: all N_x*N_y*N_z boxes per ray.
 * mode 1 = separable early-out: a (k, j) pair whose z/y-interval overlap is <= tau is
 *          skipped before the i loop.  Identical output (the full overlap of such a box
 *          is <= that partial overlap <= tau, so mode 0 drops it too); tested equal.
 * mode 2 = mode 1, and the i loop visits only the cells whose x-slab can meet the (k, j)
 *          overlap [lo, hi]: floor(u_x(lo)) - 1 .. floor(u_x(hi)) + 1 (the slab intervals are
 *          monotone in i; the margin of one cell absorbs rounding).  A skipped box has an
 *          x-interval disjoint from [lo, hi], i.e. l <= 0, so mode 0 drops it too; tested equal.
 *          (Used for the full-sinogram sweeps of the 2D fan beam, SURVEY 8(c) reading 21.)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n[3];     /* N_x, N_y, N_z */
    double d[3];      /* d_x, d_y, d_z */
    double x_lo, y_hi, z_hi;
} oracle_grid;

/* index-space origin u0 and velocity w of a physical ray p + t*theta */
static void to_index_space(const oracle_grid* g, const double* p, const double* th,
                           double* u0, double* w) {
    u0[0] = (p[0] - g->x_lo) / g->d[0];
    u0[1] = (g->y_hi - p[1]) / g->d[1];
    u0[2] = (g->z_hi - p[2]) / g->d[2];
    w[0] = th[0] / g->d[0];
    w[1] = -th[1] / g->d[1];
    w[2] = -th[2] / g->d[2];
}

/* slab t-interval of cell c on one axis; returns 0 when the ray never enters it */
static int slab(double u0, double w, int64_t c, double* lo, double* hi) {
    if (w == 0.0) {
        if ((double)c <= u0 && u0 < (double)(c + 1)) {
            *lo = -INFINITY;
            *hi = INFINITY;
            return 1;
        }
        return 0;
    }
    double t0 = ((double)c - u0) / w;
    double t1 = ((double)(c + 1) - u0) / w;
    if (t0 <= t1) { *lo = t0; *hi = t1; } else { *lo = t1; *hi = t0; }
    return 1;
}

typedef struct {
    double* lo[3];
    double* hi[3];
    char* ok[3];
} axis_tab;

static int tab_alloc(axis_tab* T, const oracle_grid* g) {
    for (int a = 0; a < 3; ++a) {
        T->lo[a] = (double*)malloc(sizeof(double) * (size_t)g->n[a]);
        T->hi[a] = (double*)malloc(sizeof(double) * (size_t)g->n[a]);
        T->ok[a] = (char*)malloc((size_t)g->n[a]);
        if (!T->lo[a] || !T->hi[a] || !T->ok[a]) return 0;
    }
    return 1;
}

static void tab_free(axis_tab* T) {
    for (int a = 0; a < 3; ++a) { free(T->lo[a]); free(T->hi[a]); free(T->ok[a]); }
}

/* Visit every unit box of one ray; call emit(I, l) for l > tau, in ascending I. */
typedef void (*emit_fn)(void* ctx, int64_t I, double l);

static void ray_row(const oracle_grid* g, const double* p, const double* th, double tau,
                    int mode, axis_tab* T, emit_fn emit, void* ctx) {
    double u0[3], w[3];
    to_index_space(g, p, th, u0, w);
    for (int a = 0; a < 3; ++a)
        for (int64_t c = 0; c < g->n[a]; ++c)
            T->ok[a][c] = (char)slab(u0[a], w[a], c, &T->lo[a][c], &T->hi[a][c]);
    const int64_t nx = g->n[0], ny = g->n[1], nz = g->n[2];
    for (int64_t k = 0; k < nz; ++k) {
        if (!T->ok[2][k]) continue;
        for (int64_t j = 0; j < ny; ++j) {
            if (!T->ok[1][j]) continue;
            double lo_kj = fmax(T->lo[2][k], T->lo[1][j]);
            double hi_kj = fmin(T->hi[2][k], T->hi[1][j]);
            if (mode >= 1 && !(hi_kj - lo_kj > tau)) continue;
            int64_t i0 = 0, i1 = nx;
            if (mode == 2) {
                if (w[0] == 0.0) {
                    i0 = (int64_t)floor(u0[0]) - 1;
                    i1 = i0 + 3;
                } else {
                    /* (lo, hi) may be infinite when the y and z axes are both fixed */
                    const double lim = (double)nx + 4.0;
                    const double ua = fmin(fmax(u0[0] + w[0] * lo_kj, -4.0), lim);
                    const double ub = fmin(fmax(u0[0] + w[0] * hi_kj, -4.0), lim);
                    i0 = (int64_t)floor(fmin(ua, ub)) - 1;
                    i1 = (int64_t)floor(fmax(ua, ub)) + 2;
                }
                if (i0 < 0) i0 = 0;
                if (i1 > nx) i1 = nx;
            }
            for (int64_t i = i0; i < i1; ++i) {
                if (!T->ok[0][i]) continue;
                double c_low = fmax(lo_kj, T->lo[0][i]);
                double c_up = fmin(hi_kj, T->hi[0][i]);
                double l = c_up - c_low;
                if (l > tau) emit(ctx, (k * ny + j) * nx + i, l);
            }
        }
    }
}

/* ---- emitters ---------------------------------------------------------------- */
typedef struct { int64_t n; } cnt_ctx;
static void emit_count(void* c, int64_t I, double l) { (void)I; (void)l; ((cnt_ctx*)c)->n++; }

typedef struct { int64_t pos; int64_t* cols; double* lens; } fill_ctx;
static void emit_fill(void* c, int64_t I, double l) {
    fill_ctx* f = (fill_ctx*)c;
    f->cols[f->pos] = I;
    f->lens[f->pos] = l;
    f->pos++;
}

typedef struct { const float* img; double acc; } fwd_ctx;
static void emit_fwd(void* c, int64_t I, double l) {
    fwd_ctx* f = (fwd_ctx*)c;
    f->acc += (double)f->img[I] * l;
}

typedef struct { double y; double* img; } adj_ctx;
static void emit_adj(void* c, int64_t I, double l) {
    adj_ctx* a = (adj_ctx*)c;
    double v = a->y * l;
#ifdef _OPENMP
#pragma omp atomic
#endif
    a->img[I] += v;
}

/* ---- exported API (ctypes) ----------------------------------------------------- */

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* counts[m] = |row m| */
int oracle_count(const oracle_grid* g, int64_t nr, const double* p, const double* th,
                 double tau, int mode, int64_t* counts) {
    int fail = 0;
#pragma omp parallel
    {
        axis_tab T;
        if (!tab_alloc(&T, g)) fail = 1;
        else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t m = 0; m < nr; ++m) {
                cnt_ctx c = {0};
                ray_row(g, p + 3 * m, th + 3 * m, tau, mode, &T, emit_count, &c);
                counts[m] = c.n;
            }
        }
        tab_free(&T);
    }
    return fail ? -1 : 0;
}

/* CSR fill: row m occupies [row_ptr[m], row_ptr[m+1]) of cols / lens */
int oracle_fill(const oracle_grid* g, int64_t nr, const double* p, const double* th,
                double tau, int mode, const int64_t* row_ptr, int64_t* cols, double* lens) {
    int fail = 0;
#pragma omp parallel
    {
        axis_tab T;
        if (!tab_alloc(&T, g)) fail = 1;
        else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t m = 0; m < nr; ++m) {
                fill_ctx c = {row_ptr[m], cols, lens};
                ray_row(g, p + 3 * m, th + 3 * m, tau, mode, &T, emit_fill, &c);
            }
        }
        tab_free(&T);
    }
    return fail ? -1 : 0;
}

/* out[m] = sum_I img[I] * l_I(ray m), fp64 accumulation in ascending I */
int oracle_forward(const oracle_grid* g, int64_t nr, const double* p, const double* th,
                   double tau, int mode, const float* img, double* out) {
    int fail = 0;
#pragma omp parallel
    {
        axis_tab T;
        if (!tab_alloc(&T, g)) fail = 1;
        else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t m = 0; m < nr; ++m) {
                fwd_ctx c = {img, 0.0};
                ray_row(g, p + 3 * m, th + 3 * m, tau, mode, &T, emit_fwd, &c);
                out[m] = c.acc;
            }
        }
        tab_free(&T);
    }
    return fail ? -1 : 0;
}

/* img[I] += sum_m y[m] * l_I(ray m)  (img is NOT cleared; fp64) */
int oracle_adjoint(const oracle_grid* g, int64_t nr, const double* p, const double* th,
                   double tau, int mode, const double* y, double* img) {
    int fail = 0;
#pragma omp parallel
    {
        axis_tab T;
        if (!tab_alloc(&T, g)) fail = 1;
        else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t m = 0; m < nr; ++m) {
                if (y[m] == 0.0) continue;
                adj_ctx c = {y[m], img};
                ray_row(g, p + 3 * m, th + 3 * m, tau, mode, &T, emit_adj, &c);
            }
        }
        tab_free(&T);
    }
    return fail ? -1 : 0;
}
