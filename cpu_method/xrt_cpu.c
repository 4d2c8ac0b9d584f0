/*
 * cpu_method/xrt_cpu.c -- the paper's O(N)-per-ray enumeration on the host cores (SURVEY 8(f) N3:
 * "CPU multi-core implementation of the paper's O(N)/ray enumeration (fp64) -- fair CPU baseline
 * beside the brute-force oracle").  Not the product (the product is the CUDA path) and not the
 * oracle (the oracle clips every ray against every unit): this is Algorithm 2.1 / 3.1 (P:224-235,
 * P:508-521) in its incremental form, one OpenMP thread per ray.
 *
 * Per ray, in index space (u_x = (x - x_lo)/d_x, u_y = (y_hi - y)/d_y, u_z = (z_hi - z)/d_z; units
 * are half-open [i, i+1) x [j, j+1) x [k, k+1), reading 2):
 *   * clip the line to the image box -> [t_in, t_out] (eq:condition_nonzero_3D P:433-441);
 *   * along each moving axis the ray enters successive slabs at T_a(b) = (b - u0_a) / w_a (the
 *     paper's C_x, C_y, C_z, eq:C_xC_yC_z P:446-450); walking the three crossing sequences in merged
 *     order visits exactly the units with C_low < C_up (eq:conditions_3D_1 P:460-468): for a slice of
 *     one axis the units visited inside it are the valid band of the other indices
 *     (eq:restriction_j_3D, eq:restriction_k_3D_1 P:479-499);
 *   * length l = C_up - C_low = next crossing - previous crossing (eq:range_length_3D P:503-506);
 *     units with l <= tau are dropped (reading 4).
 * Rays are given in PHYSICAL coordinates (point p, unit direction theta, |theta_a| <= 1e-12 snapped
 * to 0 by the caller).  fp64 throughout.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n[3];
    double d[3];
    double x_lo, y_hi, z_hi;
} cpu_grid;

/* walk one ray; if img != NULL return sum f * l, else the number of units */
static double walk(const cpu_grid* g, const double* p, const double* th, const float* img, double tau,
                   int64_t* count) {
    double u0[3], w[3], iw[3];
    u0[0] = (p[0] - g->x_lo) / g->d[0];
    u0[1] = (g->y_hi - p[1]) / g->d[1];
    u0[2] = (g->z_hi - p[2]) / g->d[2];
    w[0] = th[0] / g->d[0];
    w[1] = -th[1] / g->d[1];
    w[2] = -th[2] / g->d[2];
    double t_in = -INFINITY, t_out = INFINITY;
    int cell[3], moving[3];
    for (int a = 0; a < 3; ++a) {
        if (w[a] == 0.0) {
            if (!(u0[a] >= 0.0 && u0[a] < (double)g->n[a])) { *count = 0; return 0.0; }
            moving[a] = 0;
            iw[a] = 0.0;
            cell[a] = (int)floor(u0[a]);
        } else {
            moving[a] = 1;
            iw[a] = 1.0 / w[a];
            const double t0 = (0.0 - u0[a]) * iw[a], t1 = ((double)g->n[a] - u0[a]) * iw[a];
            t_in = fmax(t_in, fmin(t0, t1));
            t_out = fmin(t_out, fmax(t0, t1));
        }
    }
    if (!(t_out - t_in > tau)) { *count = 0; return 0.0; }
    double T[3];
    int bnd[3], sgn[3];
    for (int a = 0; a < 3; ++a) {
        if (!moving[a]) { T[a] = INFINITY; bnd[a] = 0; sgn[a] = 0; continue; }
        const int64_t N = g->n[a];
        int c = (int)floor(u0[a] + t_in * w[a]);
        c = c < 0 ? 0 : (c > N - 1 ? (int)N - 1 : c);
        /* entry cell consistent with the crossing values T(b) = (b - u0) / w */
        if (w[a] > 0.0) {
            if (c + 1 <= N - 1 && ((double)(c + 1) - u0[a]) * iw[a] <= t_in) c += 1;
            else if (c >= 1 && ((double)c - u0[a]) * iw[a] > t_in) c -= 1;
        } else {
            if (c >= 1 && ((double)c - u0[a]) * iw[a] <= t_in) c -= 1;
            else if (c + 1 <= N - 1 && ((double)(c + 1) - u0[a]) * iw[a] > t_in) c += 1;
        }
        cell[a] = c;
        sgn[a] = w[a] > 0.0 ? 1 : -1;
        bnd[a] = sgn[a] > 0 ? c + 1 : c;
        T[a] = ((double)bnd[a] - u0[a]) * iw[a];
    }
    double t = t_in, acc = 0.0;
    int64_t n = 0;
    const int64_t budget = 2 + g->n[0] + g->n[1] + g->n[2];
    for (int64_t it = 0; it < budget; ++it) {
        const double tn = fmin(fmin(T[0], T[1]), fmin(T[2], t_out));
        const double l = tn - t;
        if (l > tau) {
            ++n;
            if (img) acc += (double)img[((int64_t)cell[2] * g->n[1] + cell[1]) * g->n[0] + cell[0]] * l;
        }
        if (tn >= t_out) break;
        const int a = (tn == T[0]) ? 0 : ((tn == T[1]) ? 1 : 2);
        cell[a] += sgn[a];
        bnd[a] += sgn[a];
        T[a] = ((double)bnd[a] - u0[a]) * iw[a];
        t = tn;
    }
    *count = n;
    return acc;
}

/* forward: out[m] = sum_I img[I] l_I(ray m); counts (may be NULL) = |units of ray m| */
void xrt_cpu_forward(const cpu_grid* g, int64_t n_rays, const double* p, const double* th,
                     const float* img, double tau, double* out, int64_t* counts) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t m = 0; m < n_rays; ++m) {
        int64_t c = 0;
        out[m] = walk(g, p + 3 * m, th + 3 * m, img, tau, &c);
        if (counts) counts[m] = c;
    }
}

int xrt_cpu_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
