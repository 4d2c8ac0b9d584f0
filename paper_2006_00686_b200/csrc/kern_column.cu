// kern_column.cu -- one warp per detector column: the paper's Algorithm 3.1 split between the
// warp (shared in-plane band) and its lanes (per-row z band).  3D beams only (par3d, cone,
// helical): every ray of a detector column has the same projection onto the xy plane
// (equispaced flat detector: alpha depends on the column only, so phi1 = phi1' + alpha and
// s1 = D sin(alpha) are shared; par3d: phi1 and s1 per column).
//
// Per column (warp-cooperative, lane = one major-axis slice i):
//   slice i of the major in-plane axis spans sigma in [T_a(i), T_a(i+1)]; the valid band of the
//   minor in-plane index inside it is one or two cells (eq:restriction_j_3D: the
//   band C_1 - tan(phi1) - 1 < j < C_1 has width <= 2 when |tan| <= 1), split at the minor
//   crossing.  The (cell, sigma_start, d_sigma) segments go to shared memory in path order;
//   d_sigma = C_up - C_low of the in-plane unit (eq:range_length P:217-220), in units of the
//   in-plane arc length sigma.
// Per ray (lane = one detector row):
//   z(sigma) is linear along the shared path, so inside an in-plane segment the valid k band
//   (eq:restriction_k_3D_1) is {k_s, k_e}: the cell at the segment's start and, if
//   the ray's next z-plane crossing tau falls inside the segment, the next cell k_s + dk (at most
//   one plane per segment, checked at plan time).  The lengths are C_up - C_low of the two units
//   (eq:range_length_3D): l_e = max(sigma_e - tau, 0), l_s = d_sigma - l_e.  The
//   crossing values tau_m = t0z + m dtz are evaluated in sigma (well conditioned also for rays
//   almost parallel to the z planes) and shared by the two units they separate.  The loop is
//   branch-free (predicated); the volume copy is zero-padded in z so a ray outside the z slab
//   (before entry / after exit through a z face) reads zeros -- the z faces are ordinary
//   crossings.  The physical length is d sigma / cos(beta) (|theta_xy| = cos beta), applied once
//   per ray.
//
// Memory: the kernels read / accumulate a z-FASTEST, z-padded copy of the volume
// (work[(j * N_x + i) * NzP + pad + k]), so the 32 lanes of a warp (adjacent detector rows ->
// adjacent k) touch consecutive addresses; transposes to / from the caller's [k][j][i] image
// run inside xrt_forward / xrt_adjoint.
//
// CTA = kWarps adjacent detector columns of one view x one band of 64 NP detector rows (warp =
// column, 2 NP rays per lane) x one xy tile.  1D grid, band-major: blockIdx = band * n_items + item,
// items = (view, column group, tile) sorted by tile (plan time, build_column_items), so every view
// and column crossing one tile of one band's z slab runs while that slab is L2-resident.  Tiling
// and rays per lane are chosen per operator (capi.cu).
//
// Operators (template kOp): 0 forward, 1 adjoint (red.global.add), 2 / 3 the attenuated forward /
// adjoint of the SPECT weight (DESIGN reading 23; untiled).  Also here: the
// voxel-driven gather adjoint (k_gather, XRT_ALGO_GATHER) and the z-fastest transposes.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "xrt_internal.cuh"

namespace xrt {

namespace {

#ifndef XRT_COL_WARPS
#define XRT_COL_WARPS 4   // measured: 4 columns per CTA 0.5-2 % faster than 8 on cfg 3 / 4 / 5, 2 slower
#endif
constexpr int kWarps = XRT_COL_WARPS;  // warps per CTA = adjacent detector columns per CTA (one per warp)
// CTA of the (f, delta f) forward: kFdCols adjacent columns x kFdViews adjacent views, one warp each.
// Neighbouring views' columns cross nearly the same cells, so the CTA's warps share L1 lines: the
// compulsory L2 -> L1 traffic per ray-segment of cfg 4 falls from ~5.7 B (4 columns x 1 view) to
// ~3.4 B (4 x 2) and ~2.5 B (4 x 4) (scratch estimate).
#ifndef XRT_FD_COLS
#define XRT_FD_COLS 4
#endif
#ifndef XRT_FD_VIEWS
#define XRT_FD_VIEWS 1   // with the z-mirror forward (cfg 4): 4 x 1 100.4 ms vs 4 x 2 104.2, 4 x 4 106.7, 8 x 1 102.6
#endif
constexpr int kFdCols = XRT_FD_COLS, kFdViews = XRT_FD_VIEWS, kFdWarps = kFdCols * kFdViews;
#ifndef XRT_KPASSES
#define XRT_KPASSES 4
#endif
constexpr int kPasses = XRT_KPASSES; // 32-slice path-generation passes per chunk (chunk = 128 major slices)
#ifndef XRT_FWD2_SHORT_CHUNK
#define XRT_FWD2_SHORT_CHUNK 1
#endif

struct __align__(16) Seg {
    unsigned long long ptr;  // address of (cell, padded k = 0) in the z-fastest volume
    float se;                // sigma at the segment end
    float ds;                // segment length in sigma (C_up - C_low in the plane)
};

struct ColumnPath {
    bool hit;
    float L;          // sigma length of the in-plane chord (end of the last segment)
    int a;            // major in-plane axis (0 = x, 1 = y)
    int n_slices;     // number of major-axis slices inside (0, L)
    float t0a, dta;   // major crossings: T_a(m) = t0a + m * dta
    float t0b, dtb;   // minor crossings (INF if the minor axis is fixed)
    int cell_a0, step_a;   // major cell of slice 0 and its step (+-1)
    int cell_b0, step_b;   // minor cell at the entry and its step
    int nb_face;      // number of interior minor crossings
    float idtb;       // 1 / dtb (estimate only; decisions use the fmaf crossing values)
    int sa, sb;       // flat xy strides of the major / minor axis
    double sig_in;    // absolute sigma of the square entry (fp64)
    double ux0, uy0;  // in-plane index coordinates at sigma_rel = 0 (the square entry)
    double wx, wy;    // d u / d sigma
};

// fp64 in-plane line of the column (the paper's per-column parameters), u = detector coordinate.
__host__ __device__ __forceinline__ void column_line(const ViewRec& V, const DetC& dc, int c, double& qx,
                                            double& qy, double& ex, double& ey, double& ca_out) {
    const double u = ((double)c - dc.cu) * dc.du + dc.off_u;
    if (dc.beam == XRT_PAR3D) {
        // xy line of (s1, phi1): foot s1 theta_1, direction (cos phi1, sin phi1)
        ex = V.c1; ey = V.s1;
        qx = -u * V.s1; qy = u * V.c1;
        ca_out = 1.0;
    } else {
        const double D = dc.D;
        double ca, sa;
        if (dc.curved) {                                 // equiangular column: alpha = u / sdd
            ca = cos(u / dc.sdd); sa = sin(u / dc.sdd);
        } else {
            const double t = u * D / dc.sdd;
            const double sq = sqrt(D * D + t * t);
            ca = D / sq; sa = t / sq;                    // alpha = arctan(t / D)
        }
        const double s1 = D * sa;
        const double c1 = V.c1 * ca - V.s1 * sa;         // phi1 = phi1' + alpha
        const double n1 = V.s1 * ca + V.c1 * sa;
        ex = c1; ey = n1;
        qx = -s1 * n1; qy = s1 * c1;
        ca_out = ca;
    }
    if (fabs(ex) <= kSnap) ex = 0.0;
    if (fabs(ey) <= kSnap) ey = 0.0;
}

__device__ __forceinline__ int entry_cell(double u0, double w, double s_in, int N) {
    const double iw = 1.0 / w;
    int cc = (int)floor(u0 + s_in * w);
    cc = cc < 0 ? 0 : (cc > N - 1 ? N - 1 : cc);
    if (w > 0.0) {
        if (cc + 1 <= N - 1 && ((double)(cc + 1) - u0) * iw <= s_in) cc += 1;
        else if (cc >= 1 && ((double)cc - u0) * iw > s_in) cc -= 1;
    } else {
        if (cc >= 1 && ((double)cc - u0) * iw <= s_in) cc -= 1;
        else if (cc + 1 <= N - 1 && ((double)(cc + 1) - u0) * iw > s_in) cc += 1;
    }
    return cc;
}

// fp32 description of one column's in-plane path (computed redundantly by every lane).
__device__ __forceinline__ void column_path(const ViewRec& V, const DetC& dc, const GridC& g,
                                            int c, ColumnPath& P, double& ca) {
    double qx, qy, ex, ey;
    column_line(V, dc, c, qx, qy, ex, ey, ca);
    const double ux = (qx - g.x_lo) / g.d[0], uy = (g.y_hi - qy) / g.d[1];
    const double wx = ex / g.d[0], wy = -ey / g.d[1];
    double s_in = -INFINITY, s_out = INFINITY;
    P.hit = true;
    if (wx == 0.0) {
        if (!(ux >= 0.0 && ux < (double)g.n[0])) P.hit = false;
    } else {
        const double iw = 1.0 / wx;
        const double t0 = (0.0 - ux) * iw, t1 = ((double)g.n[0] - ux) * iw;
        s_in = fmax(s_in, fmin(t0, t1));
        s_out = fmin(s_out, fmax(t0, t1));
    }
    if (wy == 0.0) {
        if (!(uy >= 0.0 && uy < (double)g.n[1])) P.hit = false;
    } else {
        const double iw = 1.0 / wy;
        const double t0 = (0.0 - uy) * iw, t1 = ((double)g.n[1] - uy) * iw;
        s_in = fmax(s_in, fmin(t0, t1));
        s_out = fmin(s_out, fmax(t0, t1));
    }
    if (!P.hit || !(s_out - s_in > 0.0)) { P.hit = false; P.n_slices = 0; P.L = 0.f; return; }
    P.sig_in = s_in;
    P.ux0 = ux + s_in * wx;
    P.uy0 = uy + s_in * wy;
    P.wx = wx;
    P.wy = wy;
    const int cx = wx == 0.0 ? (int)floor(ux) : entry_cell(ux, wx, s_in, g.n[0]);
    const int cy = wy == 0.0 ? (int)floor(uy) : entry_cell(uy, wy, s_in, g.n[1]);
    // major axis: the one crossed most often per unit sigma
    const int a = fabs(wx) >= fabs(wy) ? 0 : 1;
    P.a = a;
    const double wa = a == 0 ? wx : wy, wb = a == 0 ? wy : wx;
    const double ua = a == 0 ? ux : uy, ub = a == 0 ? uy : ux;
    const int na = a == 0 ? g.n[0] : g.n[1], nb = a == 0 ? g.n[1] : g.n[0];
    const int cella = a == 0 ? cx : cy, cellb = a == 0 ? cy : cx;
    float L = (float)(s_out - s_in);
    int ma_face;
    {
        const double iw = 1.0 / wa;
        const int pos = wa > 0.0;
        const int bf = pos ? cella + 1 : cella;
        ma_face = pos ? (na - bf) : bf;
        P.t0a = (float)(((double)bf - ua) * iw - s_in);
        P.dta = (float)fabs(iw);
        P.step_a = pos ? 1 : -1;
        P.cell_a0 = cella;
        L = fminf(L, fmaf((float)ma_face, P.dta, P.t0a));
    }
    if (wb != 0.0) {
        const double iw = 1.0 / wb;
        const int pos = wb > 0.0;
        const int bf = pos ? cellb + 1 : cellb;
        const int m_face = pos ? (nb - bf) : bf;
        P.t0b = (float)(((double)bf - ub) * iw - s_in);
        P.dtb = (float)fabs(iw);
        P.step_b = pos ? 1 : -1;
        P.nb_face = m_face;
        L = fminf(L, fmaf((float)m_face, P.dtb, P.t0b));
    } else {
        P.t0b = INFINITY;
        P.dtb = 0.f;
        P.step_b = 0;
        P.nb_face = 0;
    }
    P.cell_b0 = cellb;
    P.L = L;
    P.idtb = P.step_b != 0 ? 1.f / P.dtb : 0.f;
    P.sa = a == 0 ? 1 : g.n[0];
    P.sb = a == 0 ? g.n[0] : 1;
    // slices = 1 + number of major crossings strictly inside (0, L)
    const float est = (L - P.t0a) / P.dta;
    int m = est < 0.f ? 0 : (est > (float)ma_face ? ma_face : (int)est);
    while (m < ma_face && fmaf((float)m, P.dta, P.t0a) < L) ++m;
    while (m > 0 && !(fmaf((float)(m - 1), P.dta, P.t0a) < L)) --m;
    P.n_slices = m + 1;
}

// Segments of major slice n: 1 or 2 in-plane units (cell, sigma_start, sigma_end), keeping only
// those whose cell lies in the tile [ti0, ti1) x [tj0, tj1).  The minor crossings at or before the
// slice start are counted against the SAME fmaf expression the neighbouring slices use, so every
// crossing value is produced exactly once (telescoping, also across tiles).
__device__ __forceinline__ int slice_segments(const ColumnPath& P, int n, int ti0, int ti1, int tj0,
                                              int tj1, float& e0s, float& e0e, int& e0c, float& e1s,
                                              float& e1e, int& e1c) {
    const float t_lo = n == 0 ? 0.f : fminf(fmaf((float)(n - 1), P.dta, P.t0a), P.L);
    const float t_hi = n + 1 >= P.n_slices ? P.L : fminf(fmaf((float)n, P.dta, P.t0a), P.L);
    const int ca = P.cell_a0 + P.step_a * n;
    int mb = 0;
    bool split = false;
    float tb = 0.f;
    if (P.step_b != 0) {
        // estimate (exact up to one step), then one fix-up step each way
        int m = __float2int_rd((t_lo - P.t0b) * P.idtb) + 1;
        m = max(0, min(m, P.nb_face));
        if (m < P.nb_face && fmaf((float)m, P.dtb, P.t0b) <= t_lo) ++m;
        if (m > 0 && fmaf((float)(m - 1), P.dtb, P.t0b) > t_lo) --m;
        mb = m;
        tb = fmaf((float)m, P.dtb, P.t0b);
        split = m < P.nb_face && tb < t_hi;
    }
    const int cb0 = P.cell_b0 + P.step_b * mb;
    const int cb1 = split ? cb0 + P.step_b : cb0;
    const int ii = P.a == 0 ? ca : cb0, jj0 = P.a == 0 ? cb0 : ca;
    const bool a_in = P.a == 0 ? (ca >= ti0 && ca < ti1) : (ca >= tj0 && ca < tj1);
    const bool b0_in = P.a == 0 ? (cb0 >= tj0 && cb0 < tj1) : (cb0 >= ti0 && cb0 < ti1);
    const bool b1_in = P.a == 0 ? (cb1 >= tj0 && cb1 < tj1) : (cb1 >= ti0 && cb1 < ti1);
    (void)ii; (void)jj0;
    const int c0 = ca * P.sa + cb0 * P.sb;
    const int c1 = ca * P.sa + cb1 * P.sb;
    const float m1 = split ? tb : t_hi;
    int cnt = 0;
    if (a_in && b0_in) { e0s = t_lo; e0e = m1; e0c = c0; cnt = 1; }
    if (split && a_in && b1_in) {
        if (cnt == 0) { e0s = tb; e0e = t_hi; e0c = c1; }
        else { e1s = tb; e1e = t_hi; e1c = c1; }
        ++cnt;
    }
    return cnt;
}

// Per-(view, column) path descriptor: the in-plane path (fp32 crossing sequences, cells) and the
// fp64 terms the per-ray z setup needs.  Depends on the geometry only: built once at plan creation
// (k_col_desc) instead of by every warp of every band and tile.
struct __align__(16) ColDesc {
    float L, t0a, dta, t0b;
    float dtb, idtb;
    int n_slices, flags;              // flags: bit0 hit, bit1 major axis (0 = x, 1 = y)
    int cell_a0, cell_b0, nb_face, steps;  // steps: (step_a + 1) | (step_b + 1) << 2
    float ux0, uy0, wx, wy;           // in-plane index coordinates at sigma = 0 and d/dsigma (tile clip)
    double sig_in, ca;                // absolute sigma of the square entry; cos(alpha) of the column
};

__global__ void k_col_desc(const ViewRec* __restrict__ views, DetC dc, GridC g, int64_t n,
                           ColDesc* __restrict__ out) {
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const int v = (int)(id / dc.cols), c = (int)(id - (int64_t)v * dc.cols);
    ColumnPath P;
    double ca;
    column_path(views[v], dc, g, c, P, ca);
    ColDesc d;
    d.L = P.L; d.t0a = P.t0a; d.dta = P.dta; d.t0b = P.t0b; d.dtb = P.dtb; d.idtb = P.idtb;
    d.n_slices = P.hit ? P.n_slices : 0;
    d.flags = (P.hit ? 1 : 0) | (P.a << 1);
    d.cell_a0 = P.cell_a0; d.cell_b0 = P.cell_b0; d.nb_face = P.nb_face;
    d.steps = (P.step_a + 1) | ((P.step_b + 1) << 2);
    d.ux0 = (float)P.ux0; d.uy0 = (float)P.uy0; d.wx = (float)P.wx; d.wy = (float)P.wy;
    d.sig_in = P.sig_in;
    d.ca = ca;
    out[id] = d;
}

__device__ __forceinline__ void load_path(const ColDesc* __restrict__ dsc, int nx, ColumnPath& P,
                                          double& ca, float& ux0, float& uy0, float& wx, float& wy) {
    const float4 q0 = __ldg(reinterpret_cast<const float4*>(dsc) + 0);
    const float4 q1 = __ldg(reinterpret_cast<const float4*>(dsc) + 1);
    const int4 q2 = __ldg(reinterpret_cast<const int4*>(dsc) + 2);
    const float4 q3 = __ldg(reinterpret_cast<const float4*>(dsc) + 3);
    const double2 q4 = __ldg(reinterpret_cast<const double2*>(dsc) + 4);
    P.L = q0.x; P.t0a = q0.y; P.dta = q0.z; P.t0b = q0.w;
    P.dtb = q1.x; P.idtb = q1.y;
    P.n_slices = __float_as_int(q1.z);
    const int flags = __float_as_int(q1.w);
    P.hit = flags & 1;
    P.a = (flags >> 1) & 1;
    P.cell_a0 = q2.x; P.cell_b0 = q2.y; P.nb_face = q2.z;
    P.step_a = (q2.w & 3) - 1;
    P.step_b = ((q2.w >> 2) & 3) - 1;
    P.sa = P.a == 0 ? 1 : nx;
    P.sb = P.a == 0 ? nx : 1;
    ux0 = q3.x; uy0 = q3.y; wx = q3.z; wy = q3.w;
    P.sig_in = q4.x;
    ca = q4.y;
}

// The in-plane fields slice_segments reads, re-read per chunk from the (L1-resident) descriptor with
// volatile loads: not hoisted, so they do not stay live across the walk (at 64 registers they were
// spilled to local memory and written back to L2 every chunk).
__device__ __forceinline__ void load_path_chunk(const ColDesc* __restrict__ dsc, int nx, ColumnPath& P) {
    unsigned a0, a1, a2, a3, b0, b1, b2, b3, c0, c1, c2, c3;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "l"(dsc));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4+16];" : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "l"(dsc));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4+32];" : "=r"(c0), "=r"(c1), "=r"(c2), "=r"(c3) : "l"(dsc));
    P.L = __uint_as_float(a0); P.t0a = __uint_as_float(a1); P.dta = __uint_as_float(a2); P.t0b = __uint_as_float(a3);
    P.dtb = __uint_as_float(b0); P.idtb = __uint_as_float(b1);
    P.n_slices = (int)b2;
    P.hit = b3 & 1;
    P.a = (b3 >> 1) & 1;
    P.cell_a0 = (int)c0; P.cell_b0 = (int)c1; P.nb_face = (int)c2;
    P.step_a = (int)(c3 & 3) - 1;
    P.step_b = (int)((c3 >> 2) & 3) - 1;
    P.sa = P.a == 0 ? 1 : nx;
    P.sb = P.a == 0 ? nx : 1;
}

// Per-ray z description along the shared path (sigma from the square entry): the z cell at the
// square entry and the z-plane crossings tau_m = t0z + m dtz, evaluated in sigma (well conditioned
// also for rays almost parallel to the z planes).
struct RayZ {
    bool active;      // ray exists (row in range) and the column hits the square
    int kp;           // padded z index (k + pad) of the cell at sigma = 0
    int dk;           // +1 / -1 per z-plane crossing, 0 when z is fixed
    float t0z, dtz;   // z-plane crossings tau_m = t0z + m dtz (INF when fixed)
    float scale;      // 1 / cos(beta): physical length per unit sigma
};

__device__ __forceinline__ void ray_z(const ViewRec& V, const DetC& dc, const GridC& g,
                                      const ColumnPath& P, double ca, int r, int pad, RayZ& Z) {
    Z.active = false;
    Z.kp = pad; Z.dk = 0; Z.t0z = INFINITY; Z.dtz = 0.f; Z.scale = 1.f;
    if (r >= dc.rows || !P.hit) return;
    const double v = ((double)r - dc.cv) * dc.dv + dc.off_v;
    double tb, z0;  // tan(beta), z at absolute sigma 0
    if (dc.beam == XRT_PAR3D) {
        // z(sigma) = s2 / cos(phi2) + sigma tan(phi2), sigma = t cos(phi2) - s2 sin(phi2)
        if (fabs(V.s2) <= kSnap) { tb = 0.0; z0 = v * V.c2; }
        else { tb = V.pad[0]; z0 = v * V.pad[1]; }      // tan(phi2), 1 / cos(phi2) (plan)
    } else {
        if (dc.curved) {
            // cylindrical detector: tan(beta) = v / sdd, z(sigma=0) = s2 / cos(beta) = D cos(alpha)
            // tan(beta) + H  (P:622, P:654 divided by cos(beta))
            tb = v / dc.sdd;
            z0 = dc.D * ca * tb + V.H;
        } else {
            // tan(beta) = h / sqrt(D^2 + t^2) = h cos(alpha) / D, z(sigma=0) = s2 / cos(beta) = h cos^2
            // (alpha) + H  (P:636, P:660 divided by cos(beta))
            const double h = v * dc.D / dc.sdd;
            tb = h * ca * dc.inv_D;
            z0 = h * (ca * ca) + V.H;
        }
        if (fabs(tb) <= kSnap) tb = 0.0;
    }
    Z.scale = sqrtf(1.f + (float)(tb * tb));           // 1 / cos(beta)
    if (tb == 0.0) {
        // fixed z: the half-open cell floor(u0); rays outside the slab read padding
        double kk = floor((g.z_hi - z0) / g.d[2]);
        kk = fmin(fmax(kk, (double)(-pad)), (double)(g.n[2] + pad - 1));
        Z.kp = (int)kk + pad;
    } else {
        const double uz0 = (g.z_hi - (z0 + P.sig_in * tb)) * g.inv_dz;   // u_z at sigma = 0
        const double iw = -g.d[2] * __drcp_rn(tb);                          // 1 / (d u_z / d sigma)
        double kk = floor(uz0);
        kk = fmin(fmax(kk, (double)(-pad)), (double)(g.n[2] + pad - 1));
        Z.kp = (int)kk + pad;
        const double bf = iw > 0.0 ? kk + 1.0 : kk;                          // first plane ahead
        const double t0 = (bf - uz0) * iw, dt = fabs(iw);
        Z.t0z = (float)t0;
        Z.dtz = (float)dt;
        Z.dk = iw > 0.0 ? 1 : -1;
    }
    Z.active = true;
}

// Work item of the tiled launch: (view, column group, tile); items are sorted by tile so that all
// views and columns crossing one volume tile run while the tile is L2-resident.
struct ColumnLaunch {
    const uint2* items;   // nullptr: untiled, (view, cgroup) from the block id
    int n_items;
    int n_views, n_cgroups, n_bands;
    int band0;            // first band of this launch (bands band0 .. band0 + grid / n_items - 1)
    int tile, n_tx;       // tile side in cells, tiles along x
    int nzp, pad;
};

// z state of two rays of one lane (rows lane + 32 q), packed so the per-segment arithmetic of the
// pair issues as f32x2 instructions (FADD2 / FFMA2 / FMUL2).  The padded z cell is carried as the
// float kp + 1.5 * 2^23, whose bit pattern is 0x4B400000 + kp: a crossing adds +-1.0 (exact), and
// the segment pointers are stored pre-offset by -4 * 0x4B400000 bytes, so the address of the cell is
// ptr + 4 * bits(kpf) with no float -> int conversion.
constexpr float kMagic = 12582912.0f;          // 1.5 * 2^23
constexpr unsigned kMagicBits = 0x4B400000u;   // bits(kMagic)
constexpr float kNoCross = -1.0e30f;           // -(next crossing) of a ray with fixed z (finite: x * 0 = 0)

struct RayPair {
    float2 ntz;        // -(next z-plane crossing) = -(t0z + mz dtz)
    float2 mz;         // z-plane crossings taken so far
    float2 ndtz, nt0z; // -dtz, -t0z   (0, kNoCross when z is fixed)
    float2 kpf;        // padded z cell of the current segment, + kMagic
    float2 dkf;        // +-1 per crossing (0 when fixed), as float
    float2 acc0, acc1; // forward: sum f_s d_sigma, sum (f_e - f_s)(sigma_e - tau)
    float2 w;          // forward: 1 / cos(beta); adjoint: y / cos(beta)
    float2 sc;         // 1 / cos(beta) (attenuated operators: physical length = sigma length * sc)
    int dk0, dk1;      // +-1 / 0 as int (neighbour offset in the mixed-direction loop)
    bool live0, live1; // ray exists and (adjoint) carries a non-zero value
};

__device__ __forceinline__ void pair_init(RayPair& P, const RayZ& Za, const RayZ& Zb, float ya, float yb,
                                          bool kAdj) {
    P.kpf = make_float2((float)Za.kp + kMagic, (float)Zb.kp + kMagic);
    P.dk0 = Za.dk; P.dk1 = Zb.dk;
    P.dkf = make_float2((float)Za.dk, (float)Zb.dk);
    P.mz = make_float2(0.f, 0.f);
    P.ndtz = make_float2(Za.dk ? -Za.dtz : 0.f, Zb.dk ? -Zb.dtz : 0.f);
    P.nt0z = make_float2(Za.dk ? -Za.t0z : kNoCross, Zb.dk ? -Zb.t0z : kNoCross);
    P.ntz = P.nt0z;
    P.acc0 = make_float2(0.f, 0.f);
    P.acc1 = make_float2(0.f, 0.f);
    P.w = kAdj ? make_float2(ya * Za.scale, yb * Zb.scale) : make_float2(Za.scale, Zb.scale);
    P.sc = make_float2(Za.scale, Zb.scale);
    P.live0 = Za.active && (!kAdj || ya != 0.f);
    P.live1 = Zb.active && (!kAdj || yb != 0.f);
}

// z state at sigma_first (the first in-tile segment start): crossings tau_m < sigma_first taken.
__device__ __forceinline__ void z_skip(float& kpf, int dk, float& mzv, float& ntzv, float ndtz, float nt0z,
                                       float sf) {
    if (dk == 0) return;
    const float t0z = -nt0z, dtz = -ndtz;
    int m0 = (int)ceilf((sf - t0z) / dtz);
    m0 = m0 < 0 ? 0 : m0;
    if (fmaf((float)m0, dtz, t0z) < sf) ++m0;
    if (m0 > 0 && !(fmaf((float)(m0 - 1), dtz, t0z) < sf)) --m0;
    kpf += (float)(dk * m0);
    mzv = (float)m0;
    ntzv = -fmaf(mzv, dtz, t0z);
}

// Debug build (-DXRT_DEBUG_BOUNDS=1, tests only): every walk load / reduction address is checked
// against the buffer the launch walks (set per launch, stream-ordered); a miss prints and traps.
#ifndef XRT_DEBUG_BOUNDS
#define XRT_DEBUG_BOUNDS 0
#endif
#if XRT_DEBUG_BOUNDS
__device__ unsigned long long g_dbg_range[2];
#endif
__device__ __forceinline__ void dbg_chk(const void* a, int bytes) {
#if XRT_DEBUG_BOUNDS
    const unsigned long long x = (unsigned long long)a;
    if (x < g_dbg_range[0] || x + (unsigned long long)bytes > g_dbg_range[1]) {
        printf("xrt debug: address %llx outside [%llx, %llx) block %d thread %d\n", x, g_dbg_range[0],
               g_dbg_range[1], (int)blockIdx.x, (int)threadIdx.x);
        __trap();
    }
#else
    (void)a; (void)bytes;
#endif
}
__device__ __forceinline__ float ldg_chk(const float* a) { dbg_chk(a, 4); return __ldg(a); }

// red.global.add.f32 on an address built by integer arithmetic (a plain atomicAdd on such a generic
// pointer compiles to a generic ATOM with a shared-window check and CAS fallback)
__device__ __forceinline__ void red_add(float* a, float v, unsigned long long pol) {
    dbg_chk(a, 4);
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}

// L2 policies: the adjoint's accumulator tile is re-used by every view of a band -> evict_last;
// sinogram elements are touched once or twice -> evict_first (do not displace the tile).  (The
// forward's plain __ldg measured faster than ld.global.nc.L2::cache_hint.)
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float ld_stream(const float* a, unsigned long long pol) {
    float v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void red_sino(float* a, float v, unsigned long long pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" :: "l"(a), "f"(v), "l"(pol) : "memory");
}

// 1.0f if x > 0 else 0.0f (one FSET)
__device__ __forceinline__ float gt0(float x) {
    float r;
    asm("set.gt.f32.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
    return r;
}

// Units of the chunk's segments for the lane's 2*NP rays.  Per segment (cell, sigma_e, d_sigma)
// and ray: the cell k_s at the segment start and, if the ray's next z crossing tau < sigma_e, the
// cell k_s + dk; l_e = max(sigma_e - tau, 0) and l_s = d_sigma - l_e are C_up - C_low of the two
// units (eq:range_length_3D).  DK = +1 / -1: every ray of the warp steps that way (or is
// fixed), so the neighbour cell is an immediate offset; DK = 0: per-ray offsets.
__device__ __forceinline__ uint4 lds128(unsigned saddr) {
    uint4 raw;   // one 128-bit shared load per segment (broadcast to the warp)
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w) : "r"(saddr));
    return raw;
}

// one 128-bit shared store of a segment record (32-bit shared address: no generic conversion)
__device__ __forceinline__ void sts_seg(unsigned saddr, unsigned long long ptr, float se, float ds) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};"
                 :: "r"(saddr), "r"((unsigned)ptr), "r"((unsigned)(ptr >> 32)), "r"(__float_as_uint(se)),
                    "r"(__float_as_uint(ds)) : "memory");
}

__device__ __forceinline__ unsigned long long seg_ptr(const uint4& raw) {
    return ((unsigned long long)raw.y << 32) | raw.x;
}

// segment pointer + 4 bits(kpf) (float cells): shift-and-add (LEA / LEA.HI.X on the ALU pipe) or
// IMAD.WIDE (FMA-heavy pipe) -- XRT_COL_LEA
#ifndef XRT_COL_LEA
#define XRT_COL_LEA 0
#endif
__device__ __forceinline__ float* col_addr(unsigned long long ptr, float kpf) {
#if XRT_COL_LEA
    unsigned long long a;
    asm("{ .reg .u64 t; cvt.u64.u32 t, %2; shl.b64 t, t, 2; add.s64 %0, %1, t; }" : "=l"(a) : "l"(ptr), "r"(__float_as_uint(kpf)));
    return (float*)a;
#else
    return (float*)(ptr + 4ull * __float_as_uint(kpf));
#endif
}

// z crossing inside the segment: cr = 1 if tau < sigma_e, lm = l_e = max(sigma_e - tau, 0); then
// the ray's z state advances to the next segment.
template <int DK>
__device__ __forceinline__ void z_step(RayPair& P, const float2 se2, float2& cr, float2& lm) {
    const float2 m1 = make_float2(-1.f, -1.f);
    const float2 le = __fadd2_rn(se2, P.ntz);               // sigma_e - tau
    cr = make_float2(gt0(le.x), gt0(le.y));
    lm = __fmul2_rn(le, cr);
    if (DK > 0) P.kpf = __fadd2_rn(P.kpf, cr);
    else if (DK < 0) P.kpf = __ffma2_rn(cr, m1, P.kpf);
    else P.kpf = __ffma2_rn(cr, P.dkf, P.kpf);
    P.mz = __fadd2_rn(P.mz, cr);
    P.ntz = __ffma2_rn(P.mz, P.ndtz, P.nt0z);                 // -(t0z + mz dtz)
}

// Forward units of the chunk's segments for the lane's 2*NP rays.  Per segment (cell, sigma_e,
// d_sigma) and ray: the cell k_s at the segment start and, if the ray's next z crossing
// tau < sigma_e, the cell k_s + dk; l_e = max(sigma_e - tau, 0) and l_s = d_sigma - l_e are
// C_up - C_low of the two units (eq:range_length_3D):
//     acc += f_s d_sigma + (f_e - f_s) l_e.
// DK = +1 / -1: every ray of the warp steps that way (or is fixed), so the neighbour cell is an
// immediate offset; DK = 0: per-ray offsets.  Software-pipelined one segment deep: the z state
// decides the next segment's cells before this segment's arithmetic, so the next loads are in
// flight while this segment's values are consumed.
#ifndef XRT_FWD_UNROLL
#define XRT_FWD_UNROLL 2
#endif
constexpr int kFwdUnroll = XRT_FWD_UNROLL;

template <int NP, int DK>
__device__ __forceinline__ void column_segments_fwd(unsigned seg, int total, RayPair (&P)[NP]) {
    const float2 m1 = make_float2(-1.f, -1.f);
    uint4 raw = lds128(seg);
    float2 f0[NP], f1[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const float* a0 = col_addr(seg_ptr(raw), P[p].kpf.x);
        const float* a1 = col_addr(seg_ptr(raw), P[p].kpf.y);
        const int o0 = DK != 0 ? DK : P[p].dk0, o1 = DK != 0 ? DK : P[p].dk1;
        f0[p] = make_float2(ldg_chk(a0), ldg_chk(a1));
        f1[p] = make_float2(ldg_chk(a0 + o0), ldg_chk(a1 + o1));
    }
#pragma unroll kFwdUnroll
    for (int s = 0; s < total; ++s) {
        const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
        const float2 se2 = make_float2(qse, qse), ds2 = make_float2(qds, qds);
        const uint4 nraw = lds128(seg + 16u * (unsigned)min(s + 1, total - 1));   // last trip: reload
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float2 cr, lm;
            z_step<DK>(P[p], se2, cr, lm);
            // next segment's loads (cells from the advanced z state)
            const float* a0 = col_addr(seg_ptr(nraw), P[p].kpf.x);
            const float* a1 = col_addr(seg_ptr(nraw), P[p].kpf.y);
            const int o0 = DK != 0 ? DK : P[p].dk0, o1 = DK != 0 ? DK : P[p].dk1;
            const float2 g0 = make_float2(ldg_chk(a0), ldg_chk(a1));
            const float2 g1 = make_float2(ldg_chk(a0 + o0), ldg_chk(a1 + o1));
            // this segment's arithmetic
            P[p].acc0 = __ffma2_rn(f0[p], ds2, P[p].acc0);        // f_s * d_sigma
            const float2 d = __ffma2_rn(f0[p], m1, f1[p]);        // f_e - f_s
            P[p].acc1 = __ffma2_rn(d, lm, P[p].acc1);             // (f_e - f_s) * l_e
            f0[p] = g0;
            f1[p] = g1;
        }
        raw = nraw;
    }
}

// Every ray of the warp keeps one z cell (horizontal rays: the 3D parallel beam without tilt,
// reading 5): each segment is one unit per ray, l = d_sigma, no z state to advance.
template <int NP>
__device__ __forceinline__ void column_segments_fwd_flat(unsigned seg, int total, RayPair (&P)[NP]) {
#pragma unroll 4
    for (int s = 0; s < total; ++s) {
        const uint4 raw = lds128(seg + 16u * (unsigned)s);
        const float qds = __uint_as_float(raw.w);
        const float2 ds2 = make_float2(qds, qds);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float* a0 = col_addr(seg_ptr(raw), P[p].kpf.x);
            const float* a1 = col_addr(seg_ptr(raw), P[p].kpf.y);
            P[p].acc0 = __ffma2_rn(make_float2(ldg_chk(a0), ldg_chk(a1)), ds2, P[p].acc0);
        }
    }
}

template <int NP>
__device__ __forceinline__ void column_segments_adj_flat(unsigned seg, int total, RayPair (&P)[NP], unsigned klo,
                                                         unsigned kn) {
    const unsigned long long pol = l2_evict_last();
#pragma unroll 4
    for (int s = 0; s < total; ++s) {
        const uint4 raw = lds128(seg + 16u * (unsigned)s);
        const float qds = __uint_as_float(raw.w);
        const float2 ds2 = make_float2(qds, qds);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float* a0 = col_addr(seg_ptr(raw), P[p].kpf.x);
            float* a1 = col_addr(seg_ptr(raw), P[p].kpf.y);
            const float2 ws = __fmul2_rn(P[p].w, ds2);
            if (P[p].live0 && __float_as_uint(P[p].kpf.x) - klo < kn) red_add(a0, ws.x, pol);
            if (P[p].live1 && __float_as_uint(P[p].kpf.y) - klo < kn) red_add(a1, ws.y, pol);
        }
    }
}

#ifndef XRT_ADJ_UNROLL
#define XRT_ADJ_UNROLL 2
#endif
constexpr int kAdjUnroll = XRT_ADJ_UNROLL;
// Adjoint: the same units, y l scattered with red.global.add (the second unit only when the z
// crossing lies inside the segment).
template <int NP, int DK>
__device__ __forceinline__ void column_segments_adj(unsigned seg, int total, RayPair (&P)[NP], unsigned klo,
                                                    unsigned kn) {
    const float2 m1 = make_float2(-1.f, -1.f);
    const unsigned long long pol = l2_evict_last();
    float kpf_in0[NP], kpf_in1[NP];
#pragma unroll kAdjUnroll
    for (int s = 0; s < total; ++s) {
        const uint4 raw = lds128(seg + 16u * (unsigned)s);
        const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
        const float2 se2 = make_float2(qse, qse), ds2 = make_float2(qds, qds);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float* a0 = col_addr(seg_ptr(raw), P[p].kpf.x);
            float* a1 = col_addr(seg_ptr(raw), P[p].kpf.y);
            const int o0 = DK != 0 ? DK : P[p].dk0, o1 = DK != 0 ? DK : P[p].dk1;
            kpf_in0[p] = P[p].kpf.x;
            kpf_in1[p] = P[p].kpf.y;
            float2 cr, lm;
            z_step<DK>(P[p], se2, cr, lm);
            const float2 ls = __ffma2_rn(lm, m1, ds2);               // l_s = d_sigma - l_e
            const float2 ws = __fmul2_rn(P[p].w, ls), we = __fmul2_rn(P[p].w, lm);
            // only cells inside the image: a ray outside the z range (its start cell in the zero
            // padding) adds nothing the caller keeps, so it must not cost an L2 reduction.
            // (bits(kpf) - kMagicBits - pad) < N_z as unsigned <=> pad <= k < pad + N_z
            const unsigned kb0 = __float_as_uint(kpf_in0[p]) - klo, kb1 = __float_as_uint(kpf_in1[p]) - klo;
            if (P[p].live0 && kb0 < kn) red_add(a0, ws.x, pol);
            if (P[p].live1 && kb1 < kn) red_add(a1, ws.y, pol);
            if (P[p].live0 && cr.x != 0.f && kb0 + (unsigned)o0 < kn) red_add(a0 + o0, we.x, pol);
            if (P[p].live1 && cr.y != 0.f && kb1 + (unsigned)o1 < kn) red_add(a1 + o1, we.y, pol);
        }
    }
}

// ---------------------------------------------------------------- attenuated operators (N4)
// The units of a ray in path order (segment start cell, then the crossing cell), each of physical
// length L = l_sigma / cos(beta): x = mu L, phi(x) = (1 - e^-x) / x, e = e^-x = 1 - x phi, and
//     forward:  S <- S e + f L phi                       (S = sum_I f_I e^-A_I L_I phi_I at the end)
//     adjoint:  A_le += x;  img_I += y L phi e^-(A - A_le) (A = the ray's total attenuation)
// (DESIGN reading 23; the same weights as k_forward_att / k_adjoint_att).  phi by its Taylor series
// for |x| <= 1/8 (truncation x^5 / 720 < 5e-8 relative); kExact: e^-x by ex2 and the quotient where
// |x| > 1/8 (chosen per launch from max |mu| * the longest unit).
template <bool kExact>
__device__ __forceinline__ float2 att_phi(float2 x, float2& e) {
    const float2 c5 = make_float2(1.f / 120.f, 1.f / 120.f), c4 = make_float2(-1.f / 24.f, -1.f / 24.f);
    const float2 c3 = make_float2(1.f / 6.f, 1.f / 6.f), c2 = make_float2(-0.5f, -0.5f), c1 = make_float2(1.f, 1.f);
    const float2 mx = make_float2(-x.x, -x.y);
    float2 phi = __ffma2_rn(x, c5, c4);
    phi = __ffma2_rn(phi, x, c3);
    phi = __ffma2_rn(phi, x, c2);
    phi = __ffma2_rn(phi, x, c1);
    e = __ffma2_rn(mx, phi, c1);                         // 1 - x phi
    if (kExact) {
        if (fabsf(x.x) > 0.125f) { e.x = __expf(-x.x); phi.x = __fdividef(1.f - e.x, x.x); }
        if (fabsf(x.y) > 0.125f) { e.y = __expf(-x.y); phi.y = __fdividef(1.f - e.y, x.y); }
    }
    return phi;
}

// forward: cells are float2 (f, mu) of the interleaved z-fastest buffer (8 bytes per cell)
template <int NP, int DK, bool kExact>
__device__ __forceinline__ void column_segments_fwd_att(unsigned seg, int total, RayPair (&P)[NP]) {
    const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll 2
    for (int s = 0; s < total; ++s) {
        const uint4 raw = lds128(seg + 16u * (unsigned)s);
        const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
        const float2 se2 = make_float2(qse, qse), ds2 = make_float2(qds, qds);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2* a0 = (const float2*)(seg_ptr(raw) + 8ull * __float_as_uint(P[p].kpf.x));
            const float2* a1 = (const float2*)(seg_ptr(raw) + 8ull * __float_as_uint(P[p].kpf.y));
            const int o0 = DK != 0 ? DK : P[p].dk0, o1 = DK != 0 ? DK : P[p].dk1;
            const float2 v00 = __ldg(a0), v01 = __ldg(a1), v10 = __ldg(a0 + o0), v11 = __ldg(a1 + o1);
            float2 cr, lm;
            z_step<DK>(P[p], se2, cr, lm);
            const float2 Ls = __fmul2_rn(__ffma2_rn(lm, m1, ds2), P[p].sc);   // (d_sigma - l_e) / cos(beta)
            const float2 Le = __fmul2_rn(lm, P[p].sc);
            float2 es, ee;
            const float2 xs = __fmul2_rn(make_float2(v00.y, v01.y), Ls);
            const float2 ps = att_phi<kExact>(xs, es);
            P[p].acc0 = __ffma2_rn(make_float2(v00.x, v01.x), __fmul2_rn(Ls, ps), __fmul2_rn(P[p].acc0, es));
            const float2 xe = __fmul2_rn(make_float2(v10.y, v11.y), Le);
            P[p].acc1 = __fadd2_rn(P[p].acc1, __fadd2_rn(xs, xe));   // the piece's attenuation (tiled)
            const float2 pe = att_phi<kExact>(xe, ee);
            P[p].acc0 = __ffma2_rn(make_float2(v10.x, v11.x), __fmul2_rn(Le, pe), __fmul2_rn(P[p].acc0, ee));
        }
    }
}

// adjoint: cells of mu at the segment pointer (z-fastest float), the accumulator at + dacc bytes;
// acc0 = A_le (running), acc1 = A (the ray's total attenuation, from the plain forward of mu)
template <int NP, int DK, bool kExact>
__device__ __forceinline__ void column_segments_adj_att(unsigned seg, int total, RayPair (&P)[NP], long long dacc,
                                                        unsigned klo, unsigned kn) {
    const float2 m1 = make_float2(-1.f, -1.f);
    const unsigned long long pol = l2_evict_last();
#pragma unroll 2
    for (int s = 0; s < total; ++s) {
        const uint4 raw = lds128(seg + 16u * (unsigned)s);
        const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
        const float2 se2 = make_float2(qse, qse), ds2 = make_float2(qds, qds);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float* a0 = col_addr(seg_ptr(raw), P[p].kpf.x);
            const float* a1 = col_addr(seg_ptr(raw), P[p].kpf.y);
            const int o0 = DK != 0 ? DK : P[p].dk0, o1 = DK != 0 ? DK : P[p].dk1;
            const float2 mus = make_float2(__ldg(a0), __ldg(a1)), mue = make_float2(__ldg(a0 + o0), __ldg(a1 + o1));
            const unsigned kb0 = __float_as_uint(P[p].kpf.x) - klo, kb1 = __float_as_uint(P[p].kpf.y) - klo;
            float2 cr, lm;
            z_step<DK>(P[p], se2, cr, lm);
            const float2 ls = __ffma2_rn(lm, m1, ds2);
            const float2 Ls = __fmul2_rn(ls, P[p].sc), Le = __fmul2_rn(lm, P[p].sc);
            float2 es, ee;
            const float2 xs = __fmul2_rn(mus, Ls);
            const float2 ps = att_phi<kExact>(xs, es);
            P[p].acc0 = __fadd2_rn(P[p].acc0, xs);
            const float2 ts = __fadd2_rn(P[p].acc0, __fmul2_rn(P[p].acc1, m1));   // A_le - A
            const float2 vs = __fmul2_rn(__fmul2_rn(P[p].w, ls), ps);             // y L phi
            const float2 xe = __fmul2_rn(mue, Le);
            const float2 pe = att_phi<kExact>(xe, ee);
            P[p].acc0 = __fadd2_rn(P[p].acc0, xe);
            const float2 te = __fadd2_rn(P[p].acc0, __fmul2_rn(P[p].acc1, m1));
            const float2 ve = __fmul2_rn(__fmul2_rn(P[p].w, lm), pe);
            float* w0 = (float*)((const char*)a0 + dacc);
            float* w1 = (float*)((const char*)a1 + dacc);
            if (P[p].live0 && kb0 < kn) red_add(w0, vs.x * __expf(ts.x), pol);
            if (P[p].live1 && kb1 < kn) red_add(w1, vs.y * __expf(ts.y), pol);
            if (P[p].live0 && cr.x != 0.f && kb0 + (unsigned)o0 < kn) red_add(w0 + o0, ve.x * __expf(te.x), pol);
            if (P[p].live1 && cr.y != 0.f && kb1 + (unsigned)o1 < kn) red_add(w1 + o1, ve.y * __expf(te.y), pol);
        }
    }
}

template <int NP, int kOp, bool kExact>
__device__ __forceinline__ void att_walk(unsigned seg, int total, RayPair (&P)[NP], int mode, long long dacc,
                                         unsigned klo, unsigned kn) {
    if (kOp == 3) {
        if (mode == 1) column_segments_adj_att<NP, 1, kExact>(seg, total, P, dacc, klo, kn);
        else if (mode == -1) column_segments_adj_att<NP, -1, kExact>(seg, total, P, dacc, klo, kn);
        else column_segments_adj_att<NP, 0, kExact>(seg, total, P, dacc, klo, kn);
    } else {
        if (mode == 1) column_segments_fwd_att<NP, 1, kExact>(seg, total, P);
        else if (mode == -1) column_segments_fwd_att<NP, -1, kExact>(seg, total, P);
        else column_segments_fwd_att<NP, 0, kExact>(seg, total, P);
    }
}

// CTA = kWarps adjacent detector columns of one view, one band of 64 NP rows, one xy tile.  Each
// warp owns one column: it generates the column's in-plane path chunk by chunk (lane = one major
// slice, warp scan, segments in its own shared-memory buffer; no CTA barrier) and walks it for its
// 2 NP rays per lane (rows band*64NP + 32q + lane: adjacent rows in adjacent lanes, so the lanes'
// loads of one segment fall on consecutive addresses of the z-fastest volume).
// Occupancy targets as resident threads per SM (the launch bounds' minimum CTAs = threads / CTA size),
// each the measured best at 4 columns per CTA: 2 pairs per lane 640 (96 registers; cfg 4 forward
// 139.4 -> 135.0 ms vs 768), adjoint with 1 pair 896 (73 registers), forward with 1 pair 768,
// attenuated and 4-pair kernels 512.
#ifndef XRT_COL_MINB
#define XRT_COL_MINB (640 / (32 * XRT_COL_WARPS))
#endif

// kOp: 0 forward, 1 adjoint, 2 attenuated forward, 3 attenuated adjoint (N4), 4 the forward per tile
// piece (pass 1 of the tiled attenuated adjoint)
// kFlat: every ray of the plan keeps one z cell (3D parallel beam without tilt, reading 5): only the
// flat walks are compiled, so the kernel fits 64 registers and runs XRT_FLAT_THREADS per SM.
#ifndef XRT_FLAT_THREADS
#define XRT_FLAT_THREADS 1024
#endif
template <int kOp, int NP, bool kFlat = false>
#ifndef XRT_ATT_THREADS
#define XRT_ATT_THREADS 896   // attenuated kernels: cfg 4 forward 344.5 -> 304.5 ms, adjoint 738.8 -> 626.6 ms vs 512
#endif
#ifndef XRT_COL_MINB_ADJ1
#define XRT_COL_MINB_ADJ1 (896 / (32 * XRT_COL_WARPS))
#endif
#ifndef XRT_COL_MINB_FWD1
#define XRT_COL_MINB_FWD1 (768 / (32 * XRT_COL_WARPS))
#endif
__global__ void __launch_bounds__(kWarps * 32, kFlat ? XRT_FLAT_THREADS / (32 * kWarps) : ((kOp == 2 || kOp == 3) ? XRT_ATT_THREADS / (32 * kWarps) : (NP == 1 ? (kOp == 1 ? XRT_COL_MINB_ADJ1 : XRT_COL_MINB_FWD1) : XRT_COL_MINB))) k_column(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                       const float* __restrict__ vol, float* __restrict__ volw,
                                                       const float* __restrict__ sino_in,
                                                       float* __restrict__ sino_out, int view0,
                                                       const ColDesc* __restrict__ desc, ColumnLaunch L,
                                                       const float* __restrict__ sino_aux, const float* __restrict__ att_mumax,
                                                       float att_lmax) {
    constexpr bool kAdjoint = kOp == 1 || kOp == 3;
    constexpr bool kAtt = kOp == 2 || kOp == 3;
    constexpr int R = 2 * NP;
    // chunk length: 32 slices for the 2-pair forward (measured 2.4 % faster on cfg 4: shorter
    // segment lists stay closer in time to the loads they feed), else kPasses x 32
    constexpr int kP = (kOp == 0 && NP == 2 && XRT_FWD2_SHORT_CHUNK) ? 1 : kPasses;
    __shared__ Seg s_seg[kWarps][2 * 32 * kP];
    __shared__ float s_first[kWarps];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned bid = blockIdx.x;
    // band-major order: every view / column / tile of one band of detector rows (one z slab of
    // the volume) runs before the next band, so the volume working set is that slab
    const int band = L.band0 + (int)(bid / (unsigned)L.n_items);
    const unsigned it = bid % (unsigned)L.n_items;
    int vv, cg, ti0 = 0, ti1 = g.n[0], tj0 = 0, tj1 = g.n[1];
    if (L.items) {
        const uint2 w = L.items[it];
        vv = (int)w.x;
        cg = (int)(w.y & 0xffffu);
        const int t = (int)(w.y >> 16);
        ti0 = (t % L.n_tx) * L.tile; ti1 = min(ti0 + L.tile, g.n[0]);
        tj0 = (t / L.n_tx) * L.tile; tj1 = min(tj0 + L.tile, g.n[1]);
    } else {
        cg = (int)(it % (unsigned)L.n_cgroups);
        vv = (int)(it / (unsigned)L.n_cgroups);
    }
    const bool tiled = L.items != nullptr;
    const int c = cg * kWarps + warp;
    if (c >= dc.cols) return;                      // warp-uniform; no CTA barrier below
    const int v = view0 + vv;
    const ViewRec V = views[v];
    ColumnPath Pth;
    double ca = 1.0;
    float pux = 0.f, puy = 0.f, pwx = 0.f, pwy = 0.f;
    load_path(desc + ((int64_t)v * dc.cols + c), g.n[0], Pth, ca, pux, puy, pwx, pwy);
    if (!Pth.hit) return;
    // slice range of the tile: clip the in-plane line to the tile box, then widen (segments
    // outside the tile are filtered exactly by slice_segments)
    int na = 0, nb = Pth.n_slices;
    if (tiled) {
        float lo = -INFINITY, hi = INFINITY;
        if (pwx != 0.f) {
            const float a0 = (ti0 - pux) / pwx, a1 = (ti1 - pux) / pwx;
            lo = fmaxf(lo, fminf(a0, a1)); hi = fminf(hi, fmaxf(a0, a1));
        } else if (!(pux >= ti0 - 1e-3f && pux <= ti1 + 1e-3f)) { hi = -INFINITY; }
        if (pwy != 0.f) {
            const float a0 = (tj0 - puy) / pwy, a1 = (tj1 - puy) / pwy;
            lo = fmaxf(lo, fminf(a0, a1)); hi = fminf(hi, fmaxf(a0, a1));
        } else if (!(puy >= tj0 - 1e-3f && puy <= tj1 + 1e-3f)) { hi = -INFINITY; }
        if (!(hi >= lo)) return;
        const float ida = 1.f / Pth.dta;
        na = max(0, __float2int_rd((lo - Pth.t0a) * ida) - 1);
        nb = min(Pth.n_slices, __float2int_rd((hi - Pth.t0a) * ida) + 3);
    }
    // the lane's rays: rows (band * R + q) * 32 + lane
    RayPair P[NP];
    bool any_live = false, pos = true, neg = true;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        RayZ Za, Zb;
        const int ra = (band * R + 2 * p) * 32 + lane, rb = ra + 32;
        ray_z(V, dc, g, Pth, ca, ra, L.pad, Za);
        ray_z(V, dc, g, Pth, ca, rb, L.pad, Zb);
        const float ya = (kAdjoint && Za.active) ? ld_stream(sino_in + ((int64_t)v * dc.rows + ra) * dc.cols + c, l2_evict_first()) : 0.f;
        const float yb = (kAdjoint && Zb.active) ? ld_stream(sino_in + ((int64_t)v * dc.rows + rb) * dc.cols + c, l2_evict_first()) : 0.f;
        pair_init(P[p], Za, Zb, ya, yb, kAdjoint);
        if (kOp == 3 && !tiled) {   // the ray's total attenuation (plain forward of mu)
            P[p].acc1 = make_float2(Za.active ? sino_aux[((int64_t)v * dc.rows + ra) * dc.cols + c] : 0.f,
                                    Zb.active ? sino_aux[((int64_t)v * dc.rows + rb) * dc.cols + c] : 0.f);
        } else if (kOp == 3) {      // tiled: the attenuation from this tile's piece to the ray's end
            const int t = (int)(L.items[it].y >> 16);
            const int ntile = L.n_tx * ((g.n[1] + L.tile - 1) / L.tile);
            const int64_t ia = ((int64_t)v * (R * 32) + 2 * p * 32 + lane) * dc.cols + c;
            const int64_t ib = ia + 32 * (int64_t)dc.cols;
            P[p].acc1 = make_float2(Za.active ? sino_aux[3 * (ia * ntile + t) + 2] : 0.f,
                                    Zb.active ? sino_aux[3 * (ib * ntile + t) + 2] : 0.f);
        }
        any_live |= P[p].live0 | P[p].live1;
        pos &= Za.dk >= 0 && Zb.dk >= 0;
        neg &= Za.dk <= 0 && Zb.dk <= 0;
    }
    if (!__any_sync(0xffffffffu, any_live)) return;
    // warp-uniform z stepping direction (2: every ray keeps its z cell)
    const bool all_pos = __all_sync(0xffffffffu, pos), all_neg = __all_sync(0xffffffffu, neg);
    const int mode = all_pos && all_neg ? 2 : (all_pos ? 1 : (all_neg ? -1 : 0));
    Seg* seg = s_seg[warp];
    const unsigned seg_s = (unsigned)__cvta_generic_to_shared(seg);
    // segment pointers pre-offset by -4 kMagicBits bytes (see RayPair)
    // attenuated: the forward reads (f, mu) float2 cells; the adjoint reads mu at the pointer and
    // reduces into volw at + dacc
    constexpr unsigned long long kEsz = kOp == 2 ? 8ull : 4ull;
    const unsigned long long base = (unsigned long long)((kAdjoint && !kAtt) ? (const float*)volw : vol) -
                                    kEsz * kMagicBits;
    const unsigned long long cstride = kEsz * (unsigned long long)L.nzp;
    const long long dacc = kOp == 3 ? (long long)((const char*)volw - (const char*)vol) : 0ll;
    const bool exact = kAtt && (*att_mumax) * att_lmax > 0.125f;
    bool zinit = !tiled;  // untiled: the z state at sigma = 0 is the initial one
    float sig_piece = 0.f;  // attenuated, tiled: sigma where this tile's piece of the path starts
    const unsigned klo = kMagicBits + (unsigned)L.pad, kn = (unsigned)g.n[2];   // interior z cells
    for (int n0 = na; n0 < nb; n0 += 32 * kP) {
        // ---- warp-cooperative: kP passes of 32 slices (slice n = n0 + 32 pass + lane) ->
        //      in-tile segments, in path order
        int total = 0;
#pragma unroll
        for (int pass = 0; pass < kP; ++pass) {
            const int n = n0 + 32 * pass + lane;
            if (n0 + 32 * pass >= nb) break;   // warp-uniform
            float a0s = 0.f, a0e = 0.f, a1s = 0.f, a1e = 0.f;
            int c0 = 0, c1 = 0, cnt = 0;
            if (n < nb) cnt = slice_segments(Pth, n, ti0, ti1, tj0, tj1, a0s, a0e, c0, a1s, a1e, c1);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int b = total + incl - cnt;
            if (cnt > 0) {
                sts_seg(seg_s + 16u * (unsigned)b, base + cstride * (unsigned)c0, a0e, a0e - a0s);
                if (b == 0) s_first[warp] = a0s;
            }
            if (cnt > 1) {
                sts_seg(seg_s + 16u * (unsigned)(b + 1), base + cstride * (unsigned)c1, a1e, a1e - a1s);
            }
            total += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (total > 0) {
            if (!zinit) {
                zinit = true;
                const float sf = s_first[warp];
                sig_piece = sf;
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    z_skip(P[p].kpf.x, P[p].dk0, P[p].mz.x, P[p].ntz.x, P[p].ndtz.x, P[p].nt0z.x, sf);
                    z_skip(P[p].kpf.y, P[p].dk1, P[p].mz.y, P[p].ntz.y, P[p].ndtz.y, P[p].nt0z.y, sf);
                }
            }
            if constexpr (kFlat) {
                if (kAdjoint) column_segments_adj_flat<NP>(seg_s, total, P, klo, kn);
                else column_segments_fwd_flat<NP>(seg_s, total, P);
            } else if (kAtt) {
                if (exact) att_walk<NP, kOp, true>(seg_s, total, P, mode == 2 ? 0 : mode, dacc, klo, kn);
                else att_walk<NP, kOp, false>(seg_s, total, P, mode == 2 ? 0 : mode, dacc, klo, kn);
            } else if (mode == 2) {
                if (kAdjoint) column_segments_adj_flat<NP>(seg_s, total, P, klo, kn);
                else column_segments_fwd_flat<NP>(seg_s, total, P);
            } else if (kAdjoint) {
                if (mode > 0) column_segments_adj<NP, 1>(seg_s, total, P, klo, kn);
                else if (mode < 0) column_segments_adj<NP, -1>(seg_s, total, P, klo, kn);
                else column_segments_adj<NP, 0>(seg_s, total, P, klo, kn);
            } else {
                if (mode > 0) column_segments_fwd<NP, 1>(seg_s, total, P);
                else if (mode < 0) column_segments_fwd<NP, -1>(seg_s, total, P);
                else column_segments_fwd<NP, 0>(seg_s, total, P);
            }
        }
        __syncwarp();  // the next chunk overwrites the segments
    }
    if (!kAdjoint) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const RayPair& Q = P[q >> 1];
            if (!((q & 1) ? Q.live1 : Q.live0)) continue;
            const float a = (q & 1) ? Q.acc0.y + Q.acc1.y : Q.acc0.x + Q.acc1.x;
            const float out = kAtt ? ((q & 1) ? Q.acc0.y : Q.acc0.x) : a * ((q & 1) ? Q.w.y : Q.w.x);
            const int64_t m = ((int64_t)v * dc.rows + (band * R + q) * 32 + lane) * dc.cols + c;
            if ((kAtt || kOp == 4) && tiled) {
                // kOp 2: the attenuated piece (sigma, S_t, A_t); kOp 4 (the plain forward with volw =
                // the pieces buffer): (sigma, -, A_t) of mu -- pass 1 of the tiled attenuated adjoint
                // (sigma_start, S_t, A_t) of this tile's piece, slot (ray of the band, tile); the
                // pieces are combined in path order by k_att_combine (rays that miss the tile keep
                // the zero slot, which the combine treats as the identity)
                if (!zinit) continue;
                const int t = (int)(L.items[it].y >> 16);
                const int n_ty = (g.n[1] + L.tile - 1) / L.tile;
                const int64_t rib = ((int64_t)v * (R * 32) + q * 32 + lane) * dc.cols + c;   // ray in band
                float* slot = volw + 3 * (rib * (L.n_tx * n_ty) + t);
                slot[0] = sig_piece;
                if (kAtt) {
                    slot[1] = out;
                    slot[2] = (q & 1) ? Q.acc1.y : Q.acc1.x;
                } else {
                    slot[2] = out;
                }
            } else if (tiled) { if (out != 0.f) red_sino(sino_out + m, out, l2_evict_first()); }
            else __stcs(sino_out + m, out);
        }
    }
}

// [rows][cols] (row stride in_ld, column offset in_off) -> [cols][rows] (row stride out_ld,
// offset out_off): scatters [N_z][N_xy] into the padded z-fastest [N_xy][NzP] and back.
__global__ void k_transpose(const float* __restrict__ in, float* __restrict__ out, int64_t rows,
                            int64_t cols, int64_t in_ld, int64_t in_off, int64_t out_ld,
                            int64_t out_off) {
    __shared__ float tile[32][33];
    const int64_t bx = (int64_t)blockIdx.x * 32;
    for (int64_t by = (int64_t)blockIdx.y * 32; by < rows; by += (int64_t)gridDim.y * 32) {
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = by + j, cc = bx + threadIdx.x;
            if (r < rows && cc < cols) tile[j][threadIdx.x] = in[r * in_ld + in_off + cc];
        }
        __syncthreads();
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = bx + j, cc = by + threadIdx.x;  // out is [cols][rows]
            if (r < cols && cc < rows) out[r * out_ld + out_off + cc] = tile[threadIdx.x][j];
        }
        __syncthreads();
    }
}

inline cudaError_t transpose(const float* in, float* out, int64_t rows, int64_t cols, int64_t in_ld,
                             int64_t in_off, int64_t out_ld, int64_t out_off, cudaStream_t s) {
    const int64_t gy = (rows + 31) / 32;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)(gy < 32768 ? gy : 32768));
    k_transpose<<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols, in_ld, in_off, out_ld, out_off);
    return cudaGetLastError();
}

// ================================================================= forward on (f, delta f) cells
// The forward's volume copy with the crossing cell folded in: cell column c (flat xy index
// j N_x + i) holds 2 NzP float2,
//     fd[c][0][kp] = (f[k], f[k+1] - f[k]),    fd[c][1][kp] = (f[k], f[k-1] - f[k]),   kp = k + pad,
// zero outside the image (the padding next to the image carries +-f of the edge cell).  A ray whose
// z index steps +1 walks half 0, one stepping -1 walks half 1 (its padded index is offset by NzP),
// a ray with fixed z half 0.  Per segment and ray ONE 8-byte load gives the start cell's f_s and
// the difference f_e - f_s to the cell after the ray's z crossing, so the units of
// eq:range_length_3D accumulate as acc += f_s d_sigma + (f_e - f_s) l_e with
// l_e = max(sigma_e - tau, 0): one load instead of two (the LSU issue rate bounds the walk:
// LDG.32 1.69 / LDG.64 2.0 SM-cycles per warp instruction, profiles/issue_peak.json).

// [N_z][N_xy] image -> fd (rows k = -1 .. N_z of every column; the rest of the padding stays 0).
// Tile of 32 columns x 32 k (+1 halo on each side) through shared memory; writes are coalesced
// along k (float4 = two float2 cells of one half).
#ifndef XRT_TOFD_KFAST
#define XRT_TOFD_KFAST 1   // k tiles fastest: 1.75 -> 0.95 ms per cfg-4 forward (ncu)
#endif
__global__ void __launch_bounds__(256) k_to_fd(const float* __restrict__ img, float2* __restrict__ fd,
                                               int64_t nxy, int nz, int64_t nzp, int pad, int ka, int kb) {
    __shared__ float t[34][33];
#if XRT_TOFD_KFAST
    // consecutive blocks: consecutive k tiles of the same 32 columns (the writes of neighbouring
    // blocks continue each other's 256-byte runs of a column)
    const int64_t c0 = (int64_t)blockIdx.y * 32;
    const int k0 = ka + (int)blockIdx.x * 32;
#else
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    const int k0 = ka + (int)blockIdx.y * 32;          // first k of this tile's rows (ka .. kb - 1)
#endif
    // load k = k0 - 1 .. k0 + 32 (34 rows), columns c0 .. c0 + 31
    for (int r = threadIdx.y; r < 34; r += 8) {
        const int k = k0 - 1 + r;
        const int64_t c = c0 + threadIdx.x;
        t[r][threadIdx.x] = (k >= 0 && k < nz && c < nxy) ? img[(int64_t)k * nxy + c] : 0.f;
    }
    __syncthreads();
    // write: warp w handles columns w, w + 8, ...; lane = k offset
    for (int cc = threadIdx.y; cc < 32; cc += 8) {
        const int64_t c = c0 + cc;
        const int k = k0 + (int)threadIdx.x;
        if (c >= nxy || k >= kb) continue;
        const float f = t[threadIdx.x + 1][cc];
        const float fp = t[threadIdx.x + 2][cc], fm = t[threadIdx.x][cc];
        float2* col = fd + c * 2 * nzp + pad + k;
        col[0] = make_float2(f, fp - f);
        col[nzp] = make_float2(f, fm - f);
    }
}

// One lane's pair of rays on the fd volume.
struct FdPair {
    float2 kpf;    // magic float: bits = kMagicBits + half * NzP + pad + k (the current cell)
    float2 kpf0;   // kpf at the ray's entry state (crossing count = (kpf - kpf0) * dk)
    float2 dkf;    // +1 / -1 per crossing, 0 fixed
    float2 ntz;    // -(next crossing - sigma_c), sigma_c the current chunk's origin
    float2 ndtz;   // -dtz (0 fixed)
    float2 t0z;    // first crossing, sigma from the square entry (kNoCrossPos fixed)
    float acc0a, acc0b, acc1a, acc1b;
};
constexpr float kNoCrossPos = 1.0e30f;

__device__ __forceinline__ void fd_init(FdPair& P, const RayZ& Za, const RayZ& Zb, int nzp) {
    const float ha = Za.dk < 0 ? (float)nzp : 0.f, hb = Zb.dk < 0 ? (float)nzp : 0.f;
    P.kpf = make_float2((float)Za.kp + ha + kMagic, (float)Zb.kp + hb + kMagic);
    P.kpf0 = P.kpf;
    P.dkf = make_float2((float)Za.dk, (float)Zb.dk);
    P.ndtz = make_float2(Za.dk ? -Za.dtz : 0.f, Zb.dk ? -Zb.dtz : 0.f);
    P.t0z = make_float2(Za.dk ? Za.t0z : kNoCrossPos, Zb.dk ? Zb.t0z : kNoCrossPos);
    P.ntz = make_float2(-P.t0z.x, -P.t0z.y);
    P.acc0a = P.acc0b = P.acc1a = P.acc1b = 0.f;
}

// 1 / cos(beta) of a ray from its z-crossing spacing: dtz = d_z / |tan(beta)| (ray_z); fixed-z
// rays (tan(beta) snapped to 0) have 1
__device__ __forceinline__ float fd_scale(float ndtz, float dz) {
    if (ndtz == 0.f) return 1.f;
    const float tb = dz / ndtz;
    return sqrtf(fmaf(tb, tb, 1.f));
}

// crossings tau_m = t0z + m dtz with tau_m < sf taken (the ray's state at sigma_first, tiled)
__device__ __forceinline__ void fd_skip(float& kpf, float kpf0, float dkf, float t0z, float ndtz, float sf) {
    if (dkf == 0.f) return;
    const float dtz = -ndtz;
    int m0 = (int)ceilf((sf - t0z) / dtz);
    m0 = m0 < 0 ? 0 : m0;
    if (fmaf((float)m0, dtz, t0z) < sf) ++m0;
    if (m0 > 0 && !(fmaf((float)(m0 - 1), dtz, t0z) < sf)) --m0;
    kpf = fmaf((float)m0, dkf, kpf0);
}

// the next crossing relative to the chunk origin sigma_c, from the exact crossing count
__device__ __forceinline__ void fd_anchor(FdPair& P, float sc) {
    const float2 m = __fmul2_rn(__fadd2_rn(P.kpf, make_float2(-P.kpf0.x, -P.kpf0.y)), P.dkf);
    const float2 tau = __ffma2_rn(m, make_float2(-P.ndtz.x, -P.ndtz.y), P.t0z);
    P.ntz = make_float2(sc - tau.x, sc - tau.y);
}

// segment pointer + 8 bits(kpf): shift-and-add (LEA / LEA.HI.X, ALU pipe) instead of IMAD.WIDE
// (FMA-heavy pipe, which the walk's packed FP32 ops keep ~61 % busy) -- XRT_FD_LEA
#ifndef XRT_FD_LEA
#define XRT_FD_LEA 1   // cfg 4 121.0 -> 116.5 ms, cfg 5 17.5 -> 16.7
#endif
__device__ __forceinline__ unsigned long long fd_addr(unsigned long long ptr, float kpf) {
#if XRT_FD_LEA
    unsigned long long a;
    asm("{ .reg .u64 t; cvt.u64.u32 t, %2; shl.b64 t, t, 3; add.s64 %0, %1, t; }" : "=l"(a) : "l"(ptr), "r"(__float_as_uint(kpf)));
    return a;
#else
    return ptr + 8ull * __float_as_uint(kpf);
#endif
}

#ifndef XRT_FD_LDHINT
#define XRT_FD_LDHINT 1   // walk-load cache hint: 1 L1::evict_last (cfg 4 115.8 -> 115.5 ms), 2 L2::256B (115.9), 3 L1::evict_first (172.4: the L1 reuse between the CTA warps matters), 0 none
#endif
// the crossing flag [le > 0] as 1.0 / 0.0: FSET (ALU pipe) or le * 2^127 saturated (FMA pipe; exact:
// with FTZ any positive le >= 2^-126 maps to >= 2 -> 1, le <= 0 -> 0) -- XRT_FD_CR_SAT
#ifndef XRT_FD_CR_SAT
#define XRT_FD_CR_SAT 1   // cfg 4 115.4 -> 114.7 ms (ALU 46 % vs FMA-heavy 38 % busy)
#endif
__device__ __forceinline__ float fd_cr(float le) {
#if XRT_FD_CR_SAT
    float r;
    asm("mul.ftz.sat.f32 %0, %1, 0f7F000000;" : "=f"(r) : "f"(le));
    return r;
#else
    return gt0(le);
#endif
}

__device__ __forceinline__ float2 ldg_f2(unsigned long long a) {
    dbg_chk((const void*)a, 8);
    float2 v;
#if XRT_FD_LDHINT == 1
    asm("ld.global.nc.L1::evict_last.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#elif XRT_FD_LDHINT == 2
    asm("ld.global.nc.L2::256B.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#elif XRT_FD_LDHINT == 3
    asm("ld.global.nc.L1::evict_first.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#elif XRT_FD_LDHINT == 4
    asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#elif XRT_FD_LDHINT == 5
    asm("ld.global.nc.L1::evict_normal.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#else
    asm("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
#endif
    return v;
}

// the chunk's segments for the lane's 2 NP rays: per segment (pointer, sigma_e - sigma_c, d_sigma)
// and ray, z crossing cr = [tau < sigma_e], l_e = max(sigma_e - tau, 0), then the state advances;
// software-pipelined one segment deep (the next segment's loads issue before this one's FMAs).
// segments per trip: cfg 4 (NP = 2) 121.0 ms at 2 vs 140.2 (1) / 134.2 (4); cfg 5 (NP = 1) 18.4 ms at
// 4 vs 19.6 (2)
#ifndef XRT_FD_UNROLL
#define XRT_FD_UNROLL 0   // 0: by NP
#endif
// mirrored ray (kM): the cell z -> -z of the walked ray's, bits(kpf') = Kb - bits(kpf) (see k_fwd_fd),
// address = ptr + 8 bits(kpf'): IADD3 + IMAD.WIDE.U32
// mirrored cell of the two-half layout: bits(kpf') = Kb - bits(kpf), address = ptr + 8 bits(kpf') by
// IADD3 + shift-and-add (ALU pipe).  Measured on cfg 4 (profiles/r2_forward_fd.md): 94.7 ms, vs 100.3 ms
// with IMAD.WIDE.U32 for the mirrored address and 111.2 ms with IMAD.WIDE.U32 for both (FMA-heavy pipe)
__device__ __forceinline__ unsigned long long fd_addr_m(unsigned long long ptr, float kpf, unsigned Kb) {
    unsigned long long a;
    asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(a) : "r"(Kb - __float_as_uint(kpf)), "l"(ptr));
    return a;
}

struct FdMirror {
    float acc0a, acc0b, acc1a, acc1b;   // the mirrored rays of the pair's rays a / b
};

// interleaved z-mirror layout (kF4): one 16-byte load gives the walked ray's (f, f[k+1] - f[k]) and its
// mirror's (f', f'[k'-1] - f'), k' = N_z - 1 + 2 pad - k: address = ptr + 16 bits(kpf)
__device__ __forceinline__ float4 ldg_f4(unsigned long long ptr, float kpf) {
    unsigned long long a;
    asm("{ .reg .u64 t; cvt.u64.u32 t, %1; shl.b64 t, t, 4; add.s64 %0, %2, t; }" : "=l"(a) : "r"(__float_as_uint(kpf)), "l"(ptr));
    dbg_chk((const void*)a, 16);
    float4 v;
    asm("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a));
    return v;
}

template <int NP, bool kM = false, bool kF4 = false>
__device__ __forceinline__ void fd_segments(unsigned seg, int total, FdPair (&P)[NP], FdMirror (&Mr)[NP],
                                            unsigned Kb) {
    constexpr int kFdUnroll = XRT_FD_UNROLL > 0 ? XRT_FD_UNROLL : (NP == 1 ? 4 : 2);   // z-mirror (NP 1): 92.6 ms at 4 vs 94.7 at 2
    if constexpr (kF4) {
        uint4 raw = lds128(seg);
        float4 qa[NP], qb[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            qa[p] = ldg_f4(seg_ptr(raw), P[p].kpf.x);
            qb[p] = ldg_f4(seg_ptr(raw), P[p].kpf.y);
        }
#pragma unroll kFdUnroll
        for (int s = 0; s < total; ++s) {
            const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
            const float2 se2 = make_float2(qse, qse);
            const uint4 nraw = lds128(seg + 16u * (unsigned)(s + 1));
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float2 le = __fadd2_rn(se2, P[p].ntz);
                const float2 cr = make_float2(fd_cr(le.x), fd_cr(le.y));
                const float2 lm = __fmul2_rn(le, cr);
                const float lma = lm.x, lmb = lm.y;
                P[p].kpf = __ffma2_rn(cr, P[p].dkf, P[p].kpf);
                P[p].ntz = __ffma2_rn(cr, P[p].ndtz, P[p].ntz);
                const float4 na = ldg_f4(seg_ptr(nraw), P[p].kpf.x);
                const float4 nb = ldg_f4(seg_ptr(nraw), P[p].kpf.y);
                P[p].acc0a = fmaf(qa[p].x, qds, P[p].acc0a);
                P[p].acc1a = fmaf(qa[p].y, lma, P[p].acc1a);
                P[p].acc0b = fmaf(qb[p].x, qds, P[p].acc0b);
                P[p].acc1b = fmaf(qb[p].y, lmb, P[p].acc1b);
                Mr[p].acc0a = fmaf(qa[p].z, qds, Mr[p].acc0a);
                Mr[p].acc1a = fmaf(qa[p].w, lma, Mr[p].acc1a);
                Mr[p].acc0b = fmaf(qb[p].z, qds, Mr[p].acc0b);
                Mr[p].acc1b = fmaf(qb[p].w, lmb, Mr[p].acc1b);
                qa[p] = na;
                qb[p] = nb;
            }
            raw = nraw;
        }
        return;
    }
    uint4 raw = lds128(seg);
    float2 va[NP], vb[NP], wa[NP], wb[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        va[p] = ldg_f2(fd_addr(seg_ptr(raw), P[p].kpf.x));
        vb[p] = ldg_f2(fd_addr(seg_ptr(raw), P[p].kpf.y));
        if (kM) {
            wa[p] = ldg_f2(fd_addr_m(seg_ptr(raw), P[p].kpf.x, Kb));
            wb[p] = ldg_f2(fd_addr_m(seg_ptr(raw), P[p].kpf.y, Kb));
        }
    }
#pragma unroll kFdUnroll
    for (int s = 0; s < total; ++s) {
        const float qse = __uint_as_float(raw.z), qds = __uint_as_float(raw.w);
        const float2 se2 = make_float2(qse, qse);
        const uint4 nraw = lds128(seg + 16u * (unsigned)(s + 1));   // record `total` repeats the last one
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2 le = __fadd2_rn(se2, P[p].ntz);                 // sigma_e - tau
            const float2 cr = make_float2(fd_cr(le.x), fd_cr(le.y));
            const float2 lm = __fmul2_rn(le, cr);                        // l_e = max(sigma_e - tau, 0)
            const float lma = lm.x, lmb = lm.y;
            P[p].kpf = __ffma2_rn(cr, P[p].dkf, P[p].kpf);
            P[p].ntz = __ffma2_rn(cr, P[p].ndtz, P[p].ntz);
            const float2 na = ldg_f2(fd_addr(seg_ptr(nraw), P[p].kpf.x));
            const float2 nb = ldg_f2(fd_addr(seg_ptr(nraw), P[p].kpf.y));
            float2 ma = make_float2(0.f, 0.f), mb = make_float2(0.f, 0.f);
            if (kM) {
                ma = ldg_f2(fd_addr_m(seg_ptr(nraw), P[p].kpf.x, Kb));
                mb = ldg_f2(fd_addr_m(seg_ptr(nraw), P[p].kpf.y, Kb));
            }
            P[p].acc0a = fmaf(va[p].x, qds, P[p].acc0a);                  // f_s d_sigma
            P[p].acc1a = fmaf(va[p].y, lma, P[p].acc1a);                  // (f_e - f_s) l_e
            P[p].acc0b = fmaf(vb[p].x, qds, P[p].acc0b);
            P[p].acc1b = fmaf(vb[p].y, lmb, P[p].acc1b);
            va[p] = na;
            vb[p] = nb;
            if (kM) {
                Mr[p].acc0a = fmaf(wa[p].x, qds, Mr[p].acc0a);
                Mr[p].acc1a = fmaf(wa[p].y, lma, Mr[p].acc1a);
                Mr[p].acc0b = fmaf(wb[p].x, qds, Mr[p].acc0b);
                Mr[p].acc1b = fmaf(wb[p].y, lmb, Mr[p].acc1b);
                wa[p] = ma;
                wb[p] = mb;
            }
        }
        raw = nraw;
    }
}


#ifndef XRT_FD_THREADS
#define XRT_FD_THREADS 1024  // resident threads per SM targeted by the launch bounds (2 pairs per lane):
#endif                       // cfg 4 124.0 ms vs 136.0 (768), 138.9 (512); 4 x 4 CTAs 126.6
#ifndef XRT_FD_THREADS1
#define XRT_FD_THREADS1 1280 // ... 1 pair per lane (cfg 5: 15.55 ms at 1280 vs 16.20 at 1024, 16.0 at 768)
#endif
#ifndef XRT_FD_THREADSM
#define XRT_FD_THREADSM 1024 // ... the z-mirror forward (cfg 4: 92.6 ms vs 98.4 at 1280, 102.7 at 768)
#endif
#define XRT_FD_MINBM (XRT_FD_THREADSM / (32 * kFdWarps) > 0 ? XRT_FD_THREADSM / (32 * kFdWarps) : 1)
#define XRT_FD_MINB (XRT_FD_THREADS / (32 * kFdWarps) > 0 ? XRT_FD_THREADS / (32 * kFdWarps) : 1)

#define XRT_FD_MINB1 (XRT_FD_THREADS1 / (32 * kFdWarps) > 0 ? XRT_FD_THREADS1 / (32 * kFdWarps) : 1)

// CTA / warp / band layout as k_column (kOp 0): warp = one detector column, 2 NP rays per lane (rows
// band 64 NP + 32 q + lane), band-major over (view, column group, tile) items.
//
// kM (mirror, circular cone symmetric in z: grid centred at z = 0, detector rows centred, H = 0):
// the ray of row r' = rows - 1 - r is the mirror image of row r under z -> -z (v, tan(beta), z(sigma)
// odd in v): it crosses the mirrored units (i, j, N_z - 1 - k) at the same sigma with the same lengths.
// A lane walks rows r of the upper half (band b: rows 64 b + lane, + 32) and accumulates their
// mirrors from the same z state: padded cell kp' = N_z - 1 + 2 pad - kp in the other half of the fd
// column (the z direction flips), i.e. bits(kpf') = 2 kMagicBits + NzP + N_z - 1 + 2 pad - bits(kpf).
// Each mirrored ray's units and C_up - C_low are those of its walked ray mirrored (the fp32 walk's
// decisions, not an independent fp32 walk of row r'); the self-mirror middle row (odd rows) is walked
// only.  Saves the z-state arithmetic of half the rays.
//
// kF4 (with kM): the interleaved layout fd4[cell][k_p] = (f[k], f[k+1] - f[k], f[k'], f[k'-1] - f[k']) of
// k_to_fd4 (k' the mirrored cell): the walked ray (its z steps +1: the upper rows of the z-symmetric
// cone) and its mirror from ONE 16-byte load.
template <int NP, bool kM, bool kF4 = false>
__global__ void __launch_bounds__(kFdWarps * 32, kM ? XRT_FD_MINBM : (NP == 1 ? XRT_FD_MINB1 : XRT_FD_MINB))
k_fwd_fd(const ViewRec* __restrict__ views, DetC dc, GridC g, const float2* __restrict__ fd,
         float* __restrict__ sino_out, int view0, const ColDesc* __restrict__ desc, ColumnLaunch L) {
    constexpr int R = 2 * NP;
    const int rows_top = kM ? (dc.rows + 1) / 2 : dc.rows;
    __shared__ Seg s_seg[kFdWarps][2 * 32 + 1];   // + a copy of the chunk's last record (look-ahead)
    __shared__ float s_first[kFdWarps];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned bid = blockIdx.x;
    const int band = L.band0 + (int)(bid / (unsigned)L.n_items);
    const unsigned it = bid % (unsigned)L.n_items;
    int vv, cg, ti0 = 0, ti1 = g.n[0], tj0 = 0, tj1 = g.n[1];
    if (L.items) {
        const uint2 w = L.items[it];
        vv = (int)w.x;
        cg = (int)(w.y & 0xffffu);
        const int t = (int)(w.y >> 16);
        ti0 = (t % L.n_tx) * L.tile; ti1 = min(ti0 + L.tile, g.n[0]);
        tj0 = (t / L.n_tx) * L.tile; tj1 = min(tj0 + L.tile, g.n[1]);
    } else {
        cg = (int)(it % (unsigned)L.n_cgroups);
        vv = (int)(it / (unsigned)L.n_cgroups);
    }
    const bool tiled = L.items != nullptr;
    const int c = cg * kFdCols + warp % kFdCols;
    vv = vv * kFdViews + warp / kFdCols;           // items count view blocks of kFdViews views
    if (c >= dc.cols || vv >= L.n_views) return;  // warp-uniform; no CTA barrier below
    const int v = view0 + vv;
    const ViewRec V = views[v];
    ColumnPath Pth;
    double ca = 1.0;
    float pux = 0.f, puy = 0.f, pwx = 0.f, pwy = 0.f;
    load_path(desc + ((int64_t)v * dc.cols + c), g.n[0], Pth, ca, pux, puy, pwx, pwy);
    if (!Pth.hit) return;
    int na = 0, nb = Pth.n_slices;
    if (tiled) {
        float lo = -INFINITY, hi = INFINITY;
        if (pwx != 0.f) {
            const float a0 = (ti0 - pux) / pwx, a1 = (ti1 - pux) / pwx;
            lo = fmaxf(lo, fminf(a0, a1)); hi = fminf(hi, fmaxf(a0, a1));
        } else if (!(pux >= ti0 - 1e-3f && pux <= ti1 + 1e-3f)) { hi = -INFINITY; }
        if (pwy != 0.f) {
            const float a0 = (tj0 - puy) / pwy, a1 = (tj1 - puy) / pwy;
            lo = fmaxf(lo, fminf(a0, a1)); hi = fminf(hi, fmaxf(a0, a1));
        } else if (!(puy >= tj0 - 1e-3f && puy <= tj1 + 1e-3f)) { hi = -INFINITY; }
        if (!(hi >= lo)) return;
        const float ida = 1.f / Pth.dta;
        na = max(0, __float2int_rd((lo - Pth.t0a) * ida) - 1);
        nb = min(Pth.n_slices, __float2int_rd((hi - Pth.t0a) * ida) + 3);
    }
    FdPair P[NP];
    FdMirror Mr[NP];
    bool any_live = false;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        RayZ Za, Zb;
        const int ra = (band * R + 2 * p) * 32 + lane, rb = ra + 32;
        // z-mirror: rows past the upper half (last band) walk as inactive rays (flat, in the zero padding)
        ray_z(V, dc, g, Pth, ca, (!kM || ra < rows_top) ? ra : dc.rows, L.pad, Za);
        ray_z(V, dc, g, Pth, ca, (!kM || rb < rows_top) ? rb : dc.rows, L.pad, Zb);
        fd_init(P[p], Za, Zb, L.nzp);
        Mr[p].acc0a = Mr[p].acc0b = Mr[p].acc1a = Mr[p].acc1b = 0.f;
        any_live |= (Za.active && ra < rows_top) | (Zb.active && rb < rows_top);
    }
    // mirrored cell: bits(kpf') = Kb - bits(kpf), Kb = 2 kMagicBits + NzP + N_z - 1 + 2 pad (< 2^32)
    const unsigned Kb = 2u * kMagicBits + (unsigned)L.nzp + (unsigned)(g.n[2] - 1 + 2 * L.pad);
    if (!__any_sync(0xffffffffu, any_live)) return;
    Seg* seg = s_seg[warp];
    const unsigned seg_s = (unsigned)__cvta_generic_to_shared(seg);
    // segment pointers pre-offset by -8 kMagicBits bytes: address = ptr + 8 bits(kpf)
    // (kF4: 16-byte cells, nzp of them per column -- the same column stride)
    const unsigned long long base = (unsigned long long)fd - (kF4 ? 16ull : 8ull) * kMagicBits;
    const unsigned long long cstride = 16ull * (unsigned long long)L.nzp;
    bool zinit = !tiled;  // untiled: the z state at sigma = 0 is the initial one
    const ColDesc* dsc = desc + ((int64_t)v * dc.cols + c);
    for (int n0 = na; n0 < nb; n0 += 32) {
        ColumnPath Pc;
        load_path_chunk(dsc, g.n[0], Pc);
        // chunk origin: the start of slice n0 (the same fmaf every lane and the slices use)
        const float sc = n0 == 0 ? 0.f : fminf(fmaf((float)(n0 - 1), Pc.dta, Pc.t0a), Pc.L);
        const int n = n0 + lane;
        float a0s = 0.f, a0e = 0.f, a1s = 0.f, a1e = 0.f;
        int c0 = 0, c1 = 0, cnt = 0;
        if (n < nb) cnt = slice_segments(Pc, n, ti0, ti1, tj0, tj1, a0s, a0e, c0, a1s, a1e, c1);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int b = incl - cnt;
        if (cnt > 0) {
            sts_seg(seg_s + 16u * (unsigned)b, base + cstride * (unsigned)c0, a0e - sc, a0e - a0s);
            if (b == 0) s_first[warp] = a0s;
        }
        if (cnt > 1) sts_seg(seg_s + 16u * (unsigned)(b + 1), base + cstride * (unsigned)c1, a1e - sc, a1e - a1s);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        // the lane holding the last record also writes it at index `total` (the walk's look-ahead
        // reads one record past the end instead of clamping its index)
        if (cnt > 0 && b + cnt == total) {
            if (cnt > 1) sts_seg(seg_s + 16u * (unsigned)total, base + cstride * (unsigned)c1, a1e - sc, a1e - a1s);
            else sts_seg(seg_s + 16u * (unsigned)total, base + cstride * (unsigned)c0, a0e - sc, a0e - a0s);
        }
        __syncwarp();
        if (total > 0) {
            if (!zinit) {
                zinit = true;
                const float sf = s_first[warp];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    fd_skip(P[p].kpf.x, P[p].kpf0.x, P[p].dkf.x, P[p].t0z.x, P[p].ndtz.x, sf);
                    fd_skip(P[p].kpf.y, P[p].kpf0.y, P[p].dkf.y, P[p].t0z.y, P[p].ndtz.y, sf);
                }
            }
#pragma unroll
            for (int p = 0; p < NP; ++p) fd_anchor(P[p], sc);
            fd_segments<NP, kM, kF4>(seg_s, total, P, Mr, Kb);
        }
        __syncwarp();  // the next chunk overwrites the segments
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const FdPair& Q = P[q >> 1];
        const int r = (band * R + q) * 32 + lane;
        if (r >= rows_top) continue;               // ray_z's `active` (the column hits the square)
        const float a = (q & 1) ? (Q.acc0b + Q.acc1b) * fd_scale(Q.ndtz.y, (float)g.d[2])
                                : (Q.acc0a + Q.acc1a) * fd_scale(Q.ndtz.x, (float)g.d[2]);
        const int64_t m = ((int64_t)v * dc.rows + r) * dc.cols + c;
        if (tiled) { if (a != 0.f) red_sino(sino_out + m, a, l2_evict_first()); }
        else __stcs(sino_out + m, a);
        if constexpr (kM) {
            const int rm = dc.rows - 1 - r;
            if (rm == r) continue;                 // the self-mirror middle row
            const FdMirror& M = Mr[q >> 1];
            const float sc = (q & 1) ? fd_scale(Q.ndtz.y, (float)g.d[2]) : fd_scale(Q.ndtz.x, (float)g.d[2]);
            const float b = ((q & 1) ? (M.acc0b + M.acc1b) : (M.acc0a + M.acc1a)) * sc;
            const int64_t mm = ((int64_t)v * dc.rows + rm) * dc.cols + c;
            if (tiled) { if (b != 0.f) red_sino(sino_out + mm, b, l2_evict_first()); }
            else __stcs(sino_out + mm, b);
        }
    }
}

// ============================================================================ voxel-driven gather
// The adjoint as a GATHER (north_star: "a voxel-driven gather that reuses the same
// per-ray unit condition"): every voxel sums y_m l_I(ray m) over the rays that cross it, with no
// atomics.  A warp owns one in-plane cell (i, j) and 32 Q consecutive voxels k of its z column
// (lane = k0 + lane + 32 q).  For each view, the detector columns whose in-plane lines can cross the
// cell come from the cell's four corners projected on the detector (+-1 column margin; a candidate
// that misses contributes exactly 0).  For each candidate column the in-plane part of the unit
// condition is the slab clip of the column's line (the same per-(view, column) descriptor the
// column kernels walk) with the cell: sigma in [C_low, C_up] of the in-plane unit
// (eq:conditions_3D_1 P:460-468 restricted to x, y; half-open for a fixed axis).  For
// each voxel, the candidate detector rows are those whose z line reaches z cell k inside that sigma
// range (z is affine in the row coordinate at fixed sigma); per row the z slab [k, k+1) gives the
// third pair of bounds and l = C_up - C_low of the 3D unit (eq:range_length_3D P:503-506) in
// physical units (the 1 / cos(beta) factor is folded into y by k_gather_prep).

// y'[v][c][r] = y[v][r][c] / cos(beta(r, c)), per-view 32x32 smem transposes (rows fastest, so the
// gather's lanes -- consecutive voxels k, consecutive rows r -- read consecutive addresses).
__global__ void k_gather_prep(const ViewRec* __restrict__ views, DetC dc, const ColDesc* __restrict__ desc,
                              const float* __restrict__ sino, float* __restrict__ yp, int v0) {
    __shared__ float tile[32][33];
    const int v = v0 + blockIdx.z;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    const ViewRec V = views[v];
    (void)V;
    for (int jj = threadIdx.y; jj < 32; jj += 8) {
        const int r = r0 + jj, c = c0 + threadIdx.x;
        float val = 0.f;
        if (r < dc.rows && c < dc.cols) {
            double tb;
            if (dc.beam == XRT_PAR3D) {
                tb = fabs(V.s2) <= kSnap ? 0.0 : V.pad[0];
            } else {
                const double vr = ((double)r - dc.cv) * dc.dv + dc.off_v;
                const double h = vr * dc.D / dc.sdd;
                const double ca = __ldg(reinterpret_cast<const double2*>(desc + ((int64_t)v * dc.cols + c)) + 4).y;
                tb = dc.curved ? vr / dc.sdd : h * ca * dc.inv_D;
                if (fabs(tb) <= kSnap) tb = 0.0;
            }
            const float scale = sqrtf(1.f + (float)(tb * tb));   // as ray_z
            val = sino[((int64_t)v * dc.rows + r) * dc.cols + c] * scale;
        }
        tile[jj][threadIdx.x] = val;
    }
    __syncthreads();
    for (int jj = threadIdx.y; jj < 32; jj += 8) {
        const int c = c0 + jj, r = r0 + threadIdx.x;
        if (r < dc.rows && c < dc.cols) yp[((int64_t)(v - v0) * dc.cols + c) * dc.rows + r] = tile[threadIdx.x][jj];
    }
}

template <int Q>
__global__ void __launch_bounds__(256) k_gather(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                const ColDesc* __restrict__ desc, const float* __restrict__ yp,
                                                float* __restrict__ work, int64_t nzp, int pad, int v0, int v1,
                                                int first) {
    extern __shared__ int s_kfix[];   // par3d without tilt: fixed z cell of every detector row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = blockIdx.x * 8 + warp, j = blockIdx.y;
    const int kb = blockIdx.z * 32 * Q;
    const bool par = dc.beam == XRT_PAR3D;
    const ViewRec V0 = views[v0];
    const bool par_flat = par && fabs(V0.s2) <= kSnap;
    if (par_flat) {
        // the half-open cell floor((z_hi - z) / d_z) of each (horizontal) row, in fp64 exactly as
        // ray_z / the oracle decide it (rows often lie exactly on z planes)
        for (int r = threadIdx.x; r < dc.rows; r += blockDim.x) {
            const double vr = ((double)r - dc.cv) * dc.dv + dc.off_v;
            s_kfix[r] = (int)floor((g.z_hi - vr * V0.c2) / g.d[2]);
        }
        __syncthreads();
    }
    if (i >= g.n[0]) return;
    const float x0 = (float)(g.x_lo + i * g.d[0]), x1 = (float)(g.x_lo + (i + 1) * g.d[0]);
    const float y1 = (float)(g.y_hi - j * g.d[1]), y0 = (float)(g.y_hi - (j + 1) * g.d[1]);
    const float inv_du = (float)(1.0 / dc.du), Df = (float)dc.D, sddf = (float)dc.sdd;
    float acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.f;
    // row coordinate <-> z-line parameter h: cone h = v D / sdd (P:636 with t, h scaled to the iso
    // plane, reading 8); par3d h = v.
    const float hscale = par ? 1.f : (float)(dc.D / dc.sdd);
    const float row_of_h = (float)(1.0 / (hscale * dc.dv));
    const float row_off = (float)(dc.cv - dc.off_v / dc.dv);
    const float h_of_row = (float)(hscale * dc.dv);
    const float h_off = (float)(hscale * (dc.off_v - dc.cv * dc.dv));
    const double h_of_row_d = (par ? 1.0 : dc.D / dc.sdd) * dc.dv;
    const double h_off_d = (par ? 1.0 : dc.D / dc.sdd) * (dc.off_v - dc.cv * dc.dv);
    // the (at most one) row with h == 0 exactly: a horizontal cone ray (fixed z cell per view)
    const double r0d = dc.cv - dc.off_v / dc.dv;
    const int r_flat = (!par && r0d == floor(r0d) && r0d >= 0 && r0d < dc.rows) ? (int)r0d : -1;
    const float kb_lo = (float)kb, kb_hi = (float)(kb + 32 * Q);
    const float vmin = (float)((0 - dc.cv) * dc.dv + dc.off_v), vmax = (float)((dc.rows - 1 - dc.cv) * dc.dv + dc.off_v);
    const float inv_sdd = (float)(1.0 / dc.sdd), inv_dzf = (float)g.inv_dz;
    for (int v = v0; v < v1; ++v) {
        const ViewRec V = views[v];
        const float c1 = (float)V.c1, s1 = (float)V.s1;
        // detector u of the four corners -> candidate columns; rho = distance from the source along
        // the central ray (cone: a ray through detector row v is at z = H + v rho / sdd there)
        float umin = INFINITY, umax = -INFINITY, rmin = INFINITY, rmax = -INFINITY;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float px = (t & 1) ? x1 : x0, py = (t & 2) ? y1 : y0;
            float u;
            if (par) {
                u = -px * s1 + py * c1;
            } else {
                const float ddx = px + Df * c1, ddy = py + Df * s1;   // P - S
                const float rho = ddx * c1 + ddy * s1;
                u = dc.curved ? sddf * atan2f(-ddx * s1 + ddy * c1, rho)        // arc length on the cylinder
                              : sddf * __fdividef(-ddx * s1 + ddy * c1, rho);
                // z = H + v rho / sdd along the ray: rho = distance along the central ray (flat) or
                // the in-plane distance from the source (cylindrical detector)
                const float rz = dc.curved ? sqrtf(ddx * ddx + ddy * ddy) : rho;
                rmin = fminf(rmin, rz);
                rmax = fmaxf(rmax, rz);
            }
            umin = fminf(umin, u);
            umax = fmaxf(umax, u);
        }
        if (!par) {
            // z cells any ray of this view can reach in the cell column; skip the view if that
            // misses the warp's k block (helical: most views)
            const float za = fminf(vmin * rmin, vmin * rmax) * inv_sdd, zb = fmaxf(vmax * rmin, vmax * rmax) * inv_sdd;
            const float Hf = (float)V.H;
            const float ua = ((float)g.z_hi - (Hf + zb)) * inv_dzf, ub = ((float)g.z_hi - (Hf + za)) * inv_dzf;
            if (ub < kb_lo - 2.f || ua > kb_hi + 2.f) continue;
        }
        // a column line crosses the cell iff its u lies inside the corners' u range (the fan is
        // monotone in u); 0.01-column margin for rounding (a spurious candidate adds exactly 0)
        const int c_lo = max(0, (int)ceilf((umin - (float)dc.off_u) * inv_du + (float)dc.cu - 0.01f));
        const int c_hi = min(dc.cols - 1, (int)floorf((umax - (float)dc.off_u) * inv_du + (float)dc.cu + 0.01f));
        for (int c = c_lo; c <= c_hi; ++c) {
            const ColDesc* dsc = desc + ((int64_t)v * dc.cols + c);
            const float4 q3 = __ldg(reinterpret_cast<const float4*>(dsc) + 3);   // ux0 uy0 wx wy
            const int flags = __ldg(reinterpret_cast<const int*>(dsc) + 7);
            if (!(flags & 1)) continue;
            // in-plane clip of the column's line with cell (i, j): [C_low, C_up] in sigma.  A fixed
            // (minor) axis keeps the descriptor's fp64 half-open cell.
            const int cell_b = __ldg(reinterpret_cast<const int*>(dsc) + 9);
            float lo = -INFINITY, hi = INFINITY;
            if (q3.z != 0.f) {
                const float iw = 1.f / q3.z;
                const float a = ((float)i - q3.x) * iw, b = ((float)(i + 1) - q3.x) * iw;
                lo = fmaxf(lo, fminf(a, b)); hi = fminf(hi, fmaxf(a, b));
            } else if (i != cell_b) continue;
            if (q3.w != 0.f) {
                const float iw = 1.f / q3.w;
                const float a = ((float)j - q3.y) * iw, b = ((float)(j + 1) - q3.y) * iw;
                lo = fmaxf(lo, fminf(a, b)); hi = fminf(hi, fmaxf(a, b));
            } else if (j != cell_b) continue;
            if (!(hi > lo)) continue;
            // z line of row h along the column: u_z(sigma) = A - T sigma - h (G0 + G1 sigma)
            // (cone / helical, from ray_z: tan(beta) = h ca / D, z(0) = h ca^2 + H; par3d: rows
            // parallel in the (sigma, z) plane, u_z = A - T sigma - h G0)
            const double2 q4 = __ldg(reinterpret_cast<const double2*>(dsc) + 4);   // sig_in, ca
            double Ad, G0d, G1d, Td;
            if (par) {
                const double tb = par_flat ? 0.0 : V.pad[0], zv = par_flat ? V.c2 : V.pad[1];
                Ad = (g.z_hi - q4.x * tb) * g.inv_dz;
                G0d = zv * g.inv_dz;
                G1d = 0.0;
                Td = tb * g.inv_dz;
            } else {
                // z(sigma) = H + h (lam + sigma_abs kap): flat lam = ca^2, kap = ca / D; curved
                // (tan(beta) = v / sdd = h / D, z(0) = D ca tan(beta)) lam = ca, kap = 1 / D
                const double lam = dc.curved ? q4.y : q4.y * q4.y, kap = dc.curved ? dc.inv_D : q4.y * dc.inv_D;
                Ad = (g.z_hi - V.H) * g.inv_dz;
                G0d = (lam + q4.x * kap) * g.inv_dz;
                G1d = kap * g.inv_dz;
                Td = 0.0;
            }
            const float A = (float)Ad, G0 = (float)G0d, G1 = (float)G1d, T = (float)Td;
            const float Gs = fmaf(lo, G1, G0), Ge = fmaf(hi, G1, G0);   // > 0
            // z range of all rows of this column inside the cell; skip if it misses the warp's k block
            {
                const float hA = fmaf(0.f, h_of_row, h_off), hB = fmaf((float)(dc.rows - 1), h_of_row, h_off);
                const float za = A - T * lo, zb = A - T * hi;
                const float u1 = za - hA * Gs, u2 = za - hB * Gs, u3 = zb - hA * Ge, u4 = zb - hB * Ge;
                const float umn = fminf(fminf(u1, u2), fminf(u3, u4)), umx = fmaxf(fmaxf(u1, u2), fmaxf(u3, u4));
                if (umx < kb_lo - 1.f || umn > kb_hi + 1.f) continue;
            }
            const float iGs = 1.f / Gs, iGe = 1.f / Ge;
            int kflat = INT_MIN;   // cone: the h == 0 row's fixed cell (fp64, as ray_z)
            if (r_flat >= 0) kflat = (int)floor((g.z_hi - V.H) / g.d[2]);
            const float* yc = yp + ((int64_t)(v - v0) * dc.cols + c) * dc.rows;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int k = kb + lane + 32 * q;
                if (k >= g.n[2]) continue;
                // rows whose z line reaches [k, k+1) for some sigma in [lo, hi]:
                // A - T s - h G(s) in [k, k+1)  <=>  h in ((A - T s - k - 1) / G, (A - T s - k) / G]
                const float as = A - T * lo - (float)k, ae = A - T * hi - (float)k;
                const float h1 = fminf((as - 1.f) * iGs, (ae - 1.f) * iGe);
                const float h2 = fmaxf(as * iGs, ae * iGe);
                const float ra = fmaf(h1, row_of_h, row_off), rb = fmaf(h2, row_of_h, row_off);
                const int r_lo = max(0, (int)ceilf(fminf(ra, rb) - 0.01f));
                const int r_hi = min(dc.rows - 1, (int)floorf(fmaxf(ra, rb) + 0.01f));
                float sum = 0.f;
                for (int r = r_lo; r <= r_hi; ++r) {
                    float l;
                    if (par_flat) {
                        l = s_kfix[r] == k ? hi - lo : 0.f;
                    } else if (r == r_flat) {
                        l = kflat == k ? hi - lo : 0.f;
                    } else {
                        // u_z(sigma) in [k, k+1)  <=>  sigma in (base - 1, base] / slope (sorted).
                        // base = u_z(0) - k in fp64: u_z(0) is a difference of O(N) terms and a
                        // u error becomes a sigma error / slope (shallow rays), as in ray_z
                        const double hd = fma((double)r, h_of_row_d, h_off_d);
                        const double base = fma(-hd, G0d, Ad) - (double)k;
                        const double is = 1.0 / fma(hd, G1d, Td);
                        const float t0 = (float)((base - 1.0) * is), t1 = (float)(base * is);
                        l = fminf(hi, fmaxf(t0, t1)) - fmaxf(lo, fminf(t0, t1));
                    }
                    if (l > 0.f) sum = fmaf(__ldg(yc + r), l, sum);
                }
                acc[q] += sum;
            }
        }
    }
    float* col = work + ((int64_t)j * g.n[0] + i) * nzp + pad;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int k = kb + lane + 32 * q;
        if (k < g.n[2]) col[k] = first ? acc[q] : col[k] + acc[q];
    }
}

}  // namespace

// Adjoint by the voxel-driven gather: sino -> z-fastest accumulator (interior rows fully written).
// Views are processed in blocks whose rescaled, transposed sinogram (workspace) stays L2-resident.
cudaError_t launch_adjoint_gather(const xrt_plan_s* p, const float* sino, float* vol_zfast, cudaStream_t s) {
    const ColDesc* d = (const ColDesc*)p->d_coldesc;
    const int64_t vb = p->gather_views;
    const int Q = p->grid.n[2] > 64 ? 4 : (p->grid.n[2] > 32 ? 2 : 1);
    for (int64_t v0 = 0; v0 < p->n_views; v0 += vb) {
        const int64_t v1 = std::min(p->n_views, v0 + vb);
        dim3 gp((unsigned)((p->det.cols + 31) / 32), (unsigned)((p->det.rows + 31) / 32), (unsigned)(v1 - v0));
        k_gather_prep<<<gp, dim3(32, 8), 0, s>>>(p->d_views, p->det, d, sino, p->d_gather_y, (int)v0);
        dim3 gg((unsigned)((p->grid.n[0] + 7) / 8), (unsigned)p->grid.n[1],
                (unsigned)((p->grid.n[2] + 32 * Q - 1) / (32 * Q)));
        const int first = v0 == 0;
        const size_t smem = sizeof(int) * (size_t)p->det.rows;   // par3d fixed-cell table
        if (Q == 4)
            k_gather<4><<<gg, 256, smem, s>>>(p->d_views, p->det, p->grid, d, p->d_gather_y, vol_zfast, p->nzp,
                                           (int)p->zpad, (int)v0, (int)v1, first);
        else if (Q == 2)
            k_gather<2><<<gg, 256, smem, s>>>(p->d_views, p->det, p->grid, d, p->d_gather_y, vol_zfast, p->nzp,
                                           (int)p->zpad, (int)v0, (int)v1, first);
        else
            k_gather<1><<<gg, 256, smem, s>>>(p->d_views, p->det, p->grid, d, p->d_gather_y, vol_zfast, p->nzp,
                                           (int)p->zpad, (int)v0, (int)v1, first);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int64_t gather_launches(const xrt_plan_s* p) {
    return 2 * ((p->n_views + p->gather_views - 1) / p->gather_views);
}

namespace {

}  // namespace

// padded z-fastest work [N_xy][NzP] -> image rows [k0, k1) of [N_z][N_xy] (staged adjoint)
cudaError_t launch_from_zfast_rows(const xrt_plan_s* p, const float* work, float* img, int64_t k0, int64_t k1,
                                   cudaStream_t s) {
    return transpose(work, img + k0 * p->grid.nxy, p->grid.nxy, k1 - k0, p->nzp, p->zpad + k0, p->grid.nxy, 0, s);
}

// image [N_z][N_xy] -> padded z-fastest work [N_xy][NzP] (interior rows pad .. pad + N_z)
cudaError_t launch_to_zfast(const xrt_plan_s* p, const float* img, float* work, cudaStream_t s) {
    return transpose(img, work, p->grid.n[2], p->grid.nxy, p->grid.nxy, 0, p->nzp, p->zpad, s);
}

// padded z-fastest work [N_xy][NzP] -> image [N_z][N_xy]
cudaError_t launch_from_zfast(const xrt_plan_s* p, const float* work, float* img, cudaStream_t s) {
    return transpose(work, img, p->grid.nxy, p->grid.n[2], p->nzp, p->zpad, p->grid.nxy, 0, s);
}

ColumnLaunch make_launch(const xrt_plan_s* p, int64_t v0, int64_t v1, int& nblk, bool adj, bool untiled = false) {
    ColumnLaunch L;
    const int rows_per_band = column_band_rows(p, adj);
    L.n_views = (int)(v1 - v0);
    L.n_cgroups = (p->det.cols + kWarps - 1) / kWarps;
    L.n_bands = (p->det.rows + rows_per_band - 1) / rows_per_band;
    L.nzp = (int)p->nzp;
    L.pad = (int)p->zpad;
    static const xrt_plan_s::ColTiling kUntiled{};
    const xrt_plan_s::ColTiling& T = untiled ? kUntiled : p->ct[adj ? 1 : 0];
    L.tile = T.tile;
    L.n_tx = T.n_tx;
    if (T.d_items) {
        L.items = (const uint2*)T.d_items;
        L.n_items = (int)T.n_items;
    } else {
        L.items = nullptr;
        L.n_items = L.n_views * L.n_cgroups;
    }
    L.band0 = 0;
    nblk = L.n_items * L.n_bands;
    return L;
}

static cudaError_t set_dbg_range(const void* lo, size_t bytes, cudaStream_t s) {
#if XRT_DEBUG_BOUNDS
    const unsigned long long r[2] = {(unsigned long long)lo, lo ? (unsigned long long)lo + bytes : ~0ull};
    return cudaMemcpyToSymbolAsync(g_dbg_range, r, sizeof(r), 0, cudaMemcpyHostToDevice, s);
#else
    (void)lo; (void)bytes; (void)s;
    return cudaSuccess;
#endif
}

template <int kOp>
cudaError_t launch_column_op(const xrt_plan_s* p, const float* vol, float* volw, const float* sino_in,
                             float* sino_out, int64_t v0, const ColumnLaunch& L, int nblk, cudaStream_t s,
                             const float* sino_aux = nullptr, const float* att_mumax = nullptr, float att_lmax = 0.f,
                             int np_override = 0) {
    constexpr bool kAdj = kOp == 1 || kOp == 3;
    const ColDesc* d = (const ColDesc*)p->d_coldesc;
    if (nblk <= 0) return cudaSuccess;
    const int np = np_override ? np_override : (kAdj ? p->col_np_adj : p->col_np);
    {
        const size_t vb = 4ull * (size_t)p->grid.nxy * (size_t)p->nzp;   // z-fastest float volume
        const cudaError_t e = kOp == 0 ? set_dbg_range(vol, vb, s) : kOp == 1 ? set_dbg_range(volw, vb, s)
                                                                        : set_dbg_range(nullptr, 0, s);
        if (e != cudaSuccess) return e;
    }
    // every ray keeps its z cell: the flat-only forward (cfg 3 1.99 -> 1.88 ms; the flat-only adjoint
    // measured 2.14 -> 2.17 ms, not used)
    if (kOp == 0 && p->flat_z && !std::getenv("XRT_NO_FLAT_KERNEL")) {
        if (np == 1)
            k_column<kOp, 1, true><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, vol, volw, sino_in, sino_out,
                                                                (int)v0, d, L, sino_aux, att_mumax, att_lmax);
        else if (np == 2)
            k_column<kOp, 2, true><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, vol, volw, sino_in, sino_out,
                                                                (int)v0, d, L, sino_aux, att_mumax, att_lmax);
        else
            return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    if (np == 1)
        k_column<kOp, 1><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, vol, volw, sino_in, sino_out, (int)v0, d, L,
                                                      sino_aux, att_mumax, att_lmax);
    else if (np == 2)
        k_column<kOp, 2><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, vol, volw, sino_in, sino_out, (int)v0, d, L,
                                                      sino_aux, att_mumax, att_lmax);
    else
        return cudaErrorInvalidValue;   // only 1 or 2 ray pairs per lane are built (plan rejects others)
    return cudaGetLastError();
}

template <bool kAdj>
cudaError_t launch_column(const xrt_plan_s* p, const float* vol, float* volw, const float* sino_in,
                          float* sino_out, int64_t v0, const ColumnLaunch& L, int nblk, cudaStream_t s) {
    return launch_column_op<kAdj ? 1 : 0>(p, vol, volw, sino_in, sino_out, v0, L, nblk, s);
}

cudaError_t launch_forward_column(const xrt_plan_s* p, const float* vol_zfast, float* sino,
                                  int64_t v0, int64_t v1, cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, v0, v1, nblk, false);
    if (L.items && !(v0 == 0 && v1 == p->n_views)) return cudaErrorInvalidValue;
    // rays whose column misses the image (or, tiled, every ray: partial sums) need zeros
    cudaError_t e = cudaMemsetAsync(sino + v0 * p->det.per_view, 0, sizeof(float) * (size_t)((v1 - v0) * p->det.per_view), s);
    if (e != cudaSuccess) return e;
    return launch_column<false>(p, vol_zfast, nullptr, nullptr, sino, v0, L, nblk, s);
}

// All views, detector-row bands [b0, b1) only (host pipelines: the sinogram rows of one band are
// transferred while the next band computes).  Rows of band b: [b * rows_per_band, ...).
int column_band_rows(const xrt_plan_s* p, bool adj) { return 64 * (adj ? p->col_np_adj : p->col_np); }
int column_bands(const xrt_plan_s* p, bool adj) {
    const int rb = column_band_rows(p, adj);
    return (p->det.rows + rb - 1) / rb;
}

// ---- forward on the (f, delta f) volume (AUTO forward of the 3D column path)
// fd rows [ka, kb) (ka >= -1, kb <= N_z + 1; the rows -1 .. N_z are the ones with data)
cudaError_t launch_to_fd_rows(const xrt_plan_s* p, const float* img, float2* fd, int ka, int kb, cudaStream_t s) {
    if (kb <= ka) return cudaSuccess;
    dim3 grid((unsigned)((p->grid.nxy + 31) / 32), (unsigned)((kb - ka + 31) / 32));
#if XRT_TOFD_KFAST
    if (grid.x <= 65535u) grid = dim3(grid.y, grid.x);
#endif
    k_to_fd<<<grid, dim3(32, 8), 0, s>>>(img, fd, p->grid.nxy, p->grid.n[2], p->nzp, (int)p->zpad, ka, kb);
    return cudaGetLastError();
}

cudaError_t launch_to_fd(const xrt_plan_s* p, const float* img, float2* fd, cudaStream_t s) {
    return launch_to_fd_rows(p, img, fd, -1, p->grid.n[2] + 1, s);
}

// interleaved z-mirror layout: fd4[cell][j] = (F[j], F[j+1] - F[j], F[C-j], F[C-j-1] - F[C-j]), F the
// zero-padded column (F[j] = f[j - pad]), C = N_z - 1 + 2 pad; rows j = pad - 1 .. pad + N_z hold data
// (the rest of the buffer stays zero from its allocation)
__global__ void __launch_bounds__(256) k_to_fd4(const float* __restrict__ img, float4* __restrict__ fd4, int64_t nxy,
                                                int nz, int64_t nzp, int pad, int j_lo, int j_hi) {
    __shared__ float t[33][33], u[33][33];
    const int64_t c0 = (int64_t)blockIdx.y * 32;
    const int j0 = j_lo + (int)blockIdx.x * 32;
    const int C = nz - 1 + 2 * pad;
    for (int r = threadIdx.y; r < 33; r += 8) {
        const int64_t c = c0 + threadIdx.x;
        const int k1 = j0 + r - pad, k2 = C - j0 - r - pad;
        t[r][threadIdx.x] = (k1 >= 0 && k1 < nz && c < nxy) ? img[(int64_t)k1 * nxy + c] : 0.f;
        u[r][threadIdx.x] = (k2 >= 0 && k2 < nz && c < nxy) ? img[(int64_t)k2 * nxy + c] : 0.f;
    }
    __syncthreads();
    for (int cc = threadIdx.y; cc < 32; cc += 8) {
        const int64_t c = c0 + cc;
        const int j = j0 + (int)threadIdx.x;
        if (c >= nxy || j >= j_hi) continue;
        const float f = t[threadIdx.x][cc], fn = t[threadIdx.x + 1][cc];
        const float g = u[threadIdx.x][cc], gn = u[threadIdx.x + 1][cc];
        fd4[c * nzp + j] = make_float4(f, fn - f, g, gn - g);
    }
}

#ifndef XRT_FD_F4
#define XRT_FD_F4 1   // device-path z-mirror forward on the interleaved layout (XRT_FD_F4=0 per launch: two halves)
#endif
bool fd_f4_on(const xrt_plan_s* p) {
    if (!fd_mirror_on_x(p)) return false;
    const char* e = std::getenv("XRT_FD_F4");
    return e ? std::atoi(e) != 0 : XRT_FD_F4 != 0;
}

// image rows k in [ka, kb) (ka >= -1, kb <= N_z + 1), i.e. padded rows j = pad + k
cudaError_t launch_to_fd4_rows(const xrt_plan_s* p, const float* img, float4* fd4, int ka, int kb, cudaStream_t s) {
    const int j_lo = std::max(0, (int)p->zpad + ka), j_hi = (int)p->zpad + kb;
    if (j_hi <= j_lo) return cudaSuccess;
    dim3 grid((unsigned)((j_hi - j_lo + 31) / 32), (unsigned)((p->grid.nxy + 31) / 32));
    k_to_fd4<<<grid, dim3(32, 8), 0, s>>>(img, fd4, p->grid.nxy, p->grid.n[2], p->nzp, (int)p->zpad, j_lo, j_hi);
    return cudaGetLastError();
}

cudaError_t launch_to_fd4(const xrt_plan_s* p, const float* img, float4* fd4, cudaStream_t s) {
    return launch_to_fd4_rows(p, img, fd4, -1, p->grid.n[2] + 1, s);
}

static cudaError_t launch_fd(const xrt_plan_s* p, const float2* fd, float* sino, const ColumnLaunch& L, int nblk,
                             cudaStream_t s) {
    if (nblk <= 0) return cudaSuccess;
    if (cudaError_t e = set_dbg_range(fd, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e != cudaSuccess) return e;
    const ColDesc* d = (const ColDesc*)p->d_coldesc;
    if (p->col_np == 1)
        k_fwd_fd<1, false><<<nblk, kFdWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, fd, sino, 0, d, L);
    else if (p->col_np == 2)
        k_fwd_fd<2, false><<<nblk, kFdWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, fd, sino, 0, d, L);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

int fd_mirror_bands(const xrt_plan_s* p);
bool fd_f4_on(const xrt_plan_s* p);
#ifndef XRT_FD_MIRROR_NP
#define XRT_FD_MIRROR_NP 1   // walked ray pairs per lane of the z-mirror forward (rows per band 64 NP)
#endif
constexpr int kMirNP = XRT_FD_MIRROR_NP;
// mirrored forward (k_fwd_fd<kMirNP, true>): read per launch, XRT_FWD_MIRROR=0 disables (A/B)
static bool fd_mirror_on(const xrt_plan_s* p) {
    const char* e = std::getenv("XRT_FWD_MIRROR");
    return p->fd_mirror && !(e && std::atoi(e) == 0);
}

// all views and bands [b0, b1) (rows b * 64 NP ...); sinogram rows of those bands pre-zeroed
cudaError_t launch_forward_fd_bands(const xrt_plan_s* p, const float2* fd, float* sino, int b0, int b1,
                                    cudaStream_t s) {
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    L.n_cgroups = (p->det.cols + kFdCols - 1) / kFdCols;
    if (p->ct_fd.d_items) {
        L.tile = p->ct_fd.tile;
        L.n_tx = p->ct_fd.n_tx;
        L.items = (const uint2*)p->ct_fd.d_items;
        L.n_items = (int)p->ct_fd.n_items;
    } else {
        L.items = nullptr;
        L.n_items = (int)((p->n_views + kFdViews - 1) / kFdViews) * L.n_cgroups;
    }
    const int rb = column_band_rows(p, false);
    const int r0 = b0 * rb, r1 = std::min(p->det.rows, b1 * rb);
    if (r1 <= r0) return cudaSuccess;
    const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
    cudaError_t e = cudaMemset2DAsync(sino + (int64_t)r0 * p->det.cols, pitch, 0,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views, s);
    if (e != cudaSuccess) return e;
    if (fd_f4_on(p)) {
        // the interleaved layout (built by fwd_prepare's launch_to_fd4) serves only the full-range call
        if (!(r0 == 0 && r1 == p->det.rows) || !p->d_work_fd4) return cudaErrorInvalidValue;
        L.band0 = 0;
        if (cudaError_t e2 = set_dbg_range(p->d_work_fd4, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess)
            return e2;
        k_fwd_fd<kMirNP, true, true><<<L.n_items * fd_mirror_bands(p), kFdWarps * 32, 0, s>>>(
            p->d_views, p->det, p->grid, (const float2*)p->d_work_fd4, sino, 0, (const ColDesc*)p->d_coldesc, L);
        return cudaGetLastError();
    }
    if (fd_mirror_on(p) && r0 == 0 && r1 == p->det.rows) {
        // all rows: bands of 64 upper-half rows, each with its mirrored rows (same L2 slab budget:
        // two 64-row slabs per band instead of one 128-row slab)
        L.band0 = 0;
        if (cudaError_t e2 = set_dbg_range(fd, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess)
            return e2;
        k_fwd_fd<kMirNP, true><<<L.n_items * fd_mirror_bands(p), kFdWarps * 32, 0, s>>>(
            p->d_views, p->det, p->grid, fd, sino, 0, (const ColDesc*)p->d_coldesc, L);
        return cudaGetLastError();
    }
    L.band0 = b0;
    return launch_fd(p, fd, sino, L, L.n_items * (b1 - b0), s);
}

bool fd_mirror_active(const xrt_plan_s* p) { return fd_mirror_on(p); }
bool fd_mirror_on_x(const xrt_plan_s* p) { return fd_mirror_on(p); }
int fd_mirror_bands(const xrt_plan_s* p) { return ((p->det.rows + 1) / 2 + 64 * kMirNP - 1) / (64 * kMirNP); }
int fd_mirror_band_rows() { return 64 * kMirNP; }

// mirror bands [b0, b1) (upper rows [64 b0, 64 b1) and their mirrors; those sinogram rows zeroed first)
cudaError_t launch_forward_fd_mirror_bands(const xrt_plan_s* p, const float2* fd, float* sino, int b0, int b1,
                                           cudaStream_t s) {
    if (b1 <= b0) return cudaSuccess;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    L.n_cgroups = (p->det.cols + kFdCols - 1) / kFdCols;
    if (p->ct_fd.d_items) {
        L.tile = p->ct_fd.tile;
        L.n_tx = p->ct_fd.n_tx;
        L.items = (const uint2*)p->ct_fd.d_items;
        L.n_items = (int)p->ct_fd.n_items;
    } else {
        L.items = nullptr;
        L.n_items = (int)((p->n_views + kFdViews - 1) / kFdViews) * L.n_cgroups;
    }
    const int rows = p->det.rows, top = (rows + 1) / 2;
    const int r0 = 64 * kMirNP * b0, r1 = std::min(top, 64 * kMirNP * b1);
    if (r1 <= r0) return cudaSuccess;
    const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
    cudaError_t e = cudaMemset2DAsync(sino + (int64_t)r0 * p->det.cols, pitch, 0,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views, s);
    if (e == cudaSuccess)
        e = cudaMemset2DAsync(sino + (int64_t)(rows - r1) * p->det.cols, pitch, 0,
                              sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views, s);
    if (e != cudaSuccess) return e;
    L.band0 = b0;
    if (fd_f4_on(p) && p->d_work_fd4) {   // host pipeline on the interleaved layout
        if (cudaError_t e2 = set_dbg_range(p->d_work_fd4, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess)
            return e2;
        k_fwd_fd<kMirNP, true, true><<<L.n_items * (b1 - b0), kFdWarps * 32, 0, s>>>(
            p->d_views, p->det, p->grid, (const float2*)p->d_work_fd4, sino, 0, (const ColDesc*)p->d_coldesc, L);
        return cudaGetLastError();
    }
    if (cudaError_t e2 = set_dbg_range(fd, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess) return e2;
    k_fwd_fd<kMirNP, true><<<L.n_items * (b1 - b0), kFdWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, fd, sino, 0,
                                                                     (const ColDesc*)p->d_coldesc, L);
    return cudaGetLastError();
}

int fd_view_block() { return kFdViews; }

// band b, views [fd_part_view[part], fd_part_view[part + 1]) only (tiled plans; see xrt_plan_s::kFwdParts)
cudaError_t launch_forward_fd_band_part(const xrt_plan_s* p, const float2* fd, float* sino, int b, int part,
                                        cudaStream_t s) {
    if (!p->d_fd_part_items || part < 0 || part >= xrt_plan_s::kFwdParts) return cudaErrorInvalidValue;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    L.n_cgroups = (p->det.cols + kFdCols - 1) / kFdCols;
    L.tile = p->ct_fd.tile;
    L.n_tx = p->ct_fd.n_tx;
    L.items = (const uint2*)p->d_fd_part_items + p->fd_part_off[part];
    L.n_items = (int)(p->fd_part_off[part + 1] - p->fd_part_off[part]);
    const int rb = column_band_rows(p, false);
    const int r0 = b * rb, r1 = std::min(p->det.rows, (b + 1) * rb);
    const int64_t v0 = p->fd_part_view[part], v1 = p->fd_part_view[part + 1];
    if (r1 <= r0 || v1 <= v0) return cudaSuccess;
    const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
    cudaError_t e = cudaMemset2DAsync(sino + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch, 0,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0), s);
    if (e != cudaSuccess) return e;
    L.band0 = b;
    return launch_fd(p, fd, sino, L, L.n_items, s);
}

// z-mirror band b, views [fd_part_view[part], fd_part_view[part + 1]) only (tiled plans)
cudaError_t launch_forward_fd_mirror_band_part(const xrt_plan_s* p, const float2* fd, float* sino, int b, int part,
                                               cudaStream_t s) {
    if (!p->d_fd_part_items || part < 0 || part >= xrt_plan_s::kFwdParts) return cudaErrorInvalidValue;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    L.n_cgroups = (p->det.cols + kFdCols - 1) / kFdCols;
    L.tile = p->ct_fd.tile;
    L.n_tx = p->ct_fd.n_tx;
    L.items = (const uint2*)p->d_fd_part_items + p->fd_part_off[part];
    L.n_items = (int)(p->fd_part_off[part + 1] - p->fd_part_off[part]);
    const int rows = p->det.rows, top = (rows + 1) / 2;
    const int r0 = 64 * kMirNP * b, r1 = std::min(top, 64 * kMirNP * (b + 1));
    const int64_t v0 = p->fd_part_view[part], v1 = p->fd_part_view[part + 1];
    if (r1 <= r0 || v1 <= v0 || L.n_items <= 0) return cudaSuccess;
    const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
    cudaError_t e = cudaMemset2DAsync(sino + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch, 0,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0), s);
    if (e == cudaSuccess)
        e = cudaMemset2DAsync(sino + v0 * p->det.per_view + (int64_t)(rows - r1) * p->det.cols, pitch, 0,
                              sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0), s);
    if (e != cudaSuccess) return e;
    L.band0 = b;
    if (fd_f4_on(p) && p->d_work_fd4) {
        if (cudaError_t e2 = set_dbg_range(p->d_work_fd4, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess)
            return e2;
        k_fwd_fd<kMirNP, true, true><<<L.n_items, kFdWarps * 32, 0, s>>>(
            p->d_views, p->det, p->grid, (const float2*)p->d_work_fd4, sino, 0, (const ColDesc*)p->d_coldesc, L);
        return cudaGetLastError();
    }
    if (cudaError_t e2 = set_dbg_range(fd, 16ull * (size_t)p->grid.nxy * (size_t)p->nzp, s); e2 != cudaSuccess) return e2;
    k_fwd_fd<kMirNP, true><<<L.n_items, kFdWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, fd, sino, 0,
                                                              (const ColDesc*)p->d_coldesc, L);
    return cudaGetLastError();
}

cudaError_t launch_forward_column_bands(const xrt_plan_s* p, const float* vol_zfast, float* sino, int b0,
                                        int b1, cudaStream_t s) {
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    const int rb = column_band_rows(p, false);
    const int r0 = b0 * rb, r1 = std::min(p->det.rows, b1 * rb);
    if (r1 <= r0) return cudaSuccess;
    const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
    cudaError_t e = cudaMemset2DAsync(sino + (int64_t)r0 * p->det.cols, pitch, 0,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views, s);
    if (e != cudaSuccess) return e;
    L.band0 = b0;
    return launch_column<false>(p, vol_zfast, nullptr, nullptr, sino, 0, L, L.n_items * (b1 - b0), s);
}

cudaError_t launch_adjoint_column_bands(const xrt_plan_s* p, const float* sino, float* vol_zfast, int b0,
                                        int b1, cudaStream_t s) {
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, true);
    L.band0 = b0;
    return launch_column<true>(p, nullptr, vol_zfast, sino, nullptr, 0, L, L.n_items * (b1 - b0), s);
}

// band b of the adjoint, views [adj_part_view[part], adj_part_view[part + 1]) only (tiled plans)
cudaError_t launch_adjoint_column_band_part(const xrt_plan_s* p, const float* sino, float* vol_zfast, int b,
                                            int part, cudaStream_t s) {
    if (!p->d_adj_part_items || part < 0 || part >= xrt_plan_s::kFwdParts) return cudaErrorInvalidValue;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, true);
    L.items = (const uint2*)p->d_adj_part_items + p->adj_part_off[part];
    L.n_items = (int)(p->adj_part_off[part + 1] - p->adj_part_off[part]);
    L.band0 = b;
    return launch_column<true>(p, nullptr, vol_zfast, sino, nullptr, 0, L, L.n_items, s);
}

cudaError_t launch_adjoint_column(const xrt_plan_s* p, const float* sino, float* vol_zfast,
                                  int64_t v0, int64_t v1, cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, v0, v1, nblk, true);
    if (L.items && !(v0 == 0 && v1 == p->n_views)) return cudaErrorInvalidValue;
    return launch_column<true>(p, nullptr, vol_zfast, sino, nullptr, v0, L, nblk, s);
}

// ---------------------------------------------------------------- attenuated operators (N4)
namespace {
// [rows][cols] -> the .x (comp 0) or .y (comp 1) field of the float2 z-fastest [cols][NzP] buffer
__global__ void k_transpose_f2(const float* __restrict__ in, float* __restrict__ out2, int64_t rows, int64_t cols,
                               int64_t out_ld, int64_t out_off, int comp) {
    __shared__ float tile[32][33];
    const int64_t bx = (int64_t)blockIdx.x * 32;
    for (int64_t by = (int64_t)blockIdx.y * 32; by < rows; by += (int64_t)gridDim.y * 32) {
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = by + j, cc = bx + threadIdx.x;
            if (r < rows && cc < cols) tile[j][threadIdx.x] = in[r * cols + cc];
        }
        __syncthreads();
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = bx + j, cc = by + threadIdx.x;
            if (r < cols && cc < rows) out2[2 * (r * out_ld + out_off + cc) + comp] = tile[threadIdx.x][j];
        }
        __syncthreads();
    }
}

// max |mu| (as the bits of a non-negative float, whose integer order is the float order)
__global__ void k_absmax(const float* __restrict__ a, int64_t n, unsigned* __restrict__ out) {
    unsigned m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, __float_as_uint(fabsf(a[i])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
}  // namespace

cudaError_t launch_att_prepare(const xrt_plan_s* p, const float* img, const float* mu, float* work2,
                               unsigned* mumax, cudaStream_t s) {
    const int64_t rows = p->grid.n[2], cols = p->grid.nxy;
    const int64_t gy = (rows + 31) / 32;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)(gy < 32768 ? gy : 32768));
    if (img) {
        k_transpose_f2<<<grid, dim3(32, 8), 0, s>>>(img, work2, rows, cols, p->nzp, p->zpad, 0);
        k_transpose_f2<<<grid, dim3(32, 8), 0, s>>>(mu, work2, rows, cols, p->nzp, p->zpad, 1);
    }
    cudaError_t e = cudaMemsetAsync(mumax, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_absmax<<<4 * 148, 256, 0, s>>>(mu, p->grid.nxyz, mumax);
    return cudaGetLastError();
}

// longest physical unit (the cell diagonal): bounds x = mu l for the choice of the phi evaluation
static float att_lmax(const xrt_plan_s* p) {
    return (float)std::sqrt(p->grid.d[0] * p->grid.d[0] + p->grid.d[1] * p->grid.d[1] + p->grid.d[2] * p->grid.d[2]);
}

namespace {
// S of every ray of band `band` from its tile pieces: sorted by the piece's start sigma, then
// S <- S e^-A_t + S_t (the unit recurrence at piece level).  Zero slots (tiles the ray misses) are
// identities wherever they sort.
__global__ void k_att_combine(const float* __restrict__ pieces, int n_tiles, int rows_band, int band, DetC dc,
                              int64_t n_views, float* __restrict__ sino) {
    const int64_t rib = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_view = (int64_t)rows_band * dc.cols;
    if (rib >= n_views * per_view) return;
    const int64_t v = rib / per_view;
    const int64_t rem = rib - v * per_view;
    const int rr = (int)(rem / dc.cols), c = (int)(rem - (int64_t)rr * dc.cols);
    const int row = band * rows_band + rr;
    if (row >= dc.rows) return;
    float sg[kMaxAttTiles], S[kMaxAttTiles], A[kMaxAttTiles];
    const int nt = n_tiles;   // <= kMaxAttTiles: att_tiled() routes larger tilings to the untiled path
    for (int t = 0; t < nt; ++t) {
        const float* q = pieces + 3 * (rib * n_tiles + t);
        sg[t] = q[0]; S[t] = q[1]; A[t] = q[2];
    }
    for (int i = 1; i < nt; ++i)            // insertion sort by sigma (at most a handful of pieces)
        for (int j = i; j > 0 && sg[j] < sg[j - 1]; --j) {
            float a = sg[j]; sg[j] = sg[j - 1]; sg[j - 1] = a;
            a = S[j]; S[j] = S[j - 1]; S[j - 1] = a;
            a = A[j]; A[j] = A[j - 1]; A[j - 1] = a;
        }
    float T = 0.f;
    for (int t = 0; t < nt; ++t) T = fmaf(T, __expf(-A[t]), S[t]);
    sino[(v * dc.rows + row) * dc.cols + c] = T;
}
}  // namespace

cudaError_t launch_forward_att_column(const xrt_plan_s* p, const float* work2, const unsigned* mumax, float* sino,
                                      float* pieces, cudaStream_t s) {
    int nblk = 0;
    const xrt_plan_s::ColTiling& T = p->ct[0];
    if (!att_tiled(p) || !pieces) {
        // untiled: every ray's whole path in one CTA
        ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false, true);
        cudaError_t e = cudaMemsetAsync(sino, 0, sizeof(float) * (size_t)(p->n_views * p->det.per_view), s);
        if (e != cudaSuccess) return e;
        return launch_column_op<2>(p, work2, nullptr, nullptr, sino, 0, L, nblk, s, nullptr, (const float*)mumax,
                                   att_lmax(p));
    }
    // tiled (L2-resident slabs): per band, each tile piece's (sigma, S_t, A_t), then the combine
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, false);
    const int rb = column_band_rows(p, false), nb = column_bands(p, false);
    const int n_tiles = T.n_tx * T.n_ty;
    const int64_t rays_band = p->n_views * (int64_t)rb * p->det.cols;
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < nb && e == cudaSuccess; ++b) {
        e = cudaMemsetAsync(pieces, 0, sizeof(float) * 3 * (size_t)(rays_band * n_tiles), s);
        L.band0 = b;
        if (e == cudaSuccess)
            e = launch_column_op<2>(p, work2, pieces, nullptr, nullptr, 0, L, L.n_items, s, nullptr,
                                    (const float*)mumax, att_lmax(p));
        if (e == cudaSuccess) {
            k_att_combine<<<(unsigned)((rays_band + 255) / 256), 256, 0, s>>>(pieces, n_tiles, rb, b, p->det,
                                                                            p->n_views, sino);
            e = cudaGetLastError();
        }
    }
    return e;
}

// The tiled attenuated operators combine a ray's tile pieces in registers (k_att_combine /
// k_att_suffix hold kMaxAttTiles slots), so they serve tilings of at most kMaxAttTiles tiles; a plan
// with more tiles (large in-plane grids or small XRT_COLUMN_TILE) runs the untiled attenuated path.
bool att_tiled(const xrt_plan_s* p) {
    const xrt_plan_s::ColTiling& T = p->ct[0];
    return T.d_items != nullptr && T.n_tx * T.n_ty <= kMaxAttTiles && !std::getenv("XRT_ATT_UNTILED");
}

int64_t att_piece_floats(const xrt_plan_s* p) {
    const xrt_plan_s::ColTiling& T = p->ct[0];
    if (!att_tiled(p)) return 0;
    return 3 * p->n_views * (int64_t)column_band_rows(p, false) * p->det.cols * T.n_tx * T.n_ty;
}

namespace {
// per ray of a band: the pieces' (sigma, A_t) in path order -> slot[2] = B_t = sum of A over this
// piece and the later ones (the attenuation from the piece's start to the ray's end)
__global__ void k_att_suffix(float* __restrict__ pieces, int n_tiles, int64_t rays_band) {
    const int64_t rib = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (rib >= rays_band) return;
    float sg[kMaxAttTiles], A[kMaxAttTiles];
    int id[kMaxAttTiles];
    const int nt = n_tiles;   // <= kMaxAttTiles (att_tiled)
    for (int t = 0; t < nt; ++t) {
        sg[t] = pieces[3 * (rib * n_tiles + t)];
        A[t] = pieces[3 * (rib * n_tiles + t) + 2];
        id[t] = t;
    }
    for (int i = 1; i < nt; ++i)
        for (int j = i; j > 0 && sg[j] < sg[j - 1]; --j) {
            float a = sg[j]; sg[j] = sg[j - 1]; sg[j - 1] = a;
            a = A[j]; A[j] = A[j - 1]; A[j - 1] = a;
            const int k = id[j]; id[j] = id[j - 1]; id[j - 1] = k;
        }
    float B = 0.f;
    for (int t = nt - 1; t >= 0; --t) {
        B += A[t];
        pieces[3 * (rib * n_tiles + id[t]) + 2] = B;
    }
}
}  // namespace

// tiled attenuated adjoint: per band, pass 1 = the plain forward of mu per piece, (sigma, -, A_t),
// the suffix sums B_t, then the scatter with A_le running from each piece's start
cudaError_t launch_adjoint_att_tiled(const xrt_plan_s* p, const float* mu_zfast, float* pieces,
                                     const unsigned* mumax, const float* y, float* acc_zfast, cudaStream_t s) {
    const xrt_plan_s::ColTiling& T = p->ct[0];
    if (!att_tiled(p) || !pieces) return cudaErrorNotSupported;
    // both passes on the forward's tiles, bands and rays per lane (the pieces' layout)
    const int rbf = column_band_rows(p, false);
    int nblk = 0;
    ColumnLaunch Lf = make_launch(p, 0, p->n_views, nblk, false);
    ColumnLaunch La = Lf;
    const int nb = column_bands(p, false);
    const int n_tiles = T.n_tx * T.n_ty;
    const int64_t rays_band = p->n_views * (int64_t)rbf * p->det.cols;
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < nb && e == cudaSuccess; ++b) {
        e = cudaMemsetAsync(pieces, 0, sizeof(float) * 3 * (size_t)(rays_band * n_tiles), s);
        Lf.band0 = La.band0 = b;
        if (e == cudaSuccess)
            e = launch_column_op<4>(p, mu_zfast, pieces, nullptr, nullptr, 0, Lf, Lf.n_items, s);
        if (e == cudaSuccess) {
            k_att_suffix<<<(unsigned)((rays_band + 255) / 256), 256, 0, s>>>(pieces, n_tiles, rays_band);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            e = launch_column_op<3>(p, mu_zfast, acc_zfast, y, nullptr, 0, La, La.n_items, s, pieces,
                                    (const float*)mumax, att_lmax(p), p->col_np);
    }
    return e;
}

cudaError_t launch_adjoint_att_column(const xrt_plan_s* p, const float* mu_zfast, float* sinoA,
                                      const unsigned* mumax, const float* y, float* acc_zfast, cudaStream_t s) {
    // pass 1: A per ray = the plain forward of mu (tiled, L2-resident); its rounding differs from the
    // running sums of pass 2 by ~1e-7 A, i.e. the weights by a factor 1 +- 1e-7 A
    cudaError_t e = launch_forward_column(p, mu_zfast, sinoA, 0, p->n_views, s);
    if (e != cudaSuccess) return e;
    int nblk = 0;
    ColumnLaunch L = make_launch(p, 0, p->n_views, nblk, true, true);    // untiled: A_le runs from the entry
    return launch_column_op<3>(p, mu_zfast, acc_zfast, y, nullptr, 0, L, nblk, s, sinoA, (const float*)mumax,
                               att_lmax(p));
}

// Rays per lane 2 NP, NP in {1, 2}: the fewest idle rows in the last band of 64 NP rows (ties:
// more rays per lane, i.e. each segment descriptor shared by more rays).
int choose_col_np(int rows) {
    if (const char* e = std::getenv("XRT_COL_NP")) {   // experiments: 1 or 2 pairs per lane
        const int v = std::atoi(e);
        if (v == 1 || v == 2) return v;
    }
    int best = 1, best_waste = 1 << 30;
    for (int np = 1; np <= 2; ++np) {
        const int per = 64 * np;
        const int waste = (rows + per - 1) / per * per - rows;
        if (waste <= best_waste) { best_waste = waste; best = np; }
    }
    return best;
}

int column_cta_columns() { return kWarps; }

size_t column_desc_bytes() { return sizeof(ColDesc); }

cudaError_t launch_col_desc(const xrt_plan_s* p, cudaStream_t s) {
    const int64_t n = p->n_views * (int64_t)p->det.cols;
    k_col_desc<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(p->d_views, p->det, p->grid, n,
                                                         (ColDesc*)p->d_coldesc);
    return cudaGetLastError();
}

// Host: work list of the tiled launch.  For every view and column group, the tiles crossed by
// any of the group's in-plane lines (walked in fp64 over the tile grid); items sorted by tile.
int build_column_items(const xrt_plan_s* p, const ViewRec* views_host, int ts, int ntx, int nty,
                       std::vector<uint2>& items, bool fd) {
    const GridC& g = p->grid;
    const DetC& dc = p->det;
    const int C = fd ? kFdCols : kWarps;          // columns per CTA
    const int VB = fd ? kFdViews : 1;             // views per CTA (item .x = view block)
    const int ncg = (dc.cols + C - 1) / C;
    const int64_t nvb = (p->n_views + VB - 1) / VB;
    std::vector<std::vector<uint2>> per_tile((size_t)ntx * nty);
    std::vector<int64_t> mark((size_t)ntx * nty, -1);
    for (int64_t vb = 0; vb < nvb; ++vb) {
        for (int cgi = 0; cgi < ncg; ++cgi) {
            const int64_t stamp = vb * ncg + cgi;
            for (int64_t v = vb * VB; v < std::min<int64_t>(p->n_views, (vb + 1) * VB); ++v)
            for (int c = cgi * C; c < std::min(dc.cols, (cgi + 1) * C); ++c) {
                double qx, qy, ex, ey, ca;
                column_line(views_host[v], dc, c, qx, qy, ex, ey, ca);
                const double ux = (qx - g.x_lo) / g.d[0], uy = (g.y_hi - qy) / g.d[1];
                const double wx = ex / g.d[0], wy = -ey / g.d[1];
                // test every tile box (expanded by a margin); tiles are few (<= 64)
                for (int ty = 0; ty < nty; ++ty)
                    for (int tx = 0; tx < ntx; ++tx) {
                        const int t = ty * ntx + tx;
                        if (mark[t] == stamp) continue;
                        const double x0 = tx * ts - 1e-3, x1 = std::min(g.n[0], (tx + 1) * ts) + 1e-3;
                        const double y0 = ty * ts - 1e-3, y1 = std::min(g.n[1], (ty + 1) * ts) + 1e-3;
                        double lo = -INFINITY, hi = INFINITY;
                        bool ok = true;
                        if (wx != 0.0) {
                            const double a0 = (x0 - ux) / wx, a1 = (x1 - ux) / wx;
                            lo = std::max(lo, std::min(a0, a1)); hi = std::min(hi, std::max(a0, a1));
                        } else ok = ux >= x0 && ux <= x1;
                        if (wy != 0.0) {
                            const double a0 = (y0 - uy) / wy, a1 = (y1 - uy) / wy;
                            lo = std::max(lo, std::min(a0, a1)); hi = std::min(hi, std::max(a0, a1));
                        } else ok = ok && uy >= y0 && uy <= y1;
                        if (ok && hi >= lo) {
                            mark[t] = stamp;
                            per_tile[t].push_back(make_uint2((unsigned)vb, (unsigned)cgi | ((unsigned)t << 16)));
                        }
                    }
            }
        }
    }
    items.clear();
    for (auto& vt : per_tile) items.insert(items.end(), vt.begin(), vt.end());
    return (int)items.size();
}

}  // namespace xrt
