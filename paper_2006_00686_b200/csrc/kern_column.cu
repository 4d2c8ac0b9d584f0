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
// Launch order: blockIdx.x = view (fastest), y = column group, z = row band: the CTAs resident at
// any time are (nearly) all views of one or two column groups, whose in-plane lines all lie in a
// thin annulus |s1| ~ const of the image -- a small, L2-resident working set reused by every view.
#include <cuda_runtime.h>

#include <cstdlib>

#include "xrt_internal.cuh"

namespace xrt {

namespace {

constexpr int kColsPerCta = 4;
constexpr int kRowWarps = 2;                     // warps per column (64 rows per CTA)
constexpr int kWarps = kColsPerCta * kRowWarps;  // 8 warps = 256 threads
constexpr int kSlices = 64;                      // major slices per chunk (2 x 32 lanes)
constexpr int kSegCap = 2 * kSlices + 1;         // segments per chunk + end sentinel

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
};

// fp64 in-plane line of the column (the paper's per-column parameters), u = detector coordinate.
__device__ __forceinline__ void column_line(const ViewRec& V, const DetC& dc, int c, double& qx,
                                            double& qy, double& ex, double& ey, double& ca_out) {
    const double u = ((double)c - dc.cu) * dc.du + dc.off_u;
    if (dc.beam == XRT_PAR3D) {
        // xy line of (s1, phi1): foot s1 theta_1, direction (cos phi1, sin phi1)
        ex = V.c1; ey = V.s1;
        qx = -u * V.s1; qy = u * V.c1;
        ca_out = 1.0;
    } else {
        const double D = dc.D;
        const double t = u * D / dc.sdd;
        const double sq = sqrt(D * D + t * t);
        const double ca = D / sq, sa = t / sq;           // alpha = arctan(t / D)
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

// Sigma at which slice n starts (slice 0 starts at the square entry, 0).
__device__ __forceinline__ float slice_start(const ColumnPath& P, int n) {
    return n == 0 ? 0.f : (n >= P.n_slices ? P.L : fminf(fmaf((float)(n - 1), P.dta, P.t0a), P.L));
}

// Segments of major slice n: 1 or 2 in-plane units (cell, sigma_start, sigma_end).  The minor
// crossings at or before the slice start are counted against the SAME fmaf expression the
// neighbouring slices use, so every crossing value is produced exactly once (telescoping).
__device__ __forceinline__ int slice_segments(const ColumnPath& P, int n, float& s0, float& s1,
                                              float& s2, int& c0, int& c1) {
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
    c0 = ca * P.sa + (P.cell_b0 + P.step_b * mb) * P.sb;
    s0 = t_lo;
    s2 = t_hi;
    s1 = split ? tb : t_hi;
    c1 = split ? c0 + P.step_b * P.sb : c0;
    return split ? 2 : 1;
}

// Per-ray z description along the shared path (sigma from the square entry).
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
    double tb, z0, cb;  // tan(beta), z at absolute sigma 0, cos(beta)
    if (dc.beam == XRT_PAR3D) {
        // z(sigma) = s2 / cos(phi2) + sigma tan(phi2), sigma = t cos(phi2) - s2 sin(phi2)
        cb = V.c2;
        tb = V.s2 / V.c2;
        z0 = v / V.c2;
        if (fabs(V.s2) <= kSnap) { tb = 0.0; z0 = v * V.c2; }
    } else {
        const double D = dc.D;
        const double h = v * D / dc.sdd;
        // tan(beta) = h / sqrt(D^2 + t^2) = h cos(alpha) / D; |theta_xy| = cos(beta)
        const double tanb = h * ca / D;
        cb = 1.0 / sqrt(1.0 + tanb * tanb);
        const double s2 = h * (ca * ca) * cb + V.H * cb;
        tb = tanb;
        z0 = s2 / cb;
        if (fabs(tanb * cb) <= kSnap) { tb = 0.0; z0 = s2; }
    }
    Z.scale = (float)(1.0 / cb);
    const double uz0 = (g.z_hi - (z0 + P.sig_in * tb)) / g.d[2];   // u_z at sigma = 0
    const double wz = -tb / g.d[2];
    double kk = floor(uz0);                                         // half-open cell
    if (kk < (double)(-pad)) kk = (double)(-pad);
    if (kk > (double)(g.n[2] + pad - 1)) kk = (double)(g.n[2] + pad - 1);
    Z.kp = (int)kk + pad;
    if (wz != 0.0) {
        const double iw = 1.0 / wz;
        const double bf = wz > 0.0 ? kk + 1.0 : kk;                 // first plane ahead
        Z.t0z = (float)((bf - uz0) * iw);
        Z.dtz = (float)fabs(iw);
        Z.dk = wz > 0.0 ? 1 : -1;
    }
    Z.active = true;
}

template <bool kAdjoint>
__global__ void __launch_bounds__(kWarps * 32, 3) k_column(const ViewRec* __restrict__ views, DetC dc,
                                                         GridC g, const float* __restrict__ vol,
                                                         float* __restrict__ volw,
                                                         const float* __restrict__ sino_in,
                                                         float* __restrict__ sino_out, int view0,
                                                         int n_views, int n_cgroups, int nzp, int pad,
                                                         int order) {
    __shared__ Seg s_seg[kWarps][kSegCap];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // 1D grid; order 0: id = (band * n_cgroups + cgroup) * n_views + view (views fastest)
    //          order 1: id = (band * n_views + view) * n_cgroups + cgroup (columns fastest)
    const unsigned bid = blockIdx.x;
    int vv, cg, band;
    if (order == 0) {
        vv = (int)(bid % (unsigned)n_views);
        const unsigned rest = bid / (unsigned)n_views;
        cg = (int)(rest % (unsigned)n_cgroups);
        band = (int)(rest / (unsigned)n_cgroups);
    } else {
        cg = (int)(bid % (unsigned)n_cgroups);
        const unsigned rest = bid / (unsigned)n_cgroups;
        vv = (int)(rest % (unsigned)n_views);
        band = (int)(rest / (unsigned)n_views);
    }
    const int c = cg * kColsPerCta + (warp % kColsPerCta);
    const int r = (band * kRowWarps + warp / kColsPerCta) * 32 + lane;
    const int v = view0 + vv;
    if (c >= dc.cols) return;  // warp-uniform
    const ViewRec V = views[v];
    ColumnPath P;
    double ca;
    column_path(V, dc, g, c, P, ca);
    RayZ Z;
    ray_z(V, dc, g, P, ca, r, pad, Z);
    const int64_t m = ((int64_t)v * dc.rows + r) * dc.cols + c;
    float y = 0.f;
    if (kAdjoint && Z.active) y = sino_in[m] * Z.scale;
    const bool live = kAdjoint ? (Z.active && y != 0.f) : Z.active;
    float acc_s = 0.f, acc_e = 0.f;
    Seg* seg = s_seg[warp];
    const unsigned long long base = (unsigned long long)(kAdjoint ? (const float*)volw : vol);
    const unsigned long long cstride = 4ull * (unsigned long long)nzp;
    unsigned kp = (unsigned)Z.kp;
    (void)0;
    float tz = Z.t0z, mz = 0.f;
    if (__any_sync(0xffffffffu, live)) {
        for (int n0 = 0; n0 < P.n_slices; n0 += kSlices) {
            // ---- warp-cooperative: slices n0 .. n0+63 -> segments in path order
            int total = 0;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int n = n0 + half * 32 + lane;
                float a0 = 0.f, a1 = 0.f, a2 = 0.f;
                int c0 = 0, c1 = 0, cnt = 0;
                if (n < P.n_slices) cnt = slice_segments(P, n, a0, a1, a2, c0, c1);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                const int b = total + incl - cnt;
                if (cnt > 0) {
                    Seg q; q.ptr = base + cstride * (unsigned)c0; q.se = a1; q.ds = a1 - a0;
                    seg[b] = q;
                }
                if (cnt > 1) {
                    Seg q; q.ptr = base + cstride * (unsigned)c1; q.se = a2; q.ds = a2 - a1;
                    seg[b + 1] = q;
                }
                total += __shfl_sync(0xffffffffu, incl, 31);
            }
            __syncwarp();
            if (live) {
                // ---- units of each segment: cell k_s, and k_s + dk after the z crossing tz
#pragma unroll 4
                for (int s = 0; s < total; ++s) {
                    const uint4 raw = *reinterpret_cast<const uint4*>(&seg[s]);
                    Seg q;
                    q.ptr = ((unsigned long long)raw.y << 32) | raw.x;
                    q.se = __uint_as_float(raw.z);
                    q.ds = __uint_as_float(raw.w);
                    const bool cross = tz < q.se;
                    const float l_e = fmaxf(q.se - tz, 0.f);         // C_up - C_low, cell k_e
                    const float l_s = q.ds - l_e;                    // C_up - C_low, cell k_s
                    if (kAdjoint) {
                        atomicAdd((float*)(q.ptr + 4ull * kp), y * l_s);
                    } else {
                        acc_s = fmaf(__ldg((const float*)(q.ptr + 4ull * kp)), l_s, acc_s);
                    }
                    if (cross) {
                        kp += Z.dk;
                        if (kAdjoint) {
                            atomicAdd((float*)(q.ptr + 4ull * kp), y * l_e);
                        } else {
                            acc_e = fmaf(__ldg((const float*)(q.ptr + 4ull * kp)), l_e, acc_e);
                        }
                        mz += 1.f;
                        tz = fmaf(mz, Z.dtz, Z.t0z);
                    }
                }
            }
            __syncwarp();
        }
    }
    const float acc = acc_s + acc_e, acc2 = 0.f;
    if (!kAdjoint && r < dc.rows) sino_out[m] = (acc + acc2) * Z.scale;
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

int column_order() {
    static int o = [] {
        const char* e = getenv("XRT_COLUMN_ORDER");
        return e ? atoi(e) : 1;
    }();
    return o;
}

}  // namespace

// image [N_z][N_xy] -> padded z-fastest work [N_xy][NzP] (interior rows pad .. pad + N_z)
cudaError_t launch_to_zfast(const xrt_plan_s* p, const float* img, float* work, cudaStream_t s) {
    return transpose(img, work, p->grid.n[2], p->grid.nxy, p->grid.nxy, 0, p->nzp, p->zpad, s);
}

// padded z-fastest work [N_xy][NzP] -> image [N_z][N_xy]
cudaError_t launch_from_zfast(const xrt_plan_s* p, const float* work, float* img, cudaStream_t s) {
    return transpose(work, img, p->grid.nxy, p->grid.n[2], p->nzp, p->zpad, p->grid.nxy, 0, s);
}

cudaError_t launch_forward_column(const xrt_plan_s* p, const float* vol_zfast, float* sino,
                                  int64_t v0, int64_t v1, cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    const int rows_per_cta = kRowWarps * 32;
    const int ncg = (p->det.cols + kColsPerCta - 1) / kColsPerCta;
    const int nband = (p->det.rows + rows_per_cta - 1) / rows_per_cta;
    const unsigned nblk = (unsigned)((v1 - v0) * ncg * nband);
    k_column<false><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, vol_zfast, nullptr,
                                                nullptr, sino, (int)v0,
        (int)(v1 - v0), ncg, (int)p->nzp, (int)p->zpad, column_order());
    return cudaGetLastError();
}

cudaError_t launch_adjoint_column(const xrt_plan_s* p, const float* sino, float* vol_zfast,
                                  int64_t v0, int64_t v1, cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    const int rows_per_cta = kRowWarps * 32;
    const int ncg = (p->det.cols + kColsPerCta - 1) / kColsPerCta;
    const int nband = (p->det.rows + rows_per_cta - 1) / rows_per_cta;
    const unsigned nblk = (unsigned)((v1 - v0) * ncg * nband);
    k_column<true><<<nblk, kWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, nullptr, vol_zfast,
                                               sino, nullptr, (int)v0,
        (int)(v1 - v0), ncg, (int)p->nzp, (int)p->zpad, column_order());
    return cudaGetLastError();
}

}  // namespace xrt
