// kern_ray.cu -- one thread per ray: forward (fp32), adjoint scatter (fp32 red.add) and the
// fp64 CSR count / fill passes.  Works for every beam and every direction (including the
// paper's Cases 2-4: axis-parallel and plane-parallel rays).
//
// The per-ray enumeration is the paper's method in incremental form.  Along each axis a with
// w_a != 0 the ray enters successive unit slabs at the crossing values
//     T_a(b) = (b - u0_a) / w_a                                   (the paper's C_x, C_y, C_z:
//                                                                  eq:C_xC_y P:170-172,
//                                                                  eq:C_xC_yC_z P:446-450)
// and a unit (i, j, k) is intersected non-vanishingly iff C_low < C_up with
// C_low = max of its slab entries, C_up = min of its slab exits (eq:conditions_2D_1 P:180-187,
// eq:conditions_3D_1 P:460-468).  Walking the three monotone crossing sequences in merged order
// visits exactly the units with C_low < C_up -- for a slice i of one axis, the units visited
// inside it are the valid band of the other index (eq:restriction_j P:197-212,
// eq:restriction_j_3D / eq:restriction_k_3D_1 P:479-499), found with one comparison per band
// member instead of a search -- and the length of the current unit is
//     l = C_up - C_low = (next crossing) - (previous crossing)   (eq:range_length P:217-220).
// Each crossing value is computed once and shared by the two units it separates
// ("telescoping", SURVEY hard part 1), which keeps fp32 sums accurate.  Axes with w_a == 0 keep
// the half-open cell floor(u0_a) (ties to the bigger index).
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "xrt_internal.cuh"

namespace xrt {

namespace {

// fp32 per-ray state, relative to t_in (all times >= 0).
struct Ray32 {
    float T[3];    // next crossing time per axis (INF if the axis is fixed)
    float t1[3];   // first crossing time
    float dt[3];   // crossing spacing 1/|w|
    float m[3];    // crossings taken so far
    int step[3];   // signed flat-index stride
    float tend;    // end of the last unit (<= the fp32 face-crossing time of every axis)
    int budget;    // 1 + number of interior crossings: hard cap on loop trips
    int64_t idx;   // flat index of the current unit
};

__device__ __forceinline__ void to_ray32(const Ray64& R, const GridC& g, Ray32& S) {
    const int64_t strides[3] = {1, (int64_t)g.n[0], g.nxy};
    float tend = (float)(R.t_out - R.t_in);
    int budget = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        S.m[a] = 0.f;
        if (!R.moving[a]) {
            S.T[a] = INFINITY;
            S.t1[a] = INFINITY;
            S.dt[a] = 0.f;
            S.step[a] = 0;
            continue;
        }
        const int pos = R.w[a] > 0.0;
        const int b_first = pos ? R.cell[a] + 1 : R.cell[a];
        const int m_face = pos ? (g.n[a] - b_first) : b_first;  // interior crossings before the face
        S.t1[a] = (float)(((double)b_first - R.u0[a]) * R.inv_w[a] - R.t_in);
        S.dt[a] = (float)fabs(R.inv_w[a]);
        S.step[a] = (int)(pos ? strides[a] : -strides[a]);
        S.T[a] = S.t1[a];
        budget += m_face;
        // the face crossing computed exactly as the loop would compute it: no axis can ever
        // step past its last interior boundary before tend (keeps every load in bounds)
        tend = fminf(tend, fmaf((float)m_face, S.dt[a], S.t1[a]));
    }
    S.tend = tend;
    S.budget = budget;
    S.idx = ((int64_t)R.cell[2] * g.n[1] + R.cell[1]) * g.n[0] + R.cell[0];
}

// Advance the axis whose crossing defined tn (one axis per call; ties advance on the next
// iteration with a zero-length unit in between).
__device__ __forceinline__ void advance(Ray32& S, float tn) {
    if (tn == S.T[0]) {
        S.m[0] += 1.f; S.T[0] = fmaf(S.m[0], S.dt[0], S.t1[0]); S.idx += S.step[0];
    } else if (tn == S.T[1]) {
        S.m[1] += 1.f; S.T[1] = fmaf(S.m[1], S.dt[1], S.t1[1]); S.idx += S.step[1];
    } else if (tn == S.T[2]) {
        S.m[2] += 1.f; S.T[2] = fmaf(S.m[2], S.dt[2], S.t1[2]); S.idx += S.step[2];
    }
}

__device__ __forceinline__ void ray_of(int64_t m, const DetC& dc, int& v, int& r, int& c) {
    const int64_t pv = dc.per_view;
    v = (int)(m / pv);
    const int64_t rem = m - (int64_t)v * pv;
    r = (int)(rem / dc.cols);
    c = (int)(rem - (int64_t)r * dc.cols);
}

#ifndef XRT_RAY_BS
#define XRT_RAY_BS 128   // cfg 2 forward 0.442 -> 0.426 ms vs 256 (tail balance of 2160 -> 4320 CTAs)
#endif
#ifndef XRT_RAY_MINB
#define XRT_RAY_MINB 1
#endif
__global__ void __launch_bounds__(XRT_RAY_BS, XRT_RAY_MINB) k_forward_ray(const ViewRec* __restrict__ views, DetC dc,
                                                      GridC g, const float* __restrict__ img,
                                                      float* __restrict__ sino, int64_t ray0,
                                                      int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    float acc = 0.f;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        Ray32 S;
        to_ray32(R, g, S);
        float tc = 0.f;
        for (int it = 0; tc < S.tend && it < S.budget; ++it) {
            const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
            acc = fmaf(__ldg(img + S.idx), tn - tc, acc);  // f_I * (C_up - C_low)
            tc = tn;
            advance(S, tn);
        }
    }
    sino[m] = acc;
}

// 2D beams: the same merged walk with two moving axes at most and a branch-free advance (the axis
// whose crossing defined tn steps; on a tie x first, y on the next trip after a zero-length unit --
// the generic walk's order), 32-bit cell index.  cfg 2 0.438 -> 0.412 ms (loading the next unit
// one trip ahead: 0.445; 64 / 256-thread blocks: 0.409 / 0.439, cfg 1 slower at 64).
#ifndef XRT_RAY2D_MINB
#define XRT_RAY2D_MINB 16   // 2048 threads per SM (32 registers): cfg 2 0.412 -> 0.389 ms
#endif
__global__ void __launch_bounds__(XRT_RAY_BS, XRT_RAY2D_MINB) k_forward_ray2d(const ViewRec* __restrict__ views, DetC dc,
                                                        GridC g, const float* __restrict__ img,
                                                        float* __restrict__ sino, int64_t ray0,
                                                        int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    float acc = 0.f;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        Ray32 S;
        to_ray32(R, g, S);
        float tx = S.T[0], ty = S.T[1], mx = 0.f, my = 0.f;
        const float t1x = S.t1[0], t1y = S.t1[1], dtx = S.dt[0], dty = S.dt[1], tend = S.tend;
        const int sx = S.step[0], sy = S.step[1];
        int idx = (int)S.idx;
        float tc = 0.f;
#pragma unroll 2
        for (int it = 0; tc < tend && it < S.budget; ++it) {
            const float tn = fminf(fminf(tx, ty), tend);
            acc = fmaf(__ldg(img + idx), tn - tc, acc);   // f_I * (C_up - C_low)
            tc = tn;
            const bool bx = tn == tx, by = !bx && tn == ty;
            mx = bx ? mx + 1.f : mx;
            my = by ? my + 1.f : my;
            tx = fmaf(mx, dtx, t1x);
            ty = fmaf(my, dty, t1y);
            idx += bx ? sx : (by ? sy : 0);
        }
    }
    sino[m] = acc;
}

// 2D beams, pieces: the same walk split into K pieces per ray along the major axis (the axis with
// the most crossings), one thread per piece, the K partial sums combined in shared memory in a fixed
// order.  Piece p covers major slices [p S, (p + 1) S) (S = ceil(slices / K); slice n spans
// [T_a(n - 1), T_a(n)], T_a(-1) = 0, T_a(n_a) = tend) and starts in the state the sequential walk has
// after taking major crossing p S - 1: the minor crossings T_b(m) < t_s taken (a minor crossing AT
// t_s is then taken on the first trip with a zero-length unit, as the sequential walk's tie order
// may do).  Every crossing value is the same fmaf(m, dt, t1) the sequential walk evaluates, so each
// unit's C_up - C_low is bit-identical to k_forward_ray2d's; only the summation order differs.
// The per-ray fp32 state (Ray2DW) is built once at plan creation (k_ray2d_walk_desc) from the fp64
// setup, so a piece costs a 32-byte load instead of the fp64 ray setup.
struct __align__(16) Ray2DW {
    float t1a, dta, t1b, dtb;   // major / minor first crossing and spacing (minor fixed: INF, 0)
    float tend;                 // end of the last unit (0: the ray misses the image)
    int idx0;                   // flat index of the entry unit (~index into imgT for x-major rays)
    int sa, sb;                 // signed flat strides of the major / minor axis (in the image walked)
};

__global__ void k_ray2d_walk_desc(const ViewRec* __restrict__ views, DetC dc, GridC g, int64_t n,
                                  Ray2DW* __restrict__ out) {
    const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray2DW d;
    d.t1a = d.t1b = INFINITY; d.dta = d.dtb = 0.f; d.tend = 0.f; d.idx0 = 0; d.sa = d.sb = 0;
    Ray64 R;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        Ray32 S;
        to_ray32(R, g, S);
        // major axis: the moving one with the smaller crossing spacing
        const int a = (S.step[0] != 0 && (S.step[1] == 0 || S.dt[0] <= S.dt[1])) ? 0 : 1, b = 1 - a;
        d.t1a = S.t1[a]; d.dta = S.dt[a];
        d.t1b = S.t1[b]; d.dtb = S.dt[b];
        d.tend = S.tend;
        const int cx = (int)(S.idx % g.n[0]), cy = (int)(S.idx / g.n[0]);
        if (a == 0) {
            // x-major: walk the transposed copy imgT[i][j] (flat i N_y + j), so the adjacent rays of a
            // warp, one x slice apart at most, read adjacent addresses; flagged by idx0 < 0
            d.idx0 = ~(cx * g.n[1] + cy);
            d.sa = S.step[0] > 0 ? g.n[1] : -g.n[1];
            d.sb = S.step[1] > 0 ? 1 : (S.step[1] < 0 ? -1 : 0);
        } else {
            d.idx0 = (int)S.idx;
            d.sa = S.step[1];
            d.sb = S.step[0];
        }
    }
    out[m] = d;
}

#ifndef XRT_RAY2D_PIECES
#define XRT_RAY2D_PIECES 4   // cfg 2 forward on f (transposed x-major walk) 0.363 / 0.301 / 0.280 / 0.282 ms at
                             // 1 / 2 / 4 / 8 pieces; on (f, delta f) 0.371 / 0.285 / 0.250 / 0.249 (AUTO: fd, 4)
#endif
#ifndef XRT_ADJ2D_PIECES
#define XRT_ADJ2D_PIECES 4   // pieces when the 2D adjoint in pieces is selected (not AUTO)
#endif
// One piece of a ray: forward (kAdj false) acc += f_I l_I; adjoint red.add of y l_I into the
// accumulator the ray walks (row-major for y-major rays, transposed for x-major rays).
template <int K, bool kAdj>
__device__ __forceinline__ float ray2d_piece(const Ray2DW* __restrict__ dsc, int64_t m, int p,
                                             const float* __restrict__ img, const float* __restrict__ imgT,
                                             float* acc_img, float* acc_imgT, float y) {
    float acc = 0.f;
    const float4 q0 = __ldg(reinterpret_cast<const float4*>(dsc + m));
    const int4 q1 = __ldg(reinterpret_cast<const int4*>(dsc + m) + 1);
    const float t1a = q0.x, dta = q0.y, t1b = q0.z, dtb = q0.w;
    const float tend = __int_as_float(q1.x);
    const int sa = q1.z, sb = q1.w;
    const bool tr = q1.y < 0;                       // x-major: the transposed copy
    const int idx0 = tr ? ~q1.y : q1.y;
    const float* __restrict__ src = tr ? imgT : img;
    float* dst = tr ? acc_imgT : acc_img;
    if (!(tend > 0.f)) return 0.f;
    // major crossings strictly inside (0, tend): the slices are nm + 1
    int nm = (int)((tend - t1a) / dta) + 1;
    nm = nm < 0 ? 0 : nm;
    while (nm > 0 && !(fmaf((float)(nm - 1), dta, t1a) < tend)) --nm;
    while (fmaf((float)nm, dta, t1a) < tend) ++nm;
    const int S = (nm + K) / K;
    const int s0 = p * S;
    if (s0 > nm) return 0.f;
    const int s1 = min(s0 + S, nm + 1);
    const float ts = s0 == 0 ? 0.f : fmaf((float)(s0 - 1), dta, t1a);
    const float te = s1 == nm + 1 ? tend : fmaf((float)(s1 - 1), dta, t1a);
    int mb = 0;
    float tb = INFINITY;
    int budget = s1 - s0 + 2;
    if (dtb > 0.f) {
        mb = (int)ceilf((ts - t1b) / dtb);
        mb = mb < 0 ? 0 : mb;
        while (mb > 0 && !(fmaf((float)(mb - 1), dtb, t1b) < ts)) --mb;
        while (fmaf((float)mb, dtb, t1b) < ts) ++mb;
        tb = fmaf((float)mb, dtb, t1b);
        budget += (int)((te - ts) / dtb) + 2;
    }
    int idx = idx0 + s0 * sa + mb * sb;
    float ma = (float)s0, mbf = (float)mb;
    float ta = fmaf(ma, dta, t1a);
    float tc = ts;
#pragma unroll 2
    for (int it = 0; tc < te && it < budget; ++it) {
        const float tn = fminf(fminf(ta, tb), te);
        if (kAdj) {   // unconditional: a zero-length unit (a tie) adds 0 to an in-image cell
            asm volatile("red.global.add.f32 [%0], %1;" :: "l"(dst + idx), "f"(y * (tn - tc)) : "memory");
        } else {
            acc = fmaf(__ldg(src + idx), tn - tc, acc);   // f_I * (C_up - C_low)
        }
        tc = tn;
        const bool ba = tn == ta, bb = !ba && tn == tb;
        ma = ba ? ma + 1.f : ma;
        mbf = bb ? mbf + 1.f : mbf;
        ta = fmaf(ma, dta, t1a);
        tb = fmaf(mbf, dtb, t1b);
        idx += ba ? sa : (bb ? sb : 0);
    }
    return acc;
}

template <int K>
__global__ void __launch_bounds__(XRT_RAY_BS, XRT_RAY2D_MINB) k_forward_ray2d_pc(const Ray2DW* __restrict__ dsc,
                                                                           const float* __restrict__ img,
                                                                           const float* __restrict__ imgT,
                                                                           float* __restrict__ sino, int64_t ray0,
                                                                           int64_t ray1) {
    // block = K groups of RB = XRT_RAY_BS / K adjacent rays; group p walks piece p of each (a warp's
    // lanes walk adjacent rays, as in the sequential kernel)
    constexpr int RB = XRT_RAY_BS / K;
    __shared__ float part[XRT_RAY_BS];
    const int p = (int)threadIdx.x / RB, rl = (int)threadIdx.x % RB;
    const int64_t m = ray0 + (int64_t)blockIdx.x * RB + rl;
    float acc = 0.f;
    if (m < ray1) acc = ray2d_piece<K, false>(dsc, m, p, img, imgT, nullptr, nullptr, 0.f);
    part[threadIdx.x] = acc;   // no early exit above: the block meets at the barrier
    __syncthreads();
    if (p == 0 && m < ray1) {
        float sum = part[rl];
#pragma unroll
        for (int q = 1; q < K; ++q) sum += part[q * RB + rl];   // fixed order: deterministic
        sino[m] = sum;
    }
}

// 2D forward in pieces on (f, delta f) images: per major slice n, [t_lo, t_hi] with t_hi = T_a(n) (the
// piece's last slice of the ray: tend), the minor crossing tau = T_b(m) decides cr = [tau < t_hi] and
// l_e = max(t_hi - tau, 0) (C_up - C_low of the second unit, eq:range_length P:217-220), and
//     acc += f(c) (t_hi - t_lo) + (f(c + s_b) - f(c)) l_e  =  f(c) l_s + f(c + s_b) l_e,
// one 8-byte load of (f, f[+-1] - f) per slice (the valid band of eq:restriction_j P:197-212 is
// {c_b, c_b + s_b} when |w_b| <= |w_a|).  Crossing values are the same fmaf(m, dt, t1) as the
// sequential walk's.  Rays within 2^-8 of 45 degrees (two minor crossings per slice possible in fp32)
// take the unit walk on the f components.  The four images (row-major / transposed x minor step
// +1 / -1) are built per call by k_fd2d.
__global__ void __launch_bounds__(256) k_fd2d(const float* __restrict__ img, float2* __restrict__ fd, int nx,
                                              int ny) {
    __shared__ float t[34][35];
    const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 34; r += 8)
        for (int q = threadIdx.x; q < 34; q += 32) {
            const int j = j0 - 1 + r, i = i0 - 1 + q;
            t[r][q] = (j >= 0 && j < ny && i >= 0 && i < nx) ? img[(int64_t)j * nx + i] : 0.f;
        }
    __syncthreads();
    const int64_t nxy = (int64_t)nx * ny;
    for (int r = threadIdx.y; r < 32; r += 8) {       // row-major, minor = x: lane = i
        const int j = j0 + r, i = i0 + (int)threadIdx.x;
        if (j < ny && i < nx) {
            const float f = t[r + 1][threadIdx.x + 1];
            fd[(int64_t)j * nx + i] = make_float2(f, t[r + 1][threadIdx.x + 2] - f);
            fd[nxy + (int64_t)j * nx + i] = make_float2(f, t[r + 1][threadIdx.x] - f);
        }
    }
    for (int r = threadIdx.y; r < 32; r += 8) {       // transposed [i][j], minor = y: lane = j
        const int i = i0 + r, j = j0 + (int)threadIdx.x;
        if (j < ny && i < nx) {
            const float f = t[threadIdx.x + 1][r + 1];
            fd[2 * nxy + (int64_t)i * ny + j] = make_float2(f, t[threadIdx.x + 2][r + 1] - f);
            fd[3 * nxy + (int64_t)i * ny + j] = make_float2(f, t[threadIdx.x][r + 1] - f);
        }
    }
}

constexpr float kMagicF = 12582912.0f;          // 1.5 * 2^23: bits(kMagicF + c) = 0x4B400000 + c (c < 2^22)
constexpr unsigned kMagicFBits = 0x4B400000u;

#ifndef XRT_RAY2D_FD_UNROLL
#define XRT_RAY2D_FD_UNROLL 4
#endif
constexpr int kFdUnroll2d = XRT_RAY2D_FD_UNROLL;
template <int K>
__device__ __forceinline__ float ray2d_piece_fd(const Ray2DW* __restrict__ dsc, int64_t m, int p,
                                                const float2* __restrict__ fd, int64_t nxy) {
    const float4 q0 = __ldg(reinterpret_cast<const float4*>(dsc + m));
    const int4 q1 = __ldg(reinterpret_cast<const int4*>(dsc + m) + 1);
    const float t1a = q0.x, dta = q0.y, dtb = q0.w;
    float t1b = q0.z;
    const float tend = __int_as_float(q1.x);
    const int sa = q1.z, sb = q1.w;
    const bool tr = q1.y < 0;
    const int idx0 = tr ? ~q1.y : q1.y;
    if (!(tend > 0.f)) return 0.f;
    int nm = (int)((tend - t1a) / dta) + 1;
    nm = nm < 0 ? 0 : nm;
    while (nm > 0 && !(fmaf((float)(nm - 1), dta, t1a) < tend)) --nm;
    while (fmaf((float)nm, dta, t1a) < tend) ++nm;
    const int S = (nm + K) / K;
    const int s0 = p * S;
    if (s0 > nm) return 0.f;
    const int s1 = min(s0 + S, nm + 1);
    const float ts = s0 == 0 ? 0.f : fmaf((float)(s0 - 1), dta, t1a);
    int mb = 0;
    if (dtb > 0.f) {
        mb = (int)ceilf((ts - t1b) / dtb);
        mb = mb < 0 ? 0 : mb;
        while (mb > 0 && !(fmaf((float)(mb - 1), dtb, t1b) < ts)) --mb;
        while (fmaf((float)mb, dtb, t1b) < ts) ++mb;
    } else {
        t1b = 1.0e30f;   // fixed minor axis: no crossing (finite, so l_e = d * 0 = 0)
    }
    const float2* __restrict__ img = fd + (tr ? 2 * nxy : 0) + (sb < 0 ? nxy : 0);
    const int idx = idx0 + s0 * sa + mb * sb;
    float acc0 = 0.f, acc1 = 0.f;
    if (dtb > 0.f && dtb < dta * (1.f + 1.f / 256.f)) {
        // near 45 degrees: the unit walk (ties: the major axis first, as the pieces walk)
        const float* __restrict__ f = reinterpret_cast<const float*>(img);
        const float te = s1 == nm + 1 ? tend : fmaf((float)(s1 - 1), dta, t1a);
        float ma = (float)s0, mbf = (float)mb;
        float ta = fmaf(ma, dta, t1a), tb = fmaf(mbf, dtb, t1b), tc = ts;
        int id = idx;
        const int budget = s1 - s0 + (int)((te - ts) / dtb) + 4;
        for (int it = 0; tc < te && it < budget; ++it) {
            const float tn = fminf(fminf(ta, tb), te);
            acc0 = fmaf(__ldg(f + 2 * (int64_t)id), tn - tc, acc0);
            tc = tn;
            const bool ba = tn == ta, bb = !ba && tn == tb;
            ma = ba ? ma + 1.f : ma;
            mbf = bb ? mbf + 1.f : mbf;
            ta = fmaf(ma, dta, t1a);
            tb = fmaf(mbf, dtb, t1b);
            id += ba ? sa : (bb ? sb : 0);
        }
        return acc0;
    }
    const unsigned long long base = (unsigned long long)img - 8ull * kMagicFBits;
    const float saf = (float)sa, sbf = (float)sb;
    float idxf = kMagicF + (float)idx, mbf = (float)mb, tb = fmaf(mbf, dtb, t1b), tlo = ts, nf = (float)s0;
    const int nlast = min(s1, nm);   // slices ending at a major crossing T_a(n)
#pragma unroll kFdUnroll2d
    for (int n = s0; n < nlast; ++n) {
        const float thi = fmaf(nf, dta, t1a);
        nf += 1.f;
        const float d = thi - tb;
        float cr;
        asm("mul.ftz.sat.f32 %0, %1, 0f7F000000;" : "=f"(cr) : "f"(d));   // [tau < t_hi]
        float2 v;
        asm("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(base + 8ull * __float_as_uint(idxf)));
        acc0 = fmaf(v.x, thi - tlo, acc0);
        acc1 = fmaf(v.y, d * cr, acc1);
        mbf += cr;
        tb = fmaf(mbf, dtb, t1b);
        idxf = fmaf(cr, sbf, idxf) + saf;
        tlo = thi;
    }
    if (s1 == nm + 1) {   // the ray's last slice ends at tend
        const float d = tend - tb;
        float cr;
        asm("mul.ftz.sat.f32 %0, %1, 0f7F000000;" : "=f"(cr) : "f"(d));
        float2 v;
        asm("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(base + 8ull * __float_as_uint(idxf)));
        acc0 = fmaf(v.x, tend - tlo, acc0);
        acc1 = fmaf(v.y, d * cr, acc1);
    }
    return acc0 + acc1;
}

template <int K>
__global__ void __launch_bounds__(XRT_RAY_BS, XRT_RAY2D_MINB) k_forward_ray2d_fd(const Ray2DW* __restrict__ dsc,
                                                                           const float2* __restrict__ fd,
                                                                           int64_t nxy, float* __restrict__ sino,
                                                                           int64_t ray0, int64_t ray1) {
    constexpr int RB = XRT_RAY_BS / K;
    __shared__ float part[XRT_RAY_BS];
    const int p = (int)threadIdx.x / RB, rl = (int)threadIdx.x % RB;
    const int64_t m = ray0 + (int64_t)blockIdx.x * RB + rl;
    float acc = 0.f;
    if (m < ray1) acc = ray2d_piece_fd<K>(dsc, m, p, fd, nxy);
    part[threadIdx.x] = acc;
    __syncthreads();
    if (p == 0 && m < ray1) {
        float sum = part[rl];
#pragma unroll
        for (int q = 1; q < K; ++q) sum += part[q * RB + rl];
        sino[m] = sum;
    }
}

// 2D slice adjoint in pieces (AUTO for the 2D beams): the lockstep slice adjoint of kern_gather2d.cu
// (k_slice2d_adj: a warp = 32 adjacent detector columns of one view walking major slice by major
// slice, at most two units per slice, reductions to consecutive addresses), its lockstep trips split
// into K pieces run by K warps (the r2k capture of k_slice2d_adj had 58 % warps active: warps of very
// different lengths).  A lane enters a piece in the state the walk has after its previous slices:
// slice n0, t_lo = T_a(n0 - 1), the minor crossings T_b(m) < t_lo taken (a crossing AT a slice end is
// taken in the next slice, le = t_hi - T_b > 0 there) -- the same fmaf values, so each unit's y l is
// bit-identical to the unsplit kernel's.  Per-ray fp32 state from the plan's Ray2DW descriptors (no
// fp64 setup per warp).  Lanes whose ray is steeper than the warp's major axis or travels against it
// walk their ray alone (piece 0 only).
template <int K>
__global__ void __launch_bounds__(128) k_slice2d_adj_pc(const Ray2DW* __restrict__ dsc, DetC dc, GridC g,
                                                       const float* __restrict__ y_in, float* __restrict__ acc_img,
                                                       float* __restrict__ acc_imgT, int n_views, int gpv) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * 128 + threadIdx.x) >> 5;
    const int p = (int)(gw % K);
    const int64_t grp = gw / K;
    const int v = (int)(grp / gpv), cgp = (int)(grp - (int64_t)v * gpv);
    if (v >= n_views) return;                               // warp-uniform
    const int c = cgp * 32 + lane;
    const int nx = g.n[0], ny = g.n[1];
    float t1a = INFINITY, dta = 0.f, t1b = INFINITY, dtb = 0.f, tend = 0.f, y = 0.f;
    int idx0 = 0, sa = 0, sb = 0;
    bool tr = false, hit = false;
    if (c < dc.cols) {
        const int64_t m = (int64_t)v * dc.cols + c;
        const float4 q0 = __ldg(reinterpret_cast<const float4*>(dsc + m));
        const int4 q1 = __ldg(reinterpret_cast<const int4*>(dsc + m) + 1);
        t1a = q0.x; dta = q0.y; t1b = q0.z; dtb = q0.w;
        tend = __int_as_float(q1.x);
        tr = q1.y < 0; idx0 = tr ? ~q1.y : q1.y; sa = q1.z; sb = q1.w;
        hit = tend > 0.f;
        y = __ldg(y_in + m);
    }
    const unsigned bh = __ballot_sync(0xffffffffu, hit);
    if (bh == 0u) return;
    // warp major axis by majority of the lanes' own major axes (x-major rays walk the transposed image)
    const unsigned bx = __ballot_sync(0xffffffffu, hit && tr);
    const bool wtr = 2 * __popc(bx) >= __popc(bh);
    const int len = wtr ? ny : nx;                          // walked row length (minor extent)
    const int sgn = sa > 0 ? 1 : -1;
    const unsigned bw = __ballot_sync(0xffffffffu, hit && tr == wtr);
    const int dir = __shfl_sync(0xffffffffu, hit && tr == wtr ? sgn : 0, bw ? __ffs(bw) - 1 : 0);   // common travel direction
    const bool alone = hit && (tr != wtr || sgn != dir || dir == 0);
    if (alone && p == 0 && y != 0.f) {
        // the ray's own unit walk (its own major axis, its own walked image)
        float* dst = tr ? acc_imgT : acc_img;
        float tc = 0.f, ta = t1a, tb = t1b, ma = 0.f, mbf = 0.f;
        int id = idx0;
        const int budget = (tr ? nx : ny) + (tr ? ny : nx) + 2;
        for (int it = 0; it < budget && tc < tend; ++it) {
            const float tn = fminf(fminf(ta, tb), tend);
            const float l = tn - tc;
            if (l > 0.f) asm volatile("red.global.add.f32 [%0], %1;" :: "l"(dst + id), "f"(y * l) : "memory");
            tc = tn;
            if (tn == ta) { ma += 1.f; ta = fmaf(ma, dta, t1a); id += sa; }
            else if (tn == tb) { mbf += 1.f; tb = fmaf(mbf, dtb, t1b); id += sb; }
        }
    }
    const bool live = hit && !alone && y != 0.f;
    const int ca = live ? idx0 / len : 0, cb = live ? idx0 - ca * len : 0;
    int n_sl = 0;
    if (live) {
        int m = (int)((tend - t1a) / dta) + 1;
        m = m < 0 ? 0 : m;
        while (m > 0 && !(fmaf((float)(m - 1), dta, t1a) < tend)) --m;
        while (fmaf((float)m, dta, t1a) < tend) ++m;
        n_sl = m + 1;
    }
    int kfirst = live ? ca * dir : INT_MAX;
    int klast = live ? (ca + dir * (n_sl - 1)) * dir : INT_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kfirst = min(kfirst, __shfl_xor_sync(0xffffffffu, kfirst, o));
        klast = max(klast, __shfl_xor_sync(0xffffffffu, klast, o));
    }
    if (kfirst > klast) return;
    const int n_trips = klast - kfirst + 1;
    const int B = (n_trips + K - 1) / K;
    const int k0 = p * B, k1 = min(n_trips, k0 + B);
    if (k0 >= k1) return;
    const int start = live ? ca * dir - kfirst : 0;        // lockstep trip of the lane's first slice
    const int n0 = max(k0 - start, 0);                     // the lane's first slice in this piece
    float mb = 0.f, t_lo = 0.f;
    if (live && n0 > 0 && n0 < n_sl) {
        t_lo = fmaf((float)(n0 - 1), dta, t1a);
        if (sb != 0) {
            int q = (int)ceilf((t_lo - t1b) / dtb);
            q = q < 0 ? 0 : q;
            while (q > 0 && !(fmaf((float)(q - 1), dtb, t1b) < t_lo)) --q;
            while (fmaf((float)q, dtb, t1b) < t_lo) ++q;
            mb = (float)q;
        }
    }
    float cbf = kMagicF + (float)(cb + (int)mb * sb);
    const float sbf = (float)sb;
    const float ndtb = sb != 0 ? -dtb : 0.f;
    const float ntb0 = sb != 0 ? -t1b : -1.0e30f;
    float ntb = fmaf(mb, ndtb, ntb0);
    float ma = (float)n0;
    float* acco = wtr ? acc_imgT : acc_img;
    const long long rstep = (long long)dir * 4ll * len;
    unsigned long long row = (unsigned long long)acco - 4ull * kMagicFBits +
                             (unsigned long long)((long long)(ca + dir * n0) * 4ll * len);
    for (int k = k0; k < k1; ++k) {
        const int rel = k - start;
        if (live && (unsigned)rel < (unsigned)n_sl) {
            const float Ta = fmaf(ma, dta, t1a);
            const float t_hi = fminf(Ta, tend);
            const float dlt = t_hi - t_lo;
            const float le = t_hi + ntb;                    // t_hi - T_b
            float cr;
            asm("set.gt.f32.f32 %0, %1, 0f00000000;" : "=f"(cr) : "f"(le));
            const float lm = fmaxf(le, 0.f);
            float* p0 = (float*)(row + 4ull * __float_as_uint(cbf));
            asm volatile("red.global.add.f32 [%0], %1;" :: "l"(p0), "f"(y * (dlt - lm)) : "memory");
            if (cr != 0.f) asm volatile("red.global.add.f32 [%0], %1;" :: "l"(p0 + sb), "f"(y * lm) : "memory");
            cbf = fmaf(cr, sbf, cbf);
            mb += cr;
            ntb = fmaf(mb, ndtb, ntb0);
            ma += 1.f;
            t_lo = t_hi;
            row += (unsigned long long)rstep;
        }
    }
}

// 2D adjoint in pieces (the forward's pieces and transposed x-major walk; scatter with red.add into
// acc_img / acc_imgT, summed by the plan's finishing transpose)
template <int K>
__global__ void __launch_bounds__(XRT_RAY_BS, XRT_RAY2D_MINB) k_adjoint_ray2d_pc(const Ray2DW* __restrict__ dsc,
                                                                           const float* __restrict__ sino,
                                                                           float* __restrict__ acc_img,
                                                                           float* __restrict__ acc_imgT, int64_t ray0,
                                                                           int64_t ray1) {
    constexpr int RB = XRT_RAY_BS / K;
    const int p = (int)threadIdx.x / RB, rl = (int)threadIdx.x % RB;
    const int64_t m = ray0 + (int64_t)blockIdx.x * RB + rl;
    if (m >= ray1) return;
    const float y = __ldg(sino + m);
    if (y == 0.f) return;
    ray2d_piece<K, true>(dsc, m, p, nullptr, nullptr, acc_img, acc_imgT, y);
}

__global__ void __launch_bounds__(256) k_adjoint_ray(const ViewRec* __restrict__ views, DetC dc,
                                                      GridC g, const float* __restrict__ sino,
                                                      float* __restrict__ img, int64_t ray0,
                                                      int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    const float y = sino[m];
    if (y == 0.f) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    if (!setup_ray(views[v], dc, g, r, c, R)) return;
    Ray32 S;
    to_ray32(R, g, S);
    float tc = 0.f;
    for (int it = 0; tc < S.tend && it < S.budget; ++it) {
        const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
        const float l = tn - tc;
        if (l > 0.f) atomicAdd(img + S.idx, y * l);
        tc = tn;
        advance(S, tn);
    }
}

// fp32 lengths / fp64 accumulation (SURVEY 8(f) N2's mixed mode): the fp32 walk of
// k_forward_ray (the same telescoped lengths C_up - C_low), products and sums in fp64 over fp64
// images / sinograms.  The adjoint walks the same lengths, so the pair is adjoint to fp64 rounding.
__global__ void __launch_bounds__(128) k_forward_mixed(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                       const double* __restrict__ img, double* __restrict__ sino,
                                                       int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    double acc = 0.0;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        Ray32 S;
        to_ray32(R, g, S);
        float tc = 0.f;
        for (int it = 0; tc < S.tend && it < S.budget; ++it) {
            const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
            acc = fma(__ldg(img + S.idx), (double)(tn - tc), acc);
            tc = tn;
            advance(S, tn);
        }
    }
    sino[m] = acc;
}

__global__ void __launch_bounds__(128) k_adjoint_mixed(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                       const double* __restrict__ sino, double* __restrict__ img,
                                                       int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    const double y = sino[m];
    if (y == 0.0) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    if (!setup_ray(views[v], dc, g, r, c, R)) return;
    Ray32 S;
    to_ray32(R, g, S);
    float tc = 0.f;
    for (int it = 0; tc < S.tend && it < S.budget; ++it) {
        const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
        const float l = tn - tc;
        if (l > 0.f) atomicAdd(img + S.idx, y * (double)l);
        tc = tn;
        advance(S, tn);
    }
}

// fp64 enumeration for the CSR dump: crossing values recomputed exactly as the clip computed
// the face values, so an axis never steps through the image face (see setup_ray).
template <bool kFill>
__device__ __forceinline__ int64_t units64(const Ray64& R, const GridC& g, int64_t* cols,
                                           double* lens) {
    int cell[3] = {R.cell[0], R.cell[1], R.cell[2]};
    double T[3];
    int bnd[3];
    int sgn[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!R.moving[a]) { T[a] = INFINITY; bnd[a] = 0; sgn[a] = 0; continue; }
        sgn[a] = R.w[a] > 0.0 ? 1 : -1;
        bnd[a] = sgn[a] > 0 ? cell[a] + 1 : cell[a];
        T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
    }
    double t = R.t_in;
    int64_t n = 0;
    const int budget = 2 + g.n[0] + g.n[1] + g.n[2];
    for (int it = 0; it < budget; ++it) {
        const double tn = fmin(fmin(T[0], T[1]), fmin(T[2], R.t_out));
        const double l = tn - t;  // C_up - C_low
        if (l > g.tau) {
            if (kFill) {
                cols[n] = ((int64_t)cell[2] * g.n[1] + cell[1]) * g.n[0] + cell[0];
                lens[n] = l;
            }
            ++n;
        }
        if (tn >= R.t_out) break;
        int a = (tn == T[0]) ? 0 : ((tn == T[1]) ? 1 : 2);
        cell[a] += sgn[a];
        bnd[a] += sgn[a];
        T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
        t = tn;
    }
    return n;
}

__global__ void __launch_bounds__(128) k_units_count(const ViewRec* __restrict__ views, DetC dc,
                                                      GridC g, int64_t ray0, int64_t ray1,
                                                      int64_t* __restrict__ counts) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = ray0 + i;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    int64_t n = 0;
    if (setup_ray(views[v], dc, g, r, c, R)) n = units64<false>(R, g, nullptr, nullptr);
    counts[i] = n;
}

__global__ void __launch_bounds__(128) k_units_fill(const ViewRec* __restrict__ views, DetC dc,
                                                     GridC g, int64_t ray0, int64_t ray1,
                                                     const int64_t* __restrict__ row_ptr,
                                                     int64_t* __restrict__ cols,
                                                     double* __restrict__ lens) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = ray0 + i;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        const int64_t o = row_ptr[i];
        units64<true>(R, g, cols + o, lens + o);
    }
}

// fp64 forward / adjoint (the paper's own precision option: "switching float ...
// into double"): the same fp64 enumeration as the CSR dump (units64), lengths and sums in
// double.  One thread per ray.
__global__ void __launch_bounds__(128) k_forward64(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                    const double* __restrict__ img, double* __restrict__ sino,
                                                    int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    double acc = 0.0;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        int cell[3] = {R.cell[0], R.cell[1], R.cell[2]};
        double T[3];
        int bnd[3], sgn[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (!R.moving[a]) { T[a] = INFINITY; bnd[a] = 0; sgn[a] = 0; continue; }
            sgn[a] = R.w[a] > 0.0 ? 1 : -1;
            bnd[a] = sgn[a] > 0 ? cell[a] + 1 : cell[a];
            T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
        }
        double t = R.t_in;
        const int budget = 2 + g.n[0] + g.n[1] + g.n[2];
        for (int it = 0; it < budget; ++it) {
            const double tn = fmin(fmin(T[0], T[1]), fmin(T[2], R.t_out));
            const double l = tn - t;   // C_up - C_low (eq:range_length_3D)
            if (l > g.tau) acc = fma(img[((int64_t)cell[2] * g.n[1] + cell[1]) * g.n[0] + cell[0]], l, acc);
            if (tn >= R.t_out) break;
            const int a = (tn == T[0]) ? 0 : ((tn == T[1]) ? 1 : 2);
            cell[a] += sgn[a];
            bnd[a] += sgn[a];
            T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
            t = tn;
        }
    }
    sino[m] = acc;
}

__global__ void __launch_bounds__(128) k_adjoint64(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                    const double* __restrict__ sino, double* __restrict__ img,
                                                    int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    const double y = sino[m];
    if (y == 0.0) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    if (!setup_ray(views[v], dc, g, r, c, R)) return;
    int cell[3] = {R.cell[0], R.cell[1], R.cell[2]};
    double T[3];
    int bnd[3], sgn[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!R.moving[a]) { T[a] = INFINITY; bnd[a] = 0; sgn[a] = 0; continue; }
        sgn[a] = R.w[a] > 0.0 ? 1 : -1;
        bnd[a] = sgn[a] > 0 ? cell[a] + 1 : cell[a];
        T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
    }
    double t = R.t_in;
    const int budget = 2 + g.n[0] + g.n[1] + g.n[2];
    for (int it = 0; it < budget; ++it) {
        const double tn = fmin(fmin(T[0], T[1]), fmin(T[2], R.t_out));
        const double l = tn - t;
        if (l > g.tau) atomicAdd(img + ((int64_t)cell[2] * g.n[1] + cell[1]) * g.n[0] + cell[0], y * l);
        if (tn >= R.t_out) break;
        const int a = (tn == T[0]) ? 0 : ((tn == T[1]) ? 1 : 2);
        cell[a] += sgn[a];
        bnd[a] += sgn[a];
        T[a] = ((double)bnd[a] - R.u0[a]) * R.inv_w[a];
        t = tn;
    }
}

// ---------------------------------------------------------------- attenuated transform (N4)
// R_Phi f with Phi = exp(-int_t^inf mu) (eq:generalizedRadontransform; DESIGN reading 23)
// for unit-basis f and mu: a unit I of length l contributes
//     f_I int_0^l exp(-(mu_I (l - s) + A_I)) ds = f_I exp(-A_I) (1 - exp(-mu_I l)) / mu_I,
// A_I the attenuation of the units after I along theta.  The walk runs along +theta (t grows from
// the source side to the detector side), the same unit walk as k_forward_ray.

// e = exp(-mu l) and the unit weight g = (1 - e) / mu = l phi(x), x = mu l, phi(x) = (1 - e^-x) / x
// (= l at mu = 0).  phi by its Taylor series for |x| <= 1/8 (truncation x^6 / 5040 < 1e-9; no
// cancellation in 1 - e), else by the quotient (cancellation <= 2^-24 / (1/8) relative).
__device__ __forceinline__ void att_unit(float mu, float l, float& e, float& gw) {
    const float x = mu * l;
    e = __expf(-x);
    float phi;
    if (fabsf(x) <= 0.125f)
        phi = fmaf(x, fmaf(x, fmaf(x, fmaf(x, fmaf(x, -1.f / 720.f, 1.f / 120.f), -1.f / 24.f), 1.f / 6.f), -0.5f), 1.f);
    else
        phi = __fdividef(1.f - e, x);
    gw = l * phi;
}

// forward: S_n = S_{n-1} exp(-mu_n l_n) + f_n g_n in path order, so every earlier unit picks up the
// attenuation of every later one (S_N = sum_I f_I exp(-A_I) g_I); no exponent can overflow.
__global__ void __launch_bounds__(256) k_forward_att(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                      const float* __restrict__ img, const float* __restrict__ mu,
                                                      float* __restrict__ sino, int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    float acc = 0.f;
    if (setup_ray(views[v], dc, g, r, c, R)) {
        Ray32 S;
        to_ray32(R, g, S);
        float tc = 0.f;
        for (int it = 0; tc < S.tend && it < S.budget; ++it) {
            const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
            float e, gw;
            att_unit(__ldg(mu + S.idx), tn - tc, e, gw);
            acc = fmaf(acc, e, __ldg(img + S.idx) * gw);
            tc = tn;
            advance(S, tn);
        }
    }
    sino[m] = acc;
}

// adjoint: pass 1 sums the ray's total attenuation A = sum mu l; pass 2 repeats the walk with the
// running sum A_le (through the end of the current unit) and scatters y exp(-(A - A_le)) g.  Both
// passes evaluate the same fmaf sequence, so A - A_le is exactly 0 on the last unit.
__global__ void __launch_bounds__(256) k_adjoint_att(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                      const float* __restrict__ sino, const float* __restrict__ mu,
                                                      float* __restrict__ img, int64_t ray0, int64_t ray1) {
    const int64_t m = ray0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= ray1) return;
    const float y = sino[m];
    if (y == 0.f) return;
    int v, r, c;
    ray_of(m, dc, v, r, c);
    Ray64 R;
    if (!setup_ray(views[v], dc, g, r, c, R)) return;
    Ray32 S;
    to_ray32(R, g, S);
    float A = 0.f, tc = 0.f;
    for (int it = 0; tc < S.tend && it < S.budget; ++it) {
        const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
        A = fmaf(__ldg(mu + S.idx), tn - tc, A);
        tc = tn;
        advance(S, tn);
    }
    to_ray32(R, g, S);
    float Ale = 0.f;
    tc = 0.f;
    for (int it = 0; tc < S.tend && it < S.budget; ++it) {
        const float tn = fminf(fminf(S.T[0], S.T[1]), fminf(S.T[2], S.tend));
        const float l = tn - tc;
        const float mui = __ldg(mu + S.idx);
        Ale = fmaf(mui, l, Ale);
        if (l > 0.f) {
            float e, gw;
            att_unit(mui, l, e, gw);
            atomicAdd(img + S.idx, y * __expf(Ale - A) * gw);
        }
        tc = tn;
        advance(S, tn);
    }
}

inline unsigned blocks_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

cudaError_t launch_forward_ray(const xrt_plan_s* p, const float* img, float* sino, int64_t ray0,
                               int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    const bool generic = std::getenv("XRT_RAY_GENERIC") != nullptr;   // (read per launch: tests toggle it)
    int pieces = XRT_RAY2D_PIECES;
    if (const char* e = std::getenv("XRT_RAY2D_PIECES")) pieces = std::atoi(e);   // experiments: 1, 2, 4, 8
    if (p->dim == 2 && !generic && ray2d_fd_on(p) && (pieces > 1 || pieces == -1)) {
        const unsigned nb = blocks_for((ray1 - ray0) * (pieces > 0 ? pieces : 1), XRT_RAY_BS);
        const Ray2DW* d = (const Ray2DW*)p->d_ray2d_walk;
        const int64_t nxy = p->grid.nxy;
        if (pieces == -1) k_forward_ray2d_fd<1><<<nb, XRT_RAY_BS, 0, s>>>(d, p->d_fd2d, nxy, sino, ray0, ray1);
        else if (pieces == 2) k_forward_ray2d_fd<2><<<nb, XRT_RAY_BS, 0, s>>>(d, p->d_fd2d, nxy, sino, ray0, ray1);
        else if (pieces == 8) k_forward_ray2d_fd<8><<<nb, XRT_RAY_BS, 0, s>>>(d, p->d_fd2d, nxy, sino, ray0, ray1);
        else k_forward_ray2d_fd<4><<<blocks_for((ray1 - ray0) * 4, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, p->d_fd2d, nxy, sino, ray0, ray1);
    } else if (p->dim == 2 && !generic && p->d_ray2d_walk && (pieces > 1 || pieces == -1)) {   // -1: one piece (A/B)
        const unsigned nb = blocks_for((ray1 - ray0) * pieces, XRT_RAY_BS);
        const Ray2DW* d = (const Ray2DW*)p->d_ray2d_walk;
        if (pieces == -1) k_forward_ray2d_pc<1><<<blocks_for(ray1 - ray0, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, img, p->d_fwd_t, sino, ray0, ray1);
        else if (pieces == 2) k_forward_ray2d_pc<2><<<nb, XRT_RAY_BS, 0, s>>>(d, img, p->d_fwd_t, sino, ray0, ray1);
        else if (pieces == 8) k_forward_ray2d_pc<8><<<nb, XRT_RAY_BS, 0, s>>>(d, img, p->d_fwd_t, sino, ray0, ray1);
        else k_forward_ray2d_pc<4><<<blocks_for((ray1 - ray0) * 4, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, img, p->d_fwd_t, sino, ray0, ray1);
    } else if (p->dim == 2 && !generic)
        k_forward_ray2d<<<blocks_for(ray1 - ray0, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(p->d_views, p->det, p->grid, img,
                                                                     sino, ray0, ray1);
    else
        k_forward_ray<<<blocks_for(ray1 - ray0, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(p->d_views, p->det, p->grid, img,
                                                                   sino, ray0, ray1);
    return cudaGetLastError();
}

// The 2D adjoint in pieces is an A/B option (XRT_ADJ2D_PIECES=K, read per launch): cfg 2 0.78 ms at
// K = 4 (1.01 / 0.88 / 0.80 at 1 / 2 / 8) vs 0.45 ms for the lockstep slice adjoint (AUTO), whose
// warps reduce into consecutive addresses; the free-running pieces' reductions do not coalesce.
bool adjoint2d_pieces(const xrt_plan_s* p) {
    const char* e = std::getenv("XRT_ADJ2D_PIECES");
    return p->d_ray2d_walk && e && std::atoi(e) > 0;
}

cudaError_t launch_adjoint_ray2d_pc(const xrt_plan_s* p, const float* sino, float* acc_img, float* acc_imgT,
                                    cudaStream_t s) {
    int pieces = XRT_ADJ2D_PIECES;
    if (const char* e = std::getenv("XRT_ADJ2D_PIECES")) pieces = std::atoi(e);
    const int64_t n = p->n_rays;
    const Ray2DW* d = (const Ray2DW*)p->d_ray2d_walk;
    if (pieces == 1) k_adjoint_ray2d_pc<1><<<blocks_for(n, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, sino, acc_img, acc_imgT, 0, n);
    else if (pieces == 2) k_adjoint_ray2d_pc<2><<<blocks_for(2 * n, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, sino, acc_img, acc_imgT, 0, n);
    else if (pieces == 8) k_adjoint_ray2d_pc<8><<<blocks_for(8 * n, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, sino, acc_img, acc_imgT, 0, n);
    else k_adjoint_ray2d_pc<4><<<blocks_for(4 * n, XRT_RAY_BS), XRT_RAY_BS, 0, s>>>(d, sino, acc_img, acc_imgT, 0, n);
    return cudaGetLastError();
}

#ifndef XRT_SLICE2D_PIECES
#define XRT_SLICE2D_PIECES 4
#endif
// 2D slice adjoint in pieces (AUTO when the plan has the walk descriptors; XRT_SLICE2D_PIECES=0:
// the unsplit k_slice2d_adj, read per launch)
bool slice2d_pieces_on(const xrt_plan_s* p) {
    const char* e = std::getenv("XRT_SLICE2D_PIECES");
    return p->d_ray2d_walk && !(e && std::atoi(e) == 0);
}

cudaError_t launch_slice2d_adj_pc(const xrt_plan_s* p, const float* y_in, float* acc_img, float* acc_imgT,
                                  cudaStream_t s) {
    int pieces = XRT_SLICE2D_PIECES;
    if (const char* e = std::getenv("XRT_SLICE2D_PIECES")) pieces = std::atoi(e);
    const int gpv = (p->det.cols + 31) / 32;
    const Ray2DW* d = (const Ray2DW*)p->d_ray2d_walk;
    const int64_t warps = p->n_views * (int64_t)gpv * pieces;
    const unsigned nb = blocks_for(warps * 32, 128);
    if (pieces == 1) k_slice2d_adj_pc<1><<<nb, 128, 0, s>>>(d, p->det, p->grid, y_in, acc_img, acc_imgT, (int)p->n_views, gpv);
    else if (pieces == 2) k_slice2d_adj_pc<2><<<nb, 128, 0, s>>>(d, p->det, p->grid, y_in, acc_img, acc_imgT, (int)p->n_views, gpv);
    else if (pieces == 8) k_slice2d_adj_pc<8><<<nb, 128, 0, s>>>(d, p->det, p->grid, y_in, acc_img, acc_imgT, (int)p->n_views, gpv);
    else k_slice2d_adj_pc<4><<<blocks_for(p->n_views * (int64_t)gpv * 4 * 32, 128), 128, 0, s>>>(d, p->det, p->grid, y_in, acc_img, acc_imgT, (int)p->n_views, gpv);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_ray(const xrt_plan_s* p, const float* sino, float* img, int64_t ray0,
                               int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_adjoint_ray<<<blocks_for(ray1 - ray0, 256), 256, 0, s>>>(p->d_views, p->det, p->grid, sino,
                                                               img, ray0, ray1);
    return cudaGetLastError();
}

cudaError_t launch_forward_att(const xrt_plan_s* p, const float* img, const float* mu, float* sino, int64_t ray0,
                               int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_forward_att<<<blocks_for(ray1 - ray0, 256), 256, 0, s>>>(p->d_views, p->det, p->grid, img, mu, sino, ray0,
                                                               ray1);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_att(const xrt_plan_s* p, const float* sino, const float* mu, float* img, int64_t ray0,
                               int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_adjoint_att<<<blocks_for(ray1 - ray0, 256), 256, 0, s>>>(p->d_views, p->det, p->grid, sino, mu, img, ray0,
                                                               ray1);
    return cudaGetLastError();
}

cudaError_t launch_forward64(const xrt_plan_s* p, const double* img, double* sino, int64_t ray0,
                             int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_forward64<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, img, sino, ray0, ray1);
    return cudaGetLastError();
}

cudaError_t launch_adjoint64(const xrt_plan_s* p, const double* sino, double* img, int64_t ray0,
                             int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_adjoint64<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, sino, img, ray0, ray1);
    return cudaGetLastError();
}

cudaError_t launch_forward_mixed(const xrt_plan_s* p, const double* img, double* sino, int64_t ray0,
                                 int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_forward_mixed<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, img, sino, ray0, ray1);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_mixed(const xrt_plan_s* p, const double* sino, double* img, int64_t ray0,
                                 int64_t ray1, cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_adjoint_mixed<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, sino, img, ray0, ray1);
    return cudaGetLastError();
}

size_t ray2d_walk_bytes() { return sizeof(Ray2DW); }

// the 2D forward in pieces on (f, delta f) images (AUTO; XRT_RAY2D_FD=0: on f, read per launch)
bool ray2d_fd_on(const xrt_plan_s* p) {
    const char* e = std::getenv("XRT_RAY2D_FD");
    return p->d_ray2d_walk && p->d_fd2d && !(e && std::atoi(e) == 0);
}

cudaError_t launch_fd2d(const xrt_plan_s* p, const float* img, cudaStream_t s) {
    const int nx = p->grid.n[0], ny = p->grid.n[1];
    k_fd2d<<<dim3((unsigned)((nx + 31) / 32), (unsigned)((ny + 31) / 32)), dim3(32, 8), 0, s>>>(img, p->d_fd2d, nx, ny);
    return cudaGetLastError();
}

cudaError_t launch_ray2d_walk_desc(const xrt_plan_s* p, cudaStream_t s) {
    k_ray2d_walk_desc<<<blocks_for(p->n_rays, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, p->n_rays,
                                                                 (Ray2DW*)p->d_ray2d_walk);
    return cudaGetLastError();
}

cudaError_t launch_units_count(const xrt_plan_s* p, int64_t ray0, int64_t ray1, int64_t* counts,
                               cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_units_count<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, ray0,
                                                               ray1, counts);
    return cudaGetLastError();
}

cudaError_t launch_units_fill(const xrt_plan_s* p, int64_t ray0, int64_t ray1,
                              const int64_t* row_ptr, int64_t* cols, double* lens,
                              cudaStream_t s) {
    if (ray1 <= ray0) return cudaSuccess;
    k_units_fill<<<blocks_for(ray1 - ray0, 128), 128, 0, s>>>(p->d_views, p->det, p->grid, ray0,
                                                              ray1, row_ptr, cols, lens);
    return cudaGetLastError();
}

}  // namespace xrt
