// kern_gather2d.cu -- the adjoint of the 2D beams (par2d, fan2d) as a pixel-driven GATHER
// (north_star: "a voxel-driven gather that reuses the same per-ray unit condition ...
// the faster variant is picked by measurement").  One thread per pixel (i, j); for every view the
// candidate detector columns come from the pixel's four corners projected on the detector (the
// fan / parallel family is monotone in u), and for each candidate the pixel's length on that ray
// is C_up - C_low of the slab intervals (eq:conditions_2D_1 P:180-187, eq:range_length P:217-220),
// with the half-open rule on a fixed axis.  No atomics; every pixel is written once.
#include <cuda_runtime.h>

#include <climits>

#include "xrt_internal.cuh"

namespace xrt {

namespace {

// Per-(view, column) ray in index space, from the paper's transforms in fp64 (paper_ray): the entry
// point of the image square, d u / d t, and for an axis-parallel ray the fp64 half-open cell of
// the fixed axis (so ties are decided exactly as the RAY kernels and the oracle decide them).
struct __align__(16) RayDesc2D {
    float ux0, uy0, wx, wy;   // u(t) = u0 + t w, t = physical length from the entry
    int flags;                // bit0 hit, bit1 x fixed, bit2 y fixed
    int fix;                  // fixed-axis cell (floor of its u, fp64)
    int pad0, pad1;
};

__global__ void k_raydesc2d(const ViewRec* __restrict__ views, DetC dc, GridC g, int64_t n,
                            RayDesc2D* __restrict__ out) {
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const int v = (int)(id / dc.cols), c = (int)(id - (int64_t)v * dc.cols);
    RayDesc2D d;
    d.flags = 0; d.fix = 0; d.pad0 = d.pad1 = 0;
    d.ux0 = d.uy0 = d.wx = d.wy = 0.f;
    Ray64 R;
    if (setup_ray(views[v], dc, g, 0, c, R)) {
        d.flags = 1 | (R.moving[0] ? 0 : 2) | (R.moving[1] ? 0 : 4);
        d.fix = !R.moving[0] ? R.cell[0] : (!R.moving[1] ? R.cell[1] : 0);
        d.ux0 = (float)(R.u0[0] + R.t_in * R.w[0]);
        d.uy0 = (float)(R.u0[1] + R.t_in * R.w[1]);
        d.wx = (float)R.w[0];
        d.wy = (float)R.w[1];
    }
    out[id] = d;
}

__global__ void __launch_bounds__(256) k_gather2d(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                  const RayDesc2D* __restrict__ desc,
                                                  const float* __restrict__ sino, float* __restrict__ img,
                                                  int n_views) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= g.n[0]) return;
    const bool par = dc.beam == XRT_PAR2D;
    const float x0 = (float)(g.x_lo + i * g.d[0]), x1 = (float)(g.x_lo + (i + 1) * g.d[0]);
    const float y1 = (float)(g.y_hi - j * g.d[1]), y0 = (float)(g.y_hi - (j + 1) * g.d[1]);
    const float inv_du = (float)(1.0 / dc.du), cu = (float)dc.cu, off_u = (float)dc.off_u;
    const float Df = (float)dc.D, sddf = (float)dc.sdd;
    const float fi = (float)i, fj = (float)j;
    float acc = 0.f;
    // pixel length on ray (v, c): C_up - C_low of the slab intervals (half-open fixed axis)
    auto unit = [&](int64_t m) -> float {
        const float4 q = __ldg(reinterpret_cast<const float4*>(desc + m));
        const int2 fl = __ldg(reinterpret_cast<const int2*>(desc + m) + 2);
        float lo = -INFINITY, hi = INFINITY;
        bool ok = fl.x & 1;
        if (fl.x & 2) {
            ok = ok && fl.y == i;
        } else {
            const float iw = __frcp_rn(q.z);
            const float a = (fi - q.x) * iw, b = (fi + 1.f - q.x) * iw;
            lo = fmaxf(lo, fminf(a, b)); hi = fminf(hi, fmaxf(a, b));
        }
        if (fl.x & 4) {
            ok = ok && fl.y == j;
        } else {
            const float iw = __frcp_rn(q.w);
            const float a = (fj - q.y) * iw, b = (fj + 1.f - q.y) * iw;
            lo = fmaxf(lo, fminf(a, b)); hi = fminf(hi, fmaxf(a, b));
        }
        return ok ? fmaxf(hi - lo, 0.f) : 0.f;
    };
#pragma unroll 4
    for (int v = 0; v < n_views; ++v) {
        const ViewRec V = views[v];
        const float c1 = (float)V.c1, s1 = (float)V.s1;
        // detector u of the pixel corners: par2d u = P . theta_perp; fan: the source is
        // S = -D e_d with e_d = (c1, s1), +u = (-s1, c1) (readings 7-9); flat u = sdd tan, curved
        // u = sdd * angle
        float umin = INFINITY, umax = -INFINITY;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float px = (t & 1) ? x1 : x0, py = (t & 2) ? y1 : y0;
            float u;
            if (par) {
                u = -px * s1 + py * c1;
            } else {
                const float ddx = px + Df * c1, ddy = py + Df * s1;
                const float a = -ddx * s1 + ddy * c1, b = ddx * c1 + ddy * s1;
                u = dc.curved ? sddf * atan2f(a, b) : sddf * __fdividef(a, b);
            }
            umin = fminf(umin, u);
            umax = fmaxf(umax, u);
        }
        const int c_lo = max(0, (int)ceilf((umin - off_u) * inv_du + cu - 0.01f));
        const int c_hi = min(dc.cols - 1, (int)floorf((umax - off_u) * inv_du + cu + 0.01f));
        const int64_t m0 = (int64_t)v * dc.cols;
        // the first three candidates without a data-dependent loop (independent loads), the rest
        // (pixels wider than ~2 detector bins) in a loop
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int c = c_lo + k;
            const bool in = c <= c_hi;
            const int cc = in ? c : c_lo;
            const float l = unit(m0 + cc);
            const float y = __ldg(sino + m0 + cc);
            acc = fmaf(y, in ? l : 0.f, acc);
        }
        for (int c = c_lo + 3; c <= c_hi; ++c) acc = fmaf(__ldg(sino + m0 + c), unit(m0 + c), acc);
    }
    img[(int64_t)j * g.n[0] + i] = acc;
}

}  // namespace

size_t raydesc2d_bytes() { return sizeof(RayDesc2D); }

cudaError_t launch_raydesc2d(const xrt_plan_s* p, cudaStream_t s) {
    const int64_t n = p->n_views * (int64_t)p->det.cols;
    k_raydesc2d<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(p->d_views, p->det, p->grid, n,
                                                             (RayDesc2D*)p->d_raydesc2d);
    return cudaGetLastError();
}

cudaError_t launch_adjoint_gather2d(const xrt_plan_s* p, const float* sino, float* img, cudaStream_t s) {
    dim3 grid((unsigned)((p->grid.n[0] + 255) / 256), (unsigned)p->grid.n[1]);
    k_gather2d<<<grid, 256, 0, s>>>(p->d_views, p->det, p->grid, (const RayDesc2D*)p->d_raydesc2d, sino, img,
                                     (int)p->n_views);
    return cudaGetLastError();
}

// ============================================================================ 2D slice kernels
// Forward and adjoint of the 2D beams with the 32 rays of a warp (32 adjacent detector columns of
// one view) walking the image in LOCKSTEP by major-axis slice (the paper's Algorithm 2.1 loop over
// the slices of one axis, with the valid band of the other index, eq:restriction_j
// P:197-212, found from the merged crossing values).  At every trip the lanes are in one slice, in
// adjacent cells of the minor axis, so their loads / reductions fall on consecutive addresses: the
// image is read (the adjoint accumulated) row-major for y-major warps and through a transposed copy
// for x-major warps.  Per ray the walk is the RAY kernel's: crossing values T(m) = t1 + m dt (FFMA)
// relative to the ray's entry, shared by the two units they separate; fixed axes half-open.
namespace {

struct Ray2S {
    float Ta, Tb;     // next crossing of the major / minor axis (relative to the entry)
    float ta1, tb1;   // first crossings
    float dta, dtb;   // spacings (0 when fixed)
    float ma, mb;     // crossings taken
    float tend;       // end of the chord
    int ca, cb;       // current major / minor cell
    int sa, sb;       // +-1 steps (0 when fixed)
};

template <bool kAdj>
__device__ __forceinline__ void slice_units(Ray2S& S, float& tc, float thi, const float* src, float* dst,
                                            int64_t row, float y, float& acc) {
    // units of one major slice: minor cells between tc and thi (a few; a ray steeper than the
    // warp's major axis crosses more)
    for (;;) {
        const float e = fminf(S.Tb, thi);
        const float l = e - tc;
        const int64_t addr = row + S.cb;
        if (kAdj) { if (l > 0.f) atomicAdd(dst + addr, y * l); }
        else acc = fmaf(__ldg(src + addr), l, acc);
        tc = e;
        if (!(S.Tb < thi)) break;
        S.mb += 1.f; S.Tb = fmaf(S.mb, S.dtb, S.tb1); S.cb += S.sb;
    }
}

#ifndef XRT_SLICE_WARPS
#define XRT_SLICE_WARPS 4   // cfg 2 slice adjoint 0.498 -> 0.487 ms vs 8
#endif
constexpr int kSliceWarps = XRT_SLICE_WARPS;
template <bool kAdj>
__global__ void __launch_bounds__(kSliceWarps * 32) k_slice2d(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                 const float* __restrict__ img, const float* __restrict__ imgT,
                                                 const float* __restrict__ y_in, float* __restrict__ sino_out,
                                                 float* __restrict__ acc_img, float* __restrict__ acc_imgT,
                                                 int n_views, int groups_per_view) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = blockIdx.x * kSliceWarps + warp;
    const int v = gid / groups_per_view, cgp = gid - v * groups_per_view;
    if (v >= n_views) return;                              // warp-uniform
    const int c = cgp * 32 + lane;
    const bool col_ok = c < dc.cols;
    Ray64 R;
    bool hit = false;
    if (col_ok) hit = setup_ray(views[v], dc, g, 0, c, R);
    const unsigned bh = __ballot_sync(0xffffffffu, hit);
    if (bh == 0u) {
        if (!kAdj && col_ok) sino_out[(int64_t)v * dc.cols + c] = 0.f;
        return;
    }
    // warp major axis by majority of the lanes' |w|
    const unsigned bx = __ballot_sync(0xffffffffu, hit && fabs(R.w[0]) >= fabs(R.w[1]));
    const int a = 2 * __popc(bx) >= __popc(bh) ? 0 : 1, b = 1 - a;
    Ray2S S;
    float y = 0.f;
    if (hit) {
        float T1[2], DT[2];
        int st[2];
        float tend = (float)(R.t_out - R.t_in);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            if (!R.moving[x]) { T1[x] = INFINITY; DT[x] = 0.f; st[x] = 0; continue; }
            const int pos = R.w[x] > 0.0;
            const int bf = pos ? R.cell[x] + 1 : R.cell[x];
            const int mface = pos ? (g.n[x] - bf) : bf;
            T1[x] = (float)(((double)bf - R.u0[x]) * R.inv_w[x] - R.t_in);
            DT[x] = (float)fabs(R.inv_w[x]);
            st[x] = pos ? 1 : -1;
            tend = fminf(tend, fmaf((float)mface, DT[x], T1[x]));   // never step through a face
        }
        S.ta1 = T1[a]; S.tb1 = T1[b]; S.dta = DT[a]; S.dtb = DT[b];
        S.Ta = S.ta1; S.Tb = S.tb1; S.ma = 0.f; S.mb = 0.f;
        S.ca = R.cell[a]; S.cb = R.cell[b]; S.sa = st[a]; S.sb = st[b];
        S.tend = tend;
        if (kAdj) y = y_in[(int64_t)v * dc.cols + c];
    }
    const float* src = a == 1 ? img : imgT;          // y-major: img[j][i]; x-major: imgT[i][j]
    float* dst = a == 1 ? acc_img : acc_imgT;
    const int64_t ld = a == 1 ? g.n[0] : g.n[1];
    // common direction of travel along the major axis
    const int dir = __shfl_sync(0xffffffffu, hit ? S.sa : 0, __ffs(bh) - 1);
    float acc = 0.f, tc = 0.f;
    bool live = hit;
    // a lane travelling against the warp's direction (or with a fixed major axis) walks its ray alone
    if (hit && (S.sa != dir || dir == 0)) {
        while (tc < S.tend) {
            const float thi = fminf(S.Ta, S.tend);
            slice_units<kAdj>(S, tc, thi, src, dst, (int64_t)S.ca * ld, y, acc);
            if (!(S.Ta <= S.tend)) break;
            S.ma += 1.f; S.Ta = fmaf(S.ma, S.dta, S.ta1); S.ca += S.sa;
        }
        live = false;
    }
    // lockstep range of major cells: the warp's entry cells to its exit cells (+-1)
    int kmin = INT_MAX, kmax = INT_MIN;
    if (live) {
        const int steps = S.tend > S.ta1 ? (int)floorf(__fdividef(S.tend - S.ta1, S.dta)) + 1 : 0;
        const int ex = max(0, min(g.n[a] - 1, S.ca + S.sa * steps));
        kmin = min(S.ca, ex); kmax = max(S.ca, ex);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (kmin <= kmax) {
        kmin = max(kmin - 1, 0);
        kmax = min(kmax + 1, g.n[a] - 1);
        const int ns = kmax - kmin + 1;
        const int k0 = dir > 0 ? kmin : kmax;
        for (int k = 0; k < ns; ++k) {
            const int M = k0 + dir * k;
            if (live && S.ca == M) {
                const float thi = fminf(S.Ta, S.tend);
                slice_units<kAdj>(S, tc, thi, src, dst, (int64_t)M * ld, y, acc);
                if (S.Ta <= S.tend && tc < S.tend) {
                    S.ma += 1.f; S.Ta = fmaf(S.ma, S.dta, S.ta1); S.ca += S.sa;
                } else {
                    live = false;
                }
            }
        }
    }
    if (!kAdj && col_ok) sino_out[(int64_t)v * dc.cols + c] = acc;
}

// ---------------------------------------------------------------------------------------------
// Slice adjoint v2 (AUTO on the 2D beams): the same lockstep walk, with at most TWO units per major
// slice for every lane whose ray is no steeper than the warp's major axis (|w_b| <= |w_a|: within one
// slice the minor coordinate changes by <= 1 cell, so the valid band of eq:restriction_j P:197-212 is
// {c_b, c_b + s_b}).  Per slice and lane, branch-free: the slice's span [t_lo, t_hi], the minor
// crossing T_b, cr = [T_b < t_hi], l_e = max(t_hi - T_b, 0) (C_up - C_low of the second unit,
// eq:range_length P:217-220), l_s = (t_hi - t_lo) - l_e.  Crossing values are T(m) = t1 + m dt (FFMA
// of the count, shared by the two units they separate): red.global.add of y l_s and (if cr) y l_e,
// the address of the minor cell a magic-float add (no conversion).  Lanes steeper than the major
// axis or travelling against the warp walk their rays alone (RAY walk).
constexpr float kMagic2 = 12582912.0f;          // 1.5 * 2^23: bits(kMagic2 + c) = 0x4B400000 + c
constexpr unsigned kMagicBits2 = 0x4B400000u;

__device__ __forceinline__ float gt0f(float x) {
    float r;
    asm("set.gt.f32.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void red_f(float* a, float v) {
    asm volatile("red.global.add.f32 [%0], %1;" :: "l"(a), "f"(v) : "memory");
}

#ifndef XRT_SLICE2_WARPS
#define XRT_SLICE2_WARPS 4
#endif
constexpr int kSlice2Warps = XRT_SLICE2_WARPS;

// (adjoint only: the forward variant on (f, f[+-1] - f) rows, and a variant staging 128^2 image
// tiles in shared memory, measured slower than the RAY forward on cfg 2 -- profiles/r2_2d.md)
__global__ void __launch_bounds__(kSlice2Warps * 32) k_slice2d_adj(const ViewRec* __restrict__ views, DetC dc, GridC g,
                                                 const float* __restrict__ y_in,
                                                 float* __restrict__ acc_img, float* __restrict__ acc_imgT,
                                                 int n_views, int groups_per_view) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = blockIdx.x * kSlice2Warps + warp;
    const int v = gid / groups_per_view, cgp = gid - v * groups_per_view;
    if (v >= n_views) return;                              // warp-uniform
    const int c = cgp * 32 + lane;
    Ray64 R;
    bool hit = false;
    if (c < dc.cols) hit = setup_ray(views[v], dc, g, 0, c, R);
    const unsigned bh = __ballot_sync(0xffffffffu, hit);
    if (bh == 0u) return;
    const unsigned bx = __ballot_sync(0xffffffffu, hit && fabs(R.w[0]) >= fabs(R.w[1]));
    const int a = 2 * __popc(bx) >= __popc(bh) ? 0 : 1, b = 1 - a;
    const int na = g.n[a], nb = g.n[b];
    // per-ray fp32 state relative to its entry (the RAY kernel's construction)
    float ta1 = INFINITY, dta = 0.f, tb1 = INFINITY, dtb = 0.f, tend = 0.f;
    int ca = 0, cb = 0, sa = 0, sb = 0;
    float y = 0.f;
    if (hit) {
        float T1[2], DT[2];
        int st[2];
        tend = (float)(R.t_out - R.t_in);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            if (!R.moving[x]) { T1[x] = INFINITY; DT[x] = 0.f; st[x] = 0; continue; }
            const int pos = R.w[x] > 0.0;
            const int bf = pos ? R.cell[x] + 1 : R.cell[x];
            const int mface = pos ? (g.n[x] - bf) : bf;
            T1[x] = (float)(((double)bf - R.u0[x]) * R.inv_w[x] - R.t_in);
            DT[x] = (float)fabs(R.inv_w[x]);
            st[x] = pos ? 1 : -1;
            tend = fminf(tend, fmaf((float)mface, DT[x], T1[x]));   // never step through a face
        }
        ta1 = T1[a]; tb1 = T1[b]; dta = DT[a]; dtb = DT[b];
        ca = R.cell[a]; cb = R.cell[b]; sa = st[a]; sb = st[b];
        y = y_in[(int64_t)v * dc.cols + c];
    }
    const int dir = __shfl_sync(0xffffffffu, hit ? sa : 0, __ffs(bh) - 1);
    // lanes that cannot take the lockstep walk: against the warp's direction, fixed major axis, or
    // steeper than the major axis (more than one minor crossing per slice): the RAY walk, alone
    const bool alone = hit && (sa != dir || dir == 0 || (sb != 0 && dtb < dta));
    if (alone && y != 0.f) {
        float tc = 0.f, Ta = ta1, Tb = tb1, ma = 0.f, mb = 0.f;
        int cca = ca, ccb = cb;
        for (int it = 0; it < na + nb + 2 && tc < tend; ++it) {
            const float tn = fminf(fminf(Ta, Tb), tend);
            const float l = tn - tc;
            const int64_t I = a == 1 ? (int64_t)cca * g.n[0] + ccb : (int64_t)ccb * g.n[0] + cca;   // y-major
            if (l > 0.f) red_f(acc_img + I, y * l);
            tc = tn;
            if (tn == Ta) { ma += 1.f; Ta = fmaf(ma, dta, ta1); cca += sa; }
            else if (tn == Tb) { mb += 1.f; Tb = fmaf(mb, dtb, tb1); ccb += sb; }
        }
    }
    const bool live = hit && !alone && y != 0.f;
    // lockstep slices: lane's first major cell ca, n_sl slices (1 + major crossings inside the chord)
    int n_sl = 0;
    if (live) {
        int m = tend > ta1 ? (int)((tend - ta1) / dta) : -1;
        m = max(-1, min(m, na));
        while (m + 1 <= na && fmaf((float)(m + 1), dta, ta1) < tend) ++m;
        while (m >= 0 && !(fmaf((float)m, dta, ta1) < tend)) --m;
        n_sl = m + 2;
    }
    int kfirst = live ? ca * dir : INT_MAX;   // position along dir
    int klast = live ? (ca + dir * (n_sl - 1)) * dir : INT_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kfirst = min(kfirst, __shfl_xor_sync(0xffffffffu, kfirst, o));
        klast = max(klast, __shfl_xor_sync(0xffffffffu, klast, o));
    }
    if (kfirst > klast) return;
    const int start = live ? ca * dir - kfirst : 0;     // lockstep trip at which this lane enters
    // minor cell as a magic float: address = row + 4 bits(cbf)
    float cbf = kMagic2 + (float)cb;
    const float sbf = (float)sb;
    const float ndtb = sb != 0 ? -dtb : 0.f;
    const float ntb0 = sb != 0 ? -tb1 : -1.0e30f;
    float ntb = ntb0;                        // -(next minor crossing)
    float mb = 0.f, t_lo = 0.f, ma = 0.f;
    float* acco = a == 1 ? acc_img : acc_imgT;   // y-major: img[j][i]; x-major: the transposed accumulator
    const long long rstep = (long long)dir * 4ll * nb;   // bytes per major step
    unsigned long long row = (unsigned long long)acco - 4ull * kMagicBits2 + (unsigned long long)((long long)ca * 4ll * nb);
    const int n_trips = klast - kfirst + 1;
    for (int k = 0; k < n_trips; ++k) {
        const int rel = k - start;
        if (live && (unsigned)rel < (unsigned)n_sl) {
            const float Ta = fmaf(ma, dta, ta1);
            const float t_hi = fminf(Ta, tend);
            const float dlt = t_hi - t_lo;
            const float le = t_hi + ntb;                    // t_hi - T_b
            const float cr = gt0f(le);
            const float lm = fmaxf(le, 0.f);
            float* p0 = (float*)(row + 4ull * __float_as_uint(cbf));
            red_f(p0, y * (dlt - lm));
            if (cr != 0.f) red_f(p0 + sb, y * lm);
            cbf = fmaf(cr, sbf, cbf);
            mb += cr;
            ntb = fmaf(mb, ndtb, ntb0);
            ma += 1.f;
            t_lo = t_hi;
            row += (unsigned long long)rstep;
        }
    }
}

}  // namespace

namespace {
// out[cols][rows] (+)= in[rows][cols]
template <bool kAdd>
__global__ void k_transpose2d(const float* __restrict__ in, float* __restrict__ out, int rows, int cols) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = by + j, c = bx + threadIdx.x;
        if (r < rows && c < cols) tile[j][threadIdx.x] = in[(int64_t)r * cols + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = bx + j, c = by + threadIdx.x;   // out row r (= in column), out column c
        if (r < cols && c < rows) {
            float* o = out + (int64_t)r * rows + c;
            *o = kAdd ? *o + tile[threadIdx.x][j] : tile[threadIdx.x][j];
        }
    }
}
}  // namespace

cudaError_t launch_transpose2d(const float* in, float* out, int rows, int cols, bool add, cudaStream_t s) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    if (add) k_transpose2d<true><<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols);
    else k_transpose2d<false><<<grid, dim3(32, 8), 0, s>>>(in, out, rows, cols);
    return cudaGetLastError();
}

cudaError_t launch_slice2d_adj(const xrt_plan_s* p, const float* y_in, float* acc_img, float* acc_imgT,
                               cudaStream_t s) {
    const int gpv = (p->det.cols + 31) / 32;
    const int64_t warps = p->n_views * (int64_t)gpv;
    const unsigned blocks = (unsigned)((warps + kSlice2Warps - 1) / kSlice2Warps);
    k_slice2d_adj<<<blocks, kSlice2Warps * 32, 0, s>>>(p->d_views, p->det, p->grid, y_in, acc_img, acc_imgT,
                                                      (int)p->n_views, gpv);
    return cudaGetLastError();
}

cudaError_t launch_slice2d(const xrt_plan_s* p, bool adjoint, const float* img, const float* imgT,
                           const float* y_in, float* sino_out, float* acc_img, float* acc_imgT,
                           cudaStream_t s) {
    const int gpv = (p->det.cols + 31) / 32;
    const int64_t warps = p->n_views * (int64_t)gpv;
    const unsigned blocks = (unsigned)((warps + kSliceWarps - 1) / kSliceWarps);
    if (adjoint)
        k_slice2d<true><<<blocks, kSliceWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, nullptr, nullptr, y_in, nullptr,
                                               acc_img, acc_imgT, (int)p->n_views, gpv);
    else
        k_slice2d<false><<<blocks, kSliceWarps * 32, 0, s>>>(p->d_views, p->det, p->grid, img, imgT, nullptr, sino_out,
                                                nullptr, nullptr, (int)p->n_views, gpv);
    return cudaGetLastError();
}

}  // namespace xrt
