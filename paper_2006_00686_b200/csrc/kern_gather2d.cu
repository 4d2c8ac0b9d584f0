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

}  // namespace xrt
