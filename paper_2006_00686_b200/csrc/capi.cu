// capi.cu -- the extern "C" boundary declared in include/xrt.h: validation, the fp64 plan
// builder (per-view ray families), dispatch to the kernels, the host-buffer
// pipeline and the CSR dump (count -> scan -> fill -> per-row sort).
#include <cuda_runtime.h>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "xrt_internal.cuh"

// NVTX ranges around the entry points (header-only nvtx3: no library dependency; visible in nsys /
// ncu --nvtx when a tool is attached, no cost otherwise)
#include <nvtx3/nvToolsExt.h>

namespace {

struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;

xrt_status fail(xrt_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

xrt_status cuda_fail(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) return fail(XRT_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
    return fail(XRT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define XRT_CUDA(call)                                         \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
    } while (0)

struct DevGuard {
    int prev = -1, want;
    explicit DevGuard(int d) : want(d) {
        cudaGetDevice(&prev);
        if (prev != want) cudaSetDevice(want);
    }
    ~DevGuard() {
        if (prev >= 0 && prev != want) cudaSetDevice(prev);
    }
};


xrt_status validate(const xrt_geometry* g) {
    if (!g) return fail(XRT_ERR_INVALID_ARG, "geometry is NULL");
    if (g->flags & ~XRT_DET_CURVED) return fail(XRT_ERR_INVALID_ARG, "unknown flags 0x%x", (unsigned)g->flags);
    if (g->beam < XRT_PAR2D || g->beam > XRT_HELICAL) return fail(XRT_ERR_INVALID_ARG, "unknown beam %d", g->beam);
    const bool is2d = g->beam == XRT_PAR2D || g->beam == XRT_FAN2D;
    const bool divergent = g->beam == XRT_FAN2D || g->beam == XRT_CONE || g->beam == XRT_HELICAL;
    for (int a = 0; a < 3; ++a) {
        if (is2d && a == 2) continue;
        if (g->n[a] < 1) return fail(XRT_ERR_INVALID_ARG, "n[%d] = %lld must be >= 1", a, (long long)g->n[a]);
        if (g->n[a] > (1 << 20)) return fail(XRT_ERR_UNSUPPORTED, "n[%d] too large", a);
        if (!(std::isfinite(g->spacing[a]) && g->spacing[a] > 0))
            return fail(XRT_ERR_INVALID_ARG, "spacing[%d] must be finite and > 0", a);
        if (!std::isfinite(g->center[a])) return fail(XRT_ERR_INVALID_ARG, "center[%d] not finite", a);
    }
    if (is2d && g->n[2] != 1) return fail(XRT_ERR_INVALID_ARG, "2D beams need n[2] == 1");
    const long double vox = (long double)g->n[0] * g->n[1] * (is2d ? 1 : g->n[2]);
    if (vox > 4.0e9L) return fail(XRT_ERR_UNSUPPORTED, "image larger than 2^32 units");
    if (g->n_views < 1) return fail(XRT_ERR_INVALID_ARG, "n_views must be >= 1");
    if (!g->angles) return fail(XRT_ERR_INVALID_ARG, "angles is NULL");
    for (int64_t v = 0; v < g->n_views; ++v)
        if (!std::isfinite(g->angles[v])) return fail(XRT_ERR_INVALID_ARG, "angles[%lld] not finite", (long long)v);
    if (g->det_cols < 1 || g->det_rows < 1) return fail(XRT_ERR_INVALID_ARG, "detector dims must be >= 1");
    if (g->det_cols > INT_MAX || g->det_rows > INT_MAX) return fail(XRT_ERR_UNSUPPORTED, "detector too large");
    if (is2d && g->det_rows != 1) return fail(XRT_ERR_INVALID_ARG, "2D beams need det_rows == 1");
    for (int a = 0; a < 2; ++a) {
        if (!(std::isfinite(g->det_spacing[a]) && g->det_spacing[a] > 0))
            return fail(XRT_ERR_INVALID_ARG, "det_spacing[%d] must be finite and > 0", a);
        if (!std::isfinite(g->det_offset[a])) return fail(XRT_ERR_INVALID_ARG, "det_offset[%d] not finite", a);
    }
    if (divergent) {
        if (!(std::isfinite(g->sod) && g->sod > 0)) return fail(XRT_ERR_INVALID_ARG, "sod must be > 0");
        if (!(std::isfinite(g->sdd) && g->sdd > g->sod)) return fail(XRT_ERR_INVALID_ARG, "sdd must be > sod");
    }
    if ((g->flags & XRT_DET_CURVED) && !divergent)
        return fail(XRT_ERR_INVALID_ARG, "XRT_DET_CURVED needs a fan / cone / helical beam");
    if (g->flags & XRT_DET_CURVED) {
        const double half = ((g->det_cols - 1) / 2.0) * g->det_spacing[0] + std::fabs(g->det_offset[0]);
        if (!(half / g->sdd < M_PI / 2)) return fail(XRT_ERR_INVALID_ARG, "curved detector fan half-angle >= pi/2");
    }
    if (g->beam == XRT_HELICAL && !(std::isfinite(g->pitch) && std::isfinite(g->z0)))
        return fail(XRT_ERR_INVALID_ARG, "pitch / z0 not finite");
    if (g->beam == XRT_PAR3D && !(std::isfinite(g->tilt) && std::fabs(g->tilt) < M_PI / 2))
        return fail(XRT_ERR_INVALID_ARG, "tilt must satisfy |tilt| < pi/2");
    return XRT_OK;
}

// Per-view terms of the paper's beam -> parallel-beam transforms (xrt_internal.cuh; P:132-138,
// P:260-272; readings 7-11).  Evaluated with the host libm.
xrt::ViewRec view_record(const xrt_geometry* g, double ang) {
    xrt::ViewRec r;
    std::memset(&r, 0, sizeof r);
    double a = ang;
    if (g->beam == XRT_FAN2D) a = ang - M_PI / 2;  // phi = gamma + (alpha - pi/2)
    r.c1 = std::cos(a);
    r.s1 = std::sin(a);
    if (g->beam == XRT_PAR3D) {
        r.c2 = std::cos(g->tilt);
        r.s2 = std::sin(g->tilt);
        r.pad[0] = r.s2 / r.c2;
        r.pad[1] = 1.0 / r.c2;
    }
    if (g->beam == XRT_HELICAL) r.H = g->z0 + g->pitch * ang / (2.0 * M_PI);  // reading 11
    return r;
}

// z padding (per side) of the column kernels' z-fastest volume: every ray's u_z over the
// in-plane chord stays inside [-pad, N_z + pad).  Bound: |z| <= |z0| + R tan(beta) with R the
// largest distance of an image-square point from the z axis (|sigma_abs| <= R).
int64_t column_zpad(const xrt_geometry* g, const xrt::GridC& G) {
    const double hx = G.n[0] * G.d[0] / 2 + std::fabs(g->center[0]);
    const double hy = G.n[1] * G.d[1] / 2 + std::fabs(g->center[1]);
    const double R = std::sqrt(hx * hx + hy * hy);
    const double v0 = (0 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    const double v1 = ((g->det_rows - 1) - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    const double vmax = std::max(std::fabs(v0), std::fabs(v1));
    double zmax;
    if (g->beam == XRT_PAR3D) {
        const double c2 = std::cos(g->tilt), t2 = std::fabs(std::tan(g->tilt));
        zmax = vmax / c2 + R * t2;
    } else {
        const double hmax = vmax * g->sod / g->sdd;
        double Hmax = 0.0;
        if (g->beam == XRT_HELICAL)
            for (int64_t v = 0; v < g->n_views; ++v)
                Hmax = std::max(Hmax, std::fabs(g->z0 + g->pitch * g->angles[v] / (2.0 * M_PI)));
        zmax = hmax + Hmax + R * hmax / g->sod;
    }
    const double half = G.n[2] * G.d[2] / 2;
    const double over = (zmax + std::fabs(g->center[2]) - half) / G.d[2];
    int64_t pad = over > 0 ? (int64_t)std::ceil(over) : 0;
    return pad + 4;
}

// Physical z range [zlo, zhi] that the rays of detector rows [r0, r1] can reach (all views): z of a
// ray at in-plane distance rho from the source (divergent) or in-plane arc sigma (parallel) is affine
// in the row coordinate v, so the extreme rows and extreme rho bound it (+ the helical H range).
static void band_z_range(const xrt_geometry* g, const xrt::GridC& G, int64_t r0, int64_t r1, double& zlo,
                         double& zhi) {
    const double hx = G.n[0] * G.d[0] / 2 + std::fabs(g->center[0]);
    const double hy = G.n[1] * G.d[1] / 2 + std::fabs(g->center[1]);
    const double R = std::sqrt(hx * hx + hy * hy);
    const double v0 = (r0 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    const double v1 = (r1 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    if (g->beam == XRT_PAR3D) {
        const double c2 = std::cos(g->tilt), t2 = std::fabs(std::tan(g->tilt));
        zlo = std::min(v0, v1) / c2 - R * t2;
        zhi = std::max(v0, v1) / c2 + R * t2;
        return;
    }
    const double rmin = std::max(0.0, g->sod - R), rmax = g->sod + R;
    const double a[4] = {v0 * rmin / g->sdd, v0 * rmax / g->sdd, v1 * rmin / g->sdd, v1 * rmax / g->sdd};
    zlo = std::min(std::min(a[0], a[1]), std::min(a[2], a[3]));
    zhi = std::max(std::max(a[0], a[1]), std::max(a[2], a[3]));
    if (g->beam == XRT_HELICAL) {
        double hmin = INFINITY, hmax = -INFINITY;
        for (int64_t v = 0; v < g->n_views; ++v) {
            const double H = g->z0 + g->pitch * g->angles[v] / (2.0 * M_PI);
            hmin = std::min(hmin, H);
            hmax = std::max(hmax, H);
        }
        zlo += hmin;
        zhi += hmax;
    }
}

// Largest number of z cells that the rays of one band of `band_rows` detector rows can reach inside
// the image (over all views).  z of a ray at in-plane distance rho from the source (divergent) or at
// in-plane arc sigma (parallel) is affine in the row coordinate v, so the extreme rows and extreme
// rho bound it.  Used only to size the xy tiles (performance), never for correctness.
double column_band_slab(const xrt_geometry* g, const xrt::GridC& G, int band_rows) {
    const double hx = G.n[0] * G.d[0] / 2 + std::fabs(g->center[0]);
    const double hy = G.n[1] * G.d[1] / 2 + std::fabs(g->center[1]);
    const double R = std::sqrt(hx * hx + hy * hy);
    double worst = 0.0;
    for (int64_t r0 = 0; r0 < g->det_rows; r0 += band_rows) {
        const int64_t r1 = std::min<int64_t>(g->det_rows, r0 + band_rows) - 1;
        const double v0 = (r0 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
        const double v1 = (r1 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
        double zlo, zhi;
        if (g->beam == XRT_PAR3D) {
            const double c2 = std::cos(g->tilt), t2 = std::fabs(std::tan(g->tilt));
            zlo = std::min(v0, v1) / c2 - R * t2;
            zhi = std::max(v0, v1) / c2 + R * t2;
        } else {
            const double rmin = std::max(0.0, g->sod - R), rmax = g->sod + R;
            double a[4] = {v0 * rmin / g->sdd, v0 * rmax / g->sdd, v1 * rmin / g->sdd, v1 * rmax / g->sdd};
            zlo = std::min(std::min(a[0], a[1]), std::min(a[2], a[3]));
            zhi = std::max(std::max(a[0], a[1]), std::max(a[2], a[3]));
            if (g->beam == XRT_HELICAL) {
                double hmin = INFINITY, hmax = -INFINITY;
                for (int64_t v = 0; v < g->n_views; ++v) {
                    const double H = g->z0 + g->pitch * g->angles[v] / (2.0 * M_PI);
                    hmin = std::min(hmin, H);
                    hmax = std::max(hmax, H);
                }
                zlo += hmin;
                zhi += hmax;
            }
        }
        const double c = g->center[2], half = G.n[2] * G.d[2] / 2;
        zlo = std::max(zlo, c - half);
        zhi = std::min(zhi, c + half);
        worst = std::max(worst, (zhi - zlo) / G.d[2] + 1.0);
    }
    return worst;
}

// The column kernels split an in-plane segment at no more than one z plane: need
// max segment length (the in-plane unit diagonal) * max |d u_z / d sigma| < 1.
bool column_single_crossing(const xrt_geometry* g, const xrt::GridC& G) {
    const double v0 = (0 - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    const double v1 = ((g->det_rows - 1) - (g->det_rows - 1) / 2.0) * g->det_spacing[1] + g->det_offset[1];
    const double vmax = std::max(std::fabs(v0), std::fabs(v1));
    const double tanb = g->beam == XRT_PAR3D ? std::fabs(std::tan(g->tilt)) : vmax * g->sod / g->sdd / g->sod;
    const double diag = std::sqrt(G.d[0] * G.d[0] + G.d[1] * G.d[1]);
    return diag * tanb / G.d[2] < 0.999;
}

xrt_status alloc_stage(xrt_plan p) {
    if (!p->d_stage_img) XRT_CUDA(cudaMalloc(&p->d_stage_img, sizeof(float) * (size_t)p->grid.nxyz));
    if (!p->d_stage_sino) XRT_CUDA(cudaMalloc(&p->d_stage_sino, sizeof(float) * (size_t)p->n_rays));
    if (!p->aux_stream) {
        cudaStream_t s;
        XRT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        p->aux_stream = s;
    }
    if (!p->aux_stream2) {
        cudaStream_t s;
        XRT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        p->aux_stream2 = s;
    }
    if (!p->aux_stream3) {
        cudaStream_t s;
        XRT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        p->aux_stream3 = s;
    }
    return XRT_OK;
}

// AUTO, by measurement: 3D beams whose rays share an xy line per detector
// column -> COLUMN for both operators; 2D beams -> RAY forward (0.45 vs 0.51 ms, cfg 2) and the
// lockstep slice adjoint (0.50 vs 1.35 ms); anything else (ray lists, steep rays) -> RAY.
int resolve(const xrt_plan_s* p, int op) {
    const int want = op == XRT_OP_FORWARD ? p->algo_fwd : p->algo_adj;
    if (want != XRT_ALGO_AUTO) return want;
    if (p->column_ok) return XRT_ALGO_COLUMN;
    if (p->d_img_t && op == XRT_OP_ADJOINT) return XRT_ALGO_COLUMN;
    return XRT_ALGO_RAY;
}

// Forward over views [v0, v1).  COLUMN reads the plan's z-fastest copy of the image, which
// fwd_prepare() builds once per call (img -> work_fwd transpose).
xrt_status fwd_prepare(xrt_plan p, const float* img, cudaStream_t s) {
    if (resolve(p, XRT_OP_FORWARD) == XRT_ALGO_RAY && p->dim == 2 && p->d_fwd_t) {
        // 2D RAY forward in pieces: the (f, delta f) images, or x-major rays walk the transposed image
        cudaError_t e = xrt::ray2d_fd_on(p) ? xrt::launch_fd2d(p, img, s)
                                            : xrt::launch_transpose2d(img, p->d_fwd_t, p->grid.n[1], p->grid.n[0], false, s);
        p->launches += 1;
        if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
        return XRT_OK;
    }
    if (resolve(p, XRT_OP_FORWARD) != XRT_ALGO_COLUMN) return XRT_OK;
    if (p->dim == 2) {   // slice kernels: x-major warps read the transposed image
        cudaError_t e = xrt::launch_transpose2d(img, p->d_img_t, p->grid.n[1], p->grid.n[0], false, s);
        p->launches += 1;
        if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
        return XRT_OK;
    }
    if (p->fd_forward && xrt::fd_f4_on(p)) {
        if (!p->d_work_fd4) {   // first use: the interleaved z-mirror volume (same size as the fd volume), zeroed
            const size_t b4 = sizeof(float4) * (size_t)(p->grid.nxy * p->nzp);
            XRT_CUDA(cudaMalloc(&p->d_work_fd4, b4));
            XRT_CUDA(cudaMemsetAsync(p->d_work_fd4, 0, b4, s));
        }
        cudaError_t e = xrt::launch_to_fd4(p, img, p->d_work_fd4, s);
        p->launches += 1;
        if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
        return XRT_OK;
    }
    cudaError_t e = p->fd_forward ? xrt::launch_to_fd(p, img, p->d_work_fd, s) : xrt::launch_to_zfast(p, img, p->d_work_fwd, s);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
    return XRT_OK;
}

xrt_status forward_range(xrt_plan p, const float* img, float* sino, int64_t v0, int64_t v1,
                         cudaStream_t s) {
    const int64_t pv = p->det.per_view;
    const int algo = resolve(p, XRT_OP_FORWARD);
    cudaError_t e = cudaSuccess;
    if (algo == XRT_ALGO_RAY) {
        e = xrt::launch_forward_ray(p, img, sino, v0 * pv, v1 * pv, s);
    } else if (algo == XRT_ALGO_COLUMN && p->dim == 2) {
        if (!(v0 == 0 && v1 == p->n_views)) return fail(XRT_ERR_UNSUPPORTED, "2D slice kernels run all views at once");
        e = xrt::launch_slice2d(p, false, img, p->d_img_t, nullptr, sino, nullptr, nullptr, s);
    } else if (algo == XRT_ALGO_COLUMN && p->fd_forward) {
        if (!(v0 == 0 && v1 == p->n_views)) return fail(XRT_ERR_UNSUPPORTED, "column forward runs all views at once");
        e = xrt::launch_forward_fd_bands(p, p->d_work_fd, sino, 0, xrt::column_bands(p, false), s);
    } else if (algo == XRT_ALGO_COLUMN) {
        e = xrt::launch_forward_column(p, p->d_work_fwd, sino, v0, v1, s);
    } else {
        return fail(XRT_ERR_UNSUPPORTED, "forward algorithm %d not built", algo);
    }
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "forward launch");
    return XRT_OK;
}

// Adjoint: adj_begin() clears the accumulator, adjoint_range() adds views [v0, v1),
// adj_finish() writes the caller's image (COLUMN: work_adj -> img transpose).
xrt_status adj_begin(xrt_plan p, float* img, cudaStream_t s) {
    const int algo = resolve(p, XRT_OP_ADJOINT);
    if (algo == XRT_ALGO_GATHER) return XRT_OK;   // the gather writes every interior voxel
    const bool col = algo == XRT_ALGO_COLUMN && p->dim == 3;
    if (algo == XRT_ALGO_COLUMN && p->dim == 2)
        XRT_CUDA(cudaMemsetAsync(p->d_img_t, 0, sizeof(float) * (size_t)p->grid.nxy, s));
    if (col) XRT_CUDA(cudaMemsetAsync(p->d_work_adj, 0, sizeof(float) * (size_t)(p->grid.nxy * p->nzp), s));
    else XRT_CUDA(cudaMemsetAsync(img, 0, sizeof(float) * (size_t)p->grid.nxyz, s));
    return XRT_OK;
}

xrt_status adjoint_range(xrt_plan p, const float* sino, float* img, int64_t v0, int64_t v1,
                         cudaStream_t s) {
    const int64_t pv = p->det.per_view;
    const int algo = resolve(p, XRT_OP_ADJOINT);
    cudaError_t e = cudaSuccess;
    if (algo == XRT_ALGO_RAY) {
        e = xrt::launch_adjoint_ray(p, sino, img, v0 * pv, v1 * pv, s);
    } else if (algo == XRT_ALGO_COLUMN && p->dim == 2) {
        if (!(v0 == 0 && v1 == p->n_views)) return fail(XRT_ERR_UNSUPPORTED, "2D slice kernels run all views at once");
        e = p->slice_v1 ? xrt::launch_slice2d(p, true, nullptr, nullptr, sino, nullptr, img, p->d_img_t, s)
            : xrt::adjoint2d_pieces(p) ? xrt::launch_adjoint_ray2d_pc(p, sino, img, p->d_img_t, s)
            : xrt::slice2d_pieces_on(p) ? xrt::launch_slice2d_adj_pc(p, sino, img, p->d_img_t, s)
                                        : xrt::launch_slice2d_adj(p, sino, img, p->d_img_t, s);
    } else if (algo == XRT_ALGO_COLUMN) {
        e = xrt::launch_adjoint_column(p, sino, p->d_work_adj, v0, v1, s);
    } else if (algo == XRT_ALGO_GATHER) {
        if (!(v0 == 0 && v1 == p->n_views)) return fail(XRT_ERR_UNSUPPORTED, "gather adjoint runs all views at once");
        if (p->dim == 2) {
            e = xrt::launch_adjoint_gather2d(p, sino, img, s);
        } else {
            if (!p->d_gather_y)
                XRT_CUDA(cudaMalloc(&p->d_gather_y, sizeof(float) * (size_t)(p->gather_views * p->det.per_view)));
            e = xrt::launch_adjoint_gather(p, sino, p->d_work_adj, s);
            p->launches += xrt::gather_launches(p) - 1;
        }
    } else {
        return fail(XRT_ERR_UNSUPPORTED, "adjoint algorithm %d not built", algo);
    }
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "adjoint launch");
    return XRT_OK;
}

xrt_status adj_finish(xrt_plan p, float* img, cudaStream_t s) {
    const int algo = resolve(p, XRT_OP_ADJOINT);
    if (algo == XRT_ALGO_COLUMN && p->dim == 2) {   // img += transpose(x-major accumulator)
        cudaError_t e = xrt::launch_transpose2d(p->d_img_t, img, p->grid.n[0], p->grid.n[1], true, s);
        p->launches += 1;
        if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
        return XRT_OK;
    }
    if (algo != XRT_ALGO_COLUMN && !(algo == XRT_ALGO_GATHER && p->dim == 3)) return XRT_OK;
    cudaError_t e = xrt::launch_from_zfast(p, p->d_work_adj, img, s);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
    return XRT_OK;
}

xrt_status count_units(xrt_plan p, int64_t* out, cudaStream_t s) {
    const int64_t chunk = (int64_t)1 << 24;
    int64_t* d_counts = nullptr;
    int64_t* d_sum = nullptr;
    void* d_tmp = nullptr;
    size_t tmp_bytes = 0;
    XRT_CUDA(cub::DeviceReduce::Sum(nullptr, tmp_bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)chunk, s));
    XRT_CUDA(cudaMalloc(&d_counts, sizeof(int64_t) * chunk));
    XRT_CUDA(cudaMalloc(&d_sum, sizeof(int64_t)));
    XRT_CUDA(cudaMalloc(&d_tmp, tmp_bytes));
    int64_t total = 0;
    xrt_status st = XRT_OK;
    for (int64_t r0 = 0; r0 < p->n_rays && st == XRT_OK; r0 += chunk) {
        const int64_t r1 = std::min(p->n_rays, r0 + chunk);
        cudaError_t e = xrt::launch_units_count(p, r0, r1, d_counts, s);
        p->launches += 1;
        if (e == cudaSuccess) e = cub::DeviceReduce::Sum(d_tmp, tmp_bytes, d_counts, d_sum, (int)(r1 - r0), s);
        int64_t part = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&part, d_sum, sizeof part, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_fail(e, "count_units");
        total += part;
    }
    cudaFree(d_counts);
    cudaFree(d_sum);
    cudaFree(d_tmp);
    if (st == XRT_OK) *out = total;
    return st;
}

}  // namespace

extern "C" {

int32_t xrt_version(void) { return (XRT_VERSION_MAJOR << 16) | XRT_VERSION_MINOR; }

const char* xrt_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace {
// rays != nullptr: an explicit ray list (xrt_plan_create_rays) laid out as one view of n_rays
// detector columns; only the RAY kernel family serves it.
xrt_status plan_create_impl(const xrt_geometry* g, int cuda_device, xrt_plan* out, const double* rays,
                            int ray_dim) {
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
        return fail(XRT_ERR_INVALID_ARG, "cuda_device %d not available (%d devices)", cuda_device, ndev);
    DevGuard guard(cuda_device);
    xrt_plan p = new (std::nothrow) xrt_plan_s();
    if (!p) return fail(XRT_ERR_OOM, "host allocation");
    const bool is2d = g->beam == XRT_PAR2D || g->beam == XRT_FAN2D;
    p->device = cuda_device;
    p->beam = g->beam;
    p->dim = is2d ? 2 : 3;
    xrt::GridC& G = p->grid;
    for (int a = 0; a < 3; ++a) {
        G.n[a] = (int)(is2d && a == 2 ? 1 : g->n[a]);
        G.d[a] = is2d && a == 2 ? 1.0 : g->spacing[a];
    }
    const double cz = is2d ? 0.0 : g->center[2];
    G.x_lo = g->center[0] - G.n[0] * G.d[0] / 2.0;
    G.y_hi = g->center[1] + G.n[1] * G.d[1] / 2.0;
    G.z_hi = cz + G.n[2] * G.d[2] / 2.0;
    G.tau = 1e-9 * std::min(G.d[0], std::min(G.d[1], is2d ? G.d[0] : G.d[2]));
    G.inv_dz = 1.0 / G.d[2];
    G.nxy = (int64_t)G.n[0] * G.n[1];
    G.nxyz = G.nxy * G.n[2];
    xrt::DetC& D = p->det;
    D.beam = g->beam;
    D.curved = (g->flags & XRT_DET_CURVED) ? 1 : 0;
    D.D = g->sod;
    D.sdd = g->sdd;
    D.inv_D = g->sod > 0 ? 1.0 / g->sod : 0.0;
    D.cols = (int)g->det_cols;
    D.rows = (int)g->det_rows;
    D.du = g->det_spacing[0];
    D.dv = g->det_spacing[1];
    D.cu = (g->det_cols - 1) / 2.0;
    D.cv = (g->det_rows - 1) / 2.0;
    D.off_u = g->det_offset[0];
    D.off_v = is2d ? 0.0 : g->det_offset[1];
    D.per_view = (int64_t)D.cols * D.rows;
    p->n_views = g->n_views;
    p->n_rays = D.per_view * g->n_views;
    std::vector<xrt::ViewRec> views((size_t)g->n_views);
    for (int64_t v = 0; v < g->n_views; ++v) views[v] = view_record(g, g->angles[v]);
    cudaError_t e = cudaMalloc(&p->d_views, sizeof(xrt::ViewRec) * views.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_views, views.data(), sizeof(xrt::ViewRec) * views.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        xrt_plan_destroy(p);
        return cuda_fail(e, "plan tables");
    }
    if (rays) {
        // explicit rays (Remark 3.5): per-ray paper parameters in a device table
        p->beam = XRT_RAYS;
        D.beam = XRT_RAYS;
        D.ray_dim = ray_dim;
        e = cudaMalloc(&p->d_rays, sizeof(double) * 4 * (size_t)p->n_rays);
        if (e == cudaSuccess)
            e = cudaMemcpy(p->d_rays, rays, sizeof(double) * 4 * (size_t)p->n_rays, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            xrt_plan_destroy(p);
            return cuda_fail(e, "ray table");
        }
        D.rays = p->d_rays;
    }
    if (!rays && (g->beam == XRT_PAR2D || g->beam == XRT_FAN2D)) {
        // 2D gather: per-(view, column) rays in index space
        e = cudaMalloc(&p->d_raydesc2d, xrt::raydesc2d_bytes() * (size_t)(p->n_views * D.cols));
        if (e == cudaSuccess) e = cudaMalloc(&p->d_img_t, sizeof(float) * (size_t)G.nxy);
        p->slice_v1 = std::getenv("XRT_SLICE_V1") != nullptr;
        if (e == cudaSuccess) e = xrt::launch_raydesc2d(p, (cudaStream_t)0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            xrt_plan_destroy(p);
            return cuda_fail(e, "2D ray descriptors");
        }
    }
    if (p->dim == 2 && (int64_t)p->n_rays < (1ll << 26)) {
        // 2D RAY forward in pieces: per-ray fp32 walk state (32 B per ray; cfg 2: 17.7 MB)
        e = cudaMalloc(&p->d_ray2d_walk, xrt::ray2d_walk_bytes() * (size_t)p->n_rays);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_fwd_t, sizeof(float) * (size_t)G.nxy);
        if (e == cudaSuccess && G.nxy < (1ll << 22))   // magic-float cell index: < 2^22 cells
            e = cudaMalloc(&p->d_fd2d, 4 * sizeof(float2) * (size_t)G.nxy);
        if (e == cudaSuccess) e = xrt::launch_ray2d_walk_desc(p, (cudaStream_t)0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            xrt_plan_destroy(p);
            return cuda_fail(e, "2D walk descriptors");
        }
    }
    p->column_ok = !rays && (g->beam == XRT_PAR3D || g->beam == XRT_CONE || g->beam == XRT_HELICAL) &&
                   column_single_crossing(g, G);
    if (p->column_ok) {
        p->zpad = column_zpad(g, G);
        p->col_np = xrt::choose_col_np(D.rows);
        p->col_np_adj = 1;
        if (const char* e = std::getenv("XRT_COL_NP_ADJ")) {   // experiments: 1 or 2 pairs per lane
            const int v = std::atoi(e);
            if (v == 1 || v == 2) p->col_np_adj = v;
        }
        p->nzp = (G.n[2] + 2 * p->zpad + 3) / 4 * 4;   // 16-byte cell columns (vector reds); tail rows stay 0
        const size_t bytes = sizeof(float) * (size_t)(G.nxy * p->nzp);
        e = cudaMalloc(&p->d_work_fwd, bytes);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_work_adj, bytes);
        if (e == cudaSuccess) e = cudaMemset(p->d_work_fwd, 0, bytes);  // zero padding stays zero
        // forward on the (f, delta f) volume, except where no ray crosses a z plane (3D parallel beam
        // without tilt: the legacy kernel's flat walk, one 4-byte load per unit, is faster there)
        p->fd_forward = !std::getenv("XRT_FWD_LEGACY") && !(g->beam == XRT_PAR3D && g->tilt == 0.0);
        p->flat_z = g->beam == XRT_PAR3D && g->tilt == 0.0;
        // circular cone symmetric in z (grid centred at z = 0, detector rows centred): the fd forward
        // walks the upper rows and accumulates their mirror images from the same z state (k_fwd_fd<NP, true>)
        p->fd_mirror = p->fd_forward && g->beam == XRT_CONE && g->center[2] == 0.0 && D.off_v == 0.0 &&
                       D.rows >= 2 && !std::getenv("XRT_NO_MIRROR");
        if (e == cudaSuccess && p->fd_forward) {
            const size_t fdb = 2 * sizeof(float2) * (size_t)(G.nxy * p->nzp);
            e = cudaMalloc(&p->d_work_fd, fdb);
            if (e == cudaSuccess) e = cudaMemset(p->d_work_fd, 0, fdb);   // padding beyond the edge rows stays 0
        }
        if (e == cudaSuccess)
            e = cudaMalloc(&p->d_coldesc, xrt::column_desc_bytes() * (size_t)(p->n_views * D.cols));
        if (e == cudaSuccess) e = xrt::launch_col_desc(p, (cudaStream_t)0);
        // gather workspace: one block of views of the rescaled, transposed sinogram (~40 MB, so the
        // block stays L2-resident while every voxel reads it)
        p->gather_views = std::max<int64_t>(1, std::min<int64_t>(g->n_views, (40ll << 20) / (4 * D.per_view)));
        // (the gather's workspace, ~40 MB, is allocated on first use: AUTO never runs the gather)
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        // xy tiling, per operator: the largest power-of-two tile whose z-fastest columns, restricted
        // to the z slab one band of detector rows can reach (the kernels run band-major), fit the
        // operator's budget, 64 MB for both (cfg 4: 256^2 tiles).  Measured alternative for the
        // adjoint: untiled in xy (budget >= 160 MB) runs 3 % faster on cfg 4 (197.6 vs 203.8 ms) but
        // writes 58 GB of partially reduced lines back to DRAM per launch instead of 7.6 GB
        // (profiles/r1d_cfg4.md); the L2-resident tiling is kept.
        for (int op = 0; op < 2 && e == cudaSuccess; ++op) {
            const char* env = std::getenv(op ? "XRT_ADJ_L2_MB" : "XRT_FWD_L2_MB");
            const double budget = (env ? std::atof(env) : 64.0) * 1024 * 1024;
            const int rows = 64 * (op ? p->col_np_adj : p->col_np);
            const double slab = std::min((double)p->nzp, column_band_slab(g, G, rows) + 2.0);
            // bytes per cell one band touches: 8 on the forward's (f, delta f) volume (one half per
            // row direction), 4 on the float z-fastest copies; the fewest tiles per axis that fit
            const double cell_bytes = (op == 0 && p->fd_forward) ? 8.0 : 4.0;
            const int nmax = std::max(G.n[0], G.n[1]);
            int ts = nmax;
            for (int nt = 1; ts > 32; ++nt) {
                ts = (nmax + nt - 1) / nt;
                if ((double)ts * ts * slab * cell_bytes <= budget) break;
            }
            if (const char* f = std::getenv("XRT_COLUMN_TILE")) ts = std::max(4, std::atoi(f));  // testing
            xrt_plan_s::ColTiling& T = p->ct[op];
            if (ts >= std::max(G.n[0], G.n[1])) {
                T.tile = std::max(G.n[0], G.n[1]);
                T.n_tx = T.n_ty = 1;
            } else {
                T.tile = ts;
                T.n_tx = (G.n[0] + ts - 1) / ts;
                T.n_ty = (G.n[1] + ts - 1) / ts;
                std::vector<uint2> items;
                xrt::build_column_items(p, views.data(), T.tile, T.n_tx, T.n_ty, items);
                T.n_items = (int64_t)items.size();
                if (!items.empty()) e = cudaMalloc(&T.d_items, sizeof(uint2) * items.size());
                if (e == cudaSuccess && !items.empty())
                    e = cudaMemcpy(T.d_items, items.data(), sizeof(uint2) * items.size(), cudaMemcpyHostToDevice);
                constexpr int Q = xrt_plan_s::kFwdParts;
                if (op == 1 && e == cudaSuccess && !items.empty() && p->n_views >= Q) {
                    // the adjoint items regrouped by view range (item .x = view), tile order kept
                    std::vector<uint2> parts;
                    parts.reserve(items.size());
                    for (int q = 0; q < Q; ++q) {
                        const int64_t v0 = p->n_views * q / Q, v1 = p->n_views * (q + 1) / Q;
                        p->adj_part_off[q] = (int64_t)parts.size();
                        p->adj_part_view[q] = v0;
                        for (const uint2& w : items)
                            if ((int64_t)w.x >= v0 && (int64_t)w.x < v1) parts.push_back(w);
                    }
                    p->adj_part_off[Q] = (int64_t)parts.size();
                    p->adj_part_view[Q] = p->n_views;
                    e = cudaMalloc(&p->d_adj_part_items, sizeof(uint2) * parts.size());
                    if (e == cudaSuccess)
                        e = cudaMemcpy(p->d_adj_part_items, parts.data(), sizeof(uint2) * parts.size(),
                                       cudaMemcpyHostToDevice);
                }
                if (op == 0 && p->fd_forward && e == cudaSuccess) {   // the fd forward's CTAs: views x columns
                    xrt_plan_s::ColTiling& F = p->ct_fd;
                    F.tile = T.tile; F.n_tx = T.n_tx; F.n_ty = T.n_ty;
                    xrt::build_column_items(p, views.data(), T.tile, T.n_tx, T.n_ty, items, true);
                    F.n_items = (int64_t)items.size();
                    if (!items.empty()) e = cudaMalloc(&F.d_items, sizeof(uint2) * items.size());
                    if (e == cudaSuccess && !items.empty())
                        e = cudaMemcpy(F.d_items, items.data(), sizeof(uint2) * items.size(), cudaMemcpyHostToDevice);
                    // the same items regrouped by view range (parts of whole view blocks), tile order kept
                    const int64_t VBk = xrt::fd_view_block();
                    const int64_t nvb = (p->n_views + VBk - 1) / VBk;
                    if (e == cudaSuccess && !items.empty() && nvb >= Q) {
                        std::vector<uint2> parts;
                        parts.reserve(items.size());
                        for (int q = 0; q < Q; ++q) {
                            const int64_t b0 = nvb * q / Q, b1 = nvb * (q + 1) / Q;
                            p->fd_part_off[q] = (int64_t)parts.size();
                            p->fd_part_view[q] = std::min<int64_t>(p->n_views, b0 * VBk);
                            for (const uint2& w : items)
                                if ((int64_t)w.x >= b0 && (int64_t)w.x < b1) parts.push_back(w);
                        }
                        p->fd_part_off[Q] = (int64_t)parts.size();
                        p->fd_part_view[Q] = p->n_views;
                        e = cudaMalloc(&p->d_fd_part_items, sizeof(uint2) * parts.size());
                        if (e == cudaSuccess)
                            e = cudaMemcpy(p->d_fd_part_items, parts.data(), sizeof(uint2) * parts.size(),
                                           cudaMemcpyHostToDevice);
                    }
                }
            }
        }
        if (e != cudaSuccess) {
            xrt_plan_destroy(p);
            return cuda_fail(e, "plan workspace");
        }
        // forward bands' image rows (host pipeline: the image arrives in z chunks, band b starts once
        // the rows it reaches are built)
        {
            const int nbf = xrt::column_bands(p, false), rbf = xrt::column_band_rows(p, false);
            p->fwd_band_k.assign(2 * (size_t)nbf, 0);
            for (int b = 0; b < nbf; ++b) {
                double zlo, zhi;
                band_z_range(g, G, (int64_t)b * rbf, std::min<int64_t>(g->det_rows, (int64_t)(b + 1) * rbf) - 1, zlo, zhi);
                p->fwd_band_k[2 * b] = std::max<int64_t>(0, (int64_t)std::floor((G.z_hi - zhi) / G.d[2]) - 2);
                p->fwd_band_k[2 * b + 1] = std::min<int64_t>(G.n[2], (int64_t)std::floor((G.z_hi - zlo) / G.d[2]) + 3);
            }
            if (p->fd_mirror) {
                const int64_t rows = g->det_rows, top = (rows + 1) / 2;
                const int nbm = xrt::fd_mirror_bands(p);
                p->fwdm_band_k.assign(4 * (size_t)nbm, 0);
                for (int b = 0; b < nbm; ++b) {
                    const int64_t mr = xrt::fd_mirror_band_rows();
                    const int64_t r0 = mr * b, r1 = std::min<int64_t>(top, mr * (b + 1));
                    const int64_t ra[2] = {r0, rows - r1}, rz[2] = {r1 - 1, rows - 1 - r0};
                    for (int h = 0; h < 2; ++h) {
                        double zlo, zhi;
                        band_z_range(g, G, ra[h], rz[h], zlo, zhi);
                        p->fwdm_band_k[4 * b + 2 * h] = std::max<int64_t>(0, (int64_t)std::floor((G.z_hi - zhi) / G.d[2]) - 2);
                        p->fwdm_band_k[4 * b + 2 * h + 1] =
                            std::min<int64_t>(G.n[2], (int64_t)std::floor((G.z_hi - zlo) / G.d[2]) + 3);
                    }
                }
            }
        }
        // staged adjoint (xrt_adjoint_stages): band b of the adjoint touches image rows
        // [klo_b, khi_b] (conservative, 2-cell margin); rows no later band touches are final after b.
        // Bands run in row order, i.e. monotone in z; a non-monotone tail folds into the last stage.
        const int nb = xrt::column_bands(p, true), rb = xrt::column_band_rows(p, true);
        std::vector<int64_t> klo(nb), khi(nb);
        for (int b = 0; b < nb; ++b) {
            double zlo, zhi;
            band_z_range(g, G, (int64_t)b * rb, std::min<int64_t>(g->det_rows, (int64_t)(b + 1) * rb) - 1, zlo, zhi);
            klo[b] = std::max<int64_t>(0, (int64_t)std::floor((G.z_hi - zhi) / G.d[2]) - 2);
            khi[b] = std::min<int64_t>(G.n[2] - 1, (int64_t)std::floor((G.z_hi - zlo) / G.d[2]) + 2);
        }
        std::vector<char> done((size_t)G.n[2], 0);
        p->adj_stage_k.assign(2 * (size_t)nb, 0);
        for (int b = 0; b < nb; ++b) {
            std::vector<char> later((size_t)G.n[2], 0);
            for (int b2 = b + 1; b2 < nb; ++b2)
                for (int64_t k = klo[b2]; k <= khi[b2]; ++k) later[(size_t)k] = 1;
            int64_t k0 = -1, k1 = -1;
            bool ok = true;
            for (int64_t k = 0; k < G.n[2]; ++k) {
                if (done[(size_t)k] || later[(size_t)k]) continue;
                if (k0 < 0) k0 = k;
                else if (k != k1) ok = false;       // not one contiguous range: defer
                k1 = k + 1;
            }
            if (!ok || k0 < 0) { p->adj_stage_k[2 * b] = p->adj_stage_k[2 * b + 1] = 0; continue; }
            for (int64_t k = k0; k < k1; ++k) done[(size_t)k] = 1;
            p->adj_stage_k[2 * b] = k0;
            p->adj_stage_k[2 * b + 1] = k1;
        }
        // the last stage finishes everything left (deferred ranges included): check contiguity
        int64_t k0 = -1, k1 = -1;
        bool ok = true;
        for (int64_t k = 0; k < G.n[2]; ++k) {
            if (done[(size_t)k]) continue;
            if (k0 < 0) k0 = k;
            else if (k != k1) ok = false;
            k1 = k + 1;
        }
        if (!ok) {   // fall back to one stage
            p->adj_stage_k.assign(2 * (size_t)nb, 0);
            p->adj_stage_k[2 * (nb - 1)] = 0;
            p->adj_stage_k[2 * (nb - 1) + 1] = G.n[2];
        } else if (k0 >= 0) {
            const int64_t a = p->adj_stage_k[2 * (nb - 1)], bnd = p->adj_stage_k[2 * (nb - 1) + 1];
            p->adj_stage_k[2 * (nb - 1)] = bnd > a ? std::min(a, k0) : k0;
            p->adj_stage_k[2 * (nb - 1) + 1] = bnd > a ? std::max(bnd, k1) : k1;
        }
    }
    *out = p;
    return XRT_OK;
}
}  // namespace

extern "C" {

xrt_status xrt_plan_create(const xrt_geometry* g, int cuda_device, xrt_plan* out) {
    NvtxRange nvtx_("xrt_plan_create");
    if (!out) return fail(XRT_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    xrt_status st = validate(g);
    if (st != XRT_OK) return st;
    return plan_create_impl(g, cuda_device, out, nullptr, 0);
}

xrt_status xrt_plan_create_rays(const xrt_ray_list* r, int cuda_device, xrt_plan* out) {
    NvtxRange nvtx_("xrt_plan_create_rays");
    if (!out) return fail(XRT_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!r) return fail(XRT_ERR_INVALID_ARG, "ray list is NULL");
    if (r->flags != 0) return fail(XRT_ERR_INVALID_ARG, "flags must be 0");
    if (r->dim != 2 && r->dim != 3) return fail(XRT_ERR_INVALID_ARG, "dim must be 2 or 3");
    if (r->n_rays < 1 || r->n_rays > INT_MAX) return fail(XRT_ERR_INVALID_ARG, "n_rays must be in [1, 2^31)");
    if (!r->params) return fail(XRT_ERR_INVALID_ARG, "params is NULL");
    for (int64_t i = 0; i < 4 * r->n_rays; ++i)
        if (!std::isfinite(r->params[i])) return fail(XRT_ERR_INVALID_ARG, "params[%lld] not finite", (long long)i);
    // the grid is validated through an xrt_geometry of the matching parallel beam
    static const double zero_angle = 0.0;
    xrt_geometry g;
    std::memset(&g, 0, sizeof g);
    g.beam = r->dim == 2 ? XRT_PAR2D : XRT_PAR3D;
    for (int a = 0; a < 3; ++a) {
        g.n[a] = r->n[a];
        g.spacing[a] = r->spacing[a];
        g.center[a] = r->center[a];
    }
    g.n_views = 1;
    g.angles = &zero_angle;
    g.det_cols = r->n_rays;
    g.det_rows = 1;
    g.det_spacing[0] = g.det_spacing[1] = 1.0;
    xrt_status st = validate(&g);
    if (st != XRT_OK) return st;
    return plan_create_impl(&g, cuda_device, out, r->params, r->dim);
}

xrt_status xrt_plan_destroy(xrt_plan p) {
    if (!p) return XRT_OK;
    DevGuard guard(p->device);
    cudaFree(p->d_views);
    cudaFree(p->d_work_fwd);
    cudaFree(p->d_work_adj);
    cudaFree(p->d_work_fd);
    cudaFree(p->d_work_att);
    cudaFree(p->d_att_A);
    cudaFree(p->d_att_pieces);
    cudaFree(p->d_att_mumax);
    cudaFree(p->ct[0].d_items);
    cudaFree(p->ct[1].d_items);
    cudaFree(p->ct_fd.d_items);
    cudaFree(p->d_fd_part_items);
    cudaFree(p->d_adj_part_items);
    cudaFree(p->d_coldesc);
    cudaFree(p->d_gather_y);
    cudaFree(p->d_rays);
    cudaFree(p->d_raydesc2d);
    cudaFree(p->d_ray2d_walk);
    cudaFree(p->d_fwd_t);
    cudaFree(p->d_work_fd4);
    cudaFree(p->d_fd2d);
    cudaFree(p->d_img_t);
    cudaFree(p->d_stage_img);
    cudaFree(p->d_stage_sino);
    if (p->aux_stream) cudaStreamDestroy((cudaStream_t)p->aux_stream);
    if (p->aux_stream2) cudaStreamDestroy((cudaStream_t)p->aux_stream2);
    if (p->aux_stream3) cudaStreamDestroy((cudaStream_t)p->aux_stream3);
    delete p;
    return XRT_OK;
}

xrt_status xrt_plan_query(xrt_plan p, int64_t* n_rays, int64_t* n_units) {
    if (!p) return fail(XRT_ERR_INVALID_ARG, "plan is NULL");
    if (n_rays) *n_rays = p->n_rays;
    if (n_units) {
        if (p->n_units < 0) {
            DevGuard guard(p->device);
            xrt_status st = count_units(p, &p->n_units, (cudaStream_t)0);
            if (st != XRT_OK) return st;
        }
        *n_units = p->n_units;
    }
    return XRT_OK;
}

xrt_status xrt_plan_set_algorithm(xrt_plan p, int32_t op, int32_t algo) {
    if (!p) return fail(XRT_ERR_INVALID_ARG, "plan is NULL");
    if (op != XRT_OP_FORWARD && op != XRT_OP_ADJOINT) return fail(XRT_ERR_INVALID_ARG, "bad op %d", op);
    if (algo < XRT_ALGO_AUTO || algo > XRT_ALGO_GATHER) return fail(XRT_ERR_INVALID_ARG, "bad algo %d", algo);
    if (algo == XRT_ALGO_GATHER && op != XRT_OP_ADJOINT)
        return fail(XRT_ERR_UNSUPPORTED, "the gather algorithm is an adjoint");
    if (algo == XRT_ALGO_GATHER && !(p->d_raydesc2d || (p->column_ok && p->det.rows <= 12288)))
        return fail(XRT_ERR_UNSUPPORTED, "gather algorithm does not serve this geometry");
    if (algo == XRT_ALGO_COLUMN && !p->column_ok && !p->d_img_t)
        return fail(XRT_ERR_UNSUPPORTED, "column algorithm does not serve this geometry");
    if (op == XRT_OP_FORWARD) p->algo_fwd = algo; else p->algo_adj = algo;
    return XRT_OK;
}

int64_t xrt_plan_launch_count(xrt_plan p) { return p ? p->launches : -1; }

xrt_status xrt_forward(xrt_plan p, const float* img, float* sino, void* cuda_stream) {
    NvtxRange nvtx_("xrt_forward");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    xrt_status st = fwd_prepare(p, img, s);
    if (st != XRT_OK) return st;
    return forward_range(p, img, sino, 0, p->n_views, s);
}

xrt_status xrt_adjoint(xrt_plan p, const float* sino, float* img, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    xrt_status st = adj_begin(p, img, s);
    if (st == XRT_OK) st = adjoint_range(p, sino, img, 0, p->n_views, s);
    if (st == XRT_OK) st = adj_finish(p, img, s);
    return st;
}

xrt_status xrt_forward_f64(xrt_plan p, const double* img, double* sino, void* cuda_stream) {
    NvtxRange nvtx_("xrt_forward_f64");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaError_t e = xrt::launch_forward64(p, img, sino, 0, p->n_rays, (cudaStream_t)cuda_stream);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "forward_f64 launch");
    return XRT_OK;
}

xrt_status xrt_adjoint_f64(xrt_plan p, const double* sino, double* img, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint_f64");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    XRT_CUDA(cudaMemsetAsync(img, 0, sizeof(double) * (size_t)p->grid.nxyz, s));
    cudaError_t e = xrt::launch_adjoint64(p, sino, img, 0, p->n_rays, s);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "adjoint_f64 launch");
    return XRT_OK;
}

xrt_status xrt_forward_mixed(xrt_plan p, const double* img, double* sino, void* cuda_stream) {
    NvtxRange nvtx_("xrt_forward_mixed");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaError_t e = xrt::launch_forward_mixed(p, img, sino, 0, p->n_rays, (cudaStream_t)cuda_stream);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "forward_mixed launch");
    return XRT_OK;
}

xrt_status xrt_adjoint_mixed(xrt_plan p, const double* sino, double* img, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint_mixed");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    XRT_CUDA(cudaMemsetAsync(img, 0, sizeof(double) * (size_t)p->grid.nxyz, s));
    cudaError_t e = xrt::launch_adjoint_mixed(p, sino, img, 0, p->n_rays, s);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "adjoint_mixed launch");
    return XRT_OK;
}

// Attenuated transform: the column kernels for the 3D beams they serve (tiled per
// band with a per-ray combine of the tile pieces, xrt::att_tiled; untiled otherwise), else the RAY
// family.  Workspace on first use: the forward's interleaved (f, mu) z-fastest volume, the tile
// pieces (both operators, tiled), the per-ray total attenuation (untiled adjoint only).
static cudaError_t att_alloc(xrt_plan p, bool adjoint) {
    cudaError_t e = cudaSuccess;
    const bool tiled = xrt::att_tiled(p);
    if (!p->d_att_mumax) e = cudaMalloc(&p->d_att_mumax, sizeof(unsigned));
    if (e == cudaSuccess && !adjoint && !p->d_work_att) {
        const size_t bytes = 2 * sizeof(float) * (size_t)(p->grid.nxy * p->nzp);
        e = cudaMalloc(&p->d_work_att, bytes);
        if (e == cudaSuccess) e = cudaMemset(p->d_work_att, 0, bytes);   // zero padding stays zero
    }
    if (e == cudaSuccess && tiled && !p->d_att_pieces)
        e = cudaMalloc(&p->d_att_pieces, sizeof(float) * (size_t)xrt::att_piece_floats(p));
    if (e == cudaSuccess && adjoint && !tiled && !p->d_att_A)
        e = cudaMalloc(&p->d_att_A, sizeof(float) * (size_t)(p->n_views * p->det.per_view));
    return e;
}

xrt_status xrt_forward_attenuated(xrt_plan p, const float* img, const float* mu, float* sino, void* cuda_stream) {
    NvtxRange nvtx_("xrt_forward_attenuated");
    if (!p || !img || !mu || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    cudaError_t e;
    if (p->dim == 3 && resolve(p, XRT_OP_FORWARD) == XRT_ALGO_COLUMN) {
        e = att_alloc(p, false);
        if (e == cudaSuccess) e = xrt::launch_att_prepare(p, img, mu, p->d_work_att, p->d_att_mumax, s);
        if (e == cudaSuccess) e = xrt::launch_forward_att_column(p, p->d_work_att, p->d_att_mumax, sino, p->d_att_pieces, s);
        p->launches += 4;
    } else {
        e = xrt::launch_forward_att(p, img, mu, sino, 0, p->n_rays, s);
        p->launches += 1;
    }
    if (e != cudaSuccess) return cuda_fail(e, "forward_attenuated launch");
    return XRT_OK;
}

xrt_status xrt_adjoint_attenuated(xrt_plan p, const float* sino, const float* mu, float* img, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint_attenuated");
    if (!p || !img || !mu || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    cudaError_t e;
    if (p->dim == 3 && resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_COLUMN) {
        // mu z-fastest in work_fwd; tiled plans: per band, the pieces' attenuation A_t (the plain
        // forward of mu per piece), their suffix sums B_t, then the scatter y e^-(B_t - A_le) L phi
        // with A_le from each piece's start; untiled: A = X mu per ray, then the untiled scatter
        const bool tiled = xrt::att_tiled(p);
        e = att_alloc(p, true);
        if (e == cudaSuccess) e = xrt::launch_to_zfast(p, mu, p->d_work_fwd, s);
        if (e == cudaSuccess) e = xrt::launch_att_prepare(p, nullptr, mu, nullptr, p->d_att_mumax, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(p->d_work_adj, 0, sizeof(float) * (size_t)(p->grid.nxy * p->nzp), s);
        if (tiled) {
            if (e == cudaSuccess)
                e = xrt::launch_adjoint_att_tiled(p, p->d_work_fwd, p->d_att_pieces, p->d_att_mumax, sino,
                                                  p->d_work_adj, s);
        } else if (e == cudaSuccess) {
            e = xrt::launch_adjoint_att_column(p, p->d_work_fwd, p->d_att_A, p->d_att_mumax, sino, p->d_work_adj, s);
        }
        if (e == cudaSuccess) e = xrt::launch_from_zfast(p, p->d_work_adj, img, s);
        p->launches += 5;
    } else {
        e = cudaMemsetAsync(img, 0, sizeof(float) * (size_t)p->grid.nxyz, s);
        if (e == cudaSuccess) e = xrt::launch_adjoint_att(p, sino, mu, img, 0, p->n_rays, s);
        p->launches += 1;
    }
    if (e != cudaSuccess) return cuda_fail(e, "adjoint_attenuated launch");
    return XRT_OK;
}

xrt_status xrt_adjoint_stages(xrt_plan p, int32_t* n_stages, int64_t* k_begin, int64_t* k_end) {
    if (!p || !n_stages) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    const bool staged = resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_COLUMN && p->dim == 3 && !p->adj_stage_k.empty();
    const int32_t S = staged ? (int32_t)(p->adj_stage_k.size() / 2) : 1;
    *n_stages = S;
    if (k_begin && k_end) {
        for (int32_t s = 0; s < S; ++s) {
            k_begin[s] = staged ? p->adj_stage_k[2 * s] : 0;
            k_end[s] = staged ? p->adj_stage_k[2 * s + 1] : p->grid.n[2];
        }
    }
    return XRT_OK;
}

xrt_status xrt_adjoint_stage(xrt_plan p, const float* sino, float* img, int32_t stage, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint_stage");
    if (!p || !img || !sino) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const bool staged = resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_COLUMN && p->dim == 3 && !p->adj_stage_k.empty();
    const int32_t S = staged ? (int32_t)(p->adj_stage_k.size() / 2) : 1;
    if (stage < 0 || stage >= S) return fail(XRT_ERR_INVALID_ARG, "stage %d outside [0, %d)", stage, S);
    if (!staged) return xrt_adjoint(p, sino, img, cuda_stream);
    xrt_status st = XRT_OK;
    if (stage == 0) st = adj_begin(p, img, s);
    if (st != XRT_OK) return st;
    cudaError_t e = xrt::launch_adjoint_column_bands(p, sino, p->d_work_adj, stage, stage + 1, s);
    p->launches += 1;
    if (e != cudaSuccess) return cuda_fail(e, "adjoint stage launch");
    const int64_t k0 = p->adj_stage_k[2 * stage], k1 = p->adj_stage_k[2 * stage + 1];
    if (k1 > k0) {
        e = xrt::launch_from_zfast_rows(p, p->d_work_adj, img, k0, k1, s);
        p->launches += 1;
        if (e != cudaSuccess) return cuda_fail(e, "transpose launch");
    }
    return XRT_OK;
}

// Host-buffer forward: H2D(image) -> per view chunk: kernel, then D2H of that chunk on the aux
// stream, so the sinogram download overlaps the next chunk's kernel.
xrt_status xrt_forward_host(xrt_plan p, const float* img_host, float* sino_host, void* cuda_stream) {
    NvtxRange nvtx_("xrt_forward_host");
    if (!p || !img_host || !sino_host) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    xrt_status st = alloc_stage(p);
    if (st != XRT_OK) return st;
    cudaStream_t s = (cudaStream_t)cuda_stream, a = (cudaStream_t)p->aux_stream;
    if (resolve(p, XRT_OP_FORWARD) == XRT_ALGO_COLUMN && p->dim == 3 && p->fd_forward && xrt::fd_mirror_active(p) &&
        !p->fwdm_band_k.empty()) {
        // z-mirror fd forward: mirror band b needs image rows at both ends of z, so the image goes up
        // from both ends towards the middle (two fronts, alternating chunks on the aux stream), each
        // front building its fd rows as soon as their neighbour rows are present; band b waits for
        // the chunk after which both of its row ranges are built; its upper and mirrored sinogram
        // rows go down on a second aux stream while later bands compute
        const int nz = p->grid.n[2];
        const int64_t nxy = p->grid.nxy;
        const int nbm = xrt::fd_mirror_bands(p), rows = p->det.rows, top = (rows + 1) / 2;
        const int CH = std::max(32, (nz + 15) / 16);
        cudaStream_t d = (cudaStream_t)p->aux_stream2;
        cudaStream_t cs[2] = {s, (cudaStream_t)p->aux_stream3};
        struct Step { int lo, hi; bool asc; };
        std::vector<Step> steps;
        for (int alo = 0, dhi = nz; alo < dhi;) {
            const int ahi = std::min(dhi, alo + CH);
            steps.push_back({alo, ahi, true});
            alo = ahi;
            if (alo >= dhi) break;
            const int dlo = std::max(alo, dhi - CH);
            steps.push_back({dlo, dhi, false});
            dhi = dlo;
        }
        const int nst = (int)steps.size();
        std::vector<cudaEvent_t> evc((size_t)nst), evb((size_t)nbm), evp((size_t)xrt_plan_s::kFwdParts);
        for (auto& x : evc) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : evb) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : evp) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        cudaEvent_t ev0, ev_end;
        XRT_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        XRT_CUDA(cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming));
        XRT_CUDA(cudaEventRecord(ev0, s));
        XRT_CUDA(cudaStreamWaitEvent(a, ev0, 0));
        XRT_CUDA(cudaStreamWaitEvent(cs[1], ev0, 0));
        cudaError_t e = cudaSuccess;
        // interleaved layout (device-path layout, also here when on): fd4 row k needs image rows k, k + 1
        // and their mirrors N_z - 1 - k, N_z - 2 - k; two halves: fd row k needs k - 1, k, k + 1.
        // After every upload step, the rows (k = -1 .. N_z) whose image rows are all present are built
        // (runs of consecutive rows per launch); built_at[k] = the step after which row k exists.
        const bool f4 = xrt::fd_f4_on(p);
        if (f4 && !p->d_work_fd4) {
            const size_t b4 = sizeof(float4) * (size_t)(nxy * p->nzp);
            XRT_CUDA(cudaMalloc(&p->d_work_fd4, b4));
            XRT_CUDA(cudaMemsetAsync(p->d_work_fd4, 0, b4, a));
        }
        std::vector<char> up((size_t)nz, 0);
        std::vector<int> built_at((size_t)nz + 2, -1);   // index k + 1
        auto present = [&](int k) { return k < 0 || k >= nz || up[(size_t)k]; };
        for (int i = 0; i < nst && e == cudaSuccess; ++i) {
            const Step& S = steps[i];
            e = cudaMemcpyAsync(p->d_stage_img + S.lo * nxy, img_host + S.lo * nxy,
                                sizeof(float) * (size_t)((S.hi - S.lo) * nxy), cudaMemcpyHostToDevice, a);
            for (int k = S.lo; k < S.hi; ++k) up[(size_t)k] = 1;
            int run0 = -2;
            for (int k = -1; k <= nz + 1 && e == cudaSuccess; ++k) {
                bool ready = false;
                if (k <= nz && built_at[(size_t)k + 1] < 0)
                    ready = f4 ? (present(k) && present(k + 1) && present(nz - 1 - k) && present(nz - 2 - k))
                               : (present(k - 1) && present(k) && present(k + 1));
                if (ready) {
                    built_at[(size_t)k + 1] = i;
                    if (run0 == -2) run0 = k;
                } else if (run0 != -2) {
                    e = f4 ? xrt::launch_to_fd4_rows(p, p->d_stage_img, p->d_work_fd4, run0, k, a)
                           : xrt::launch_to_fd_rows(p, p->d_stage_img, p->d_work_fd, run0, k, a);
                    p->launches += 1;
                    run0 = -2;
                }
            }
            if (e == cudaSuccess) e = cudaEventRecord(evc[i], a);
        }
        const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
        for (int b = 0; b < nbm && e == cudaSuccess; ++b) {
            // the step after which every row the band reads is built (f4: the walked rows' range only,
            // their mirrors sit in the same fd4 rows)
            int need = 0;
            for (int h = 0; h < (f4 ? 1 : 2); ++h) {
                const int x0 = std::max(-1, (int)p->fwdm_band_k[4 * b + 2 * h] - 1);
                const int x1 = std::min(nz + 1, (int)p->fwdm_band_k[4 * b + 2 * h + 1] + 1);
                for (int k = x0; k < x1; ++k) need = std::max(need, built_at[(size_t)k + 1]);
            }
            if (need < 0) need = nst - 1;
            const int mr = xrt::fd_mirror_band_rows();
            const int r0 = mr * b, r1 = std::min(top, mr * (b + 1));
            const int q0[2] = {r0, rows - r1};
            if (b == nbm - 1 && p->d_fd_part_items) {
                // the last band part by part (view ranges): each part's rows go down while the next
                // part computes, so only the last part's copy is exposed
                for (int q = 0; q < xrt_plan_s::kFwdParts && e == cudaSuccess; ++q) {
                    const int64_t v0 = p->fd_part_view[q], v1 = p->fd_part_view[q + 1];
                    cudaStream_t c = cs[(b + q) & 1];
                    e = cudaStreamWaitEvent(c, evc[need], 0);
                    if (e == cudaSuccess)
                        e = xrt::launch_forward_fd_mirror_band_part(p, p->d_work_fd, p->d_stage_sino, b, q, c);
                    p->launches += 1;
                    if (e == cudaSuccess) e = cudaEventRecord(evp[q], c);
                    if (e == cudaSuccess) e = cudaStreamWaitEvent(d, evp[q], 0);
                    for (int h = 0; h < 2 && e == cudaSuccess && v1 > v0; ++h)
                        e = cudaMemcpy2DAsync(sino_host + v0 * p->det.per_view + (int64_t)q0[h] * p->det.cols, pitch,
                                              p->d_stage_sino + v0 * p->det.per_view + (int64_t)q0[h] * p->det.cols,
                                              pitch, sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0),
                                              cudaMemcpyDeviceToHost, d);
                }
                continue;
            }
            cudaStream_t c = cs[b & 1];
            e = cudaStreamWaitEvent(c, evc[need], 0);
            if (e == cudaSuccess) e = xrt::launch_forward_fd_mirror_bands(p, p->d_work_fd, p->d_stage_sino, b, b + 1, c);
            p->launches += 1;
            if (e == cudaSuccess) e = cudaEventRecord(evb[b], c);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(d, evb[b], 0);
            for (int h = 0; h < 2 && e == cudaSuccess; ++h)
                e = cudaMemcpy2DAsync(sino_host + (int64_t)q0[h] * p->det.cols, pitch,
                                      p->d_stage_sino + (int64_t)q0[h] * p->det.cols, pitch,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views,
                                      cudaMemcpyDeviceToHost, d);
        }
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, evc[nst - 1], 0);   // the stage buffers are reused
        if (e == cudaSuccess) e = cudaEventRecord(ev_end, cs[1]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_end, 0);
        cudaError_t e1 = cudaStreamSynchronize(a);
        cudaError_t e2 = cudaStreamSynchronize(s);
        cudaError_t e3 = cudaStreamSynchronize(d);
        cudaError_t e4 = cudaStreamSynchronize(cs[1]);
        if (e3 == cudaSuccess) e3 = e4;
        for (auto& x : evc) cudaEventDestroy(x);
        for (auto& x : evb) cudaEventDestroy(x);
        for (auto& x : evp) cudaEventDestroy(x);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev_end);
        if (e != cudaSuccess) return cuda_fail(e, "forward_host mirrored pipeline");
        if (e1 != cudaSuccess) return cuda_fail(e1, "forward_host sync");
        if (e2 != cudaSuccess) return cuda_fail(e2, "forward_host sync");
        if (e3 != cudaSuccess) return cuda_fail(e3, "forward_host sync");
        return XRT_OK;
    }
    if (resolve(p, XRT_OP_FORWARD) == XRT_ALGO_COLUMN && p->dim == 3 && p->fd_forward && !p->fwd_band_k.empty()) {
        // fd column forward: the image goes up in z chunks on the aux stream, each chunk's fd rows
        // built there as soon as its neighbour rows are present; band b waits only for the rows
        // it reaches (bands run in row order, i.e. monotone in z: the chunks are sent in the order
        // the bands need them); band b's sinogram rows go down on a second aux stream
        const int nz = p->grid.n[2];
        const int64_t nxy = p->grid.nxy;
        const int nb = xrt::column_bands(p, false), rb = xrt::column_band_rows(p, false);
        const bool desc = p->fwd_band_k[0] + p->fwd_band_k[1] >= nz;    // band 0 at high k
        const int CH = std::max(32, (nz + 15) / 16);
        const int nch = (nz + CH - 1) / CH;
        cudaStream_t d = (cudaStream_t)p->aux_stream2;
        // bands alternate between two compute streams (disjoint sinogram rows), so one band's
        // last CTAs overlap the next band's first ones; both start after the caller's prior work
        // on s, as does the upload stream
        cudaStream_t cs[2] = {s, (cudaStream_t)p->aux_stream3};
        std::vector<cudaEvent_t> evc((size_t)nch), evb((size_t)nb), evp((size_t)xrt_plan_s::kFwdParts);
        for (auto& x : evc) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : evb) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : evp) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        cudaEvent_t ev0, ev_end;
        XRT_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        XRT_CUDA(cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming));
        XRT_CUDA(cudaEventRecord(ev0, s));
        XRT_CUDA(cudaStreamWaitEvent(a, ev0, 0));
        XRT_CUDA(cudaStreamWaitEvent(cs[1], ev0, 0));
        // XRT_HOST_TRACE=1: per-phase device times on stderr (diagnostic)
        const bool trace = std::getenv("XRT_HOST_TRACE") != nullptr;
        std::vector<cudaEvent_t> tev;
        auto tmark = [&](cudaStream_t st) {
            if (!trace) return;
            cudaEvent_t x;
            cudaEventCreate(&x);
            cudaEventRecord(x, st);
            tev.push_back(x);
        };
        tmark(s);
        // chunk i covers image rows [lo_i, hi_i) in send order; built fd rows after chunk i:
        // desc: [lo_i + 1 .. nz] (row lo_i waits for its lower neighbour), asc: [-1 .. hi_i - 1)
        cudaError_t e = cudaSuccess;
        int built_lo = nz + 1, built_hi = -1;   // fd rows [built_lo, nz] (desc) or [-1, built_hi) (asc)
        std::vector<int> done_lo((size_t)nch), done_hi((size_t)nch);
        for (int i = 0; i < nch && e == cudaSuccess; ++i) {
            const int lo = desc ? std::max(0, nz - (i + 1) * CH) : i * CH;
            const int hi = desc ? nz - i * CH : std::min(nz, (i + 1) * CH);
            e = cudaMemcpyAsync(p->d_stage_img + lo * nxy, img_host + lo * nxy, sizeof(float) * (size_t)((hi - lo) * nxy),
                                cudaMemcpyHostToDevice, a);
            if (desc) {
                const int ka = lo == 0 ? -1 : lo + 1, kb = built_lo;
                if (e == cudaSuccess) e = xrt::launch_to_fd_rows(p, p->d_stage_img, p->d_work_fd, ka, kb, a);
                built_lo = ka;
            } else {
                const int ka = built_hi < 0 ? -1 : built_hi, kb = hi == nz ? nz + 1 : hi - 1;
                if (e == cudaSuccess) e = xrt::launch_to_fd_rows(p, p->d_stage_img, p->d_work_fd, ka, kb, a);
                built_hi = kb;
            }
            p->launches += 1;
            done_lo[i] = desc ? built_lo : -1;
            done_hi[i] = desc ? nz + 1 : built_hi;
            if (e == cudaSuccess) e = cudaEventRecord(evc[i], a);
        }
        const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
        for (int b = 0; b < nb && e == cudaSuccess; ++b) {
            // the first chunk after which the band's rows (with their fd neighbours) are built
            const int k0 = (int)p->fwd_band_k[2 * b] - 1, k1 = (int)p->fwd_band_k[2 * b + 1] + 1;
            int need = nch - 1;
            for (int i = 0; i < nch; ++i)
                if (done_lo[i] <= std::max(k0, -1) && done_hi[i] >= std::min(k1, nz + 1)) { need = i; break; }
            const int r0 = b * rb, r1 = std::min(p->det.rows, r0 + rb);
            if (b == nb - 1 && p->d_fd_part_items) {
                // the last band part by part (view ranges): each part's rows go down while the next
                // part computes, so only the last part's copy is exposed
                for (int q = 0; q < xrt_plan_s::kFwdParts && e == cudaSuccess; ++q) {
                    const int64_t v0 = p->fd_part_view[q], v1 = p->fd_part_view[q + 1];
                    cudaStream_t c = cs[(b + q) & 1];
                    e = cudaStreamWaitEvent(c, evc[need], 0);
                    if (e == cudaSuccess) e = xrt::launch_forward_fd_band_part(p, p->d_work_fd, p->d_stage_sino, b, q, c);
                    p->launches += 1;
                    if (e == cudaSuccess) e = cudaEventRecord(evp[q], c);
                    if (e == cudaSuccess) e = cudaStreamWaitEvent(d, evp[q], 0);
                    if (e == cudaSuccess && v1 > v0)
                        e = cudaMemcpy2DAsync(sino_host + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch,
                                              p->d_stage_sino + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch,
                                              sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0),
                                              cudaMemcpyDeviceToHost, d);
                }
                continue;
            }
            cudaStream_t c = cs[b & 1];
            e = cudaStreamWaitEvent(c, evc[need], 0);
            tmark(c);
            if (e == cudaSuccess) e = xrt::launch_forward_fd_bands(p, p->d_work_fd, p->d_stage_sino, b, b + 1, c);
            tmark(c);
            p->launches += 1;
            if (e == cudaSuccess) e = cudaEventRecord(evb[b], c);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(d, evb[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(sino_host + (int64_t)r0 * p->det.cols, pitch,
                                      p->d_stage_sino + (int64_t)r0 * p->det.cols, pitch,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views,
                                      cudaMemcpyDeviceToHost, d);
        }
        tmark(a);
        tmark(d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, evc[nch - 1], 0);   // the stage buffers are reused
        if (e == cudaSuccess) e = cudaEventRecord(ev_end, cs[1]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_end, 0);
        cudaError_t e1 = cudaStreamSynchronize(a);
        cudaError_t e2 = cudaStreamSynchronize(s);
        cudaError_t e3 = cudaStreamSynchronize(d);
        cudaError_t e4 = cudaStreamSynchronize(cs[1]);
        if (e3 == cudaSuccess) e3 = e4;
        for (auto& x : evc) cudaEventDestroy(x);
        for (auto& x : evb) cudaEventDestroy(x);
        for (auto& x : evp) cudaEventDestroy(x);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev_end);
        if (trace && !tev.empty()) {
            std::fprintf(stderr, "xrt forward_host trace (ms from start):");
            for (size_t i = 1; i < tev.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, tev[0], tev[i]);
                std::fprintf(stderr, " %.2f", ms);
            }
            std::fprintf(stderr, "\n");
        }
        for (auto& x : tev) cudaEventDestroy(x);
        if (e != cudaSuccess) return cuda_fail(e, "forward_host chunked pipeline");
        if (e1 != cudaSuccess) return cuda_fail(e1, "forward_host sync");
        if (e2 != cudaSuccess) return cuda_fail(e2, "forward_host sync");
        if (e3 != cudaSuccess) return cuda_fail(e3, "forward_host sync");
        return XRT_OK;
    }
    XRT_CUDA(cudaMemcpyAsync(p->d_stage_img, img_host, sizeof(float) * (size_t)p->grid.nxyz,
                             cudaMemcpyHostToDevice, s));
    st = fwd_prepare(p, p->d_stage_img, s);
    if (st != XRT_OK) return st;
    if (resolve(p, XRT_OP_FORWARD) == XRT_ALGO_COLUMN && p->dim == 3) {
        // COLUMN: one launch per band of detector rows; the band's sinogram rows (every view) go
        // back on the aux stream while the next band computes
        const int nb = xrt::column_bands(p, false), rb = xrt::column_band_rows(p, false);
        const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
        std::vector<cudaEvent_t> ev((size_t)nb);
        for (auto& x : ev) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (int b = 0; b < nb && st == XRT_OK; ++b) {
            const int r0 = b * rb, r1 = std::min(p->det.rows, r0 + rb);
            cudaError_t e = p->fd_forward ? xrt::launch_forward_fd_bands(p, p->d_work_fd, p->d_stage_sino, b, b + 1, s)
                                          : xrt::launch_forward_column_bands(p, p->d_work_fwd, p->d_stage_sino, b, b + 1, s);
            p->launches += 1;
            if (e == cudaSuccess) e = cudaEventRecord(ev[b], s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(a, ev[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpy2DAsync(sino_host + (int64_t)r0 * p->det.cols, pitch,
                                      p->d_stage_sino + (int64_t)r0 * p->det.cols, pitch,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)p->n_views,
                                      cudaMemcpyDeviceToHost, a);
            if (e != cudaSuccess) st = cuda_fail(e, "forward_host band pipeline");
        }
        cudaError_t e1 = cudaStreamSynchronize(a);
        cudaError_t e2 = cudaStreamSynchronize(s);
        for (auto& x : ev) cudaEventDestroy(x);
        if (st != XRT_OK) return st;
        if (e1 != cudaSuccess) return cuda_fail(e1, "forward_host sync");
        if (e2 != cudaSuccess) return cuda_fail(e2, "forward_host sync");
        return XRT_OK;
    }
    const bool whole = resolve(p, XRT_OP_FORWARD) == XRT_ALGO_COLUMN;   // 2D slice kernels
    const int64_t nchunk = whole ? 1 : std::min<int64_t>(8, p->n_views);
    const int64_t pv = p->det.per_view;
    std::vector<cudaEvent_t> ev((size_t)nchunk);
    for (auto& x : ev) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (int64_t k = 0; k < nchunk && st == XRT_OK; ++k) {
        const int64_t v0 = p->n_views * k / nchunk, v1 = p->n_views * (k + 1) / nchunk;
        st = forward_range(p, p->d_stage_img, p->d_stage_sino, v0, v1, s);
        if (st != XRT_OK) break;
        cudaError_t e = cudaEventRecord(ev[k], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(a, ev[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(sino_host + v0 * pv, p->d_stage_sino + v0 * pv,
                                sizeof(float) * (size_t)((v1 - v0) * pv), cudaMemcpyDeviceToHost, a);
        if (e != cudaSuccess) st = cuda_fail(e, "forward_host pipeline");
    }
    cudaError_t e1 = cudaStreamSynchronize(a);
    cudaError_t e2 = cudaStreamSynchronize(s);
    for (auto& x : ev) cudaEventDestroy(x);
    if (st != XRT_OK) return st;
    if (e1 != cudaSuccess) return cuda_fail(e1, "forward_host sync");
    if (e2 != cudaSuccess) return cuda_fail(e2, "forward_host sync");
    return XRT_OK;
}

// Host-buffer adjoint: per view chunk H2D(sino chunk) on the aux stream overlapping the previous
// chunk's kernel, then D2H(image).
xrt_status xrt_adjoint_host(xrt_plan p, const float* sino_host, float* img_host, void* cuda_stream) {
    NvtxRange nvtx_("xrt_adjoint_host");
    if (!p || !img_host || !sino_host) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    DevGuard guard(p->device);
    xrt_status st = alloc_stage(p);
    if (st != XRT_OK) return st;
    cudaStream_t s = (cudaStream_t)cuda_stream, a = (cudaStream_t)p->aux_stream;
    st = adj_begin(p, p->d_stage_img, s);
    if (st != XRT_OK) return st;
    if (resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_COLUMN && p->dim == 3 && !p->adj_stage_k.empty()) {
        // COLUMN, staged: the sinogram rows of band b (every view) are uploaded on the aux stream
        // while band b - 1 computes; after band b the image rows no later band reaches are
        // transposed out and downloaded on a second aux stream while the next bands compute, so
        // only the last stage's rows wait for the end (xrt_adjoint_stages)
        const int nb = xrt::column_bands(p, true), rb = xrt::column_band_rows(p, true);
        const size_t pitch = sizeof(float) * (size_t)p->det.per_view;
        cudaStream_t d = (cudaStream_t)p->aux_stream2;
        std::vector<cudaEvent_t> ev((size_t)nb), evd((size_t)nb);
        for (auto& x : ev) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (auto& x : evd) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        const int64_t nxy = p->grid.nxy;
        std::vector<cudaEvent_t> evp((size_t)xrt_plan_s::kFwdParts);
        for (auto& x : evp) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
        for (int b = 0; b < nb && st == XRT_OK; ++b) {
            const int r0 = b * rb, r1 = std::min(p->det.rows, r0 + rb);
            cudaError_t e = cudaSuccess;
            if (b == 0 && p->d_adj_part_items) {
                // the first band part by part (view ranges): each part computes as soon as its rows
                // are up, so only the first part's upload is exposed
                for (int q = 0; q < xrt_plan_s::kFwdParts && e == cudaSuccess; ++q) {
                    const int64_t v0 = p->adj_part_view[q], v1 = p->adj_part_view[q + 1];
                    if (v1 > v0)
                        e = cudaMemcpy2DAsync(p->d_stage_sino + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch,
                                              sino_host + v0 * p->det.per_view + (int64_t)r0 * p->det.cols, pitch,
                                              sizeof(float) * (size_t)(r1 - r0) * p->det.cols, (size_t)(v1 - v0),
                                              cudaMemcpyHostToDevice, a);
                    if (e == cudaSuccess) e = cudaEventRecord(evp[q], a);
                    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, evp[q], 0);
                    if (e == cudaSuccess) e = xrt::launch_adjoint_column_band_part(p, p->d_stage_sino, p->d_work_adj, b, q, s);
                    p->launches += 1;
                }
            } else {
                e = cudaMemcpy2DAsync(p->d_stage_sino + (int64_t)r0 * p->det.cols, pitch,
                                      sino_host + (int64_t)r0 * p->det.cols, pitch,
                                      sizeof(float) * (size_t)(r1 - r0) * p->det.cols,
                                      (size_t)p->n_views, cudaMemcpyHostToDevice, a);
                if (e == cudaSuccess) e = cudaEventRecord(ev[b], a);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[b], 0);
                if (e == cudaSuccess) e = xrt::launch_adjoint_column_bands(p, p->d_stage_sino, p->d_work_adj, b, b + 1, s);
                p->launches += 1;
            }
            const int64_t k0 = p->adj_stage_k[2 * b], k1 = p->adj_stage_k[2 * b + 1];
            if (e == cudaSuccess && k1 > k0) {
                e = xrt::launch_from_zfast_rows(p, p->d_work_adj, p->d_stage_img, k0, k1, s);
                p->launches += 1;
                if (e == cudaSuccess) e = cudaEventRecord(evd[b], s);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(d, evd[b], 0);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(img_host + k0 * nxy, p->d_stage_img + k0 * nxy, sizeof(float) * (size_t)((k1 - k0) * nxy),
                                        cudaMemcpyDeviceToHost, d);
            }
            if (e != cudaSuccess) st = cuda_fail(e, "adjoint_host staged pipeline");
        }
        cudaError_t e1 = cudaStreamSynchronize(s);
        cudaError_t e2 = cudaStreamSynchronize(a);
        cudaError_t e3 = cudaStreamSynchronize(d);
        for (auto& x : ev) cudaEventDestroy(x);
        for (auto& x : evd) cudaEventDestroy(x);
        for (auto& x : evp) cudaEventDestroy(x);
        if (st != XRT_OK) return st;
        if (e1 != cudaSuccess) return cuda_fail(e1, "adjoint_host sync");
        if (e2 != cudaSuccess) return cuda_fail(e2, "adjoint_host sync");
        if (e3 != cudaSuccess) return cuda_fail(e3, "adjoint_host sync");
        return XRT_OK;
    }
    const bool whole = resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_GATHER ||
                       resolve(p, XRT_OP_ADJOINT) == XRT_ALGO_COLUMN;   // 2D slice kernels
    const int64_t nchunk = whole ? 1 : std::min<int64_t>(8, p->n_views);
    const int64_t pv = p->det.per_view;
    std::vector<cudaEvent_t> ev((size_t)nchunk);
    for (auto& x : ev) XRT_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    // all uploads on the aux stream, each kernel waits for its chunk
    for (int64_t k = 0; k < nchunk && st == XRT_OK; ++k) {
        const int64_t v0 = p->n_views * k / nchunk, v1 = p->n_views * (k + 1) / nchunk;
        cudaError_t e = cudaMemcpyAsync(p->d_stage_sino + v0 * pv, sino_host + v0 * pv,
                                        sizeof(float) * (size_t)((v1 - v0) * pv), cudaMemcpyHostToDevice, a);
        if (e == cudaSuccess) e = cudaEventRecord(ev[k], a);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[k], 0);
        if (e != cudaSuccess) { st = cuda_fail(e, "adjoint_host pipeline"); break; }
        st = adjoint_range(p, p->d_stage_sino, p->d_stage_img, v0, v1, s);
    }
    if (st == XRT_OK) st = adj_finish(p, p->d_stage_img, s);
    if (st == XRT_OK) {
        cudaError_t e = cudaMemcpyAsync(img_host, p->d_stage_img, sizeof(float) * (size_t)p->grid.nxyz,
                                        cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = cuda_fail(e, "adjoint_host D2H");
    }
    cudaError_t e1 = cudaStreamSynchronize(s);
    cudaError_t e2 = cudaStreamSynchronize(a);
    for (auto& x : ev) cudaEventDestroy(x);
    if (st != XRT_OK) return st;
    if (e1 != cudaSuccess) return cuda_fail(e1, "adjoint_host sync");
    if (e2 != cudaSuccess) return cuda_fail(e2, "adjoint_host sync");
    return XRT_OK;
}

xrt_status xrt_ray_units(xrt_plan p, int64_t ray_begin, int64_t ray_end, int64_t* row_ptr,
                         int64_t* cols, double* lens, int64_t capacity, int64_t* nnz_out,
                         void* cuda_stream) {
    NvtxRange nvtx_("xrt_ray_units");
    if (!p || !row_ptr || !nnz_out) return fail(XRT_ERR_INVALID_ARG, "NULL argument");
    if (ray_begin < 0 || ray_end < ray_begin || ray_end > p->n_rays)
        return fail(XRT_ERR_INVALID_ARG, "ray range [%lld, %lld) outside [0, %lld)", (long long)ray_begin,
                    (long long)ray_end, (long long)p->n_rays);
    if ((cols == nullptr) != (lens == nullptr)) return fail(XRT_ERR_INVALID_ARG, "cols and lens must both be set or both NULL");
    DevGuard guard(p->device);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int64_t n = ray_end - ray_begin;
    if (n > INT_MAX) return fail(XRT_ERR_UNSUPPORTED, "more than 2^31-1 rays in one call");
    XRT_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s));
    if (n == 0) {
        *nnz_out = 0;
        return XRT_OK;
    }
    int64_t* d_counts = nullptr;
    void* d_tmp = nullptr;
    size_t tmp_bytes = 0;
    xrt_status st = XRT_OK;
    cudaError_t e = cudaMallocAsync(&d_counts, sizeof(int64_t) * (size_t)n, s);
    if (e == cudaSuccess) { e = xrt::launch_units_count(p, ray_begin, ray_end, d_counts, s); p->launches += 1; }
    if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, d_counts, row_ptr + 1, (int)n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_tmp, tmp_bytes, s);
    if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(d_tmp, tmp_bytes, d_counts, row_ptr + 1, (int)n, s);
    int64_t nnz = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nnz, row_ptr + n, sizeof nnz, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (d_tmp) cudaFreeAsync(d_tmp, s);
    if (d_counts) cudaFreeAsync(d_counts, s);
    d_tmp = nullptr;
    if (e != cudaSuccess) return cuda_fail(e, "ray_units count");
    *nnz_out = nnz;
    if (!cols) return XRT_OK;
    if (capacity < nnz) return fail(XRT_ERR_CAPACITY, "capacity %lld < nnz %lld", (long long)capacity, (long long)nnz);
    if (nnz > INT_MAX) return fail(XRT_ERR_UNSUPPORTED, "nnz > 2^31-1 in one call; split the ray range");
    if (nnz == 0) return XRT_OK;
    // fill in traversal order into scratch, then sort each row by flat index into the caller's arrays
    int64_t* k_in = nullptr;
    double* v_in = nullptr;
    e = cudaMallocAsync(&k_in, sizeof(int64_t) * (size_t)nnz, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&v_in, sizeof(double) * (size_t)nnz, s);
    if (e == cudaSuccess) { e = xrt::launch_units_fill(p, ray_begin, ray_end, row_ptr, k_in, v_in, s); p->launches += 1; }
    tmp_bytes = 0;
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::SortPairs(nullptr, tmp_bytes, k_in, cols, v_in, lens, (int)nnz, (int)n,
                                                row_ptr, row_ptr + 1, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_tmp, tmp_bytes, s);
    if (e == cudaSuccess)
        e = cub::DeviceSegmentedSort::SortPairs(d_tmp, tmp_bytes, k_in, cols, v_in, lens, (int)nnz, (int)n,
                                                row_ptr, row_ptr + 1, s);
    if (d_tmp) cudaFreeAsync(d_tmp, s);
    if (k_in) cudaFreeAsync(k_in, s);
    if (v_in) cudaFreeAsync(v_in, s);
    if (e != cudaSuccess) st = cuda_fail(e, "ray_units fill");
    return st;
}

}  // extern "C"
