/*
 * xrt.h -- C ABI of the B200-native discrete X-ray transform (arXiv 2006.00686,
 * Chen, Wang, Bajaj, Oektem, "A Fast and Adaptive Algorithm to Compute the X-ray
 * Transform").  Citations: P:n = line n of the paper's LaTeX source.
 *
 * What the library computes
 *   forward  (xrt_forward):  sino[m] = sum_I img[I] * l_I(ray m)          Eq. (1.4)
 *   adjoint  (xrt_adjoint):  img[I]  = sum_m sino[m] * l_I(ray m)          P:59 ("transpose of
 *                                                                          the projection matrix")
 *   rows     (xrt_ray_units): {(I, l_I(ray m)) : l_I > tau}, one CSR row per ray
 * where l_I(ray) is the length of the ray inside unit I (eq:intersection_length P:153-156,
 * eq:intersection_length_3D P:429-432), enumerated by the paper's sufficient-and-necessary
 * condition for non-vanishing intersectability (eq:restriction_j P:197-212,
 * eq:restriction_j_3D / eq:restriction_k_3D_1 P:479-499) and evaluated by its analytic formula
 * l = C_up - C_low (eq:range_length P:217-220, eq:range_length_3D P:503-506).  Ties (a ray on a
 * grid line / plane) go to the unit with the bigger 1D index: units are half-open
 * in index space (reading 2).
 *
 * Conventions (DESIGN.md section 3 lists every reading of the paper):
 *   image   fp32, C-contiguous [N_z][N_y][N_x]; flat index I = (k*N_y + j)*N_x + i (P:106, P:318,
 *           reading 1); i runs along +x, j along -y, k along -z.
 *           The image box is [center - N*spacing/2, center + N*spacing/2] per axis.
 *   sino    fp32, C-contiguous [n_views][det_rows][det_cols]; ray id m = (v*rows + r)*cols + c.
 *   detector bin positions u_c = (c - (det_cols-1)/2)*du + off_u, v_r = (r - (det_rows-1)/2)*dv
 *           + off_v (reading 9).  Lengths are physical (spacing units).
 *   beams   (readings 7-11):
 *     XRT_PAR2D   ray (s, phi) = (u_c, angle_v): theta = (cos phi, sin phi), point s*theta_perp.
 *     XRT_FAN2D   source S = sod*(-sin a, cos a); flat detector at sdd, +u = (cos a, sin a).
 *     XRT_PAR3D   (s1, s2, phi1, phi2) = (u_c, v_r, angle_v, tilt) with the Euler frame
 *                 theta, theta_1, theta_2 of P:404-412.
 *     XRT_CONE    source S = (-sod cos p, -sod sin p, 0); flat detector at sdd,
 *                 +u = (-sin p, cos p, 0), +v = +z.
 *     XRT_HELICAL as XRT_CONE with source height H(p) = z0 + pitch*p/(2 pi) (detector moves
 *                 with the source; angles are unwrapped and may exceed 2 pi).
 *   detector  flat by default (equispaced columns, P:268-272 / P:627-642).  flags & XRT_DET_CURVED
 *             (fan / cone / helical only): a cylinder of radius sdd about the source, columns
 *             equiangular with fan angle alpha_c = u_c / sdd, rows flat with tan(beta) = v_r / sdd;
 *             rays by the paper's equiangular transforms.
 *
 * Ownership: every image / sinogram / CSR buffer is caller-allocated device memory (e.g. a torch
 * tensor's data_ptr()) unless the function name ends in _host.  The plan owns only its geometry
 * tables and internal workspace (allocated at create time; the _host and _attenuated entry
 * points additionally allocate staging / attenuation buffers on first use).  Nothing returned to
 * the caller is library-allocated.
 *
 * Asynchrony: functions taking a cuda_stream enqueue on that stream (NULL = legacy default stream)
 * and return; kernel faults surface as XRT_ERR_CUDA from a later call.  Functions that return a
 * host-side count (xrt_ray_units' nnz_out, xrt_plan_query's n_units) synchronise the stream.
 * Concurrency: calls on one plan share its workspace, so they must be ordered (one stream, or
 * streams the caller serialises); independent plans may run concurrently on different streams.
 *
 * Errors: every function returns an xrt_status; on a non-OK status xrt_last_error() returns a
 * thread-local human-readable message.  Invalid arguments never launch work.
 */
#ifndef XRT_H
#define XRT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XRT_VERSION_MAJOR 0
#define XRT_VERSION_MINOR 1

typedef struct xrt_plan_s* xrt_plan; /* opaque */

typedef enum {
    XRT_OK = 0,
    XRT_ERR_INVALID_ARG = 1, /* bad geometry or argument; nothing was launched            */
    XRT_ERR_UNSUPPORTED = 2, /* valid request outside what this build implements            */
    XRT_ERR_CUDA = 3,        /* a CUDA runtime call or an earlier asynchronous launch failed */
    XRT_ERR_OOM = 4,         /* device allocation failed                                     */
    XRT_ERR_CAPACITY = 5     /* xrt_ray_units: caller capacity < nnz (nnz_out still set)     */
} xrt_status;

#define XRT_DET_CURVED 1 /* xrt_geometry.flags: cylindrical (equiangular-column) detector */

typedef enum {
    XRT_PAR2D = 0,
    XRT_FAN2D = 1,
    XRT_PAR3D = 2,
    XRT_CONE = 3,
    XRT_HELICAL = 4,
    XRT_RAYS = 5   /* plan built by xrt_plan_create_rays (not valid in xrt_geometry.beam)         */
} xrt_beam;

/* Acquisition geometry.  All lengths in the same physical unit (e.g. mm), angles in radians. */
typedef struct {
    int32_t beam;            /* xrt_beam                                                         */
    int32_t flags;           /* XRT_DET_CURVED or 0; other bits must be 0                        */
    int64_t n[3];            /* N_x, N_y, N_z >= 1 (N_z = 1 for 2D beams)                         */
    double spacing[3];       /* d_x, d_y, d_z > 0 (anisotropic allowed; d_z ignored for 2D)       */
    double center[3];        /* physical centre of the image box (z ignored for 2D)              */
    int64_t n_views;         /* >= 1                                                              */
    const double* angles;    /* HOST array [n_views]: phi (par2d), alpha (fan), phi1 (par3d),
                                phi1' (cone / helical); copied at create time                    */
    int64_t det_cols;        /* >= 1                                                              */
    int64_t det_rows;        /* >= 1 (must be 1 for 2D beams)                                     */
    double det_spacing[2];   /* du, dv > 0, measured on the detector                              */
    double det_offset[2];    /* detector-centre shift along +u, +v                                */
    double sod;              /* source-to-origin distance (fan / cone / helical; > 0)             */
    double sdd;              /* source-to-detector distance (> sod)                               */
    double pitch;            /* helical: source z advance per 2 pi of angle; else ignored         */
    double z0;               /* helical: source z at angle 0; else ignored                        */
    double tilt;             /* par3d: Euler angle phi2 of every view, |tilt| < pi/2      */
} xrt_geometry;

/* Algorithm selectors for xrt_plan_set_algorithm (testing / benchmarking).  AUTO picks by
 * geometry; every algorithm computes the same operator. */
typedef enum { XRT_OP_FORWARD = 0, XRT_OP_ADJOINT = 1 } xrt_op;
typedef enum {
    XRT_ALGO_AUTO = 0,
    XRT_ALGO_RAY = 1,    /* one thread per ray, per-ray unit enumeration (any geometry)          */
    XRT_ALGO_COLUMN = 2, /* one warp per detector column: shared in-plane unit band, per-lane
                            z band (3D beams whose rays have a common xy line per column)        */
    XRT_ALGO_GATHER = 3  /* adjoint only: voxel-driven gather (a warp per cell column, no atomics);
                            same geometries as XRT_ALGO_COLUMN                                   */
} xrt_algo;

/* Validate `g`, build the per-view geometry tables on `cuda_device` and allocate workspace.
 * Errors: XRT_ERR_INVALID_ARG (non-finite values, n <= 0, spacing <= 0, n_views <= 0,
 * angles == NULL, det_rows != 1 for 2D, sod <= 0 or sdd <= sod for divergent beams,
 * |tilt| >= pi/2, unknown flags, XRT_DET_CURVED with a parallel beam or a fan half-angle
 * >= pi/2); XRT_ERR_OOM; XRT_ERR_CUDA. */
xrt_status xrt_plan_create(const xrt_geometry* g, int cuda_device, xrt_plan* out);

/* Explicit ray list (Remark 3.5: any beam reduces to parallel-beam parameters; SURVEY
 * 8(f) N1).  Each ray is given by the paper's own parameters: dim 2 -> (s, phi, -, -), the line
 * {t theta + s theta_perp} of P:132-138; dim 3 -> (s1, s2, phi1, phi2), the line
 * {t theta + s1 theta_1 + s2 theta_2} of P:404-414.  The plan behaves as one view of n_rays detector
 * columns: sino is [1][1][n_rays] (ray i at index i); forward / adjoint / ray_units / f64 use the RAY
 * kernel family.  params: HOST [n_rays][4] fp64, copied at create time (unused entries ignored).
 * Errors: XRT_ERR_INVALID_ARG (dim not 2/3, n_rays < 1, non-finite params, invalid grid, flags). */
typedef struct {
    int32_t dim;             /* 2 or 3                                                           */
    int32_t flags;           /* must be 0                                                        */
    int64_t n[3];            /* image grid as in xrt_geometry (n[2] = 1 for dim 2)               */
    double spacing[3];
    double center[3];
    int64_t n_rays;          /* >= 1                                                              */
    const double* params;    /* HOST [n_rays][4]                                                  */
} xrt_ray_list;
xrt_status xrt_plan_create_rays(const xrt_ray_list* r, int cuda_device, xrt_plan* out);
xrt_status xrt_plan_destroy(xrt_plan p);

/* n_rays = n_views*det_rows*det_cols.  n_units (may be NULL) = nnz of the whole projection
 * matrix, counted exactly by the fp64 enumeration on first request (synchronous, cached). */
xrt_status xrt_plan_query(xrt_plan p, int64_t* n_rays, int64_t* n_units);

/* Select the kernel family used by xrt_forward / xrt_adjoint (default XRT_ALGO_AUTO).
 * XRT_ERR_UNSUPPORTED if the algorithm cannot serve this geometry. */
xrt_status xrt_plan_set_algorithm(xrt_plan p, int32_t op, int32_t algo);

/* Cumulative number of CUDA kernels this plan has launched (instrumentation). */
int64_t xrt_plan_launch_count(xrt_plan p);

/* Forward projection.  img: device fp32 [N_z][N_y][N_x] (read only); sino: device fp32
 * [n_views][det_rows][det_cols] (fully overwritten).  fp32 arithmetic, fp32 accumulation. */
xrt_status xrt_forward(xrt_plan p, const float* img, float* sino, void* cuda_stream);

/* Adjoint (backprojection).  sino: device fp32 (read only); img: device fp32, fully
 * overwritten with A^T sino. */
xrt_status xrt_adjoint(xrt_plan p, const float* sino, float* img, void* cuda_stream);

/* Staged adjoint, for overlapping a multi-GPU reduction of the image with the backprojection
 * (rays are independent).  The COLUMN adjoint runs band-major over blocks of
 * detector rows, each a z slab of the image (bands in row order: monotone in z).  xrt_adjoint_stages
 * reports S stages and, per stage s, the image rows [k_begin[s], k_end[s]) of [N_z][N_y][N_x] that
 * are FINAL after stage s (no later band reaches them; conservative, 2-cell margin); the ranges are
 * disjoint and cover [0, N_z) (an empty range: begin == end).  k_begin / k_end: host arrays of
 * capacity >= S, or both NULL to query S only.  xrt_adjoint_stage(p, sino, img, s, stream), called
 * for s = 0 .. S-1 in order on one stream, adds stage s's rows and writes img[k_begin[s]:k_end[s]]
 * (fully overwritten); after stage S-1 img = A^T sino, identical to xrt_adjoint.  A caller can
 * reduce img[k_begin[s]:k_end[s]] across ranks while stage s+1 computes.  Algorithms other than the
 * 3D COLUMN adjoint: S = 1 (the whole image).  Errors: XRT_ERR_INVALID_ARG (NULL, stage out of range). */
xrt_status xrt_adjoint_stages(xrt_plan p, int32_t* n_stages, int64_t* k_begin, int64_t* k_end);
xrt_status xrt_adjoint_stage(xrt_plan p, const float* sino, float* img, int32_t stage, void* cuda_stream);

/* fp64 variants (the paper's "switching float ... into double"): the same
 * operator with the fp64 unit enumeration of xrt_ray_units (units with l <= tau dropped) and fp64
 * sums.  img: device fp64 [N_z][N_y][N_x]; sino: device fp64 [n_views][det_rows][det_cols]; the
 * output is fully overwritten.  One thread per ray (RAY family), every geometry.  The adjoint
 * accumulates with fp64 atomics, so its last bits depend on the order of execution. */
xrt_status xrt_forward_f64(xrt_plan p, const double* img, double* sino, void* cuda_stream);
xrt_status xrt_adjoint_f64(xrt_plan p, const double* sino, double* img, void* cuda_stream);

/* Mixed precision (SURVEY 8(f) N2's "fp32-length / fp64-accumulate"): the fp32 unit walk of
 * the RAY family (the telescoped fp32 lengths C_up - C_low of xrt_forward), each product and every
 * sum in fp64.  img / sino: device fp64, layouts as xrt_forward_f64; the output is fully overwritten.
 * Forward and adjoint walk identical fp32 lengths, so <A x, y> = <x, A^T y> to fp64 rounding; the
 * adjoint accumulates with fp64 atomics (last bits order dependent).  Errors: XRT_ERR_INVALID_ARG
 * on NULL pointers; launch errors as XRT_ERR_CUDA. */
xrt_status xrt_forward_mixed(xrt_plan p, const double* img, double* sino, void* cuda_stream);
xrt_status xrt_adjoint_mixed(xrt_plan p, const double* sino, double* img, void* cuda_stream);

/* Attenuated X-ray transform (the generalized transform R_Phi of eq:generalizedRadontransform,
 * P:36-40, with the SPECT weight Phi(theta, x, t) = exp(-int_t^inf mu(x + s theta) ds); SURVEY 8(f)
 * N4, reading 23).  f = img and mu are unit-basis images on the plan's grid (eq:f_represent,
 * P:42-50), so per ray, with the units I in the order of t along theta (from the source towards the
 * detector; parallel beams: the paper's theta, P:132-138 / P:404-412):
 *     sino = sum_I f_I exp(-A_I) g(mu_I, l_I),   g(mu, l) = (1 - exp(-mu l)) / mu  (= l at mu = 0),
 * A_I = sum over the units J after I of mu_J l_J, l the intersection lengths of xrt_forward.
 * mu = 0 everywhere gives xrt_forward.  The adjoint is img_I = sum_m y_m exp(-A_mI) g(mu_I, l_mI).
 *   img, mu, sino: device fp32, layouts as xrt_forward (mu read only, same shape as img); the
 *   output is fully overwritten.  mu in physical 1/length (any finite value; mu >= 0 physically).
 * Kernels: on the 3D beams the column path (AUTO) walks each ray's units in path order, per band
 * of detector rows and xy tile (L2-resident), and combines a ray's tile pieces in path order
 * (S <- S exp(-A_t) + S_t); tilings of more than 16 tiles run untiled.  2D beams, ray lists and
 * steep rays: one thread per ray (RAY family).  fp32 arithmetic, the attenuation running product
 * in path order.  Errors: XRT_ERR_INVALID_ARG on NULL pointers. */
xrt_status xrt_forward_attenuated(xrt_plan p, const float* img, const float* mu, float* sino,
                                  void* cuda_stream);
xrt_status xrt_adjoint_attenuated(xrt_plan p, const float* sino, const float* mu, float* img,
                                  void* cuda_stream);

/* As xrt_forward / xrt_adjoint but with HOST buffers (pageable or pinned): the host->device copy
 * of the input, the kernels and the device->host copy of the output all run inside the call,
 * pipelined over view chunks; returns after the output is in host memory. */
xrt_status xrt_forward_host(xrt_plan p, const float* img_host, float* sino_host, void* cuda_stream);
xrt_status xrt_adjoint_host(xrt_plan p, const float* sino_host, float* img_host, void* cuda_stream);

/* CSR intersection dump for rays [ray_begin, ray_end), fp64 enumeration (reading 4:
 * units with l <= tau = 1e-9 * min(spacing) are dropped).  Row r (ray ray_begin + r) is
 * cols[row_ptr[r] .. row_ptr[r+1]) / lens[...], ascending flat index, lengths physical.
 *   row_ptr: device int64 [ray_end - ray_begin + 1] (required)
 *   cols, lens: device int64 / fp64 arrays of `capacity` entries, or both NULL for a count-only
 *              pass (two-phase use: count, allocate, fill)
 *   nnz_out: host, receives the total count (synchronous).
 * Errors: XRT_ERR_INVALID_ARG (range outside [0, n_rays), ray_end < ray_begin, NULL row_ptr or
 * nnz_out, exactly one of cols/lens NULL); XRT_ERR_CAPACITY (capacity < nnz; nothing written
 * to cols/lens); XRT_ERR_UNSUPPORTED (nnz > 2^31 - 1 in one call: split the range). */
xrt_status xrt_ray_units(xrt_plan p, int64_t ray_begin, int64_t ray_end, int64_t* row_ptr,
                         int64_t* cols, double* lens, int64_t capacity, int64_t* nnz_out,
                         void* cuda_stream);

/* Thread-local message describing the last non-OK status returned on this thread. */
const char* xrt_last_error(void);

/* (major << 16) | minor */
int32_t xrt_version(void);

#ifdef __cplusplus
}
#endif

#endif /* XRT_H */
