// xrt_internal.cuh -- plan layout and the per-ray geometry shared by every kernel.
//
// A plan stores, per view v, the view-dependent terms of the paper's transformation of that
// view's rays to parallel-beam parameters (DESIGN.md section 5 "Plan"); every ray is then
// built in fp64 exactly as the paper parameterises it:
//   2D   ray (s, phi):  theta = (cos phi, sin phi), foot point s theta_perp
//   3D   ray (s1, s2, phi1, phi2): theta, theta_1, theta_2 of P:404-412, foot point
//        s1 theta_1 + s2 theta_2
//   fan  s = D t / sqrt(D^2 + t^2), phi = arctan(t / D) + alpha - pi/2
//   cone phi1 = phi1' + alpha, phi2 = beta, s1 = D sin(alpha), s2 = h cos^2(alpha) cos(beta),
//        alpha = arctan(t / D), beta = arctan(h / sqrt(D^2 + t^2))
//   helix s2 += H cos(beta)
// with t = u sod / sdd, h = v sod / sdd (flat detector at sdd, reading 8).  Sums of angles are
// formed with the addition theorem from per-view cos/sin (host, libm) and the per-ray
// cos/sin of arctan (algebraic), so no per-ray transcendental is evaluated.  Parameterising at
// the paper's foot point (not at the source) also makes the fixed coordinate of an
// axis-parallel ray exact (e.g. the central fan ray of a view at alpha = pi/2 has y = s = 0
// exactly, where the source has y = D cos(pi/2) = 6e-14), which the half-open tie rule needs.
#pragma once

#include <cstdint>
#include <cmath>

#include "../../include/xrt.h"

namespace xrt {

struct ViewRec {
    // par2d: cos/sin(phi); fan: cos/sin(alpha - pi/2); par3d: cos/sin(phi1);
    // cone / helical: cos/sin(phi1')
    double c1, s1;
    double c2, s2;  // par3d: cos/sin(phi2 = tilt); unused otherwise
    double H;       // helical source height H(phi1'); 0 otherwise
    double pad[3];  // par3d: pad[0] = tan(phi2), pad[1] = 1 / cos(phi2)
};

struct GridC {
    int n[3];          // N_x, N_y, N_z
    double d[3];       // spacing
    double x_lo, y_hi, z_hi;
    double tau;        // drop threshold for the fp64 CSR path (reading 4)
    double inv_dz;     // 1 / d_z
    int64_t nxy, nxyz;
};

struct DetC {
    int beam;                              // xrt_beam
    int curved;                            // 1: cylindrical detector (equiangular columns, XRT_DET_CURVED)
    int ray_dim;                           // XRT_RAYS: 2 or 3
    const double* rays;                    // XRT_RAYS: device [n_rays][4] paper parameters
    double D, sdd;                         // source-to-origin / -detector distances
    double inv_D;                          // 1 / D
    int cols, rows;
    double du, dv, cu, cv, off_u, off_v;  // u_c = (c - cu) du + off_u
    int64_t per_view;                      // rows * cols
};

constexpr double kSnap = 1e-12;  // |theta_a| <= kSnap -> 0 (reading 2/5)

// Index-space description of one ray: u(t) = u0 + t w, t the physical arc length.
// Unit (i, j, k) is [i, i+1) x [j, j+1) x [k, k+1) in u (P:151, P:427 shifted/scaled; reading 2).
struct Ray64 {
    double u0[3];
    double w[3];
    double inv_w[3];
    double t_in, t_out;  // clip of the line to the image box
    int cell[3];         // unit containing u(t) just after t_in
    int moving[3];       // w != 0
};

// Compute the ray of detector bin (view v, row r, col c) and clip it to the image box (fp64).
// Returns false when the ray has no unit with length > tau (the whole chord is <= tau).
__device__ __forceinline__ void paper_ray(const ViewRec& V, const DetC& dc, int r, int c,
                                          double p[3], double th[3]) {
    const double u = ((double)c - dc.cu) * dc.du + dc.off_u;
    const double v = ((double)r - dc.cv) * dc.dv + dc.off_v;
    const double D = dc.D;
    switch (dc.beam) {
        case XRT_RAYS: {   // explicit ray c of the list (Remark 3.5)
            const double* q = dc.rays + 4 * (int64_t)c;
            if (dc.ray_dim == 2) {   // (s, phi): theta = (cos phi, sin phi), point s theta_perp
                double sp, cp;
                sincos(q[1], &sp, &cp);
                th[0] = cp; th[1] = sp; th[2] = 0.0;
                p[0] = -q[0] * sp; p[1] = q[0] * cp; p[2] = 0.0;
            } else {                 // (s1, s2, phi1, phi2): theta, theta_1, theta_2 of P:404-412
                double a1, b1, a2, b2;   // sin/cos phi1, sin/cos phi2
                sincos(q[2], &a1, &b1);
                sincos(q[3], &a2, &b2);
                th[0] = b2 * b1; th[1] = b2 * a1; th[2] = a2;
                p[0] = q[0] * (-a1) + q[1] * (-a2 * b1);
                p[1] = q[0] * b1 + q[1] * (-a2 * a1);
                p[2] = q[1] * b2;
            }
            break;
        }
        case XRT_PAR2D: {  // (s, phi) = (u, angle_v)
            th[0] = V.c1; th[1] = V.s1; th[2] = 0.0;
            p[0] = -u * V.s1; p[1] = u * V.c1; p[2] = 0.0;
            break;
        }
        case XRT_FAN2D: {  // fan: equispaced (flat, t on the iso plane) or equiangular (curved)
            double cg, sg;
            if (dc.curved) {                                  // gamma = u / sdd
                sincos(u / dc.sdd, &sg, &cg);
            } else {
                const double t = u * D / dc.sdd;
                const double den = sqrt(D * D + t * t);
                cg = D / den; sg = t / den;                   // cos/sin(arctan(t/D))
            }
            const double s = D * sg;                          // s = D sin(gamma)
            const double cp = V.c1 * cg - V.s1 * sg;          // cos(gamma + alpha - pi/2)
            const double sp = V.s1 * cg + V.c1 * sg;
            th[0] = cp; th[1] = sp; th[2] = 0.0;
            p[0] = -s * sp; p[1] = s * cp; p[2] = 0.0;
            break;
        }
        case XRT_PAR3D: {  // (s1, s2, phi1, phi2) = (u, v, angle_v, tilt)
            const double c1 = V.c1, s1 = V.s1, c2 = V.c2, s2 = V.s2;
            th[0] = c2 * c1; th[1] = c2 * s1; th[2] = s2;
            p[0] = u * (-s1) + v * (-s2 * c1);
            p[1] = u * c1 + v * (-s2 * s1);
            p[2] = v * c2;
            break;
        }
        default: {  // cone / helical
            double ca, sa, cb, sb, s2;
            if (dc.curved) {
                // equiangular columns alpha = u / sdd, flat rows tan(beta) = v / sdd:
                // s1 = D sin(alpha), s2 = D cos(alpha) sin(beta) (+ H cos(beta))
                sincos(u / dc.sdd, &sa, &ca);
                const double tb = v / dc.sdd, r3 = sqrt(1.0 + tb * tb);
                cb = 1.0 / r3; sb = tb / r3;
                s2 = D * ca * sb + V.H * cb;
            } else {
                const double t = u * D / dc.sdd;
                const double h = v * D / dc.sdd;
                const double q = D * D + t * t;
                const double sq = sqrt(q);
                ca = D / sq; sa = t / sq;                     // alpha = arctan(t / D)
                const double r3 = sqrt(q + h * h);
                cb = sq / r3; sb = h / r3;                    // beta = arctan(h / sqrt(D^2+t^2))
                s2 = h * (ca * ca) * cb + V.H * cb;
            }
            const double s1 = D * sa;
            const double c1 = V.c1 * ca - V.s1 * sa;          // phi1 = phi1' + alpha
            const double n1 = V.s1 * ca + V.c1 * sa;
            th[0] = cb * c1; th[1] = cb * n1; th[2] = sb;
            p[0] = s1 * (-n1) + s2 * (-sb * c1);
            p[1] = s1 * c1 + s2 * (-sb * n1);
            p[2] = s2 * cb;
            break;
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (fabs(th[a]) <= kSnap) th[a] = 0.0;
}

__device__ __forceinline__ bool setup_ray(const ViewRec& V, const DetC& dc, const GridC& g,
                                          int r, int c, Ray64& R) {
    double o[3], th[3];
    paper_ray(V, dc, r, c, o, th);
    // index-space frame (P:140-151 / P:416-427 with spacing and centre: reading 2, 13, 14)
    R.u0[0] = (o[0] - g.x_lo) / g.d[0];
    R.u0[1] = (g.y_hi - o[1]) / g.d[1];
    R.u0[2] = (g.z_hi - o[2]) / g.d[2];
    R.w[0] = th[0] / g.d[0];
    R.w[1] = -th[1] / g.d[1];
    R.w[2] = -th[2] / g.d[2];
    double t_in = -INFINITY, t_out = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (R.w[a] == 0.0) {
            // fixed axis: inside slab c iff c <= u0 < c + 1 (half-open)
            if (!(R.u0[a] >= 0.0 && R.u0[a] < (double)g.n[a])) return false;
            R.moving[a] = 0;
            R.inv_w[a] = 0.0;
            R.cell[a] = (int)floor(R.u0[a]);
        } else {
            R.moving[a] = 1;
            R.inv_w[a] = 1.0 / R.w[a];
            const double t0 = (0.0 - R.u0[a]) * R.inv_w[a];
            const double t1 = ((double)g.n[a] - R.u0[a]) * R.inv_w[a];
            t_in = fmax(t_in, fmin(t0, t1));
            t_out = fmin(t_out, fmax(t0, t1));
        }
    }
    if (!(t_out - t_in > g.tau)) return false;
    R.t_in = t_in;
    R.t_out = t_out;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (!R.moving[a]) continue;
        const int N = g.n[a];
        int cc = (int)floor(R.u0[a] + t_in * R.w[a]);
        cc = cc < 0 ? 0 : (cc > N - 1 ? N - 1 : cc);
        // make the entry cell consistent with the crossing times T(b) = (b - u0) / w
        if (R.w[a] > 0.0) {
            if (cc + 1 <= N - 1 && ((double)(cc + 1) - R.u0[a]) * R.inv_w[a] <= t_in) cc += 1;
            else if (cc >= 1 && ((double)cc - R.u0[a]) * R.inv_w[a] > t_in) cc -= 1;
        } else {
            if (cc >= 1 && ((double)cc - R.u0[a]) * R.inv_w[a] <= t_in) cc -= 1;
            else if (cc + 1 <= N - 1 && ((double)(cc + 1) - R.u0[a]) * R.inv_w[a] > t_in) cc += 1;
        }
        R.cell[a] = cc;
    }
    return true;
}

}  // namespace xrt

// ---------------------------------------------------------------------------------- host side
#include <vector>
struct xrt_plan_s {
    int device = 0;
    int beam = 0;
    int dim = 3;
    xrt::GridC grid{};
    xrt::DetC det{};
    int64_t n_views = 0;
    int64_t n_rays = 0;
    int64_t n_units = -1;
    xrt::ViewRec* d_views = nullptr;   // device [n_views]
    float* d_work_fwd = nullptr;       // z-fastest, z-padded copy of the forward input (COLUMN)
    float* d_work_adj = nullptr;       // z-fastest, z-padded adjoint accumulator (COLUMN)
    float2* d_work_fd = nullptr;       // forward (COLUMN): per cell 2 x NzP (f, f[k+-1] - f[k]) cells
    float4* d_work_fd4 = nullptr;      // z-mirror forward, device path: interleaved (f, df, f', df') cells (first use)
    bool fd_forward = true;            // AUTO forward on the (f, delta f) volume (XRT_FWD_LEGACY=1: k_column)
    bool flat_z = false;               // every ray keeps one z cell (par3d, tilt 0): flat column kernels
    bool fd_mirror = false;            // circular cone symmetric in z: the fd forward walks the upper rows and their mirrors
    int64_t zpad = 0, nzp = 0;         // z padding per side and padded column length
    // xy tiling of the column kernels (L2 residency), per operator: [0] forward, [1] adjoint
    struct ColTiling {
        int tile = 0, n_tx = 1, n_ty = 1;
        void* d_items = nullptr;       // device uint2 work list (tiled) or nullptr (one tile)
        int64_t n_items = 0;
    } ct[2], ct_fd;                    // ct_fd: the (f, delta f) forward's items (view blocks x column groups)
    // ct_fd's items regrouped into kFwdParts contiguous view ranges (each part still sorted by tile):
    // the host pipeline launches the last band part by part, so a part's sinogram rows travel to the
    // host while the next part computes
    static constexpr int kFwdParts = 4;
    void* d_fd_part_items = nullptr;
    int64_t fd_part_off[kFwdParts + 1] = {0, 0, 0, 0, 0};
    int64_t fd_part_view[kFwdParts + 1] = {0, 0, 0, 0, 0};   // first view of each part (+ end)
    // the same for the adjoint's items (ct[1]): the host pipeline uploads and runs its FIRST band
    // part by part, so only the first part's upload is exposed
    void* d_adj_part_items = nullptr;
    int64_t adj_part_off[kFwdParts + 1] = {0, 0, 0, 0, 0};
    int64_t adj_part_view[kFwdParts + 1] = {0, 0, 0, 0, 0};
    int col_np = 2;                    // ray pairs per lane of the forward column kernel (rows per band = 64 col_np)
    int col_np_adj = 1;                // ... of the adjoint column kernel (measured: 1 pair is faster, cfg 3 / 4)
    // attenuated operators on the column path (allocated on first use)
    float* d_work_att = nullptr;       // z-fastest float2 (f, mu) cells
    float* d_att_A = nullptr;          // per-ray total attenuation (sinogram-shaped)
    float* d_att_pieces = nullptr;     // tiled attenuated forward: (sigma, S_t, A_t) per ray of a band and tile
    unsigned* d_att_mumax = nullptr;   // max |mu| (float bits)
    void* d_coldesc = nullptr;         // per-(view, column) path descriptors (COLUMN, GATHER)
    double* d_rays = nullptr;          // explicit ray list (XRT_RAYS)
    void* d_raydesc2d = nullptr;       // per-(view, column) rays in index space (2D GATHER)
    void* d_ray2d_walk = nullptr;      // 2D RAY forward in pieces: per-ray fp32 walk state (32 B per ray)
    float* d_fwd_t = nullptr;          // 2D RAY forward in pieces: transposed input (x-major rays walk it)
    float2* d_fd2d = nullptr;          // 2D forward in pieces on (f, f[+-1] - f): 4 images (row-major / transposed, +-1)
    float* d_img_t = nullptr;          // 2D COLUMN (slice) kernels: transposed image / accumulator
    bool slice_v1 = false;             // XRT_SLICE_V1=1: the round-1 slice adjoint (A/B)
    float* d_gather_y = nullptr;       // GATHER workspace: rescaled, transposed sinogram of one view block
    int64_t gather_views = 0;          // views per GATHER launch
    // host-pipeline staging (allocated on first *_host call)
    float* d_stage_img = nullptr;
    float* d_stage_sino = nullptr;
    void* aux_stream = nullptr;
    void* aux_stream2 = nullptr;       // host pipelines: downloads of final image rows (staged adjoint)
    void* aux_stream3 = nullptr;       // forward host pipeline: every other band's kernels (band tails overlap)
    int algo_fwd = XRT_ALGO_AUTO;
    int algo_adj = XRT_ALGO_AUTO;
    bool column_ok = false;            // geometry admits the column-shared kernels
    std::vector<int64_t> adj_stage_k;  // staged adjoint: per band b, image rows [k0, k1) final after b
    std::vector<int64_t> fwd_band_k;   // forward bands: per band b, the image rows [k0, k1) its rays reach
    std::vector<int64_t> fwdm_band_k;  // z-mirror forward bands: per band b, [k0, k1) of its upper rows, then of their mirrors
    int64_t launches = 0;
};

namespace xrt {
// kernels (kern_ray.cu)
cudaError_t launch_forward_ray(const xrt_plan_s* p, const float* img, float* sino, int64_t ray0,
                               int64_t ray1, cudaStream_t s);
cudaError_t launch_adjoint_ray(const xrt_plan_s* p, const float* sino, float* img, int64_t ray0,
                               int64_t ray1, cudaStream_t s);
cudaError_t launch_units_count(const xrt_plan_s* p, int64_t ray0, int64_t ray1, int64_t* counts,
                               cudaStream_t s);
size_t ray2d_walk_bytes();
bool adjoint2d_pieces(const xrt_plan_s* p);
bool ray2d_fd_on(const xrt_plan_s* p);
bool slice2d_pieces_on(const xrt_plan_s* p);
cudaError_t launch_slice2d_adj_pc(const xrt_plan_s* p, const float* y_in, float* acc_img, float* acc_imgT,
                                  cudaStream_t s);
cudaError_t launch_fd2d(const xrt_plan_s* p, const float* img, cudaStream_t s);
cudaError_t launch_adjoint_ray2d_pc(const xrt_plan_s* p, const float* sino, float* acc_img, float* acc_imgT,
                                    cudaStream_t s);
cudaError_t launch_ray2d_walk_desc(const xrt_plan_s* p, cudaStream_t s);
cudaError_t launch_forward_att(const xrt_plan_s* p, const float* img, const float* mu, float* sino, int64_t ray0,
                               int64_t ray1, cudaStream_t s);
cudaError_t launch_adjoint_att(const xrt_plan_s* p, const float* sino, const float* mu, float* img, int64_t ray0,
                               int64_t ray1, cudaStream_t s);
cudaError_t launch_att_prepare(const xrt_plan_s* p, const float* img, const float* mu, float* work2,
                               unsigned* mumax, cudaStream_t s);
cudaError_t launch_forward_att_column(const xrt_plan_s* p, const float* work2, const unsigned* mumax, float* sino,
                                      float* pieces, cudaStream_t s);
constexpr int kMaxAttTiles = 16;   // tile pieces per ray the attenuated combine holds (att_tiled)
bool att_tiled(const xrt_plan_s* p);
int64_t att_piece_floats(const xrt_plan_s* p);
cudaError_t launch_adjoint_att_tiled(const xrt_plan_s* p, const float* mu_zfast, float* pieces,
                                     const unsigned* mumax, const float* y, float* acc_zfast, cudaStream_t s);
cudaError_t launch_adjoint_att_column(const xrt_plan_s* p, const float* mu_zfast, float* sinoA,
                                      const unsigned* mumax, const float* y, float* acc_zfast, cudaStream_t s);
cudaError_t launch_forward64(const xrt_plan_s* p, const double* img, double* sino, int64_t ray0,
                             int64_t ray1, cudaStream_t s);
cudaError_t launch_adjoint64(const xrt_plan_s* p, const double* sino, double* img, int64_t ray0,
                             int64_t ray1, cudaStream_t s);
cudaError_t launch_forward_mixed(const xrt_plan_s* p, const double* img, double* sino, int64_t ray0,
                                 int64_t ray1, cudaStream_t s);
cudaError_t launch_adjoint_mixed(const xrt_plan_s* p, const double* sino, double* img, int64_t ray0,
                                 int64_t ray1, cudaStream_t s);
cudaError_t launch_units_fill(const xrt_plan_s* p, int64_t ray0, int64_t ray1,
                              const int64_t* row_ptr, int64_t* cols, double* lens, cudaStream_t s);
// kernels (kern_column.cu)
cudaError_t launch_to_zfast(const xrt_plan_s* p, const float* img, float* work, cudaStream_t s);
cudaError_t launch_from_zfast(const xrt_plan_s* p, const float* work, float* img, cudaStream_t s);
cudaError_t launch_from_zfast_rows(const xrt_plan_s* p, const float* work, float* img, int64_t k0, int64_t k1,
                                   cudaStream_t s);
cudaError_t launch_forward_column(const xrt_plan_s* p, const float* vol_zfast, float* sino,
                                  int64_t v0, int64_t v1, cudaStream_t s);
cudaError_t launch_adjoint_column(const xrt_plan_s* p, const float* sino, float* vol_zfast,
                                  int64_t v0, int64_t v1, cudaStream_t s);
}  // namespace xrt
#include <vector>
namespace xrt {
int build_column_items(const xrt_plan_s* p, const ViewRec* views_host, int ts, int ntx, int nty,
                       std::vector<uint2>& items, bool fd = false);
size_t column_desc_bytes();
int choose_col_np(int rows);
int column_cta_columns();
cudaError_t launch_col_desc(const xrt_plan_s* p, cudaStream_t s);
cudaError_t launch_adjoint_gather(const xrt_plan_s* p, const float* sino, float* vol_zfast, cudaStream_t s);
int64_t gather_launches(const xrt_plan_s* p);
int column_band_rows(const xrt_plan_s* p, bool adj);
size_t raydesc2d_bytes();
cudaError_t launch_raydesc2d(const xrt_plan_s* p, cudaStream_t s);
cudaError_t launch_adjoint_gather2d(const xrt_plan_s* p, const float* sino, float* img, cudaStream_t s);
cudaError_t launch_transpose2d(const float* in, float* out, int rows, int cols, bool add, cudaStream_t s);
cudaError_t launch_slice2d_adj(const xrt_plan_s* p, const float* y_in, float* acc_img, float* acc_imgT,
                               cudaStream_t s);
cudaError_t launch_slice2d(const xrt_plan_s* p, bool adjoint, const float* img, const float* imgT,
                           const float* y_in, float* sino_out, float* acc_img, float* acc_imgT,
                           cudaStream_t s);
int column_bands(const xrt_plan_s* p, bool adj);
cudaError_t launch_forward_column_bands(const xrt_plan_s* p, const float* vol_zfast, float* sino, int b0,
                                        int b1, cudaStream_t s);
cudaError_t launch_to_fd(const xrt_plan_s* p, const float* img, float2* fd, cudaStream_t s);
cudaError_t launch_to_fd_rows(const xrt_plan_s* p, const float* img, float2* fd, int ka, int kb, cudaStream_t s);
cudaError_t launch_forward_fd_bands(const xrt_plan_s* p, const float2* fd, float* sino, int b0, int b1,
                                    cudaStream_t s);
int fd_view_block();                 // views per CTA of the fd forward (kFdViews)
bool fd_mirror_active(const xrt_plan_s* p);
bool fd_mirror_on_x(const xrt_plan_s* p);
bool fd_f4_on(const xrt_plan_s* p);
cudaError_t launch_to_fd4(const xrt_plan_s* p, const float* img, float4* fd4, cudaStream_t s);
cudaError_t launch_to_fd4_rows(const xrt_plan_s* p, const float* img, float4* fd4, int ka, int kb, cudaStream_t s);
int fd_mirror_bands(const xrt_plan_s* p);
int fd_mirror_band_rows();           // upper-half rows per z-mirror band
cudaError_t launch_forward_fd_mirror_bands(const xrt_plan_s* p, const float2* fd, float* sino, int b0, int b1,
                                           cudaStream_t s);
cudaError_t launch_forward_fd_mirror_band_part(const xrt_plan_s* p, const float2* fd, float* sino, int b, int part,
                                               cudaStream_t s);
cudaError_t launch_adjoint_column_band_part(const xrt_plan_s* p, const float* sino, float* vol_zfast, int b,
                                            int part, cudaStream_t s);
cudaError_t launch_forward_fd_band_part(const xrt_plan_s* p, const float2* fd, float* sino, int b, int part,
                                        cudaStream_t s);
cudaError_t launch_adjoint_column_bands(const xrt_plan_s* p, const float* sino, float* vol_zfast, int b0,
                                        int b1, cudaStream_t s);
}  // namespace xrt
