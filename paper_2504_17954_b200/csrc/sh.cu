// Stage-1 spherical-harmonics colour (forward + backward), float64.
//
// eval_sh / eval_sh_backward / view_dirs / view_dirs_backward
// (gaussians.py:427-529): one thread per Gaussian; the basis and its
// direction derivatives are rebuilt in registers (the reference materialises
// (N,B) and (N,B,3) arrays).  HBM-bound: 24 + 24*nb B in, 24 B out per
// Gaussian forward; backward adds d_rgb in and d_coeffs out.  Products
// follow numpy's left-to-right evaluation of each basis expression.
#include "ivr_common.cuh"

namespace ivr {

constexpr double kShC0 = 0.28209479177387814;
constexpr double kShC1 = 0.4886025119029199;
__constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
__constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

struct ShDir {
    double v[3], n, u[3];
};

// view_dirs: normalize_rows(mu - pos, eps=1e-12) (_mathutil.py:31-36)
__device__ __forceinline__ ShDir sh_dir(const double *mu, int64_t i, const double p[3]) {
    ShDir d;
    for (int k = 0; k < 3; ++k) d.v[k] = dsub(mu[3 * i + k], p[k]);
    d.n = norm3(d.v[0], d.v[1], d.v[2]);
    const double ne = d.n > 1e-12 ? d.n : 1e-12;
    for (int k = 0; k < 3; ++k) d.u[k] = ddiv(d.v[k], ne);
    return d;
}

// sh_basis (gaussians.py:427-494): B[b] and, when D != nullptr, dB[b]/d(x,y,z)
template <int DEG>
__device__ __forceinline__ void sh_basis(double x, double y, double z, double *B, double (*D)[3]) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    if (D)
        for (int b = 0; b < NB; ++b) D[b][0] = D[b][1] = D[b][2] = 0.0;
    B[0] = kShC0;
    if (DEG >= 1) {
        B[1] = dmul(-kShC1, y);
        B[2] = dmul(kShC1, z);
        B[3] = dmul(-kShC1, x);
        if (D) {
            D[1][1] = -kShC1;
            D[2][2] = kShC1;
            D[3][0] = -kShC1;
        }
    }
    if (DEG >= 2) {
        const double xx = dmul(x, x), yy = dmul(y, y), zz = dmul(z, z);
        B[4] = dmul(dmul(kShC2[0], x), y);
        B[5] = dmul(dmul(kShC2[1], y), z);
        B[6] = dmul(kShC2[2], dsub(dsub(dmul(2.0, zz), xx), yy));
        B[7] = dmul(dmul(kShC2[3], x), z);
        B[8] = dmul(kShC2[4], dsub(xx, yy));
        if (D) {
            D[4][0] = dmul(kShC2[0], y);
            D[4][1] = dmul(kShC2[0], x);
            D[5][1] = dmul(kShC2[1], z);
            D[5][2] = dmul(kShC2[1], y);
            D[6][0] = dmul(kShC2[2], dmul(-2.0, x));
            D[6][1] = dmul(kShC2[2], dmul(-2.0, y));
            D[6][2] = dmul(kShC2[2], dmul(4.0, z));
            D[7][0] = dmul(kShC2[3], z);
            D[7][2] = dmul(kShC2[3], x);
            D[8][0] = dmul(kShC2[4], dmul(2.0, x));
            D[8][1] = dmul(kShC2[4], dmul(-2.0, y));
        }
    }
    if (DEG >= 3) {
        const double xx = dmul(x, x), yy = dmul(y, y), zz = dmul(z, z);
        B[9] = dmul(dmul(kShC3[0], y), dsub(dmul(3.0, xx), yy));
        B[10] = dmul(dmul(dmul(kShC3[1], x), y), z);
        B[11] = dmul(dmul(kShC3[2], y), dsub(dsub(dmul(4.0, zz), xx), yy));
        B[12] = dmul(dmul(kShC3[3], z), dsub(dsub(dmul(2.0, zz), dmul(3.0, xx)), dmul(3.0, yy)));
        B[13] = dmul(dmul(kShC3[4], x), dsub(dsub(dmul(4.0, zz), xx), yy));
        B[14] = dmul(dmul(kShC3[5], z), dsub(xx, yy));
        B[15] = dmul(dmul(kShC3[6], x), dsub(xx, dmul(3.0, yy)));
        if (D) {
            D[9][0] = dmul(dmul(dmul(kShC3[0], 6.0), x), y);
            D[9][1] = dmul(kShC3[0], dsub(dmul(3.0, xx), dmul(3.0, yy)));
            D[10][0] = dmul(dmul(kShC3[1], y), z);
            D[10][1] = dmul(dmul(kShC3[1], x), z);
            D[10][2] = dmul(dmul(kShC3[1], x), y);
            D[11][0] = dmul(kShC3[2], dmul(dmul(-2.0, x), y));
            D[11][1] = dmul(kShC3[2], dsub(dsub(dmul(4.0, zz), xx), dmul(3.0, yy)));
            D[11][2] = dmul(kShC3[2], dmul(dmul(8.0, y), z));
            D[12][0] = dmul(kShC3[3], dmul(dmul(-6.0, x), z));
            D[12][1] = dmul(kShC3[3], dmul(dmul(-6.0, y), z));
            D[12][2] = dmul(kShC3[3], dsub(dsub(dmul(6.0, zz), dmul(3.0, xx)), dmul(3.0, yy)));
            D[13][0] = dmul(kShC3[4], dsub(dsub(dmul(4.0, zz), dmul(3.0, xx)), yy));
            D[13][1] = dmul(kShC3[4], dmul(dmul(-2.0, x), y));
            D[13][2] = dmul(kShC3[4], dmul(dmul(8.0, x), z));
            D[14][0] = dmul(kShC3[5], dmul(dmul(2.0, x), z));
            D[14][1] = dmul(kShC3[5], dmul(dmul(-2.0, y), z));
            D[14][2] = dmul(kShC3[5], dsub(xx, yy));
            D[15][0] = dmul(kShC3[6], dsub(dmul(3.0, xx), dmul(3.0, yy)));
            D[15][1] = dmul(kShC3[6], dmul(dmul(-6.0, x), y));
        }
    }
}

struct ShArgs {
    int64_t n;
    const double *mu, *coeffs;
    double pos[3];
    const double *d_rgb;
    double *rgb, *d_coeffs, *d_mu;
};

template <int DEG>
__global__ void __launch_bounds__(128) sh_eval_kernel(ShArgs A) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const ShDir d = sh_dir(A.mu, i, A.pos);
    double B[NB];
    sh_basis<DEG>(d.u[0], d.u[1], d.u[2], B, nullptr);
    const double *c = A.coeffs + (int64_t)NB * 3 * i;
    for (int ch = 0; ch < 3; ++ch) {
        double s = dmul(B[0], c[ch]);
#pragma unroll
        for (int b = 1; b < NB; ++b) s = dadd(s, dmul(B[b], c[3 * b + ch]));
        const double raw = dadd(s, 0.5);
        A.rgb[3 * i + ch] = raw > 0.0 ? raw : (raw < 0.0 ? 0.0 : raw);  // np.maximum(raw, 0)
    }
}

template <int DEG>
__global__ void __launch_bounds__(128) sh_bwd_kernel(ShArgs A) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const ShDir d = sh_dir(A.mu, i, A.pos);
    double B[NB], D[NB][3];
    sh_basis<DEG>(d.u[0], d.u[1], d.u[2], B, D);
    const double *c = A.coeffs + (int64_t)NB * 3 * i;
    double g[3];
    for (int ch = 0; ch < 3; ++ch) {
        double s = dmul(B[0], c[ch]);
#pragma unroll
        for (int b = 1; b < NB; ++b) s = dadd(s, dmul(B[b], c[3 * b + ch]));
        const double raw = dadd(s, 0.5);
        g[ch] = raw > 0.0 ? A.d_rgb[3 * i + ch] : 0.0;  // gate = raw > 0
    }
    double *dc = A.d_coeffs + (int64_t)NB * 3 * i;
    double dd[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        for (int ch = 0; ch < 3; ++ch) dc[3 * b + ch] = dmul(B[b], g[ch]);
        const double inner = dadd(dadd(dmul(c[3 * b], g[0]), dmul(c[3 * b + 1], g[1])),
                                  dmul(c[3 * b + 2], g[2]));
        for (int k = 0; k < 3; ++k) dd[k] = dadd(dd[k], dmul(inner, D[b][k]));
    }
    if (A.d_mu) {
        // normalize_rows_backward(v, d_dir) (_mathutil.py:39-44), no eps
        double u[3];
        for (int k = 0; k < 3; ++k) u[k] = ddiv(d.v[k], d.n);
        const double pr = dot3(dd, u);
        for (int k = 0; k < 3; ++k)
            A.d_mu[3 * i + k] = dadd(A.d_mu[3 * i + k], ddiv(dsub(dd[k], dmul(pr, u[k])), d.n));
    }
}

// sh_basis as an array function: basis (n, NB) and its direction
// derivatives (n, NB, 3) for given unit directions (gaussians.py:429-494)
template <int DEG>
__global__ void __launch_bounds__(128)
sh_basis_kernel(int64_t n, const double *dirs, double *basis, double *dbasis) {
    constexpr int NB = (DEG + 1) * (DEG + 1);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double B[NB], D[NB][3];
    sh_basis<DEG>(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], B, D);
    for (int b = 0; b < NB; ++b) {
        basis[(int64_t)NB * i + b] = B[b];
        if (dbasis)
            for (int k = 0; k < 3; ++k) dbasis[((int64_t)NB * i + b) * 3 + k] = D[b][k];
    }
}

static int sh_launch(bool bwd, int degree, const ShArgs &A, cudaStream_t st) {
    const int blocks = (int)((A.n + 127) / 128);
#define IVR_SH_CASE(DG)                                                          \
    case DG:                                                                     \
        if (bwd) sh_bwd_kernel<DG><<<blocks, 128, 0, st>>>(A);                   \
        else sh_eval_kernel<DG><<<blocks, 128, 0, st>>>(A);                      \
        break;
    switch (degree) {
        IVR_SH_CASE(0)
        IVR_SH_CASE(1)
        IVR_SH_CASE(2)
        IVR_SH_CASE(3)
    }
#undef IVR_SH_CASE
    return check_launch(bwd ? "sh_bwd_kernel" : "sh_eval_kernel");
}

}  // namespace ivr

extern "C" int ivr_sh_eval(int64_t n, int32_t degree, const double *mu, const double *coeffs,
                           const double cam_pos[3], double *rgb, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || degree < 0 || degree > 3 || !cam_pos || (n > 0 && (!mu || !coeffs || !rgb))) {
        set_error("ivr_sh_eval: bad argument (degree must be 0..3)");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    ShArgs A{};
    A.n = n;
    A.mu = mu;
    A.coeffs = coeffs;
    for (int k = 0; k < 3; ++k) A.pos[k] = cam_pos[k];
    A.rgb = rgb;
    return sh_launch(false, degree, A, (cudaStream_t)stream);
}

extern "C" int ivr_sh_bwd(int64_t n, int32_t degree, const double *mu, const double *coeffs,
                          const double cam_pos[3], const double *d_rgb, double *d_coeffs,
                          double *d_mu, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || degree < 0 || degree > 3 || !cam_pos ||
        (n > 0 && (!mu || !coeffs || !d_rgb || !d_coeffs))) {
        set_error("ivr_sh_bwd: bad argument (degree must be 0..3)");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    ShArgs A{};
    A.n = n;
    A.mu = mu;
    A.coeffs = coeffs;
    for (int k = 0; k < 3; ++k) A.pos[k] = cam_pos[k];
    A.d_rgb = d_rgb;
    A.d_coeffs = d_coeffs;
    A.d_mu = d_mu;
    return sh_launch(true, degree, A, (cudaStream_t)stream);
}

extern "C" int ivr_sh_basis(int64_t n, int32_t degree, const double *dirs, double *basis,
                            double *dbasis, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || degree < 0 || degree > 3 || (n > 0 && (!dirs || !basis))) {
        set_error("ivr_sh_basis: bad argument (degree must be 0..3)");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    const int blocks = (int)((n + 127) / 128);
    cudaStream_t st = (cudaStream_t)stream;
    switch (degree) {
        case 0: sh_basis_kernel<0><<<blocks, 128, 0, st>>>(n, dirs, basis, dbasis); break;
        case 1: sh_basis_kernel<1><<<blocks, 128, 0, st>>>(n, dirs, basis, dbasis); break;
        case 2: sh_basis_kernel<2><<<blocks, 128, 0, st>>>(n, dirs, basis, dbasis); break;
        default: sh_basis_kernel<3><<<blocks, 128, 0, st>>>(n, dirs, basis, dbasis); break;
    }
    return check_launch("sh_basis_kernel");
}
