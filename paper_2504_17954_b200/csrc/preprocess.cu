// K1 -- fused per-Gaussian preprocess (float64, one thread per Gaussian).
//
// Replaces, bit-faithfully up to transcendental ulps:
//   scene.apply_edits            scene.py:199-228   (opacity logit round trip)
//   shading.shade_gaussians      shading.py:225-329 (Blinn-Phong, coeff transform)
//   gaussians.project_gaussians  gaussians.py:296-346 (EWA, dgemm FMA chains)
//   rasterizer.rasterize_forward rasterizer.py:88-121 (radius/rect/count),
//                                rasterizer.py:134-153 (f32 packing)
// and emits the float32 blend record plus the conservative sigma threshold
// `hi` that lets the blend skip a pair in float32 only when the reference's
// float64 alpha test certainly skips it.
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {

struct ShadeOut {
    double rgb[3];
    double amb[3], dif[3], spec;
};

// shading.py:236-297 for one splat.  `nrm` is the unit normal (eps 1e-12).
__device__ __forceinline__ void shade_one(const ivr_shading &S, const ivr_frame_params &P,
                                          int64_t i, int32_t sid, const double mu[3],
                                          const double nrm[3], ShadeOut &o) {
    const ivr_camera &cam = P.cam;
    double w[3] = {dsub(cam.position[0], mu[0]), dsub(cam.position[1], mu[1]),
                   dsub(cam.position[2], mu[2])};
    const double wn = dmax(norm3(w[0], w[1], w[2]), 1e-12);
    const double v[3] = {ddiv(w[0], wn), ddiv(w[1], wn), ddiv(w[2], wn)};
    double l[3], h[3];
    if (!P.orbital) {
        for (int k = 0; k < 3; ++k) l[k] = h[k] = v[k];
    } else {
        double u[3];
        for (int k = 0; k < 3; ++k) {
            l[k] = P.light_dir[k];
            u[k] = dadd(v[k], l[k]);
        }
        const double un = dmax(norm3(u[0], u[1], u[2]), 1e-12);
        for (int k = 0; k < 3; ++k) h[k] = ddiv(u[k], un);
    }
    const double sa = sigmoid_ref(S.k_a_raw[i]);
    const double sd = sigmoid_ref(S.k_d_raw[i]);
    const double ss = sigmoid_ref(S.k_s_raw[i]);
    const double beta1 = dadd(exp(S.log_beta[i]), 1.0);
    const double ta = dadd(dmul(P.lam[0], sa), P.b[0]);
    const double td = dadd(dmul(P.lam[1], sd), P.b[1]);
    const double tsp = dadd(dmul(P.lam[2], ss), P.b[2]);
    const double tb = dadd(dmul(P.lam[3], beta1), P.b[3]);
    const double k_a = dmul(P.term_scales[0], clip01(ta));
    const double k_d = dmul(P.term_scales[1], clip01(td));
    const double k_s = dmul(P.term_scales[2], clip01(tsp));
    const double beta = dmul(P.term_scales[3], dmax(tb, 1.0));
    const double *cp = S.per_splat_palette ? S.palette + 3 * i : S.palette + 3 * (int64_t)sid;
    double cv[3];
    for (int k = 0; k < 3; ++k) cv[k] = clip01(dadd(cp[k], S.delta_c[3 * i + k]));
    const double a_ndl = fabs(dot3(nrm, l));
    const double a_ndh = fabs(dot3(nrm, h));
    double spow = 0.0;
    if (a_ndh > 0.0) spow = pow(dmax(a_ndh, 1e-300), beta);
    if (!(a_ndl > 0.0)) spow = 0.0;
    const double kdl = dmul(k_d, a_ndl);
    o.spec = dmul(dmul(k_s, spow), 1.0);
    for (int k = 0; k < 3; ++k) {
        o.amb[k] = dmul(k_a, cv[k]);
        o.dif[k] = dmul(kdl, cv[k]);
        o.rgb[k] = dadd(dadd(o.amb[k], o.dif[k]), o.spec);
    }
}

__device__ __forceinline__ void preprocess_one(const ivr_gaussians &G, const ivr_shading &S,
                                               int has_shading, const ivr_edits &E, int has_edits,
                                               const ivr_frame_params &P, const ivr_layout &L,
                                               const ivr_proj_out &O, int f64_mode, int64_t i) {
    const ivr_camera &cam = P.cam;
    const int32_t sid = (has_edits && E.scene_id) ? E.scene_id[i] : 0;

    // ---- effective opacity (scene.py:214-220; every splat when any scale != 1)
    double o_logit = G.o_logit[i];
    if (has_edits && P.rescale_opacity && E.opacity_scale) {
        double p = dmul(E.opacity_scale[sid], sigmoid_ref(o_logit));
        p = p < 1e-12 ? 1e-12 : (p > 1.0 - 1e-9 ? 1.0 - 1e-9 : p);
        o_logit = log(ddiv(p, dsub(1.0, p)));
    }
    const double opacity = sigmoid_ref(o_logit);

    // ---- projection (gaussians.py:302-339)
    const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
    const double qr[4] = {G.q_raw[4 * i], G.q_raw[4 * i + 1], G.q_raw[4 * i + 2],
                          G.q_raw[4 * i + 3]};
    const double qn = norm4(qr[0], qr[1], qr[2], qr[3]);
    const double qw = ddiv(qr[0], qn), qx = ddiv(qr[1], qn), qy = ddiv(qr[2], qn),
                 qz = ddiv(qr[3], qn);
    const double s[3] = {exp(G.log_s[3 * i]), exp(G.log_s[3 * i + 1]), exp(G.log_s[3 * i + 2])};
    const double *W = cam.rotation;
    const double d[3] = {dsub(mu[0], cam.position[0]), dsub(mu[1], cam.position[1]),
                         dsub(mu[2], cam.position[2])};
    double t[3];
    for (int j = 0; j < 3; ++j) t[j] = chain3(d[0], W[3 * j], d[1], W[3 * j + 1], d[2], W[3 * j + 2]);
    const double tz = t[2];
    bool valid = tz > kNearPlane;
    const double tzs = valid ? tz : 1.0;
    const double f = cam.focal;
    const double mx = dadd(ddiv(dmul(f, t[0]), tzs), cam.cx);
    const double my = dadd(ddiv(dmul(f, t[1]), tzs), cam.cy);

    // quat_to_rot (gaussians.py:222-236)
    double R[9];
    R[0] = dsub(1.0, dmul(2.0, dadd(dmul(qy, qy), dmul(qz, qz))));
    R[1] = dmul(2.0, dsub(dmul(qx, qy), dmul(qw, qz)));
    R[2] = dmul(2.0, dadd(dmul(qx, qz), dmul(qw, qy)));
    R[3] = dmul(2.0, dadd(dmul(qx, qy), dmul(qw, qz)));
    R[4] = dsub(1.0, dmul(2.0, dadd(dmul(qx, qx), dmul(qz, qz))));
    R[5] = dmul(2.0, dsub(dmul(qy, qz), dmul(qw, qx)));
    R[6] = dmul(2.0, dsub(dmul(qx, qz), dmul(qw, qy)));
    R[7] = dmul(2.0, dadd(dmul(qy, qz), dmul(qw, qx)));
    R[8] = dsub(1.0, dmul(2.0, dadd(dmul(qx, qx), dmul(qy, qy))));
    double M3[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) M3[3 * r + c] = dmul(R[3 * r + c], s[c]);
    double C3[9];  // M3 @ M3^T
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            C3[3 * r + c] = chain3(M3[3 * r], M3[3 * c], M3[3 * r + 1], M3[3 * c + 1],
                                   M3[3 * r + 2], M3[3 * c + 2]);
    double J[6] = {ddiv(f, tzs), 0.0, ddiv(dmul(-f, t[0]), dmul(tzs, tzs)),
                   0.0, ddiv(f, tzs), ddiv(dmul(-f, t[1]), dmul(tzs, tzs))};
    double M[6];  // J @ W
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            M[3 * r + c] = chain3(J[3 * r], W[c], J[3 * r + 1], W[3 + c], J[3 * r + 2], W[6 + c]);
    double A[6];  // M @ cov3d
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            A[3 * r + c] = chain3(M[3 * r], C3[c], M[3 * r + 1], C3[3 + c], M[3 * r + 2], C3[6 + c]);
    double C2[4];  // A @ M^T
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c)
            C2[2 * r + c] = chain3(A[3 * r], M[3 * c], A[3 * r + 1], M[3 * c + 1], A[3 * r + 2],
                                   M[3 * c + 2]);
    C2[0] = dadd(C2[0], kCov2dDilation);
    C2[3] = dadd(C2[3], kCov2dDilation);
    const double ca = C2[0], cb = C2[1], cc = C2[3];
    const double det = dsub(dmul(ca, cc), dmul(cb, cb));
    const double dets = det > 0.0 ? det : 1.0;
    const double q0 = ddiv(cc, dets), q1 = ddiv(-cb, dets), q2 = ddiv(ca, dets);
    valid = valid && (det > 0.0);

    // ---- radius / visibility / tile rect (rasterizer.py:88-118)
    const double half_tr = dmul(0.5, dadd(ca, cc));
    const double dac = dsub(ca, cc);
    const double disc = dadd(dmul(0.25, dmul(dac, dac)), dmul(cb, cb));
    const double lam_max = dadd(half_tr, sqrt(dmax(disc, 0.0)));
    const double cut = sqrt(dmul(2.0, log(dmax(ddiv(opacity, kAlphaSkip), 1.0))));
    const double radius = dadd(ceil(dmul(sqrt(dmax(lam_max, 0.0)), cut)), 1.0);
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    bool visible = valid && (opacity >= kAlphaSkip) && (radius > 0.0);
    visible = visible && (dadd(mx, radius) >= 0.0) && (dsub(mx, radius) < (double)cam.width) &&
              (dadd(my, radius) >= 0.0) && (dsub(my, radius) < (double)cam.height);
    auto tclip = [](double x, int hi) -> int {
        x = floor(x / 16.0);
        x = x < 0.0 ? 0.0 : (x > (double)hi ? (double)hi : x);
        return (int)x;
    };
    int tx0 = 0, tx1 = -1, ty0 = 0, ty1 = -1, cnt = 0;
    if (visible) {
        tx0 = tclip(dsub(mx, radius), ntx - 1);
        tx1 = tclip(dadd(mx, radius), ntx - 1);
        ty0 = tclip(dsub(my, radius), nty - 1);
        ty1 = tclip(dadd(my, radius), nty - 1);
        cnt = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
    }
    O.depth_key[i] = visible ? (uint64_t)__double_as_longlong(tz) : ~0ull;
    O.count[i] = cnt;
    ushort4 rc;
    rc.x = (unsigned short)tx0; rc.y = (unsigned short)(tx1 < 0 ? 0 : tx1);
    rc.z = (unsigned short)ty0; rc.w = (unsigned short)(ty1 < 0 ? 0 : ty1);
    reinterpret_cast<ushort4 *>(O.rect)[i] = rc;

    // ---- normals (GaussianGeometry.normals, eps 1e-12)
    const double nr[3] = {G.n_raw[3 * i], G.n_raw[3 * i + 1], G.n_raw[3 * i + 2]};
    const double nn = dmax(norm3(nr[0], nr[1], nr[2]), 1e-12);
    const double nrm[3] = {ddiv(nr[0], nn), ddiv(nr[1], nn), ddiv(nr[2], nn)};

    ShadeOut sh;
    if (has_shading) shade_one(S, P, i, sid, mu, nrm, sh);

    // ---- float32 blend record (rasterizer.py:151-153 casts) + skip threshold
    const float mx32 = (float)mx, my32 = (float)my;
    const float a32 = (float)q0, b32 = (float)q1, c32 = (float)q2, o32 = (float)opacity;
    float hi32 = __int_as_float(0x7f800000);  // +inf: always take the exact path
    float thr32 = 0.0f;                         // ln(o / (1/255)): alpha-skip exponent
    {
        const double a = a32, b = b32, c = c32;
        const double oo = f64_mode ? opacity : (double)o32;
        const double thr = log(oo / kAlphaSkip);
        if (thr == thr && fabs(thr) < 1e30) thr32 = (float)thr;
        const double hm = 0.5 * (a + c), dd = sqrt(0.25 * (a - c) * (a - c) + b * b);
        const double lmin = hm - dd, lmaxq = hm + dd;
        if (lmin > 0.0 && a > 0.0 && c > 0.0 && thr == thr) {
            const double cT = (fmax(a, c) + fabs(b)) / lmin;
            const double eps_f = (f64_mode ? 40.0 : 32.0) * 5.9604644775390625e-08;
            double hi = (thr + 1e-9 * (1.0 + fabs(thr))) * (1.0 + eps_f * cT) + 1e-7;
            if (f64_mode) {
                const double e = 1.1920928955078125e-07 * (fabs(mx) + fabs(my) + 1.0);
                hi += 1.5 * sqrt(2.0 * fmax(hi, 0.0) * lmaxq) * e + lmaxq * e * e;
            }
            hi32 = __double2float_ru(hi);
        }
    }
    float4 *rec = reinterpret_cast<float4 *>(O.rec) + 2 * i;
    rec[0] = make_float4(mx32, my32, o32, hi32);
    rec[1] = make_float4(0.5f * a32, b32, 0.5f * c32, thr32);
    if (O.rec64) {
        double *r = O.rec64 + 8 * i;
        r[0] = mx; r[1] = my; r[2] = q0; r[3] = q1; r[4] = q2; r[5] = opacity; r[6] = tz; r[7] = 0.0;
    }

    // ---- packed values (rasterizer.py:134-149)
    const int K = L.k;
    float *vrow = O.values + (int64_t)K * i;
    double *vrow64 = O.values64 ? O.values64 + (int64_t)K * i : nullptr;
    auto put = [&](int col, double x) {
        vrow[col] = (float)x;
        if (vrow64) vrow64[col] = x;
    };
    if (L.col_color >= 0) {
        for (int k = 0; k < 3; ++k)
            put(L.col_color + k, has_shading ? sh.rgb[k] : (L.colors ? L.colors[3 * i + k] : 0.0));
    }
    if (L.col_alpha >= 0) put(L.col_alpha, 1.0);
    if (L.col_depth >= 0) put(L.col_depth, tz);
    if (L.col_normal >= 0)
        for (int k = 0; k < 3; ++k) put(L.col_normal + k, nrm[k]);
    for (int a = 0; a < L.n_attr; ++a) {
        const int w = L.attr_width[a];
        for (int k = 0; k < w; ++k) put(L.attr_col[a] + k, L.attr[a][(int64_t)w * i + k]);
    }

    // ---- optional float64 parity outputs
    if (O.mean2d) { O.mean2d[2 * i] = mx; O.mean2d[2 * i + 1] = my; }
    if (O.conic) { O.conic[3 * i] = q0; O.conic[3 * i + 1] = q1; O.conic[3 * i + 2] = q2; }
    if (O.cov2d) for (int k = 0; k < 4; ++k) O.cov2d[4 * i + k] = C2[k];
    if (O.depth) O.depth[i] = tz;
    if (O.opacity) O.opacity[i] = opacity;
    if (O.radius) O.radius[i] = radius;
    if (O.valid) O.valid[i] = valid ? 1 : 0;
    if (O.rgb && has_shading) for (int k = 0; k < 3; ++k) O.rgb[3 * i + k] = sh.rgb[k];
}

// Per-frame parameters (camera, light, transform, rescale flag) are staged in
// shared memory once per block, from kernel parameters or from device memory.
__device__ __forceinline__ void stage_params(const ivr_frame_params *src, ivr_frame_params &dst) {
    static_assert(sizeof(ivr_frame_params) % 4 == 0, "params must be word-sized");
    constexpr int kWords = (int)(sizeof(ivr_frame_params) / 4);
    for (int w = threadIdx.x; w < kWords; w += blockDim.x)
        reinterpret_cast<int *>(&dst)[w] = reinterpret_cast<const int *>(src)[w];
    __syncthreads();
}

__global__ void __launch_bounds__(256)
preprocess_kernel(ivr_gaussians G, ivr_shading S, int has_shading, ivr_edits E, int has_edits,
                  ivr_frame_params Pv, const ivr_frame_params *__restrict__ Pd, ivr_layout L,
                  ivr_proj_out O, int f64_mode) {
    __shared__ ivr_frame_params sp;
    stage_params(Pd ? Pd : &Pv, sp);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.n) return;
    preprocess_one(G, S, has_shading, E, has_edits, sp, L, O, f64_mode, i);
}

__global__ void __launch_bounds__(256)
shade_kernel(ivr_gaussians G, ivr_shading S, const int32_t *scene_id, ivr_frame_params Pv,
             double *rgb, double *terms) {
    __shared__ ivr_frame_params sp;
    stage_params(&Pv, sp);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.n) return;
    const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
    const double nr[3] = {G.n_raw[3 * i], G.n_raw[3 * i + 1], G.n_raw[3 * i + 2]};
    const double nn = dmax(norm3(nr[0], nr[1], nr[2]), 1e-12);
    const double nrm[3] = {ddiv(nr[0], nn), ddiv(nr[1], nn), ddiv(nr[2], nn)};
    ShadeOut sh;
    shade_one(S, sp, i, scene_id ? scene_id[i] : 0, mu, nrm, sh);
    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = sh.rgb[k];
    if (terms) {
        for (int k = 0; k < 3; ++k) {
            terms[9 * i + k] = sh.amb[k];
            terms[9 * i + 3 + k] = sh.dif[k];
            terms[9 * i + 6 + k] = sh.spec;
        }
    }
}

ivr_frame_params params_from(const ivr_camera &cam, const ivr_shading *S, const ivr_edits *E) {
    ivr_frame_params P{};
    P.cam = cam;
    if (S) {
        P.orbital = S->orbital;
        for (int k = 0; k < 3; ++k) P.light_dir[k] = S->light_dir[k];
        for (int k = 0; k < 4; ++k) {
            P.term_scales[k] = S->term_scales[k];
            P.lam[k] = S->lam[k];
            P.b[k] = S->b[k];
        }
    }
    P.rescale_opacity = E ? E->rescale_opacity : 0;
    return P;
}

}  // namespace ivr

extern "C" int ivr_preprocess_fwd(const ivr_gaussians *g, const ivr_shading *shading,
                                  const ivr_edits *edits, const ivr_camera *cam,
                                  const ivr_layout *layout, ivr_proj_out *out, int32_t f64_mode,
                                  ivr_stream_t stream) {
    if (!g || !cam || !layout || !out || g->n < 0) {
        ivr::set_error("ivr_preprocess_fwd: null argument");
        return IVR_ERR_ARG;
    }
    if (!out->depth_key || !out->count || !out->rect || !out->rec || !out->values || layout->k < 1 ||
        layout->n_attr < 0 || layout->n_attr > IVR_MAX_ATTRS || cam->width < 1 || cam->height < 1) {
        ivr::set_error("ivr_preprocess_fwd: missing output buffer or bad layout");
        return IVR_ERR_ARG;
    }
    if (f64_mode && (!out->rec64 || !out->values64)) {
        ivr::set_error("ivr_preprocess_fwd: float64 mode needs rec64 and values64");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    ivr_shading S{};
    ivr_edits E{};
    if (shading) S = *shading;
    if (edits) E = *edits;
    const int threads = 256;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    ivr_frame_params P = ivr::params_from(*cam, shading, edits);
    ivr::preprocess_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        *g, S, shading != nullptr, E, edits != nullptr, P, nullptr, *layout, *out, f64_mode);
    return ivr::check_launch("preprocess_kernel");
}

extern "C" int ivr_preprocess_fwd_params(const ivr_gaussians *g, const ivr_shading *shading,
                                         const ivr_edits *edits, const ivr_frame_params *params,
                                         int32_t width, int32_t height, const ivr_layout *layout,
                                         ivr_proj_out *out, int32_t f64_mode,
                                         ivr_stream_t stream) {
    if (!g || !params || !layout || !out || g->n < 0 || width < 1 || height < 1) {
        ivr::set_error("ivr_preprocess_fwd_params: null argument");
        return IVR_ERR_ARG;
    }
    if (!out->depth_key || !out->count || !out->rect || !out->rec || !out->values || layout->k < 1 ||
        layout->n_attr < 0 || layout->n_attr > IVR_MAX_ATTRS ||
        (f64_mode && (!out->rec64 || !out->values64))) {
        ivr::set_error("ivr_preprocess_fwd_params: missing output buffer or bad layout");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    ivr_shading S{};
    ivr_edits E{};
    if (shading) S = *shading;
    if (edits) E = *edits;
    const int threads = 256;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    ivr_frame_params Pv{};
    Pv.cam.width = width;
    Pv.cam.height = height;
    ivr::preprocess_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        *g, S, shading != nullptr, E, edits != nullptr, Pv, params, *layout, *out, f64_mode);
    return ivr::check_launch("preprocess_kernel(params)");
}

extern "C" int ivr_shade_fwd(const ivr_gaussians *g, const ivr_shading *shading,
                             const int32_t *scene_id, const ivr_camera *cam, double *rgb,
                             double *terms, ivr_stream_t stream) {
    if (!g || !shading || !cam || !rgb || g->n < 0) {
        ivr::set_error("ivr_shade_fwd: null argument");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    const int threads = 256;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    ivr_frame_params P = ivr::params_from(*cam, shading, nullptr);
    ivr::shade_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(*g, *shading, scene_id, P, rgb,
                                                                   terms);
    return ivr::check_launch("shade_kernel");
}
