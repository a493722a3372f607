// Exact per-Gaussian projection and shading forward, shared by K1 (forward
// preprocess) and K4 (backward recompute) so both see bit-identical values.
//
// Reference: gaussians.project_gaussians (gaussians.py:296-346) and
// shading.shade_gaussians (shading.py:225-329); OpenBLAS dgemm k-chains are
// reproduced with chain3 (see ivr_common.cuh).
#pragma once

#include "ivr_common.cuh"

namespace ivr {

struct Proj {
    double t[3], tzs;
    bool valid;
    double mx, my;
    double q[4];   // unit quaternion
    double s[3];   // scales
    double R[9];
    double C3[9];  // cov3d
    double J[6];
    double M[6];   // J @ W
    double C2[4];  // cov2d (+ dilation)
    double conic[3];
};

__device__ __forceinline__ void quat_rot(const double q[4], double R[9]) {
    const double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    R[0] = dsub(1.0, dmul(2.0, dadd(dmul(qy, qy), dmul(qz, qz))));
    R[1] = dmul(2.0, dsub(dmul(qx, qy), dmul(qw, qz)));
    R[2] = dmul(2.0, dadd(dmul(qx, qz), dmul(qw, qy)));
    R[3] = dmul(2.0, dadd(dmul(qx, qy), dmul(qw, qz)));
    R[4] = dsub(1.0, dmul(2.0, dadd(dmul(qx, qx), dmul(qz, qz))));
    R[5] = dmul(2.0, dsub(dmul(qy, qz), dmul(qw, qx)));
    R[6] = dmul(2.0, dsub(dmul(qx, qz), dmul(qw, qy)));
    R[7] = dmul(2.0, dadd(dmul(qy, qz), dmul(qw, qx)));
    R[8] = dsub(1.0, dmul(2.0, dadd(dmul(qx, qx), dmul(qy, qy))));
}

// Camera-independent part of the projection (gaussians.py:222-275, 305-310):
// unit quaternion, scales, rotation and cov3d = (R S)(R S)^T.
__device__ __forceinline__ void cov3d_one(const ivr_gaussians &G, int64_t i, Proj &p) {
    const double qr[4] = {G.q_raw[4 * i], G.q_raw[4 * i + 1], G.q_raw[4 * i + 2],
                          G.q_raw[4 * i + 3]};
    const double qn = norm4(qr[0], qr[1], qr[2], qr[3]);
    for (int k = 0; k < 4; ++k) p.q[k] = ddiv(qr[k], qn);
    for (int k = 0; k < 3; ++k) p.s[k] = exp(G.log_s[3 * i + k]);
    quat_rot(p.q, p.R);
    double M3[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) M3[3 * r + c] = dmul(p.R[3 * r + c], p.s[c]);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            p.C3[3 * r + c] = chain3(M3[3 * r], M3[3 * c], M3[3 * r + 1], M3[3 * c + 1],
                                     M3[3 * r + 2], M3[3 * c + 2]);
}

// Per-Gaussian static cache (ivr_preprocess_static): cov3d (xx xy xz yy yz
// zz), unit normal, sigmoid(o_logit), sigmoid(k_a/k_d/k_s raw),
// exp(log_beta)+1, has-shading flag, pad.
constexpr int kCacheStride = 16;

// gaussians.py:302-339, operation by operation.  With G.cache the
// camera-independent cov3d comes from the cache (bit-identical values; q, s,
// R are then not filled -- the geometry backward never uses a cache).
__device__ __forceinline__ void project_one(const ivr_gaussians &G, int64_t i,
                                            const ivr_camera &cam, Proj &p) {
    const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
    if (G.cache) {
        const double *c = G.cache + kCacheStride * i;
        p.C3[0] = c[0]; p.C3[1] = c[1]; p.C3[2] = c[2];
        p.C3[3] = c[1]; p.C3[4] = c[3]; p.C3[5] = c[4];
        p.C3[6] = c[2]; p.C3[7] = c[4]; p.C3[8] = c[5];
    } else {
        cov3d_one(G, i, p);
    }
    const double *W = cam.rotation;
    const double d[3] = {dsub(mu[0], cam.position[0]), dsub(mu[1], cam.position[1]),
                         dsub(mu[2], cam.position[2])};
    for (int j = 0; j < 3; ++j) p.t[j] = chain3(d[0], W[3 * j], d[1], W[3 * j + 1], d[2], W[3 * j + 2]);
    const double tz = p.t[2];
    p.valid = tz > kNearPlane;
    p.tzs = p.valid ? tz : 1.0;
    const double f = cam.focal;
    p.mx = dadd(ddiv(dmul(f, p.t[0]), p.tzs), cam.cx);
    p.my = dadd(ddiv(dmul(f, p.t[1]), p.tzs), cam.cy);
    const double tzs = p.tzs;
    p.J[0] = ddiv(f, tzs);
    p.J[1] = 0.0;
    p.J[2] = ddiv(dmul(-f, p.t[0]), dmul(tzs, tzs));
    p.J[3] = 0.0;
    p.J[4] = ddiv(f, tzs);
    p.J[5] = ddiv(dmul(-f, p.t[1]), dmul(tzs, tzs));
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            p.M[3 * r + c] = chain3(p.J[3 * r], W[c], p.J[3 * r + 1], W[3 + c], p.J[3 * r + 2], W[6 + c]);
    double A[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
            A[3 * r + c] = chain3(p.M[3 * r], p.C3[c], p.M[3 * r + 1], p.C3[3 + c], p.M[3 * r + 2],
                                  p.C3[6 + c]);
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c)
            p.C2[2 * r + c] = chain3(A[3 * r], p.M[3 * c], A[3 * r + 1], p.M[3 * c + 1], A[3 * r + 2],
                                     p.M[3 * c + 2]);
    p.C2[0] = dadd(p.C2[0], kCov2dDilation);
    p.C2[3] = dadd(p.C2[3], kCov2dDilation);
    const double ca = p.C2[0], cb = p.C2[1], cc = p.C2[3];
    const double det = dsub(dmul(ca, cc), dmul(cb, cb));
    const double dets = det > 0.0 ? det : 1.0;
    p.conic[0] = ddiv(cc, dets);
    p.conic[1] = ddiv(-cb, dets);
    p.conic[2] = ddiv(ca, dets);
    p.valid = p.valid && (det > 0.0);
}

// GaussianGeometry.normals (eps 1e-12)
__device__ __forceinline__ void unit_normal(const ivr_gaussians &G, int64_t i, double nrm[3]) {
    if (G.cache) {
        const double *c = G.cache + kCacheStride * i;
        for (int k = 0; k < 3; ++k) nrm[k] = c[6 + k];
        return;
    }
    const double nr[3] = {G.n_raw[3 * i], G.n_raw[3 * i + 1], G.n_raw[3 * i + 2]};
    const double nn = dmax(norm3(nr[0], nr[1], nr[2]), 1e-12);
    for (int k = 0; k < 3; ++k) nrm[k] = ddiv(nr[k], nn);
}

// Effective opacity after the per-scene opacity edit (scene.py:214-220);
// sig_o = sigmoid(o_logit) (computed here or taken from the static cache).
__device__ __forceinline__ double effective_opacity_s(double sig_o, bool rescale, double scale) {
    if (rescale) {
        double p = dmul(scale, sig_o);
        p = p < 1e-12 ? 1e-12 : (p > 1.0 - 1e-9 ? 1.0 - 1e-9 : p);
        return sigmoid_ref(log(ddiv(p, dsub(1.0, p))));
    }
    return sig_o;
}
__device__ __forceinline__ double effective_opacity(double o_logit, bool rescale, double scale) {
    return effective_opacity_s(sigmoid_ref(o_logit), rescale, scale);
}

// Shading forward state (shading.py:236-297) kept for the backward.
struct ShadeState {
    double rgb[3], amb[3], dif[3], spec;
    double v[3], l[3], h[3], u[3], w_cam[3];
    double sig[3], beta1;
    double k[4];      // k_a, k_d, k_s, beta (after transform, clamps, term scales)
    bool gates[4];
    double c_v[3];
    bool open[3];
    double ndl, ndh, a_ndl, a_ndh, spow;
    bool gate;
};

// EXACT (K1, shade_kernel): the reference's operations; EXACT = false (K4b's
// gradient-only recomputation): the two unit vectors use one reciprocal each
// instead of three IEEE divisions (<= 1 ulp; gradient tolerance 1e-3)
template <bool EXACT = true>
__device__ __forceinline__ void shade_state(const ivr_shading &S, const ivr_frame_params &P,
                                            int64_t i, int32_t sid, const double mu[3],
                                            const double nrm[3], ShadeState &o,
                                            const double *cache = nullptr) {
    const ivr_camera &cam = P.cam;
    for (int k = 0; k < 3; ++k) o.w_cam[k] = dsub(cam.position[k], mu[k]);
    const double wn = dmax(norm3(o.w_cam[0], o.w_cam[1], o.w_cam[2]), 1e-12);
    if (EXACT) {
        for (int k = 0; k < 3; ++k) o.v[k] = ddiv(o.w_cam[k], wn);
    } else {
        const double iw = 1.0 / wn;
        for (int k = 0; k < 3; ++k) o.v[k] = o.w_cam[k] * iw;
    }
    if (!P.orbital) {
        for (int k = 0; k < 3; ++k) {
            o.l[k] = o.h[k] = o.v[k];
            o.u[k] = 0.0;
        }
    } else {
        for (int k = 0; k < 3; ++k) {
            o.l[k] = P.light_dir[k];
            o.u[k] = dadd(o.v[k], o.l[k]);
        }
        const double un = dmax(norm3(o.u[0], o.u[1], o.u[2]), 1e-12);
        if (EXACT) {
            for (int k = 0; k < 3; ++k) o.h[k] = ddiv(o.u[k], un);
        } else {
            const double iu = 1.0 / un;
            for (int k = 0; k < 3; ++k) o.h[k] = o.u[k] * iu;
        }
    }
    if (cache && cache[kCacheStride * i + 14] != 0.0) {
        const double *c = cache + kCacheStride * i;
        o.sig[0] = c[10];
        o.sig[1] = c[11];
        o.sig[2] = c[12];
        o.beta1 = c[13];
    } else {
        o.sig[0] = sigmoid_ref(S.k_a_raw[i]);
        o.sig[1] = sigmoid_ref(S.k_d_raw[i]);
        o.sig[2] = sigmoid_ref(S.k_s_raw[i]);
        o.beta1 = dadd(exp(S.log_beta[i]), 1.0);
    }
    double t[4];
    for (int k = 0; k < 3; ++k) t[k] = dadd(dmul(P.lam[k], o.sig[k]), P.b[k]);
    t[3] = dadd(dmul(P.lam[3], o.beta1), P.b[3]);
    for (int k = 0; k < 3; ++k) {
        o.gates[k] = (t[k] > 0.0) && (t[k] < 1.0);
        o.k[k] = dmul(P.term_scales[k], clip01(t[k]));
    }
    o.gates[3] = t[3] > 1.0;
    o.k[3] = dmul(P.term_scales[3], dmax(t[3], 1.0));
    const double *cp = S.per_splat_palette ? S.palette + 3 * i : S.palette + 3 * (int64_t)sid;
    for (int k = 0; k < 3; ++k) {
        const double pre = dadd(cp[k], S.delta_c[3 * i + k]);
        o.open[k] = (pre > 0.0) && (pre < 1.0);
        o.c_v[k] = clip01(pre);
    }
    o.ndl = dot3(nrm, o.l);
    o.ndh = dot3(nrm, o.h);
    o.a_ndl = fabs(o.ndl);
    o.a_ndh = fabs(o.ndh);
    o.gate = o.a_ndl > 0.0;
    double spow = 0.0;
    if (o.a_ndh > 0.0) spow = pow(dmax(o.a_ndh, 1e-300), o.k[3]);
    if (!o.gate) spow = 0.0;
    o.spow = spow;
    const double kdl = dmul(o.k[1], o.a_ndl);
    o.spec = dmul(dmul(o.k[2], spow), 1.0);
    for (int k = 0; k < 3; ++k) {
        o.amb[k] = dmul(o.k[0], o.c_v[k]);
        o.dif[k] = dmul(kdl, o.c_v[k]);
        o.rgb[k] = dadd(dadd(o.amb[k], o.dif[k]), o.spec);
    }
}

// FAST-mode colour (K1 packs colours as float32 and the image contract is
// 1e-4): the same Blinn-Phong as shade_state in float32 arithmetic, from the
// static cache's sigmoids.  Keys, rects and the blend record stay float64.
__device__ __forceinline__ void shade_rgb_f32(const ivr_shading &S, const ivr_frame_params &P,
                                              int64_t i, int32_t sid, const double mu[3],
                                              const double nrm[3], const double *c, float rgb[3]) {
    const ivr_camera &cam = P.cam;
    float v[3], l[3], h[3], n[3];
    for (int k = 0; k < 3; ++k) {
        v[k] = (float)(cam.position[k] - mu[k]);
        n[k] = (float)nrm[k];
    }
    const float vn = rsqrtf(fmaxf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2], 1e-24f));
    for (int k = 0; k < 3; ++k) v[k] *= vn;
    if (!P.orbital) {
        for (int k = 0; k < 3; ++k) l[k] = h[k] = v[k];
    } else {
        for (int k = 0; k < 3; ++k) {
            l[k] = (float)P.light_dir[k];
            h[k] = v[k] + l[k];
        }
        const float hn = rsqrtf(fmaxf(h[0] * h[0] + h[1] * h[1] + h[2] * h[2], 1e-24f));
        for (int k = 0; k < 3; ++k) h[k] *= hn;
    }
    float kk[4];
    for (int k = 0; k < 3; ++k) {
        const float t = (float)P.lam[k] * (float)c[10 + k] + (float)P.b[k];
        kk[k] = (float)P.term_scales[k] * fminf(fmaxf(t, 0.0f), 1.0f);
    }
    kk[3] = (float)P.term_scales[3] * fmaxf((float)P.lam[3] * (float)c[13] + (float)P.b[3], 1.0f);
    const float a_ndl = fabsf(n[0] * l[0] + n[1] * l[1] + n[2] * l[2]);
    const float a_ndh = fabsf(n[0] * h[0] + n[1] * h[1] + n[2] * h[2]);
    const float spow = (a_ndl > 0.0f && a_ndh > 0.0f) ? powf(a_ndh, kk[3]) : 0.0f;
    const float spec = kk[2] * spow, kdl = kk[1] * a_ndl;
    const double *cp = S.per_splat_palette ? S.palette + 3 * i : S.palette + 3 * (int64_t)sid;
    for (int k = 0; k < 3; ++k) {
        const float cv = fminf(fmaxf((float)(cp[k] + S.delta_c[3 * i + k]), 0.0f), 1.0f);
        rgb[k] = kk[0] * cv + kdl * cv + spec;
    }
}

}  // namespace ivr
