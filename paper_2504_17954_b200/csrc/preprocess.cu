// K1 -- fused per-Gaussian preprocess (float64, one thread per Gaussian).
//
// Replaces, bit-faithfully up to transcendental ulps:
//   scene.apply_edits            scene.py:199-228   (opacity logit round trip)
//   shading.shade_gaussians      shading.py:225-329 (Blinn-Phong, coeff transform)
//   gaussians.project_gaussians  gaussians.py:296-346 (EWA, dgemm FMA chains)
//   rasterizer.rasterize_forward rasterizer.py:88-121 (radius/rect/count),
//                                rasterizer.py:134-153 (f32 packing)
// and emits the float32 blend record plus the conservative exponent bound
// `hi` (sigma32 > hi implies the reference's float64 alpha < 1/255) and the
// alpha-skip exponent thr = ln(255 o) used by K3.
#include <math.h>

#include "project.cuh"

namespace ivr {

constexpr int kK1Threads = 64;

__device__ __forceinline__ void preprocess_one(const ivr_gaussians &G, const ivr_shading &S,
                                               int has_shading, const ivr_edits &E, int has_edits,
                                               const ivr_frame_params &P, const ivr_layout &L,
                                               const ivr_proj_out &O, int mode, int64_t i) {
    // mode bit 0 (IVR_PRE_F64): dtype=float64 semantics; bit 1
    // (IVR_PRE_EXACT_RGB): the float64 shading chain even with a static cache
    const bool f64_mode = (mode & IVR_PRE_F64) != 0;
    const ivr_camera &cam = P.cam;
    const int32_t sid = (has_edits && E.scene_id) ? E.scene_id[i] : 0;
    const bool rescale = has_edits && P.rescale_opacity && E.opacity_scale;
    const double sig_o = G.cache ? G.cache[kCacheStride * i + 9] : sigmoid_ref(G.o_logit[i]);
    const double opacity = effective_opacity_s(sig_o, rescale, rescale ? E.opacity_scale[sid] : 1.0);

    Proj p;
    project_one(G, i, cam, p);
    const double tz = p.t[2];
    const double mx = p.mx, my = p.my;
    const double ca = p.C2[0], cb = p.C2[1], cc = p.C2[3];

    // ---- radius / visibility / tile rect (rasterizer.py:88-118)
    const double half_tr = dmul(0.5, dadd(ca, cc));
    const double dac = dsub(ca, cc);
    const double disc = dadd(dmul(0.25, dmul(dac, dac)), dmul(cb, cb));
    const double lam_max = dadd(half_tr, sqrt(dmax(disc, 0.0)));
    const double cut = sqrt(dmul(2.0, log(dmax(ddiv(opacity, kAlphaSkip), 1.0))));
    const double radius = dadd(ceil(dmul(sqrt(dmax(lam_max, 0.0)), cut)), 1.0);
    const int ntx = (cam.width + kTile - 1) / kTile, nty = (cam.height + kTile - 1) / kTile;
    bool visible = p.valid && (opacity >= kAlphaSkip) && (radius > 0.0);
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

    double nrm[3];
    unit_normal(G, i, nrm);
    ShadeState sh;
    float rgb32[3] = {0.0f, 0.0f, 0.0f};
    // FAST mode with a shading cache and no float64 colour output: float32 colour
    const bool fast_rgb = has_shading && !f64_mode && !(mode & IVR_PRE_EXACT_RGB) && !O.rgb && G.cache &&
                          G.cache[kCacheStride * i + 14] != 0.0;
    if (has_shading) {
        const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
        if (fast_rgb)
            shade_rgb_f32(S, P, i, sid, mu, nrm, G.cache + kCacheStride * i, rgb32);
        else
            shade_state(S, P, i, sid, mu, nrm, sh, G.cache);
    }

    // ---- float32 blend record (rasterizer.py:151-153 casts) + skip bounds
    const float mx32 = (float)mx, my32 = (float)my;
    const float a32 = (float)p.conic[0], b32 = (float)p.conic[1], c32 = (float)p.conic[2];
    const float o32 = (float)opacity;
    float hi32 = __int_as_float(0x7f800000);  // +inf: always take the exact path
    float thr32 = 0.0f;                         // ln(o / (1/255))
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
        r[0] = mx; r[1] = my; r[2] = p.conic[0]; r[3] = p.conic[1]; r[4] = p.conic[2];
        r[5] = opacity; r[6] = tz; r[7] = 0.0;
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
            put(L.col_color + k, fast_rgb ? (double)rgb32[k]
                                 : has_shading ? sh.rgb[k] : (L.colors ? L.colors[3 * i + k] : 0.0));
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
    if (O.conic) for (int k = 0; k < 3; ++k) O.conic[3 * i + k] = p.conic[k];
    if (O.cov2d) for (int k = 0; k < 4; ++k) O.cov2d[4 * i + k] = p.C2[k];
    if (O.depth) O.depth[i] = tz;
    if (O.opacity) O.opacity[i] = opacity;
    if (O.radius) O.radius[i] = radius;
    if (O.valid) O.valid[i] = p.valid ? 1 : 0;
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

__global__ void __launch_bounds__(kK1Threads)
preprocess_kernel(ivr_gaussians G, ivr_shading S, int has_shading, ivr_edits E, int has_edits,
                  ivr_frame_params Pv, const ivr_frame_params *__restrict__ Pd, ivr_layout L,
                  ivr_proj_out O, int f64_mode) {
    pdl_begin();
    __shared__ ivr_frame_params sp;
    stage_params(Pd ? Pd : &Pv, sp);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < G.n) preprocess_one(G, S, has_shading, E, has_edits, sp, L, O, f64_mode, i);
    if (!O.depth_minmax) return;
    // [min, max] of the visible depth keys for K2's coarse keys: warp and
    // block reduction, one atomic pair per block
    const unsigned long long key = i < G.n ? O.depth_key[i] : ~0ull;
    unsigned long long lo = key, hi = key == ~0ull ? 0ull : key;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    constexpr int kW = kK1Threads / 32;
    __shared__ unsigned long long s_lo[kW], s_hi[kW];
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kW; ++w) {
            lo = s_lo[w] < lo ? s_lo[w] : lo;
            hi = s_hi[w] > hi ? s_hi[w] : hi;
        }
        if (lo != ~0ull) {
            atomicMin(O.depth_minmax, lo);
            atomicMax(O.depth_minmax + 1, hi);
        }
    }
}

__global__ void __launch_bounds__(256)
shade_kernel(ivr_gaussians G, ivr_shading S, const int32_t *scene_id, ivr_frame_params Pv,
             double *rgb, double *terms) {
    __shared__ ivr_frame_params sp;
    stage_params(&Pv, sp);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.n) return;
    const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
    double nrm[3];
    unit_normal(G, i, nrm);
    ShadeState sh;
    shade_state(S, sp, i, scene_id ? scene_id[i] : 0, mu, nrm, sh);
    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = sh.rgb[k];
    if (terms) {
        for (int k = 0; k < 3; ++k) {
            terms[9 * i + k] = sh.amb[k];
            terms[9 * i + 3 + k] = sh.dif[k];
            terms[9 * i + 6 + k] = sh.spec;
        }
    }
}

// Camera- and edit-independent per-Gaussian values for repeated frames of a
// resident scene (same functions as the per-frame path: bit-identical).
__global__ void __launch_bounds__(256)
static_kernel(ivr_gaussians G, ivr_shading S, int has_shading, double *cache) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.n) return;
    ivr_gaussians Gn = G;
    Gn.cache = nullptr;
    Proj p;
    cov3d_one(Gn, i, p);
    double nrm[3];
    unit_normal(Gn, i, nrm);
    double *c = cache + kCacheStride * i;
    c[0] = p.C3[0]; c[1] = p.C3[1]; c[2] = p.C3[2];
    c[3] = p.C3[4]; c[4] = p.C3[5]; c[5] = p.C3[8];
    for (int k = 0; k < 3; ++k) c[6 + k] = nrm[k];
    c[9] = sigmoid_ref(G.o_logit[i]);
    if (has_shading) {
        c[10] = sigmoid_ref(S.k_a_raw[i]);
        c[11] = sigmoid_ref(S.k_d_raw[i]);
        c[12] = sigmoid_ref(S.k_s_raw[i]);
        c[13] = dadd(exp(S.log_beta[i]), 1.0);
        c[14] = 1.0;
    } else {
        c[10] = c[11] = c[12] = c[13] = c[14] = 0.0;
    }
    c[15] = 0.0;
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
    } else {
        for (int k = 0; k < 4; ++k) {
            P.term_scales[k] = 1.0;
            P.lam[k] = 1.0;
        }
    }
    P.rescale_opacity = E ? E->rescale_opacity : 0;
    return P;
}

}  // namespace ivr

extern "C" int ivr_preprocess_static(const ivr_gaussians *g, const ivr_shading *shading,
                                     double *cache, ivr_stream_t stream) {
    using namespace ivr;
    if (!g || !cache || g->n < 0 || (g->n > 0 && (!g->q_raw || !g->log_s || !g->o_logit || !g->n_raw))) {
        set_error("ivr_preprocess_static: bad argument");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    ivr_shading S{};
    if (shading) S = *shading;
    const int threads = 256;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    static_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(*g, S, shading ? 1 : 0, cache);
    return check_launch("static_kernel");
}

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
    if ((f64_mode & IVR_PRE_F64) && (!out->rec64 || !out->values64)) {
        ivr::set_error("ivr_preprocess_fwd: float64 mode needs rec64 and values64");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    ivr_shading S{};
    ivr_edits E{};
    if (shading) S = *shading;
    if (edits) E = *edits;
    const int threads = ivr::kK1Threads;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    ivr_frame_params P = ivr::params_from(*cam, shading, edits);
    ivr::launch<3>(ivr::preprocess_kernel, blocks, threads, 0, (cudaStream_t)stream, *g, S,
                (int)(shading != nullptr), E, (int)(edits != nullptr), P,
                (const ivr_frame_params *)nullptr, *layout, *out, (int)f64_mode);
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
        ((f64_mode & IVR_PRE_F64) && (!out->rec64 || !out->values64))) {
        ivr::set_error("ivr_preprocess_fwd_params: missing output buffer or bad layout");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    ivr_shading S{};
    ivr_edits E{};
    if (shading) S = *shading;
    if (edits) E = *edits;
    const int threads = ivr::kK1Threads;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    ivr_frame_params Pv{};
    Pv.cam.width = width;
    Pv.cam.height = height;
    ivr::launch<3>(ivr::preprocess_kernel, blocks, threads, 0, (cudaStream_t)stream, *g, S,
                (int)(shading != nullptr), E, (int)(edits != nullptr), Pv, params, *layout, *out,
                (int)f64_mode);
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
