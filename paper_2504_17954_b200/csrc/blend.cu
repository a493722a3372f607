// K3 -- per-tile front-to-back alpha blend (forward).
//
// Replaces _kernels.composite_forward (_kernels.py:31-72).  One CTA per 16x16
// tile (tiles launched heaviest-first when a tile order is given), one thread
// per pixel.  The tile's depth-sorted pair list is streamed through shared
// memory in batches of 256 pairs; while a batch is staged each thread tests
// one pair against the whole tile in float64 (minimum of the Gaussian exponent
// over the tile rectangle) and culls pairs the reference's alpha test rejects
// at every pixel of the tile.  Survivors are compacted in list order (warp
// ballots), so each pixel walks exactly the reference list minus provably
// skipped pairs, and the CTA retires once every pixel has passed T < 1e-4.
//
// Decisions (sigma < 0, alpha < 1/255, T < 1e-4) must match the reference's
// float64 arithmetic exactly -- a flipped alpha-skip moves a pixel by
// ~T/255 >> 1e-4 (SURVEY.md finding 4).  Two modes:
//  * EXACT: every non-skipped pair is re-evaluated with the reference's
//    float64 arithmetic (separately rounded, exp, cap, skip, T *= 1-alpha,
//    float32 accumulation rounding) -> bit-faithful images.
//  * FAST: the exponent is evaluated in float32 together with a rigorous
//    per-evaluation error bound E.  Pairs certainly on one side of the
//    alpha-skip threshold use float32 alpha; only pairs inside the +-E band
//    take the exact float64 path.  T is tracked in float32 with a running
//    relative error bound; if T lands inside its band around 1e-4 the pixel
//    is replayed in EXACT mode.  Decisions therefore still match the
//    reference; only the accumulated values carry float32 rounding
//    (~1e-6, tolerance 1e-4).
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {

constexpr int kBlendThreads = 256;
constexpr int kModeExact = 0;
constexpr int kModeFast = 1;

// Can splat (record r0, r1) reach alpha >= 1/255 anywhere in the pixel
// rectangle [px0, px1] x [py0, py1]?  Conservative: true unless the float64
// minimum of the exponent over the rectangle exceeds hi (>= ln(255 o) + margins).
__device__ __forceinline__ bool tile_touch(const float4 r0, const float4 r1, int px0, int px1,
                                           int py0, int py1) {
    const double hi = r0.w;
    if (!(hi < 1e30)) return true;
    const double a = 2.0 * (double)r1.x, b = r1.y, c = 2.0 * (double)r1.z;
    if (!(a > 0.0 && c > 0.0 && a * c - b * b > 0.0)) return true;
    const double mx = r0.x, my = r0.y;
    const double ex0 = px0 - mx, ex1 = px1 - mx, ey0 = py0 - my, ey1 = py1 - my;
    if (ex0 <= 0.0 && ex1 >= 0.0 && ey0 <= 0.0 && ey1 >= 0.0) return true;
    const double ia = 1.0 / a, ic = 1.0 / c;
    double best = 1e300;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double e = k ? ex1 : ex0;
        double dy = -b * e * ic;
        dy = dy < ey0 ? ey0 : (dy > ey1 ? ey1 : dy);
        const double s = 0.5 * (a * e * e + c * dy * dy) + b * e * dy;
        best = s < best ? s : best;
        const double f = k ? ey1 : ey0;
        double dx = -b * f * ia;
        dx = dx < ex0 ? ex0 : (dx > ex1 ? ex1 : dx);
        const double t = 0.5 * (a * dx * dx + c * f * f) + b * dx * f;
        best = t < best ? t : best;
    }
    return !(best > hi);
}

// Reference alpha for one (pixel, splat) in float64 (_kernels.py:51-61);
// returns a negative value when the reference skips the pair.
__device__ __forceinline__ double exact_alpha(double dpx, double dpy, double mx, double my,
                                              double ca, double cb, double cc, double o) {
    const double ddx = dsub(dpx, mx), ddy = dsub(dpy, my);
    const double sg = dadd(dmul(0.5, dadd(dmul(dmul(ca, ddx), ddx), dmul(dmul(cc, ddy), ddy))),
                           dmul(dmul(cb, ddx), ddy));
    if (sg < 0.0) return -1.0;
    double al = dmul(o, exp(-sg));
    if (al > kAlphaCap) al = kAlphaCap;
    if (al < kAlphaSkip) return -1.0;
    return al;
}

// EXACT replay of one pixel over its whole tile list (global memory).  Used
// by FAST mode when T lands in its ambiguity band around T_STOP.
template <int KMAX, bool F64>
__device__ void replay_pixel(int s0, int s1, const int32_t *__restrict__ pair_splat,
                             const float4 *__restrict__ rec, const float *__restrict__ values,
                             const double *__restrict__ rec64, const double *__restrict__ values64,
                             int K, int px, int py, float *acc, double *acc64, double &T, int &nc,
                             int &last) {
    const double dpx = px, dpy = py;
    const float fpx = px, fpy = py;
    T = 1.0;
    nc = 0;
    last = s0;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) acc[c] = 0.0f;
#pragma unroll
    for (int c = 0; c < (F64 ? KMAX : 1); ++c) acc64[c] = 0.0;
    for (int j = s0; j < s1; ++j) {
        const int sp = pair_splat[j];
        if (sp < 0) continue;  // culled for the whole tile (never contributes)
        const float4 a0 = __ldg(rec + 2 * sp), a1 = __ldg(rec + 2 * sp + 1);
        const float dx = fpx - a0.x, dy = fpy - a0.y;
        const float sig = fmaf(fmaf(a1.x, dx, a1.y * dy), dx, (a1.z * dy) * dy);
        if (sig > a0.w) continue;
        double al;
        if (F64) {
            const double *r = rec64 + 8 * (int64_t)sp;
            al = exact_alpha(dpx, dpy, r[0], r[1], r[2], r[3], r[4], r[5]);
        } else {
            al = exact_alpha(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y, 2.0 * (double)a1.z, a0.z);
        }
        if (al < 0.0) continue;
        const double w = dmul(T, al);
        if (F64) {
            for (int c = 0; c < K; ++c) acc64[c] = dadd(acc64[c], dmul(w, values64[(int64_t)K * sp + c]));
        } else {
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) acc[c] = (float)dadd((double)acc[c], dmul(w, (double)__ldg(values + (int64_t)K * sp + c)));
        }
        T = dmul(T, dsub(1.0, al));
        ++nc;
        last = j + 1;
        if (T < kTStop) break;
    }
}

template <int KMAX, bool F64, int MODE>
__global__ void __launch_bounds__(kBlendThreads, 3)
blend_fwd_kernel(const int32_t *__restrict__ ranges, const int32_t *__restrict__ pair_splat,
                 int ntx, const float4 *__restrict__ rec, const float *__restrict__ values,
                 const double *__restrict__ rec64, const double *__restrict__ values64, int K,
                 int W, int H, float *__restrict__ out, double *__restrict__ out64,
                 int32_t *__restrict__ contrib, int32_t *__restrict__ last_pos,
                 double *__restrict__ t_final, const int32_t *__restrict__ tile_order,
                 int preculled) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool kStage64 = F64 && MODE == kModeExact;
    constexpr bool kStageMean64 = F64 && MODE == kModeFast;
    float4 *s_r0 = reinterpret_cast<float4 *>(smem);
    float4 *s_r1 = s_r0 + kBlendThreads;
    int *s_j = reinterpret_cast<int *>(s_r1 + kBlendThreads);
    int *s_sp = s_j + kBlendThreads;
    float *s_v = reinterpret_cast<float *>(s_sp + kBlendThreads);
    double *s_r64 = reinterpret_cast<double *>(s_v + kBlendThreads * KMAX);  // 6/pair
    double *s_v64 = s_r64 + (kStage64 ? 6 * kBlendThreads : (kStageMean64 ? 2 * kBlendThreads : 0));
    __shared__ int s_wsum[kBlendThreads / 32];

    const int tile = tile_order ? tile_order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % ntx, ty = tile / ntx;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int px = tx * kTile + (tid & 15), py = ty * kTile + (tid >> 4);
    const bool inside = px < W && py < H;
    const int s0 = ranges[tile], s1 = ranges[tile + 1];
    const int px0 = tx * kTile, py0 = ty * kTile;
    const int px1 = min(px0 + kTile - 1, W - 1), py1 = min(py0 + kTile - 1, H - 1);
    const float fpx = (float)px, fpy = (float)py;
    const double dpx = (double)px, dpy = (double)py;

    double T = 1.0;     // EXACT mode transmittance (float64, reference arithmetic)
    float Tf = 1.0f;    // FAST mode transmittance
    float errT = 0.0f;  // FAST: bound on |Tf - T_ref| / T_ref
    float acc[KMAX];
    double acc64[F64 ? KMAX : 1];
#pragma unroll
    for (int c = 0; c < KMAX; ++c) acc[c] = 0.0f;
#pragma unroll
    for (int c = 0; c < (F64 ? KMAX : 1); ++c) acc64[c] = 0.0;
    int nc = 0, last = s0;
    bool done = !inside, replay = false;

    for (int base = s0; base < s1; base += kBlendThreads) {
        if (__syncthreads_count(!done) == 0) break;
        // ---- stage + cull one batch (each thread one pair)
        const int j = base + tid;
        bool keep = false;
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
        int sp = 0;
        if (j < s1) {
            sp = pair_splat[j];
            if (preculled) {
                keep = sp >= 0;  // bit 31 = culled by ivr_bin_sort_cull
                if (keep) {
                    r0 = __ldg(rec + 2 * sp);
                    r1 = __ldg(rec + 2 * sp + 1);
                }
            } else {
                r0 = __ldg(rec + 2 * sp);
                r1 = __ldg(rec + 2 * sp + 1);
                keep = tile_touch(r0, r1, px0, px1, py0, py1);
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_wsum[warp] = __popc(m);
        __syncthreads();
        int off = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kBlendThreads / 32; ++w) {
            const int c = s_wsum[w];
            off += (w < warp) ? c : 0;
            total += c;
        }
        if (keep) {
            const int q = off + __popc(m & lanemask_lt());
            s_r0[q] = r0;
            s_r1[q] = r1;
            s_j[q] = j;
            s_sp[q] = sp;
            const float *v = values + (int64_t)K * sp;
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) s_v[q * KMAX + c] = __ldg(v + c);
            if (kStageMean64) {
                s_r64[2 * q] = __ldg(rec64 + 8 * (int64_t)sp);
                s_r64[2 * q + 1] = __ldg(rec64 + 8 * (int64_t)sp + 1);
            }
            if (kStage64) {
                const double *r = rec64 + 8 * (int64_t)sp;
#pragma unroll
                for (int c = 0; c < 6; ++c) s_r64[q * 6 + c] = __ldg(r + c);
                const double *v64 = values64 + (int64_t)K * sp;
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c < K) s_v64[q * KMAX + c] = __ldg(v64 + c);
            }
        }
        __syncthreads();
        if (done) continue;
        // ---- per-pixel walk over the survivors, in list order
        for (int q = 0; q < total; ++q) {
            const float4 a0 = s_r0[q];
            const float4 a1 = s_r1[q];
            const float dx = fpx - a0.x, dy = fpy - a0.y;
            const float bdy = a1.y * dy, hcdy = a1.z * dy;
            const float sig = fmaf(fmaf(a1.x, dx, bdy), dx, hcdy * dy);
            if (sig > a0.w) continue;  // reference alpha < 1/255 for certain
            if (MODE == kModeExact) {
                double al;
                if (kStage64) {
                    const double *r = s_r64 + q * 6;
                    al = exact_alpha(dpx, dpy, r[0], r[1], r[2], r[3], r[4], r[5]);
                } else {
                    al = exact_alpha(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                     2.0 * (double)a1.z, a0.z);
                }
                if (al < 0.0) continue;
                const double w = dmul(T, al);
                if (F64) {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c)
                        if (c < K) acc64[c] = dadd(acc64[c], dmul(w, s_v64[q * KMAX + c]));
                } else {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c)
                        if (c < K)
                            acc[c] = (float)dadd((double)acc[c], dmul(w, (double)s_v[q * KMAX + c]));
                }
                T = dmul(T, dsub(1.0, al));
                ++nc;
                last = s_j[q] + 1;
                if (T < kTStop) {
                    done = true;
                    break;
                }
            } else {
                // candidate: recompute with the float64 mean in dtype=float64 mode
                float cdx = dx, cdy = dy, cbdy = bdy, chcdy = hcdy, csig = sig;
                if (kStageMean64) {
                    cdx = (float)dsub(dpx, s_r64[2 * q]);
                    cdy = (float)dsub(dpy, s_r64[2 * q + 1]);
                    cbdy = a1.y * cdy;
                    chcdy = a1.z * cdy;
                    csig = fmaf(fmaf(a1.x, cdx, cbdy), cdx, chcdy * cdy);
                }
                // rigorous bound on |csig - sigma_ref|: ~17 ulp of the term
                // magnitudes (dx/dy rounding, 5 ops, float32 conic rounding)
                const float terms = fmaf(a1.x * cdx, cdx, fmaf(chcdy, cdy, fabsf(cbdy * cdx)));
                const float E = 1.0e-6f * terms + 1e-30f;
                const float sig_c = csig;
                const float thr = a1.w;
                const float tm = 2.4e-7f * fabsf(thr) + 1e-7f;  // thr rounding + exp/1/255 margin
                float al;
                float dal;  // relative error bound of al
                if (sig_c - E > 0.0f && sig_c + E < thr - tm) {
                    al = a0.z * exp2f(-1.4426950408889634f * sig_c);
                    al = fminf(al, 0.99f);
                    dal = E + 6e-7f * (1.0f + sig_c);
                } else if (sig_c - E > thr + tm) {
                    continue;  // certainly skipped by the reference
                } else {
                    double ad;
                    if (F64) {
                        const double *r = rec64 + 8 * (int64_t)s_sp[q];
                        ad = exact_alpha(dpx, dpy, r[0], r[1], r[2], r[3], r[4], r[5]);
                    } else {
                        ad = exact_alpha(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                         2.0 * (double)a1.z, a0.z);
                    }
                    if (ad < 0.0) continue;
                    al = (float)ad;
                    dal = 1.2e-7f;
                }
                const float w = Tf * al;
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c < K) acc[c] = fmaf(w, s_v[q * KMAX + c], acc[c]);
                Tf = Tf * (1.0f - al);
                errT += al * dal * __frcp_rn(1.0f - al) * 1.01f + 1.2e-7f;
                ++nc;
                last = s_j[q] + 1;
                if (Tf < 1e-4f * (1.0f + errT + 1e-6f)) {
                    if (Tf < 1e-4f * (1.0f - errT - 1e-6f)) {
                        done = true;  // reference also stopped here
                    } else {
                        done = true;  // ambiguous: replay this pixel exactly
                        replay = true;
                    }
                    break;
                }
            }
        }
    }
    if (!inside) return;
    if (MODE == kModeFast) {
        if (replay) {
            replay_pixel<KMAX, F64>(s0, s1, pair_splat, rec, values, rec64, values64, K, px, py,
                                    acc, acc64, T, nc, last);
            if (F64) {
#pragma unroll
                for (int c = 0; c < KMAX; ++c) acc[c] = (float)acc64[c];
            }
        } else {
            T = (double)Tf;
        }
    }
    const int64_t pix = (int64_t)py * W + px;
    if (F64) {
        double *o = out64 + pix * K;
        if (MODE == kModeExact) {
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) o[c] = acc64[c];
        } else {
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) o[c] = replay ? acc64[c] : (double)acc[c];
        }
    } else {
        float *o = out + pix * K;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < K) o[c] = acc[c];
    }
    if (contrib) contrib[pix] = nc;
    if (last_pos) last_pos[pix] = last;
    if (t_final) t_final[pix] = T;
}

template <int KMAX, bool F64, int MODE>
size_t blend_smem_bytes() {
    return (size_t)kBlendThreads * (16 + 16 + 4 + 4 + 4 * KMAX) +
           ((F64 && MODE == kModeExact) ? (size_t)kBlendThreads * 8 * (6 + KMAX) : 0) +
           ((F64 && MODE == kModeFast) ? (size_t)kBlendThreads * 16 : 0);
}

template <int KMAX, bool F64, int MODE>
int launch_blend(const int32_t *ranges, const int32_t *pair_splat, int ntx, int nty,
                 const float *rec, const float *values, const double *rec64,
                 const double *values64, int K, int W, int H, float *out, double *out64,
                 int32_t *contrib, int32_t *last_pos, double *t_final, const int32_t *tile_order,
                 int preculled, cudaStream_t st) {
    const size_t sm = blend_smem_bytes<KMAX, F64, MODE>();
    auto fn = blend_fwd_kernel<KMAX, F64, MODE>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fn<<<ntx * nty, kBlendThreads, sm, st>>>(ranges, pair_splat, ntx,
                                            reinterpret_cast<const float4 *>(rec), values, rec64,
                                            values64, K, W, H, out, out64, contrib, last_pos,
                                            t_final, tile_order, preculled);
    return check_launch("blend_fwd_kernel");
}

// ----------------------------------------------------------------- tile order
// Heaviest tiles first: a tile's CTA runtime grows with its pair count, and the
// longest tiles otherwise start in the last wave and set the frame's tail.
// Single CTA bitonic sort of (count desc, tile asc) for up to 4096 tiles.
__global__ void __launch_bounds__(1024)
tile_order_kernel(const int32_t *ranges, int ntiles, int32_t *order) {
    __shared__ unsigned long long key[4096];
    const int n2 = 4096;
    for (int i = threadIdx.x; i < n2; i += 1024) {
        unsigned long long k = ~0ull;
        if (i < ntiles) {
            const uint32_t cnt = (uint32_t)(ranges[i + 1] - ranges[i]);
            k = ((unsigned long long)(0xffffffffu - cnt) << 32) | (uint32_t)i;
        }
        key[i] = k;
    }
    __syncthreads();
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < n2 / 2; i += 1024) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const unsigned long long a = key[lo], b = key[hi];
                if ((a > b) == up) {
                    key[lo] = b;
                    key[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < ntiles; i += 1024) order[i] = (int32_t)(key[i] & 0xffffffffu);
}

}  // namespace ivr

extern "C" int ivr_tile_order(const int32_t *tile_ranges, int32_t ntiles, int32_t *order,
                              ivr_stream_t stream) {
    using namespace ivr;
    if (!tile_ranges || !order || ntiles < 1) {
        set_error("ivr_tile_order: bad argument");
        return IVR_ERR_ARG;
    }
    if (ntiles > 4096) {  // identity order for very large frames
        set_error("ivr_tile_order: more than 4096 tiles");
        return IVR_ERR_ARG;
    }
    tile_order_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(tile_ranges, ntiles, order);
    return check_launch("tile_order_kernel");
}

extern "C" int ivr_blend_fwd(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                             int32_t nty, const float *rec, const float *values,
                             const double *rec64, const double *values64, int32_t k,
                             int32_t width, int32_t height, float *out, double *out64,
                             int32_t *contrib, int32_t *last_pos, double *t_final,
                             const int32_t *tile_order, int32_t flags, ivr_stream_t stream) {
    using namespace ivr;
    cudaStream_t st = (cudaStream_t)stream;
    if (!tile_ranges || !pair_splat || !rec || !values || k < 1 || k > 32 || width < 1 ||
        height < 1 || ntx != (width + kTile - 1) / kTile || nty != (height + kTile - 1) / kTile) {
        set_error("ivr_blend_fwd: bad argument");
        return IVR_ERR_ARG;
    }
    const bool f64 = out64 != nullptr;
    if (f64 ? (!rec64 || !values64) : (out == nullptr)) {
        set_error("ivr_blend_fwd: float64 mode needs rec64/values64/out64; float32 needs out");
        return IVR_ERR_ARG;
    }
    const bool exact = (flags & IVR_BLEND_EXACT) != 0;
    const int preculled = (flags & IVR_BLEND_PRECULLED) != 0 ? 1 : 0;
#define IVR_BLEND_M(KM, F, M)                                                                    \
    return launch_blend<KM, F, M>(tile_ranges, pair_splat, ntx, nty, rec, values, rec64, values64, \
                                  k, width, height, out, out64, contrib, last_pos, t_final,       \
                                  tile_order, preculled, st)
#define IVR_BLEND(KM)                                                                             \
    if (f64) {                                                                                    \
        if (exact) { IVR_BLEND_M(KM, true, kModeExact); }                                         \
        IVR_BLEND_M(KM, true, kModeFast);                                                         \
    }                                                                                             \
    if (exact) { IVR_BLEND_M(KM, false, kModeExact); }                                            \
    IVR_BLEND_M(KM, false, kModeFast)
    if (k <= 4) { IVR_BLEND(4); }
    if (k <= 8) { IVR_BLEND(8); }
    if (k <= 16) { IVR_BLEND(16); }
    IVR_BLEND(32);
#undef IVR_BLEND
#undef IVR_BLEND_M
}
