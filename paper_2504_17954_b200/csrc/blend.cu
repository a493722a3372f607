// K3 -- per-tile front-to-back alpha blend (forward).
//
// Replaces _kernels.composite_forward (_kernels.py:31-72).  One CTA per 16x16
// tile, one thread per pixel.  The tile's depth-sorted pair list is streamed
// through shared memory in batches of 256 pairs; while a batch is staged every
// thread tests one pair against the whole tile in float64 (minimum of the
// Gaussian exponent over the tile rectangle) and culls pairs that the
// reference's alpha test rejects at every pixel of the tile.  Survivors are
// compacted in list order (warp ballots), so the per-pixel walk sees exactly
// the reference's list minus provably-skipped pairs.
//
// Per (pixel, pair) the exponent is first evaluated in float32; when it
// exceeds the per-splat bound `hi` (computed in K1 so that sigma32 > hi
// implies the reference's float64 alpha < 1/255) the pair is skipped.  Every
// other pair is re-evaluated with the reference's float64 arithmetic
// (separately rounded, no FMA, exp, 0.99 cap, 1/255 skip, T *= 1-alpha,
// float32 accumulation rounding in float32 mode), so contributor counts,
// last_pos and the image match the reference.
// The CTA retires as soon as every pixel has passed T < 1e-4.
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {

constexpr int kBlendThreads = 256;

// Can splat (record r0, r1) reach alpha >= 1/255 anywhere in the pixel
// rectangle [px0, px1] x [py0, py1]?  Conservative: returns true unless the
// float64 minimum of the exponent over the rectangle exceeds the per-splat
// bound hi (>= ln(255 o) + margins).
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

template <int KMAX, bool F64>
__global__ void __launch_bounds__(kBlendThreads)
blend_fwd_kernel(const int32_t *__restrict__ ranges, const int32_t *__restrict__ pair_splat,
                 int ntx, const float4 *__restrict__ rec, const float *__restrict__ values,
                 const double *__restrict__ rec64, const double *__restrict__ values64, int K,
                 int W, int H, float *__restrict__ out, double *__restrict__ out64,
                 int32_t *__restrict__ contrib, int32_t *__restrict__ last_pos,
                 double *__restrict__ t_final, const int32_t *__restrict__ tile_order) {
    extern __shared__ __align__(16) unsigned char smem[];
    float4 *s_r0 = reinterpret_cast<float4 *>(smem);
    float4 *s_r1 = s_r0 + kBlendThreads;
    int *s_j = reinterpret_cast<int *>(s_r1 + kBlendThreads);
    float *s_v = reinterpret_cast<float *>(s_j + kBlendThreads);
    double *s_r64 = reinterpret_cast<double *>(s_v + kBlendThreads * KMAX);  // F64: 6/pair
    double *s_v64 = s_r64 + (F64 ? 6 * kBlendThreads : 0);                   // F64: KMAX/pair
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

    double T = 1.0;
    float acc[KMAX];
    double acc64[F64 ? KMAX : 1];
#pragma unroll
    for (int c = 0; c < KMAX; ++c) acc[c] = 0.0f;
#pragma unroll
    for (int c = 0; c < (F64 ? KMAX : 1); ++c) acc64[c] = 0.0;
    int nc = 0, last = s0;
    bool done = !inside;

    for (int base = s0; base < s1; base += kBlendThreads) {
        if (__syncthreads_count(!done) == 0) break;
        // ---- stage + cull one batch (each thread one pair)
        const int j = base + tid;
        bool keep = false;
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
        int sp = 0;
        if (j < s1) {
            sp = pair_splat[j];
            r0 = __ldg(rec + 2 * sp);
            r1 = __ldg(rec + 2 * sp + 1);
            keep = tile_touch(r0, r1, px0, px1, py0, py1);
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
            const float *v = values + (int64_t)K * sp;
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) s_v[q * KMAX + c] = __ldg(v + c);
            if (F64) {
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
            const float sig = fmaf(fmaf(a1.x, dx, a1.y * dy), dx, (a1.z * dy) * dy);
            if (sig > a0.w) continue;  // reference alpha < 1/255 for certain
            // exact float64 evaluation (_kernels.py:51-61)
            double mx, my, ca, cb, cc, o;
            if (F64) {
                const double *r = s_r64 + q * 6;
                mx = r[0]; my = r[1]; ca = r[2]; cb = r[3]; cc = r[4]; o = r[5];
            } else {
                mx = a0.x; my = a0.y;
                ca = 2.0 * (double)a1.x; cb = a1.y; cc = 2.0 * (double)a1.z;
                o = a0.z;
            }
            const double ddx = dsub(dpx, mx), ddy = dsub(dpy, my);
            const double sg = dadd(dmul(0.5, dadd(dmul(dmul(ca, ddx), ddx), dmul(dmul(cc, ddy), ddy))),
                                   dmul(dmul(cb, ddx), ddy));
            if (sg < 0.0) continue;
            double al = dmul(o, exp(-sg));
            if (al > kAlphaCap) al = kAlphaCap;
            if (al < kAlphaSkip) continue;
            const double w = dmul(T, al);
            if (F64) {
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c < K) acc64[c] = dadd(acc64[c], dmul(w, s_v64[q * KMAX + c]));
            } else {
#pragma unroll
                for (int c = 0; c < KMAX; ++c)
                    if (c < K) acc[c] = (float)dadd((double)acc[c], dmul(w, (double)s_v[q * KMAX + c]));
            }
            T = dmul(T, dsub(1.0, al));
            ++nc;
            last = s_j[q] + 1;
            if (T < kTStop) {
                done = true;
                break;
            }
        }
    }
    if (!inside) return;
    const int64_t pix = (int64_t)py * W + px;
    if (F64) {
        double *o = out64 + pix * K;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < K) o[c] = acc64[c];
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

template <int KMAX, bool F64>
size_t blend_smem_bytes() {
    return (size_t)kBlendThreads * (16 + 16 + 4 + 4 * KMAX) +
           (F64 ? (size_t)kBlendThreads * 8 * (6 + KMAX) : 0);
}

template <int KMAX, bool F64>
int launch_blend(const int32_t *ranges, const int32_t *pair_splat, int ntx, int nty,
                 const float *rec, const float *values, const double *rec64,
                 const double *values64, int K, int W, int H, float *out, double *out64,
                 int32_t *contrib, int32_t *last_pos, double *t_final, const int32_t *tile_order,
                 cudaStream_t st) {
    const size_t sm = blend_smem_bytes<KMAX, F64>();
    auto fn = blend_fwd_kernel<KMAX, F64>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    fn<<<ntx * nty, kBlendThreads, sm, st>>>(ranges, pair_splat, ntx,
                                            reinterpret_cast<const float4 *>(rec), values, rec64,
                                            values64, K, W, H, out, out64, contrib, last_pos,
                                            t_final, tile_order);
    return check_launch("blend_fwd_kernel");
}

}  // namespace ivr

extern "C" int ivr_blend_fwd(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                             int32_t nty, const float *rec, const float *values,
                             const double *rec64, const double *values64, int32_t k,
                             int32_t width, int32_t height, float *out, double *out64,
                             int32_t *contrib, int32_t *last_pos, double *t_final,
                             const int32_t *tile_order, ivr_stream_t stream) {
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
#define IVR_BLEND(KM)                                                                             \
    return f64 ? launch_blend<KM, true>(tile_ranges, pair_splat, ntx, nty, rec, values, rec64,    \
                                        values64, k, width, height, out, out64, contrib,          \
                                        last_pos, t_final, tile_order, st)                        \
               : launch_blend<KM, false>(tile_ranges, pair_splat, ntx, nty, rec, values, rec64,   \
                                         values64, k, width, height, out, out64, contrib,         \
                                         last_pos, t_final, tile_order, st)
    if (k <= 4) { IVR_BLEND(4); }
    if (k <= 8) { IVR_BLEND(8); }
    if (k <= 16) { IVR_BLEND(16); }
    IVR_BLEND(32);
#undef IVR_BLEND
}
