// Photometric loss: L1 + (1 - SSIM) with its analytic gradient, float64.
//
// Replaces losses.ssim / losses.photometric_loss (losses.py:45-138): an
// 11x11 Gaussian window (sigma 1.5) evaluated where it fits ("valid"),
// population statistics, C1 = 0.01^2, C2 = 0.03^2, mean over windows and
// channels; the gradient is the adjoint ("full") filtering of the per-window
// partials.  The reference runs 8 scipy convolutions per channel; here two
// shared-memory tiled kernels do the work of all of them:
//   A) per 16x32 block of windows: stage the 26x42 input patch of x and y,
//      horizontal then vertical 11-tap passes for x, y, x^2, y^2, xy, the
//      SSIM value, and the three partial maps dL/d(ux), dL/d(uxx), dL/d(uxy);
//   B) per 16x32 block of pixels: stage the 26x42 patch of the three maps
//      (zero outside the valid windows), full 11-tap passes, then
//      d_pred = a * sign(x - y) + b * (F(d_ux) + 2x F(d_uxx) + y F(d_uxy))
//      and the |x - y| sum for the L1 term.
// Per-block partial sums are reduced in a fixed order (deterministic).
// Bound: FP64 issue (~ (5 + 3) x 22 DFMA per pixel and channel) and the
// f64 traffic of x, y, three maps and d_pred (~ 7 x 8 B per pixel-channel).
#include "ivr_common.cuh"

namespace ivr {
namespace ssimk {

constexpr int R = 5, WIN = 2 * R + 1;
constexpr int TH = 32, TW = 32;                 // output tile (windows in A, pixels in B)
constexpr int IH = TH + WIN - 1, IW = TW + WIN - 1;  // 42 x 42 staged patch
// register blocking: every filtering thread produces RB consecutive outputs of
// its row (horizontal) or column (vertical), streaming the RB + 10 inputs once
// from shared memory (RB + 10 loads for RB outputs instead of 11 RB); the
// taps of each output are still accumulated in ascending order
constexpr int RB = 4;
static_assert((TH / RB) * TW == 256, "one vertical strip per thread");
constexpr int kStageIt = (IH * IW + 255) / 256;  // staging elements per thread
constexpr int kThreads = 256;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

struct Args {
    const double *x, *y;  // (H, W, C)
    // optional prediction source: channel c of pixel p = xf[p * xs + xcol[c]]
    // (K3's float32 (H, W, k) frame read in place; promotion to f64 is exact)
    const float *xf;
    int xs, xcol[4];
    int H, W, C, Hv, Wv;
    double g[WIN];
    double up;            // 1 / (Hv * Wv * C)
    double a, b;          // d_pred = a * sign(x - y) + b * d(mean SSIM)/dx
    double *m_ux, *m_uxx, *m_uxy;  // (C, Hv, Wv)
    double *partA, *partB;         // per-block partial sums
    double *d_pred;                // (H, W, C)
};

__device__ __forceinline__ double load_x(const Args &A, int64_t pix, int c) {
    return A.xf ? (double)__ldg(A.xf + pix * A.xs + A.xcol[c]) : A.x[pix * A.C + c];
}

__device__ __forceinline__ double block_sum(double v, double *s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) t += s_red[w];
    return t;
}

// A: window statistics -> SSIM partial sum + the three partial maps
__global__ void __launch_bounds__(kThreads) ssim_window_kernel(Args A) {
    ::ivr::pdl_begin();
    extern __shared__ __align__(16) double sm[];
    double *sx = sm, *sy = sx + IH * IW;
    double *hq = sy + IH * IW;  // [5][IH][TW]
    __shared__ double s_red[kThreads / 32];
    const int i0 = blockIdx.y * TH, j0 = blockIdx.x * TW;
    const int tid = threadIdx.x;
    double ssum = 0.0;
    for (int c = 0; c < A.C; ++c) {
        __syncthreads();
        // staging: fully unrolled so every load of the patch is in flight at once
        // (a rolled loop serialises one global round trip per 256 elements)
        {
            double vx[kStageIt], vy[kStageIt];
#pragma unroll
            for (int it = 0; it < kStageIt; ++it) {
                const int k = it * kThreads + tid;
                const int r = k / IW, q = k % IW, gi = i0 + r, gj = j0 + q;
                const bool ok = k < IH * IW && gi < A.H && gj < A.W;
                const int64_t px = (int64_t)gi * A.W + gj, o = px * A.C + c;
                vx[it] = ok ? load_x(A, px, c) : 0.0;
                vy[it] = ok ? A.y[o] : 0.0;
            }
#pragma unroll
            for (int it = 0; it < kStageIt; ++it) {
                const int k = it * kThreads + tid;
                if (k < IH * IW) {
                    sx[k] = vx[it];
                    sy[k] = vy[it];
                }
            }
        }
        __syncthreads();
        for (int k = tid; k < IH * (TW / RB); k += kThreads) {
            const int r = k / (TW / RB), q0 = (k % (TW / RB)) * RB;
            double h[5][RB];
#pragma unroll
            for (int o = 0; o < RB; ++o)
#pragma unroll
                for (int m = 0; m < 5; ++m) h[m][o] = 0.0;
#pragma unroll
            for (int jj = 0; jj < RB + WIN - 1; ++jj) {
                const double xv = sx[r * IW + q0 + jj], yv = sy[r * IW + q0 + jj];
                const double xx = xv * xv, yy = yv * yv, xy = xv * yv;
#pragma unroll
                for (int o = 0; o < RB; ++o) {
                    const int t = jj - o;
                    if (t < 0 || t >= WIN) continue;
                    const double g = A.g[t];
                    h[0][o] = fma(g, xv, h[0][o]);
                    h[1][o] = fma(g, yv, h[1][o]);
                    h[2][o] = fma(g, xx, h[2][o]);
                    h[3][o] = fma(g, yy, h[3][o]);
                    h[4][o] = fma(g, xy, h[4][o]);
                }
            }
#pragma unroll
            for (int m = 0; m < 5; ++m)
#pragma unroll
                for (int o = 0; o < RB; ++o) hq[m * IH * TW + r * TW + q0 + o] = h[m][o];
        }
        __syncthreads();
        {
            const int q = tid % TW, r0 = (tid / TW) * RB;
            double u[5][RB];
#pragma unroll
            for (int m = 0; m < 5; ++m) {
#pragma unroll
                for (int o = 0; o < RB; ++o) u[m][o] = 0.0;
#pragma unroll
                for (int ii = 0; ii < RB + WIN - 1; ++ii) {
                    const double v = hq[m * IH * TW + (r0 + ii) * TW + q];
#pragma unroll
                    for (int o = 0; o < RB; ++o) {
                        const int t = ii - o;
                        if (t < 0 || t >= WIN) continue;
                        u[m][o] = fma(A.g[t], v, u[m][o]);
                    }
                }
            }
            const int wj = j0 + q;
#pragma unroll
            for (int o = 0; o < RB; ++o) {
                const int wi = i0 + r0 + o;
                if (wi >= A.Hv || wj >= A.Wv) continue;
                const double ux = u[0][o], uy = u[1][o];
                const double vx = u[2][o] - ux * ux, vy = u[3][o] - uy * uy, vxy = u[4][o] - ux * uy;
                const double a1 = 2.0 * ux * uy + kC1, a2 = 2.0 * vxy + kC2;
                const double b1 = ux * ux + uy * uy + kC1, b2 = vx + vy + kC2;
                const double bb = b1 * b2;
                const double s = (a1 * a2) / bb;  // the reference's SSIM value
                ssum += s;
                // gradient-only partials from one reciprocal (1/b1 = b2/bb, 1/b2 = b1/bb)
                const double ibb = 1.0 / bb, sup = s * ibb * A.up;
                const double da1 = a2 * ibb * A.up, da2 = a1 * ibb * A.up;
                const double db1 = -sup * b2, db2 = -sup * b1;
                const double d_uxy = 2.0 * da2;
                const double d_uxx = db2;
                const double d_ux = 2.0 * uy * da1 + 2.0 * ux * db1 - 2.0 * ux * db2 - uy * d_uxy;
                const int64_t o2 = ((int64_t)c * A.Hv + wi) * A.Wv + wj;
                A.m_ux[o2] = d_ux;
                A.m_uxx[o2] = d_uxx;
                A.m_uxy[o2] = d_uxy;
            }
        }
    }
    const double t = block_sum(ssum, s_red);
    if (tid == 0) A.partA[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// B: adjoint filtering of the maps -> d_pred, plus the L1 partial sum
// 3 CTAs/SM (80 registers, no spills; 74 KB of shared memory each): the
// staging loads were 45% of the warp stalls at 2 CTAs/SM (C4 loss 0.172 ->
// 0.158 ms, C3 losses 0.282 -> 0.269 ms)
template <bool SSIM>
__global__ void __launch_bounds__(kThreads, 3) ssim_grad_kernel(Args A) {
    ::ivr::pdl_begin();
    extern __shared__ __align__(16) double sm[];
    double *mq = sm;                    // [3][IH][IW]
    double *hq = mq + 3 * IH * IW;      // [3][IH][TW]
    __shared__ double s_red[kThreads / 32];
    const int i0 = blockIdx.y * TH, j0 = blockIdx.x * TW;
    const int tid = threadIdx.x;
    double l1 = 0.0;
    for (int c = 0; c < A.C; ++c) {
        if (SSIM) {
            __syncthreads();
            double v0[kStageIt], v1[kStageIt], v2[kStageIt];
#pragma unroll
            for (int it = 0; it < kStageIt; ++it) {
                const int k = it * kThreads + tid;
                const int r = k / IW, q = k % IW, wi = i0 - (WIN - 1) + r, wj = j0 - (WIN - 1) + q;
                const bool ok = k < IH * IW && wi >= 0 && wj >= 0 && wi < A.Hv && wj < A.Wv;
                const int64_t o = ((int64_t)c * A.Hv + wi) * A.Wv + wj;
                v0[it] = ok ? A.m_ux[o] : 0.0;
                v1[it] = ok ? A.m_uxx[o] : 0.0;
                v2[it] = ok ? A.m_uxy[o] : 0.0;
            }
#pragma unroll
            for (int it = 0; it < kStageIt; ++it) {
                const int k = it * kThreads + tid;
                if (k < IH * IW) {
                    mq[0 * IH * IW + k] = v0[it];
                    mq[1 * IH * IW + k] = v1[it];
                    mq[2 * IH * IW + k] = v2[it];
                }
            }
            __syncthreads();
            for (int k = tid; k < IH * (TW / RB); k += kThreads) {
                const int r = k / (TW / RB), q0 = (k % (TW / RB)) * RB;
                double h[3][RB];
#pragma unroll
                for (int o = 0; o < RB; ++o)
#pragma unroll
                    for (int m = 0; m < 3; ++m) h[m][o] = 0.0;
                // output q0 + o takes tap t from column q0 + o + 10 - t: stream
                // the columns right to left so every output's taps ascend
#pragma unroll
                for (int jj = RB + WIN - 2; jj >= 0; --jj) {
                    double v[3];
#pragma unroll
                    for (int m = 0; m < 3; ++m) v[m] = mq[m * IH * IW + r * IW + q0 + jj];
#pragma unroll
                    for (int o = 0; o < RB; ++o) {
                        const int t = o + (WIN - 1) - jj;
                        if (t < 0 || t >= WIN) continue;
                        const double g = A.g[t];
#pragma unroll
                        for (int m = 0; m < 3; ++m) h[m][o] = fma(g, v[m], h[m][o]);
                    }
                }
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                    for (int o = 0; o < RB; ++o) hq[m * IH * TW + r * TW + q0 + o] = h[m][o];
            }
            __syncthreads();
        }
        const int q = tid % TW, r0 = (tid / TW) * RB;
        double f[3][RB];
#pragma unroll
        for (int m = 0; m < 3; ++m)
#pragma unroll
            for (int o = 0; o < RB; ++o) f[m][o] = 0.0;
        if (SSIM) {
#pragma unroll
            for (int m = 0; m < 3; ++m) {
#pragma unroll
                for (int ii = RB + WIN - 2; ii >= 0; --ii) {
                    const double v = hq[m * IH * TW + (r0 + ii) * TW + q];
#pragma unroll
                    for (int o = 0; o < RB; ++o) {
                        const int t = o + (WIN - 1) - ii;
                        if (t < 0 || t >= WIN) continue;
                        f[m][o] = fma(A.g[t], v, f[m][o]);
                    }
                }
            }
        }
        const int pj = j0 + q;
#pragma unroll
        for (int o = 0; o < RB; ++o) {
            const int pi = i0 + r0 + o;
            if (pi >= A.H || pj >= A.W) continue;
            const int64_t px = (int64_t)pi * A.W + pj, oo = px * A.C + c;
            const double xv = load_x(A, px, c), yv = A.y[oo];
            const double df = xv - yv;
            l1 += fabs(df);
            double d = A.a * (df > 0.0 ? 1.0 : (df < 0.0 ? -1.0 : 0.0));
            if (SSIM) d += A.b * (f[0][o] + 2.0 * xv * f[1][o] + yv * f[2][o]);
            A.d_pred[oo] = d;
        }
    }
    const double t = block_sum(l1, s_red);
    if (tid == 0) A.partB[blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// sums[0] = sum of SSIM over windows and channels, sums[1] = sum |x - y|
__global__ void __launch_bounds__(kThreads) ssim_finish_kernel(const double *partA, int na,
                                                               const double *partB, int nb,
                                                               double *sums) {
    ::ivr::pdl_begin();
    __shared__ double s_red[kThreads / 32];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < na; i += kThreads) a += partA[i];
    for (int i = threadIdx.x; i < nb; i += kThreads) b += partB[i];
    const double ta = block_sum(a, s_red);
    const double tb = block_sum(b, s_red);
    if (threadIdx.x == 0) {
        sums[0] = ta;
        sums[1] = tb;
    }
}

struct Plan {
    int64_t maps;  // doubles per map
    int na, nb;
    size_t bytes;
};

inline Plan plan(int H, int W, int C) {
    Plan p{};
    const int Hv = H - WIN + 1 > 0 ? H - WIN + 1 : 0, Wv = W - WIN + 1 > 0 ? W - WIN + 1 : 0;
    p.maps = (int64_t)C * Hv * Wv;
    p.na = ((Wv + TW - 1) / TW) * ((Hv + TH - 1) / TH);
    p.nb = ((W + TW - 1) / TW) * ((H + TH - 1) / TH);
    p.bytes = 8 * (size_t)(3 * p.maps + p.na + p.nb + 2);
    return p;
}

}  // namespace ssimk
}  // namespace ivr

extern "C" size_t ivr_photometric_workspace_size(int32_t height, int32_t width, int32_t channels) {
    return ivr::ssimk::plan(height, width, channels).bytes;
}

static int photometric(const double *pred, const float *frame, int32_t frame_k,
                       const int32_t *cols, const double *gt, int32_t height, int32_t width,
                       int32_t channels, const double window[11], double a, double b,
                       int32_t with_ssim, double *d_pred, double *sums, void *workspace,
                       size_t workspace_bytes, ivr_stream_t stream) {
    using namespace ivr;
    using namespace ivr::ssimk;
    if ((!pred && !frame) || !gt || !d_pred || !sums || !window || height < 1 || width < 1 || channels < 1 ||
        (with_ssim && (height < WIN || width < WIN))) {
        set_error("ivr_photometric_loss: bad argument (images smaller than the 11x11 window?)");
        return IVR_ERR_ARG;
    }
    const Plan p = plan(height, width, channels);
    if (!workspace || workspace_bytes < p.bytes) {
        set_error("ivr_photometric_loss: workspace too small");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Args A{};
    A.x = pred;
    A.xf = frame;
    if (frame) {
        if (channels > 4 || !cols || frame_k < 1) {
            set_error("ivr_photometric_loss_frame: needs 1..4 channels and a column map");
            return IVR_ERR_ARG;
        }
        A.xs = frame_k;
        for (int c = 0; c < channels; ++c) {
            if (cols[c] < 0 || cols[c] >= frame_k) {
                set_error("ivr_photometric_loss_frame: column out of range");
                return IVR_ERR_ARG;
            }
            A.xcol[c] = cols[c];
        }
    }
    A.y = gt;
    A.H = height;
    A.W = width;
    A.C = channels;
    A.Hv = height - WIN + 1;
    A.Wv = width - WIN + 1;
    for (int t = 0; t < WIN; ++t) A.g[t] = window[t];
    A.up = with_ssim ? 1.0 / ((double)A.Hv * A.Wv * channels) : 0.0;
    A.a = a;
    A.b = b;
    double *ws = (double *)workspace;
    A.m_ux = ws;
    A.m_uxx = ws + p.maps;
    A.m_uxy = ws + 2 * p.maps;
    A.partA = ws + 3 * p.maps;
    A.partB = A.partA + p.na;
    A.d_pred = d_pred;
    const size_t smA = 8 * (size_t)(2 * IH * IW + 5 * IH * TW);
    const size_t smB = 8 * (size_t)(3 * IH * IW + 3 * IH * TW);
    int na = 0;
    if (with_ssim) {
        cudaFuncSetAttribute(ssim_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
        const dim3 gA((A.Wv + TW - 1) / TW, (A.Hv + TH - 1) / TH);
        ivr::launch<3>(ssim_window_kernel, gA, kThreads, smA, st, A);
        na = p.na;
        cudaFuncSetAttribute(ssim_grad_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB);
    }
    const dim3 gB((width + TW - 1) / TW, (height + TH - 1) / TH);
    if (with_ssim)
        ivr::launch<3>(ssim_grad_kernel<true>, gB, kThreads, smB, st, A);
    else
        ivr::launch<3>(ssim_grad_kernel<false>, gB, kThreads, 0, st, A);
    ivr::launch<3>(ssim_finish_kernel, 1, kThreads, 0, st, (const double *)A.partA, na, (const double *)A.partB, p.nb, sums);
    return check_launch("ivr_photometric_loss");
}

extern "C" int ivr_photometric_loss(const double *pred, const double *gt, int32_t height,
                                    int32_t width, int32_t channels, const double window[11],
                                    double a, double b, int32_t with_ssim, double *d_pred,
                                    double *sums, void *workspace, size_t workspace_bytes,
                                    ivr_stream_t stream) {
    if (!pred) {
        ivr::set_error("ivr_photometric_loss: bad argument (null prediction)");
        return IVR_ERR_ARG;
    }
    return photometric(pred, nullptr, 0, nullptr, gt, height, width, channels, window, a, b,
                       with_ssim, d_pred, sums, workspace, workspace_bytes, stream);
}

extern "C" int ivr_photometric_loss_frame(const float *frame, int32_t frame_k,
                                          const int32_t *cols, const double *gt, int32_t height,
                                          int32_t width, int32_t channels,
                                          const double window[11], double a, double b,
                                          int32_t with_ssim, double *d_pred, double *sums,
                                          void *workspace, size_t workspace_bytes,
                                          ivr_stream_t stream) {
    if (!frame) {
        ivr::set_error("ivr_photometric_loss_frame: bad argument (null frame)");
        return IVR_ERR_ARG;
    }
    return photometric(nullptr, frame, frame_k, cols, gt, height, width, channels, window, a, b,
                       with_ssim, d_pred, sums, workspace, workspace_bytes, stream);
}
