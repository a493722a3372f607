// Training-step map terms, fused: the upstream image gradient d_out (H,W,K)
// for K4a in one pass over the rendered maps.
//
// Replaces, per pixel (float64 arithmetic, as the reference):
//   * packing of the photometric gradient into the colour / alpha channels
//     (trainer.py:355-366);
//   * pseudo_normal_from_depth + normal_consistency_loss (losses.py:141-206):
//     camera-space points from depth, forward differences (backward at the
//     last row / column), cross product, unit normal facing the camera,
//     rotated to world; mean L2 distance over pixels with alpha > 1e-3;
//   * offset_sparsity_loss on the delta_c maps (losses.py:256-260);
//   * bilateral_smoothness on the k_a, k_d, k_s, beta maps
//     (losses.py:209-253): edge weights exp(-sum |grad gt|) / (H W), gradient
//     gathered from the 4-neighbourhood (no atomics).
// The reference / torch restatement builds each of these with tens of full-map
// array operations; here they are two kernels: a first pass (normal-mask
// count -- the normal loss divides by it -- and the bilateral edge-weight
// map, and the pseudo normals it needs, stored for the second pass) and the
// fused gradient + per-block loss partial sums.
#include "ivr_common.cuh"

namespace ivr {
namespace regk {

constexpr int kThreads = 256;

struct Args {
    const float *out;  // (H, W, K) K3 output
    int K, H, W;
    int c_color, c_alpha, c_depth, c_normal, c_delta, n_bil;
    int c_bil[4];
    const double *gt;      // (H, W, 4)
    const double *d_rgba;  // (H, W, 4) photometric gradient (or null)
    const double *camp;    // device: f, cx, cy, rot[9] (world -> camera, row-major)
    double w_normal, w_offset, w_bil;
    int *mask_count;       // device: pixels in the normal mask
    double *wmap;          // (H, W) bilateral edge weights / (H W), from the first pass
    double4 *nmap;         // (H, W) world pseudo normal + mask flag, from the first pass
    float *d_out;          // (H, W, K)
    double *part;          // per block: normal, |offset| sum, bilateral sum
};

__device__ __forceinline__ double depth_at(const Args &A, int y, int x) {
    return (double)A.out[((int64_t)y * A.W + x) * A.K + A.c_depth];
}

// camera-space point of pixel (y, x), evaluated as numpy does
// (losses.py:157-161: (px - cx) * d / f, each operation rounded).  The pseudo
// normal is a cross product of neighbour differences: where the surface is
// nearly flat those differences cancel and one ulp in a point moves the normal
// (and the mask / facing decisions) visibly, so every step keeps the
// reference's rounding.
__device__ __forceinline__ void point(const Args &A, double f, double cx, double cy, int y, int x,
                                      double p[3]) {
    const double d = depth_at(A, y, x);
    p[0] = ((double)x - cx) * d / f;
    p[1] = ((double)y - cy) * d / f;
    p[2] = d;
}

// pseudo normal (world) at (y, x) and whether it is in the mask
__device__ __forceinline__ bool pseudo_normal(const Args &A, int y, int x, double nw[3]) {
    const double f = A.camp[0], cx = A.camp[1], cy = A.camp[2];
    const double *rot = A.camp + 3;
    double p[3], q[3], dx[3], dy[3];
    point(A, f, cx, cy, y, x, p);
    if (x + 1 < A.W) {
        point(A, f, cx, cy, y, x + 1, q);
        for (int k = 0; k < 3; ++k) dx[k] = q[k] - p[k];
    } else {
        double r[3];
        point(A, f, cx, cy, y, x - 1, r);
        for (int k = 0; k < 3; ++k) dx[k] = p[k] - r[k];
    }
    if (y + 1 < A.H) {
        point(A, f, cx, cy, y + 1, x, q);
        for (int k = 0; k < 3; ++k) dy[k] = q[k] - p[k];
    } else {
        double r[3];
        point(A, f, cx, cy, y - 1, x, r);
        for (int k = 0; k < 3; ++k) dy[k] = p[k] - r[k];
    }
    // np.cross (products rounded, then the difference)
    double n[3] = {dx[1] * dy[2] - dx[2] * dy[1], dx[2] * dy[0] - dx[0] * dy[2],
                   dx[0] * dy[1] - dx[1] * dy[0]};
    // np.linalg.norm: sqrt((n0^2 + n1^2) + n2^2); n / max(norm, 1e-12)
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    const bool good = nn > 1e-12;
    for (int k = 0; k < 3; ++k) n[k] = good ? n[k] / fmax(nn, 1e-12) : 0.0;
    if (n[0] * p[0] + n[1] * p[1] + n[2] * p[2] > 0.0)
        for (int k = 0; k < 3; ++k) n[k] = -n[k];
    // n @ R (OpenBLAS dgemm: the k-ascending FMA chain, ivr_common.cuh chain3)
    for (int j = 0; j < 3; ++j) nw[j] = fma(n[2], rot[6 + j], fma(n[1], rot[3 + j], n[0] * rot[j]));
    const double alpha = (double)A.out[((int64_t)y * A.W + x) * A.K + A.c_alpha];
    return good && alpha > 1e-3;
}

__device__ __forceinline__ double block_sum(double v, double *s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kThreads / 32; ++w) t += s_red[w];
    return t;
}

// bilateral edge weight at (y, x): exp(-sum_c |gt(x+1)-gt| - sum_c |gt(y+1)-gt|)
__device__ __forceinline__ double edge_weight(const Args &A, int y, int x) {
    const double *g = A.gt + ((int64_t)y * A.W + x) * 4;
    double s = 0.0;
    if (x + 1 < A.W) {
        const double *h = g + 4;
        s += fabs(h[0] - g[0]) + fabs(h[1] - g[1]) + fabs(h[2] - g[2]);
    }
    if (y + 1 < A.H) {
        const double *h = g + 4 * (int64_t)A.W;
        s += fabs(h[0] - g[0]) + fabs(h[1] - g[1]) + fabs(h[2] - g[2]);
    }
    return exp(-s);
}

__global__ void __launch_bounds__(kThreads) mask_count_kernel(Args A) {
    ::ivr::pdl_begin();
    __shared__ int s_c;
    if (threadIdx.x == 0) s_c = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    int c = 0;
    if (i < (int64_t)A.H * A.W) {
        const int y = (int)(i / A.W), x = (int)(i % A.W);
        if (A.w_normal > 0.0) {
            double nw[3];
            c = pseudo_normal(A, y, x, nw) ? 1 : 0;
            A.nmap[i] = make_double4(nw[0], nw[1], nw[2], (double)c);
        }
        if (A.w_bil > 0.0 && A.n_bil > 0)
            A.wmap[i] = edge_weight(A, y, x) / ((double)A.H * A.W);  // losses.py:239
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_c, c);
    __syncthreads();
    if (threadIdx.x == 0 && s_c) atomicAdd(A.mask_count, s_c);
}

__device__ __forceinline__ double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// The block's 256 consecutive pixels (their K-channel rows are contiguous) are
// staged through shared memory in both directions: coalesced loads of the
// rendered maps and coalesced stores of d_out, instead of K scattered 4-byte
// accesses per pixel at a 4K-byte stride.
__global__ void __launch_bounds__(kThreads) reg_grad_kernel(Args A) {
    ::ivr::pdl_begin();
    __shared__ double s_red[kThreads / 32];
    extern __shared__ float s_reg[];  // [kThreads * K] maps in, [kThreads * K] d_out
    const int tid = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * kThreads;
    const int64_t i = p0 + tid;
    const int64_t npx = (int64_t)A.H * A.W;
    const int nloc = (int)(npx - p0 < kThreads ? npx - p0 : kThreads);
    const int K = A.K, nflt = nloc * K;
    float *s_in = s_reg, *s_out = s_reg + kThreads * K;
    for (int q = tid; q < nflt; q += kThreads) {
        s_in[q] = A.out[p0 * K + q];
        s_out[q] = 0.0f;
    }
    __syncthreads();
    double l_normal = 0.0, l_offset = 0.0, l_bil = 0.0;
    if (i < npx) {
        const int y = (int)(i / A.W), x = (int)(i % A.W);
        const float *o = s_in + tid * K;
        float *d = s_out + tid * K;
        // x-neighbours from the staged rows when inside the block, else global
        auto left = [&](int c) { return tid > 0 ? o[c - K] : A.out[(i - 1) * K + c]; };
        auto right = [&](int c) { return tid + 1 < nloc ? o[K + c] : A.out[(i + 1) * K + c]; };
        if (A.d_rgba) {
            const double *g = A.d_rgba + 4 * i;
            d[A.c_color] = (float)g[0];
            d[A.c_color + 1] = (float)g[1];
            d[A.c_color + 2] = (float)g[2];
            d[A.c_alpha] = (float)g[3];
        }
        if (A.w_normal > 0.0) {
            const double4 nm = A.nmap[i];  // computed once by the first pass
            const double nw[3] = {nm.x, nm.y, nm.z};
            const bool m = nm.w != 0.0;
            const double cnt = (double)max(*A.mask_count, 1);
            if (m) {
                double df[3];
                for (int k = 0; k < 3; ++k) df[k] = (double)o[A.c_normal + k] - nw[k];
                const double nn = sqrt(df[0] * df[0] + df[1] * df[1] + df[2] * df[2]);
                l_normal = nn / cnt;
                if (nn > 1e-12)
                    for (int k = 0; k < 3; ++k)
                        d[A.c_normal + k] = (float)(A.w_normal * (df[k] / nn / cnt));
            }
        }
        if (A.w_offset > 0.0) {
            const double inv = 1.0 / (3.0 * (double)npx);
            for (int k = 0; k < 3; ++k) {
                const double m = (double)o[A.c_delta + k];
                l_offset += fabs(m);
                d[A.c_delta + k] = (float)(A.w_offset * sgn(m) * inv);
            }
        }
        if (A.w_bil > 0.0 && A.n_bil > 0) {
            const double w0 = A.wmap[i];
            const double wl = x > 0 ? A.wmap[i - 1] : 0.0;
            const double wu = y > 0 ? A.wmap[i - A.W] : 0.0;
            for (int b = 0; b < A.n_bil; ++b) {
                const int c = A.c_bil[b];
                const double k0 = (double)o[c];
                double g = 0.0;
                if (x + 1 < A.W) {
                    const double gx = (double)right(c) - k0;
                    l_bil += fabs(gx) * w0;
                    g -= sgn(gx) * w0;
                }
                if (y + 1 < A.H) {
                    const double gy = (double)A.out[(i + A.W) * K + c] - k0;
                    l_bil += fabs(gy) * w0;
                    g -= sgn(gy) * w0;
                }
                if (x > 0) g += sgn(k0 - (double)left(c)) * wl;
                if (y > 0) g += sgn(k0 - (double)A.out[(i - A.W) * K + c]) * wu;
                d[c] = (float)(A.w_bil * g);
            }
        }
    }
    __syncthreads();
    for (int q = tid; q < nflt; q += kThreads) A.d_out[p0 * K + q] = s_out[q];
    const double a = block_sum(l_normal, s_red);
    const double b = block_sum(l_offset, s_red);
    const double c = block_sum(l_bil, s_red);
    if (threadIdx.x == 0) {
        A.part[3 * blockIdx.x] = a;
        A.part[3 * blockIdx.x + 1] = b;
        A.part[3 * blockIdx.x + 2] = c;
    }
}

// terms[0] = normal loss, [1] = mean |delta_c|, [2] = bilateral sum (all maps)
__global__ void __launch_bounds__(kThreads) reg_finish_kernel(const double *part, int nb, int64_t npx,
                                                              double *terms) {
    ::ivr::pdl_begin();
    __shared__ double s_red[kThreads / 32];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < nb; i += kThreads) {
        a += part[3 * i];
        b += part[3 * i + 1];
        c += part[3 * i + 2];
    }
    const double ta = block_sum(a, s_red), tb = block_sum(b, s_red), tc = block_sum(c, s_red);
    if (threadIdx.x == 0) {
        terms[0] = ta;
        terms[1] = tb / (3.0 * (double)npx);
        terms[2] = tc;
    }
}

}  // namespace regk
}  // namespace ivr

extern "C" size_t ivr_regularize_workspace_size(int32_t height, int32_t width) {
    const int64_t npx = (int64_t)height * width;
    const int64_t nb = (npx + ivr::regk::kThreads - 1) / ivr::regk::kThreads;
    return 256 + 8 * (size_t)(3 * nb) + 8 * (size_t)npx + 32 + 32 * (size_t)npx;
}

extern "C" int ivr_regularize(const float *out, int32_t k, int32_t height, int32_t width,
                              const int32_t cols[5], const int32_t *bil_cols, int32_t n_bil,
                              const double *gt, const double *d_rgba, const double *cam_params,
                              double w_normal, double w_offset, double w_bil, float *d_out,
                              double *terms, void *workspace, size_t workspace_bytes,
                              ivr_stream_t stream) {
    using namespace ivr;
    using namespace ivr::regk;
    if (!out || !cols || !d_out || !terms || k < 1 || height < 2 || width < 2 || n_bil < 0 ||
        n_bil > 4 || (n_bil > 0 && !bil_cols) || (w_bil > 0.0 && n_bil > 0 && !gt) ||
        (w_normal > 0.0 && (!cam_params || cols[1] < 0 || cols[2] < 0 || cols[3] < 0)) ||
        (w_offset > 0.0 && cols[4] < 0) || (d_rgba && (cols[0] < 0 || cols[1] < 0))) {
        set_error("ivr_regularize: bad argument");
        return IVR_ERR_ARG;
    }
    if (!workspace || workspace_bytes < ivr_regularize_workspace_size(height, width)) {
        set_error("ivr_regularize: workspace too small");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    Args A{};
    A.out = out;
    A.K = k;
    A.H = height;
    A.W = width;
    A.c_color = cols[0];
    A.c_alpha = cols[1];
    A.c_depth = cols[2];
    A.c_normal = cols[3];
    A.c_delta = cols[4];
    A.n_bil = n_bil;
    for (int b = 0; b < n_bil; ++b) A.c_bil[b] = bil_cols[b];
    A.gt = gt;
    A.d_rgba = d_rgba;
    A.camp = cam_params;
    A.w_normal = w_normal;
    A.w_offset = w_offset;
    A.w_bil = w_bil;
    char *ws = (char *)workspace;
    A.mask_count = reinterpret_cast<int *>(ws);
    A.part = reinterpret_cast<double *>(ws + 256);
    A.d_out = d_out;
    const int64_t npx = (int64_t)height * width;
    const int nb = (int)((npx + kThreads - 1) / kThreads);
    A.wmap = A.part + 3 * (int64_t)nb;
    A.nmap = reinterpret_cast<double4 *>(((uintptr_t)(A.wmap + npx) + 31) & ~(uintptr_t)31);
    if (cudaMemsetAsync(A.mask_count, 0, sizeof(int), st) != cudaSuccess)
        return check_launch("ivr_regularize memset");
    if (w_normal > 0.0 || (w_bil > 0.0 && n_bil > 0)) ivr::launch<3>(mask_count_kernel, nb, kThreads, 0, st, A);
    const size_t sm_grad = 2 * (size_t)kThreads * k * sizeof(float);
    if (sm_grad > 48 * 1024)
        cudaFuncSetAttribute(reg_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_grad);
    ivr::launch<3>(reg_grad_kernel, nb, kThreads, sm_grad, st, A);
    ivr::launch<3>(reg_finish_kernel, 1, kThreads, 0, st, (const double *)A.part, nb, npx, terms);
    return check_launch("ivr_regularize");
}
