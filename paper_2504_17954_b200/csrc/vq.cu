// K5/K6 -- scalar-codebook VQ assign and decode (bandwidth kernels).
//
// The reference's codebooks are 1-D (one scalar codebook per attribute,
// shared across components; vq.py:1-6, 137-147) and assignment is
// np.searchsorted over float64 centroid midpoints (vq.py:90-96).  Nearest
// codeword search in 1-D is a binary search, not a distance GEMM: there is no
// contraction dimension to put on tensor cores (SURVEY.md finding 5), so
// these kernels are HBM-bound (6 B per value in + out).  Midpoints live in
// shared memory (K=4096 -> 32 KB); ~12 compares per value.
#include "ivr_common.cuh"

namespace ivr {

constexpr int kVqThreads = 256;
constexpr int kVqSmemMids = 6144;  // 48 KB of float64 midpoints

template <bool SMEM>
__global__ void __launch_bounds__(kVqThreads)
vq_assign_kernel(const double *__restrict__ values, int64_t n, const double *__restrict__ cents,
                 int k, uint16_t *__restrict__ out) {
    __shared__ double s_mid[SMEM ? kVqSmemMids : 1];
    if (SMEM) {
        for (int i = threadIdx.x; i < k - 1; i += kVqThreads)
            s_mid[i] = 0.5 * (cents[i + 1] + cents[i]);
        __syncthreads();
    }
    // searchsorted(mids, v, 'left') = number of mids < v.  Fixed-trip-count
    // binary search over kVqIlp independent values per thread, interleaved so
    // the shared-memory loads of different values overlap (the search is
    // latency-bound, not bandwidth-bound).
    const int nm = k - 1;
    int top = 1;
    while ((top << 1) <= nm) top <<= 1;
    constexpr int kVqIlp = 8;
    const int64_t chunk = (int64_t)kVqThreads * kVqIlp;
    for (int64_t base = (int64_t)blockIdx.x * chunk; base < n; base += (int64_t)gridDim.x * chunk) {
        double v[kVqIlp];
        int pos[kVqIlp];
#pragma unroll
        for (int r = 0; r < kVqIlp; ++r) {
            const int64_t i = base + r * kVqThreads + threadIdx.x;
            v[r] = i < n ? values[i] : 0.0;
            pos[r] = 0;
        }
        for (int step = top; step > 0; step >>= 1) {
#pragma unroll
            for (int r = 0; r < kVqIlp; ++r) {
                const int m = pos[r] + step;
                if (m <= nm) {
                    const double mid = SMEM ? s_mid[m - 1]
                                            : 0.5 * (__ldg(cents + m) + __ldg(cents + m - 1));
                    if (mid < v[r]) pos[r] = m;
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kVqIlp; ++r) {
            const int64_t i = base + r * kVqThreads + threadIdx.x;
            if (i < n) out[i] = (uint16_t)(v[r] != v[r] ? nm : pos[r]);  // NaN sorts last
        }
    }
}

__global__ void __launch_bounds__(kVqThreads)
vq_decode_kernel(const uint16_t *__restrict__ idx, int64_t n, const double *__restrict__ cents,
                 int k, double *__restrict__ out, long long *bad) {
    for (int64_t i = (int64_t)blockIdx.x * kVqThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kVqThreads) {
        const int j = idx[i];
        if (j >= k) {
            atomicMax(bad, (long long)j);
            out[i] = 0.0;
        } else {
            out[i] = __ldg(cents + j);
        }
    }
}

static int grid_for(int64_t n) {
    int64_t b = (n + kVqThreads - 1) / kVqThreads;
    const int64_t cap = 148 * 16;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace ivr

extern "C" int ivr_vq_assign(const double *values, int64_t n, const double *centroids, int32_t k,
                             uint16_t *indices, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || k < 1 || k > 65536 || (n > 0 && (!values || !centroids || !indices))) {
        set_error("ivr_vq_assign: bad argument");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (k - 1 <= kVqSmemMids)
        vq_assign_kernel<true><<<grid_for(n), kVqThreads, 0, st>>>(values, n, centroids, k, indices);
    else
        vq_assign_kernel<false><<<grid_for(n), kVqThreads, 0, st>>>(values, n, centroids, k, indices);
    return check_launch("vq_assign_kernel");
}

extern "C" int ivr_vq_decode(const uint16_t *indices, int64_t n, const double *centroids, int32_t k,
                             double *out, int64_t *bad, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || k < 1 || !bad || (n > 0 && (!indices || !centroids || !out))) {
        set_error("ivr_vq_decode: bad argument");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    vq_decode_kernel<<<grid_for(n), kVqThreads, 0, (cudaStream_t)stream>>>(
        indices, n, centroids, k, out, reinterpret_cast<long long *>(bad));
    return check_launch("vq_decode_kernel");
}
