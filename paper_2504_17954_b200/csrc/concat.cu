// Compose on the device: ComposedScene.compose / GaussianGeometry.concat /
// ShadingAttributes.concat (scene.py:147-186, gaussians.py:98-106,
// shading.py:168-176) as one batched copy of device-resident models into the
// concatenated SoA + per-splat scene ids.  HBM-bound (read + write each byte).
#include "ivr_common.cuh"

namespace ivr {

constexpr int kConcatMax = 64;

struct ConcatArgs {
    const double *src[kConcatMax];
    int64_t row0[kConcatMax + 1];  // exclusive prefix of rows
    int n_src, width;
    double *dst;
    int32_t *scene_id;
};

__global__ void __launch_bounds__(256) concat_kernel(ConcatArgs A) {
    const int m = blockIdx.y;
    const int64_t rows = A.row0[m + 1] - A.row0[m];
    const int64_t count = rows * A.width;
    const double *s = A.src[m];
    double *d = A.dst + A.row0[m] * A.width;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        d[i] = s[i];
    if (A.scene_id)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
             i += (int64_t)gridDim.x * blockDim.x)
            A.scene_id[A.row0[m] + i] = m;
}

}  // namespace ivr

extern "C" int ivr_concat(const double *const *srcs, const int64_t *rows, int32_t n_src,
                          int32_t width, double *dst, int32_t *scene_id, ivr_stream_t stream) {
    using namespace ivr;
    if (!srcs || !rows || !dst || n_src < 1 || n_src > kConcatMax || width < 1) {
        set_error("ivr_concat: bad argument (1..64 sources)");
        return IVR_ERR_ARG;
    }
    ConcatArgs A{};
    A.row0[0] = 0;
    int64_t most = 0;
    for (int m = 0; m < n_src; ++m) {
        if (rows[m] < 0 || (rows[m] > 0 && !srcs[m])) {
            set_error("ivr_concat: bad source");
            return IVR_ERR_ARG;
        }
        A.src[m] = srcs[m];
        A.row0[m + 1] = A.row0[m] + rows[m];
        most = rows[m] * width > most ? rows[m] * width : most;
    }
    A.n_src = n_src;
    A.width = width;
    A.dst = dst;
    A.scene_id = scene_id;
    if (most == 0) return IVR_OK;
    int64_t bx = (most + 255) / 256;
    if (bx > 148 * 4) bx = 148 * 4;
    concat_kernel<<<dim3((unsigned)bx, (unsigned)n_src), 256, 0, (cudaStream_t)stream>>>(A);
    return check_launch("concat_kernel");
}
