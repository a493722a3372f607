// Shared device helpers for the B200 editable-Gaussian hot path (sm_100a).
//
// Exactness: every TU is compiled with -fmad=false; float64 arithmetic that
// must reproduce the reference's numpy/numba evaluation uses the explicitly
// rounded intrinsics below, and FMAs appear only where the reference itself
// fuses (OpenBLAS dgemm k-chains).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/ivrgs.h"

namespace ivr {

// _kernels.py:14-16, gaussians.py:21-22
constexpr double kAlphaCap = 0.99;
constexpr double kAlphaSkip = 1.0 / 255.0;
constexpr double kTStop = 1e-4;
constexpr double kNearPlane = 0.01;
constexpr double kCov2dDilation = 0.3;
constexpr int kTile = IVR_TILE;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

// numpy's np.clip / np.maximum on ordered (non-NaN) inputs
__device__ __forceinline__ double clip01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : (a < b ? b : a); }

// _mathutil.sigmoid (_mathutil.py:6-13): branch on sign
__device__ __forceinline__ double sigmoid_ref(double x) {
    if (x >= 0.0) return ddiv(1.0, dadd(1.0, exp(-x)));
    const double e = exp(x);
    return ddiv(e, dadd(1.0, e));
}

// np.linalg.norm(v, axis=-1) for length-3/4 rows: sequential add.reduce
__device__ __forceinline__ double norm3(double x, double y, double z) {
    return sqrt(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z)));
}
__device__ __forceinline__ double norm4(double w, double x, double y, double z) {
    return sqrt(dadd(dadd(dadd(dmul(w, w), dmul(x, x)), dmul(y, y)), dmul(z, z)));
}
// np.sum(a*b, axis=-1) for 3-vectors
__device__ __forceinline__ double dot3(const double a[3], const double b[3]) {
    return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]));
}

// OpenBLAS dgemm inner product over k = 0..2 as measured on the reference
// machine: fma(a2, b2, fma(a1, b1, a0 * b0)).
__device__ __forceinline__ double chain3(double a0, double b0, double a1, double b1,
                                         double a2, double b2) {
    return dfma(a2, b2, dfma(a1, b1, dmul(a0, b0)));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Programmatic dependent launch (sm_90+).  A kernel started by `launch`
// below may be scheduled while its stream predecessor drains; pdl_begin()
// first waits for that predecessor's completion and memory flush (so nothing
// before it may touch global memory), then lets the NEXT kernel of the stream
// be scheduled onto SMs this grid's retiring CTAs free.  Without the launch
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// IVR_PDL: 0 off; 1 (default) K2's chain outside graph capture; 2 K2's chain
// always; 3 every kernel launched through here (K1, K3 and the training /
// inverse step kernels too).  Inside a captured graph the programmatic edges
// measured neutral for the isolated C2 frame, -3% for the 6-slot frame stream
// (CTAs waiting at griddepcontrol.wait hold SM slots other frames could use)
// and -3% / -1% for the C3 / C4 steps; eager launches gain ~13 us of K2 per
// frame.
int pdl_level();

// kernel<<<grid, block, smem, stream>>>(args...) with the programmatic
// stream-serialisation attribute when IVR_PDL allows it for LEVEL
template <int LEVEL = 1, typename... P, typename... A>
inline cudaError_t launch(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, A &&...args) {
    const int lvl = pdl_level();
    bool pdl = lvl >= LEVEL && lvl > 0;
    if (pdl && lvl == 1) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
            // the legacy stream while another thread captures globally: no
            // programmatic edge, and the query's error is not this launch's
            (void)cudaGetLastError();
            pdl = false;
        } else {
            pdl = cs == cudaStreamCaptureStatusNone;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

}  // namespace ivr

// error plumbing shared by the C-ABI wrappers
namespace ivr {
void set_error(const char *msg);
int check_launch(const char *what);
}  // namespace ivr
