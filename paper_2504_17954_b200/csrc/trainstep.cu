// Training-step plumbing in three launches (replacing ~50 small tensor ops
// per step: the C3 step was host-bound on their dispatch).
//
//  * ivr_stage2_attrs: the stage-2 attribute channels packed by K1
//    (trainer.py:379-404): k_a/k_d/k_s = sigmoid(raw) (_mathutil.py:6-13),
//    beta = exp(log_beta) + 1 (shading.py:132-134).
//  * ivr_step_assemble: the per-Gaussian tail of _stage1_step /
//    _stage2_step (trainer.py:386-394, 410-444): value-channel chain rule
//    into the shading parameters (delta_c += d_values[delta_c];
//    d_k_raw += d_k sigma'(raw); d_log_beta += d_beta (beta - 1)), the
//    opacity-L1 gradient w o (1 - o) / n (losses.py:263-268), the densify
//    statistic |d_mean2d| + |d_n_raw| (trainer.py:443), and per-block
//    partial sums of o for the opacity-L1 value.
//  * ivr_loss_finalize: the step's scalar loss (losses.py:118-138 +
//    trainer.py:355-366, 410-431) from the fused kernels' sums, with the
//    reference's divergence bookkeeping (first non-finite photometric loss).
// All float64 (the TU is built with -fmad=false).
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {
namespace stepk {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 4;  // fixed grid: deterministic partial sums

__global__ void __launch_bounds__(kThreads)
attrs_kernel(int64_t n, const double *ka, const double *kd, const double *ks, const double *lb,
             double *oa, double *od, double *os, double *ob) {
    ::ivr::pdl_begin();
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        oa[i] = sigmoid_ref(ka[i]);
        od[i] = sigmoid_ref(kd[i]);
        os[i] = sigmoid_ref(ks[i]);
        ob[i] = dadd(exp(lb[i]), 1.0);
    }
}

// d * sigma(raw) * (1 - sigma(raw)), in the trainer's evaluation order
__device__ __forceinline__ double dsig(double d, double raw) {
    const double s = sigmoid_ref(raw);
    return dmul(dmul(d, s), dsub(1.0, s));
}

__global__ void __launch_bounds__(kThreads) assemble_kernel(ivr_step_grads A) {
    ::ivr::pdl_begin();
    __shared__ double s_red[kThreads / 32];
    double osum = 0.0;
    const int K = A.k;
    const double dn = (double)A.n;
    // captured steps: sticky overflow gate (0 -> 1 only, so blocks reading the
    // word before or after block 0 updates it compute the same value)
    bool gated = false;
    if (A.gate) {
        gated = *A.gate != 0 || (int64_t)*A.n_pairs > A.pair_capacity;
        if (blockIdx.x == 0 && threadIdx.x == 0) *A.gate = gated ? 1 : 0;
    }
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < A.n;
         i += (int64_t)gridDim.x * kThreads) {
        const double *dv = A.d_values ? A.d_values + (int64_t)K * i : nullptr;
        if (A.o_logit) {
            const double o = sigmoid_ref(A.o_logit[i]);
            osum = dadd(osum, o);
            if (A.d_o_logit && A.w_opacity_l1 > 0.0)
                A.d_o_logit[i] = dadd(A.d_o_logit[i],
                                      ddiv(dmul(dmul(A.w_opacity_l1, o), dsub(1.0, o)), dn));
        }
        if (dv) {
            if (A.d_delta_c && A.col_delta_c >= 0)
                for (int c = 0; c < 3; ++c)
                    A.d_delta_c[3 * i + c] = dadd(A.d_delta_c[3 * i + c], dv[A.col_delta_c + c]);
            if (A.d_k_a_raw && A.col_k_a >= 0)
                A.d_k_a_raw[i] = dadd(A.d_k_a_raw[i], dsig(dv[A.col_k_a], A.k_a_raw[i]));
            if (A.d_k_d_raw && A.col_k_d >= 0)
                A.d_k_d_raw[i] = dadd(A.d_k_d_raw[i], dsig(dv[A.col_k_d], A.k_d_raw[i]));
            if (A.d_k_s_raw && A.col_k_s >= 0)
                A.d_k_s_raw[i] = dadd(A.d_k_s_raw[i], dsig(dv[A.col_k_s], A.k_s_raw[i]));
            if (A.d_log_beta && A.col_beta >= 0) {
                const double beta = dadd(exp(A.log_beta[i]), 1.0);
                A.d_log_beta[i] = dadd(A.d_log_beta[i], dmul(dv[A.col_beta], dsub(beta, 1.0)));
            }
        }
        if (A.stat) {
            const double *m = A.d_mean2d + 2 * i, *r = A.d_n_raw + 3 * i;
            const double st = dadd(sqrt(dadd(dmul(m[0], m[0]), dmul(m[1], m[1]))),
                                   norm3(r[0], r[1], r[2]));
            A.stat[i] = st;
            if (A.stat_sum && !gated) A.stat_sum[i] = dadd(A.stat_sum[i], st);
        }
    }
    if (!A.o_partial) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) osum += __shfl_xor_sync(0xffffffffu, osum, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = osum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t = dadd(t, s_red[w]);
        A.o_partial[blockIdx.x] = t;
    }
}

constexpr int kFinThreads = 256;

__global__ void __launch_bounds__(kFinThreads)
finalize_kernel(ivr_loss_terms T, double *loss, int64_t *state, double *last_bad) {
    ::ivr::pdl_begin();
    // opacity partials: fixed strided split + fixed-order tree (deterministic);
    // one thread summing them serially put ~25 us of dependent loads on the
    // step's critical path
    __shared__ double s_part[kFinThreads];
    double ps = 0.0;
    if (T.o_partial)
        for (int b = threadIdx.x; b < T.n_partial; b += kFinThreads) ps = dadd(ps, T.o_partial[b]);
    s_part[threadIdx.x] = ps;
    __syncthreads();
    for (int h = kFinThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) s_part[threadIdx.x] = dadd(s_part[threadIdx.x], s_part[threadIdx.x + h]);
        __syncthreads();
    }
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    // photometric part (losses.photometric_loss): l1 * mean|x - y| + s * (1 - mean SSIM)
    double photo = dmul(T.l1_weight, ddiv(T.photo_sums[1], T.numel));
    if (T.ssim_weight > 0.0)
        photo = dadd(photo, dmul(T.ssim_weight, dsub(1.0, ddiv(T.photo_sums[0], T.windows))));
    double L = photo;
    if (T.terms) {
        if (T.w_normal > 0.0) L = dadd(L, dmul(T.w_normal, T.terms[0]));
        if (T.w_offset > 0.0) L = dadd(L, dmul(T.w_offset, T.terms[1]));
        if (T.w_bil > 0.0) L = dadd(L, dmul(T.w_bil, T.terms[2]));
    }
    if (T.o_partial && T.w_opacity_l1 > 0.0) L = dadd(L, dmul(T.w_opacity_l1, ddiv(s_part[0], T.n)));
    *loss = L;
    if (state) {  // [step count, first step with a non-finite photometric loss or -1]
        state[0] += 1;
        if (!isfinite(photo) && state[1] < 0) {
            state[1] = state[0];
            if (last_bad) *last_bad = photo;
        }
    }
}

}  // namespace stepk
}  // namespace ivr

using namespace ivr::stepk;

namespace {
unsigned grid_for(int64_t n) {
    int64_t b = (n + kThreads - 1) / kThreads;
    if (b > kMaxBlocks) b = kMaxBlocks;
    return (unsigned)(b < 1 ? 1 : b);
}
}  // namespace

extern "C" int ivr_stage2_attrs(int64_t n, const double *k_a_raw, const double *k_d_raw,
                                const double *k_s_raw, const double *log_beta, double *k_a,
                                double *k_d, double *k_s, double *beta, ivr_stream_t stream) {
    if (n < 0 || (n > 0 && (!k_a_raw || !k_d_raw || !k_s_raw || !log_beta || !k_a || !k_d ||
                            !k_s || !beta))) {
        ivr::set_error("ivr_stage2_attrs: bad argument");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    ivr::launch<3>(attrs_kernel, grid_for(n), kThreads, 0, (cudaStream_t)stream, n, k_a_raw, k_d_raw, k_s_raw,
                                                                     log_beta, k_a, k_d, k_s, beta);
    return ivr::check_launch("attrs_kernel");
}

extern "C" int32_t ivr_step_partials(int64_t n) { return (int32_t)grid_for(n); }

extern "C" int ivr_step_assemble(const ivr_step_grads *a, ivr_stream_t stream) {
    if (!a || a->n < 0 || a->k < 0 || (a->d_values && a->k < 1) ||
        (a->stat && (!a->d_mean2d || !a->d_n_raw)) ||
        (a->d_k_a_raw && a->col_k_a >= 0 && !a->k_a_raw) ||
        (a->d_k_d_raw && a->col_k_d >= 0 && !a->k_d_raw) ||
        (a->d_k_s_raw && a->col_k_s >= 0 && !a->k_s_raw) ||
        (a->d_log_beta && a->col_beta >= 0 && !a->log_beta) ||
        (a->o_partial && !a->o_logit)) {
        ivr::set_error("ivr_step_assemble: bad argument");
        return IVR_ERR_ARG;
    }
    if (a->n == 0) return IVR_OK;
    ivr::launch<3>(assemble_kernel, grid_for(a->n), kThreads, 0, (cudaStream_t)stream, *a);
    return ivr::check_launch("assemble_kernel");
}

extern "C" int ivr_loss_finalize(const ivr_loss_terms *t, double *loss, int64_t *state,
                                 double *last_bad, ivr_stream_t stream) {
    if (!t || !t->photo_sums || !loss || (t->o_partial && t->n_partial < 1)) {
        ivr::set_error("ivr_loss_finalize: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::launch<3>(finalize_kernel, 1, kFinThreads, 0, (cudaStream_t)stream, *t, loss, state, last_bad);
    return ivr::check_launch("finalize_kernel");
}
