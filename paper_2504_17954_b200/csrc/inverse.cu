// Device-side transform step of the inverse exploration loop
// (inverse.optimize_to_reference, inverse.py:205-244), so that whole
// iterations -- render, loss, backward, Adam, parameter refresh -- replay as
// one CUDA graph with no host round trip per iteration.
//
//  * ivr_inverse_pack (per view): the view's photometric loss from the
//    fused L1 + SSIM sums (losses.py:118-138, default weights), its packed
//    gradient [d_c_p (3S), d_scale * sigmoid(opacity_raw) (S), d_lam (4),
//    d_b (4), d_polar, d_azimuth (orbital only)] (inverse.py:161-190)
//    accumulated over views, and the pair-capacity overflow flag.
//  * ivr_inverse_update (per iteration): mean over views, the loss record,
//    the reference's per-group Adam with the 1e-12 gradient floor
//    (inverse.py:229-238; trainer.Adam, trainer.py:109-120), then the frame
//    tables every view reads next iteration: palettes, softplus opacity
//    scales and the rescale flag (scene.py:214-220), lam, b, the orbital
//    light direction and its angle derivatives.
// An overflowed or non-finite iteration gates every later update (sticky)
// and records its index, so the host can grow the capacity and resume from
// it, or raise DivergedLoss at it.  Single thread: the state is 4S+10 floats.
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {
namespace invk {

__global__ void pack_kernel(ivr_inverse_step A, const double *photo_sums, double numel,
                            double windows, const double *d_c_p, const double *d_scale,
                            const double *d_globals, const int32_t *n_pairs, int64_t capacity) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int S = A.n_scenes;
    double *g = A.grad;
    // photometric_loss with LossWeights() defaults (l1 0.8, ssim 0.2)
    const double l1 = dmul(0.8, ddiv(photo_sums[1], numel));
    const double loss = dadd(l1, dmul(0.2, dsub(1.0, ddiv(photo_sums[0], windows))));
    *A.loss_sum = dadd(*A.loss_sum, loss);
    for (int k = 0; k < 3 * S; ++k) g[k] = dadd(g[k], d_c_p[k]);
    for (int s = 0; s < S; ++s)
        g[3 * S + s] = dadd(g[3 * S + s], dmul(d_scale[s], sigmoid_ref(A.x[3 * S + s])));
    for (int k = 0; k < 8; ++k) g[4 * S + k] = dadd(g[4 * S + k], d_globals[k]);
    if (A.orbital)
        for (int k = 8; k < 10; ++k) g[4 * S + k] = dadd(g[4 * S + k], d_globals[k]);
    if ((int64_t)*n_pairs > capacity) A.ctl[2] |= IVR_INV_OVERFLOW;
}

__device__ double softplus_d(double x) {  // np.logaddexp(0, x)
    return dadd(x > 0.0 ? x : 0.0, log1p(exp(-fabs(x))));
}

__global__ void update_kernel(ivr_inverse_step A) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int S = A.n_scenes, N = 4 * S + 10;
    int64_t *ctl = A.ctl;  // [iteration, first gated iteration, reason bits]
    const int64_t it = ctl[0];
    const double nv = (double)A.n_views;
    const double loss = ddiv(*A.loss_sum, nv);
    bool gate = ctl[1] >= 0;
    if (!gate) {
        if (!isfinite(loss)) ctl[2] |= IVR_INV_DIVERGED;
        if (ctl[2] != 0) {
            ctl[1] = it;
            gate = true;
        }
    }
    if (it < A.iters) A.losses[it] = loss;
    if (!gate) {
        double *x = A.x;
        // groups: c_p, opacity_raw, lam, b, angles (inverse.py:229-238)
        const int off[5] = {0, 3 * S, 4 * S, 4 * S + 4, 4 * S + 8};
        const int len[5] = {3 * S, S, 4, 4, 2};
        for (int q = 0; q < 5; ++q) {
            if (!(A.learnable & (1 << q))) continue;
            if (q == 4 && !A.orbital) continue;
            double gmax = 0.0;
            for (int k = 0; k < len[q]; ++k) {
                const double gk = fabs(ddiv(A.grad[off[q] + k], nv));
                gmax = gk > gmax ? gk : gmax;
            }
            if (!(gmax > 1e-12)) continue;
            const int64_t t = ++A.t[q];
            const double bc1 = dsub(1.0, pow(A.beta1, (double)t));
            const double bc2 = dsub(1.0, pow(A.beta2, (double)t));
            for (int k = 0; k < len[q]; ++k) {
                const int j = off[q] + k;
                const double gj = ddiv(A.grad[j], nv);
                const double m = dadd(dmul(A.beta1, A.m[j]), dmul(dsub(1.0, A.beta1), gj));
                const double v = dadd(dmul(A.beta2, A.v[j]), dmul(dmul(dsub(1.0, A.beta2), gj), gj));
                A.m[j] = m;
                A.v[j] = v;
                const double mhat = ddiv(m, bc1), vhat = ddiv(v, bc2);
                x[j] = dsub(x[j], ddiv(dmul(A.lr, mhat), dadd(sqrt(vhat), A.eps)));
            }
        }
        // frame tables for the next iteration
        bool rescale = false;
        for (int k = 0; k < 3 * S; ++k) A.tab[k] = x[k];
        for (int s = 0; s < S; ++s) {
            const double sc = softplus_d(x[3 * S + s]);
            A.tab[3 * S + s] = sc;
            rescale = rescale || sc != 1.0;
        }
        const double p = x[4 * S + 8], a = x[4 * S + 9];
        const double cp = cos(p), sp = sin(p), ca = cos(a), sa = sin(a);
        for (int v = 0; v < A.n_views; ++v) {
            ivr_frame_params &P = A.params[v];
            for (int k = 0; k < 4; ++k) {
                P.lam[k] = x[4 * S + k];
                P.b[k] = x[4 * S + 4 + k];
            }
            P.rescale_opacity = rescale ? 1 : 0;
            if (A.orbital) {
                P.light_dir[0] = dmul(cp, ca);
                P.light_dir[1] = dmul(cp, sa);
                P.light_dir[2] = sp;
                P.dl_dp[0] = dmul(-sp, ca);
                P.dl_dp[1] = dmul(-sp, sa);
                P.dl_dp[2] = cp;
                P.dl_da[0] = dmul(-cp, sa);
                P.dl_da[1] = dmul(cp, ca);
                P.dl_da[2] = 0.0;
            }
        }
    }
    for (int j = 0; j < N; ++j) A.grad[j] = 0.0;
    *A.loss_sum = 0.0;
    ctl[0] = it + 1;
}

}  // namespace invk
}  // namespace ivr

namespace {
bool bad_state(const ivr_inverse_step *a) {
    return !a || a->n_scenes < 1 || a->n_views < 1 || !a->x || !a->m || !a->v || !a->t ||
           !a->grad || !a->loss_sum || !a->losses || !a->ctl || !a->params || !a->tab ||
           a->iters < 1;
}
}  // namespace

extern "C" int ivr_inverse_pack(const ivr_inverse_step *a, const double *photo_sums, double numel,
                                double windows, const double *d_c_p, const double *d_scale,
                                const double *d_globals, const int32_t *n_pairs,
                                int64_t pair_capacity, ivr_stream_t stream) {
    if (bad_state(a) || !photo_sums || !d_c_p || !d_scale || !d_globals || !n_pairs ||
        !(numel > 0.0) || !(windows > 0.0)) {
        ivr::set_error("ivr_inverse_pack: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::invk::pack_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*a, photo_sums, numel, windows,
                                                               d_c_p, d_scale, d_globals, n_pairs,
                                                               pair_capacity);
    return ivr::check_launch("inverse pack_kernel");
}

extern "C" int ivr_inverse_update(const ivr_inverse_step *a, ivr_stream_t stream) {
    if (bad_state(a)) {
        ivr::set_error("ivr_inverse_update: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::invk::update_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*a);
    return ivr::check_launch("inverse update_kernel");
}
