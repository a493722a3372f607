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
// it, or raise DivergedLoss at it.
#include <math.h>

#include "ivr_common.cuh"

namespace ivr {
namespace invk {

// Both kernels run as one block whose threads own the state elements (the
// state is 4S+10 floats, S <= kMaxScenes): a single thread walking it would
// chain ~100 dependent global round trips (~25 us) onto every iteration.
constexpr int kThreads = 128;
constexpr int kMaxScenes = 1024;

__global__ void __launch_bounds__(kThreads)
pack_kernel(ivr_inverse_step A, const double *photo_sums, double numel, double windows,
            const double *d_c_p, const double *d_scale, const double *d_globals,
            const int32_t *n_pairs, int64_t capacity) {
    ::ivr::pdl_begin();
    const int S = A.n_scenes, N = 4 * S + 10;
    double *g = A.grad;
    for (int j = threadIdx.x; j < N; j += kThreads) {
        double v;
        if (j < 3 * S) v = d_c_p[j];
        else if (j < 4 * S) v = dmul(d_scale[j - 3 * S], sigmoid_ref(A.x[j]));
        else if (j < 4 * S + 8) v = d_globals[j - 4 * S];
        else v = A.orbital ? d_globals[j - 4 * S] : 0.0;
        g[j] = dadd(g[j], v);
    }
    if (threadIdx.x == 0) {
        // photometric_loss with LossWeights() defaults (l1 0.8, ssim 0.2)
        const double l1 = dmul(0.8, ddiv(photo_sums[1], numel));
        const double loss = dadd(l1, dmul(0.2, dsub(1.0, ddiv(photo_sums[0], windows))));
        *A.loss_sum = dadd(*A.loss_sum, loss);
        // overflow count next to the loss: all-reduced with the gradient when
        // views are sharded, so every rank gates the same iterations
        if ((int64_t)*n_pairs > capacity) A.loss_sum[1] = dadd(A.loss_sum[1], 1.0);
    }
}

__device__ double softplus_d(double x) {  // np.logaddexp(0, x)
    return dadd(x > 0.0 ? x : 0.0, log1p(exp(-fabs(x))));
}

__global__ void __launch_bounds__(kThreads) update_kernel(ivr_inverse_step A) {
    ::ivr::pdl_begin();
    const int S = A.n_scenes, N = 4 * S + 10;
    const int tid = threadIdx.x;
    __shared__ double s_g[4 * kMaxScenes + 10];
    __shared__ double s_max[5][kThreads / 32];
    __shared__ double s_bc[5][2];  // per group: 1 - beta^t (0 = group not stepped)
    __shared__ int s_gate, s_rescale;
    const double nv = A.view_div > 0.0 ? A.view_div : (double)A.n_views;
    // groups: c_p, opacity_raw, lam, b, angles (inverse.py:229-238)
    auto group = [S](int j) {
        return j < 3 * S ? 0 : (j < 4 * S ? 1 : (j < 4 * S + 4 ? 2 : (j < 4 * S + 8 ? 3 : 4)));
    };
    double mx[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int j = tid; j < N; j += kThreads) {
        const double gj = ddiv(A.grad[j], nv);
        s_g[j] = gj;
        const int q = group(j);
        mx[q] = fabs(gj) > mx[q] ? fabs(gj) : mx[q];
    }
    for (int q = 0; q < 5; ++q) {  // per-warp max, then 4 entries per group below
        double m = mx[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, m, o);
            m = y > m ? y : m;
        }
        if ((tid & 31) == 0) s_max[q][tid >> 5] = m;
    }
    if (tid == 0) s_rescale = 0;
    __syncthreads();
    if (tid == 0) {
        int64_t *ctl = A.ctl;  // [iteration, first gated iteration, reason bits]
        const int64_t it = ctl[0];
        const double loss = ddiv(*A.loss_sum, nv);
        bool gate = ctl[1] >= 0;
        if (A.loss_sum[1] > 0.0) ctl[2] |= IVR_INV_OVERFLOW;
        if (!gate) {
            if (!isfinite(loss)) ctl[2] |= IVR_INV_DIVERGED;
            if (ctl[2] != 0) {
                ctl[1] = it;
                gate = true;
            }
        }
        if (it < A.iters) A.losses[it] = loss;
        for (int q = 0; q < 5; ++q) {
            double gm = 0.0;
            for (int k = 0; k < kThreads / 32; ++k) gm = s_max[q][k] > gm ? s_max[q][k] : gm;
            s_bc[q][0] = s_bc[q][1] = 0.0;
            const bool learn = (A.learnable & (1 << q)) && (q != 4 || A.orbital);
            if (gate || !learn || !(gm > 1e-12)) continue;
            const int64_t t = ++A.t[q];
            s_bc[q][0] = dsub(1.0, pow(A.beta1, (double)t));
            s_bc[q][1] = dsub(1.0, pow(A.beta2, (double)t));
        }
        s_gate = gate ? 1 : 0;
        ctl[0] = it + 1;
        A.loss_sum[0] = 0.0;
        A.loss_sum[1] = 0.0;
    }
    __syncthreads();
    if (s_gate) {
        for (int j = tid; j < N; j += kThreads) A.grad[j] = 0.0;
        return;
    }
    double *x = A.x;
    for (int j = tid; j < N; j += kThreads) {
        const int q = group(j);
        const double bc1 = s_bc[q][0], bc2 = s_bc[q][1];
        double xj = x[j];
        if (bc1 != 0.0) {
            const double gj = s_g[j];
            const double m = dadd(dmul(A.beta1, A.m[j]), dmul(dsub(1.0, A.beta1), gj));
            const double v = dadd(dmul(A.beta2, A.v[j]), dmul(dmul(dsub(1.0, A.beta2), gj), gj));
            A.m[j] = m;
            A.v[j] = v;
            const double mhat = ddiv(m, bc1), vhat = ddiv(v, bc2);
            xj = dsub(xj, ddiv(dmul(A.lr, mhat), dadd(sqrt(vhat), A.eps)));
            x[j] = xj;
        }
        A.grad[j] = 0.0;
        // frame tables for the next iteration
        if (j < 3 * S) {
            A.tab[j] = xj;
        } else if (j < 4 * S) {
            const double sc = softplus_d(xj);
            A.tab[j] = sc;
            if (sc != 1.0) atomicOr(&s_rescale, 1);
        }
        s_g[j] = xj;  // updated parameters for the frame params below
    }
    __syncthreads();
    const double p = s_g[4 * S + 8], a = s_g[4 * S + 9];
    for (int v = tid; v < A.n_views; v += kThreads) {
        ivr_frame_params &P = A.params[v];
        for (int k = 0; k < 4; ++k) {
            P.lam[k] = s_g[4 * S + k];
            P.b[k] = s_g[4 * S + 4 + k];
        }
        P.rescale_opacity = s_rescale;
        if (A.orbital) {
            const double cp = cos(p), sp = sin(p), ca = cos(a), sa = sin(a);
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

}  // namespace invk
}  // namespace ivr

namespace {
// n_views may be 0 on a rank that holds no view of a sharded fit (it only
// joins the all-reduce and applies the update; view_div > 0 then)
bool bad_state(const ivr_inverse_step *a) {
    return !a || a->n_scenes < 1 || a->n_scenes > ivr::invk::kMaxScenes || a->n_views < 0 ||
           (a->n_views == 0 && !(a->view_div > 0.0)) ||
           !a->x || !a->m || !a->v || !a->t || !a->grad || !a->loss_sum || !a->losses || !a->ctl || !a->params || !a->tab ||
           a->iters < 1;
}
}  // namespace

extern "C" int ivr_inverse_pack(const ivr_inverse_step *a, const double *photo_sums, double numel,
                                double windows, const double *d_c_p, const double *d_scale,
                                const double *d_globals, const int32_t *n_pairs,
                                int64_t pair_capacity, ivr_stream_t stream) {
    if (bad_state(a) || a->n_views < 1 || !photo_sums || !d_c_p || !d_scale || !d_globals || !n_pairs ||
        !(numel > 0.0) || !(windows > 0.0)) {
        ivr::set_error("ivr_inverse_pack: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::invk::pack_kernel<<<1, ivr::invk::kThreads, 0, (cudaStream_t)stream>>>(*a, photo_sums, numel, windows,
                                                               d_c_p, d_scale, d_globals, n_pairs,
                                                               pair_capacity);
    return ivr::check_launch("inverse pack_kernel");
}

extern "C" int ivr_inverse_update(const ivr_inverse_step *a, ivr_stream_t stream) {
    if (bad_state(a)) {
        ivr::set_error("ivr_inverse_update: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::invk::update_kernel<<<1, ivr::invk::kThreads, 0, (cudaStream_t)stream>>>(*a);
    return ivr::check_launch("inverse update_kernel");
}
