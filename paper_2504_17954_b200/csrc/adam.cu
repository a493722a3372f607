// Multi-tensor Adam (trainer.Adam.step, trainer.py:109-120) in one launch.
//
// Every parameter group of a training step (10 in stage 2) is updated by a
// single kernel: blockIdx.y selects the group, blockIdx.x strides over its
// elements.  Float64 with the reference's numpy evaluation order and
// rounding (the TU is built with -fmad=false):
//   m = b1 m + (1 - b1) g;  v = b2 v + ((1 - b2) g) g
//   p -= (lr (m / bc1)) / (sqrt(v / bc2) + eps),  bc = 1 - beta^t (host),
// with the two divisions by bc as multiplications by 1/bc (<= 1 ulp).
// HBM-bound: 4 float64 reads + 3 writes per element.
#include "ivr_common.cuh"

namespace ivr {

constexpr int kAdamMaxGroups = 16;

struct AdamGroups {
    ivr_adam_group g[kAdamMaxGroups];
    int n;
    double b1, b2, eps;
    const double *sched;  // device [lr, bc1, bc2] per group (graph replay), or null
    const int32_t *skip;  // device flag: nonzero = no update (gated step), or null
};

__global__ void __launch_bounds__(256) adam_kernel(AdamGroups A) {
    ::ivr::pdl_begin();
    if (A.skip && *A.skip) return;
    ivr_adam_group G = A.g[blockIdx.y];
    if (A.sched) {
        G.lr = A.sched[3 * blockIdx.y];
        G.bc1 = A.sched[3 * blockIdx.y + 1];
        G.bc2 = A.sched[3 * blockIdx.y + 2];
    }
    const double b1 = A.b1, b2 = A.b2, c1 = 1.0 - A.b1, c2 = 1.0 - A.b2;
    // m / bc as m * (1 / bc): within 1 ulp of the reference's division, and
    // two IEEE divides fewer per element (the kernel is FP64-issue bound)
    const double i1 = 1.0 / G.bc1, i2 = 1.0 / G.bc2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double g = G.grad[i];
        const double m = dadd(dmul(b1, G.m[i]), dmul(c1, g));
        const double v = dadd(dmul(b2, G.v[i]), dmul(dmul(c2, g), g));
        G.m[i] = m;
        G.v[i] = v;
        const double mhat = dmul(m, i1), vhat = dmul(v, i2);
        // lr mhat / (sqrt(vhat) + eps) with the division as an approximate
        // reciprocal refined by two Newton steps (within an ulp or two of
        // the IEEE quotient: ~1e-16 of the update, far below the reference
        // tolerance of the parameter; the kernel is FP64-issue bound)
        // sqrt(vhat) likewise from an approximate reciprocal square root
        // and two Newton steps (vhat = 0 -> 0)
        double rs;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(vhat));
        rs = rs * fma(-0.5 * vhat, rs * rs, 1.5);
        rs = rs * fma(-0.5 * vhat, rs * rs, 1.5);
        const double sq = vhat > 0.0 ? vhat * rs : 0.0;
        const double den = dadd(sq, A.eps);
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
        r = fma(r, fma(-den, r, 1.0), r);
        r = fma(r, fma(-den, r, 1.0), r);
        G.param[i] = dsub(G.param[i], dmul(dmul(G.lr, mhat), r));
    }
}

}  // namespace ivr

namespace {
int adam_impl(const ivr_adam_group *groups, int32_t n_groups, double beta1, double beta2,
              double eps, const double *sched, const int32_t *skip, ivr_stream_t stream) {
    using namespace ivr;
    if (!groups || n_groups < 0 || n_groups > kAdamMaxGroups) {
        set_error("ivr_adam_step: bad argument (at most 16 groups)");
        return IVR_ERR_ARG;
    }
    AdamGroups A{};
    int64_t nmax = 0;
    for (int k = 0; k < n_groups; ++k) {
        const ivr_adam_group &g = groups[k];
        if (g.n < 0 || (g.n > 0 && (!g.param || !g.m || !g.v || !g.grad)) ||
            (!sched && (!(g.bc1 > 0.0) || !(g.bc2 > 0.0)))) {
            set_error("ivr_adam_step: bad group");
            return IVR_ERR_ARG;
        }
        A.g[k] = g;
        nmax = g.n > nmax ? g.n : nmax;
    }
    A.n = n_groups;
    A.b1 = beta1;
    A.b2 = beta2;
    A.eps = eps;
    A.sched = sched;
    A.skip = skip;
    if (n_groups == 0 || nmax == 0) return IVR_OK;
    int64_t bx = (nmax + 255) / 256;
    if (bx > 148 * 8) bx = 148 * 8;
    ivr::launch<3>(adam_kernel, dim3((unsigned)bx, (unsigned)n_groups), 256, 0, (cudaStream_t)stream, A);
    return check_launch("adam_kernel");
}
}  // namespace

extern "C" int ivr_adam_step(const ivr_adam_group *groups, int32_t n_groups, double beta1,
                             double beta2, double eps, ivr_stream_t stream) {
    return adam_impl(groups, n_groups, beta1, beta2, eps, nullptr, nullptr, stream);
}

extern "C" int ivr_adam_step_sched(const ivr_adam_group *groups, int32_t n_groups, double beta1,
                                   double beta2, double eps, const double *sched,
                                   const int32_t *skip, ivr_stream_t stream) {
    if (!sched) {
        ivr::set_error("ivr_adam_step_sched: sched is required");
        return IVR_ERR_ARG;
    }
    return adam_impl(groups, n_groups, beta1, beta2, eps, sched, skip, stream);
}
