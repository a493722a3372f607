/*
 * TEST INFRASTRUCTURE ONLY -- never linked into the product path.
 *
 * Plain-C restatement of the reference's numba tile compositor
 * (/root/reference/pkg/src/voxsplat/_kernels.py).  It exists so that the
 * parity tests and the bench's CPU-baseline leg have a fast, exact CPU
 * checker on machines where the reference package is absent.
 *
 * Arithmetic contract (verified against the numba machine code, see
 * DESIGN.md "oracle"): every operation is a separately rounded IEEE double
 * op (numba emits no FMA for these loops), exp() is glibc's (numba calls the
 * libm `exp` symbol), and in float32 mode the running pixel sum is rounded to
 * float after every accumulation because the reference accumulates into a
 * float32 array (`out[py, px, k] += w * values[sp, k]`, _kernels.py:64).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* _kernels.py:14-16 */
static const double ORC_ALPHA_CAP = 0.99;
static const double ORC_ALPHA_SKIP = 1.0 / 255.0;
static const double ORC_T_STOP = 1e-4;

int orc_abi_version(void) { return 1; }

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Gaussian exponent exactly as _kernels.py:51-54 evaluates it. */
static inline double orc_sigma(const double *conic, double dx, double dy) {
    double t0 = conic[0] * dx;
    t0 = t0 * dx;
    double t2 = conic[2] * dy;
    t2 = t2 * dy;
    double q = 0.5 * (t0 + t2);
    double t1 = conic[1] * dx;
    t1 = t1 * dy;
    return q + t1;
}

/*
 * composite_forward  (_kernels.py:31-72)
 *  tile_ranges (ntiles+1) int64, pair_splat (P) int64,
 *  mean2d (N,2), conic (N,3), opacity (N), values (N,nch): doubles holding the
 *  kernel inputs (float32-rounded values promoted exactly in float32 mode),
 *  out (H,W,nch) zero-initialised, contrib (H,W), last_pos (H,W), t_final (H,W).
 */
void orc_composite_forward(const int64_t *tile_ranges, int64_t ntiles,
                           const int64_t *pair_splat, const double *mean2d,
                           const double *conic, const double *opacity,
                           const double *values, int64_t nch, int64_t width,
                           int64_t height, int64_t tile_size, int64_t ntx,
                           int round_f32, double *out, int32_t *contrib,
                           int64_t *last_pos, double *t_final, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t tile = 0; tile < ntiles; ++tile) {
        const int64_t s0 = tile_ranges[tile], s1 = tile_ranges[tile + 1];
        const int64_t tx = tile % ntx, ty = tile / ntx;
        const int64_t x1 = (tx + 1) * tile_size < width ? (tx + 1) * tile_size : width;
        const int64_t y1 = (ty + 1) * tile_size < height ? (ty + 1) * tile_size : height;
        for (int64_t py = ty * tile_size; py < y1; ++py) {
            for (int64_t px = tx * tile_size; px < x1; ++px) {
                double T = 1.0;
                int64_t last = s0;
                int32_t nc = 0;
                double *o = out + (py * width + px) * nch;
                for (int64_t j = s0; j < s1; ++j) {
                    const int64_t sp = pair_splat[j];
                    const double dx = (double)px - mean2d[2 * sp];
                    const double dy = (double)py - mean2d[2 * sp + 1];
                    const double sigma = orc_sigma(conic + 3 * sp, dx, dy);
                    if (sigma < 0.0) continue;
                    double alpha = opacity[sp] * exp(-sigma);
                    if (alpha > ORC_ALPHA_CAP) alpha = ORC_ALPHA_CAP;
                    if (alpha < ORC_ALPHA_SKIP) continue;
                    const double w = T * alpha;
                    const double *v = values + sp * nch;
                    for (int64_t k = 0; k < nch; ++k) {
                        double acc = o[k] + w * v[k];
                        o[k] = round_f32 ? (double)(float)acc : acc;
                    }
                    T *= 1.0 - alpha;
                    nc += 1;
                    last = j + 1;
                    if (T < ORC_T_STOP) break;
                }
                contrib[py * width + px] = nc;
                last_pos[py * width + px] = last;
                t_final[py * width + px] = T;
            }
        }
    }
}

/*
 * composite_backward  (_kernels.py:75-135): back-to-front replay with
 * transmittance recovered by division; gradients land in per-pair slots.
 */
void orc_composite_backward(const int64_t *tile_ranges, int64_t ntiles,
                            const int64_t *pair_splat, const double *mean2d,
                            const double *conic, const double *opacity,
                            const double *values, int64_t nch, int64_t width,
                            int64_t height, int64_t tile_size, int64_t ntx,
                            const double *d_out, const int64_t *last_pos,
                            const double *t_final, double *pair_dv,
                            double *pair_dmean, double *pair_dconic,
                            double *pair_dopac, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel
    {
        double *suffix = (double *)malloc(sizeof(double) * (size_t)(nch > 0 ? nch : 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t tile = 0; tile < ntiles; ++tile) {
            const int64_t s0 = tile_ranges[tile], s1 = tile_ranges[tile + 1];
            if (s1 == s0) continue;
            const int64_t tx = tile % ntx, ty = tile / ntx;
            const int64_t x1 = (tx + 1) * tile_size < width ? (tx + 1) * tile_size : width;
            const int64_t y1 = (ty + 1) * tile_size < height ? (ty + 1) * tile_size : height;
            for (int64_t py = ty * tile_size; py < y1; ++py) {
                for (int64_t px = tx * tile_size; px < x1; ++px) {
                    const int64_t last = last_pos[py * width + px];
                    if (last <= s0) continue;
                    double T = t_final[py * width + px];
                    for (int64_t k = 0; k < nch; ++k) suffix[k] = 0.0;
                    const double *dout = d_out + (py * width + px) * nch;
                    for (int64_t j = last - 1; j >= s0; --j) {
                        const int64_t sp = pair_splat[j];
                        const double dx = (double)px - mean2d[2 * sp];
                        const double dy = (double)py - mean2d[2 * sp + 1];
                        const double *q = conic + 3 * sp;
                        const double sigma = orc_sigma(q, dx, dy);
                        if (sigma < 0.0) continue;
                        const double g = exp(-sigma);
                        const double alpha_u = opacity[sp] * g;
                        double alpha = alpha_u;
                        if (alpha > ORC_ALPHA_CAP) alpha = ORC_ALPHA_CAP;
                        if (alpha < ORC_ALPHA_SKIP) continue;
                        T = T / (1.0 - alpha);
                        const double w = T * alpha;
                        double d_alpha = 0.0;
                        const double *v = values + sp * nch;
                        for (int64_t k = 0; k < nch; ++k) {
                            const double dok = dout[k];
                            const double vk = v[k];
                            d_alpha += dok * (T * vk - suffix[k] / (1.0 - alpha));
                            pair_dv[j * nch + k] += dok * w;
                            suffix[k] += w * vk;
                        }
                        if (alpha_u < ORC_ALPHA_CAP) {
                            pair_dopac[j] += g * d_alpha;
                            const double d_sigma = -alpha_u * d_alpha;
                            pair_dconic[3 * j + 0] += 0.5 * dx * dx * d_sigma;
                            pair_dconic[3 * j + 1] += dx * dy * d_sigma;
                            pair_dconic[3 * j + 2] += 0.5 * dy * dy * d_sigma;
                            const double gx = q[0] * dx + q[1] * dy;
                            const double gy = q[1] * dx + q[2] * dy;
                            pair_dmean[2 * j + 0] += -d_sigma * gx;
                            pair_dmean[2 * j + 1] += -d_sigma * gy;
                        }
                    }
                }
            }
        }
        free(suffix);
    }
}

/*
 * VQ assignment (vq.py:90-96): index = searchsorted(mids, v, side='left'),
 * mids = 0.5*(c[1:]+c[:-1]); a NaN value sorts after every mid -> K-1.
 */
void orc_vq_assign(const double *values, int64_t n, const double *centroids,
                   int64_t k, int64_t *out, int nthreads) {
    set_threads(nthreads);
    double *mids = (double *)malloc(sizeof(double) * (size_t)(k > 1 ? k - 1 : 1));
    for (int64_t i = 0; i + 1 < k; ++i) mids[i] = 0.5 * (centroids[i + 1] + centroids[i]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double v = values[i];
        if (k <= 1) { out[i] = 0; continue; }
        if (v != v) { out[i] = k - 1; continue; }
        int64_t lo = 0, hi = k - 1; /* first index with mids[idx] >= v */
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (mids[mid] < v) lo = mid + 1; else hi = mid;
        }
        out[i] = lo;
    }
    free(mids);
}
