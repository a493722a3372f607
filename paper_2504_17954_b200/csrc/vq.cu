// K5/K6 -- scalar-codebook VQ assign and decode (bandwidth kernels), and the
// k-means that builds the codebooks (K5s: k-means++ seeding, Lloyd steps).
//
// The reference's codebooks are 1-D (one scalar codebook per attribute,
// shared across components; vq.py:1-6, 137-147) and assignment is
// np.searchsorted over float64 centroid midpoints (vq.py:90-96).  Nearest
// codeword search in 1-D is a binary search, not a distance GEMM: there is no
// contraction dimension to put on tensor cores (SURVEY.md finding 5), so
// these kernels are HBM-bound (6 B per value in + out).  Midpoints live in
// shared memory (K=4096 -> 32 KB) next to a uniform bucket table that cuts
// the search to ~2 compares per value.
#include <cooperative_groups.h>

#include "ivr_common.cuh"

namespace ivr {

constexpr int kVqThreads = 256;
constexpr int kVqSmemMids = 4096;  // 32 KB of float64 midpoints (+16 KB bucket table)
constexpr int kLut = 8192;         // uniform buckets over [mid_0, mid_last]

__device__ __forceinline__ double vq_mid(const double *c, int i) { return 0.5 * (c[i + 1] + c[i]); }

// lut[b] = number of midpoints < lo + b * w  (b < kLut); params = {lo, w, inv_w,
// float32 buckets safe}
template <int NB = kLut>
__global__ void __launch_bounds__(kVqThreads)
vq_lut_kernel(const double *__restrict__ cents, int k, uint16_t *lut, double *params) {
    const int nm = k - 1;
    const double lo = vq_mid(cents, 0), hi = vq_mid(cents, nm - 1);
    const double w = (hi - lo) / NB;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        params[0] = lo;
        params[1] = w;
        params[2] = w > 0.0 ? 1.0 / w : 0.0;
        // 1 when the float32 bucket of any value inside [lo, hi] is within a
        // quarter bucket of its true bucket (|v| 2^-23 relative rounding of v,
        // lo and the product, over the bucket width): the [b-1, b+2) window
        // then provably holds the answer and the edge checks can be skipped
        const double mag = fmax(fabs(lo), fabs(hi));
        params[3] = (w > 0.0 && mag * 4.0 * 1.1920928955078125e-07 + w * 1e-6 < 0.25 * w) ? 1.0 : 0.0;
    }
    const int b = blockIdx.x * kVqThreads + threadIdx.x;
    if (b >= NB) return;
    const double e = lo + (double)b * w;
    int a = 0, z = nm;  // count of mids < e
    while (a < z) {
        const int m = (a + z) >> 1;
        if (vq_mid(cents, m) < e) a = m + 1;
        else z = m;
    }
    lut[b] = (uint16_t)a;
}

// searchsorted(mids, v, 'left') = number of mids < v.  A uniform bucket table
// narrows the interval to the mids between the edges of the neighbouring
// buckets (typically 0-3 mids); the answer is then checked against the
// interval ends with exact float64 compares and, if a rounding corner case
// put v outside the interval, recomputed by a full binary search.  Midpoints
// and the table live in shared memory.
__device__ __forceinline__ int vq_full_search(const double *mid, int nm, double v) {
    int a = 0, z = nm;
    while (a < z) {
        const int m = (a + z) >> 1;
        if (mid[m] < v) a = m + 1;
        else z = m;
    }
    return a;
}

template <bool SMEM>
__global__ void __launch_bounds__(kVqThreads)
vq_assign_kernel(const double *__restrict__ values, int64_t n, const double *__restrict__ cents,
                 int k, const uint16_t *__restrict__ lut, const double *__restrict__ params,
                 uint16_t *__restrict__ out) {
    __shared__ double s_mid[SMEM ? kVqSmemMids : 1];
    __shared__ uint16_t s_lut[SMEM ? kLut : 1];
    const int nm = k - 1;
    if (SMEM) {
        for (int i = threadIdx.x; i < nm; i += kVqThreads) s_mid[i] = vq_mid(cents, i);
        for (int i = threadIdx.x; i < kLut; i += kVqThreads) s_lut[i] = lut[i];
        __syncthreads();
    }
    const double lo = params[0], inv_w = params[2];
    const bool use_lut = SMEM && inv_w > 0.0;
    const bool exact_buckets = params[3] != 0.0;
    // the bucket index only narrows the search (every answer is verified
    // against exact float64 compares), so it is computed in float32
    const float lo_f = (float)lo, inv_w_f = (float)inv_w;
    constexpr int kVqIlp = 8;
    const int64_t chunk = (int64_t)kVqThreads * kVqIlp;
    for (int64_t base = (int64_t)blockIdx.x * chunk; base < n; base += (int64_t)gridDim.x * chunk) {
        double v[kVqIlp];
#pragma unroll
        for (int r = 0; r < kVqIlp; ++r) {
            const int64_t i = base + r * kVqThreads + threadIdx.x;
            v[r] = i < n ? __ldcs(values + i) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kVqIlp; ++r) {
            const int64_t i = base + r * kVqThreads + threadIdx.x;
            if (i >= n) continue;
            int pos;
            if (v[r] != v[r]) {
                pos = nm;  // NaN sorts last
            } else if (SMEM) {
                if (use_lut) {
                    const float t = ((float)v[r] - lo_f) * inv_w_f;
                    const int b = t < 0.0f ? 0 : (t >= (float)(kLut - 1) ? kLut - 1 : (int)t);
                    int a = b >= 1 ? s_lut[b - 1] : 0;
                    const int zi = b + 2 < kLut ? s_lut[b + 2] : nm;
                    int z = zi;
                    const int a0 = a;
                    while (a < z) {
                        const int m = (a + z) >> 1;
                        if (s_mid[m] < v[r]) a = m + 1;
                        else z = m;
                    }
                    pos = a;
                    // values outside [lo, hi] land in the clamped edge buckets,
                    // whose windows end at 0 / nm: no check needed there either
                    const bool inside = t >= 0.0f && t < (float)(kLut - 1);
                    if (!(exact_buckets && inside)) {
                        const bool ok_lo = pos > a0 || a0 == 0 || s_mid[a0 - 1] < v[r];
                        const bool ok_hi = pos < zi || zi == nm || !(s_mid[zi] < v[r]);
                        if (!(ok_lo && ok_hi)) pos = vq_full_search(s_mid, nm, v[r]);
                    }
                } else {
                    pos = vq_full_search(s_mid, nm, v[r]);
                }
            } else {
                int a = 0, z = nm;
                while (a < z) {
                    const int m = (a + z) >> 1;
                    if (0.5 * (__ldg(cents + m + 1) + __ldg(cents + m)) < v[r]) a = m + 1;
                    else z = m;
                }
                pos = a;
            }
            __stcs(out + i, (uint16_t)pos);
        }
    }
}

// Assign, windowed form (K - 1 <= kVqSmemMids, at least one midpoint): a
// 32768-bucket table (kLutWin) is widened in shared memory to one word per
// bucket holding its search window [lut[b - 1], lut[b + 2]), and the window
// is searched by two branch-free binary-lifting steps (windows of <= 3
// midpoints: all of the C5 attribute values; wider windows,
// and the corner cases the float32 bucket index can hit, take the verified
// full search).  A warp moves 256 contiguous values per step: four 16-byte
// loads and four 4-byte stores (two indices each) per lane.
constexpr int kWinSteps = 2;
constexpr int kLutWin = 32768;  // buckets of the windowed search (128 KB of windows)

template <int NB>
__device__ __forceinline__ int vq_pos_win(const double *mid, const uint32_t *win, int nm, double v,
                                          float lo_f, float inv_w_f, bool exact_buckets,
                                          bool use_lut, bool &ok) {
    const float t = ((float)v - lo_f) * inv_w_f;
    const float tc = fminf(fmaxf(t, 0.0f), (float)(NB - 1));  // NaN -> 0 (handled by the caller)
    const uint32_t w = win[(int)tc];
    const int a0 = (int)(w & 0xffffu), zi = (int)(w >> 16);
    int pos = a0;
#pragma unroll
    for (int s = kWinSteps - 1; s >= 0; --s) {
        const int m = pos + (1 << s) - 1;
        const bool in = m < zi;
        const double x = mid[in ? m : 0];
        if (in && x < v) pos = m + 1;
    }
    ok = use_lut && zi - a0 < (1 << kWinSteps);
    const bool inside = t >= 0.0f && t < (float)(NB - 1);
    if (ok && !(exact_buckets && inside)) {
        const bool ok_lo = pos > a0 || a0 == 0 || mid[a0 - 1] < v;
        const bool ok_hi = pos < zi || zi == nm || !(mid[zi] < v);
        ok = ok_lo && ok_hi;
    }
    return pos;
}

constexpr int kWinThreads = 1024;  // one 32-warp CTA per SM under the 160 KB of tables
constexpr int kWinR = 2;          // 16-byte value loads per lane per step
constexpr int kWinTile = 64 * kWinR;  // values per warp per step

template <int NB>
__global__ void __launch_bounds__(kWinThreads, 1)
vq_assign_win_kernel(const double *__restrict__ values, int64_t n, const double *__restrict__ cents,
                     int k, const uint16_t *__restrict__ lut, const double *__restrict__ params,
                     uint16_t *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char sm_w[];
    double *s_mid = reinterpret_cast<double *>(sm_w);
    uint32_t *s_win = reinterpret_cast<uint32_t *>(s_mid + kVqSmemMids);
    const int nm = k - 1;
    for (int i = threadIdx.x; i < nm; i += kWinThreads) s_mid[i] = vq_mid(cents, i);
    for (int b = threadIdx.x; b < NB; b += kWinThreads) {
        const uint32_t a = b >= 1 ? lut[b - 1] : 0u;
        const uint32_t z = b + 2 < NB ? lut[b + 2] : (uint32_t)nm;
        s_win[b] = a | (z << 16);
    }
    __syncthreads();
    const double lo = params[0], inv_w = params[2];
    const bool use_lut = inv_w > 0.0;
    const bool exact_buckets = params[3] != 0.0;
    const float lo_f = (float)lo, inv_w_f = (float)inv_w;
    const int lane = threadIdx.x & 31;
    constexpr int kWarpsPerCta = kWinThreads / 32;
    const int64_t gw = (int64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
    const int64_t step = (int64_t)gridDim.x * kWarpsPerCta * kWinTile;
    // the next tile's values are loaded before this tile is searched
    auto load = [&](int64_t t, double2 *v) {
        if (t + kWinTile <= n) {
#pragma unroll
            for (int r = 0; r < kWinR; ++r)
                v[r] = __ldcs(reinterpret_cast<const double2 *>(values + t + 64 * r + 2 * lane));
        }
    };
    double2 nxt[kWinR];
    load(gw * kWinTile, nxt);
    for (int64_t tile = gw * kWinTile; tile < n; tile += step) {
        if (tile + kWinTile <= n) {
            double2 v[kWinR];
#pragma unroll
            for (int r = 0; r < kWinR; ++r) v[r] = nxt[r];
            load(tile + step, nxt);
            // every window search first (independent chains overlap), the rare
            // verified full searches after
            int p[2 * kWinR];
            bool ok[2 * kWinR];
#pragma unroll
            for (int r = 0; r < kWinR; ++r) {
                p[2 * r] = vq_pos_win<NB>(s_mid, s_win, nm, v[r].x, lo_f, inv_w_f, exact_buckets,
                                          use_lut, ok[2 * r]);
                p[2 * r + 1] = vq_pos_win<NB>(s_mid, s_win, nm, v[r].y, lo_f, inv_w_f, exact_buckets,
                                              use_lut, ok[2 * r + 1]);
            }
#pragma unroll
            for (int q = 0; q < 2 * kWinR; ++q) {
                const double x = (q & 1) ? v[q >> 1].y : v[q >> 1].x;
                if (!ok[q]) p[q] = vq_full_search(s_mid, nm, x);
                if (x != x) p[q] = nm;  // NaN sorts last
            }
#pragma unroll
            for (int r = 0; r < kWinR; ++r)
                __stcs(reinterpret_cast<uint32_t *>(out + tile + 64 * r + 2 * lane),
                       (uint32_t)p[2 * r] | ((uint32_t)p[2 * r + 1] << 16));
        } else {
            for (int j = 0; j < 2 * kWinR; ++j) {
                const int64_t i = tile + 64 * (j >> 1) + 2 * lane + (j & 1);
                if (i >= n) continue;
                const double x = values[i];
                bool okq;
                int p = vq_pos_win<NB>(s_mid, s_win, nm, x, lo_f, inv_w_f, exact_buckets, use_lut, okq);
                if (!okq) p = vq_full_search(s_mid, nm, x);
                if (x != x) p = nm;
                out[i] = (uint16_t)p;
            }
        }
    }
}

// 8 indices per thread per step: one 16-byte load, four 16-byte stores; the
// codebook is gathered from shared memory (K <= kVqSmemMids + 1)
template <bool SMEM>
__global__ void __launch_bounds__(kVqThreads)
vq_decode_kernel(const uint16_t *__restrict__ idx, int64_t n, const double *__restrict__ cents,
                 int k, double *__restrict__ out, long long *bad) {
    __shared__ double s_c[SMEM ? kVqSmemMids + 1 : 1];
    if (SMEM) {
        for (int i = threadIdx.x; i < k; i += kVqThreads) s_c[i] = cents[i];
        __syncthreads();
    }
    const double *tab = SMEM ? s_c : cents;
    const int64_t nv = n / 8;
    const bool aligned = ((reinterpret_cast<uintptr_t>(idx) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    const int64_t stride = (int64_t)gridDim.x * kVqThreads;
    int worst = -1;
    if (aligned) {
        // a warp decodes 256 contiguous indices per step; every load and
        // store instruction covers one contiguous span (128 B of indices,
        // 512 B of values), lane l holding entries 64 p + 2 l and + 1
        const int lane = threadIdx.x & 31;
        const int64_t nw = nv / 32;  // whole 256-index tiles
        const int64_t wstride = stride / 32;
        for (int64_t tw = ((int64_t)blockIdx.x * kVqThreads + threadIdx.x) / 32; tw < nw; tw += wstride) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(idx + 256 * tw) + lane;
            double2 *o = reinterpret_cast<double2 *>(out + 256 * tw) + lane;
            uint32_t w[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) w[p] = __ldcs(src + 32 * p);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int j0 = (int)(w[p] & 0xffffu), j1 = (int)(w[p] >> 16);
                if (j0 >= k) worst = max(worst, j0);
                if (j1 >= k) worst = max(worst, j1);
                const double d0 = j0 < k ? tab[j0] : 0.0;
                const double d1 = j1 < k ? tab[j1] : 0.0;
                __stcs(o + 32 * p, make_double2(d0, d1));
            }
        }
    }
    for (int64_t i = (aligned ? 256 * (nv / 32) : 0) + (int64_t)blockIdx.x * kVqThreads + threadIdx.x;
         i < n; i += stride) {
        const int j = idx[i];
        if (j >= k) worst = max(worst, j);
        out[i] = j < k ? tab[j] : 0.0;
    }
    if (worst >= 0) atomicMax(bad, (long long)worst);
}

// decode is a store stream: measured best with 2 CTAs per SM (148 x {1, 2, 3,
// 4, 7}: 0.195, 0.149, 0.153, 0.160, 0.235 ms for 60M values)
static int grid_for_decode(int64_t n) {
    int64_t b = (n / 8 + kVqThreads - 1) / kVqThreads;
    const int64_t cap = 148 * 4;  // 2 -> 4 CTAs per SM: 128 -> 111 us at C5 (more stores in flight)
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

static int grid_for(int64_t n) {
    // persistent-style grid: ~4 CTAs per SM, each staging its tables once
    int64_t b = (n + kVqThreads - 1) / kVqThreads;
    const int64_t cap = 148 * 4;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace ivr

namespace ivr {

// Fused Lloyd step: assign (as K5) + per-centroid sums / counts privatised in
// shared memory (float64 sums, u32 counts), flushed with one global atomic per
// centroid per CTA.
__global__ void __launch_bounds__(kVqThreads)
lloyd_accum_kernel(const double *__restrict__ values, int64_t n, const double *__restrict__ cents,
                   int k, const uint16_t *__restrict__ lut, const double *__restrict__ params,
                   double *sums, unsigned long long *counts) {
    extern __shared__ __align__(16) double sm_l[];
    double *s_mid = sm_l;                                   // k - 1
    double *s_sum = s_mid + kVqSmemMids;                    // k
    unsigned int *s_cnt = reinterpret_cast<unsigned int *>(s_sum + kVqSmemMids + 1);  // k
    uint16_t *s_lut = reinterpret_cast<uint16_t *>(s_cnt + kVqSmemMids + 1);        // kLut
    const int nm = k - 1;
    for (int i = threadIdx.x; i < nm; i += kVqThreads) s_mid[i] = vq_mid(cents, i);
    for (int i = threadIdx.x; i < k; i += kVqThreads) {
        s_sum[i] = 0.0;
        s_cnt[i] = 0u;
    }
    for (int i = threadIdx.x; i < kLut; i += kVqThreads) s_lut[i] = lut[i];
    __syncthreads();
    const double lo = params[0], inv_w = params[2];
    const float lo_f = (float)lo, inv_w_f = (float)inv_w;
    for (int64_t i = (int64_t)blockIdx.x * kVqThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kVqThreads) {
        const double v = values[i];
        int pos;
        if (v != v) {
            pos = nm;
        } else if (inv_w > 0.0) {
            const float t = ((float)v - lo_f) * inv_w_f;
            const int b = t < 0.0f ? 0 : (t >= (float)(kLut - 1) ? kLut - 1 : (int)t);
            int a = b >= 1 ? s_lut[b - 1] : 0;
            const int zi = b + 2 < kLut ? s_lut[b + 2] : nm;
            int z = zi;
            const int a0 = a;
            while (a < z) {
                const int m = (a + z) >> 1;
                if (s_mid[m] < v) a = m + 1;
                else z = m;
            }
            pos = a;
            const bool ok_lo = pos > a0 || a0 == 0 || s_mid[a0 - 1] < v;
            const bool ok_hi = pos < zi || zi == nm || !(s_mid[zi] < v);
            if (!(ok_lo && ok_hi)) pos = vq_full_search(s_mid, nm, v);
        } else {
            pos = vq_full_search(s_mid, nm, v);
        }
        atomicAdd(&s_sum[pos], v);
        atomicAdd(&s_cnt[pos], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += kVqThreads) {
        if (s_cnt[i]) {
            atomicAdd(&sums[i], s_sum[i]);
            atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
        }
    }
}

// new = counts > 0 ? sums / counts : c (vq.py:81-83); shift[0] = max |new - c|
__global__ void __launch_bounds__(1024)
lloyd_finish_kernel(const double *cents, int k, const double *sums, const unsigned long long *counts,
                    double *out, double *shift) {
    __shared__ double s_red[32];
    double m = 0.0;
    for (int i = threadIdx.x; i < k; i += 1024) {
        const double nw = counts[i] > 0 ? sums[i] / (double)counts[i] : cents[i];
        out[i] = nw;
        m = fmax(m, fabs(nw - cents[i]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 32; ++w) t = fmax(t, s_red[w]);
        *shift = t;
    }
}

// Lloyd step on the values in sorted order (vq.py:75-87) for `sets` centroid
// sets at once (k-means' restarts): bucket b (searchsorted on the float64
// midpoints, as K5) is the contiguous range xs[bnd[b], bnd[b + 1]) with
// bnd[b] = #{xs <= mid[b - 1]}, so the per-centroid sums are segment sums --
// one CTA per bucket, fixed tree order, no atomics -- instead of a scatter
// of float64 atomics (a CAS loop per value in shared memory).  Sums run in
// value order rather than np.bincount's index order (same float64 sums up to
// rounding, as the atomic form).
constexpr int kLlThreads = 256;

__global__ void __launch_bounds__(kLlThreads)
lloyd_bounds_kernel(const double *__restrict__ xs, int64_t n, const double *__restrict__ cents,
                    int k, int64_t *bnd, unsigned long long *shift) {
    const int r = blockIdx.y;
    const double *c = cents + (int64_t)r * k;
    int64_t *b = bnd + (int64_t)r * (k + 1);
    const int i = blockIdx.x * kLlThreads + threadIdx.x;  // boundary i + 1 (mid i)
    if (i == 0) {
        b[0] = 0;
        b[k] = n;
        shift[r] = 0ull;
    }
    if (i >= k - 1) return;
    const double m = vq_mid(c, i);
    int64_t lo = 0, hi = n;  // first position with xs > m (NaN sorts last, never <= m)
    while (lo < hi) {
        const int64_t md = (lo + hi) >> 1;
        if (__ldg(xs + md) <= m) lo = md + 1;
        else hi = md;
    }
    b[i + 1] = lo;
}

__global__ void __launch_bounds__(kLlThreads)
lloyd_segsum_kernel(const double *__restrict__ xs, const double *__restrict__ cents, int k,
                    const int64_t *__restrict__ bnd, double *out, unsigned long long *shift) {
    __shared__ double s_red[kLlThreads / 32];
    const int r = blockIdx.y, bk = blockIdx.x;
    const int64_t *b = bnd + (int64_t)r * (k + 1);
    const int64_t b0 = b[bk], b1 = b[bk + 1];
    double t = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kLlThreads) t += __ldg(xs + i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kLlThreads / 32; ++w) sum += s_red[w];
        const double old = cents[(int64_t)r * k + bk];
        const int64_t cnt = b1 - b0;
        const double nw = cnt > 0 ? sum / (double)cnt : old;  // vq.py:81-83
        out[(int64_t)r * k + bk] = nw;
        const double d = fabs(nw - old);  // max over the set: non-negative doubles order as bits
        atomicMax(shift + r, d == d ? (unsigned long long)__double_as_longlong(d)
                                    : 0x7ff8000000000000ull);
    }
}

// ----------------------------------------------------------------- k-means++
// vq._seed_plusplus (vq.py:60-72) with the reference's random stream: every
// step draws one uniform u (rng.choice(n, p = d2 / sum d2) == the first index
// whose cumulative d2 in INDEX order exceeds u * sum).  Per step two kernels:
// (A) d2 = min(d2, (x - c)^2) for the centre just chosen (d2 = (x - c0)^2 at
// the first step) with per-block partial sums in index order, (B) one block
// scans the block sums, finds the block holding u * sum and the index inside
// it, and writes the next centre.
constexpr int kSeedThreads = 256, kSeedItems = 8, kSeedChunk = kSeedThreads * kSeedItems;
constexpr int kPickThreads = 1024;

__global__ void __launch_bounds__(kSeedThreads)
seed_update_kernel(const double *x, int64_t n, double *d2, const double *center, int init,
                   double *bsum) {
    __shared__ double s_red[kSeedThreads / 32];
    const double c = *center;
    const int64_t base = (int64_t)blockIdx.x * kSeedChunk;
    double sum = 0.0;
#pragma unroll
    for (int r = 0; r < kSeedItems; ++r) {
        const int64_t i = base + r * kSeedThreads + threadIdx.x;
        if (i < n) {
            const double d = x[i] - c;
            const double v = init ? d * d : fmin(d2[i], d * d);
            d2[i] = v;
            sum += v;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kSeedThreads / 32; ++w) t += s_red[w];
        bsum[blockIdx.x] = t;
    }
}

// inclusive scan of one double per thread over the block (1024 threads)
__device__ __forceinline__ double block_scan_d(double v, double *s_w, double &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = s_w[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    if (warp > 0) v += s_w[warp - 1];
    total = s_w[31];
    __syncthreads();
    return v;
}

__global__ void __launch_bounds__(kPickThreads)
seed_pick_kernel(const double *x, int64_t n, const double *d2, const double *bsum, int nb,
                 const double *u, double *centers, int step) {
    __shared__ double s_w[32];
    __shared__ int s_blk, s_lastmass;
    __shared__ unsigned long long s_idx;
    const int tid = threadIdx.x;
    if (tid == 0) {
        s_blk = 0x7fffffff;
        s_lastmass = -1;
        s_idx = ~0ull;
    }
    // block sums: thread t owns the contiguous blocks [t * per, (t + 1) * per)
    const int per = (nb + kPickThreads - 1) / kPickThreads;
    const int b0 = tid * per, b1 = min(b0 + per, nb);
    double mine = 0.0;
    for (int b = b0; b < b1; ++b) mine += bsum[b];
    double tot;
    const double incl = block_scan_d(mine, s_w, tot);
    if (!(tot > 0.0)) {  // all mass on chosen centres: the reference repeats c0
        if (tid == 0) centers[step] = centers[0];
        return;
    }
    const double target = u[step - 1] * tot;
    double run = incl - mine;
    int last_pos = -1;  // last block with mass (rounding fallback)
    bool hit = false;
    for (int b = b0; b < b1; ++b) {
        const double v = bsum[b];
        if (v > 0.0) last_pos = b;
        if (!hit && run + v > target) {
            atomicMin(&s_blk, b);
            hit = true;
        }
        run += v;
    }
    if (last_pos >= 0) atomicMax(&s_lastmass, last_pos);
    __syncthreads();
    // u * tot at or above the rounded total: the last block with mass
    int blk = s_blk != 0x7fffffff ? s_blk : (s_lastmass >= 0 ? s_lastmass : nb - 1);
    // cumulative d2 before the block, then the index inside it
    double before = 0.0;
    {
        double part = 0.0;
        for (int b = b0; b < min(b1, blk); ++b) part += bsum[b];
        double t2;
        block_scan_d(part, s_w, t2);
        before = t2;
    }
    const int64_t e0 = (int64_t)blk * kSeedChunk;
    double v2[2];
    int64_t ix[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        ix[q] = e0 + 2 * tid + q;
        v2[q] = ix[q] < n ? d2[ix[q]] : 0.0;
    }
    double t3;
    const double inc2 = block_scan_d(v2[0] + v2[1], s_w, t3);
    double r2 = before + inc2 - (v2[0] + v2[1]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (ix[q] < n && r2 + v2[q] > target) {
            atomicMin(&s_idx, (unsigned long long)ix[q]);
            break;
        }
        r2 += v2[q];
    }
    __syncthreads();
    if (tid == 0) {
        int64_t j = (int64_t)s_idx;
        if (s_idx == ~0ull) {  // rounding: the block's last element with mass
            j = e0;
            for (int64_t q = min(e0 + kSeedChunk, n) - 1; q >= e0; --q)
                if (d2[q] > 0.0) {
                    j = q;
                    break;
                }
        }
        centers[step] = x[j];
    }
}

// ----------------------------------------------------------------- k-means++, sorted
// The same seeding in one persistent cooperative kernel that touches only the
// samples a new centre can change, for up to kSsMaxP independent seedings at
// once (k-means' restarts of every attribute: their draws do not depend on
// the data, so all of them are known before the first one runs).  Scalar
// k-means is 1-D: with the samples in value order (xs = x[order]), a centre c
// at sorted position p can only lower d2 for samples strictly between the
// chosen centres next to it (positions L < p < R); every other sample is at
// least as close to L or R, and fl((x - v)^2) is monotone in |x - v|, so
// np.minimum would keep its d2 bit for bit.  Per step: CTA r picks seeding
// r's centre from its block sums (d2 in INDEX order: 32 values per block, 64
// blocks per super-block) and publishes (index, L, R); the grid lowers d2
// over every seeding's (L, R), marking the lowered blocks; after a grid
// barrier one warp per marked super-block re-sums its marked blocks and the
// super-block (fixed order: bit-identical runs), and the CTAs arrive on a
// counter the picking CTAs wait for.  The samples updated per step fall off
// like n / i (~n ln k in all instead of n k); the step is a chain of
// dependent L2 round trips, which the seedings of one launch share.
namespace cg = cooperative_groups;

constexpr int kSsThreads = 512;
constexpr int kSsBlk = 32;      // d2 values per block sum
constexpr int kSsSup = 64;      // block sums per super-block sum
constexpr int kSsMaxK = 32768;  // chosen positions kept in shared memory
constexpr int kSsPer = 16;      // super-block sums per thread held in registers by the pick
constexpr int kSsMaxP = 64;     // seedings per launch (one picking CTA each)

struct SsProb {
    const double *x;
    const int32_t *order;
    int64_t n, nb1, first;
    int nb2;
    const double *u;  // k - 1 draws
    double *centers;  // k
    // workspace: values in sorted order, sorted position of each index, d2,
    // block sums, super-block sums, marked-block masks, two super-block lists
    // (step parity), their lengths, the published pick {j, L, R, step}
    double *xs;
    int32_t *rank;
    double *d2, *bs1, *bs2;
    unsigned long long *dmask;
    int32_t *dlist, *dcount;
    long long *ctl;
};

struct SeedSorted {
    int k, P;
    unsigned *arrive;
    unsigned long long *phase_ns;  // CTA 0's time per phase: pick, wait, update, barrier, re-sum, arrive
    SsProb pr[kSsMaxP];
};

__device__ __forceinline__ double warp_tree_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block sum: the 32 d2 values in index order, added sequentially (one thread)
__device__ __forceinline__ double ss_block_sum(const double *d2, int64_t n, int64_t blk) {
    const int64_t i0 = blk * kSsBlk;
    double t = 0.0;
    if (i0 + kSsBlk <= n) {
        const double2 *p = reinterpret_cast<const double2 *>(d2 + i0);
        double2 v[kSsBlk / 2];
#pragma unroll
        for (int q = 0; q < kSsBlk / 2; ++q) v[q] = __ldcg(p + q);
#pragma unroll
        for (int q = 0; q < kSsBlk / 2; ++q) {
            t += v[q].x;
            t += v[q].y;
        }
    } else {
        for (int64_t i = i0; i < n; ++i) t += __ldcg(d2 + i);
    }
    return t;
}

// inclusive scan over a CTA of kSsThreads threads
__device__ __forceinline__ double ss_block_scan(double v, double *s_w, double &total) {
    constexpr int kW = kSsThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = lane < kW ? s_w[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kW) s_w[lane] = w;
    }
    __syncthreads();
    if (warp > 0) v += s_w[warp - 1];
    total = s_w[kW - 1];
    __syncthreads();
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ long long ld_volatile_s64(const long long *p) {
    long long v;
    asm volatile("ld.volatile.global.s64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// CTA r's pick for seeding r at `step`: the first index whose cumulative d2
// (index order) exceeds u * sum d2, and its chosen neighbours L < p < R in
// value order (j = -1: all mass on chosen centres)
__device__ void ss_pick(const SsProb &Q, int step, int32_t *s_chosen, int nch, long long &j,
                        long long &L, long long &R) {
    __shared__ double s_w[32], s_before;
    __shared__ int s_sup, s_supmass, s_lr[2];
    __shared__ long long s_j;
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t n = Q.n;
    const int nb2 = Q.nb2;
    const double *d2 = Q.d2, *bs1 = Q.bs1, *bs2 = Q.bs2;
    const int per = (nb2 + kSsThreads - 1) / kSsThreads;
    const int q0 = min(tid * per, nb2), q1 = min(q0 + per, nb2);
    if (tid == 0) {
        s_sup = 0x7fffffff;
        s_supmass = -1;
    }
    // the thread's super-block sums in registers (independent loads; nb2 <=
    // kSsPer * kSsThreads, i.e. n <= 2^24, in one round)
    double mine = 0.0;
    double vq[kSsPer];
    for (int qb = q0; qb < q1; qb += kSsPer) {
#pragma unroll
        for (int u = 0; u < kSsPer; ++u) vq[u] = qb + u < q1 ? __ldcg(bs2 + qb + u) : 0.0;
#pragma unroll
        for (int u = 0; u < kSsPer; ++u) mine += vq[u];
    }
    const bool one = q1 - q0 <= kSsPer;  // vq holds the whole chunk
    double tot;
    const double incl = ss_block_scan(mine, s_w, tot);
    j = -1;
    L = -1;
    R = n;
    if (!(tot > 0.0)) return;  // uniform over the CTA
    const double target = Q.u[step - 1] * tot;
    double run = incl - mine, bhit = 0.0, blast = 0.0;
    int lastm = -1, hitq = 0x7fffffff;
    for (int qb = q0; qb < q1; qb += kSsPer) {
        if (!one) {
#pragma unroll
            for (int u = 0; u < kSsPer; ++u) vq[u] = qb + u < q1 ? __ldcg(bs2 + qb + u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kSsPer; ++u) {
            const int q = qb + u;
            if (q < q1) {
                const double v = vq[u];
                if (v > 0.0) {
                    lastm = q;
                    blast = run;
                }
                if (hitq == 0x7fffffff && run + v > target) {
                    hitq = q;
                    bhit = run;
                }
                run += v;
            }
        }
    }
    if (hitq != 0x7fffffff) atomicMin(&s_sup, hitq);
    if (lastm >= 0) atomicMax(&s_supmass, lastm);
    __syncthreads();
    // the cumulative sum before the chosen super-block, from its owner
    const bool fb = s_sup == 0x7fffffff;  // rounding: the last one with mass
    if (fb ? (lastm >= 0 && lastm == s_supmass) : hitq == s_sup) s_before = fb ? blast : bhit;
    __syncthreads();
    const int sup = !fb ? s_sup : (s_supmass >= 0 ? s_supmass : nb2 - 1);
    const double before = s_before;
    if (tid < 32) {
        // block inside the super-block: lane l holds blocks 2l, 2l + 1
        const int64_t bb = (int64_t)sup * kSsSup + 2 * lane;
        const double v0 = bb < Q.nb1 ? __ldcg(bs1 + bb) : 0.0;
        const double v1 = bb + 1 < Q.nb1 ? __ldcg(bs1 + bb + 1) : 0.0;
        double x = v0 + v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const double r0 = before + (x - v0 - v1);
        const bool h0 = r0 + v0 > target, h1 = !h0 && r0 + v0 + v1 > target;
        const uint32_t hm = __ballot_sync(0xffffffffu, h0 || h1);
        int blk;
        double before2 = 0.0;
        if (hm) {
            const int l = __ffs(hm) - 1;
            const int sel = __shfl_sync(0xffffffffu, h0 ? 0 : 1, l);
            blk = 2 * l + sel;
            before2 = __shfl_sync(0xffffffffu, sel ? r0 + v0 : r0, l);
        } else {  // rounding: the last block with mass
            const uint32_t m1 = __ballot_sync(0xffffffffu, v1 > 0.0);
            const uint32_t m0 = __ballot_sync(0xffffffffu, v0 > 0.0);
            const int l1 = m1 ? 31 - __clz(m1) : -1, l0 = m0 ? 31 - __clz(m0) : -1;
            blk = l1 >= 0 && 2 * l1 + 1 > 2 * l0 ? 2 * l1 + 1 : (l0 >= 0 ? 2 * l0 : 0);
        }
        // value inside the block
        const int64_t b1 = (int64_t)sup * kSsSup + blk;
        const int64_t i = b1 * kSsBlk + lane;
        const double v = i < n ? __ldcg(d2 + i) : 0.0;
        double xv = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, xv, o);
            if (lane >= o) xv += y;
        }
        const uint32_t vm = __ballot_sync(0xffffffffu, hm && before2 + xv > target);
        long long jj;
        if (vm) {
            jj = b1 * kSsBlk + (__ffs(vm) - 1);
        } else {  // rounding: the block's last value with mass
            const uint32_t mm = __ballot_sync(0xffffffffu, v > 0.0);
            jj = b1 * kSsBlk + (mm ? 31 - __clz(mm) : 0);
        }
        if (lane == 0) s_j = jj;
    }
    __syncthreads();
    j = s_j;
    // chosen neighbours L < p < R (positions are distinct: a chosen sample
    // has d2 = 0 and is never drawn again)
    const int p = __ldcg(Q.rank + j);
    int l = -1, rr = (int)n;
    for (int q = tid; q < nch; q += kSsThreads) {
        const int v = s_chosen[q];
        if (v < p && v > l) l = v;
        if (v > p && v < rr) rr = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l = max(l, __shfl_xor_sync(0xffffffffu, l, o));
        rr = min(rr, __shfl_xor_sync(0xffffffffu, rr, o));
    }
    if (tid == 0) {
        s_lr[0] = -1;
        s_lr[1] = (int)n;
    }
    __syncthreads();
    if (lane == 0) {
        atomicMax(&s_lr[0], l);
        atomicMin(&s_lr[1], rr);
    }
    __syncthreads();
    L = s_lr[0];
    R = s_lr[1];
    if (tid == 0) s_chosen[nch] = p;
}

__global__ void __launch_bounds__(kSsThreads, 1) seed_sorted_kernel(const __grid_constant__ SeedSorted S) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int32_t s_chosen[];  // CTA r < P: seeding r's chosen sorted positions
    __shared__ long long s_ctl[kSsMaxP][3];
    __shared__ int64_t s_start[kSsMaxP + 1], s_cst[kSsMaxP + 1];
    __shared__ bool s_done[kSsMaxP];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t gtid = (int64_t)blockIdx.x * kSsThreads + tid;
    const int64_t gsz = (int64_t)gridDim.x * kSsThreads;
    const int P = S.P;
    for (int r = 0; r < P; ++r) {
        const SsProb &Q = S.pr[r];
        const double c0 = Q.x[Q.first];
        for (int64_t s = gtid; s < Q.n; s += gsz) {
            const int32_t i = Q.order[s];
            Q.xs[s] = Q.x[i];
            Q.rank[i] = (int32_t)s;
        }
        for (int64_t i = gtid; i < Q.n; i += gsz) {
            const double d = Q.x[i] - c0;
            Q.d2[i] = d * d;
        }
        for (int64_t b = gtid; b < Q.nb2; b += gsz) Q.dmask[b] = 0ull;
        if (gtid == 0) {
            Q.centers[0] = c0;
            Q.dcount[0] = Q.dcount[1] = 0;
            Q.ctl[3] = 0;  // published step
        }
    }
    if (gtid == 0) S.arrive[0] = 0;  // CTAs done re-summing, cumulative
    if (tid < kSsMaxP) s_done[tid] = false;
    grid.sync();
    for (int r = 0; r < P; ++r) {
        const SsProb &Q = S.pr[r];
        for (int64_t blk = gtid; blk < Q.nb1; blk += gsz) Q.bs1[blk] = ss_block_sum(Q.d2, Q.n, blk);
    }
    grid.sync();
    for (int r = 0; r < P; ++r) {  // one warp per super-block, as re-summed
        const SsProb &Q = S.pr[r];
        for (int64_t sp = gtid >> 5; sp < Q.nb2; sp += gsz >> 5) {
            const int64_t b0 = sp * kSsSup + lane, b1 = b0 + 32;
            const double a = b0 < Q.nb1 ? __ldcg(Q.bs1 + b0) : 0.0;
            const double b = b1 < Q.nb1 ? __ldcg(Q.bs1 + b1) : 0.0;
            const double t = warp_tree_sum(a + b);
            if (lane == 0) Q.bs2[sp] = t;
        }
    }
    if (blockIdx.x < P && tid == 0) s_chosen[0] = __ldcg(S.pr[blockIdx.x].rank + S.pr[blockIdx.x].first);
    grid.sync();
    int nch = 1;
    const bool prof = blockIdx.x == 0 && tid == 0;
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0}, t0 = prof ? gtimer() : 0, t1;
    auto mark = [&](int k) {
        if (prof) {
            t1 = gtimer();
            ph[k] += t1 - t0;
            t0 = t1;
        }
    };
    for (int step = 1; step < S.k; ++step) {
        const int buf = step & 1;
        if (blockIdx.x < P) {
            // ---- CTA r picks seeding r's centre (every CTA has arrived after
            // re-summing the previous step's marked blocks)
            const int r = blockIdx.x;
            const SsProb &Q = S.pr[r];
            long long j = -1, L = -1, Rr = Q.n;
            if (!s_done[r]) ss_pick(Q, step, s_chosen, nch, j, L, Rr);
            ++nch;
            if (tid == 0) {  // publish (j = -1: all mass on chosen centres)
                if (j >= 0) Q.centers[step] = Q.x[j];
                Q.ctl[0] = j;
                Q.ctl[1] = L;
                Q.ctl[2] = Rr;
                __threadfence();
                atomicExch((unsigned long long *)(Q.ctl + 3), (unsigned long long)step);
            }
        }
        mark(0);
        // ---- every CTA: the published picks
        for (int r = tid; r < P; r += kSsThreads) {
            const SsProb &Q = S.pr[r];
            while (ld_volatile_s64(Q.ctl + 3) < step) {
            }
            __threadfence();
            s_ctl[r][0] = ld_volatile_s64(Q.ctl);
            s_ctl[r][1] = ld_volatile_s64(Q.ctl + 1);
            s_ctl[r][2] = ld_volatile_s64(Q.ctl + 2);
        }
        __syncthreads();
        mark(1);
        if (tid == 0) {  // range offsets of the seedings still running
            int64_t t = 0;
            for (int r = 0; r < P; ++r) {
                s_start[r] = t;
                if (s_ctl[r][0] >= 0) t += s_ctl[r][2] - s_ctl[r][1] - 1;
            }
            s_start[P] = t;
        }
        if (blockIdx.x < P && s_ctl[blockIdx.x][0] < 0 && !s_done[blockIdx.x]) {
            const SsProb &Q = S.pr[blockIdx.x];  // the reference repeats c0
            const double c0 = Q.x[Q.first];
            for (int q = step + tid; q < S.k; q += kSsThreads) Q.centers[q] = c0;
        }
        bool any = false;
        for (int r = 0; r < P; ++r) any |= s_ctl[r][0] >= 0;
        __syncthreads();
        for (int r = tid; r < P; r += kSsThreads)
            if (s_ctl[r][0] < 0) s_done[r] = true;
        if (!any) return;  // every seeding done (uniform over the grid)
        const int64_t tot_len = s_start[P];
        // ---- d2 = min(d2, (x - c)^2) over each seeding's (L, R); a lowered
        // block is marked in its super-block's mask, which joins the list once
        {
            int r = 0;
            double c = 0.0;
            int64_t rbeg = -1, rend = -1;
            for (int64_t g = gtid; g < tot_len; g += gsz) {
                if (g >= rend) {  // next seeding with a range (empty ranges skipped)
                    r = 0;
                    while (s_start[r + 1] <= g) ++r;
                    rbeg = s_start[r];
                    rend = s_start[r + 1];
                    c = S.pr[r].x[s_ctl[r][0]];
                }
                const SsProb &Q = S.pr[r];
                const int64_t s = s_ctl[r][1] + 1 + (g - rbeg);
                const int32_t i = __ldg(Q.order + s);
                const double d = __ldcg(Q.xs + s) - c;
                const double nv = d * d;
                if (nv < __ldcg(Q.d2 + i)) {
                    Q.d2[i] = nv;
                    const int64_t blk = i / kSsBlk;
                    const int sp = (int)(blk / kSsSup);
                    unsigned long long *dm = Q.dmask + sp;
                    const unsigned long long bit = 1ull << (blk % kSsSup);
                    if (!(__ldcg(dm) & bit)) {
                        const unsigned long long old = atomicOr(dm, bit);
                        if (old == 0ull) Q.dlist[(int64_t)buf * Q.nb2 + atomicAdd(Q.dcount + buf, 1)] = sp;
                    }
                }
            }
        }
        mark(2);
        grid.sync();
        mark(3);
        // ---- re-sum the listed super-blocks, one warp each: lane l owns blocks
        // l and l + 32 (re-summed from d2 when marked), then the tree sum
        {
            if (tid == 0) {
                s_cst[0] = 0;
                for (int r = 0; r < P; ++r) s_cst[r + 1] = s_cst[r] + __ldcg(S.pr[r].dcount + buf);
            }
            __syncthreads();
            const int64_t wg = gtid >> 5, nwg = gsz >> 5;
            bool wrote = false;
            int r = 0;
            for (int64_t q = wg; q < s_cst[P]; q += nwg) {
                while (s_cst[r + 1] <= q) ++r;
                const SsProb &Q = S.pr[r];
                const int sp = __ldcg(Q.dlist + (int64_t)buf * Q.nb2 + (q - s_cst[r]));
                unsigned long long *dm = Q.dmask + sp;
                const unsigned long long m = __ldcg(dm);
                const int64_t b0 = (int64_t)sp * kSsSup + lane, b1 = b0 + 32;
                double a = b0 < Q.nb1 ? __ldcg(Q.bs1 + b0) : 0.0;
                double b = b1 < Q.nb1 ? __ldcg(Q.bs1 + b1) : 0.0;
                const bool ma = (m >> lane) & 1ull, mb = (m >> (lane + 32)) & 1ull;
                if (ma) a = ss_block_sum(Q.d2, Q.n, b0);
                if (mb) b = ss_block_sum(Q.d2, Q.n, b1);
                if (ma) Q.bs1[b0] = a;
                if (mb) Q.bs1[b1] = b;
                const double t = warp_tree_sum(a + b);
                if (lane == 0) {
                    Q.bs2[sp] = t;
                    *dm = 0ull;
                }
                wrote = true;
            }
            if (wrote) __threadfence();
            if (gtid < P) S.pr[gtid].dcount[buf ^ 1] = 0;
        }
        __syncthreads();
        mark(4);
        // ---- arrive; the picking CTAs wait for everyone
        if (tid == 0) {
            atomicAdd(S.arrive, 1u);
            if (blockIdx.x < P) {
                const unsigned want = (unsigned)gridDim.x * (unsigned)step;
                while (*(volatile unsigned *)S.arrive < want) {
                }
                __threadfence();
            }
        }
        __syncthreads();
        mark(5);
    }
    if (prof)
        for (int q = 0; q < 6; ++q) S.phase_ns[q] = ph[q];
}

}  // namespace ivr

extern "C" size_t ivr_kmeans_lloyd_workspace_size(int32_t k) {
    return 4 * sizeof(double) + 2 * (size_t)ivr::kLut + 256 + 16 * (size_t)(k < 1 ? 1 : k);
}

extern "C" int ivr_kmeans_lloyd_step(const double *values, int64_t n, const double *centroids,
                                     int32_t k, double *new_centroids, double *shift,
                                     void *workspace, size_t workspace_bytes, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 1 || k < 2 || k - 1 > kVqSmemMids || !values || !centroids || !new_centroids ||
        !shift || !workspace || workspace_bytes < ivr_kmeans_lloyd_workspace_size(k)) {
        set_error("ivr_kmeans_lloyd_step: bad argument (2 <= k <= 4097, workspace)");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    char *ws = (char *)workspace;
    double *params = reinterpret_cast<double *>(ws);
    uint16_t *lut = reinterpret_cast<uint16_t *>(params + 4);
    char *acc = ws + ((4 * sizeof(double) + 2 * (size_t)kLut + 255) & ~(size_t)255);
    double *sums = reinterpret_cast<double *>(acc);
    unsigned long long *counts = reinterpret_cast<unsigned long long *>(sums + k);
    if (cudaMemsetAsync(acc, 0, 16 * (size_t)k, st) != cudaSuccess)
        return check_launch("ivr_kmeans_lloyd_step memset");
    vq_lut_kernel<<<(kLut + kVqThreads - 1) / kVqThreads, kVqThreads, 0, st>>>(centroids, k, lut,
                                                                              params);
    const size_t smem = 8 * (size_t)(2 * kVqSmemMids + 1) + 4 * (size_t)(kVqSmemMids + 1) +
                        2 * (size_t)kLut;
    cudaFuncSetAttribute(lloyd_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lloyd_accum_kernel<<<grid_for(n), kVqThreads, smem, st>>>(values, n, centroids, k, lut, params,
                                                              sums, counts);
    lloyd_finish_kernel<<<1, 1024, 0, st>>>(centroids, k, sums, counts, new_centroids, shift);
    return check_launch("ivr_kmeans_lloyd_step");
}

extern "C" size_t ivr_kmeans_lloyd_sorted_workspace_size(int32_t k, int32_t sets) {
    return 8 * (size_t)(k < 1 ? 1 : k + 1) * (size_t)(sets < 1 ? 1 : sets);
}

extern "C" int ivr_kmeans_lloyd_step_sorted(const double *sorted_values, int64_t n,
                                            const double *centroids, int32_t k, int32_t sets,
                                            double *new_centroids, double *shift, void *workspace,
                                            size_t workspace_bytes, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 1 || k < 2 || sets < 1 || sets > 65535 || !sorted_values || !centroids ||
        !new_centroids || !shift || !workspace ||
        workspace_bytes < ivr_kmeans_lloyd_sorted_workspace_size(k, sets)) {
        set_error("ivr_kmeans_lloyd_step_sorted: bad argument");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t *bnd = reinterpret_cast<int64_t *>(workspace);
    unsigned long long *sh = reinterpret_cast<unsigned long long *>(shift);
    lloyd_bounds_kernel<<<dim3((k - 1 + kLlThreads - 1) / kLlThreads, sets), kLlThreads, 0, st>>>(
        sorted_values, n, centroids, k, bnd, sh);
    lloyd_segsum_kernel<<<dim3(k, sets), kLlThreads, 0, st>>>(sorted_values, centroids, k, bnd,
                                                              new_centroids, sh);
    return check_launch("ivr_kmeans_lloyd_step_sorted");
}

extern "C" size_t ivr_vq_assign_workspace_size(void) {
    return 8 * sizeof(double) + 2 * (size_t)ivr::kLut + 2 * (size_t)ivr::kLutWin;
}

extern "C" int ivr_vq_assign(const double *values, int64_t n, const double *centroids, int32_t k,
                             uint16_t *indices, void *workspace, size_t workspace_bytes,
                             ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || k < 1 || k > 65536 || (n > 0 && (!values || !centroids || !indices))) {
        set_error("ivr_vq_assign: bad argument");
        return IVR_ERR_ARG;
    }
    if (n == 0) return IVR_OK;
    if (k == 1) {  // a single centroid: every index is 0
        if (cudaMemsetAsync(indices, 0, 2 * (size_t)n, (cudaStream_t)stream) != cudaSuccess)
            return check_launch("ivr_vq_assign memset");
        return IVR_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (!workspace || workspace_bytes < ivr_vq_assign_workspace_size()) {
        set_error("ivr_vq_assign: workspace too small");
        return IVR_ERR_ARG;
    }
    double *params = reinterpret_cast<double *>(workspace);
    uint16_t *lut = reinterpret_cast<uint16_t *>(params + 4);
    if (k - 1 <= kVqSmemMids) {
        const bool aligned = ((reinterpret_cast<uintptr_t>(values) & 15) == 0) &&
                             ((reinterpret_cast<uintptr_t>(indices) & 3) == 0);
        if (aligned) {
            double *params_w = params + 4 + kLut / 4;  // after the kLut table
            uint16_t *lut_w = reinterpret_cast<uint16_t *>(params_w + 4);
            vq_lut_kernel<kLutWin><<<(kLutWin + kVqThreads - 1) / kVqThreads, kVqThreads, 0, st>>>(
                centroids, k, lut_w, params_w);
            auto fn = vq_assign_win_kernel<kLutWin>;
            const size_t sm = kVqSmemMids * sizeof(double) + kLutWin * sizeof(uint32_t);
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWinThreads, sm);
            int64_t b = (n + kWinTile - 1) / kWinTile / (kWinThreads / 32);
            const int64_t cap = 148 * (int64_t)(per_sm > 0 ? per_sm : 1);
            b = b < 1 ? 1 : (b > cap ? cap : b);
            fn<<<(int)b, kWinThreads, sm, st>>>(values, n, centroids, k, lut_w, params_w, indices);
        } else {
            vq_lut_kernel<<<(kLut + kVqThreads - 1) / kVqThreads, kVqThreads, 0, st>>>(centroids, k,
                                                                                      lut, params);
            vq_assign_kernel<true><<<grid_for(n), kVqThreads, 0, st>>>(values, n, centroids, k, lut,
                                                                       params, indices);
        }
    } else {
        cudaMemsetAsync(params, 0, 4 * sizeof(double), st);
        vq_assign_kernel<false><<<grid_for(n), kVqThreads, 0, st>>>(values, n, centroids, k, lut,
                                                                    params, indices);
    }
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
    if (k <= kVqSmemMids + 1)
        vq_decode_kernel<true><<<grid_for_decode(n), kVqThreads, 0, (cudaStream_t)stream>>>(
            indices, n, centroids, k, out, reinterpret_cast<long long *>(bad));
    else
        vq_decode_kernel<false><<<grid_for(n), kVqThreads, 0, (cudaStream_t)stream>>>(
            indices, n, centroids, k, out, reinterpret_cast<long long *>(bad));
    return check_launch("vq_decode_kernel");
}

extern "C" size_t ivr_kmeans_seed_workspace_size(int64_t n) {
    const int64_t nb = (n + ivr::kSeedChunk - 1) / ivr::kSeedChunk;
    return 8 * (size_t)(n < 1 ? 1 : n) + 8 * (size_t)(nb < 1 ? 1 : nb) + 256;
}

extern "C" int ivr_kmeans_seed(const double *values, int64_t n, int32_t k, int64_t first,
                               const double *u, double *centers, void *workspace,
                               size_t workspace_bytes, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 1 || k < 1 || first < 0 || first >= n || !values || !centers || (k > 1 && !u) ||
        !workspace || workspace_bytes < ivr_kmeans_seed_workspace_size(n)) {
        set_error("ivr_kmeans_seed: bad argument");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    double *d2 = reinterpret_cast<double *>(workspace);
    const int nb = (int)((n + kSeedChunk - 1) / kSeedChunk);
    double *bsum = d2 + ((n + 31) & ~(int64_t)31);
    if (cudaMemcpyAsync(centers, values + first, sizeof(double), cudaMemcpyDeviceToDevice, st) !=
        cudaSuccess)
        return check_launch("ivr_kmeans_seed copy");
    for (int i = 1; i < k; ++i) {
        seed_update_kernel<<<nb, kSeedThreads, 0, st>>>(values, n, d2, centers + i - 1, i == 1, bsum);
        seed_pick_kernel<<<1, kPickThreads, 0, st>>>(values, n, d2, bsum, nb, u, centers, i);
    }
    return check_launch("ivr_kmeans_seed");
}

namespace {
inline size_t ss_al(size_t x) { return (x + 255) & ~(size_t)255; }
// per seeding: xs | rank | d2 | block sums | super-block sums | masks | two
// lists | lengths + published pick
size_t ss_bytes(int64_t n) {
    const int64_t nb1 = (n + ivr::kSsBlk - 1) / ivr::kSsBlk;
    const int64_t nb2 = (nb1 + ivr::kSsSup - 1) / ivr::kSsSup;
    return 2 * ss_al(8 * (size_t)n) + ss_al(4 * (size_t)n) + ss_al(8 * (size_t)nb1) +
           2 * ss_al(8 * (size_t)nb2) + ss_al(8 * (size_t)nb2) + 256;
}
}  // namespace

extern "C" size_t ivr_kmeans_seed_sorted_workspace_size(const ivr_seed_problem *problems,
                                                       int32_t count) {
    size_t t = 256;  // arrival counter + phase clock
    for (int p = 0; problems && p < count; ++p)
        t += ss_bytes(problems[p].n < 1 ? 1 : problems[p].n);
    return t;
}

extern "C" int ivr_kmeans_seed_sorted(const ivr_seed_problem *problems, int32_t count, int32_t k,
                                      void *workspace, size_t workspace_bytes,
                                      ivr_stream_t stream) {
    using namespace ivr;
    bool ok = problems && count >= 1 && count <= kSsMaxP && k >= 1 && k <= kSsMaxK && workspace &&
              workspace_bytes >= ivr_kmeans_seed_sorted_workspace_size(problems, count);
    for (int p = 0; ok && p < count; ++p) {
        const ivr_seed_problem &q = problems[p];
        ok = q.values && q.order && q.centers && q.n >= 1 && q.n <= 0x7fffffffll && q.first >= 0 &&
             q.first < q.n && (k == 1 || q.u);
    }
    if (!ok) {
        set_error("ivr_kmeans_seed_sorted: bad argument");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)workspace;
    SeedSorted S{};
    S.k = k;
    S.P = count;
    S.arrive = (unsigned *)w;
    S.phase_ns = (unsigned long long *)(w + 64);
    w += 256;
    for (int p = 0; p < count; ++p) {
        const ivr_seed_problem &q = problems[p];
        SsProb &Q = S.pr[p];
        Q.x = q.values;
        Q.order = q.order;
        Q.n = q.n;
        Q.first = q.first;
        Q.u = q.u;
        Q.centers = q.centers;
        Q.nb1 = (q.n + kSsBlk - 1) / kSsBlk;
        Q.nb2 = (int)((Q.nb1 + kSsSup - 1) / kSsSup);
        Q.xs = (double *)w;
        w += ss_al(8 * (size_t)q.n);
        Q.d2 = (double *)w;
        w += ss_al(8 * (size_t)q.n);
        Q.rank = (int32_t *)w;
        w += ss_al(4 * (size_t)q.n);
        Q.bs1 = (double *)w;
        w += ss_al(8 * (size_t)Q.nb1);
        Q.bs2 = (double *)w;
        w += ss_al(8 * (size_t)Q.nb2);
        Q.dmask = (unsigned long long *)w;
        w += ss_al(8 * (size_t)Q.nb2);
        Q.dlist = (int32_t *)w;
        w += ss_al(8 * (size_t)Q.nb2);
        Q.dcount = (int32_t *)w;
        Q.ctl = (long long *)(w + 64);
        w += 256;
    }
    const size_t smem = 4 * (size_t)k;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(seed_sorted_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return check_launch("ivr_kmeans_seed_sorted smem");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seed_sorted_kernel, kSsThreads, smem);
    if (sms < count || per_sm < 1) {
        set_error("ivr_kmeans_seed_sorted: kernel does not fit on the device");
        return IVR_ERR_ARG;
    }
    void *args[] = {&S};
    if (cudaLaunchCooperativeKernel((const void *)seed_sorted_kernel, dim3(sms), dim3(kSsThreads),
                                    args, smem, st) != cudaSuccess)
        return check_launch("ivr_kmeans_seed_sorted");
    return check_launch("ivr_kmeans_seed_sorted");
}
