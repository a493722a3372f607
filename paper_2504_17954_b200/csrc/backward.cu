// K4 -- backward pass.
//
// K4a blend_bwd_kernel replaces _kernels.composite_backward
// (_kernels.py:75-135) + the per-Gaussian np.add.at reductions
// (rasterizer.py:240-243).  Two CTAs per tile, one thread per pixel, each warp
// an independent 8x4 pixel block that streams the tile list in 32-pair chunks
// with the K3 strip cull; each pixel walks its contributors BACK to front
// from last_pos, as the reference does: the transmittance in front of
// contributor i is recovered from the forward's t_final by division,
// T_i = T_{i+1} / (1 - alpha_i), and the colour behind i is the suffix sum
// accumulated on the way (small terms first, so it keeps its relative
// precision where the front-to-back form C - A_i cancels), giving
//   dL/dalpha_i = sum_k dout_k (T_i v_ik - suffix_ik / (1 - alpha_i)).
// Decisions (skip / contribute) use the certified float32-with-bound test of
// K3, so the contributor set is the reference's.  Per (splat, warp) the 32
// pixel contributions are warp-reduced and added with one float32 atomic per
// component.
//
// K4b preprocess_bwd_kernel (one thread per Gaussian, float64) chains the
// per-Gaussian accumulators through conic -> cov2d, the channel unpack,
// project_backward, the opacity logit, and optionally shade_backward with
// the inverse-fitting per-scene reductions.
#include <math.h>
#include <stdlib.h>

#include "project.cuh"
#include "cull.cuh"

namespace ivr {

constexpr int kBwdThreads = 256;
constexpr float kSigmaErrB = 4.0e-7f;

struct BwdArgs {
    const int32_t *ranges, *pair_splat;
    int ntx;
    const float4 *rec;
    const float *values;
    const double *rec64;
    int K, W, H;
    const double *t_final;
    const int32_t *last_pos;
    const float *d_out;
    const double *d_out64;  // IVR_BLEND_DOUT_F64: the upstream gradient in float64 instead
    float *g_values, *g_mean, *g_conic, *g_opac;
    int preculled;
    const int32_t *tile_order;
    // deterministic mode: per-(pair, warp) partials in place of atomics,
    // part[((j * 8 + warp) * (K + 6)) + slot], slot = value c | K + geometry
    float *part;
};

__device__ __forceinline__ double exact_alpha_b(double dpx, double dpy, double mx, double my,
                                                double ca, double cb, double cc, double o,
                                                double &alpha_u, double &g) {
    const double ddx = dsub(dpx, mx), ddy = dsub(dpy, my);
    const double sg = dadd(dmul(0.5, dadd(dmul(dmul(ca, ddx), ddx), dmul(dmul(cc, ddy), ddy))),
                           dmul(dmul(cb, ddx), ddy));
    if (sg < 0.0) return -1.0;
    g = exp(-sg);
    alpha_u = dmul(o, g);
    double al = alpha_u;
    if (al > kAlphaCap) al = kAlphaCap;
    if (al < kAlphaSkip) return -1.0;
    return al;
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Transpose reduction of NS per-lane values: each step a lane keeps one half
// of its array and trades the other half with its partner at xor offset h, so
// after log2(NS) steps lane l holds slot (l & (NS-1)) summed over its NS-lane
// group; a final xor over the remaining lane bits completes the warp total.
// NS-1 (+1 for NS=16) shuffles in place of 5 per slot.
template <int NS, typename T = float>
__device__ __forceinline__ T warp_transpose_sum(T *x, int lane) {
#pragma unroll
    for (int h = NS / 2; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const T send = up ? x[i] : x[i + h];
            const T keep = up ? x[i + h] : x[i];
            x[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    T r = x[0];
#pragma unroll
    for (int o = NS; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    return r;
}

__device__ __forceinline__ float ex2_approx_b(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx_b(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Per-warp staging slots for one 32-pair chunk.
template <int KMAX, bool F64>
struct BwdSlots {
    float4 r0[32], r1[32];
    float v[32 * KMAX];
    int sp[32];
    double r64[F64 ? 32 * 6 : 1];
    // deferred value gradients: a batch of up to kBatch contributing pairs
    // keeps each pixel's blend weight w (bw[pair][pixel], padded rows:
    // conflict-free reads); at a flush lanes i and i + 16 form pair i's K sums
    // sum_p bw[i][p] * dout[p][c] (one half of the channels each) from the
    // warp's dout table
    float bw[16 * 33];
    __align__(16) float dout[32 * KMAX];
    int bsp[16], bj[16];
};

constexpr int kBwdWarpW = 8;  // warp footprint 8x4 pixels (as K3)

// Two CTAs per tile (4 warps each), each warp an independent 8x4 block of pixels walking
// the tile list in 32-pair chunks up to the largest last_pos of its pixels
// (same strip cull and prefetch as K3; no CTA barrier).
// 4-warp CTAs; K <= 4 (the inverse fit's float64-decision, geometry-free
// instance) at 7 CTAs/SM (72 registers: C4 K4a 0.331 -> 0.31 ms), K <= 16
// at 6 (80 registers; 7 CTAs cost the C3 instance 3%)
template <int KMAX, bool F64, bool GEOM>
__global__ void __launch_bounds__(128, KMAX <= 4 ? 7 : (KMAX <= 16 ? 6 : 2))
blend_bwd_kernel(BwdArgs A) {
    ::ivr::pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    BwdSlots<KMAX, F64> &W = reinterpret_cast<BwdSlots<KMAX, F64> *>(smem)[threadIdx.x >> 5];

    // a CTA holds blockDim.x / 32 of the tile's 8 blocks (independent warps)
    const int cpt = (kBwdThreads / 32) / (blockDim.x >> 5);  // CTAs per tile
    const int trank = blockIdx.x / cpt;
    const int tile = A.tile_order ? A.tile_order[trank] : trank;
    const int tx = tile % A.ntx, ty = tile / A.ntx;
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = (blockIdx.x % cpt) * (blockDim.x >> 5) + (tid >> 5);  // block of the tile
    constexpr int kWH = 32 / kBwdWarpW, kPerRow = kTile / kBwdWarpW;
    const int sx0 = tx * kTile + kBwdWarpW * (warp % kPerRow);
    const int sy_raw = ty * kTile + kWH * (warp / kPerRow);
    const int px = sx0 + (lane % kBwdWarpW), py = sy_raw + lane / kBwdWarpW;
    const bool inside = px < A.W && py < A.H;
    const int sx1 = min(sx0 + kBwdWarpW - 1, A.W - 1);
    const int sy0 = min(sy_raw, A.H - 1), sy1 = min(sy_raw + kWH - 1, A.H - 1);
    const int s0 = A.ranges[tile];
    const int K = A.K;
    const int64_t pix = (int64_t)py * A.W + px;
    const int last = inside ? A.last_pos[pix] : s0;
    const int stop = __reduce_max_sync(0xffffffffu, last);  // no pixel of the warp contributes past here

    // d alpha_i = sum_k dout_k (T_i v_ik - suffix_ik / (1 - alpha_i)) only
    // needs the dot products D_i = dout . v_i and the scalar suffix
    // S_i = dout . suffix_i = sum_{j > i} w_j D_j, accumulated back to front
    float dout[KMAX];
    float S = 0.0f;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) {
        dout[c] = (inside && c < K) ? (A.d_out64 ? (float)A.d_out64[pix * K + c] : A.d_out[pix * K + c])
                                    : 0.0f;
        W.dout[lane * KMAX + c] = dout[c];
    }
    int nbat = 0;  // pairs in the deferred value batch (warp-uniform)
    // flush: lanes i and i + 16 reduce pair i of the batch over the 32 pixels
    constexpr int KH = KMAX / 2;  // channels per lane at a flush
    auto flush = [&]() {
        __syncwarp();
        const int bi = lane & 15, c0 = (lane >> 4) * KH;
        if (bi < nbat) {
            float acc[KH];
#pragma unroll
            for (int c = 0; c < KH; ++c) acc[c] = 0.f;
            const float *row = W.bw + bi * 33;
#pragma unroll 4
            for (int p2 = 0; p2 < 32; ++p2) {
                const float wv = row[p2];
                const float *dr = W.dout + p2 * KMAX + c0;
                if (KH % 4 == 0) {
#pragma unroll
                    for (int c4 = 0; c4 < KH / 4; ++c4) {
                        const float4 d = reinterpret_cast<const float4 *>(dr)[c4];
                        acc[4 * c4] = fmaf(wv, d.x, acc[4 * c4]);
                        acc[4 * c4 + 1] = fmaf(wv, d.y, acc[4 * c4 + 1]);
                        acc[4 * c4 + 2] = fmaf(wv, d.z, acc[4 * c4 + 2]);
                        acc[4 * c4 + 3] = fmaf(wv, d.w, acc[4 * c4 + 3]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < KH; ++c) acc[c] = fmaf(wv, dr[c], acc[c]);
                }
            }
            if (A.part) {
                float *pp = A.part + ((int64_t)W.bj[bi] * (kBwdThreads / 32) + warp) * (K + 6);
#pragma unroll
                for (int c = 0; c < KH; ++c)
                    if (c0 + c < K && acc[c] != 0.f) pp[c0 + c] = acc[c];
            } else {
                float *gv = A.g_values + (int64_t)K * W.bsp[bi] + c0;
#pragma unroll
                for (int c = 0; c < KH; ++c)
                    if (c0 + c < K && acc[c] != 0.f) atomicAdd(gv + c, acc[c]);
            }
        }
        __syncwarp();
        nbat = 0;
    };
    // per-lane atomic target for the transposed geometry totals: lane l owns
    // slot l (< 6: mean2d x, y, conic a, b, c, opacity)
    float *gbase = nullptr;
    int gstride = 0;
    if (!GEOM) {  // opacity only (transform fits): lane 0 adds the warp sum
        if (lane == 0) {
            gbase = A.g_opac;
            gstride = 1;
        }
    } else if (lane < 2) {
        gbase = A.g_mean + lane;
        gstride = 2;
    } else if (lane < 5) {
        gbase = A.g_conic + (lane - 2);
        gstride = 3;
    } else if (lane == 5) {
        gbase = A.g_opac;
        gstride = 1;
    }
    float T = inside && last > s0 ? (float)A.t_final[pix] : 0.0f;  // behind the last contributor
    const float fpx = (float)px, fpy = (float)py;
    const double dpx = (double)px, dpy = (double)py;

    int sp = 0;
    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
    // two-stage prefetch as in K3: ids one chunk ahead of their records
    // (bit 31: culled for this tile by ivr_bin_sort_cull; -1 past the stop),
    // chunks visited from the last one back to the tile start
    auto fetch_ids = [&](int base) {
        const int j = base + lane;
        return j < stop ? __ldg(A.pair_splat + j) : -1;
    };
    auto fetch_recs = [&](int id) {
        sp = id;
        if (id >= 0) {
            r0 = __ldg(A.rec + 2 * id);
            r1 = __ldg(A.rec + 2 * id + 1);
        }
    };
    const int top = s0 < stop ? s0 + 32 * ((stop - 1 - s0) / 32) : s0 - 32;  // last chunk
    int spn = -1;
    if (top >= s0) {
        fetch_recs(fetch_ids(top));
        if (top - 32 >= s0) spn = fetch_ids(top - 32);
    }
    for (int base = top; base >= s0; base -= 32) {
        const int j = base + lane;
        const bool keep = j < stop && sp >= 0 && !tile_cull32(r0, r1, sx0, sx1, sy0, sy1);
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            W.r0[lane] = r0;
            W.r1[lane] = r1;
            W.sp[lane] = sp;
            const float *v = A.values + (int64_t)K * sp;
#pragma unroll
            for (int c = 0; c < KMAX; ++c) W.v[lane * KMAX + c] = c < K ? __ldg(v + c) : 0.0f;
            if (F64) {
                const double *r = A.rec64 + 8 * (int64_t)sp;
#pragma unroll
                for (int c = 0; c < 6; ++c) W.r64[lane * 6 + c] = __ldg(r + c);
            }
        }
        __syncwarp();
        if (base - 32 >= s0) {
            fetch_recs(spn);
            spn = base - 64 >= s0 ? fetch_ids(base - 64) : -1;
        }
        uint32_t mbits = m;
        while (mbits) {  // back to front inside the chunk
            const int q = 31 - __clz(mbits);
            mbits &= ~(1u << q);
            const float4 a0 = W.r0[q];
            const float4 a1 = W.r1[q];
            bool contrib = false;
            float al = 0.f, alu = 0.f, g = 0.f;
            float dx = 0.f, dy = 0.f;
            if (inside && base + q < last) {
                dx = fpx - a0.x;
                dy = fpy - a0.y;
                const float bdy = a1.y * dy, hcdy = a1.z * dy;
                const float sig = fmaf(fmaf(a1.x, dx, bdy), dx, hcdy * dy);
                if (!(sig > a0.w)) {
                    float cdx = dx, cdy = dy, cbdy = bdy, chcdy = hcdy, csig = sig;
                    if (F64) {
                        cdx = (float)dsub(dpx, W.r64[q * 6]);
                        cdy = (float)dsub(dpy, W.r64[q * 6 + 1]);
                        cbdy = a1.y * cdy;
                        chcdy = a1.z * cdy;
                        csig = fmaf(fmaf(a1.x, cdx, cbdy), cdx, chcdy * cdy);
                    }
                    const float terms = fmaf(a1.x * cdx, cdx, fmaf(chcdy, cdy, fabsf(cbdy * cdx)));
                    const float E = kSigmaErrB * terms + 1e-30f;
                    const float thr = a1.w;
                    const float tm = 2.4e-7f * fabsf(thr) + 1e-7f;
                    if (csig - E > 0.0f && csig + E < thr - tm) {
                        g = ex2_approx_b(-1.4426950408889634f * csig);
                        alu = a0.z * g;
                        al = fminf(alu, 0.99f);
                        contrib = true;
                    } else if (!(csig - E > a0.w)) {
                        double au, gd, ad;
                        if (F64) {
                            const double *r = W.r64 + q * 6;
                            ad = exact_alpha_b(dpx, dpy, r[0], r[1], r[2], r[3], r[4], r[5], au, gd);
                        } else {
                            ad = exact_alpha_b(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                               2.0 * (double)a1.z, a0.z, au, gd);
                        }
                        if (ad >= 0.0) {
                            al = (float)ad;
                            alu = (float)au;
                            g = (float)gd;
                            contrib = true;
                        }
                    }
                    dx = cdx;
                    dy = cdy;
                }
            }
            // per-pixel contributions: w (the value gradients dout_c * w are
            // reduced per batch), xg = d mean2d (2), d conic (3), d opacity
            // (zero when not contributing)
            float wpix = 0.f, xg[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) xg[c] = 0.f;
            if (contrib) {
                // T in front of this contributor: T / (1 - alpha) (approximate
                // reciprocal + one Newton step, ~0.5 ulp)
                const float om = 1.0f - al;
                float inv = rcp_approx_b(om);
                inv = fmaf(inv, fmaf(-om, inv, 1.0f), inv);
                T = T * inv;
                const float w = T * al;
                float Dv = 0.f;  // dout . v
                if (KMAX % 4 == 0) {
                    const float4 *vv = reinterpret_cast<const float4 *>(W.v + q * KMAX);
#pragma unroll
                    for (int c4 = 0; c4 < KMAX / 4; ++c4) {
                        const float4 v = vv[c4];
                        Dv = fmaf(dout[4 * c4], v.x, Dv);
                        Dv = fmaf(dout[4 * c4 + 1], v.y, Dv);
                        Dv = fmaf(dout[4 * c4 + 2], v.z, Dv);
                        Dv = fmaf(dout[4 * c4 + 3], v.w, Dv);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c) Dv = fmaf(dout[c], W.v[q * KMAX + c], Dv);
                }
                wpix = w;
                const float d_alpha = T * Dv - S * inv;
                S = fmaf(w, Dv, S);  // suffix seen by the contributors in front
                if (alu < 0.99f) {
                    if (GEOM) {
                        const float d_sigma = -alu * d_alpha;
                        const float ca = 2.0f * a1.x, cb = a1.y, cc = 2.0f * a1.z;
                        xg[0] = -d_sigma * (ca * dx + cb * dy);
                        xg[1] = -d_sigma * (cb * dx + cc * dy);
                        xg[2] = 0.5f * dx * dx * d_sigma;
                        xg[3] = dx * dy * d_sigma;
                        xg[4] = 0.5f * dy * dy * d_sigma;
                    }
                    xg[5] = g * d_alpha;
                }
            }
            if (__any_sync(0xffffffffu, contrib)) {
                // value gradients: this pair's pixel weights join the batch;
                // geometry: transpose reduction (7 shuffles + the remaining lane
                // bits, lane l ends with slot l % 8) and parallel atomics
                const int s = W.sp[q];
                W.bw[nbat * 33 + lane] = wpix;
                if (lane == 0) {
                    W.bsp[nbat] = s;
                    W.bj[nbat] = base + q;
                }
                if (++nbat == 16) flush();
                const float tg = GEOM ? warp_transpose_sum<8>(xg, lane) : warp_sum(xg[5]);
                if (A.part) {  // deterministic mode: plain stores, reduced in fixed order later
                    float *pp = A.part + ((int64_t)(base + q) * (kBwdThreads / 32) + warp) * (K + 6);
                    if (GEOM ? (lane < 6) : (lane == 0)) {
                        if (tg != 0.f) pp[K + (GEOM ? lane : 5)] = tg;
                    }
                } else {
                    if (gbase && tg != 0.f) atomicAdd(gbase + (int64_t)gstride * s, tg);
                }
            }
        }
        __syncwarp();  // slots are rewritten by the next chunk
    }
    if (nbat > 0) flush();
}

template <int KMAX, bool F64>
int launch_bwd(const BwdArgs &A, int ntiles, bool geom, cudaStream_t st) {
    const size_t sm = (kBwdThreads / 32) * sizeof(BwdSlots<KMAX, F64>);
    auto fn = geom ? blend_bwd_kernel<KMAX, F64, true> : blend_bwd_kernel<KMAX, F64, false>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // half-tile CTAs, as K3 (C4 K4a 0.332 -> 0.326 ms, C3 0.339 -> 0.335 ms)
    constexpr int wpc = 4;
    const int cpt = (kBwdThreads / 32) / wpc;
    launch<3>(fn, ntiles * cpt, 32 * wpc, (sm / (kBwdThreads / 32)) * wpc, st, A);
    return check_launch("blend_bwd_kernel");
}

// ----------------------------------------------------------------- deterministic K4a
// Fixed-order reduction of the per-(pair, warp) partials: one thread per
// Gaussian walks its tile rectangle row-major (the reference's pair order),
// finds its entry in each tile list by binary search on (depth key, splat)
// -- the order K2 produced -- and sums the 8 warp partials of that entry in
// warp order, in float64.  Same result on every run.
__global__ void __launch_bounds__(128)
bwd_reduce_det_kernel(int64_t n, int K, const uint64_t *depth_key, const int32_t *count,
                      const ushort4 *rect, const int32_t *ranges, const int32_t *pair_splat,
                      int ntx, int64_t cap, const float *part, float *g_values, float *g_mean,
                      float *g_conic, float *g_opac) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double acc[32 + 6];
    for (int c = 0; c < K + 6; ++c) acc[c] = 0.0;
    if (count[s] > 0) {
        const ushort4 rc = rect[s];
        const uint64_t key = depth_key[s];
        for (int ty = rc.z; ty <= rc.w; ++ty)
            for (int tx = rc.x; tx <= rc.y; ++tx) {
                const int t = ty * ntx + tx;
                int lo = ranges[t], hi = ranges[t + 1];
                lo = lo < cap ? lo : (int)cap;
                hi = hi < cap ? hi : (int)cap;
                while (lo < hi) {  // first entry not below (key, s)
                    const int mid = (lo + hi) >> 1;
                    const uint32_t sp = (uint32_t)pair_splat[mid] & 0x7fffffffu;
                    const uint64_t km = depth_key[sp];
                    if (km < key || (km == key && (int64_t)sp < s)) lo = mid + 1;
                    else hi = mid;
                }
                if (lo >= (int)cap || ((uint32_t)pair_splat[lo] & 0x7fffffffu) != (uint32_t)s) continue;
                const float *pp = part + (int64_t)lo * (kBwdThreads / 32) * (K + 6);
                for (int w = 0; w < kBwdThreads / 32; ++w)
                    for (int c = 0; c < K + 6; ++c) acc[c] += (double)pp[w * (K + 6) + c];
            }
    }
    for (int c = 0; c < K; ++c) g_values[s * K + c] = (float)acc[c];
    if (g_mean) {
        g_mean[2 * s] = (float)acc[K];
        g_mean[2 * s + 1] = (float)acc[K + 1];
    }
    if (g_conic)
        for (int c = 0; c < 3; ++c) g_conic[3 * s + c] = (float)acc[K + 2 + c];
    g_opac[s] = (float)acc[K + 5];
}

// ----------------------------------------------------------------- K4b helpers
__device__ __forceinline__ void normalize_bwd(const double v[3], const double d[3], double out[3]) {
    // _mathutil.normalize_rows_backward: (d - (d.u) u) / |v|
    const double in = 1.0 / sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    const double u[3] = {v[0] * in, v[1] * in, v[2] * in};
    const double pr = d[0] * u[0] + d[1] * u[1] + d[2] * u[2];
    for (int k = 0; k < 3; ++k) out[k] = (d[k] - pr * u[k]) * in;
}

__device__ __forceinline__ double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

// bad[id] = first row with a non-finite value in output tensor `id`
__device__ __forceinline__ void flag_bad(unsigned long long *bad, int64_t i, int id, double x) {
    if (bad && !isfinite(x)) atomicMin(bad + id, (unsigned long long)i);
}

struct BwdConst {
    ivr_gaussians G;
    ivr_shading S;
    int has_shading;
    ivr_edits E;
    int has_edits;
    ivr_layout L;
    ivr_grads R;
    int geometry;
};

// GEOM: the projection / covariance / quaternion backward is compiled in
// (training); transform fits instantiate without it (fewer registers).
template <bool GEOM>
__global__ void __launch_bounds__(128, GEOM ? 4 : 5)
preprocess_bwd_kernel(BwdConst B, ivr_frame_params Pv, const ivr_frame_params *__restrict__ Pd) {
    ::ivr::pdl_begin();
    __shared__ ivr_frame_params P;
    __shared__ double s_glob[10];
    extern __shared__ double s_scene[];  // [S][4] per-scene d_c_p (3) + d_scale
    {
        const ivr_frame_params *src = Pd ? Pd : &Pv;
        constexpr int kWords = (int)(sizeof(ivr_frame_params) / 4);
        for (int w = threadIdx.x; w < kWords; w += blockDim.x)
            reinterpret_cast<int *>(&P)[w] = reinterpret_cast<const int *>(src)[w];
        if (threadIdx.x < 10) s_glob[threadIdx.x] = 0.0;
    }
    const int nsc = B.R.per_scene;  // number of per-scene slots in s_scene (0 = none)
    for (int k = threadIdx.x; k < 4 * nsc; k += blockDim.x) s_scene[k] = 0.0;
    __syncthreads();
    const ivr_gaussians &G = B.G;
    const ivr_grads &R = B.R;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // this thread's contributions to the reductions: [0..9] the 10 global
    // transform gradients, [10..12] its scene's d_c_p, [13] its d_scale;
    // warp-reduced (transpose sum) before one shared atomic per slot
    double red[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) red[k] = 0.0;
    const bool active = i < G.n;
    int32_t sid_l = -1;
    if (active) {
        const ivr_camera &cam = P.cam;
        const int K = B.L.k;
        const int32_t sid = (B.has_edits && B.E.scene_id) ? B.E.scene_id[i] : 0;
        sid_l = sid;
        // ---- per-Gaussian upstream from K4a
        double gv_color[3] = {0, 0, 0}, gv_depth = 0.0, gv_norm[3] = {0, 0, 0};
        double gmean[2] = {0, 0}, gcon[3] = {0, 0, 0}, gop = 0.0;
        if (R.g_values) {
            const float *gv = R.g_values + (int64_t)K * i;
            if (B.L.col_color >= 0) for (int k = 0; k < 3; ++k) gv_color[k] = gv[B.L.col_color + k];
            if (B.L.col_depth >= 0) gv_depth = gv[B.L.col_depth];
            if (B.L.col_normal >= 0) for (int k = 0; k < 3; ++k) gv_norm[k] = gv[B.L.col_normal + k];
            if (R.d_values) for (int c = 0; c < K; ++c) R.d_values[(int64_t)K * i + c] = gv[c];
        }
        if (R.g_mean2d) { gmean[0] = R.g_mean2d[2 * i]; gmean[1] = R.g_mean2d[2 * i + 1]; }
        if (R.g_conic) for (int k = 0; k < 3; ++k) gcon[k] = R.g_conic[3 * i + k];
        if (R.g_opacity) gop = R.g_opacity[i];
        if (R.d_colors) for (int k = 0; k < 3; ++k) R.d_colors[3 * i + k] = gv_color[k];
        if (R.d_mean2d) { R.d_mean2d[2 * i] = gmean[0]; R.d_mean2d[2 * i + 1] = gmean[1]; }
        for (int k = 0; k < 3; ++k) flag_bad(R.bad, i, 5, gv_color[k]);

        // d_mu / d_n_raw only when asked for (transform fits skip both chains)
        const bool want_mu = R.d_mu || R.d_n_raw;
        double d_mu[3] = {0, 0, 0}, d_n_raw[3] = {0, 0, 0}, nraw[3] = {0, 0, 0};
        if (want_mu) {
            for (int k = 0; k < 3; ++k) nraw[k] = G.n_raw[3 * i + k];
            if (B.L.col_normal >= 0 && R.g_values) normalize_bwd(nraw, gv_norm, d_n_raw);
        }

        // ---- opacity: effective logit chain (rasterizer.py:278-279) + inverse scale
        const bool rescale = B.has_edits && P.rescale_opacity && B.E.opacity_scale;
        const double scale = rescale ? B.E.opacity_scale[sid] : 1.0;
        const double o_base = sigmoid_ref(G.o_logit[i]);
        double pcl = o_base, o_eff = o_base;
        bool open_gate = true;
        if (rescale) {
            const double praw = scale * o_base;
            pcl = praw < 1e-12 ? 1e-12 : (praw > 1.0 - 1e-9 ? 1.0 - 1e-9 : praw);
            open_gate = (praw > 1e-12) && (praw < 1.0 - 1e-9);
            o_eff = sigmoid_ref(log(pcl / (1.0 - pcl)));
        }
        const double d_o_logit = gop * o_eff * (1.0 - o_eff);
        if (R.d_o_logit) R.d_o_logit[i] = d_o_logit;
        flag_bad(R.bad, i, 3, d_o_logit);
        if (R.d_scale && nsc > 0) {
            const double d_p = d_o_logit / (pcl * (1.0 - pcl));
            red[13] = open_gate ? d_p * o_base : 0.0;
        }

        // ---- geometry (gaussians.project_backward)
        if (GEOM) {
            Proj p;
            project_one(G, i, cam, p);
            double dq[4] = {0, 0, 0, 0}, dls[3] = {0, 0, 0};
            if (p.valid) {
                // conic -> cov2d: dC = -Q dQ Q (symmetric split of the b term)
                const double Q[4] = {p.conic[0], p.conic[1], p.conic[1], p.conic[2]};
                const double dQ[4] = {gcon[0], 0.5 * gcon[1], 0.5 * gcon[1], gcon[2]};
                double T1[4], dC[4];
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c)
                        T1[2 * r + c] = Q[2 * r] * dQ[c] + Q[2 * r + 1] * dQ[2 + c];
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c)
                        dC[2 * r + c] = -(T1[2 * r] * Q[c] + T1[2 * r + 1] * Q[2 + c]);
                const double *W = cam.rotation;
                const double f = cam.focal, tz = p.tzs;
                // d_cov3d = M^T dC M ; dM = dC M C3^T + dC^T M C3
                double MtdC[6];  // (3x2) = M^T dC
                for (int a = 0; a < 3; ++a)
                    for (int c = 0; c < 2; ++c)
                        MtdC[2 * a + c] = p.M[a] * dC[c] + p.M[3 + a] * dC[2 + c];
                double dC3[9];
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        dC3[3 * a + b] = MtdC[2 * a] * p.M[b] + MtdC[2 * a + 1] * p.M[3 + b];
                double dM[6];
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 3; ++c) {
                        double acc = 0.0;
                        for (int m = 0; m < 2; ++m)
                            for (int k = 0; k < 3; ++k) {
                                acc += dC[2 * r + m] * p.M[3 * m + k] * p.C3[3 * c + k];
                                acc += dC[2 * m + r] * p.M[3 * m + k] * p.C3[3 * k + c];
                            }
                        dM[3 * r + c] = acc;
                    }
                double dJ[6];
                for (int r = 0; r < 2; ++r)
                    for (int k = 0; k < 3; ++k)
                        dJ[3 * r + k] = dM[3 * r] * W[3 * k] + dM[3 * r + 1] * W[3 * k + 1] +
                                        dM[3 * r + 2] * W[3 * k + 2];
                // one reciprocal instead of ten divisions (gradient tolerance 1e-3)
                const double itz = 1.0 / tz, f1 = f * itz, f2 = f1 * itz, f3 = f2 * itz;
                double dt[3];
                dt[0] = dJ[2] * (-f2) + gmean[0] * f1;
                dt[1] = dJ[5] * (-f2) + gmean[1] * f1;
                dt[2] = dJ[0] * (-f2) + dJ[4] * (-f2) + dJ[2] * (2 * p.t[0] * f3) +
                        dJ[5] * (2 * p.t[1] * f3) - gmean[0] * p.t[0] * f2 -
                        gmean[1] * p.t[1] * f2 + gv_depth;
                for (int j = 0; j < 3; ++j)
                    d_mu[j] += dt[0] * W[j] + dt[1] * W[3 + j] + dt[2] * W[6 + j];
                // covariance_backward (gaussians.py:278-289)
                double Gs[9], dM3[9];
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) Gs[3 * a + b] = dC3[3 * a + b] + dC3[3 * b + a];
                for (int a = 0; a < 3; ++a)
                    for (int k = 0; k < 3; ++k) {
                        double acc = 0.0;
                        for (int b = 0; b < 3; ++b) acc += Gs[3 * a + b] * p.R[3 * b + k] * p.s[k];
                        dM3[3 * a + k] = acc;
                    }
                double ds[3] = {0, 0, 0}, dR[9];
                for (int k = 0; k < 3; ++k)
                    for (int a = 0; a < 3; ++a) {
                        ds[k] += dM3[3 * a + k] * p.R[3 * a + k];
                        dR[3 * a + k] = dM3[3 * a + k] * p.s[k];
                    }
                // quat_to_rot_backward (gaussians.py:239-264)
                const double w = p.q[0], x = p.q[1], y = p.q[2], z = p.q[3];
                const double *g = dR;
                const double qw = 2 * (-z * g[1] + y * g[2] + z * g[3] - x * g[5] - y * g[6] + x * g[7]);
                const double qx = 2 * (y * g[1] + z * g[2] + y * g[3] - 2 * x * g[4] - w * g[5] +
                                       z * g[6] + w * g[7] - 2 * x * g[8]);
                const double qy = 2 * (-2 * y * g[0] + x * g[1] + w * g[2] + x * g[3] + z * g[5] -
                                       w * g[6] + z * g[7] - 2 * y * g[8]);
                const double qz = 2 * (-2 * z * g[0] - w * g[1] + x * g[2] + w * g[3] - 2 * z * g[4] +
                                       y * g[5] + x * g[6] + y * g[7]);
                const double qraw[4] = {G.q_raw[4 * i], G.q_raw[4 * i + 1], G.q_raw[4 * i + 2],
                                        G.q_raw[4 * i + 3]};
                const double qn = sqrt(qraw[0] * qraw[0] + qraw[1] * qraw[1] + qraw[2] * qraw[2] +
                                       qraw[3] * qraw[3]);
                const double dqv[4] = {qw, qx, qy, qz};
                double pr = 0.0;
                const double iqn = 1.0 / qn;
                for (int k = 0; k < 4; ++k) pr += dqv[k] * (qraw[k] * iqn);
                for (int k = 0; k < 4; ++k) dq[k] = (dqv[k] - pr * (qraw[k] * iqn)) * iqn;
                for (int k = 0; k < 3; ++k) dls[k] = ds[k] * p.s[k];
            }
            if (R.d_q_raw) for (int k = 0; k < 4; ++k) R.d_q_raw[4 * i + k] = dq[k];
            if (R.d_log_s) for (int k = 0; k < 3; ++k) R.d_log_s[3 * i + k] = dls[k];
            for (int k = 0; k < 4; ++k) flag_bad(R.bad, i, 1, dq[k]);
            for (int k = 0; k < 3; ++k) flag_bad(R.bad, i, 2, dls[k]);
        }

        // ---- shading (shading.shade_backward)
        if (B.has_shading) {
            const double mu[3] = {G.mu[3 * i], G.mu[3 * i + 1], G.mu[3 * i + 2]};
            double nrm[3];
            unit_normal(G, i, nrm);
            ShadeState st;
            shade_state<false>(B.S, P, i, sid, mu, nrm, st, G.cache);
            double d_rgb[3];
            for (int k = 0; k < 3; ++k)
                d_rgb[k] = gv_color[k] + (R.d_rgb_extra ? R.d_rgb_extra[3 * i + k] : 0.0);
            const double s3 = d_rgb[0] + d_rgb[1] + d_rgb[2];
            const double dot_cv = d_rgb[0] * st.c_v[0] + d_rgb[1] * st.c_v[1] + d_rgb[2] * st.c_v[2];
            const double k_a = st.k[0], k_d = st.k[1], k_s = st.k[2], beta = st.k[3];
            double d_c_v[3];
            for (int k = 0; k < 3; ++k) d_c_v[k] = (k_a + k_d * st.a_ndl) * d_rgb[k];
            const double d_k_a = dot_cv, d_k_d = st.a_ndl * dot_cv, d_k_s = st.spow * s3;
            const double d_spow = k_s * s3;
            const bool safe = st.a_ndh > 0.0;
            const double log_andh = log(safe ? st.a_ndh : 1.0);
            const double d_a_ndh = (st.gate && safe) ? d_spow * beta * exp((beta - 1.0) * log_andh) : 0.0;
            const double d_beta = (st.gate && safe) ? d_spow * st.spow * log_andh : 0.0;
            const double d_a_ndl = k_d * dot_cv;
            const double d_ndl = sgn(st.ndl) * d_a_ndl, d_ndh = sgn(st.ndh) * d_a_ndh;
            double d_n_unit[3], d_l[3], d_h[3], d_v[3];
            for (int k = 0; k < 3; ++k) {
                d_n_unit[k] = d_ndl * st.l[k] + d_ndh * st.h[k];
                d_l[k] = d_ndl * nrm[k];
                d_h[k] = d_ndh * nrm[k];
            }
            if (!P.orbital) {
                for (int k = 0; k < 3; ++k) d_v[k] = d_h[k] + d_l[k];
            } else {
                double d_u[3];
                normalize_bwd(st.u, d_h, d_u);
                for (int k = 0; k < 3; ++k) {
                    d_v[k] = d_u[k];
                    d_l[k] += d_u[k];
                }
                double dp = 0.0, da = 0.0;
                for (int k = 0; k < 3; ++k) {
                    dp += d_l[k] * P.dl_dp[k];
                    da += d_l[k] * P.dl_da[k];
                }
                red[8] = dp;
                red[9] = da;
            }
            if (want_mu) {
                double d_w[3];
                normalize_bwd(st.w_cam, d_v, d_w);
                for (int k = 0; k < 3; ++k) d_mu[k] -= d_w[k];
                double d_nr2[3];
                normalize_bwd(nraw, d_n_unit, d_nr2);
                for (int k = 0; k < 3; ++k) d_n_raw[k] += d_nr2[k];
            }
            const double e_a = d_k_a * P.term_scales[0] * (st.gates[0] ? 1.0 : 0.0);
            const double e_d = d_k_d * P.term_scales[1] * (st.gates[1] ? 1.0 : 0.0);
            const double e_s = d_k_s * P.term_scales[2] * (st.gates[2] ? 1.0 : 0.0);
            const double e_b = d_beta * P.term_scales[3] * (st.gates[3] ? 1.0 : 0.0);
            red[0] = e_a * st.sig[0];
            red[1] = e_d * st.sig[1];
            red[2] = e_s * st.sig[2];
            red[3] = e_b * st.beta1;
            red[4] = e_a;
            red[5] = e_d;
            red[6] = e_s;
            red[7] = e_b;
            const double dka = e_a * P.lam[0] * st.sig[0] * (1.0 - st.sig[0]);
            const double dkd = e_d * P.lam[1] * st.sig[1] * (1.0 - st.sig[1]);
            const double dks = e_s * P.lam[2] * st.sig[2] * (1.0 - st.sig[2]);
            const double dlb = e_b * P.lam[3] * (st.beta1 - 1.0);
            if (R.d_k_a_raw) R.d_k_a_raw[i] = dka;
            if (R.d_k_d_raw) R.d_k_d_raw[i] = dkd;
            if (R.d_k_s_raw) R.d_k_s_raw[i] = dks;
            if (R.d_log_beta) R.d_log_beta[i] = dlb;
            double dco[3];
            for (int k = 0; k < 3; ++k) dco[k] = st.open[k] ? d_c_v[k] : 0.0;
            if (R.d_delta_c) for (int k = 0; k < 3; ++k) R.d_delta_c[3 * i + k] = dco[k];
            if (R.d_c_p) {
                if (nsc > 0) {
                    for (int k = 0; k < 3; ++k) red[10 + k] = dco[k];
                } else {
                    for (int k = 0; k < 3; ++k) R.d_c_p[3 * i + k] = dco[k];
                }
            }
            flag_bad(R.bad, i, 6, dka);
            flag_bad(R.bad, i, 7, dkd);
            flag_bad(R.bad, i, 8, dks);
            flag_bad(R.bad, i, 9, dlb);
            for (int k = 0; k < 3; ++k) flag_bad(R.bad, i, 10, dco[k]);
        }
        if (R.d_mu) for (int k = 0; k < 3; ++k) R.d_mu[3 * i + k] = d_mu[k];
        if (R.d_n_raw) for (int k = 0; k < 3; ++k) R.d_n_raw[3 * i + k] = d_n_raw[k];
        if (want_mu) {
            for (int k = 0; k < 3; ++k) {
                flag_bad(R.bad, i, 0, d_mu[k]);
                flag_bad(R.bad, i, 4, d_n_raw[k]);
            }
        }
    }
    if (R.d_globals || nsc > 0) {  // transform gradients requested (fits, shade_backward)
        const int lane = threadIdx.x & 31;
        const unsigned act = __ballot_sync(0xffffffffu, active);
        if (act) {
            const int32_t sid0 = __shfl_sync(0xffffffffu, sid_l, __ffs(act) - 1);
            const bool uni = __all_sync(0xffffffffu, !active || sid_l == sid0);
            if (!uni) {  // mixed scenes in this warp: per-lane scene atomics
                if (nsc > 0 && active) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (red[10 + k] != 0.0) atomicAdd(&s_scene[4 * sid_l + k], red[10 + k]);
                }
#pragma unroll
                for (int k = 10; k < 14; ++k) red[k] = 0.0;
            }
            const double t = warp_transpose_sum<16, double>(red, lane);
            if (lane < 10) {
                if (t != 0.0) atomicAdd(&s_glob[lane], t);
            } else if (lane < 14 && nsc > 0 && uni && t != 0.0) {
                atomicAdd(&s_scene[4 * sid0 + (lane - 10)], t);
            }
        }
    }
    __syncthreads();
    if (R.scratch) {  // per-block partials; bwd_sums_kernel adds them in a fixed order
        const int nsl = 10 + 4 * nsc;
        double *pb = R.scratch + (int64_t)blockIdx.x * nsl;
        for (int k = threadIdx.x; k < nsl; k += blockDim.x)
            pb[k] = k < 10 ? (B.has_shading ? s_glob[k] : 0.0) : s_scene[k - 10];
        return;
    }
    if (R.d_globals && B.has_shading && threadIdx.x < 10) atomicAdd(&R.d_globals[threadIdx.x], s_glob[threadIdx.x]);
    for (int k = threadIdx.x; k < 4 * nsc; k += blockDim.x) {
        const double v = s_scene[k];
        if (v == 0.0) continue;
        if ((k & 3) == 3) {
            if (R.d_scale) atomicAdd(&R.d_scale[k >> 2], v);
        } else if (R.d_c_p) {
            atomicAdd(&R.d_c_p[3 * (k >> 2) + (k & 3)], v);
        }
    }
}

// Fixed-order sums of K4b's per-block partials (one block per slot): the 10
// global transform gradients and the per-scene d_c_p / d_scale, without
// contended float64 atomics and identical run to run.
__global__ void __launch_bounds__(256)
bwd_sums_kernel(const double *part, int nblocks, int nsc, int has_globals, double *d_globals,
                double *d_c_p, double *d_scale) {
    ::ivr::pdl_begin();
    __shared__ double s[256];
    const int nsl = 10 + 4 * nsc, slot = blockIdx.x;
    double t = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 256) t += part[(int64_t)b * nsl + slot];
    s[threadIdx.x] = t;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h) s[threadIdx.x] += s[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double v = s[0];
    if (slot < 10) {
        if (d_globals && has_globals) d_globals[slot] += v;
    } else {
        const int k = slot - 10;
        if ((k & 3) == 3) {
            if (d_scale) d_scale[k >> 2] += v;
        } else if (d_c_p) {
            d_c_p[3 * (k >> 2) + (k & 3)] += v;
        }
    }
}

ivr_frame_params params_from(const ivr_camera &cam, const ivr_shading *S, const ivr_edits *E);

}  // namespace ivr

namespace {
int blend_bwd_impl(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                   int32_t nty, const float *rec, const float *values, const double *rec64,
                   int32_t k, int32_t width, int32_t height, const double *t_final,
                   const int32_t *last_pos, const float *d_out, float *g_values, float *g_mean2d,
                   float *g_conic, float *g_opacity, const int32_t *tile_order, int32_t flags,
                   float *part, ivr_stream_t stream) {
    using namespace ivr;
    if (!tile_ranges || !pair_splat || !rec || !values || !t_final || !last_pos || !d_out ||
        !g_values || !g_opacity || k < 1 || k > 32 ||
        (!(flags & IVR_BLEND_NO_GEOMETRY) && (!g_mean2d || !g_conic)) ||
        ntx != (width + kTile - 1) / kTile || nty != (height + kTile - 1) / kTile) {
        set_error("ivr_blend_bwd: bad argument");
        return IVR_ERR_ARG;
    }
    BwdArgs A;
    A.ranges = tile_ranges;
    A.pair_splat = pair_splat;
    A.ntx = ntx;
    A.rec = reinterpret_cast<const float4 *>(rec);
    A.values = values;
    A.rec64 = rec64;
    A.K = k;
    A.W = width;
    A.H = height;
    A.t_final = t_final;
    A.last_pos = last_pos;
    const bool dout64 = (flags & IVR_BLEND_DOUT_F64) != 0;
    A.d_out = dout64 ? nullptr : d_out;
    A.d_out64 = dout64 ? reinterpret_cast<const double *>(d_out) : nullptr;
    A.g_values = g_values;
    A.g_mean = g_mean2d;
    A.g_conic = g_conic;
    A.g_opac = g_opacity;
    A.preculled = (flags & IVR_BLEND_PRECULLED) ? 1 : 0;
    A.tile_order = tile_order;
    A.part = part;
    cudaStream_t st = (cudaStream_t)stream;
    const int nt = ntx * nty;
    const bool f64 = rec64 != nullptr;
    const bool geom = (flags & IVR_BLEND_NO_GEOMETRY) == 0;
#define IVR_BWD(KM) return f64 ? launch_bwd<KM, true>(A, nt, geom, st) : launch_bwd<KM, false>(A, nt, geom, st)
    if (k <= 4) { IVR_BWD(4); }
    if (k <= 8) { IVR_BWD(8); }
    if (k <= 16) { IVR_BWD(16); }
    IVR_BWD(32);
#undef IVR_BWD
}
}  // namespace

extern "C" int ivr_blend_bwd(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                             int32_t nty, const float *rec, const float *values,
                             const double *rec64, int32_t k, int32_t width, int32_t height,
                             const double *t_final, const int32_t *last_pos, const float *d_out,
                             float *g_values, float *g_mean2d, float *g_conic, float *g_opacity,
                             const int32_t *tile_order, int32_t flags, ivr_stream_t stream) {
    return blend_bwd_impl(tile_ranges, pair_splat, ntx, nty, rec, values, rec64, k, width, height,
                          t_final, last_pos, d_out, g_values, g_mean2d, g_conic, g_opacity,
                          tile_order, flags, nullptr, stream);
}

extern "C" size_t ivr_blend_bwd_det_workspace_size(int64_t pair_capacity, int32_t k) {
    if (pair_capacity < 0 || k < 1 || k > 32) return 0;
    return (size_t)pair_capacity * (ivr::kBwdThreads / 32) * (size_t)(k + 6) * sizeof(float);
}

extern "C" int ivr_blend_bwd_deterministic(
    const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx, int32_t nty,
    const float *rec, const float *values, const double *rec64, int32_t k, int32_t width,
    int32_t height, const double *t_final, const int32_t *last_pos, const float *d_out,
    int64_t n, const uint64_t *depth_key, const int32_t *count, const uint16_t *rect,
    int64_t pair_capacity, void *workspace, size_t workspace_bytes, float *g_values,
    float *g_mean2d, float *g_conic, float *g_opacity, const int32_t *tile_order, int32_t flags,
    ivr_stream_t stream) {
    using namespace ivr;
    const size_t need = ivr_blend_bwd_det_workspace_size(pair_capacity, k);
    if (n < 0 || !depth_key || !count || !rect || pair_capacity < 1 ||
        pair_capacity > 0x7fffffffll || !workspace || workspace_bytes < need) {
        set_error("ivr_blend_bwd_deterministic: bad argument or workspace too small");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(workspace, 0, need, st) != cudaSuccess) {
        set_error("ivr_blend_bwd_deterministic: memset failed");
        return IVR_ERR_CUDA;
    }
    const int rc = blend_bwd_impl(tile_ranges, pair_splat, ntx, nty, rec, values, rec64, k, width,
                                  height, t_final, last_pos, d_out, g_values, g_mean2d, g_conic,
                                  g_opacity, tile_order, flags, (float *)workspace, stream);
    if (rc != IVR_OK || n == 0) return rc;
    bwd_reduce_det_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
        n, k, depth_key, count, (const ushort4 *)rect, tile_ranges, pair_splat, ntx,
        pair_capacity, (const float *)workspace, g_values, g_mean2d, g_conic, g_opacity);
    return check_launch("bwd_reduce_det_kernel");
}

// per-pair gradients (the reference's composite_backward outputs): the 8
// warp partials of each list entry summed in warp order
__global__ void __launch_bounds__(256)
pair_sum_kernel(const float *part, int64_t npairs, int stride, float *pair_out) {
    const int64_t q = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (q >= npairs * stride) return;
    const int64_t j = q / stride, c = q % stride;
    float t = 0.0f;
    constexpr int kW = ivr::kBwdThreads / 32;
    for (int w = 0; w < kW; ++w) t += part[(j * kW + w) * stride + c];
    pair_out[q] = t;
}

extern "C" int ivr_blend_bwd_pairs(const int32_t *tile_ranges, const int32_t *pair_splat,
                                   int32_t ntx, int32_t nty, const float *rec,
                                   const float *values, const double *rec64, int32_t k,
                                   int32_t width, int32_t height, const double *t_final,
                                   const int32_t *last_pos, const float *d_out, int64_t n_pairs,
                                   void *workspace, size_t workspace_bytes, float *pair_grads,
                                   ivr_stream_t stream) {
    using namespace ivr;
    const size_t need = ivr_blend_bwd_det_workspace_size(n_pairs, k);
    if (n_pairs < 0 || n_pairs > 0x7fffffffll || !pair_grads || !workspace ||
        workspace_bytes < need) {
        set_error("ivr_blend_bwd_pairs: bad argument or workspace too small");
        return IVR_ERR_ARG;
    }
    if (n_pairs == 0) return IVR_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(workspace, 0, need, st) != cudaSuccess) {
        set_error("ivr_blend_bwd_pairs: memset failed");
        return IVR_ERR_CUDA;
    }
    // the walk only writes the partials in this mode; the per-Gaussian
    // accumulator arguments are never touched (any valid pointer passes)
    const int rc = blend_bwd_impl(tile_ranges, pair_splat, ntx, nty, rec, values, rec64, k,
                                  width, height, t_final, last_pos, d_out, pair_grads, pair_grads,
                                  pair_grads, pair_grads, nullptr, 0, (float *)workspace, stream);
    if (rc != IVR_OK) return rc;
    const int stride = k + 6;
    const int64_t tot = n_pairs * stride;
    pair_sum_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>((const float *)workspace,
                                                                   n_pairs, stride, pair_grads);
    return check_launch("pair_sum_kernel");
}

extern "C" int64_t ivr_preprocess_bwd_scratch_len(int64_t n, int32_t per_scene) {
    if (n < 0 || per_scene < 0) return 0;
    return ((n + 127) / 128) * (int64_t)(10 + 4 * per_scene);
}

extern "C" int ivr_preprocess_bwd(const ivr_gaussians *g, const ivr_shading *shading,
                                  const ivr_edits *edits, const ivr_frame_params *params,
                                  const ivr_camera *cam, const ivr_layout *layout, ivr_grads *grads,
                                  int32_t geometry, ivr_stream_t stream) {
    using namespace ivr;
    if (!g || !layout || !grads || (!params && !cam) || g->n < 0 || grads->per_scene < 0 ||
        grads->per_scene > 1024) {
        set_error("ivr_preprocess_bwd: bad argument");
        return IVR_ERR_ARG;
    }
    if (g->n == 0) return IVR_OK;
    if (grads->scratch &&
        grads->scratch_len < ivr_preprocess_bwd_scratch_len(g->n, grads->per_scene)) {
        set_error("ivr_preprocess_bwd: scratch too small");
        return IVR_ERR_ARG;
    }
    BwdConst B{};
    B.G = *g;
    if (geometry) B.G.cache = nullptr;  // the geometry chain needs q, s, R (not cached)
    if (shading) B.S = *shading;
    B.has_shading = shading != nullptr;
    if (edits) B.E = *edits;
    B.has_edits = edits != nullptr;
    B.L = *layout;
    B.R = *grads;
    B.geometry = geometry;
    ivr_frame_params Pv{};
    if (!params) {
        Pv = params_from(*cam, shading, edits);
        for (int k = 0; k < 3; ++k) {
            Pv.dl_dp[k] = grads->dl_dp[k];
            Pv.dl_da[k] = grads->dl_da[k];
        }
    }
    const int threads = 128;
    const unsigned blocks = (unsigned)((g->n + threads - 1) / threads);
    const size_t sm = (size_t)grads->per_scene * 4 * sizeof(double);
    if (geometry)
        ivr::launch<3>(preprocess_bwd_kernel<true>, blocks, threads, sm, (cudaStream_t)stream, B, Pv, params);
    else
        ivr::launch<3>(preprocess_bwd_kernel<false>, blocks, threads, sm, (cudaStream_t)stream, B, Pv, params);
    if (grads->scratch) {
        const int nsl = 10 + 4 * grads->per_scene;
        bwd_sums_kernel<<<nsl, 256, 0, (cudaStream_t)stream>>>(
            grads->scratch, (int)blocks, grads->per_scene, shading ? 1 : 0, grads->d_globals,
            grads->per_scene > 0 ? grads->d_c_p : nullptr, grads->d_scale);
    }
    return check_launch("preprocess_bwd_kernel");
}
