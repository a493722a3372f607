// K3 -- per-tile front-to-back alpha blend (forward).
//
// Replaces _kernels.composite_forward (_kernels.py:31-72).  Two CTAs per 16x16
// tile (tiles launched heaviest-first when a tile order is given), one thread
// per pixel, and each warp an independent 8x4 block: the warp streams the
// tile's depth-sorted pair list in chunks of 32, culls every pair against its
// own strip (a rigorous float32 lower bound of the exponent over the strip vs
// the record's skip bound; bit 31 of a pair id = already culled for the tile
// by ivr_bin_sort_cull), stashes survivors in per-warp shared slots and walks
// them in list order.  Each pixel therefore visits exactly the reference list
// minus provably skipped pairs, and a warp retires as soon as its 32 pixels
// have passed T < 1e-4 -- there is no CTA-wide barrier.
//
// Decisions (sigma < 0, alpha < 1/255, T < 1e-4) must match the reference's
// float64 arithmetic exactly: a flipped alpha-skip moves a pixel by
// ~T/255 >> 1e-4 (SURVEY.md finding 4).  Two modes:
//  * EXACT: every non-skipped pair is re-evaluated with the reference's
//    float64 arithmetic (separately rounded, exp, cap, skip, T *= 1-alpha,
//    float32 accumulation rounding) -> bit-faithful images.
//  * FAST: the exponent is evaluated in float32 with a rigorous
//    per-evaluation error bound E.  Pairs certainly on one side of the
//    alpha-skip threshold take float32 alpha; only pairs inside the band take
//    the exact float64 path.  T is tracked in float32 with a running relative
//    error bound; a pixel whose T lands inside its band around 1e-4 is
//    flagged, and its warp re-walks the list once in EXACT mode for the
//    flagged pixels only.  Decisions therefore match the reference; values
//    carry float32 rounding (~1e-6 against the 1e-4 tolerance).
#include <math.h>
#include <stdlib.h>

#include "cull.cuh"

// K3 FAST walk: pair ids through the bulk-copy engine (A/B switch, see
// warp_walk_staged)
#ifndef IVR_K3_BULK_IDS
#define IVR_K3_BULK_IDS 0
#endif

namespace ivr {

constexpr int kBlendThreads = 256;  // one tile's 8 blocks (the CTA may hold a part of them)
constexpr int kCtaWarps = 4;        // warps (8x4 blocks) per K3 CTA
// Warp footprint width: 8 -> 8x4 pixel blocks (less perimeter per pixel than
// 16x2, so more lanes fall inside a footprint that touches the warp).
constexpr int kWarpW = 8;
constexpr int kModeExact = 0;
constexpr int kModeFast = 1;
// |sigma32 - sigma_ref| <= kSigmaErr * (|a/2 dx^2| + |b dx dy| + |c/2 dy^2|):
// 5 roundings per term + dx/dy rounding (5.1 ulp) + float32 conic rounding in
// dtype=float64 mode (1 ulp), with slack: 6.7 ulp of 2^-24.
constexpr float kSigmaErr = 4.0e-7f;

// Can splat (record r0, r1) reach alpha >= 1/255 anywhere in the pixel
// rectangle [px0, px1] x [py0, py1]?  Conservative: true unless the float64
// minimum of the exponent over the rectangle exceeds hi (>= ln(255 o) + margins).
__device__ __forceinline__ bool tile_touch(const float4 r0, const float4 r1, int px0, int px1,
                                           int py0, int py1) {
    const double hi = r0.w;
    if (!(hi < 1e30)) return true;
    const double a = 2.0 * (double)r1.x, b = r1.y, c = 2.0 * (double)r1.z;
    if (!(a > 0.0 && c > 0.0 && a * c - b * b > 0.0)) return true;
    const double mx = r0.x, my = r0.y;
    const double ex0 = px0 - mx, ex1 = px1 - mx, ey0 = py0 - my, ey1 = py1 - my;
    if (ex0 <= 0.0 && ex1 >= 0.0 && ey0 <= 0.0 && ey1 >= 0.0) return true;
    const double ia = 1.0 / a, ic = 1.0 / c;
    double best = 1e300;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double e = k ? ex1 : ex0;
        double dy = -b * e * ic;
        dy = dy < ey0 ? ey0 : (dy > ey1 ? ey1 : dy);
        const double s = 0.5 * (a * e * e + c * dy * dy) + b * e * dy;
        best = s < best ? s : best;
        const double f = k ? ey1 : ey0;
        double dx = -b * f * ia;
        dx = dx < ex0 ? ex0 : (dx > ex1 ? ex1 : dx);
        const double t = 0.5 * (a * dx * dx + c * f * f) + b * dx * f;
        best = t < best ? t : best;
    }
    return !(best > hi);
}

// Reference alpha for one (pixel, splat) in float64 (_kernels.py:51-61);
// returns a negative value when the reference skips the pair.
__device__ __forceinline__ double exact_alpha(double dpx, double dpy, double mx, double my,
                                              double ca, double cb, double cc, double o) {
    const double ddx = dsub(dpx, mx), ddy = dsub(dpy, my);
    const double sg = dadd(dmul(0.5, dadd(dmul(dmul(ca, ddx), ddx), dmul(dmul(cc, ddy), ddy))),
                           dmul(dmul(cb, ddx), ddy));
    if (sg < 0.0) return -1.0;
    double al = dmul(o, exp(-sg));
    if (al > kAlphaCap) al = kAlphaCap;
    if (al < kAlphaSkip) return -1.0;
    return al;
}

// MUFU.EX2 / MUFU.RCP without the denormal-range fix-ups of exp2f/__fdividef
// (arguments here are far from the denormal range; error bounds below assume
// the approx instructions' ~2 ulp)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct BlendArgs {
    const int32_t *ranges;
    const int32_t *pair_splat;
    int ntx;
    const float4 *rec;
    const float *values;
    const double *rec64;
    const double *values64;
    int K, W, H;
    float *out;
    double *out64;
    int32_t *contrib, *last_pos;
    double *t_final;
    const int32_t *tile_order;
    int preculled;
    long long *trace;  // debug: per (tile, block) {tile, smid, t0, t1} (globaltimer), or null
#if IVR_K3_BULK_IDS
    int ntx_nty;       // tile count: ranges[ntx_nty] = pairs in the frame
    int *bulk_fault;   // set when a bulk id copy never completed
#endif
};

template <int KMAX, bool F64>
struct PixelState {
    double T;     // EXACT: float64 transmittance (reference arithmetic)
    float Tf;     // FAST: float32 transmittance
    float errT;   // FAST: 1e-4 x bound on |Tf / T_ref - 1|
    float acc[KMAX];
    double acc64[F64 ? KMAX : 1];
    int nc, last;
    bool done, replay;

    __device__ __forceinline__ void reset(int s0, bool done0) {
        T = 1.0;
        Tf = 1.0f;
        errT = 0.0f;
#pragma unroll
        for (int c = 0; c < KMAX; ++c) acc[c] = 0.0f;
#pragma unroll
        for (int c = 0; c < (F64 ? KMAX : 1); ++c) acc64[c] = 0.0;
        nc = 0;
        last = s0;
        done = done0;
        replay = false;
    }
};

// Per-warp staging slots: one 32-pair chunk of the tile list at a time.
template <int KMAX, bool F64, int MODE>
struct WarpSlots {
    float4 r0[32], r1[32];
    float v[32 * KMAX];
    double r64[F64 ? 32 * 6 : 1];                           // mx, my, a, b, c, o
    float2 lo[F64 ? 32 : 1];  // FAST float64 mode: mean - float32(mean), per pair
    int sp[F64 ? 32 : 1];     // FAST float64 mode: splat (band pairs read rec64 lazily)
    double v64[(F64 && MODE == kModeExact) ? 32 * KMAX : 1];
};

// One warp = one 8x4 pixel block of the tile.  The warp streams the tile's pair
// list in chunks of 32 (one pair per lane): load id + record, cull against the
// strip rectangle (rigorous float32 bound), stash survivors in its own shared
// slots, then every lane walks the survivors in list order for its pixel.
// No CTA barrier anywhere: each warp retires as soon as its 32 pixels have
// passed T < 1e-4, and the next chunk's ids and records are prefetched into
// registers while the current chunk is walked.
template <int KMAX, bool F64, int MODE, int WMODE>
__device__ __forceinline__ void warp_walk(const BlendArgs &A, WarpSlots<KMAX, F64, WMODE> &W,
                                          int s0, int s1, int px, int py, int sx0, int sx1,
                                          int sy0, int sy1, PixelState<KMAX, F64> &st) {
    const int lane = threadIdx.x & 31;
    const int K = A.K;
    const float fpx = (float)px, fpy = (float)py;
    const double dpx = (double)px, dpy = (double)py;
    int sp = 0;
    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
    constexpr int KPF = KMAX <= 4 ? KMAX : 0;  // values prefetched with the record (K <= 4)
    float pv[KPF > 0 ? KPF : 1];
    // two-stage prefetch: a chunk's pair ids are loaded one chunk before its
    // records, so the dependent id -> record round trips of the list stream
    // overlap two walks instead of one (bit 31 of an id: culled for this tile
    // by ivr_bin_sort_cull; -1 past the list end)
    auto fetch_ids = [&](int base) {
        const int j = base + lane;
        return j < s1 ? __ldg(A.pair_splat + j) : -1;
    };
    auto fetch_recs = [&](int id) {
        sp = id;
        if (id >= 0) {
            r0 = __ldg(A.rec + 2 * id);
            r1 = __ldg(A.rec + 2 * id + 1);
#pragma unroll
            for (int c = 0; c < KPF; ++c) pv[c] = c < K ? __ldg(A.values + (int64_t)K * id + c) : 0.0f;
        }
    };
    int spn = -1;  // ids of the next chunk
    if (s0 < s1) {
        fetch_recs(fetch_ids(s0));
        if (s0 + 32 < s1) spn = fetch_ids(s0 + 32);
    }
    for (int base = s0; base < s1; base += 32) {
        if (__all_sync(0xffffffffu, st.done)) break;
        const int j = base + lane;
        bool keep = false;
        if (j < s1) {
            keep = sp >= 0 && !tile_cull32(r0, r1, sx0, sx1, sy0, sy1);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            W.r0[lane] = r0;
            // FAST mode reads thr_lo = thr - (thr rounding + margins) in place of thr
            W.r1[lane] = MODE == kModeFast
                             ? make_float4(r1.x, r1.y, r1.z, r1.w - (2.4e-7f * fabsf(r1.w) + 1e-7f))
                             : r1;
            if (KPF > 0) {
#pragma unroll
                for (int c = 0; c < KPF; ++c) W.v[lane * KMAX + c] = pv[c];
            } else {
                const float *v = A.values + (int64_t)K * sp;
#pragma unroll
                for (int c = 0; c < KMAX; ++c)  // zero-padded to KMAX: no channel predicates below
                    W.v[lane * KMAX + c] = c < K ? __ldg(v + c) : 0.0f;
            }
            if (F64) {
                const double *r = A.rec64 + 8 * (int64_t)sp;
                if (MODE == kModeExact) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) W.r64[lane * 6 + c] = __ldg(r + c);
                } else {
                    // mean - float32(mean) is exact in float64 and tiny: the
                    // candidate dx = (px - mx32) - lo carries <= ~1 ulp (the
                    // error bound budgets 5 ulp for dx)
                    W.lo[lane] = make_float2((float)(__ldg(r) - (double)r0.x),
                                             (float)(__ldg(r + 1) - (double)r0.y));
                    W.sp[lane] = sp;
                }
                if (MODE == kModeExact) {  // FAST walks accumulate the float32 values
                    const double *v64 = A.values64 + (int64_t)K * sp;
#pragma unroll
                    for (int c = 0; c < KMAX; ++c) W.v64[lane * KMAX + c] = c < K ? __ldg(v64 + c) : 0.0;
                }
            }
        }
        __syncwarp();
        if (base + 32 < s1) {  // prefetch during the walk: next records, ids after that
            fetch_recs(spn);
            spn = base + 64 < s1 ? fetch_ids(base + 64) : -1;
        }
        uint32_t mbits = st.done ? 0u : m;
        while (mbits) {
            const int q = __ffs(mbits) - 1;
            mbits &= mbits - 1;
            const float4 a0 = W.r0[q];
            const float4 a1 = W.r1[q];
            const float dx = fpx - a0.x, dy = fpy - a0.y;
            const float bdy = a1.y * dy, hcdy = a1.z * dy;
            const float sig = fmaf(fmaf(a1.x, dx, bdy), dx, hcdy * dy);
            if (sig > a0.w) continue;  // reference alpha < 1/255 for certain
            if (MODE == kModeExact) {
                double al;
                if (F64) {
                    const double *r = W.r64 + q * 6;
                    al = exact_alpha(dpx, dpy, r[0], r[1], r[2], r[3], r[4], r[5]);
                } else {
                    al = exact_alpha(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                     2.0 * (double)a1.z, a0.z);
                }
                if (al < 0.0) continue;
                const double w = dmul(st.T, al);
                if (F64) {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c)
                        st.acc64[c] = dadd(st.acc64[c], dmul(w, W.v64[q * KMAX + c]));
                } else {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c)
                        st.acc[c] = (float)dadd((double)st.acc[c], dmul(w, (double)W.v[q * KMAX + c]));
                }
                st.T = dmul(st.T, dsub(1.0, al));
                ++st.nc;
                st.last = base + q + 1;
                if (st.T < kTStop) {
                    st.done = true;
                    break;
                }
            } else {
                // candidate: in dtype=float64 mode recompute dx, dy from the float64 mean
                float cdx = dx, cdy = dy, cbdy = bdy, chcdy = hcdy, csig = sig;
                if (F64) {
                    const float2 lo = W.lo[q];
                    cdx = dx - lo.x;
                    cdy = dy - lo.y;
                    cbdy = a1.y * cdy;
                    chcdy = a1.z * cdy;
                    csig = fmaf(fmaf(a1.x, cdx, cbdy), cdx, chcdy * cdy);
                }
                const float terms = fmaf(a1.x * cdx, cdx, fmaf(chcdy, cdy, fabsf(cbdy * cdx)));
                const float E = kSigmaErr * terms + 1e-30f;
                float al, dal;  // alpha and a bound on |dAlpha| (absolute)
                if (csig - E > 0.0f && csig + E < a1.w) {  // a1.w = thr_lo (staged)
                    const float au = a0.z * ex2_approx(-1.4426950408889634f * csig);
                    // relative error: sigma bound, argument rounding, ex2.approx, * o
                    const float rel = E + 1.2e-7f * csig + 3.6e-7f;
                    // au certainly above the cap: the reference capped too (alpha =
                    // 0.99, |0.99f - 0.99| < 1.1e-8); otherwise the f32 error bound
                    const bool capped = au > 0.99f * (1.0f + rel);
                    al = fminf(au, 0.99f);
                    dal = capped ? 1.1e-8f : au * rel;
                } else if (csig - E > a0.w) {
                    continue;  // certainly skipped: sigma_ref >= csig - E > hi >= thr_ref
                } else {
                    double ad;
                    if (F64) {
                        const double *r = A.rec64 + 8 * (int64_t)W.sp[q];
                        ad = exact_alpha(dpx, dpy, __ldg(r), __ldg(r + 1), __ldg(r + 2),
                                         __ldg(r + 3), __ldg(r + 4), __ldg(r + 5));
                    } else {
                        ad = exact_alpha(dpx, dpy, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                         2.0 * (double)a1.z, a0.z);
                    }
                    if (ad < 0.0) continue;
                    al = (float)ad;
                    dal = 6e-8f * al;
                }
                const float w = st.Tf * al;
                if (KMAX % 4 == 0) {
                    const float4 *vv = reinterpret_cast<const float4 *>(W.v + q * KMAX);
#pragma unroll
                    for (int c4 = 0; c4 < KMAX / 4; ++c4) {
                        const float4 v = vv[c4];
                        st.acc[4 * c4] = fmaf(w, v.x, st.acc[4 * c4]);
                        st.acc[4 * c4 + 1] = fmaf(w, v.y, st.acc[4 * c4 + 1]);
                        st.acc[4 * c4 + 2] = fmaf(w, v.z, st.acc[4 * c4 + 2]);
                        st.acc[4 * c4 + 3] = fmaf(w, v.w, st.acc[4 * c4 + 3]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < KMAX; ++c) st.acc[c] = fmaf(w, W.v[q * KMAX + c], st.acc[c]);
                }
                const float om = 1.0f - al;
                st.Tf = st.Tf * om;
                // errT carried pre-scaled by 1e-4 (the stop threshold):
                // += 1e-4 * (dal / om * 1.01 + 1.3e-7); 1/om by MUFU.RCP, whose
                // error is covered by the 1.01 factor
                st.errT = fmaf(dal * rcp_approx(om), 1.01e-4f, st.errT + 1.3e-11f);
                ++st.nc;
                st.last = base + q + 1;
                if (st.Tf < 1.0000001e-4f + st.errT) {
                    st.done = true;  // certain stop, or ambiguous -> EXACT re-walk
                    st.replay = !(st.Tf < 0.9999999e-4f - st.errT);
                    break;
                }
            }
        }
        __syncwarp();  // slots are rewritten by the next chunk
    }
}

// ------------------------------------------------- FAST float32, K <= 4
// The same walk with the list records staged by asynchronous copies
// (cp.async, Ampere-style LDGSTS gathers: the records of a chunk are not
// contiguous, so a bulk/TMA copy does not apply) into a kStages-deep per-warp
// ring in shared memory: chunk c + kStages is requested as soon as chunk c
// has been walked, and its pair ids one chunk earlier, so two walks hide the
// dependent id -> record L2 round trips (the register prefetch of warp_walk
// hid one: ncu showed ~14% of K3's warp samples in long-scoreboard stalls
// at the chunk boundary), with no prefetch registers held across the walk.
constexpr int kStages = 3;

template <int KMAX>
struct StageBase {
    float4 r0[kStages][32], r1[kStages][32];
    float v[kStages][32 * KMAX];
#if IVR_K3_BULK_IDS
    int ids[2][40];                 // bulk-copied pair-id windows (36 ints used)
    unsigned long long bar[2];      // their mbarriers
#endif
};
template <int KMAX, bool F64 = false>
struct StageSlots : StageBase<KMAX> {};
// float64-decision mode: the float64 mean rides along (its float32 residual
// corrects dx, dy) and the splat id serves the band pairs' lazy float64 read
template <int KMAX>
struct StageSlots<KMAX, true> : StageBase<KMAX> {
    double2 m64[kStages][32];
    float2 lo[kStages][32];
    int sp[kStages][32];
};

#if IVR_K3_BULK_IDS
// Pair ids by the bulk-copy engine (cp.async.bulk + mbarrier): the ids of a
// chunk are contiguous, so lane 0 requests the 16-byte-aligned 144-byte
// window around them; the wait is bounded (a lost completion marks the
// frame bad instead of hanging the SM).
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(unsigned long long *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_inval(unsigned long long *b) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_ids(int *dst, const int32_t *src, unsigned long long *b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 144;" ::"r"(smem_u32(b)) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 144, [%2];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ bool bar_wait(unsigned long long *b, uint32_t phase) {
    for (int n = 0; n < (1 << 22); ++n) {
        uint32_t done;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(phase)
            : "memory");
        if (done) return true;
    }
    return false;
}
#endif

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// FAST float32 walk of one staged chunk: the survivors `mbits` (records r0,
// r1 with thr_lo in r1.w, values v zero-padded to KMAX) in list order for
// this lane's pixel; sets st.done (+ st.replay when ambiguous) at the stop.
template <int KMAX, bool F64 = false>
__device__ __forceinline__ void walk_chunk_fast(const float4 *r0s, const float4 *r1s,
                                                const float *vs, uint32_t mbits, int base, int px,
                                                int py, PixelState<KMAX, F64> &st,
                                                const float2 *los = nullptr,
                                                const int *sps = nullptr,
                                                const double *rec64 = nullptr) {
    const float fpx = (float)px, fpy = (float)py;
    while (mbits) {
        const int q = __ffs(mbits) - 1;
        mbits &= mbits - 1;
        const float4 a0 = r0s[q];
        const float4 a1 = r1s[q];
        const float dx = fpx - a0.x, dy = fpy - a0.y;
        const float bdy = a1.y * dy, hcdy = a1.z * dy;
        const float sig = fmaf(fmaf(a1.x, dx, bdy), dx, hcdy * dy);
        if (sig > a0.w) continue;  // reference alpha < 1/255 for certain
        // float64 decisions: dx, dy from the float64 mean (float32 residual)
        float cdx = dx, cdy = dy, cbdy = bdy, chcdy = hcdy, csig = sig;
        if (F64) {
            const float2 lo = los[q];
            cdx = dx - lo.x;
            cdy = dy - lo.y;
            cbdy = a1.y * cdy;
            chcdy = a1.z * cdy;
            csig = fmaf(fmaf(a1.x, cdx, cbdy), cdx, chcdy * cdy);
        }
        const float terms = fmaf(a1.x * cdx, cdx, fmaf(chcdy, cdy, fabsf(cbdy * cdx)));
        const float E = kSigmaErr * terms + 1e-30f;
        float al, dal;
        if (csig - E > 0.0f && csig + E < a1.w) {
            const float au = a0.z * ex2_approx(-1.4426950408889634f * csig);
            const float rel = E + 1.2e-7f * csig + 3.6e-7f;
            const bool capped = au > 0.99f * (1.0f + rel);
            al = fminf(au, 0.99f);
            dal = capped ? 1.1e-8f : au * rel;
        } else if (csig - E > a0.w) {
            continue;
        } else {
            double ad;
            if (F64) {
                const double *r = rec64 + 8 * (int64_t)sps[q];
                ad = exact_alpha((double)px, (double)py, __ldg(r), __ldg(r + 1), __ldg(r + 2),
                                 __ldg(r + 3), __ldg(r + 4), __ldg(r + 5));
            } else {
                ad = exact_alpha((double)px, (double)py, a0.x, a0.y, 2.0 * (double)a1.x, a1.y,
                                 2.0 * (double)a1.z, a0.z);
            }
            if (ad < 0.0) continue;
            al = (float)ad;
            dal = 6e-8f * al;
        }
        const float w = st.Tf * al;
        if (KMAX % 4 == 0) {
            const float4 *vv = reinterpret_cast<const float4 *>(vs + q * KMAX);
#pragma unroll
            for (int c4 = 0; c4 < KMAX / 4; ++c4) {
                const float4 v = vv[c4];
                st.acc[4 * c4] = fmaf(w, v.x, st.acc[4 * c4]);
                st.acc[4 * c4 + 1] = fmaf(w, v.y, st.acc[4 * c4 + 1]);
                st.acc[4 * c4 + 2] = fmaf(w, v.z, st.acc[4 * c4 + 2]);
                st.acc[4 * c4 + 3] = fmaf(w, v.w, st.acc[4 * c4 + 3]);
            }
        } else {
#pragma unroll
            for (int c2 = 0; c2 < KMAX; ++c2) st.acc[c2] = fmaf(w, vs[q * KMAX + c2], st.acc[c2]);
        }
        const float om = 1.0f - al;
        st.Tf = st.Tf * om;
        st.errT = fmaf(dal * rcp_approx(om), 1.01e-4f, st.errT + 1.3e-11f);
        ++st.nc;
        st.last = base + q + 1;
        if (st.Tf < 1.0000001e-4f + st.errT) {
            st.done = true;
            st.replay = !(st.Tf < 0.9999999e-4f - st.errT);
            return;
        }
    }
}

template <int KMAX, bool F64 = false>
__device__ __forceinline__ void warp_walk_staged(const BlendArgs &A, StageSlots<KMAX, F64> &S,
                                                 int s0, int s1, int px, int py, int sx0, int sx1,
                                                 int sy0, int sy1, PixelState<KMAX, F64> &st) {
    const int lane = threadIdx.x & 31;
    const int K = A.K;
    const int nch = (s1 - s0 + 31) >> 5;
    auto fetch_id = [&](int c) {
        const int j = s0 + 32 * c + lane;
        return c < nch && j < s1 ? __ldg(A.pair_splat + j) : -1;
    };
    // request chunk c's records (id < 0: culled for the tile or past the end)
    auto request = [&](int c, int id) {
        if (id >= 0) {
            const int g = c % kStages;
            cp_async16(&S.r0[g][lane], A.rec + 2 * id);
            cp_async16(&S.r1[g][lane], A.rec + 2 * id + 1);
            if constexpr (F64) cp_async16(&S.m64[g][lane], A.rec64 + 8 * (int64_t)id);
            if (KMAX == 4 && K == 4) {
                cp_async16(&S.v[g][lane * 4], A.values + 4 * (int64_t)id);
            } else {
#pragma unroll
                for (int c2 = 0; c2 < KMAX; ++c2)
                    if (c2 < K) cp_async4(&S.v[g][lane * KMAX + c2], A.values + (int64_t)K * id + c2);
            }
        }
        cp_async_commit();  // one group per chunk, possibly empty
    };
    int ids[kStages];  // ids[k]: pair ids of chunk c + k (constant indices: registers)
#pragma unroll
    for (int k = 0; k < kStages; ++k) ids[k] = fetch_id(k);
#pragma unroll
    for (int k = 0; k < kStages; ++k) request(k, ids[k]);
    int in = fetch_id(kStages);
#if IVR_K3_BULK_IDS
    // chunks q >= kStages + 1 come through the bulk ring: slot (q - q0) & 1,
    // parity ((q - q0) >> 1) & 1; a chunk whose 144-byte window would read
    // past the frame's last pair is loaded directly instead
    constexpr int q0 = kStages + 1;
    const int n_all = A.ranges[A.ntx_nty];
    auto bulk_ok = [&](int q) { return q < nch && ((s0 + 32 * q) & ~3) + 36 <= n_all; };
    auto bulk_issue = [&](int q) {
        if (lane == 0 && bulk_ok(q))
            bulk_ids(S.ids[(q - q0) & 1], A.pair_splat + ((s0 + 32 * q) & ~3), &S.bar[(q - q0) & 1]);
    };
    if (lane == 0) {
        bar_init(&S.bar[0]);
        bar_init(&S.bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    bulk_issue(q0);
    bulk_issue(q0 + 1);
    int c_end = 0;
#endif
    for (int c = 0; c < nch; ++c) {
        if (__all_sync(0xffffffffu, st.done)) break;
        cp_async_wait<kStages - 1>();  // this lane's copies of chunk c landed
        __syncwarp();                  // ... and every lane's
        const int g = c % kStages;
        const int base = s0 + 32 * c;
        bool keep = false;
        if (ids[0] >= 0) {
            const float4 r0 = S.r0[g][lane], r1 = S.r1[g][lane];
            keep = !tile_cull32(r0, r1, sx0, sx1, sy0, sy1);
            // the walk reads thr_lo = thr - (thr rounding + margins) in place of thr
            if (keep) S.r1[g][lane].w = r1.w - (2.4e-7f * fabsf(r1.w) + 1e-7f);
            if constexpr (F64) {
                if (keep) {  // mean - float32(mean): exact in float64, tiny
                    const double2 m = S.m64[g][lane];
                    S.lo[g][lane] = make_float2((float)(m.x - (double)r0.x), (float)(m.y - (double)r0.y));
                    S.sp[g][lane] = ids[0];
                }
            }
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if constexpr (F64)
            walk_chunk_fast<KMAX, true>(S.r0[g], S.r1[g], S.v[g], st.done ? 0u : m, base, px, py,
                                        st, S.lo[g], S.sp[g], A.rec64);
        else
            walk_chunk_fast<KMAX>(S.r0[g], S.r1[g], S.v[g], st.done ? 0u : m, base, px, py, st);
        __syncwarp();  // every lane is done reading stage g
        request(c + kStages, in);
#pragma unroll
        for (int k = 0; k + 1 < kStages; ++k) ids[k] = ids[k + 1];
        ids[kStages - 1] = in;
#if IVR_K3_BULK_IDS
        {
            const int q = c + kStages + 1;
            if (bulk_ok(q)) {
                const int sl = (q - q0) & 1;
                if (!bar_wait(&S.bar[sl], (uint32_t)(((q - q0) >> 1) & 1))) {
                    if (lane == 0) atomicExch(A.bulk_fault, 1);
                    in = -1;
                } else {
                    const int j = s0 + 32 * q + lane;
                    in = j < s1 ? S.ids[sl][((s0 + 32 * q) & 3) + lane] : -1;
                }
                __syncwarp();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_issue(q + 2);
            } else {
                in = fetch_id(q);
            }
        }
        c_end = c + 1;
#else
        in = fetch_id(c + kStages + 1);
#endif
    }
#if IVR_K3_BULK_IDS
    // drain the (at most two) bulk copies issued but not consumed
    for (int q = c_end + kStages + 1; q <= c_end + kStages + 2; ++q) {
        if (bulk_ok(q) && !bar_wait(&S.bar[(q - q0) & 1], (uint32_t)(((q - q0) >> 1) & 1)) && lane == 0)
            atomicExch(A.bulk_fault, 1);
    }
    __syncwarp();
    if (lane == 0) {
        bar_inval(&S.bar[0]);
        bar_inval(&S.bar[1]);
    }
#endif
    asm volatile("cp.async.wait_all;" ::: "memory");  // the ring may be reused (EXACT re-walk)
    __syncwarp();
}

// Wide values (FAST, 4 < K <= 16, e.g. the K=15 training forward): records
// go through the same ring, but a chunk's values (up to 64 B per pair) are
// requested only for the pairs that survive the 8x4 cull, one chunk ahead:
// at step c the warp culls chunk c + 1 (its records are in), requests those
// survivors' values, walks chunk c (values requested at step c - 1) and then
// refills chunk c's record slot with chunk c + 3.  Copy groups per step:
// values(c + 1), then records(c + 3), so `wait_group 1` at the top of step c
// leaves only records(c + 2) in flight.
template <int KMAX>
__device__ __forceinline__ void warp_walk_staged_sv(const BlendArgs &A, StageSlots<KMAX> &S,
                                                    int s0, int s1, int px, int py, int sx0,
                                                    int sx1, int sy0, int sy1,
                                                    PixelState<KMAX, false> &st) {
    static_assert(kStages == 3, "the copy-group schedule assumes a 3-deep ring");
    const int lane = threadIdx.x & 31;
    const int K = A.K;
    const int nch = (s1 - s0 + 31) >> 5;
    auto fetch_id = [&](int c) {
        const int j = s0 + 32 * c + lane;
        return c < nch && j < s1 ? __ldg(A.pair_splat + j) : -1;
    };
    auto request_rec = [&](int c, int id) {
        if (id >= 0) {
            const int g = c % kStages;
            cp_async16(&S.r0[g][lane], A.rec + 2 * id);
            cp_async16(&S.r1[g][lane], A.rec + 2 * id + 1);
        }
        cp_async_commit();
    };
    auto request_val = [&](int c, int id, bool keep) {
        if (keep) {
            const int g = c % kStages;
            const float *v = A.values + (int64_t)K * id;
#pragma unroll
            for (int c2 = 0; c2 < KMAX; ++c2)
                if (c2 < K) cp_async4(&S.v[g][lane * KMAX + c2], v + c2);
        }
        cp_async_commit();
    };
    // cull chunk c against the block (records in), stage thr_lo for the walk
    auto cull = [&](int c, int id) {
        bool keep = false;
        if (id >= 0) {
            const int g = c % kStages;
            const float4 r0 = S.r0[g][lane], r1 = S.r1[g][lane];
            keep = !tile_cull32(r0, r1, sx0, sx1, sy0, sy1);
            if (keep) S.r1[g][lane].w = r1.w - (2.4e-7f * fabsf(r1.w) + 1e-7f);
        }
        return keep;
    };
    int ids[kStages];
#pragma unroll
    for (int k = 0; k < kStages; ++k) ids[k] = fetch_id(k);
#pragma unroll
    for (int k = 0; k < kStages; ++k) request_rec(k, ids[k]);
    int in = fetch_id(kStages);
    cp_async_wait<kStages - 1>();  // records of chunk 0
    __syncwarp();
    const bool k0 = cull(0, ids[0]);
    uint32_t m_cur = __ballot_sync(0xffffffffu, k0);  // survivors of the chunk walked next
    __syncwarp();
    request_val(0, ids[0], k0);
    for (int c = 0; c < nch; ++c) {
        if (__all_sync(0xffffffffu, st.done)) break;
        if (c == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        else cp_async_wait<1>();
        __syncwarp();
        const int g = c % kStages;
        // cull the next chunk and request its survivors' values
        bool kn = false;
        if (c + 1 < nch) kn = cull(c + 1, ids[1]);
        const uint32_t m_next = __ballot_sync(0xffffffffu, kn);
        __syncwarp();
        request_val(c + 1, ids[1], kn);
        walk_chunk_fast<KMAX>(S.r0[g], S.r1[g], S.v[g], st.done ? 0u : m_cur, s0 + 32 * c, px, py, st);
        __syncwarp();  // every lane is done reading chunk c's slots
        request_rec(c + kStages, in);
#pragma unroll
        for (int k = 0; k + 1 < kStages; ++k) ids[k] = ids[k + 1];
        ids[kStages - 1] = in;
        in = fetch_id(c + kStages + 1);
        m_cur = m_next;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // the ring may be reused (EXACT re-walk)
    __syncwarp();
}

template <int KMAX, bool F64, int MODE>
constexpr bool kStaged = MODE == kModeFast && (F64 ? KMAX <= 4 : KMAX <= 16);

template <int KMAX, bool F64, int MODE>
__global__ void __launch_bounds__(kBlendThreads, (KMAX <= 4 && !F64) ? 4 : 3)
blend_fwd_kernel(BlendArgs A) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    using Slots = WarpSlots<KMAX, F64, kModeExact>;  // EXACT layout also serves FAST
    // per-warp region: WarpSlots, or (staged FAST walk) the StageSlots ring
    constexpr size_t kRegion =
        (kStaged<KMAX, F64, MODE> && sizeof(StageSlots<KMAX, F64>) > sizeof(Slots))
            ? sizeof(StageSlots<KMAX, F64>) : sizeof(Slots);
    Slots &W = *reinterpret_cast<Slots *>(smem + (threadIdx.x >> 5) * kRegion);

    // a CTA holds blockDim.x / 32 of the tile's 8 blocks (the warps are
    // independent: no CTA barrier), so CTAs can be narrower than a tile
    const int cpt = (kBlendThreads / 32) / (blockDim.x >> 5);  // CTAs per tile
    const int trank = blockIdx.x / cpt;
    const int tile = A.tile_order ? A.tile_order[trank] : trank;
    const int tx = tile % A.ntx, ty = tile / A.ntx;
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = (blockIdx.x % cpt) * (blockDim.x >> 5) + (tid >> 5);  // block of the tile
    // warp footprint kWarpW x (32 / kWarpW) pixels; lane -> (lane % kWarpW, lane / kWarpW)
    constexpr int kWarpH = 32 / kWarpW, kPerRow = kTile / kWarpW;
    const int sx0 = tx * kTile + kWarpW * (warp % kPerRow);
    const int sy_raw = ty * kTile + kWarpH * (warp / kPerRow);
    const int px = sx0 + (lane % kWarpW), py = sy_raw + lane / kWarpW;
    const bool inside = px < A.W && py < A.H;
    const int s0 = A.ranges[tile], s1 = A.ranges[tile + 1];
    const int sx1 = min(sx0 + kWarpW - 1, A.W - 1);
    const int sy0 = min(sy_raw, A.H - 1), sy1 = min(sy_raw + kWarpH - 1, A.H - 1);

    long long t_start = 0;
    if (A.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    PixelState<KMAX, F64> st;
    st.reset(s0, !inside);
    if constexpr (kStaged<KMAX, F64, MODE>) {
        // the ring aliases the warp's WarpSlots region (warp_walk runs after it)
        StageSlots<KMAX, F64> &S =
            *reinterpret_cast<StageSlots<KMAX, F64> *>(smem + (tid >> 5) * kRegion);
        if constexpr (KMAX <= 4)
            warp_walk_staged<KMAX, F64>(A, S, s0, s1, px, py, sx0, sx1, sy0, sy1, st);
        else if constexpr (!F64)
            warp_walk_staged_sv<KMAX>(A, S, s0, s1, px, py, sx0, sx1, sy0, sy1, st);
    } else {
        warp_walk<KMAX, F64, MODE, kModeExact>(A, W, s0, s1, px, py, sx0, sx1, sy0, sy1, st);
    }
    if (A.trace && lane == 0) {
        long long t_end;
        int sm_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
        long long *tr = A.trace + 4 * ((int64_t)tile * 8 + warp);
        tr[0] = tile;
        tr[1] = sm_;
        tr[2] = t_start;
        tr[3] = t_end;
    }
    bool exact_out = MODE == kModeExact;
    if (MODE == kModeFast) {
        // pixels whose T landed in the ambiguity band: one EXACT re-walk (per warp)
        const bool need = st.replay;
        if (__any_sync(0xffffffffu, need)) {
            PixelState<KMAX, F64> ex;
            ex.reset(s0, !need);
            warp_walk<KMAX, F64, kModeExact, kModeExact>(A, W, s0, s1, px, py, sx0, sx1, sy0, sy1,
                                                         ex);
            if (need) {
                st = ex;
                exact_out = true;
            }
        }
        if (!exact_out) st.T = (double)st.Tf;
    }
    if (!inside) return;
    const int64_t pix = (int64_t)py * A.W + px;
    const int K = A.K;
    if (F64) {
        double *o = A.out64 + pix * K;
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
            if (c < K) o[c] = exact_out ? st.acc64[c] : (double)st.acc[c];
    } else {
        float *o = A.out + pix * K;
        if (K == KMAX && KMAX % 4 == 0) {  // 16-byte aligned rows: vector stores
#pragma unroll
            for (int c4 = 0; c4 < KMAX / 4; ++c4)
                reinterpret_cast<float4 *>(o)[c4] =
                    make_float4(st.acc[4 * c4], st.acc[4 * c4 + 1], st.acc[4 * c4 + 2],
                                st.acc[4 * c4 + 3]);
        } else {
#pragma unroll
            for (int c = 0; c < KMAX; ++c)
                if (c < K) o[c] = st.acc[c];
        }
    }
    if (A.contrib) A.contrib[pix] = st.nc;
    if (A.last_pos) A.last_pos[pix] = st.last;
    if (A.t_final) A.t_final[pix] = st.T;
}

template <int KMAX, bool F64, int MODE>
size_t blend_smem_bytes() {
    const size_t slots = sizeof(WarpSlots<KMAX, F64, kModeExact>);
    const size_t ring = kStaged<KMAX, F64, MODE> ? sizeof(StageSlots<KMAX, F64>) : 0;
    return (kBlendThreads / 32) * (ring > slots ? ring : slots);
}

template <int KMAX, bool F64, int MODE>
int launch_blend(const BlendArgs &A, int ntiles, cudaStream_t st) {
    const size_t sm = blend_smem_bytes<KMAX, F64, MODE>();
    auto fn = blend_fwd_kernel<KMAX, F64, MODE>;
    if (sm > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // half-tile CTAs: a CTA's resources are held until its slowest warp is
    // done, so narrower CTAs release them sooner (C2 stream 3047 -> 3055 FPS,
    // C3 forward 0.539 -> 0.533 ms; 1-warp CTAs: K3 +4%)
    constexpr int wpc = kCtaWarps;
    const int cpt = (kBlendThreads / 32) / wpc;
    launch<3>(fn, ntiles * cpt, 32 * wpc, (sm / (kBlendThreads / 32)) * wpc, st, A);
    return check_launch("blend_fwd_kernel");
}

// ----------------------------------------------------------------- tile order
// Heaviest tiles first: a tile's CTA runtime grows with its pair count, and the
// longest tiles otherwise start in the last wave and set the frame's tail.
// The order is only a schedule (any permutation gives identical results), so
// a single-CTA counting sort on half-octave buckets of the pair count
// (descending) is enough: histogram, scan, scatter.
constexpr int kOrderBuckets = 64;

__global__ void __launch_bounds__(1024)
tile_order_kernel(const int32_t *ranges, int ntiles, int32_t *order) {
    __shared__ int s_hist[kOrderBuckets];
    if (threadIdx.x < kOrderBuckets) s_hist[threadIdx.x] = 0;
    __syncthreads();
    auto bucket = [](int cnt) {
        const int b = (int)(2.0f * __log2f((float)cnt + 1.0f));
        return kOrderBuckets - 1 - (b < kOrderBuckets - 1 ? b : kOrderBuckets - 1);
    };
    for (int t = threadIdx.x; t < ntiles; t += 1024) atomicAdd(&s_hist[bucket(ranges[t + 1] - ranges[t])], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int b = 0; b < kOrderBuckets; ++b) {
            const int c = s_hist[b];
            s_hist[b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += 1024)
        order[atomicAdd(&s_hist[bucket(ranges[t + 1] - ranges[t])], 1)] = t;
}

}  // namespace ivr

namespace {
long long *g_blend_trace = nullptr;  // debug hook only (tools/blend_trace.py)
}

// Debug: record {tile, smid, t_start, t_end} (ns, %globaltimer) per (tile,
// 8x4 block) of subsequent ivr_blend_fwd calls into buf (ntiles * 8 * 4
// int64), or stop with NULL.  Not for concurrent use.
extern "C" void ivr_debug_blend_trace(long long *buf) { g_blend_trace = buf; }

namespace ivr {
// Measured error of the two approximate MUFU instructions K3/K4 certify
// against (FAST mode): ex2.approx.ftz over every multiple of 2^-16 in
// [-126, 0] (alpha = o 2^(-sigma log2 e)) and rcp.approx.ftz over every
// float32 in [1/128, 1] (1 / (1 - alpha)), relative to float64; maxima as
// ordered bit patterns of positive doubles.
__global__ void mufu_err_kernel(unsigned long long *out) {
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double m_ex2 = 0.0, m_rcp = 0.0;
    for (int64_t k = t0; k <= 126ll << 16; k += stride) {
        const float x = -(float)k * 0x1p-16f;
        const double ref = exp2((double)x);
        const double rel = fabs((double)ex2_approx(x) - ref) / ref;
        m_ex2 = rel > m_ex2 ? rel : m_ex2;
    }
    const uint32_t lo = __float_as_uint(0x1p-7f), hi = __float_as_uint(1.0f);
    for (int64_t k = t0; k <= (int64_t)(hi - lo); k += stride) {
        const float x = __uint_as_float(lo + (uint32_t)k);
        const double ref = 1.0 / (double)x;
        const double rel = fabs((double)rcp_approx(x) - ref) / ref;
        m_rcp = rel > m_rcp ? rel : m_rcp;
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(m_ex2));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(m_rcp));
}

// Measured |sigma32 - sigma_ref| / (|a/2 dx^2| + |b dx dy| + |c/2 dy^2|) of
// the FAST walk's float32 exponent against the reference's float64 one on
// the same float32 record (random conics with condition <= 1e4, means up to
// 4096 px, pixels out to sigma ~ 40): the ratio kSigmaErr bounds.
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ float urand(uint32_t &st) {
    st = hash32(st + 0x9e3779b9U);
    return (float)(st >> 8) * 0x1p-24f;
}
__global__ void sigma_err_kernel(int64_t n, uint32_t seed, unsigned long long *out) {
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double worst = 0.0;
    for (int64_t i = t0; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t st = hash32((uint32_t)i * 2654435761u ^ seed);
        const float mx = 4096.0f * urand(st), my = 4096.0f * urand(st);
        const float a = exp2f(-13.0f + 16.0f * urand(st)), c = a * exp2f(-6.0f + 12.0f * urand(st));
        const float b = (2.0f * urand(st) - 1.0f) * 0.999f * sqrtf(a * c);
        // a pixel at exponent up to ~40 from the mean
        const float r = sqrtf(80.0f / fminf(a, c)) * urand(st), th = 6.2831853f * urand(st);
        const int px = (int)floorf(mx + r * cosf(th)), py = (int)floorf(my + r * sinf(th));
        // FAST walk (float32 record a/2, b, c/2)
        const float ha = 0.5f * a, hc = 0.5f * c;
        const float dx = (float)px - mx, dy = (float)py - my;
        const float bdy = b * dy, hcdy = hc * dy;
        const float sig = fmaf(fmaf(ha, dx, bdy), dx, hcdy * dy);
        // reference: float64 on the same float32 values
        const double ddx = (double)px - (double)mx, ddy = (double)py - (double)my;
        const double sref = 0.5 * ((double)a * ddx * ddx + (double)c * ddy * ddy) + (double)b * ddx * ddy;
        const double terms = 0.5 * (double)a * ddx * ddx + fabs((double)b * ddx * ddy) +
                             0.5 * (double)c * ddy * ddy;
        if (terms > 0.0) {
            const double q = fabs((double)sig - sref) / terms;
            worst = q > worst ? q : worst;
        }
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(worst));
}
}  // namespace ivr

// Debug / test: maximal |sigma32 - sigma_ref| / terms over n random
// (record, pixel) samples into out[0] (device, caller-zeroed).
extern "C" int ivr_debug_sigma_error(int64_t n, uint32_t seed, double *out, ivr_stream_t stream) {
    if (!out || n < 1) {
        ivr::set_error("ivr_debug_sigma_error: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::sigma_err_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
        n, seed, reinterpret_cast<unsigned long long *>(out));
    return ivr::check_launch("sigma_err_kernel");
}

// Debug / test: out (device, 2 doubles, caller-zeroed) receives the maximal
// relative errors of ex2.approx and rcp.approx over the ranges K3/K4 use.
extern "C" int ivr_debug_mufu_error(double *out, ivr_stream_t stream) {
    if (!out) {
        ivr::set_error("ivr_debug_mufu_error: bad argument");
        return IVR_ERR_ARG;
    }
    ivr::mufu_err_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<unsigned long long *>(out));
    return ivr::check_launch("mufu_err_kernel");
}

extern "C" int ivr_tile_order(const int32_t *tile_ranges, int32_t ntiles, int32_t *order,
                              ivr_stream_t stream) {
    using namespace ivr;
    if (!tile_ranges || !order || ntiles < 1) {
        set_error("ivr_tile_order: bad argument");
        return IVR_ERR_ARG;
    }
    tile_order_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(tile_ranges, ntiles, order);
    return check_launch("tile_order_kernel");
}

extern "C" int ivr_blend_fwd(const int32_t *tile_ranges, const int32_t *pair_splat, int32_t ntx,
                             int32_t nty, const float *rec, const float *values,
                             const double *rec64, const double *values64, int32_t k,
                             int32_t width, int32_t height, float *out, double *out64,
                             int32_t *contrib, int32_t *last_pos, double *t_final,
                             const int32_t *tile_order, int32_t flags, ivr_stream_t stream) {
    using namespace ivr;
    cudaStream_t st = (cudaStream_t)stream;
    if (!tile_ranges || !pair_splat || !rec || !values || k < 1 || k > 32 || width < 1 ||
        height < 1 || ntx != (width + kTile - 1) / kTile || nty != (height + kTile - 1) / kTile) {
        set_error("ivr_blend_fwd: bad argument");
        return IVR_ERR_ARG;
    }
    const bool f64 = out64 != nullptr;
    if (f64 ? (!rec64 || !values64) : (out == nullptr)) {
        set_error("ivr_blend_fwd: float64 mode needs rec64/values64/out64; float32 needs out");
        return IVR_ERR_ARG;
    }
    BlendArgs A;
    A.ranges = tile_ranges;
    A.pair_splat = pair_splat;
    A.ntx = ntx;
    A.rec = reinterpret_cast<const float4 *>(rec);
    A.values = values;
    A.rec64 = rec64;
    A.values64 = values64;
    A.K = k;
    A.W = width;
    A.H = height;
    A.out = out;
    A.out64 = out64;
    A.contrib = contrib;
    A.last_pos = last_pos;
    A.t_final = t_final;
    A.tile_order = tile_order;
    A.preculled = (flags & IVR_BLEND_PRECULLED) != 0 ? 1 : 0;
    A.trace = g_blend_trace;
#if IVR_K3_BULK_IDS
    A.ntx_nty = ntx * nty;
    static int *fault = nullptr;
    if (!fault) {
        cudaMalloc(&fault, sizeof(int));
        cudaMemset(fault, 0, sizeof(int));
    }
    A.bulk_fault = fault;
#endif
    const bool exact = (flags & IVR_BLEND_EXACT) != 0;
    const int nt = ntx * nty;
#define IVR_BLEND(KM)                                                                   \
    if (f64) {                                                                          \
        return exact ? launch_blend<KM, true, kModeExact>(A, nt, st)                    \
                     : launch_blend<KM, true, kModeFast>(A, nt, st);                    \
    }                                                                                   \
    return exact ? launch_blend<KM, false, kModeExact>(A, nt, st)                       \
                 : launch_blend<KM, false, kModeFast>(A, nt, st)
    if (k <= 4) { IVR_BLEND(4); }
    if (k <= 8) { IVR_BLEND(8); }
    if (k <= 16) { IVR_BLEND(16); }
    IVR_BLEND(32);
#undef IVR_BLEND
}
