// K2 -- bit-exact (tile, depth) pair ordering on device.
//
// Reproduces np.lexsort((depth[pair_splat], pair_tile)) (rasterizer.py:129)
// over the pairs of fill_pairs (_kernels.py:19-28) and the tile ranges of
// np.searchsorted (rasterizer.py:132), without materialising a composite key:
//
//  1. depth ranks.  Positive float64 depths order like their bit patterns.
//     The bits are shifted into a "coarse" key (bits - min) >> s of about
//     log2(n) + 3 bits (~8 buckets per splat; the [min, max] of the visible
//     keys comes from K1's block-reduced atomics, or from a min/max kernel
//     when the keys are supplied directly).  One histogram kernel maps the
//     keys and counts every pass's 8-bit digits; each stable LSD pass is then
//     ONE kernel (onesweep: 4096-key blocks take virtual ids in start order,
//     publish their digit counts and find their exclusive prefix per digit by
//     decoupled look-back over their predecessors, then scatter through
//     shared memory).  Invisible splats carry all ones and sort last.  Runs
//     of equal coarse keys are re-ordered by the full 64-bit key (insertion
//     sort, stable); if a run is longer than kMaxRun the last block of that
//     kernel recomputes the whole order with a full 64-bit LSD sort --
//     correctness never depends on the data.  Ties keep index order =
//     lexsort's tie break on fill_pairs' order.
//  2. counting placement: each block owns 2048 consecutive depth ranks; its
//     warps expand their ranks' pairs in fill_pairs order (load-balanced
//     warp expansion, no per-pair global searches), build a per-tile
//     histogram that is scanned per tile across blocks, and write each pair
//     once to tile_start[t] + block offset + its stable rank inside the block
//     (warp match_any ranking).  The per-tile scan kernel's last block turns
//     the tile totals into the tile ranges (P = their sum) and the K3/K4
//     tile schedule, and re-arms the min/max words for the next frame.
//  3. optional tile cull: while placing, each pair is tested in float64 for
//     whether its splat can reach alpha >= 1/255 anywhere in the tile; pairs
//     that cannot are marked with bit 31 (pair_splat & 0x7fffffff is the
//     reference list), letting the blend skip them without loading records.
// All data-dependent sizes live in device memory: the sequence is
// stream-ordered and CUDA-graph capturable (8 kernels + one control-block
// memset per frame at 1M splats).
#include "cull.cuh"

namespace ivr {
namespace sortk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                 // per thread in radix passes
constexpr int kChunk = kThreads * kItems;  // 4096 keys per radix block
constexpr int kRadix = 256;
constexpr int kMaxRun = 64;
constexpr uint32_t kInvisible = 0xffffffffu;

__global__ void init_minmax_kernel(unsigned long long *mm) {
    mm[0] = ~0ull;
    mm[1] = 0ull;
}

// Look-back status words: 2 flag bits (1 = block aggregate, 2 = inclusive
// prefix) over a 30-bit count; 0 = not yet published.
constexpr uint32_t kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}

__device__ __forceinline__ int64_t load_n(const int32_t *n_dev, int64_t n_host, int64_t cap) {
    int64_t n = n_dev ? (int64_t)(*n_dev) : n_host;
    return n < cap ? n : cap;
}

// Inclusive block scan of one uint32 per thread (kThreads threads).
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t x, uint32_t *s_warp, uint32_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kWarps ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kWarps) s_warp[lane] = w;
    }
    __syncthreads();
    if (warp > 0) x += s_warp[warp - 1];
    total = s_warp[kWarps - 1];
    __syncthreads();
    return x;
}

// ----------------------------------------------------------------- coarse keys
__global__ void __launch_bounds__(kThreads)
minmax_kernel(const uint64_t *keys, int64_t n, unsigned long long *mm /* [min, max] */) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        const unsigned long long k = keys[i];
        if (k != ~0ull) {
            lo = k < lo ? k : lo;
            hi = k > hi ? k : hi;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    // block reduction first: one atomic pair per block (per-warp atomics on
    // the same two words serialise in L2)
    __shared__ unsigned long long s_lo[kWarps], s_hi[kWarps];
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; ++w) {
            lo = s_lo[w] < lo ? s_lo[w] : lo;
            hi = s_hi[w] > hi ? s_hi[w] : hi;
        }
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

// ----------------------------------------------------------------- radix passes
// Coarse keys + every pass's digit histogram in one read of the 64-bit keys:
// visible keys get `vbits` bits ((bits - min) >> s < 2^vbits), invisible
// splats all ones (above every visible key); per-block shared histograms are
// added into the global per-pass digit counts gdig[pass][256] (zeroed by the
// frame's control-block memset).
__global__ void __launch_bounds__(kThreads)
hist_coarse_kernel(const uint64_t *full, int64_t n, const unsigned long long *mm, int vbits,
                   int passes, uint32_t *ck, uint32_t *gdig) {
    __shared__ uint32_t s[4][kRadix];
#pragma unroll
    for (int p = 0; p < 4; ++p) s[p][threadIdx.x] = 0;
    const unsigned long long lo = mm[0], hi = mm[1];
    const unsigned long long range = hi >= lo ? hi - lo : 0ull;
    const int bits = range ? 64 - __clzll((long long)range) : 0;
    const int sh = bits > vbits ? bits - vbits : 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    unsigned long long k[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + r * kThreads + threadIdx.x;
        k[r] = idx < n ? full[idx] : 0ull;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + r * kThreads + threadIdx.x;
        if (idx < n) {
            const uint32_t c = k[r] == ~0ull ? kInvisible : (uint32_t)((k[r] - lo) >> sh);
            ck[idx] = c;
            for (int p = 0; p < passes; ++p) atomicAdd(&s[p][(c >> (8 * p)) & 255u], 1u);
        }
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
        if (s[p][threadIdx.x]) atomicAdd(&gdig[p * kRadix + threadIdx.x], s[p][threadIdx.x]);
}

// One stable LSD pass (8-bit digit at `shift`) of (key, value) pairs as a
// single kernel.  vals_in == nullptr means identity values.  Blocks take
// virtual ids in the order they start (so every predecessor is running and
// look-back cannot deadlock), rank their 4096 keys by digit (warp match_any),
// publish per-digit counts, and obtain each digit's exclusive prefix over the
// earlier blocks by decoupled look-back on status[block][digit]; the digit
// bases come from the pass's global histogram (hist_coarse_kernel).
template <typename KeyT>
__global__ void __launch_bounds__(kThreads)
onesweep_kernel(const KeyT *keys, const uint32_t *vals, int64_t n, int shift,
                const uint32_t *gdig, uint32_t *status, uint32_t *vctr, KeyT *dkeys,
                uint32_t *dvals) {
    __shared__ uint32_t s_wcnt[kWarps][kRadix];
    __shared__ uint32_t s_gbase[kRadix];
    __shared__ uint32_t s_lstart[kRadix];
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_bid;
    __shared__ KeyT s_keys[kChunk];
    __shared__ uint32_t s_vals[kChunk];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_bid = atomicAdd(vctr, 1u);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_wcnt[w][tid] = 0;
    __syncthreads();
    const uint32_t bid = s_bid;
    const int64_t base = (int64_t)bid * kChunk;
    KeyT k[kItems];
    uint32_t v[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {  // all loads first (memory-level parallelism)
        const int64_t idx = base + warp * (32 * kItems) + r * 32 + lane;
        const bool ok = idx < n;
        k[r] = ok ? keys[idx] : (KeyT)0;
        v[r] = ok ? (vals ? vals[idx] : (uint32_t)idx) : 0u;
    }
    uint32_t dig[kItems], rank[kItems];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + warp * (32 * kItems) + r * 32 + lane;
        const bool ok = idx < n;
        dig[r] = ok ? ((uint32_t)(k[r] >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig[r]);
        uint32_t before = 0;
        if (ok) before = s_wcnt[warp][dig[r]];
        __syncwarp();
        if (ok && (peers & lt) == 0) s_wcnt[warp][dig[r]] = before + __popc(peers);
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    uint32_t cnt;  // this block's count of digit tid
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_wcnt[w][tid];
            s_wcnt[w][tid] = run;
            run += c;
        }
        cnt = run;
    }
    // publish the aggregate (block 0: already the inclusive prefix), then look back
    uint32_t *my = status + (int64_t)bid * kRadix + tid;
    st_volatile(my, (bid == 0 ? kFlagPrefix : kFlagAgg) | cnt);
    uint32_t excl = 0;
    if (bid > 0) {
        int64_t j = (int64_t)bid - 1;
        while (true) {
            const uint32_t w = ld_volatile(status + j * kRadix + tid);
            if ((w & ~kValMask) == 0) continue;  // predecessor not published yet
            excl += w & kValMask;
            if (w & kFlagPrefix) break;
            --j;
        }
        st_volatile(my, kFlagPrefix | (excl + cnt));
    }
    uint32_t tot;
    const uint32_t gd = gdig[tid];
    const uint32_t ginc = block_incl_scan(gd, s_warp, tot);
    s_gbase[tid] = ginc - gd + excl;
    {
        const uint32_t inc = block_incl_scan(cnt, s_warp, tot);
        s_lstart[tid] = inc - cnt;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        if (dig[r] < 256u) {
            const uint32_t lp = s_lstart[dig[r]] + s_wcnt[warp][dig[r]] + rank[r];
            s_keys[lp] = k[r];
            s_vals[lp] = v[r];
        }
    }
    __syncthreads();
    const int nvalid = (int)((n - base) < kChunk ? (n - base) : kChunk);
    for (int i = tid; i < nvalid; i += kThreads) {
        const KeyT kk = s_keys[i];
        const uint32_t d = (uint32_t)(kk >> shift) & 255u;
        const uint32_t g = s_gbase[d] + (uint32_t)i - s_lstart[d];
        dkeys[g] = kk;
        dvals[g] = s_vals[i];
    }
}

// ----------------------------------------------------------------- run fix-up
// Rare path (a coarse-key run longer than kMaxRun, i.e. many depths packed
// into one bucket by an extreme depth range): one CTA recomputes the whole
// order with a stable 8 x 8-bit LSD sort of the full 64-bit keys.
template <int NT>
__device__ void full_sort_block(const uint64_t *depth_key, int64_t n, uint64_t *kA, uint64_t *kB,
                                uint32_t *vA, uint32_t *vB) {
    constexpr int NW = NT / 32;
    __shared__ uint32_t s_off[kRadix];
    __shared__ uint32_t s_wc[NW][kRadix];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    for (int p = 0; p < 8; ++p) {
        const uint64_t *ki = p == 0 ? depth_key : ((p & 1) ? kB : kA);
        const uint32_t *vi = p == 0 ? nullptr : ((p & 1) ? vB : vA);
        uint64_t *ko = (p & 1) ? kA : kB;
        uint32_t *vo = (p & 1) ? vA : vB;
        const int sh = 8 * p;
        // digit histogram -> exclusive offsets
        for (int d = tid; d < kRadix; d += NT) s_off[d] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += NT) atomicAdd(&s_off[(ki[i] >> sh) & 255], 1u);
        __syncthreads();
        if (tid == 0) {
            uint32_t run = 0;
            for (int d = 0; d < kRadix; ++d) {
                const uint32_t c = s_off[d];
                s_off[d] = run;
                run += c;
            }
        }
        __syncthreads();
        // stable scatter, one NT-element tile at a time
        for (int64_t base = 0; base < n; base += NT) {
            for (int i = tid; i < NW * kRadix; i += NT) (&s_wc[0][0])[i] = 0;
            __syncthreads();
            const int64_t i = base + tid;
            const bool ok = i < n;
            const uint64_t k = ok ? ki[i] : 0ull;
            const uint32_t v = ok ? (vi ? vi[i] : (uint32_t)i) : 0u;
            const uint32_t d = ok ? (uint32_t)((k >> sh) & 255) : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (ok && (peers & lt) == 0) s_wc[warp][d] = __popc(peers);
            __syncthreads();
            for (int dd = tid; dd < kRadix; dd += NT) {  // exclusive scan across warps
                uint32_t run = 0;
                for (int w = 0; w < NW; ++w) {
                    const uint32_t c = s_wc[w][dd];
                    s_wc[w][dd] = run;
                    run += c;
                }
            }
            __syncthreads();
            if (ok) {
                const uint32_t pos = s_off[d] + s_wc[warp][d] + __popc(peers & lt);
                ko[pos] = k;
                vo[pos] = v;
            }
            __syncthreads();
            // advance the digit offsets by this tile's per-digit totals
            for (int dd = tid; dd < kRadix; dd += NT) s_wc[0][dd] = 0;
            __syncthreads();
            if (ok) atomicAdd(&s_wc[0][d], 1u);
            __syncthreads();
            for (int dd = tid; dd < kRadix; dd += NT) s_off[dd] += s_wc[0][dd];
            __syncthreads();
        }
    }
    // result in kA/vA after 8 passes (pass 7 writes A)
}

// Re-order runs of equal coarse keys by the full 64-bit key (stable).  A run
// longer than kMaxRun sets *need_full; the kernel's last block to finish then
// recomputes the whole order (full_sort_block) into idx.
__global__ void __launch_bounds__(kThreads)
fixup_kernel(const uint32_t *ck, uint32_t *idx, int64_t n, const uint64_t *full,
             int32_t *need_full, uint32_t *done, uint64_t *fkA, uint64_t *fkB, uint32_t *vscratch) {
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const uint32_t k = i < n ? ck[i] : kInvisible;
    const bool head = k != kInvisible && (i == 0 || ck[i - 1] != k) && i + 1 < n && ck[i + 1] == k;
    if (head) {
        int64_t e = i + 1;
        while (e < n && ck[e] == k && e - i <= kMaxRun) ++e;
        if (e - i > kMaxRun) {
            *need_full = 1;
        } else {
            const int len = (int)(e - i);
            uint32_t v[kMaxRun];
            uint64_t key[kMaxRun];
            for (int a = 0; a < len; ++a) {
                v[a] = idx[i + a];
                key[a] = full[v[a]];
            }
            for (int a = 1; a < len; ++a) {  // stable insertion sort (indices ascending on ties)
                const uint32_t tv = v[a];
                const uint64_t tk = key[a];
                int b = a - 1;
                while (b >= 0 && key[b] > tk) {
                    key[b + 1] = key[b];
                    v[b + 1] = v[b];
                    --b;
                }
                key[b + 1] = tk;
                v[b + 1] = tv;
            }
            for (int a = 0; a < len; ++a) idx[i + a] = v[a];
        }
    }
    // last block to finish: the full sort if any run was too long
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || ld_volatile((const uint32_t *)need_full) == 0) return;
    __threadfence();
    full_sort_block<kThreads>(full, n, fkA, fkB, idx, vscratch);
}

// ----------------------------------------------------------------- placement
constexpr int kRanksPerWarp = 256;
constexpr int kRanksPerBlock = kRanksPerWarp * kWarps;  // 2048 ranks per block

struct PairCtx {
    const uint32_t *order;  // rank -> splat
    const int32_t *count;   // splat -> tiles touched
    const ushort4 *rect;    // splat -> tile rect
    const float4 *rec;      // blend records (tile cull), may be null
    int64_t n;
    int ntx, nty, ntiles;
    int64_t cap;
    // tile-row band [ty_lo, ty_lo + bh) handled by this launch (frames whose
    // per-warp difference arrays exceed shared memory are placed band by band);
    // banded = false: the whole grid (bh = nty)
    int ty_lo, bh;
    bool banded;
};

// Clip a tile rectangle to the launch's band; rows become band-local.
// Returns false when the rectangle misses the band.
__device__ __forceinline__ bool band_clip(const PairCtx &C, ushort4 &rc) {
    if (!C.banded) return true;
    const int z = max((int)rc.z, C.ty_lo), w = min((int)rc.w, C.ty_lo + C.bh - 1);
    if (z > w) return false;
    rc.z = (unsigned short)(z - C.ty_lo);
    rc.w = (unsigned short)(w - C.ty_lo);
    return true;
}

// 2-D difference-array update for one tile rectangle (D is (nty+1) x (ntx+1)).
__device__ __forceinline__ void diff_add(int *D, int w1, const ushort4 rc, int v) {
    atomicAdd(&D[rc.z * w1 + rc.x], v);
    atomicAdd(&D[rc.z * w1 + rc.y + 1], -v);
    atomicAdd(&D[(rc.w + 1) * w1 + rc.x], -v);
    atomicAdd(&D[(rc.w + 1) * w1 + rc.y + 1], v);
}

// In-place 2-D inclusive prefix sum of a difference array by `nt` threads
// (thread index `t`); `sync` separates the row and column passes.
template <typename Sync>
__device__ __forceinline__ void prefix2d(int *D, int w1, int h1, int t, int nt, Sync &&sync) {
    for (int r = t; r < h1; r += nt) {
        int run = 0;
        for (int c = 0; c < w1; ++c) {
            run += D[r * w1 + c];
            D[r * w1 + c] = run;
        }
    }
    sync();
    for (int c = t; c < w1; c += nt) {
        int run = 0;
        for (int r = 0; r < h1; ++r) {
            run += D[r * w1 + c];
            D[r * w1 + c] = run;
        }
    }
    sync();
}

// Warp-cooperative, load-balanced expansion of the pairs of ranks
// [rbase, rend) in fill_pairs order (rank-major, then ty, then tx): each lane
// owns one rank of a 32-rank group; the group's pairs are visited 32 at a
// time, every lane finding its owner rank with a 5-step shuffle search over
// the group's inclusive count prefix.  f(ok, splat, tile, tx, ty) is called
// by all 32 lanes for each 32-pair chunk (convergent; ok marks real pairs).
template <typename Fn>
__device__ __forceinline__ void expand_pairs(const PairCtx &C, int64_t rbase, int64_t rend, Fn &&f) {
    const int lane = threadIdx.x & 31;
    for (int64_t g = rbase; g < rend; g += 32) {
        const int64_t r = g + lane;
        uint32_t sp = 0, cnt = 0, rx = 0, rz = 0;
        if (r < rend) {
            sp = C.order[r];
            cnt = (uint32_t)C.count[sp];
            if (cnt) {
                ushort4 rc = C.rect[sp];
                if (band_clip(C, rc)) {
                    cnt = (uint32_t)(rc.y - rc.x + 1) * (uint32_t)(rc.w - rc.z + 1);
                    rx = (uint32_t)rc.x | ((uint32_t)rc.y << 16);
                    rz = (uint32_t)rc.z | ((uint32_t)rc.w << 16);
                } else {
                    cnt = 0;
                }
            }
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t G = __shfl_sync(0xffffffffu, incl, 31);
        if (G == 0) {
            if (C.banded) continue;  // this group misses the band; later ones may not
            break;                   // invisible ranks (count 0) sort last: nothing further
        }
        const uint32_t excl = incl - cnt;
        for (uint32_t k0 = 0; k0 < G; k0 += 32) {
            const uint32_t k = k0 + lane;
            int owner = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= k) owner += step;
            }
            const uint32_t o_excl = __shfl_sync(0xffffffffu, excl, owner);
            const uint32_t o_sp = __shfl_sync(0xffffffffu, sp, owner);
            const uint32_t o_rx = __shfl_sync(0xffffffffu, rx, owner);
            const uint32_t o_rz = __shfl_sync(0xffffffffu, rz, owner);
            const bool ok = k < G;
            const uint32_t q = k - o_excl;
            const uint32_t tx0 = o_rx & 0xffffu, tx1 = o_rx >> 16, ty0 = o_rz & 0xffffu;
            const uint32_t w = tx1 - tx0 + 1;
            // q / w via a float reciprocal (q, w < 2^16) and one correction
            float rw;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rw) : "f"((float)w));
            uint32_t qy = (uint32_t)((float)q * rw);
            if (qy * w > q) --qy;
            else if ((qy + 1) * w <= q) ++qy;
            const int ty = ok ? (int)(ty0 + qy) + C.ty_lo : 0;  // global tile row
            const int tx = ok ? (int)(tx0 + (q - qy * w)) : 0;
            f(ok, o_sp, ok ? ty * C.ntx + tx : -1, tx, ty);
        }
    }
}

// per-block tile histogram -> hist[tile * nblocks + block], from a 2-D
// difference array of the block's tile rectangles (no pair expansion)
__global__ void __launch_bounds__(kThreads)
pair_hist_kernel(PairCtx C, uint32_t *hist, int nblocks) {
    extern __shared__ int smem_i32[];
    const int w1 = C.ntx + 1, h1 = C.bh + 1;
    int *D = smem_i32;
    for (int i = threadIdx.x; i < w1 * h1; i += kThreads) D[i] = 0;
    __syncthreads();
    const int64_t r0 = (int64_t)blockIdx.x * kRanksPerBlock;
    for (int k = threadIdx.x; k < kRanksPerBlock; k += kThreads) {
        const int64_t r = r0 + k;
        if (r >= C.n) break;
        const uint32_t sp = C.order[r];
        if (C.count[sp] > 0) {
            ushort4 rc = C.rect[sp];
            if (band_clip(C, rc)) diff_add(D, w1, rc, 1);
        }
    }
    __syncthreads();
    prefix2d(D, w1, h1, threadIdx.x, kThreads, [] { __syncthreads(); });
    const int tb = C.ty_lo * C.ntx;  // first tile of the band
    for (int t = threadIdx.x; t < C.ntx * C.bh; t += kThreads)
        hist[(int64_t)(tb + t) * nblocks + blockIdx.x] = (uint32_t)D[(t / C.ntx) * w1 + t % C.ntx];
}

// Per-tile exclusive scan of the per-block pair counts (hist[tile][block],
// one warp per tile row, 32 coalesced columns per step) -> tile totals; the
// kernel's last block to finish then writes tile_ranges = exclusive scan of
// the totals (P = their sum, ranges clamped to the pair capacity so an
// overflowed frame never makes K3/K4 read past pair_splat), the optional
// heaviest-first tile schedule for K3/K4 (a 64-bucket counting sort of the
// tile pair counts; scheduling only), and re-arms the depth min/max words
// that K1 of the next frame reduces into.
constexpr int kOrderBuckets = 64;

__global__ void __launch_bounds__(kThreads)
tile_scan_kernel(uint32_t *hist, int ntiles, int nblocks, uint32_t *totals, uint32_t *done,
                 int32_t *ranges, uint32_t cap, int32_t *n_pairs, int32_t *order,
                 unsigned long long *mm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int r = blockIdx.x * kWarps + warp;
    if (r < ntiles) {
        uint32_t *row = hist + (int64_t)r * nblocks;
        uint32_t carry = 0;
#pragma unroll 4
        for (int base = 0; base < nblocks; base += 32) {
            const int i = base + lane;
            const uint32_t v = i < nblocks ? row[i] : 0;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (i < nblocks) row[i] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) totals[r] = carry;
    }
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ uint32_t s_warp[kWarps];
    uint64_t carry = 0;
    for (int base = 0; base < ntiles; base += kThreads) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < ntiles ? __ldcg(totals + i) : 0;
        uint32_t tot;
        const uint32_t incl = block_incl_scan(v, s_warp, tot);
        if (i < ntiles) ranges[i] = (int32_t)min(carry + incl - v, (uint64_t)cap);
        carry += tot;
    }
    if (threadIdx.x == 0) {
        ranges[ntiles] = (int32_t)min(carry, (uint64_t)cap);
        // P = the sum of all tile counts (unclamped; saturated to int32)
        *n_pairs = carry > 0x7fffffffull ? 0x7fffffff : (int32_t)carry;
        if (mm) {
            mm[0] = ~0ull;
            mm[1] = 0ull;
        }
    }
    if (!order) return;
    __syncthreads();
    __shared__ int s_hist[kOrderBuckets];
    if (threadIdx.x < kOrderBuckets) s_hist[threadIdx.x] = 0;
    __syncthreads();
    auto bucket = [](int cnt) {
        const int b = (int)(2.0f * __log2f((float)cnt + 1.0f));
        return kOrderBuckets - 1 - (b < kOrderBuckets - 1 ? b : kOrderBuckets - 1);
    };
    for (int t = threadIdx.x; t < ntiles; t += kThreads)
        atomicAdd(&s_hist[bucket(ranges[t + 1] - ranges[t])], 1);
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
    for (int t = threadIdx.x; t < ntiles; t += kThreads)
        order[atomicAdd(&s_hist[bucket(ranges[t + 1] - ranges[t])], 1)] = t;
}

// stable placement: warp w of block b owns ranks [b*2048 + w*256, +256).
// Per-warp tile counts come from per-warp 2-D difference arrays; the pairs
// are expanded once, ranked within the warp by match_any and written.
__global__ void __launch_bounds__(kThreads)
pair_place_kernel(PairCtx C, const uint32_t *hist, int nblocks, const int32_t *ranges,
                  int32_t *pair_splat, int W, int H) {
    extern __shared__ int smem_i32[];
    const int w1 = C.ntx + 1, h1 = C.bh + 1, cells = w1 * h1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kWarps * cells; i += kThreads) smem_i32[i] = 0;
    __syncthreads();
    int *Dw = smem_i32 + warp * cells;
    const uint32_t lt = lanemask_lt();
    const int64_t rb = (int64_t)blockIdx.x * kRanksPerBlock + (int64_t)warp * kRanksPerWarp;
    const int64_t re = rb + kRanksPerWarp < C.n ? rb + kRanksPerWarp : C.n;
    // phase 1: per-warp tile counts (<= 256 per tile per warp); the warp's
    // 8 rank loads are issued together, then the dependent count / rect loads
    {
        constexpr int kPer = kRanksPerWarp / 32;
        uint32_t sps[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int64_t r = rb + lane + 32 * u;
            sps[u] = r < re ? __ldg(C.order + r) : 0xffffffffu;
        }
        int cnts[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) cnts[u] = sps[u] != 0xffffffffu ? __ldg(C.count + sps[u]) : 0;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            if (cnts[u] > 0) {
                ushort4 rc = C.rect[sps[u]];
                if (band_clip(C, rc)) diff_add(Dw, w1, rc, 1);
            }
        }
    }
    __syncwarp();
    prefix2d(Dw, w1, h1, lane, 32, [] { __syncwarp(); });
    __syncthreads();
    // phase 2: exclusive scan across warps, per tile (block total <= 2048), and
    // the block's global base per tile (tile start + earlier blocks) in smem
    uint32_t *s_base = reinterpret_cast<uint32_t *>(smem_i32 + kWarps * cells);
    const int tb = C.ty_lo * C.ntx;  // first tile of the band
    for (int tl = tid; tl < C.ntx * C.bh; tl += kThreads) {
        const int cell = (tl / C.ntx) * w1 + tl % C.ntx, t = tb + tl;
        int run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = smem_i32[w * cells + cell];
            smem_i32[w * cells + cell] = run;
            run += c;
        }
        s_base[cell] = run ? (uint32_t)ranges[t] + hist[(int64_t)t * nblocks + blockIdx.x] : 0u;
    }
    __syncthreads();
    // phase 3: expand once, place (and cull-flag) every pair
    expand_pairs(C, rb, re, [&](bool ok, uint32_t sp, int tile, int tx, int ty) {
        const uint32_t peers = __match_any_sync(0xffffffffu, tile);
        const int cell = (ty - C.ty_lo) * w1 + tx;
        // the first lane of each equal-tile group advances the warp's running
        // count for that tile and shares the old value with its peers
        const int leader = __ffs(peers) - 1;
        int before = 0;
        if (ok && lane == leader) before = atomicAdd(&Dw[cell], __popc(peers));
        before = __shfl_sync(0xffffffffu, before, leader);
        if (ok) {
            const uint32_t pos = s_base[cell] + (uint32_t)before + __popc(peers & lt);
            if ((int64_t)pos < C.cap) {
                uint32_t v = sp;
                if (C.rec) {
                    const int px0 = tx * kTile, py0 = ty * kTile;
                    const int px1 = min(px0 + kTile - 1, W - 1), py1 = min(py0 + kTile - 1, H - 1);
                    const float4 a0 = __ldg(C.rec + 2 * sp), a1 = __ldg(C.rec + 2 * sp + 1);
                    if (tile_cull32(a0, a1, px0, px1, py0, py1)) v |= 0x80000000u;
                }
                pair_splat[pos] = (int32_t)v;
            }
        }
    });
}

}  // namespace sortk
}  // namespace ivr

using namespace ivr::sortk;

namespace {
inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct Plan {
    size_t off[16];
    size_t total;
    int nbk, nbp;
    size_t ctrl_bytes;  // zeroed per frame: digit histograms, counters, flags, look-back words
};

// control block (offset 8): gdig[4][256] | vctr[4] | done_fix | done_tiles |
// need_full | pad | status[4][nbk][256]
constexpr size_t kCtrlHead = 4 * 256 * 4 + 64;

Plan plan(int64_t n, int64_t cap, int32_t ntiles) {
    Plan L{};
    L.nbk = (int)((n + kChunk - 1) / kChunk);
    L.nbp = (int)((n + kRanksPerBlock - 1) / kRanksPerBlock);
    L.ctrl_bytes = kCtrlHead + (size_t)4 * L.nbk * kRadix * 4;
    size_t sz[16] = {
        al(4 * (size_t)n), al(4 * (size_t)n),                    // 0,1 coarse keys A/B
        al(4 * (size_t)n), al(4 * (size_t)n),                    // 2,3 vals A/B
        al(8 * (size_t)n), al(8 * (size_t)n),                    // 4,5 full keys (fallback) A/B
        al(4),                                                   // 6 (unused)
        al(4),                                                   // 7 (unused)
        al(L.ctrl_bytes),                                        // 8 control block
        al(4),                                                   // 9 (unused)
        al(4 * (size_t)ntiles * (L.nbp + 1)),                    // 10 pair tile hist
        al(4 * (size_t)(ntiles + 1)),                            // 11 tile totals
        al(16),                                                  // 12 minmax (keys supplied directly)
        al(16),                                                  // 13 (unused)
        0, 0};
    size_t o = 0;
    for (int i = 0; i < 16; ++i) {
        L.off[i] = o;
        o += sz[i];
    }
    L.total = o;
    return L;
}
}  // namespace

extern "C" size_t ivr_bin_sort_workspace_size(int64_t n, int64_t pair_capacity, int32_t ntiles) {
    return plan(n < 1 ? 1 : n, pair_capacity < 1 ? 1 : pair_capacity, ntiles < 1 ? 1 : ntiles).total;
}

extern "C" int ivr_bin_sort(int64_t n, const uint64_t *depth_key, const int32_t *count,
                            const uint16_t *rect, int32_t ntx, int32_t nty, int64_t pair_capacity,
                            void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                            int32_t *tile_ranges, int32_t *n_pairs, ivr_stream_t stream) {
    return ivr_bin_sort_frame(n, depth_key, nullptr, count, rect, nullptr, ntx, nty, 0, 0,
                              pair_capacity, workspace, workspace_bytes, pair_splat, tile_ranges,
                              n_pairs, nullptr, stream);
}

extern "C" int ivr_bin_sort_cull(int64_t n, const uint64_t *depth_key, const int32_t *count,
                                 const uint16_t *rect, const float *rec, int32_t ntx, int32_t nty,
                                 int32_t width, int32_t height, int64_t pair_capacity,
                                 void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                                 int32_t *tile_ranges, int32_t *n_pairs, ivr_stream_t stream) {
    return ivr_bin_sort_frame(n, depth_key, nullptr, count, rect, rec, ntx, nty, width, height,
                              pair_capacity, workspace, workspace_bytes, pair_splat, tile_ranges,
                              n_pairs, nullptr, stream);
}

extern "C" int ivr_bin_sort_frame(int64_t n, const uint64_t *depth_key,
                                  unsigned long long *depth_minmax, const int32_t *count,
                                  const uint16_t *rect, const float *rec, int32_t ntx, int32_t nty,
                                  int32_t width, int32_t height, int64_t pair_capacity,
                                  void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                                  int32_t *tile_ranges, int32_t *n_pairs, int32_t *tile_order,
                                  ivr_stream_t stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int32_t ntiles = ntx * nty;
    // placement keeps 8 per-warp int32 difference arrays of (ntx+1)(rows+1)
    // cells plus one table of per-tile block bases in smem: frames whose tile
    // grid does not fit are placed in bands of `bh` tile rows
    const int64_t max_cells = (int64_t)(220 * 1024) / (4 * (kWarps + 1));
    int band_rows = (int)(max_cells / (ntx + 1)) - 1;
    band_rows = band_rows > nty ? nty : band_rows;
    const bool fits = band_rows >= 1;
    if (n < 0 || pair_capacity < 1 || ntx < 1 || nty < 1 || !fits || !tile_ranges ||
        !n_pairs || !pair_splat || !workspace || (rec && (width < 1 || height < 1))) {
        ivr::set_error("ivr_bin_sort: bad argument");
        return IVR_ERR_ARG;
    }
    if (n >= (1ll << 30) || pair_capacity > 0x7fffffffll) {
        ivr::set_error("ivr_bin_sort: n must be below 2^30 and the capacity fit int32");
        return IVR_ERR_ARG;
    }
    const Plan L = plan(n < 1 ? 1 : n, pair_capacity, ntiles);
    if (workspace_bytes < L.total) {
        ivr::set_error("ivr_bin_sort: workspace too small");
        return IVR_ERR_ARG;
    }
    if (n == 0) {
        cudaMemsetAsync(n_pairs, 0, 4, st);
        cudaMemsetAsync(tile_ranges, 0, 4 * (size_t)(ntiles + 1), st);
        if (tile_order) ivr_tile_order(tile_ranges, ntiles, tile_order, stream);
        return ivr::check_launch("ivr_bin_sort(empty)");
    }
    char *ws = (char *)workspace;
    uint32_t *ckA = (uint32_t *)(ws + L.off[0]), *ckB = (uint32_t *)(ws + L.off[1]);
    uint32_t *vA = (uint32_t *)(ws + L.off[2]), *vB = (uint32_t *)(ws + L.off[3]);
    uint64_t *fkA = (uint64_t *)(ws + L.off[4]), *fkB = (uint64_t *)(ws + L.off[5]);
    char *ctrl = ws + L.off[8];
    uint32_t *gdig = (uint32_t *)ctrl;
    uint32_t *vctr = gdig + 4 * 256;
    uint32_t *done_fix = vctr + 4, *done_tiles = vctr + 5;
    int32_t *need_full = (int32_t *)(vctr + 6);
    uint32_t *status = (uint32_t *)(ctrl + kCtrlHead);
    uint32_t *phist = (uint32_t *)(ws + L.off[10]);
    uint32_t *ttot = (uint32_t *)(ws + L.off[11]);
    const int nbk = L.nbk, nbp = L.nbp;
    const size_t status_pass = (size_t)nbk * kRadix;

    // ---- 1. depth ranks: coarse keys with ~8 buckets per splat (at least
    //      log2(n) + 3 bits; 8-bit digits), one onesweep kernel per pass, run fix-up
    int lg = 1;
    while (lg < 62 && (1ll << lg) < n) ++lg;
    int passes = (lg + 4 + 7) / 8;
    passes = passes < 2 ? 2 : (passes > 4 ? 4 : passes);
    const int vbits = 8 * passes - 1;
    cudaMemsetAsync(ctrl, 0, kCtrlHead + (size_t)passes * status_pass * 4, st);
    unsigned long long *mm = depth_minmax;
    if (!mm) {  // keys supplied directly: reduce their range here
        mm = (unsigned long long *)(ws + L.off[12]);
        init_minmax_kernel<<<1, 1, 0, st>>>(mm);
        int gb = (int)((n + kThreads * 8 - 1) / (kThreads * 8));
        gb = gb < 1 ? 1 : (gb > 1184 ? 1184 : gb);
        minmax_kernel<<<gb, kThreads, 0, st>>>(depth_key, n, mm);
    }
    hist_coarse_kernel<<<nbk, kThreads, 0, st>>>(depth_key, n, mm, vbits, passes, ckA, gdig);
    uint32_t *kin = ckA, *kout = ckB, *vin = nullptr, *vout = vB;
    for (int p = 0; p < passes; ++p) {
        onesweep_kernel<uint32_t><<<nbk, kThreads, 0, st>>>(kin, vin, n, 8 * p, gdig + 256 * p,
                                                           status + p * status_pass, vctr + p,
                                                           kout, vout);
        uint32_t *t = kin;
        kin = kout;
        kout = t;
        vin = vout;
        vout = (vout == vB) ? vA : vB;
    }
    // sorted (key, order) now in (kin, vin); runs fixed, long runs -> full sort
    uint32_t *ord = vin, *vscratch = (vin == vA) ? vB : vA;
    fixup_kernel<<<(int)((n + kThreads - 1) / kThreads), kThreads, 0, st>>>(
        kin, ord, n, depth_key, need_full, done_fix, fkA, fkB, vscratch);
    // ---- 2. counting placement by tile (+ optional tile cull flag); the
    // tile scan's last block writes the ranges, P = n_pairs and the schedule
    PairCtx C{};
    C.order = ord;
    C.count = count;
    C.rect = (const ushort4 *)rect;
    C.rec = (const float4 *)rec;
    C.n = n;
    C.ntx = ntx;
    C.nty = nty;
    C.ntiles = ntiles;
    C.cap = pair_capacity;
    C.banded = band_rows < nty;
    const size_t cells = (size_t)(ntx + 1) * (band_rows + 1);
    const size_t sm_hist = 4 * cells;
    const size_t sm_place = 4 * (size_t)(kWarps + 1) * cells;
    if (sm_hist > 48 * 1024)
        cudaFuncSetAttribute(pair_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_hist);
    if (sm_place > 48 * 1024)
        cudaFuncSetAttribute(pair_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_place);
    for (int y0 = 0; y0 < nty; y0 += band_rows) {  // one band unless the grid is too large
        C.ty_lo = y0;
        C.bh = y0 + band_rows <= nty ? band_rows : nty - y0;
        pair_hist_kernel<<<nbp, kThreads, sm_hist, st>>>(C, phist, nbp);
    }
    tile_scan_kernel<<<(ntiles + kWarps - 1) / kWarps, kThreads, 0, st>>>(
        phist, ntiles, nbp, ttot, done_tiles, tile_ranges, (uint32_t)pair_capacity, n_pairs,
        tile_order, depth_minmax);
    for (int y0 = 0; y0 < nty; y0 += band_rows) {
        C.ty_lo = y0;
        C.bh = y0 + band_rows <= nty ? band_rows : nty - y0;
        pair_place_kernel<<<nbp, kThreads, sm_place, st>>>(C, phist, nbp, tile_ranges, pair_splat,
                                                           width, height);
    }
    return ivr::check_launch("ivr_bin_sort");
}
