// K2 -- bit-exact (tile, depth) pair ordering on device.
//
// Reproduces np.lexsort((depth[pair_splat], pair_tile)) (rasterizer.py:129)
// over the pairs of fill_pairs (_kernels.py:19-28) and the tile ranges of
// np.searchsorted (rasterizer.py:132), without materialising a composite key:
//
//  1. depth ranks.  Positive float64 depths order like their bit patterns.
//     The bits are shifted into a "coarse" key (bits - min) >> s of
//     ceil(log2 n) bits (~1-2 buckets per splat; the [min, max] of the visible
//     keys comes from K1's block-reduced atomics, or from a min/max kernel
//     when the keys are supplied directly) and the splats are counting-sorted
//     by it: bucket counts by atomics, one exclusive scan, a scatter that
//     claims slots with an atomic cursor per bucket, then every bucket is
//     sorted by (full 64-bit key, index) -- exactly lexsort's order, ties by
//     index = fill_pairs' order (_kernels.py:21-28).  Invisible splats fill a
//     last bucket.  A bucket longer than kMaxRun (extreme depth clustering)
//     makes the sort kernel's last block recompute the whole order with a
//     full 64-bit LSD sort -- correctness never depends on the data.
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
// stream-ordered and CUDA-graph capturable (7 kernels + one control-block
// memset per frame).
#include "cull.cuh"

namespace ivr {
namespace sortk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                 // per thread in the bucket passes
constexpr int kChunk = kThreads * kItems;  // 4096 keys / counts per block
constexpr int kRadix = 256;
constexpr int kMaxRun = 64;

__global__ void init_minmax_kernel(unsigned long long *mm) {
    mm[0] = ~0ull;
    mm[1] = 0ull;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
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

// ----------------------------------------------------------------- bucket ranks
// Depth ranks by one counting sort on the coarse key: nb = 2^vbits buckets
// (~2 per splat) + one for the invisible splats (last).  Bucket counts by
// global atomics, an exclusive scan of the counts (single pass, decoupled
// look-back), a scatter that claims each splat's slot with an atomic on its
// bucket cursor (so the order inside a bucket is arbitrary), and a per-bucket
// sort by (full 64-bit key, index) -- lexsort's order, ties by index -- in
// fixup_buckets_kernel.
__global__ void __launch_bounds__(kThreads)
bucket_count_kernel(const uint64_t *full, int64_t n, const unsigned long long *mm, int vbits,
                    uint32_t *ck, uint32_t *counts) {
    pdl_begin();
    const unsigned long long lo = mm[0], hi = mm[1];
    const unsigned long long range = hi >= lo ? hi - lo : 0ull;
    const int bits = range ? 64 - __clzll((long long)range) : 0;
    const int sh = bits > vbits ? bits - vbits : 0;
    const uint32_t nb = 1u << vbits;
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
            const uint32_t c = k[r] == ~0ull ? nb : (uint32_t)((k[r] - lo) >> sh);
            ck[idx] = c;
            atomicAdd(counts + c, 1u);
        }
    }
}

// Exclusive scan of counts[0..m): each block scans its 4096 counts in place
// (block-local offsets) and leaves its total in boff[block]; the kernel's last
// block to finish turns boff into the exclusive block offsets (so a bucket
// c starts at boff[c >> 12] + counts[c]).
__global__ void __launch_bounds__(kThreads)
bucket_scan_kernel(uint32_t *counts, int64_t m, uint32_t *boff, uint32_t *done) {
    pdl_begin();
    __shared__ uint32_t s_warp[kWarps];
    __shared__ bool s_last;
    __shared__ uint32_t s_c[kChunk + kChunk / 32];  // padded: conflict-free row reads
    const int tid = threadIdx.x;
    const int64_t b0 = (int64_t)blockIdx.x * kChunk;
    auto pad = [](int i) { return i + (i >> 5); };
#pragma unroll
    for (int r = 0; r < kItems; ++r) {  // coalesced in, each thread then owns 16 in a row
        const int i = r * kThreads + tid;
        s_c[pad(i)] = b0 + i < m ? counts[b0 + i] : 0u;
    }
    __syncthreads();
    uint32_t v[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        v[r] = s_c[pad(tid * kItems + r)];
        sum += v[r];
    }
    uint32_t tot;
    const uint32_t incl = block_incl_scan(sum, s_warp, tot);
    uint32_t run = incl - sum;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        s_c[pad(tid * kItems + r)] = run;
        run += v[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int i = r * kThreads + tid;
        if (b0 + i < m) counts[b0 + i] = s_c[pad(i)];
    }
    if (tid == 0) boff[blockIdx.x] = tot;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int nb = gridDim.x;
    uint32_t carry = 0;
    for (int b0 = 0; b0 < nb; b0 += kThreads) {
        const int b = b0 + tid;
        const uint32_t x = b < nb ? __ldcg(boff + b) : 0u;
        const uint32_t inc = block_incl_scan(x, s_warp, tot);
        if (b < nb) boff[b] = carry + inc - x;
        carry += tot;
    }
}

// Scatter: each splat claims the next slot of its bucket (cursor = the
// scanned offset; afterwards cursor[c] = the start of bucket c + 1).
__global__ void __launch_bounds__(kThreads)
bucket_scatter_kernel(const uint32_t *ck, int64_t n, uint32_t *cursor, const uint32_t *boff,
                      uint32_t *idx) {
    pdl_begin();
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    uint32_t c[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t i = base + r * kThreads + threadIdx.x;
        c[r] = i < n ? ck[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t i = base + r * kThreads + threadIdx.x;
        if (i < n) idx[boff[c[r] / kChunk] + atomicAdd(cursor + c[r], 1u)] = (uint32_t)i;
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

// Sort a run of <= M ranks in registers by (full key, index).
template <int M>
__device__ __forceinline__ void sort_run(uint32_t *idx, int64_t i, int len, const uint64_t *full) {
    uint32_t v[M];
    uint64_t key[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
        v[a] = a < len ? idx[i + a] : 0xffffffffu;
        key[a] = a < len ? full[v[a]] : ~0ull;
    }
    // insertion network; padding entries (key ~0, index ~0) stay last
#pragma unroll
    for (int a = 1; a < M; ++a) {
#pragma unroll
        for (int b = a; b > 0; --b) {
            const bool sw = key[b - 1] > key[b] || (key[b - 1] == key[b] && v[b - 1] > v[b]);
            const uint64_t k0 = key[b - 1], k1 = key[b];
            const uint32_t v0 = v[b - 1], v1 = v[b];
            key[b - 1] = sw ? k1 : k0;
            key[b] = sw ? k0 : k1;
            v[b - 1] = sw ? v1 : v0;
            v[b] = sw ? v0 : v1;
        }
    }
#pragma unroll
    for (int a = 0; a < M; ++a)
        if (a < len) idx[i + a] = v[a];
}

// Per-bucket sort by (full key, index) after the scatter (bucket c spans
// [end[c - 1], end[c]) with end = the advanced cursors); a bucket larger than
// kMaxRun sets *need_full and the last block recomputes the whole order.
constexpr int kFixThreads = 1024;
constexpr int kFixPer = 4;  // buckets per thread
__global__ void __launch_bounds__(kFixThreads)
fixup_buckets_kernel(const uint32_t *end, const uint32_t *boff, uint32_t nb, uint32_t *idx,
                     int64_t n, const uint64_t *full, int32_t *need_full, uint32_t *done,
                     uint64_t *fkA, uint64_t *fkB, uint32_t *vscratch) {
    pdl_begin();
    bool flagged = false;
    const int64_t c0 = ((int64_t)blockIdx.x * kFixThreads + threadIdx.x) * kFixPer;
    uint32_t ends[kFixPer + 1];
#pragma unroll
    for (int q = 0; q <= kFixPer; ++q) {
        const int64_t c = c0 + q - 1;  // ends[q] = end of bucket c0 + q - 1
        ends[q] = c < 0 ? 0u : (c < nb ? boff[c / kChunk] + end[c] : 0u);
    }
#pragma unroll
    for (int q = 0; q < kFixPer; ++q) {
        const int64_t c = c0 + q;
        if (c >= nb) break;
        const uint32_t b = ends[q], e = ends[q + 1];
        const int len = (int)(e - b);
        if (len > kMaxRun) {
            *need_full = 1;
            flagged = true;
        } else if (len >= 2) {
            if (len <= 4) {
                sort_run<4>(idx, b, len, full);
            } else if (len <= 8) {
                sort_run<8>(idx, b, len, full);
            } else {
                uint32_t v[kMaxRun];
                uint64_t key[kMaxRun];
                for (int a = 0; a < len; ++a) {
                    v[a] = idx[b + a];
                    key[a] = full[v[a]];
                }
                for (int a = 1; a < len; ++a) {  // insertion sort by (key, index)
                    const uint32_t tv = v[a];
                    const uint64_t tk = key[a];
                    int z = a - 1;
                    while (z >= 0 && (key[z] > tk || (key[z] == tk && v[z] > tv))) {
                        key[z + 1] = key[z];
                        v[z + 1] = v[z];
                        --z;
                    }
                    key[z + 1] = tk;
                    v[z + 1] = tv;
                }
                for (int a = 0; a < len; ++a) idx[b + a] = v[a];
            }
        }
    }
    __shared__ bool s_last;
    if (__syncthreads_or(flagged)) __threadfence();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || ld_volatile((const uint32_t *)need_full) == 0) return;
    __threadfence();
    full_sort_block<kFixThreads>(full, n, fkA, fkB, idx, vscratch);
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
__device__ __forceinline__ void expand_pairs(const PairCtx &C, const uint32_t *sps,
                                             const uint32_t *cnts, const uint32_t *rxs,
                                             const uint32_t *rzs, Fn &&f) {
    // group u = the warp's ranks rb + 32u .. + 31, lane l holding rank rb + 32u + l
    // (already loaded and band-clipped by the caller: cnt 0 = no pairs)
    const int lane = threadIdx.x & 31;
    constexpr int kPer = kRanksPerWarp / 32;
#pragma unroll 1
    for (int u = 0; u < kPer; ++u) {
        const uint32_t sp = sps[u], cnt = cnts[u], rx = rxs[u], rz = rzs[u];
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

// per-block tile histogram -> hist[block * ntiles + tile] (coalesced rows), from a 2-D
// difference array of the block's tile rectangles (no pair expansion)
__global__ void __launch_bounds__(kThreads)
pair_hist_kernel(PairCtx C, uint32_t *hist, int nblocks) {
    extern __shared__ int smem_i32[];
    const int w1 = C.ntx + 1, h1 = C.bh + 1;
    int *D = smem_i32;
    for (int i = threadIdx.x; i < w1 * h1; i += kThreads) D[i] = 0;
    __syncthreads();
    pdl_begin();
    const int64_t r0 = (int64_t)blockIdx.x * kRanksPerBlock;
    // the thread's 8 ranks: rank loads together, then count and rectangle
    // loads together (K1 writes a rectangle for every splat)
    constexpr int kPer = kRanksPerBlock / kThreads;
    uint32_t sps[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int64_t r = r0 + threadIdx.x + (int64_t)kThreads * u;
        sps[u] = r < C.n ? __ldg(C.order + r) : 0xffffffffu;
    }
    int cnts[kPer];
    ushort4 rcs[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const bool ok = sps[u] != 0xffffffffu;
        cnts[u] = ok ? __ldg(C.count + sps[u]) : 0;
        rcs[u] = ok ? C.rect[sps[u]] : make_ushort4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u)
        if (cnts[u] > 0 && band_clip(C, rcs[u])) diff_add(D, w1, rcs[u], 1);
    __syncthreads();
    prefix2d(D, w1, h1, threadIdx.x, kThreads, [] { __syncthreads(); });
    const int tb = C.ty_lo * C.ntx;  // first tile of the band
    for (int t = threadIdx.x; t < C.ntx * C.bh; t += kThreads)
        hist[(int64_t)blockIdx.x * C.ntiles + tb + t] = (uint32_t)D[(t / C.ntx) * w1 + t % C.ntx];
}

// Per-tile exclusive scan of the per-block pair counts hist[block][tile], in
// place.  A CTA owns 32 consecutive tiles (lane = tile) and splits the blocks
// into 32 groups (warp = group): each thread sums its group's counts
// (coalesced 128-byte rows), the CTA scans the 32 group sums of each tile in
// shared memory, and each thread rewrites its group's counts as offsets inside
// the tile.  The kernel's last block scans the tile totals into tile_ranges
// (P = their sum, ranges clamped to the pair capacity so an overflowed frame
// never makes K3/K4 read past pair_splat), writes the optional heaviest-first
// tile schedule for K3/K4 (a 64-bucket counting sort of the tile pair counts;
// scheduling only), and re-arms the depth min/max words that K1 of the next
// frame reduces into.
constexpr int kOrderBuckets = 64;

constexpr int kScanThreads = 1024;
constexpr int kScanGroups = kScanThreads / 32;  // block groups per tile column

__global__ void __launch_bounds__(kScanThreads)
tile_scan_kernel(uint32_t *hist, int ntiles, int nblocks, uint32_t *totals, uint32_t *done,
                 int32_t *ranges, uint32_t cap, int32_t *n_pairs, int32_t *order,
                 unsigned long long *mm) {
    pdl_begin();
    __shared__ uint32_t s_grp[kScanGroups][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * 32 + lane;
    const int bpg = (nblocks + kScanGroups - 1) / kScanGroups;
    const int b0 = min(warp * bpg, nblocks), b1 = min(b0 + bpg, nblocks);
    uint32_t sum = 0;
    if (t < ntiles) {
        for (int bb = b0; bb < b1; bb += 8) {  // 8 independent loads per round
            uint32_t v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = bb + q < b1 ? hist[(int64_t)(bb + q) * ntiles + t] : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) sum += v[q];
        }
    }
    s_grp[warp][lane] = sum;
    __syncthreads();
    {  // warp w scans tile w's group sums (lane = group; padded rows: no conflicts)
        const uint32_t v = s_grp[lane][warp];
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        s_grp[lane][warp] = x - v;
        const int tw = blockIdx.x * 32 + warp;
        if (lane == 31 && tw < ntiles) {
            totals[tw] = x;
            __threadfence();  // the totals are read by the last block
        }
    }
    __syncthreads();
    if (t < ntiles) {
        uint32_t run = s_grp[warp][lane];
        for (int bb = b0; bb < b1; bb += 8) {
            uint32_t v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = bb + q < b1 ? hist[(int64_t)(bb + q) * ntiles + t] : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (bb + q < b1) hist[(int64_t)(bb + q) * ntiles + t] = run;
                run += v[q];
            }
        }
    }
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ uint32_t s_warp[32];
    uint64_t carry = 0;
    for (int base = 0; base < ntiles; base += kScanThreads) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < ntiles ? __ldcg(totals + i) : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;
        }
        __syncthreads();
        const uint32_t incl = x + (warp > 0 ? s_warp[warp - 1] : 0);
        if (i < ntiles) ranges[i] = (int32_t)min(carry + incl - v, (uint64_t)cap);
        carry += s_warp[31];
        __syncthreads();
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
    // warp-aggregated: lanes with equal buckets add once (the counts cluster)
    const uint32_t lt = lanemask_lt();
    for (int t = threadIdx.x; t < ntiles; t += kScanThreads) {
        const int b = bucket(ranges[t + 1] - ranges[t]);
        const uint32_t peers = __match_any_sync(__activemask(), b);
        if (lane == __ffs(peers) - 1) atomicAdd(&s_hist[b], __popc(peers));
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 64 buckets, two per lane
        const int c0 = s_hist[2 * lane], c1 = s_hist[2 * lane + 1];
        int x = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const int ex = x - c0 - c1;
        s_hist[2 * lane] = ex;
        s_hist[2 * lane + 1] = ex + c0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += kScanThreads) {
        const int b = bucket(ranges[t + 1] - ranges[t]);
        const uint32_t peers = __match_any_sync(__activemask(), b);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&s_hist[b], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        order[base + __popc(peers & lt)] = t;
    }
}

// stable placement: warp w of block b owns ranks [b*2048 + w*256, +256).
// Per-warp tile counts come from per-warp 2-D difference arrays; the pairs
// are expanded once, ranked within the warp by match_any and written.
__global__ void __launch_bounds__(kThreads)
pair_place_kernel(PairCtx C, const uint32_t *hist, const int32_t *ranges, int32_t *pair_splat, int W, int H) {
    extern __shared__ int smem_i32[];
    const int w1 = C.ntx + 1, h1 = C.bh + 1, cells = w1 * h1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kWarps * cells; i += kThreads) smem_i32[i] = 0;
    __syncthreads();
    pdl_begin();
    int *Dw = smem_i32 + warp * cells;
    const uint32_t lt = lanemask_lt();
    const int64_t rb = (int64_t)blockIdx.x * kRanksPerBlock + (int64_t)warp * kRanksPerWarp;
    const int64_t re = rb + kRanksPerWarp < C.n ? rb + kRanksPerWarp : C.n;
    // phase 1: per-warp tile counts (<= 256 per tile per warp); the warp's
    // 8 rank loads are issued together, then the dependent count / rect
    // loads; the band-clipped rectangles stay in registers for phase 3
    constexpr int kPer = kRanksPerWarp / 32;
    uint32_t sps[kPer], cnts[kPer], rxs[kPer], rzs[kPer];
    {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int64_t r = rb + lane + 32 * u;
            sps[u] = r < re ? __ldg(C.order + r) : 0xffffffffu;
        }
        ushort4 rcs[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const bool ok = sps[u] != 0xffffffffu;
            cnts[u] = ok ? (uint32_t)__ldg(C.count + sps[u]) : 0u;
            rcs[u] = ok ? C.rect[sps[u]] : make_ushort4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            ushort4 rc = rcs[u];
            if (cnts[u] > 0 && band_clip(C, rc)) {
                diff_add(Dw, w1, rc, 1);
                cnts[u] = (uint32_t)(rc.y - rc.x + 1) * (uint32_t)(rc.w - rc.z + 1);
                rxs[u] = (uint32_t)rc.x | ((uint32_t)rc.y << 16);
                rzs[u] = (uint32_t)rc.z | ((uint32_t)rc.w << 16);
            } else {
                cnts[u] = 0u;
                rxs[u] = rzs[u] = 0u;
            }
            if (sps[u] == 0xffffffffu) sps[u] = 0u;
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
        s_base[cell] = run ? (uint32_t)ranges[t] + hist[(int64_t)blockIdx.x * C.ntiles + t] : 0u;
    }
    __syncthreads();
    // phase 3: expand once, place (and cull-flag) every pair
    expand_pairs(C, sps, cnts, rxs, rzs, [&](bool ok, uint32_t sp, int tile, int tx, int ty) {
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
    int vbits;          // coarse-key bits: 2^vbits depth buckets (1-2 per splat)
    int64_t nbuckets;   // 2^vbits + 1 (the invisible splats' bucket last)
    int64_t nscan;      // bucket-scan blocks
    size_t ctrl_bytes;  // zeroed per frame: counters, flags, bucket counts, look-back words
};

// control block (offset 8): vctr | done_fix | done_tiles | need_full | pad (64 B)
// | bucket counts (nbuckets) | scan look-back words (nscan)
constexpr size_t kCtrlHead = 64;

Plan plan(int64_t n, int64_t cap, int32_t ntiles) {
    Plan L{};
    L.nbk = (int)((n + kChunk - 1) / kChunk);
    L.nbp = (int)((n + kRanksPerBlock - 1) / kRanksPerBlock);
    int lg = 1;
    while (lg < 29 && (1ll << lg) < n) ++lg;
    L.vbits = lg;
    L.nbuckets = (1ll << L.vbits) + 1;
    L.nscan = (L.nbuckets + kChunk - 1) / kChunk;
    L.ctrl_bytes = kCtrlHead + 4 * (size_t)L.nbuckets + 4 * (size_t)L.nscan;
    size_t sz[16] = {
        al(4 * (size_t)n), al(4),                                // 0 coarse keys, 1 (unused)
        al(4 * (size_t)n), al(4 * (size_t)n),                    // 2,3 order / fallback scratch
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
    uint32_t *ck = (uint32_t *)(ws + L.off[0]);
    uint32_t *ord = (uint32_t *)(ws + L.off[2]), *vscratch = (uint32_t *)(ws + L.off[3]);
    uint64_t *fkA = (uint64_t *)(ws + L.off[4]), *fkB = (uint64_t *)(ws + L.off[5]);
    char *ctrl = ws + L.off[8];
    uint32_t *vctr = (uint32_t *)ctrl;  // bucket-scan done counter
    uint32_t *done_fix = vctr + 1, *done_tiles = vctr + 2;
    int32_t *need_full = (int32_t *)(vctr + 3);
    uint32_t *bcount = (uint32_t *)(ctrl + kCtrlHead);
    uint32_t *sstatus = bcount + L.nbuckets;  // per scan block: total, then offset
    uint32_t *phist = (uint32_t *)(ws + L.off[10]);
    uint32_t *ttot = (uint32_t *)(ws + L.off[11]);
    const int nbk = L.nbk, nbp = L.nbp;

    // ---- 1. depth ranks: counting sort on a coarse key of ceil(log2 n) bits
    //      (1-2 buckets per splat), then each bucket sorted by (key, index)
    cudaMemsetAsync(ctrl, 0, L.ctrl_bytes, st);
    unsigned long long *mm = depth_minmax;
    if (!mm) {  // keys supplied directly: reduce their range here
        mm = (unsigned long long *)(ws + L.off[12]);
        init_minmax_kernel<<<1, 1, 0, st>>>(mm);
        int gb = (int)((n + kThreads * 8 - 1) / (kThreads * 8));
        gb = gb < 1 ? 1 : (gb > 1184 ? 1184 : gb);
        minmax_kernel<<<gb, kThreads, 0, st>>>(depth_key, n, mm);
    }
    ivr::launch(bucket_count_kernel, nbk, kThreads, 0, st, depth_key, n, mm, L.vbits, ck, bcount);
    ivr::launch(bucket_scan_kernel, (int)L.nscan, kThreads, 0, st, bcount, L.nbuckets, sstatus, vctr);
    ivr::launch(bucket_scatter_kernel, nbk, kThreads, 0, st, ck, n, bcount, sstatus, ord);
    const uint32_t nb_vis = (uint32_t)(L.nbuckets - 1);
    const int64_t fix_threads = (nb_vis + kFixPer - 1) / kFixPer;
    ivr::launch(fixup_buckets_kernel, (int)((fix_threads + kFixThreads - 1) / kFixThreads), kFixThreads,
           0, st, bcount, sstatus, nb_vis, ord, n, depth_key, need_full, done_fix, fkA, fkB,
           vscratch);
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
        ivr::launch(pair_hist_kernel, nbp, kThreads, sm_hist, st, C, phist, nbp);
    }
    ivr::launch(tile_scan_kernel, (ntiles + 31) / 32, kScanThreads, 0, st, phist, ntiles, nbp, ttot,
           done_tiles, tile_ranges, (uint32_t)pair_capacity, n_pairs, tile_order, depth_minmax);
    for (int y0 = 0; y0 < nty; y0 += band_rows) {
        C.ty_lo = y0;
        C.bh = y0 + band_rows <= nty ? band_rows : nty - y0;
        ivr::launch(pair_place_kernel, nbp, kThreads, sm_place, st, C, phist, tile_ranges, pair_splat,
               width, height);
    }
    return ivr::check_launch("ivr_bin_sort");
}
