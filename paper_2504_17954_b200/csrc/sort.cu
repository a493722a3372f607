// K2 -- bit-exact (tile, depth) pair ordering on device.
//
// Reproduces np.lexsort((depth[pair_splat], pair_tile)) (rasterizer.py:129)
// over the pairs emitted by fill_pairs (_kernels.py:19-28) without ever
// materialising an 80-bit composite key:
//   1. stable LSD radix sort of the N float64 depth keys (positive doubles
//      compare like their bit patterns; invisible splats carry ~0 and sort
//      last; ties keep index order = lexsort's tie break on pair order);
//   2. exclusive scan of the per-splat tile counts in depth-rank order and
//      emission of the (tile, splat) pairs in rank order;
//   3. stable LSD radix sort of the pairs by 16-bit tile id (2 passes);
//   4. tile ranges (np.searchsorted(pair_tile, arange(T+1))) from the run
//      boundaries of the sorted tile ids.
// All sizes that depend on the data live in device memory, so the whole
// sequence is stream-ordered and CUDA-graph capturable.
#include "ivr_common.cuh"

namespace ivr {
namespace sortk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;                       // per thread
constexpr int kChunk = kThreads * kItems;       // 2048 items per block
constexpr int kRadix = 256;

__device__ __forceinline__ int64_t load_n(const int32_t *n_dev, int64_t n_host, int64_t cap) {
    int64_t n = n_dev ? (int64_t)(*n_dev) : n_host;
    return n < cap ? n : cap;
}

// Inclusive block scan of one uint32 per thread (256 threads).
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

// ----------------------------------------------------------------- digit histograms
// All eight byte-histograms of the depth keys in one read; used to skip
// passes whose digit is constant over all keys.
__global__ void __launch_bounds__(kThreads)
key64_hist_kernel(const uint64_t *keys, int64_t n, uint32_t *hist /* [8][256] */) {
    __shared__ uint32_t s[8 * kRadix];
    for (int i = threadIdx.x; i < 8 * kRadix; i += kThreads) s[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kThreads) {
        const uint64_t k = keys[i];
#pragma unroll
        for (int p = 0; p < 8; ++p) atomicAdd(&s[p * kRadix + ((k >> (8 * p)) & 255)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * kRadix; i += kThreads)
        if (s[i]) atomicAdd(&hist[i], s[i]);
}

// cur[p] in {0: caller input (values = identity), 1: buffer A, 2: buffer B}
__global__ void pass_plan_kernel(const uint32_t *hist, int64_t n, int npass, int32_t *skip,
                                 int32_t *cur) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int c = 0;
    cur[0] = 0;
    for (int p = 0; p < npass; ++p) {
        bool trivial = false;
        for (int d = 0; d < kRadix; ++d)
            if ((int64_t)hist[p * kRadix + d] == n) trivial = true;
        skip[p] = trivial || n == 0;
        if (!skip[p]) c = (c == 1) ? 2 : 1;
        cur[p + 1] = c;
    }
}

template <typename KeyT>
struct Bufs {
    const KeyT *in_keys;      // cur == 0
    const uint32_t *in_vals;  // cur == 0 (nullptr = identity)
    KeyT *keys[2];            // cur == 1, 2
    uint32_t *vals[2];
};

template <typename KeyT>
__device__ __forceinline__ void src_of(const Bufs<KeyT> &B, int c, const KeyT *&k, const uint32_t *&v) {
    if (c == 0) { k = B.in_keys; v = B.in_vals; }
    else { k = B.keys[c - 1]; v = B.vals[c - 1]; }
}

// ----------------------------------------------------------------- upsweep
template <typename KeyT>
__global__ void __launch_bounds__(kThreads)
upsweep_kernel(Bufs<KeyT> B, const int32_t *cur, const int32_t *skip, int pass, int shift,
               const int32_t *n_dev, int64_t n_host, int64_t cap, uint32_t *blockhist,
               int nblocks) {
    if (skip && skip[pass]) return;
    const int64_t n = load_n(n_dev, n_host, cap);
    __shared__ uint32_t s[kRadix];
    s[threadIdx.x] = 0;
    __syncthreads();
    const KeyT *keys;
    const uint32_t *vals;
    src_of(B, cur ? cur[pass] : pass == 0 ? 0 : 1, keys, vals);
    const int64_t base = (int64_t)blockIdx.x * kChunk;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + r * kThreads + threadIdx.x;
        if (idx < n) atomicAdd(&s[(uint32_t)(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    blockhist[(int64_t)threadIdx.x * nblocks + blockIdx.x] = s[threadIdx.x];
}

// ----------------------------------------------------------------- per-digit row scan
// grid = 256 (one block per digit): exclusive scan of blockhist[d][0..nblocks)
__global__ void __launch_bounds__(1024)
rowscan_kernel(const int32_t *skip, int pass, uint32_t *blockhist, int nblocks,
               uint32_t *rowtotal) {
    if (skip && skip[pass]) return;
    __shared__ uint32_t s_warp[32];
    uint32_t *row = blockhist + (int64_t)blockIdx.x * nblocks;
    uint32_t carry = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < nblocks; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nblocks ? row[i] : 0;
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
        if (i < nblocks) row[i] = carry + incl - v;
        carry += s_warp[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) rowtotal[blockIdx.x] = carry;
}

// ----------------------------------------------------------------- downsweep
template <typename KeyT>
__global__ void __launch_bounds__(kThreads)
downsweep_kernel(Bufs<KeyT> B, const int32_t *cur, const int32_t *skip, int pass, int shift,
                 const int32_t *n_dev, int64_t n_host, int64_t cap,
                 const uint32_t *blockhist, const uint32_t *rowtotal, int nblocks,
                 KeyT *fixed_dst_keys, uint32_t *fixed_dst_vals) {
    if (skip && skip[pass]) return;
    const int64_t n = load_n(n_dev, n_host, cap);
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    if (base >= n) return;
    __shared__ uint32_t s_wcnt[kWarps][kRadix];
    __shared__ uint32_t s_gbase[kRadix];    // global base of digit d for this block
    __shared__ uint32_t s_lstart[kRadix];   // block-local start of digit d
    __shared__ uint32_t s_warp[kWarps];
    __shared__ KeyT s_keys[kChunk];
    __shared__ uint32_t s_vals[kChunk];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int w = 0; w < kWarps; ++w) s_wcnt[w][tid] = 0;
    // digit base = exclusive scan of the digit totals + this block's row offset
    uint32_t tot;
    const uint32_t rt = rowtotal[tid];
    const uint32_t incl = block_incl_scan(rt, s_warp, tot);
    s_gbase[tid] = incl - rt + blockhist[(int64_t)tid * nblocks + blockIdx.x];

    const int c_src = cur ? cur[pass] : (pass == 0 ? 0 : 1);
    const KeyT *keys;
    const uint32_t *vals;
    src_of(B, c_src, keys, vals);
    KeyT *dkeys = fixed_dst_keys ? fixed_dst_keys : B.keys[cur ? cur[pass + 1] - 1 : (pass & 1) ? 0 : 1];
    uint32_t *dvals = fixed_dst_vals ? fixed_dst_vals : B.vals[cur ? cur[pass + 1] - 1 : (pass & 1) ? 0 : 1];
    __syncthreads();

    KeyT k[kItems];
    uint32_t v[kItems], dig[kItems], rank[kItems];
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + warp * (32 * kItems) + r * 32 + lane;
        const bool ok = idx < n;
        k[r] = ok ? keys[idx] : (KeyT)0;
        v[r] = ok ? (vals ? vals[idx] : (uint32_t)idx) : 0u;
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
    // per digit: exclusive scan across warps; block count per digit
    {
        uint32_t run = 0;
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_wcnt[w][tid];
            s_wcnt[w][tid] = run;
            run += c;
        }
        const uint32_t inc = block_incl_scan(run, s_warp, tot);
        s_lstart[tid] = inc - run;
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

// ----------------------------------------------------------------- rank-order scan
__device__ __forceinline__ const uint32_t *sorted_vals(const Bufs<uint64_t> &B, const int32_t *cur, int npass) {
    const int c = cur[npass];
    return c == 0 ? nullptr : B.vals[c - 1];
}

__device__ __forceinline__ uint32_t count_at(const Bufs<uint64_t> &B, const int32_t *cur,
                                             int npass, const int32_t *count, int64_t r) {
    const uint32_t *sv = sorted_vals(B, cur, npass);
    const int64_t i = sv ? (int64_t)sv[r] : r;
    return (uint32_t)count[i];
}

__global__ void __launch_bounds__(kThreads)
scan_reduce_kernel(Bufs<uint64_t> B, const int32_t *cur, int npass, const int32_t *count,
                   int64_t n, uint32_t *partial) {
    __shared__ uint32_t s_warp[kWarps];
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + r * kThreads + threadIdx.x;
        if (idx < n) sum += count_at(B, cur, npass, count, idx);
    }
    uint32_t tot;
    block_incl_scan(sum, s_warp, tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024)
scan_partials_kernel(uint32_t *partial, int nb, int32_t *n_pairs) {
    __shared__ uint32_t s_warp[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t carry = 0;
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < nb ? partial[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_warp[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;
        }
        __syncthreads();
        const uint32_t incl = x + (warp > 0 ? s_warp[warp - 1] : 0);
        if (i < nb) partial[i] = (uint32_t)carry + incl - v;
        carry += s_warp[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_pairs = carry > 0x7fffffffull ? 0x7fffffff : (int32_t)carry;
}

// exclusive scan of counts in rank order, then emit this rank's pairs
__global__ void __launch_bounds__(kThreads)
emit_kernel(Bufs<uint64_t> B, const int32_t *cur, int npass, const int32_t *count,
            const ushort4 *rect, int64_t n, const uint32_t *partial, int ntx, int64_t cap,
            uint32_t *tile_key, uint32_t *pair_val) {
    __shared__ uint32_t s_warp[kWarps];
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const uint32_t *sv = sorted_vals(B, cur, npass);
    // blocked arrangement: thread t owns items base + t*kItems .. +kItems-1
    uint32_t c[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + (int64_t)threadIdx.x * kItems + r;
        c[r] = idx < n ? (uint32_t)count[sv ? (int64_t)sv[idx] : idx] : 0u;
        sum += c[r];
    }
    uint32_t tot;
    const uint32_t incl = block_incl_scan(sum, s_warp, tot);
    uint64_t off = (uint64_t)partial[blockIdx.x] + incl - sum;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const int64_t idx = base + (int64_t)threadIdx.x * kItems + r;
        if (c[r]) {
            const uint32_t i = sv ? sv[idx] : (uint32_t)idx;
            const ushort4 rc = rect[i];
            const int w = rc.y - rc.x + 1;
            for (uint32_t q = 0; q < c[r]; ++q) {
                const uint64_t pos = off + q;
                if (pos >= (uint64_t)cap) break;
                const int ty = rc.z + (int)q / w, tx = rc.x + (int)q % w;
                tile_key[pos] = (uint32_t)(ty * ntx + tx);
                pair_val[pos] = i;
            }
        }
        off += c[r];
    }
}

__global__ void __launch_bounds__(kThreads)
ranges_kernel(const uint32_t *tile_key, const int32_t *n_pairs, int64_t cap, int ntiles,
              int32_t *ranges) {
    const int64_t n = load_n(n_pairs, 0, cap);
    const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (i > n) return;
    if (n == 0) {
        for (int t = 0; t <= ntiles; ++t) ranges[t] = 0;
        return;
    }
    const int prev = i == 0 ? -1 : (int)tile_key[i - 1];
    const int here = i == n ? ntiles : (int)tile_key[i];
    for (int t = prev + 1; t <= here; ++t) ranges[t] = (int32_t)i;
}

}  // namespace sortk
}  // namespace ivr

using namespace ivr::sortk;

namespace {
struct Layout {
    size_t off[16];
    size_t total;
};

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

Layout plan(int64_t n, int64_t cap, int32_t ntiles) {
    Layout L{};
    const int64_t nb_keys = (n + kChunk - 1) / kChunk;
    const int64_t nb_pairs = (cap + kChunk - 1) / kChunk;
    const int64_t nbmax = nb_keys > nb_pairs ? nb_keys : nb_pairs;
    size_t sz[16] = {
        al(8 * (size_t)n), al(8 * (size_t)n),       // keyA keyB
        al(4 * (size_t)n), al(4 * (size_t)n),       // valA valB
        al(4 * (size_t)cap), al(4 * (size_t)cap),   // tile keys A/B
        al(4 * (size_t)cap), al(4 * (size_t)cap),   // pair vals A/B
        al(4 * (size_t)(256 * (nbmax + 1))),        // blockhist
        al(4 * 256),                                // rowtotal
        al(4 * 8 * 256),                            // key64 hist
        al(4 * 16), al(4 * 16),                     // skip, cur
        al(4 * (size_t)(nb_keys + 1)),              // scan partials
        0, 0};
    (void)ntiles;
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
    return plan(n < 1 ? 1 : n, pair_capacity < 1 ? 1 : pair_capacity, ntiles).total;
}

extern "C" int ivr_bin_sort(int64_t n, const uint64_t *depth_key, const int32_t *count,
                            const uint16_t *rect, int32_t ntx, int32_t nty, int64_t pair_capacity,
                            void *workspace, size_t workspace_bytes, int32_t *pair_splat,
                            int32_t *tile_ranges, int32_t *n_pairs, ivr_stream_t stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int32_t ntiles = ntx * nty;
    if (n < 0 || pair_capacity < 1 || ntx < 1 || nty < 1 || ntiles > 65535 || !tile_ranges ||
        !n_pairs || !pair_splat || !workspace) {
        ivr::set_error("ivr_bin_sort: bad argument");
        return IVR_ERR_ARG;
    }
    if (n > 0x7fffffffll || pair_capacity > 0x7fffffffll) {
        ivr::set_error("ivr_bin_sort: sizes must fit int32");
        return IVR_ERR_ARG;
    }
    const Layout L = plan(n < 1 ? 1 : n, pair_capacity, ntiles);
    if (workspace_bytes < L.total) {
        ivr::set_error("ivr_bin_sort: workspace too small");
        return IVR_ERR_ARG;
    }
    if (n == 0) {
        cudaMemsetAsync(n_pairs, 0, 4, st);
        cudaMemsetAsync(tile_ranges, 0, 4 * (size_t)(ntiles + 1), st);
        return ivr::check_launch("ivr_bin_sort(empty)");
    }
    char *ws = (char *)workspace;
    Bufs<uint64_t> DB{};
    DB.in_keys = depth_key;
    DB.in_vals = nullptr;
    DB.keys[0] = (uint64_t *)(ws + L.off[0]);
    DB.keys[1] = (uint64_t *)(ws + L.off[1]);
    DB.vals[0] = (uint32_t *)(ws + L.off[2]);
    DB.vals[1] = (uint32_t *)(ws + L.off[3]);
    uint32_t *tkA = (uint32_t *)(ws + L.off[4]);
    uint32_t *tkB = (uint32_t *)(ws + L.off[5]);
    uint32_t *pvA = (uint32_t *)(ws + L.off[6]);
    uint32_t *pvB = (uint32_t *)(ws + L.off[7]);
    uint32_t *blockhist = (uint32_t *)(ws + L.off[8]);
    uint32_t *rowtotal = (uint32_t *)(ws + L.off[9]);
    uint32_t *hist64 = (uint32_t *)(ws + L.off[10]);
    int32_t *skip = (int32_t *)(ws + L.off[11]);
    int32_t *cur = (int32_t *)(ws + L.off[12]);
    uint32_t *partial = (uint32_t *)(ws + L.off[13]);

    // ---- 1. stable depth sort (8 byte-passes, constant digits skipped)
    const int nbk = (int)((n + kChunk - 1) / kChunk);
    cudaMemsetAsync(hist64, 0, 4 * 8 * 256, st);
    int hb = (int)((n + kThreads * 16 - 1) / (kThreads * 16));
    hb = hb < 1 ? 1 : (hb > 1184 ? 1184 : hb);
    key64_hist_kernel<<<hb, kThreads, 0, st>>>(depth_key, n, hist64);
    pass_plan_kernel<<<1, 32, 0, st>>>(hist64, n, 8, skip, cur);
    for (int p = 0; p < 8; ++p) {
        upsweep_kernel<uint64_t><<<nbk, kThreads, 0, st>>>(DB, cur, skip, p, 8 * p, nullptr, n, n,
                                                            blockhist, nbk);
        rowscan_kernel<<<256, 1024, 0, st>>>(skip, p, blockhist, nbk, rowtotal);
        downsweep_kernel<uint64_t><<<nbk, kThreads, 0, st>>>(DB, cur, skip, p, 8 * p, nullptr, n, n,
                                                              blockhist, rowtotal, nbk, nullptr,
                                                              nullptr);
    }
    // ---- 2. counts in rank order -> offsets -> emit pairs
    scan_reduce_kernel<<<nbk, kThreads, 0, st>>>(DB, cur, 8, count, n, partial);
    scan_partials_kernel<<<1, 1024, 0, st>>>(partial, nbk, n_pairs);
    emit_kernel<<<nbk, kThreads, 0, st>>>(DB, cur, 8, count, (const ushort4 *)rect, n, partial, ntx,
                                          pair_capacity, tkA, pvA);
    // ---- 3. stable tile sort: (tkA, pvA) -> (tkB, pvB) -> (tkA, pair_splat)
    const int nbp = (int)((pair_capacity + kChunk - 1) / kChunk);
    {
        Bufs<uint32_t> P0{};
        P0.in_keys = tkA;
        P0.in_vals = pvA;
        upsweep_kernel<uint32_t><<<nbp, kThreads, 0, st>>>(P0, nullptr, nullptr, 0, 0, n_pairs, 0,
                                                            pair_capacity, blockhist, nbp);
        rowscan_kernel<<<256, 1024, 0, st>>>(nullptr, 0, blockhist, nbp, rowtotal);
        downsweep_kernel<uint32_t><<<nbp, kThreads, 0, st>>>(P0, nullptr, nullptr, 0, 0, n_pairs, 0,
                                                              pair_capacity, blockhist, rowtotal, nbp,
                                                              tkB, pvB);
        Bufs<uint32_t> P1{};
        P1.in_keys = tkB;
        P1.in_vals = pvB;
        upsweep_kernel<uint32_t><<<nbp, kThreads, 0, st>>>(P1, nullptr, nullptr, 0, 8, n_pairs, 0,
                                                            pair_capacity, blockhist, nbp);
        rowscan_kernel<<<256, 1024, 0, st>>>(nullptr, 0, blockhist, nbp, rowtotal);
        downsweep_kernel<uint32_t><<<nbp, kThreads, 0, st>>>(P1, nullptr, nullptr, 0, 8, n_pairs, 0,
                                                              pair_capacity, blockhist, rowtotal, nbp,
                                                              tkA, (uint32_t *)pair_splat);
    }
    // ---- 4. tile ranges
    const int rb = (int)((pair_capacity + 1 + kThreads - 1) / kThreads);
    ranges_kernel<<<rb, kThreads, 0, st>>>(tkA, n_pairs, pair_capacity, ntiles, tile_ranges);
    return ivr::check_launch("ivr_bin_sort");
}
