// IVRG model files straight into HBM: device CRC-32 and chunk unpacking.
//
// The IVRG format (scene.py:242-436) is little-endian float32 SoA chunks
// (META / PALT / GEOM / RAWA or QATT / EDIT) closed by a zlib CRC-32 over the
// whole body.  The reference reads the file, runs zlib.crc32 on the host and
// converts every chunk f32 -> f64 with numpy before anything reaches a
// device.  Here the raw file bytes are copied to HBM once and
//   * ivr_crc32 checks the CRC with all SMs: each thread folds one 256-byte
//     segment (slicing-by-4 tables in shared memory), then every partial CRC
//     is shifted to the end of the message by a GF(2) multiply with
//     x^(8*bytes_after) mod P and XOR-reduced (CRC is linear);
//   * ivr_unpack widens f32 -> f64 (and u8 -> u16 codebook indices) directly
//     into the SoA tensors the renderer uses; chunk payloads need not be
//     aligned (META is arbitrary-length JSON), so the loads are byte-wise
//     and the stores coalesced.
// Both are HBM-bound: CRC reads 1 B per byte; unpack reads 4 B and writes 8 B
// per float.
#include "ivr_common.cuh"

namespace ivr {
namespace crc {

constexpr uint32_t kPoly = 0xEDB88320u;  // reflected CRC-32 (zlib)
constexpr int kSeg = 256;                // bytes per thread
constexpr int kThreads = 256;
constexpr int64_t kChunk = (int64_t)kSeg * kThreads;  // bytes per CTA

// a(x) * b(x) mod P(x) in the reflected representation (zlib multmodp)
__host__ __device__ constexpr uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t p = 0;
    for (int i = 0; i < 32; ++i) {
        if (a & (0x80000000u >> i)) p ^= b;
        b = (b & 1u) ? ((b >> 1) ^ kPoly) : (b >> 1);
    }
    return p;
}

struct Tables {
    uint32_t t[4][256];      // slicing-by-4
    uint32_t x2n[32];        // x^(2^k) mod P
    uint32_t seg_shift[kThreads];  // x^(8*kSeg*j) mod P
    constexpr Tables() : t(), x2n(), seg_shift() {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? ((c >> 1) ^ kPoly) : (c >> 1);
            t[0][i] = c;
        }
        for (int s = 1; s < 4; ++s)
            for (int i = 0; i < 256; ++i) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xFFu];
        uint32_t p = 1u << 30;  // x^1
        x2n[0] = p;
        for (int k = 1; k < 32; ++k) x2n[k] = p = multmodp(p, p);
        for (int j = 0; j < kThreads; ++j) seg_shift[j] = x2nmodp((uint64_t)kSeg * j, 3);
    }
    // x^(n * 2^k) mod P
    constexpr uint32_t x2nmodp(uint64_t n, int k) const {
        uint32_t p = 1u << 31;  // x^0
        while (n) {
            if (n & 1) p = multmodp(x2n[k & 31], p);
            n >>= 1;
            ++k;
        }
        return p;
    }
};

__device__ const Tables kTables = Tables();

__device__ __forceinline__ uint32_t x2nmodp_dev(const uint32_t *x2n, uint64_t n, int k) {
    uint32_t p = 1u << 31;
    while (n) {
        if (n & 1) p = multmodp(x2n[k & 31], p);
        n >>= 1;
        ++k;
    }
    return p;
}

__global__ void __launch_bounds__(kThreads) crc32_kernel(const uint8_t *__restrict__ data, int64_t n,
                                                         uint32_t *out) {
    __shared__ uint32_t T[4][256];
    __shared__ uint32_t s_x2n[32];
    __shared__ uint32_t s_red[kThreads / 32];
    const int tid = threadIdx.x;
    for (int s = 0; s < 4; ++s) T[s][tid] = kTables.t[s][tid];
    if (tid < 32) s_x2n[tid] = kTables.x2n[tid];
    __syncthreads();

    // segments are laid on 16-byte-aligned addresses: virtual offset v = i + head
    const int head = (int)(reinterpret_cast<uintptr_t>(data) & 15);
    const uint8_t *base = data - head;
    const int64_t nv = n + head;
    const int64_t cta0 = (int64_t)blockIdx.x * kChunk;
    const int64_t cta_end = min(cta0 + kChunk, nv);
    const int64_t start = max(cta0 + (int64_t)tid * kSeg, (int64_t)head);
    const int64_t end = min(cta0 + (int64_t)tid * kSeg + kSeg, nv);
    uint32_t c = 0;  // register from 0: f(segment), linear in the data
    if (start < end) {
        if (end - start == kSeg) {
            const uint4 *p = reinterpret_cast<const uint4 *>(base + start);
#pragma unroll 4
            for (int i = 0; i < kSeg / 16; ++i) {
                const uint4 v = __ldg(p + i);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    c ^= w[k];
                    c = T[3][c & 0xFFu] ^ T[2][(c >> 8) & 0xFFu] ^ T[1][(c >> 16) & 0xFFu] ^ T[0][c >> 24];
                }
            }
        } else {
            for (int64_t i = start; i < end; ++i) c = T[0][(c ^ base[i]) & 0xFFu] ^ (c >> 8);
        }
        // shift to the end of this CTA's range
        const int64_t after = cta_end - end;
        if (after) {
            const uint32_t sh = (after % kSeg == 0 && after / kSeg < kThreads)
                                    ? kTables.seg_shift[after / kSeg]
                                    : x2nmodp_dev(s_x2n, (uint64_t)after, 3);
            c = multmodp(sh, c);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
    if ((tid & 31) == 0) s_red[tid >> 5] = c;
    __syncthreads();
    if (tid == 0) {
        uint32_t r = 0;
        for (int w = 0; w < kThreads / 32; ++w) r ^= s_red[w];
        const int64_t tail = nv - cta_end;  // bytes after this CTA
        if (tail) r = multmodp(x2nmodp_dev(s_x2n, (uint64_t)tail, 3), r);
        if (blockIdx.x == 0)  // zlib pre/post inversion: ~0 shifted over n bytes, then ~
            r ^= multmodp(x2nmodp_dev(s_x2n, (uint64_t)n, 3), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
        atomicXor(out, r);
    }
}

}  // namespace crc

// kind 0: f32 LE -> f64; kind 1: u8 -> u16; kind 2: u16 LE -> u16
__global__ void __launch_bounds__(256) unpack_kernel(const uint8_t *__restrict__ src, int64_t count,
                                                     int kind, void *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (kind == 0) {
            const uint8_t *b = src + 4 * i;
            const uint32_t u = (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) |
                               ((uint32_t)b[3] << 24);
            static_cast<double *>(dst)[i] = (double)__uint_as_float(u);
        } else if (kind == 1) {
            static_cast<uint16_t *>(dst)[i] = src[i];
        } else {
            const uint8_t *b = src + 2 * i;
            static_cast<uint16_t *>(dst)[i] = (uint16_t)(b[0] | (b[1] << 8));
        }
    }
}

// f64 -> f32 LE bytes (IVRG writer, _f32_bytes scene.py:243-244)
__global__ void __launch_bounds__(256) pack_f32_kernel(const double *__restrict__ src, int64_t count,
                                                       uint8_t *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = __float_as_uint((float)src[i]);
        uint8_t *b = dst + 4 * i;
        b[0] = u & 0xFFu;
        b[1] = (u >> 8) & 0xFFu;
        b[2] = (u >> 16) & 0xFFu;
        b[3] = u >> 24;
    }
}

static int grid_elems(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace ivr

extern "C" int ivr_crc32(const uint8_t *data, int64_t n, uint32_t *out, ivr_stream_t stream) {
    using namespace ivr;
    if (n < 0 || !out || (n > 0 && !data)) {
        set_error("ivr_crc32: bad argument");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(out, 0, sizeof(uint32_t), st) != cudaSuccess) return check_launch("ivr_crc32 memset");
    if (n == 0) return IVR_OK;
    const int64_t nv = n + (int64_t)(reinterpret_cast<uintptr_t>(data) & 15);
    const int64_t blocks = (nv + crc::kChunk - 1) / crc::kChunk;
    crc::crc32_kernel<<<(unsigned)blocks, crc::kThreads, 0, st>>>(data, n, out);
    return check_launch("crc32_kernel");
}

extern "C" int ivr_unpack(const uint8_t *src, int64_t count, int32_t kind, void *dst,
                          ivr_stream_t stream) {
    using namespace ivr;
    if (count < 0 || kind < 0 || kind > 2 || (count > 0 && (!src || !dst))) {
        set_error("ivr_unpack: bad argument");
        return IVR_ERR_ARG;
    }
    if (count == 0) return IVR_OK;
    unpack_kernel<<<grid_elems(count), 256, 0, (cudaStream_t)stream>>>(src, count, kind, dst);
    return check_launch("unpack_kernel");
}

extern "C" int ivr_pack_f32(const double *src, int64_t count, uint8_t *dst, ivr_stream_t stream) {
    using namespace ivr;
    if (count < 0 || (count > 0 && (!src || !dst))) {
        set_error("ivr_pack_f32: bad argument");
        return IVR_ERR_ARG;
    }
    if (count == 0) return IVR_OK;
    pack_f32_kernel<<<grid_elems(count), 256, 0, (cudaStream_t)stream>>>(src, count, dst);
    return check_launch("pack_f32_kernel");
}
