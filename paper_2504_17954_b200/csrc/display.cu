// Service frame path on the device: display maps, uint8 conversion and PNG.
//
// render_modes.py:31-110 turns a float render into a display image (shaded
// RGBA with the colour clipped, alpha, unit normals mapped to [0,1], depth
// normalised over covered pixels), to_uint8 = clip(round(255 x), 0, 255), and
// png_bytes encodes it with PIL; service.py:169-187 / 255-275 sends either
// the raw uint8 bytes or the PNG for every frame.  Here:
//   * ivr_display_u8 builds the uint8 display image straight from the
//     float64 render maps (round half to even, as np.round);
//   * ivr_png_encode wraps it in a valid PNG without leaving the device:
//     filter-0 rows in stored (uncompressed) deflate blocks, the zlib adler32
//     and both chunk CRC-32s computed in parallel -- the bytes differ from
//     PIL's compressed stream, the decoded pixels are identical.
// Both are HBM-bound byte kernels.
#include <string.h>

#include "ivr_common.cuh"

namespace ivr {
namespace disp {

constexpr int kThreads = 256;

struct MapArgs {
    const double *out;  // (H, W, K) float64 render
    int H, W, K;
    int c_color, c_alpha, c_depth, c_normal;
    int mode;           // 0 shaded RGBA, 1 alpha (L), 2 normal (RGB), 3 depth (L)
    const double *lohi; // depth: covered min / max
    uint8_t *dst;
};

__device__ __forceinline__ uint8_t u8(double x) {
    double r = rint(x * 255.0);  // np.round: half to even
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    return (uint8_t)r;
}

__device__ __forceinline__ double clip01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

// covered-pixel depth range (render_modes.py:83-92): d = depth / alpha
__global__ void __launch_bounds__(kThreads) depth_range_kernel(MapArgs A, unsigned long long *mm) {
    const int64_t npx = (int64_t)A.H * A.W;
    double lo = 1e308, hi = -1e308;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < npx;
         i += (int64_t)gridDim.x * kThreads) {
        const double *o = A.out + i * A.K;
        const double a = o[A.c_alpha];
        if (a > 1e-6) {
            const double d = o[A.c_depth] / a;
            lo = fmin(lo, d);
            hi = fmax(hi, d);
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, s));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, s));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        // order-preserving integer images of the doubles (sign-magnitude -> two's)
        auto key = [](double v) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(v);
            return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        };
        atomicMin(mm, key(lo));
        atomicMax(mm + 1, key(hi));
    }
}

__global__ void decode_range_kernel(const unsigned long long *mm, double *lohi) {
    auto val = [](unsigned long long k) {
        const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        return __longlong_as_double((long long)b);
    };
    const bool any = mm[0] != ~0ull;
    lohi[0] = any ? val(mm[0]) : 0.0;
    lohi[1] = any ? val(mm[1]) : 0.0;
    lohi[2] = any ? 1.0 : 0.0;
}

__global__ void __launch_bounds__(kThreads) display_kernel(MapArgs A) {
    const int64_t npx = (int64_t)A.H * A.W;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < npx;
         i += (int64_t)gridDim.x * kThreads) {
        const double *o = A.out + i * A.K;
        if (A.mode == 0) {
            uint8_t *d = A.dst + 4 * i;
            for (int c = 0; c < 3; ++c) d[c] = u8(clip01(o[A.c_color + c]));
            d[3] = u8(o[A.c_alpha]);
        } else if (A.mode == 1) {
            A.dst[i] = u8(o[A.c_alpha]);
        } else if (A.mode == 2) {
            const double n0 = o[A.c_normal], n1 = o[A.c_normal + 1], n2 = o[A.c_normal + 2];
            const double nn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
            const bool ok = nn > 1e-8;
            uint8_t *d = A.dst + 3 * i;
            const double m = fmax(nn, 1e-8);
            d[0] = u8(0.5 * ((ok ? n0 / m : 0.0) + 1.0));
            d[1] = u8(0.5 * ((ok ? n1 / m : 0.0) + 1.0));
            d[2] = u8(0.5 * ((ok ? n2 / m : 0.0) + 1.0));
        } else {
            const double a = o[A.c_alpha];
            double v = 0.0;
            if (a > 1e-6) {
                const double dd = o[A.c_depth] / a;
                const double lo = A.lohi[0], hi = A.lohi[1];
                v = hi > lo ? (dd - lo) / (hi - lo) : 1.0;
            }
            A.dst[i] = u8(v);
        }
    }
}

// ---------------------------------------------------------------- PNG
constexpr int kStored = 65535;  // max stored-block payload

struct PngArgs {
    const uint8_t *img;  // H x W x C
    int H, W, C;
    int64_t raw;         // H * (1 + W C)
    int64_t data_off;    // offset of the zlib stream in the output
    uint8_t *out;
};

// zlib stream body: stored blocks of the filtered rows
__global__ void __launch_bounds__(kThreads) png_scatter_kernel(PngArgs A) {
    const int64_t row = (int64_t)A.W * A.C + 1;
    for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < A.raw;
         r += (int64_t)gridDim.x * kThreads) {
        const int64_t y = r / row, x = r % row;
        const uint8_t v = x == 0 ? 0 : A.img[y * (row - 1) + x - 1];
        const int64_t b = r / kStored;
        uint8_t *o = A.out + A.data_off + 2 + 5 * (b + 1) + r;
        *o = v;
        if (r % kStored == 0) {  // block header before this byte
            const int64_t len = min((int64_t)kStored, A.raw - r);
            uint8_t *h = o - 5;
            h[0] = (r + len == A.raw) ? 1 : 0;  // BFINAL, BTYPE = 00 (stored)
            h[1] = len & 0xff;
            h[2] = (len >> 8) & 0xff;
            h[3] = (~len) & 0xff;
            h[4] = ((~len) >> 8) & 0xff;
        }
    }
}

// adler32 of the filtered rows: sums of d_i and of (n - i) d_i, mod 65521
__global__ void __launch_bounds__(kThreads) png_adler_kernel(PngArgs A, unsigned long long *acc) {
    const int64_t row = (int64_t)A.W * A.C + 1;
    unsigned long long s1 = 0, s2 = 0;
    for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < A.raw;
         r += (int64_t)gridDim.x * kThreads) {
        const int64_t y = r / row, x = r % row;
        const unsigned v = x == 0 ? 0u : A.img[y * (row - 1) + x - 1];
        s1 += v;
        s2 = (s2 + (unsigned long long)((A.raw - r) % 65521) * v) % 65521ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, s1 % 65521ull);
        atomicAdd(acc + 1, s2 % 65521ull);
    }
}

__global__ void png_adler_finish(PngArgs A, const unsigned long long *acc) {
    const unsigned long long a = (1ull + acc[0]) % 65521ull;
    const unsigned long long b = ((unsigned long long)(A.raw % 65521) + acc[1]) % 65521ull;
    const uint32_t ad = (uint32_t)((b << 16) | a);
    uint8_t *o = A.out + A.data_off + 2 + 5 * ((A.raw + kStored - 1) / kStored) + A.raw;
    o[0] = ad >> 24;
    o[1] = (ad >> 16) & 0xff;
    o[2] = (ad >> 8) & 0xff;
    o[3] = ad & 0xff;
}

struct Bytes {
    uint8_t d[48];
    int n;
};

// small host-built byte strings written by a kernel (stream-ordered, no sync)
__global__ void put_bytes(Bytes b, uint8_t *dst) {
    for (int i = threadIdx.x; i < b.n; i += blockDim.x) dst[i] = b.d[i];
}

__global__ void init_u64(unsigned long long *p, unsigned long long a, unsigned long long b) {
    p[0] = a;
    p[1] = b;
}

__global__ void put_be32(const uint32_t *v, uint8_t *dst) {
    const uint32_t x = *v;
    dst[0] = x >> 24;
    dst[1] = (x >> 16) & 0xff;
    dst[2] = (x >> 8) & 0xff;
    dst[3] = x & 0xff;
}

}  // namespace disp
}  // namespace ivr

extern "C" int ivr_crc32(const uint8_t *data, int64_t n, uint32_t *out, ivr_stream_t stream);

extern "C" int ivr_display_u8(const double *out, int32_t height, int32_t width, int32_t k,
                              const int32_t cols[4], int32_t mode, uint8_t *dst, void *workspace,
                              ivr_stream_t stream) {
    using namespace ivr;
    using namespace ivr::disp;
    if (!out || !cols || !dst || !workspace || height < 1 || width < 1 || k < 1 || mode < 0 ||
        mode > 3 || cols[1] < 0 || (mode == 0 && cols[0] < 0) || (mode == 2 && cols[3] < 0) ||
        (mode == 3 && cols[2] < 0)) {
        set_error("ivr_display_u8: bad argument");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    MapArgs A{};
    A.out = out;
    A.H = height;
    A.W = width;
    A.K = k;
    A.c_color = cols[0];
    A.c_alpha = cols[1];
    A.c_depth = cols[2];
    A.c_normal = cols[3];
    A.mode = mode;
    A.dst = dst;
    unsigned long long *mm = reinterpret_cast<unsigned long long *>(workspace);
    double *lohi = reinterpret_cast<double *>(mm + 2);
    A.lohi = lohi;
    const int64_t npx = (int64_t)height * width;
    int blocks = (int)((npx + kThreads - 1) / kThreads);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (mode == 3) {
        init_u64<<<1, 1, 0, st>>>(mm, ~0ull, 0ull);
        depth_range_kernel<<<blocks, kThreads, 0, st>>>(A, mm);
        decode_range_kernel<<<1, 1, 0, st>>>(mm, lohi);
    }
    display_kernel<<<blocks, kThreads, 0, st>>>(A);
    return check_launch("display_kernel");
}

extern "C" int64_t ivr_png_size(int32_t height, int32_t width, int32_t channels) {
    const int64_t raw = (int64_t)height * (1 + (int64_t)width * channels);
    const int64_t blocks = (raw + ivr::disp::kStored - 1) / ivr::disp::kStored;
    const int64_t zlen = 2 + 5 * blocks + raw + 4;
    return 8 + 25 + (12 + zlen) + 12;
}

extern "C" int ivr_png_encode(const uint8_t *img, int32_t height, int32_t width, int32_t channels,
                              uint8_t *out, int64_t out_cap, void *workspace,
                              ivr_stream_t stream) {
    using namespace ivr;
    using namespace ivr::disp;
    if (!img || !out || !workspace || height < 1 || width < 1 ||
        !(channels == 1 || channels == 3 || channels == 4) ||
        out_cap < ivr_png_size(height, width, channels)) {
        set_error("ivr_png_encode: bad argument (1, 3 or 4 channels; output capacity)");
        return IVR_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    PngArgs A{};
    A.img = img;
    A.H = height;
    A.W = width;
    A.C = channels;
    A.raw = (int64_t)height * (1 + (int64_t)width * channels);
    const int64_t blocks_z = (A.raw + kStored - 1) / kStored;
    const int64_t zlen = 2 + 5 * blocks_z + A.raw + 4;
    // host-built header: signature, IHDR (with its CRC), IDAT length + tag, zlib header
    uint8_t hdr[8 + 25 + 8 + 2];
    const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
    memcpy(hdr, sig, 8);
    auto be32 = [](uint8_t *p, uint32_t v) {
        p[0] = v >> 24; p[1] = (v >> 16) & 0xff; p[2] = (v >> 8) & 0xff; p[3] = v & 0xff;
    };
    uint8_t *ih = hdr + 8;
    be32(ih, 13);
    memcpy(ih + 4, "IHDR", 4);
    be32(ih + 8, (uint32_t)width);
    be32(ih + 12, (uint32_t)height);
    ih[16] = 8;                                                        // bit depth
    ih[17] = channels == 1 ? 0 : (channels == 3 ? 2 : 6);              // L, RGB, RGBA
    ih[18] = ih[19] = ih[20] = 0;                                      // deflate, filter, no interlace
    {
        uint32_t c = 0xffffffffu;  // host CRC-32 of the 17 IHDR bytes
        for (int i = 4; i < 21; ++i) {
            c ^= ih[i];
            for (int b = 0; b < 8; ++b) c = (c & 1u) ? ((c >> 1) ^ 0xEDB88320u) : (c >> 1);
        }
        be32(ih + 21, ~c);
    }
    uint8_t *id = hdr + 8 + 25;
    be32(id, (uint32_t)zlen);
    memcpy(id + 4, "IDAT", 4);
    id[8] = 0x78;  // zlib: deflate, 32K window
    id[9] = 0x01;  // no dictionary, fastest (check bits: 0x7801 % 31 == 0)
    {
        Bytes b{};
        static_assert(sizeof(hdr) <= sizeof(b.d), "header fits");
        memcpy(b.d, hdr, sizeof(hdr));
        b.n = (int)sizeof(hdr);
        put_bytes<<<1, 64, 0, st>>>(b, out);
    }
    A.data_off = 8 + 25 + 8;
    A.out = out;
    unsigned long long *acc = reinterpret_cast<unsigned long long *>(workspace);
    uint32_t *crc = reinterpret_cast<uint32_t *>(acc + 2);
    init_u64<<<1, 1, 0, st>>>(acc, 0ull, 0ull);
    int g = (int)((A.raw + kThreads - 1) / kThreads);
    if (g > 148 * 8) g = 148 * 8;
    png_scatter_kernel<<<g, kThreads, 0, st>>>(A);
    png_adler_kernel<<<g, kThreads, 0, st>>>(A, acc);
    png_adler_finish<<<1, 1, 0, st>>>(A, acc);
    // IDAT CRC over tag + data, then IEND
    const int64_t idat_tag = 8 + 25 + 4;
    int rc = ivr_crc32(out + idat_tag, 4 + zlen, crc, stream);
    if (rc != IVR_OK) return rc;
    put_be32<<<1, 1, 0, st>>>(crc, out + idat_tag + 4 + zlen);
    {
        const uint8_t iend[12] = {0, 0, 0, 0, 'I', 'E', 'N', 'D', 0xae, 0x42, 0x60, 0x82};
        Bytes b{};
        memcpy(b.d, iend, 12);
        b.n = 12;
        put_bytes<<<1, 64, 0, st>>>(b, out + idat_tag + 4 + zlen + 4);
    }
    return check_launch("ivr_png_encode");
}
