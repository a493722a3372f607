// Probe: one warp streams a global int array in 32-int chunks through two
// shared buffers filled by cp.async.bulk + mbarrier (the K3 id-stream
// pattern); checks the sum.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
struct Slots { __align__(16) int ids[2][40]; unsigned long long bar[2]; };
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void bulk_ids(int *dst, const int32_t *src, unsigned long long *b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 144;" ::"r"(smem_u32(b)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 144, [%2];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ int bar_try(unsigned long long *b, uint32_t phase) {
    uint32_t done;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(phase) : "memory");
    return (int)done;
}
__device__ long long walk(Slots &W, const int *a, int s0, int s1, int stop_at, int *spins);
__global__ void probe(const int *a, int s0, int s1, long long *out, int *spins) {
    __shared__ Slots W;
    // first walk breaks early (drain), second walk re-initialises and runs fully
    walk(W, a, s0, s1, 7, spins);
    long long sum = walk(W, a, s0, s1, 1 << 30, spins);
    if ((threadIdx.x & 31) == 0) *out = sum;
}
__device__ long long walk(Slots &W, const int *a, int s0, int s1, int stop_at, int *spins) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) { bar_init(&W.bar[0]); bar_init(&W.bar[1]); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    __syncwarp();
    auto issue = [&](int c) { int b = s0 + 32 * c; if (b < s1 && lane == 0) bulk_ids(W.ids[c & 1], a + (b & ~3), &W.bar[c & 1]); };
    long long sum = 0;
    int nch = (s1 - s0 + 31) / 32;
    int issued = 0;
    auto iss = [&](int c) { if (s0 + 32 * c < s1) { issue(c); issued = c + 1; } };
    iss(0); iss(1);
    int c = 0;
    for (; c < nch; ++c) {
        if (c == stop_at) break;
        int n = 0;
        while (!bar_try(&W.bar[c & 1], (uint32_t)((c >> 1) & 1))) { if (++n > 1000000) { if (lane == 0) atomicAdd(spins, 1); return 0; } }
        int b = s0 + 32 * c, j = b + lane;
        int v = j < s1 ? W.ids[c & 1][(b & 3) + lane] : 0;
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        iss(c + 2);
        sum += v;
    }
    for (int q = c; q < issued; ++q) {  // drain
        int n = 0;
        while (!bar_try(&W.bar[q & 1], (uint32_t)((q >> 1) & 1))) { if (++n > 1000000) { if (lane == 0) atomicAdd(spins, 100); return 0; } }
    }
    __syncwarp();
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    return sum;
}
int main() {
    const int N = 100000;
    int *h = new int[N + 64];
    for (int i = 0; i < N + 64; ++i) h[i] = i % 977;
    int *d; cudaMalloc(&d, sizeof(int) * (N + 64)); cudaMemcpy(d, h, sizeof(int) * (N + 64), cudaMemcpyHostToDevice);
    long long *o; int *sp; cudaMalloc(&o, 8); cudaMalloc(&sp, 4); cudaMemset(sp, 0, 4);
    int s0 = 13, s1 = 50013;
    probe<<<1, 32>>>(d, s0, s1, o, sp);
    cudaError_t e = cudaDeviceSynchronize();
    long long got; int spins; cudaMemcpy(&got, o, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&spins, sp, 4, cudaMemcpyDeviceToHost);
    long long ref = 0; for (int i = s0; i < s1; ++i) ref += h[i];
    printf("err=%s got=%lld ref=%lld stuck=%d\n", cudaGetErrorString(e), got, ref, spins);
    return 0;
}
