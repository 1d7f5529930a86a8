// Microbenchmark: tcgen05.mma kind::i8 throughput with operands streamed
// from distinct buffers (no operand reuse between consecutive MMAs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void mma_ss(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%4, %5, %6, %7}, p;\n\t}" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_ts(uint32_t tmem, uint32_t ta, uint64_t bd, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%4, %5, %6, %7}, p;\n\t}" ::"r"(tmem),
                 "r"(ta), "l"(bd), "r"(idesc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

// mode 0: SS, A 16 KB x nbuf (128 x 128 B), B NB x 128 B x nbuf; mode 1: TS (A in TMEM, 4 stages)
template <int N, int MODE>
__global__ void k(long long *out, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t fin;
    __shared__ uint32_t slot;
    constexpr int NBUF = 4;
    unsigned char *A = (unsigned char *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char *B = A + (MODE == 0 ? NBUF * 16384 : 0);
    const int bytes = (MODE == 0 ? NBUF * 16384 : 0) + NBUF * N * 128;
    for (int i = threadIdx.x; i < bytes; i += blockDim.x) A[i] = (unsigned char)(i & 1);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 4 * NBUF) {
#pragma unroll
            for (int b = 0; b < NBUF; ++b) {
                const uint64_t bd = sdesc(smem_u32(B + b * N * 128));
                if (MODE == 0) {
                    const uint64_t ad = sdesc(smem_u32(A + b * 16384));
#pragma unroll
                    for (int u = 0; u < 4; ++u) mma_ss(tmem + (u & 1) * N, ad + 2 * u, bd + 2 * u, idesc);
                } else {
                    const uint32_t ta = tmem + 256 + b * 32;
#pragma unroll
                    for (int u = 0; u < 4; ++u) mma_ts(tmem + (u & 1) * N, ta + 8 * u, bd + 2 * u, idesc);
                }
            }
        }
        mma_commit(smem_u32(&fin));
        mbar_wait(smem_u32(&fin), 0);
        long long t2 = clock64();
        out[0] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int MODE>
void run() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    size_t smem = 1024 + (MODE == 0 ? 4 * 16384 : 0) + 4 * N * 128;
    cudaFuncSetAttribute(k<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 8192;
    k<N, MODE><<<1, 128, smem>>>(d, iters);
    k<N, MODE><<<1, 128, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s N=%3d: %.1f cyc/mma (%s)\n", MODE ? "TS" : "SS", N, (double)h[0] / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    run<24, 1>();
    run<32, 1>();
    return 0;
}
