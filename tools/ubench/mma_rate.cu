// Microbenchmark: tcgen05.mma kind::i8 issue rate (cycles per MMA) for
// M=128, K=32 and several N, SS mode, one CTA.  Debug tool, not shipped.
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
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

template <int N, int M = 128>
__global__ void k(long long *out, int iters, int chains, int commit_every) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar, fin, fin2;
    __shared__ uint32_t slot;
    unsigned char *A = (unsigned char *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char *B = A + 16384;
    for (int i = threadIdx.x; i < 16384 + N * 128; i += blockDim.x) A[i] = (unsigned char)(i & 1);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fin2)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fin2)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = sdesc(smem_u32(A)), bd = sdesc(smem_u32(B));
        int phase = 0;
        long long t0 = clock64();
        if (commit_every == -2) {
            // groups of 8 MMAs + one commit (to a barrier nobody waits on)
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) mma_i8(tmem + (u % (N >= 256 ? 2 : 4)) * N, ad + 2 * (u & 3), bd + 2 * (u & 3), idesc, 1);
                mma_commit(smem_u32(&bar));
            }
        } else if (commit_every == -3) {
            // groups of 4 MMAs + 2 commits
            for (int i = 0; i < iters; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) mma_i8(tmem + u * N, ad + 2 * u, bd + 2 * u, idesc, 1);
                mma_commit(smem_u32(&bar));
                mma_commit(smem_u32(&bar));
            }
        } else if (commit_every == -4) {
            // kernel-like loop: wait a completed barrier, fence, 4 MMAs, 2 commits
            for (int i = 0; i < iters; i += 4) {
                mbar_wait(smem_u32(&fin2), 0);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int u = 0; u < 4; ++u) mma_i8(tmem + u * N, ad + 2 * u, bd + 2 * u, idesc, (i | u) != 0);
                mma_commit(smem_u32(&bar));
                mma_commit(smem_u32(&bar));
            }
        } else if (commit_every == -5) {
            // same without the fence
            for (int i = 0; i < iters; i += 4) {
                mbar_wait(smem_u32(&fin2), 0);
#pragma unroll
                for (int u = 0; u < 4; ++u) mma_i8(tmem + u * N, ad + 2 * u, bd + 2 * u, idesc, (i | u) != 0);
                mma_commit(smem_u32(&bar));
                mma_commit(smem_u32(&bar));
            }
        } else if (commit_every < 0) {
            // unrolled, fixed descriptors, independent accumulators
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) mma_i8(tmem + (u % (N >= 256 ? 2 : 4)) * N, ad, bd, idesc, 1);
            }
        } else {
            for (int i = 0; i < iters; ++i) {
                const int ch = i % chains;
                mma_i8(tmem + ch * N, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i >= chains);
                if (commit_every && (i % commit_every) == commit_every - 1) mma_commit(smem_u32(&bar));
            }
        }
        long long t1 = clock64();
        mma_commit(smem_u32(&fin));
        mbar_wait(smem_u32(&fin), 0);
        (void)phase;
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int M = 128>
void run(int chains, int commit_every) {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    size_t smem = 1024 + 16384 + N * 128;
    cudaFuncSetAttribute(k<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 4096;
    k<N, M><<<1, 128, smem>>>(d, iters, chains, commit_every);
    k<N, M><<<1, 128, smem>>>(d, iters, chains, commit_every);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("M=%d N=%3d chains=%d commit_every=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", M, N, chains, commit_every,
           (double)h[0] / iters, (double)h[1] / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    run<32, 128>(1, -3);
    run<32, 128>(1, -4);
    run<32, 128>(1, -5);
    return 0;
}
