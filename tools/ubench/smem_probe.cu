// smem_probe.cu -- on-chip ranking / accumulation primitives for the stream
// encode, over an R-MAT-like stream of 2^28 entries.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/smem_probe tools/ubench/smem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void gen(int64_t e, int scale, uint32_t *rows, uint32_t *cols) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned r = 0, c = 0;
        for (int l = 0; l < scale; l += 2) {
            unsigned long long x = mix64(i * 16 + l + 12345);
            for (int h = 0; h < 2; ++h) {
                unsigned u = h ? (unsigned)(x >> 32) : (unsigned)x;
                int rb = u >= 3264175145u, cb = (u >= 2448131276u && u < 3264175145u) || u >= 4080218931u;
                r = 2 * r + rb; c = 2 * c + cb;
            }
        }
        rows[i] = r; cols[i] = c;
    }
}

constexpr int TILE = 4096, NT = 512;

// rank by 8-bit digit with returning smem atomics, per 4096-entry tile
__global__ void __launch_bounds__(NT) k_rank_atomic(int64_t e, const uint32_t *rows, int shift, unsigned *out) {
    __shared__ unsigned cnt[256];
    unsigned acc = 0;
    for (int64_t t0 = (int64_t)blockIdx.x * TILE; t0 < e; t0 += (int64_t)gridDim.x * TILE) {
        if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < TILE / NT; ++u) {
            const unsigned d = (rows[t0 + u * NT + threadIdx.x] >> shift) & 255;
            acc += atomicAdd(cnt + d, 1u);
        }
        __syncthreads();
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

// rank by 8-bit digit with match_any + one atomic per distinct digit per warp
__global__ void __launch_bounds__(NT) k_rank_match(int64_t e, const uint32_t *rows, int shift, unsigned *out) {
    __shared__ unsigned cnt[256];
    unsigned acc = 0;
    const int lane = threadIdx.x & 31;
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int64_t t0 = (int64_t)blockIdx.x * TILE; t0 < e; t0 += (int64_t)gridDim.x * TILE) {
        if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < TILE / NT; ++u) {
            const unsigned d = (rows[t0 + u * NT + threadIdx.x] >> shift) & 255;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int leader = __ffs(peers) - 1;
            unsigned b = 0;
            if (lane == leader) b = atomicAdd(cnt + d, (unsigned)__popc(peers));
            b = __shfl_sync(0xffffffffu, b, leader);
            acc += b + __popc(peers & lt);
        }
        __syncthreads();
    }
    if (acc == 0xdeadbeef) out[0] = acc;
}

// f64 accumulation into a 256-row x K tile at (row & 255, label(col))
template <int MODE>
__global__ void __launch_bounds__(NT) k_acc(int64_t e, const uint32_t *rows, const uint32_t *cols, int k,
                                            double *out) {
    extern __shared__ double zt[];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * k; i += NT) zt[i] = 0.0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned r = rows[i] & 255, c = cols[i];
        const unsigned lab = (unsigned)((c * 2654435761u) >> 16) % (unsigned)k;
        const double x = 1.0 + (c & 7);
        const unsigned key = r * k + lab;
        if (MODE == 0) {
            atomicAdd(zt + key, x);
        } else {
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            double s = 0.0;
            // leader sums the peers' values through shuffles
            unsigned m = peers;
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                s += __shfl_sync(peers, x, l);
            }
            if (lane == __ffs(peers) - 1) atomicAdd(zt + key, s);
        }
    }
    __syncthreads();
    double s = 0;
    for (int i = threadIdx.x; i < 256 * k; i += NT) s += zt[i];
    if (s == 1234.5) out[0] = s;
}

int main() {
    const int64_t e = 1ll << 28;
    uint32_t *rows, *cols;
    unsigned *o;
    double *od;
    CK(cudaMalloc(&rows, e * 4)); CK(cudaMalloc(&cols, e * 4)); CK(cudaMalloc(&o, 64)); CK(cudaMalloc(&od, 64));
    gen<<<148 * 16, 256>>>(e, 24, rows, cols);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto T = [&](const char *name, auto fn) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-34s %8.3f ms  %7.1f G entries/s  (%s)\n", name, best, e / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    const int G = 148 * 4;
    T("rank atomic digit[16,24)", [&] { k_rank_atomic<<<G, NT>>>(e, rows, 16, o); });
    T("rank atomic digit[8,16)", [&] { k_rank_atomic<<<G, NT>>>(e, rows, 8, o); });
    T("rank atomic digit[0,8)", [&] { k_rank_atomic<<<G, NT>>>(e, rows, 0, o); });
    T("rank match digit[16,24)", [&] { k_rank_match<<<G, NT>>>(e, rows, 16, o); });
    T("rank match digit[0,8)", [&] { k_rank_match<<<G, NT>>>(e, rows, 0, o); });
    for (int k : {50, 20}) {
        const int sm = 256 * k * 8;
        cudaFuncSetAttribute(k_acc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        cudaFuncSetAttribute(k_acc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        char nm[64];
        snprintf(nm, 64, "f64 smem atomicAdd K=%d", k);
        T(nm, [&] { k_acc<0><<<148 * (k == 50 ? 2 : 2), NT, sm>>>(e, rows, cols, k, od); });
        snprintf(nm, 64, "f64 match+leader atomic K=%d", k);
        T(nm, [&] { k_acc<1><<<148 * 2, NT, sm>>>(e, rows, cols, k, od); });
    }
    return 0;
}
