// part_probe.cu -- micro-measurements that choose the stream-encode design
// (DESIGN.md §3.5): global atomics, scattered stores, gathers and shared-
// memory histograms over an R-MAT-like stream of 2^28 entries (2^24 rows).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/part_probe part_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void gen(int64_t e, int scale, int64_t *rows, int64_t *cols, float *w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        long long r = 0, c = 0;
        for (int l = 0; l < scale; l += 2) {
            unsigned long long x = mix64(i * 16 + l + 12345);
            for (int h = 0; h < 2; ++h) {
                unsigned u = h ? (unsigned)(x >> 32) : (unsigned)x;
                int rb = u >= 3264175145u, cb = (u >= 2448131276u && u < 3264175145u) || u >= 4080218931u;
                r = 2 * r + rb; c = 2 * c + cb;
            }
        }
        rows[i] = r; cols[i] = c; w[i] = 0.5f;
    }
}

__global__ void k_deg_red(int64_t e, const int64_t *rows, const float *w, double *d) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(d + rows[i], (double)w[i]);
}

__global__ void k_cnt_red(int64_t e, const int64_t *rows, unsigned *c) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(c + rows[i], 1u);
}

// per entry: returning atomic on the bucket cursor, then an 8-byte store
__global__ void k_scatter_atomic(int64_t e, const int64_t *rows, const int64_t *cols, int shift, unsigned *cur,
                                 unsigned long long *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rows[i];
        const unsigned b = (unsigned)(r >> shift);
        const unsigned p = atomicAdd(cur + b, 1u);
        out[p] = ((unsigned long long)r << 32) | (unsigned)cols[i];
    }
}

// warp-aggregated: lanes with the same bucket share one atomic
__global__ void k_scatter_wagg(int64_t e, const int64_t *rows, const int64_t *cols, int shift, unsigned *cur,
                               unsigned long long *out) {
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; i0 < e;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + lane;
        const bool ok = i < e;
        const int64_t r = ok ? rows[i] : 0;
        const unsigned b = ok ? (unsigned)(r >> shift) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (lane == leader && ok) base = atomicAdd(cur + b, (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (ok) {
            unsigned lt;
            asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
            out[base + __popc(peers & lt)] = ((unsigned long long)r << 32) | (unsigned)cols[i];
        }
    }
}

__global__ void k_gather(int64_t e, const int64_t *cols, const double2 *tab, double *out) {
    double acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = __ldg(tab + cols[i]);
        acc += v.x + v.y;
    }
    if (acc == 12345.678) out[0] = acc;
}

__global__ void k_gather8(int64_t e, const int64_t *cols, const double *tab, double *out) {
    double acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldg(tab + cols[i]);
    if (acc == 12345.678) out[0] = acc;
}

__global__ void k_stream(int64_t e, const int64_t *rows, const int64_t *cols, const float *w, double *out) {
    double acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        acc += rows[i] + cols[i] + w[i];
    if (acc == 12345.678) out[0] = acc;
}

// shared-memory histogram: 2^bits u32 counters per CTA, flushed nonzero
extern __shared__ unsigned smh[];
__global__ void k_smem_hist(int64_t e, const int64_t *rows, int shift, int nb, unsigned *g) {
    for (int i = threadIdx.x; i < nb; i += blockDim.x) smh[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(smh + (rows[i] >> shift), 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (smh[i]) atomicAdd(g + i, smh[i]);
}

int main() {
    const int scale = 24;
    const int64_t e = 1ll << 28, n = 1ll << scale;
    int64_t *rows, *cols;
    float *w;
    double *d, *out;
    double2 *tab;
    unsigned *cnt, *cur;
    unsigned long long *sc;
    CK(cudaMalloc(&rows, e * 8)); CK(cudaMalloc(&cols, e * 8)); CK(cudaMalloc(&w, e * 4));
    CK(cudaMalloc(&d, n * 8)); CK(cudaMalloc(&tab, n * 16)); CK(cudaMalloc(&cnt, n * 4));
    CK(cudaMalloc(&cur, n * 4)); CK(cudaMalloc(&sc, e * 8)); CK(cudaMalloc(&out, 64));
    void *flush; CK(cudaMalloc(&flush, 512 << 20));
    gen<<<148 * 16, 256>>>(e, scale, rows, cols, w);
    CK(cudaMemset(tab, 0, n * 16));
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    unsigned *base; CK(cudaMalloc(&base, n * 4));
    unsigned *hcnt = (unsigned *)malloc(n * 4);
    auto set_bases = [&](int shift) {
        cudaMemset(cnt, 0, n * 4);
        k_cnt_red<<<148 * 8, 256>>>(e, rows, cnt);  // per row
        cudaMemcpy(hcnt, cnt, n * 4, cudaMemcpyDeviceToHost);
        unsigned s = 0;
        for (int64_t bk = 0; bk < (n >> shift); ++bk) {
            unsigned c = 0;
            for (int64_t r = bk << shift; r < (bk + 1) << shift; ++r) c += hcnt[r];
            hcnt[bk] = s;
            s += c;
        }
        cudaMemcpy(base, hcnt, (n >> shift) * 4, cudaMemcpyHostToDevice);
    };
    int cur_shift = -1;
    auto T = [&](const char *name, auto fn, double bytes) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            cudaMemset(d, 0, n * 8); cudaMemset(cnt, 0, n * 4);
            if (cur_shift >= 0) cudaMemcpy(cur, base, (n >> cur_shift) * 4, cudaMemcpyDeviceToDevice);
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-28s %8.3f ms  %7.1f G entries/s  %7.1f GB/s  (%s)\n", name, best, e / best / 1e6,
               bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    const int G = 148 * 8, B = 256;
    T("stream rows+cols+w", [&] { k_stream<<<G, B>>>(e, rows, cols, w, out); }, 20.0 * e);
    T("deg f64 RED (2^24 rows)", [&] { k_deg_red<<<G, B>>>(e, rows, w, d); }, 12.0 * e);
    T("cnt u32 RED (2^24 rows)", [&] { k_cnt_red<<<G, B>>>(e, rows, cnt); }, 8.0 * e);
    for (int shift : {8, 14}) {
        set_bases(shift);
        cur_shift = shift;
        // cursors need bucket bases: fake them as b * cap so positions stay in range
        char nm[64];
        snprintf(nm, 64, "scatter atomic >>%d", shift);
        T(nm, [&] { k_scatter_atomic<<<G, B>>>(e, rows, cols, shift, cur, sc); }, 24.0 * e);
        snprintf(nm, 64, "scatter warp-agg >>%d", shift);
        T(nm, [&] { k_scatter_wagg<<<G, B>>>(e, rows, cols, shift, cur, sc); }, 24.0 * e);
    }
    cur_shift = -1;
    T("gather 16B (268 MB table)", [&] { k_gather<<<G, B>>>(e, cols, tab, out); }, 8.0 * e);
    T("gather 8B (134 MB table)", [&] { k_gather8<<<G, B>>>(e, cols, (const double *)tab, out); }, 8.0 * e);
    cudaFuncSetAttribute(k_smem_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
    for (int bits : {10, 16}) {
        char nm[64];
        snprintf(nm, 64, "smem hist %d bits", bits);
        T(nm, [&] { k_smem_hist<<<148, 1024, (4 << bits)>>>(e, rows, scale - bits, 1 << bits, cnt); }, 8.0 * e);
    }
    return 0;
}
