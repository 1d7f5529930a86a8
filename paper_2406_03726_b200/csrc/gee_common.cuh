// gee_common.cuh -- helpers shared by the sm_100a GEE kernels.
#pragma once

#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include <atomic>
#include <cassert>

// Device-side bounds assertions, compiled in by `make CHECKED=1` (the
// sanitizer substitute: compute-sanitizer is closed on the GPU pool).
#ifdef GEE_CHECKED
#define GEE_DASSERT(c) assert(c)
#else
#define GEE_DASSERT(c) ((void)0)
#endif

#include "gee.h"

namespace gee {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs; refined at run time via props

// ---- host-side bookkeeping -------------------------------------------------
uint64_t &launch_counter();
int cuda_status(cudaError_t e);
int num_sms();
// bench profiling: when enabled, record an event after each launch
void profile_mark(const char *name, cudaStream_t st);

// "Done once per device" flag.  Function attributes (e.g. the dynamic
// shared-memory limit) belong to each device's context, so a process-wide
// bool would skip them for a second GPU; racing threads may both set the
// attribute, which is harmless.
struct PerDevice {
    std::atomic<unsigned long long> bits{0};
    static int dev() {
        int d = 0;
        if (cudaGetDevice(&d) != cudaSuccess) d = 0;
        return d & 63;
    }
    bool done() const { return (bits.load(std::memory_order_acquire) >> dev()) & 1ull; }
    void mark() { bits.fetch_or(1ull << dev(), std::memory_order_release); }
};

// Every launch site uses a stream variable named `st`.
#define GEE_CHECK_LAUNCH(name)                                  \
    do {                                                        \
        ++::gee::launch_counter();                              \
        cudaError_t _e = cudaGetLastError();                    \
        if (_e != cudaSuccess) return ::gee::cuda_status(_e);   \
        ::gee::profile_mark(name, st);                          \
    } while (0)

#define GEE_CHECK_CUDA(call)                                    \
    do {                                                        \
        cudaError_t _e = (call);                                \
        if (_e != cudaSuccess) return ::gee::cuda_status(_e);   \
    } while (0)

// Bump allocator over a caller-provided workspace.  With base == nullptr it
// only measures (the *_workspace size queries run the same code).
struct Carver {
    char *base;
    size_t off;
    explicit Carver(void *b) : base(static_cast<char *>(b)), off(0) {}
    template <class T>
    T *take(size_t n) {
        off = (off + 255) & ~size_t(255);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += n * sizeof(T);
        return p;
    }
    size_t bytes() const { return (off + 255) & ~size_t(255); }
};

inline unsigned grid_for(int64_t n, int threads, int per_sm = 8) {
    int64_t b = (n + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (unsigned)b;
}

// ---- device helpers --------------------------------------------------------
__device__ __forceinline__ void raise_err(int32_t *err, int bits) {
    if (err) atomicOr(err, bits);
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ int warp_min(int x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

__device__ __forceinline__ unsigned warp_sum_u(unsigned x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Exponent of the least significant set bit of a finite nonzero double.
__device__ __forceinline__ int lowbit_exp(double x) {
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    int e = (int)((b >> 52) & 0x7ff);
    unsigned long long m = b & ((1ull << 52) - 1);
    if (e == 0) return -1074 + (__ffsll((long long)m) - 1);
    m |= 1ull << 52;
    return e - 1075 + (__ffsll((long long)m) - 1);
}

// Exactness certificate: if every addend is a multiple of 2^mlow and
// sum|x| < 2^(mlow+52) (one bit of slack over the 53-bit significand, which
// also absorbs the rounding of sabs itself), every partial sum in ANY order
// is exactly representable, so any summation order equals the reference's
// sequential left fold bit for bit.
struct Cert {
    int mlow;
    double sabs;
    __device__ __forceinline__ Cert() : mlow(INT_MAX), sabs(0.0) {}
    __device__ __forceinline__ void add(double x) {
        if (x != 0.0) {
            mlow = min(mlow, lowbit_exp(x));
            sabs += fabs(x);
        }
    }
};

__device__ __forceinline__ bool cert_ok(int mlow, double sabs) {
    if (mlow == INT_MAX) return true;
    if (!(sabs < 1.0e300)) return false;
    if (mlow + 52 > 1000) return false;
    return sabs < ldexp(1.0, mlow + 52);
}

// Block-wide helpers (blockDim.x multiple of 32, <= 1024).  `red` must hold
// 33 slots of the type and is reused across calls after a __syncthreads().
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned *red,
                                                         unsigned *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned w = lane < nw ? red[lane] : 0u;
        unsigned wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) red[lane] = wi - w;
        if (lane == nw - 1) red[32] = wi;
    }
    __syncthreads();
    unsigned res = red[wid] + incl - v;
    if (total) *total = red[32];
    __syncthreads();
    return res;
}

__device__ __forceinline__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < nw ? red[lane] : 0.0;
        r = warp_sum(r);
        if (lane == 0) red[0] = r;
    }
    __syncthreads();
    r = red[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ int block_min(int v, int *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    v = warp_min(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int r = lane < nw ? red[lane] : INT_MAX;
        r = warp_min(r);
        if (lane == 0) red[0] = r;
    }
    __syncthreads();
    int r = red[0];
    __syncthreads();
    return r;
}

// 1/sqrt(d) exactly as numpy computes it (IEEE sqrt, IEEE division;
// sparse.py:213-215), 0 for d == 0; d < 0 is an error.
__device__ __forceinline__ double laplacian_scale(double d, int32_t *err) {
    if (d < 0.0) {
        raise_err(err, GEE_ERR_NEG_DEGREE);
        return 0.0;
    }
    return d > 0.0 ? __ddiv_rn(1.0, __dsqrt_rn(d)) : 0.0;
}

}  // namespace gee
