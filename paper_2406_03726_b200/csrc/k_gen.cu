// k_gen.cu -- on-device synthetic graph generators.
//
// The reference draws its SBM with numpy's sequential PCG64 stream and
// geometric gap skipping (sbm.py:52-155); a sequential stream cannot be
// split across 148 SMs without replaying it.  These generators are instead
// COUNTER-BASED: every random word is a pure function of (seed, stream,
// counter) -- the t-th output of a SplitMix64 sequence keyed by
// mix(seed ^ stream * golden) -- so any thread can draw any edge, and the
// C restatement in oracle/gee_gen.c (the reference arm's and the tests'
// input generator) produces the identical arrays bit for bit.  Probability
// thresholds are integers computed once on the host, so no floating-point
// rounding separates the two implementations.
//
//   gee_gen_rmat     R-MAT, 2^scale nodes, quadrant thresholds t1<t2<t3
//                    over a 32-bit uniform per level; optional f32 weights
//                    1 - u24 * 2^-24 in (0, 1]
//   gee_gen_chunglu  endpoint pairs by inverse CDF (binary search of a
//                    host-built f64 CDF table, searchsorted side='right'),
//                    optional f64 weights 1 - u53 * 2^-53 in (0, 1]
//   gee_gen_pairs    G(n,m) candidates: key lo*n + hi of a uniform pair,
//                    -1 for a self pair (the caller keeps first occurrences)
//   gee_gen_sbm_*    SBM pair sweep: pair (i, j), i < j, is an edge when
//                    u32(i*n + j) < thr[label_i == label_j]; row-major
//                    output (count pass, caller scan, fill pass)
#include "gee_common.cuh"

namespace gee {

namespace {

constexpr unsigned long long kGolden = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// t-th word of the stream keyed `key` (= mix64(seed ^ stream * golden))
__device__ __forceinline__ unsigned long long draw(unsigned long long key, unsigned long long t) {
    return mix64(key + (t + 1) * kGolden);
}

__device__ __forceinline__ unsigned mulhi(unsigned u, unsigned n) {
    return (unsigned)(((unsigned long long)u * n) >> 32);
}

__global__ void __launch_bounds__(256) k_gen_rmat(unsigned long long key, unsigned long long wkey, int scale,
                                                  int64_t e, unsigned t1, unsigned t2, unsigned t3, int64_t *rows,
                                                  int64_t *cols, float *w) {
    const int words = (scale + 1) / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        long long r = 0, c = 0;
        for (int h = 0; h < words; ++h) {
            const unsigned long long x = draw(key, (unsigned long long)i * 16 + h);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                if (2 * h + half < scale) {
                    const unsigned u = half ? (unsigned)(x >> 32) : (unsigned)x;
                    const int rb = u >= t2;
                    const int cb = (u >= t1 && u < t2) || u >= t3;
                    r = 2 * r + rb;
                    c = 2 * c + cb;
                }
            }
        }
        rows[i] = r;
        cols[i] = c;
        if (w) {
            const unsigned u24 = (unsigned)(draw(wkey, (unsigned long long)i) >> 40);
            w[i] = 1.0f - (float)u24 * 0x1p-24f;  // exact: u24 < 2^24
        }
    }
}

__device__ __forceinline__ int64_t cdf_pick(const double *cdf, int64_t n, double u) {
    // searchsorted(cdf, u, side='right'): number of entries <= u, clipped to n-1
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cdf[mid] <= u) lo = mid + 1;
        else hi = mid;
    }
    return lo < n ? lo : n - 1;
}

__global__ void __launch_bounds__(256) k_gen_chunglu(unsigned long long rkey, unsigned long long ckey,
                                                     unsigned long long wkey, const double *__restrict__ cdf,
                                                     int64_t n, int64_t e, int64_t *rows, int64_t *cols,
                                                     double *w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const double ur = (double)(draw(rkey, (unsigned long long)i) >> 11) * 0x1p-53;
        const double uc = (double)(draw(ckey, (unsigned long long)i) >> 11) * 0x1p-53;
        rows[i] = cdf_pick(cdf, n, ur);
        cols[i] = cdf_pick(cdf, n, uc);
        if (w) w[i] = 1.0 - (double)(draw(wkey, (unsigned long long)i) >> 11) * 0x1p-53;
    }
}

__global__ void __launch_bounds__(256) k_gen_pairs(unsigned long long key, int64_t t0, int64_t count, unsigned n,
                                                   int64_t *keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = draw(key, (unsigned long long)(t0 + i));
        const unsigned a = mulhi((unsigned)x, n), b = mulhi((unsigned)(x >> 32), n);
        keys[i] = a == b ? -1 : (a < b ? (int64_t)a * n + b : (int64_t)b * n + a);
    }
}

// one warp per row i: pairs (i, j), j in (i, n)
template <bool FILL>
__global__ void __launch_bounds__(256) k_gen_sbm(unsigned long long key, int64_t n, const int64_t *__restrict__ lab,
                                                 unsigned thr_in, unsigned thr_out, int64_t *cnt,
                                                 const int64_t *__restrict__ off, int64_t *rows, int64_t *cols) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t li = lab[i];
        int64_t pos = FILL ? off[i] : 0;
        for (int64_t j0 = i + 1; j0 < n; j0 += 32) {
            const int64_t j = j0 + lane;
            bool hit = false;
            if (j < n) {
                const unsigned u = (unsigned)(draw(key, (unsigned long long)(i * n + j)) >> 32);
                hit = u < (lab[j] == li ? thr_in : thr_out);
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (FILL && hit) {
                const int64_t p = pos + __popc(m & lanemask_lt());
                rows[p] = i;
                cols[p] = j;
            }
            pos += __popc(m);
        }
        if (!FILL && lane == 0) cnt[i] = pos;
    }
}

}  // namespace

}  // namespace gee

using namespace gee;

extern "C" {

int gee_gen_rmat(uint64_t key, uint64_t wkey, int scale, int64_t n_edges, uint32_t t1, uint32_t t2, uint32_t t3,
                 int64_t *rows, int64_t *cols, float *w, void *stream) {
    if (scale < 1 || scale > 31 || n_edges < 0 || !(t1 <= t2 && t2 <= t3)) return GEE_E_ARG;
    if (n_edges && (!rows || !cols)) return GEE_E_ARG;
    if (!n_edges) return GEE_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_gen_rmat<<<grid_for(n_edges, 256, 16), 256, 0, st>>>(key, wkey, scale, n_edges, t1, t2, t3, rows, cols, w);
    GEE_CHECK_LAUNCH("k_gen_rmat");
    return GEE_OK;
}

int gee_gen_chunglu(uint64_t rkey, uint64_t ckey, uint64_t wkey, const double *cdf, int64_t n_nodes,
                    int64_t n_edges, int64_t *rows, int64_t *cols, double *w, void *stream) {
    if (n_nodes < 1 || n_edges < 0 || !cdf) return GEE_E_ARG;
    if (n_edges && (!rows || !cols)) return GEE_E_ARG;
    if (!n_edges) return GEE_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_gen_chunglu<<<grid_for(n_edges, 256, 16), 256, 0, st>>>(rkey, ckey, wkey, cdf, n_nodes, n_edges, rows, cols,
                                                              w);
    GEE_CHECK_LAUNCH("k_gen_chunglu");
    return GEE_OK;
}

int gee_gen_pairs(uint64_t key, int64_t t0, int64_t count, int64_t n_nodes, int64_t *keys, void *stream) {
    if (n_nodes < 1 || n_nodes > 0xffffffffll || count < 0 || t0 < 0 || (count && !keys)) return GEE_E_ARG;
    if (!count) return GEE_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_gen_pairs<<<grid_for(count, 256, 16), 256, 0, st>>>(key, t0, count, (unsigned)n_nodes, keys);
    GEE_CHECK_LAUNCH("k_gen_pairs");
    return GEE_OK;
}

int gee_gen_sbm_count(uint64_t key, int64_t n_nodes, const int64_t *labels, uint32_t thr_in, uint32_t thr_out,
                      int64_t *counts, void *stream) {
    if (n_nodes < 1 || n_nodes > (1ll << 31) || !labels || !counts) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    k_gen_sbm<false><<<grid_for(n_nodes * 32, 256, 16), 256, 0, st>>>(key, n_nodes, labels, thr_in, thr_out,
                                                                       counts, nullptr, nullptr, nullptr);
    GEE_CHECK_LAUNCH("k_gen_sbm_count");
    return GEE_OK;
}

int gee_gen_sbm_fill(uint64_t key, int64_t n_nodes, const int64_t *labels, uint32_t thr_in, uint32_t thr_out,
                     const int64_t *offsets, int64_t *rows, int64_t *cols, void *stream) {
    if (n_nodes < 1 || n_nodes > (1ll << 31) || !labels || !offsets || !rows || !cols) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    k_gen_sbm<true><<<grid_for(n_nodes * 32, 256, 16), 256, 0, st>>>(key, n_nodes, labels, thr_in, thr_out,
                                                                      nullptr, offsets, rows, cols);
    GEE_CHECK_LAUNCH("k_gen_sbm_fill");
    return GEE_OK;
}

}  // extern "C"
