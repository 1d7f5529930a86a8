// k_scan.cu -- exclusive prefix sum of uint32 counts into int64 offsets
// (out[0] = 0, out[n] = total).  Three coalesced passes over the counts:
// per-tile reduce, one-CTA scan of the tile sums, per-tile scan + offset.
#include "gee_common.cuh"

namespace gee {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned long long block_exclusive_scan_u64(
    unsigned long long v, unsigned long long *red, unsigned long long *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned long long w = lane < nw ? red[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) red[lane] = wi - w;
        if (lane == nw - 1) red[32] = wi;
    }
    __syncthreads();
    unsigned long long res = red[wid] + incl - v;
    if (total) *total = red[32];
    __syncthreads();
    return res;
}

__global__ void k_scan_reduce(const unsigned *__restrict__ in, int64_t n,
                              unsigned long long *__restrict__ bsum) {
    __shared__ unsigned long long red[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + (int64_t)j * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    unsigned long long tot;
    block_exclusive_scan_u64(s, red, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// in-place exclusive scan of nb tile sums by one CTA; bsum[nb] = total
__global__ void k_scan_bsums(unsigned long long *bsum, int64_t nb) {
    __shared__ unsigned long long red[33];
    unsigned long long carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        int64_t i = b0 + threadIdx.x;
        unsigned long long v = i < nb ? bsum[i] : 0ull;
        unsigned long long tot;
        unsigned long long ex = block_exclusive_scan_u64(v, red, &tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void k_scan_down(const unsigned *__restrict__ in, int64_t n,
                            const unsigned long long *__restrict__ bsum, int64_t *__restrict__ out) {
    __shared__ unsigned long long red[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    unsigned v[kScanItems];
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        v[j] = i < n ? in[i] : 0u;
        s += v[j];
    }
    unsigned long long ex = block_exclusive_scan_u64(s, red, nullptr) + bsum[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = base + j;
        if (i < n) out[i] = (int64_t)ex;
        ex += v[j];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        int64_t nb = gridDim.x;
        out[n] = (int64_t)bsum[nb];
    }
}

size_t scan_workspace(int64_t n) {
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb < 1) nb = 1;
    return (size_t)(nb + 1) * sizeof(unsigned long long) + 256;
}

// out[0..n] = exclusive scan of in[0..n); ws from scan_workspace(n)
int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st) {
    int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb < 1) nb = 1;
    unsigned long long *bsum = static_cast<unsigned long long *>(ws);
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum);
    GEE_CHECK_LAUNCH("k_scan_reduce");
    k_scan_bsums<<<1, 1024, 0, st>>>(bsum, nb);
    GEE_CHECK_LAUNCH("k_scan_bsums");
    k_scan_down<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum, out);
    GEE_CHECK_LAUNCH("k_scan_down");
    return GEE_OK;
}

}  // namespace gee
