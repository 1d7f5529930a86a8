// k_label.cu -- K1: class histogram n_k and the per-class weight 1/n_k.
//
// Replaces LabelVector.class_counts (embedding.py:68-71) and the value
// column of build_weight_matrix (embedding.py:92-107).  W itself is never
// materialised: gee_embed reads y32 + inv_nk instead of W's CSR.
#include "gee_common.cuh"

namespace gee {

constexpr int kHistSmemMax = 8192;  // classes privatised in shared memory

// labels int64 -> int32 (-1 = unlabeled), validated, histogrammed.  Small K:
// per-CTA shared histogram with warp-aggregated updates (__match_any_sync
// collapses equal labels so a hot class costs one shared atomic per warp).
__global__ void k_label_hist(const int64_t *__restrict__ labels, int64_t n, int k,
                             int32_t *__restrict__ y32, unsigned long long *__restrict__ counts,
                             int32_t *err) {
    extern __shared__ unsigned sh_hist[];
    const bool priv = k <= kHistSmemMax;
    if (priv)
        for (int c = threadIdx.x; c < k; c += blockDim.x) sh_hist[c] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) & ~int64_t(31);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        int lab = -1;
        bool valid = false;
        if (i < n) {
            int64_t v = labels[i];
            if (v < -1 || v >= k) {
                raise_err(err, GEE_ERR_LABEL);
                v = -1;
            }
            lab = (int)v;
            y32[i] = lab;
            valid = lab >= 0;
        }
        // every lane of the warp reaches here (n_round is a multiple of 32)
        unsigned key = valid ? (unsigned)lab : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, key);
        int leader = __ffs(peers) - 1;
        if (valid && (threadIdx.x & 31) == leader) {
            unsigned cnt = __popc(peers);
            if (priv)
                atomicAdd(&sh_hist[lab], cnt);
            else
                atomicAdd(&counts[lab], (unsigned long long)cnt);
        }
    }
    __syncthreads();
    if (priv)
        for (int c = threadIdx.x; c < k; c += blockDim.x)
            if (sh_hist[c]) atomicAdd(&counts[c], (unsigned long long)sh_hist[c]);
}

// inv_nk[c] = 1.0 / n_c as build_weight_matrix computes it (f64 division of
// 1.0 by the count, embedding.py:106); empty classes are never read.
__global__ void k_inv_counts(const unsigned long long *__restrict__ counts, int k,
                             double *__restrict__ inv_nk) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < k) {
        unsigned long long n = counts[c];
        inv_nk[c] = n ? __ddiv_rn(1.0, (double)n) : 0.0;
    }
}

// Small label vectors: one CTA does histogram, counts and 1/n_k in one launch
// (no memset, no second kernel).
__global__ void __launch_bounds__(1024) k_label_small(const int64_t *__restrict__ labels, int64_t n, int k,
                                                      int32_t *__restrict__ y32, long long *__restrict__ counts,
                                                      double *__restrict__ inv_nk, int32_t *err) {
    extern __shared__ unsigned sh_hist[];
    for (int c = threadIdx.x; c < k; c += blockDim.x) sh_hist[c] = 0;
    __syncthreads();
    const int64_t n_round = (n + 31) & ~int64_t(31);
    for (int64_t i = threadIdx.x; i < n_round; i += blockDim.x) {
        int lab = -1;
        bool valid = false;
        if (i < n) {
            int64_t v = labels[i];
            if (v < -1 || v >= k) {
                raise_err(err, GEE_ERR_LABEL);
                v = -1;
            }
            lab = (int)v;
            y32[i] = lab;
            valid = lab >= 0;
        }
        unsigned key = valid ? (unsigned)lab : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, key);
        if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh_hist[lab], __popc(peers));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const unsigned m = sh_hist[c];
        counts[c] = (long long)m;
        inv_nk[c] = m ? __ddiv_rn(1.0, (double)m) : 0.0;
    }
}

constexpr int64_t kLabelSmall = 1 << 18;
constexpr int kLabelWarpHistK = 384;  // 32 warp histograms of <= 384 classes: <= 48 KB
constexpr int kLabelMaxBlocks = 1024;

// Pipeline variant: each CTA histograms a contiguous slice into its own row
// of `partial` (no atomics on the result, no memset); the last CTA to finish
// sums the rows into counts, computes 1/n_k and re-arms `done` for the next
// launch or graph replay.
__global__ void __launch_bounds__(1024) k_label_multi(const int64_t *__restrict__ labels, int64_t n, int k,
                                                      int64_t per_block, int32_t *__restrict__ y32,
                                                      unsigned *__restrict__ partial, long long *__restrict__ counts,
                                                      double *__restrict__ inv_nk, unsigned *__restrict__ done,
                                                      int32_t *err) {
    extern __shared__ unsigned sh_hist[];
    __shared__ bool last;
    // few classes: one sub-histogram per warp and plain shared atomics (no
    // __match_any_sync); more: one histogram with warp-aggregated updates
    const bool per_warp = k <= kLabelWarpHistK;
    const int nh = per_warp ? (int)(blockDim.x >> 5) : 1;
    unsigned *mine = sh_hist + (per_warp ? (threadIdx.x >> 5) * k : 0);
    for (int c = threadIdx.x; c < nh * k; c += blockDim.x) sh_hist[c] = 0;
    __syncthreads();
    const int64_t i0 = (int64_t)blockIdx.x * per_block;
    const int64_t i1 = min(n, i0 + per_block);
    for (int64_t b = i0; b < i1; b += 4 * (int64_t)blockDim.x) {
        int64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = b + u * (int64_t)blockDim.x + threadIdx.x;
            v[u] = i < i1 ? labels[i] : -2;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = b + u * (int64_t)blockDim.x + threadIdx.x;
            int lab = -1;
            if (i < i1) {
                int64_t x = v[u];
                if (x < -1 || x >= k) {
                    raise_err(err, GEE_ERR_LABEL);
                    x = -1;
                }
                lab = (int)x;
                y32[i] = lab;
            }
            if (per_warp) {
                if (lab >= 0) atomicAdd(mine + lab, 1u);
            } else {
                const unsigned key = lab >= 0 ? (unsigned)lab : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, key);
                if (lab >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&sh_hist[lab], __popc(peers));
            }
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        unsigned t = 0;
        for (int h = 0; h < nh; ++h) t += sh_hist[h * k + c];
        partial[(size_t)blockIdx.x * k + c] = t;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last block sums the per-block rows with all of its threads: class c's
    // blocks are split over blockDim / k slices (one thread per class did 1024
    // dependent L2 round trips at configs[3]) and the slices meet in counts[c]
    const int nsl = (int)blockDim.x / k;
    if (nsl < 2) {  // more classes than half the block: a thread per class (configs[4]: 0.06 ms; sliced 0.13)
        for (int c = threadIdx.x; c < k; c += blockDim.x) {
            unsigned long long m = 0;
            for (unsigned b = 0; b < gridDim.x; ++b) m += __ldcg(partial + (size_t)b * k + c);
            counts[c] = (long long)m;
            inv_nk[c] = m ? __ddiv_rn(1.0, (double)m) : 0.0;
        }
        if (threadIdx.x == 0) *done = 0;
        return;
    }
    for (int c = threadIdx.x; c < k; c += blockDim.x) counts[c] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < nsl * k; t += blockDim.x) {
        const int c = t % k, sl = t / k;
        unsigned long long m = 0;
        for (unsigned b = sl; b < gridDim.x; b += nsl) m += __ldcg(partial + (size_t)b * k + c);
        if (m) atomicAdd(reinterpret_cast<unsigned long long *>(counts) + c, m);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const unsigned long long m = (unsigned long long)__ldcg(counts + c);  // the atomics' result, from L2
        inv_nk[c] = m ? __ddiv_rn(1.0, (double)m) : 0.0;
    }
    if (threadIdx.x == 0) *done = 0;
}

size_t label_partial_words(int64_t n, int k) {
    int64_t per = n > 2048 * (int64_t)kLabelMaxBlocks ? (n + kLabelMaxBlocks - 1) / kLabelMaxBlocks : 2048;
    int64_t nb = (n + per - 1) / per;
    if (nb < 1) nb = 1;
    return (size_t)nb * (size_t)k;
}

// labels -> y32, counts, 1/n_k in one launch; `done` must be zero on the
// first call (the kernel leaves it zero).  Falls back to label_hist for K
// beyond the shared-memory histogram.
int label_hist_pipeline(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts, double *inv_nk,
                        unsigned *partial, unsigned *done, int32_t *err, cudaStream_t st);

int label_hist(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts,
               double *inv_nk, int32_t *err, cudaStream_t st) {
    if (n <= kLabelSmall && k <= kHistSmemMax) {
        k_label_small<<<1, 1024, sizeof(unsigned) * (size_t)k, st>>>(labels, n, k, y32,
                                                                    reinterpret_cast<long long *>(counts),
                                                                    inv_nk, err);
        GEE_CHECK_LAUNCH("k_label_hist");
        return GEE_OK;
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (size_t)k, st));
    if (n > 0) {
        const int threads = 512;
        unsigned grid = grid_for(n, threads, 2);
        size_t smem = k <= kHistSmemMax ? sizeof(unsigned) * (size_t)k : 0;
        k_label_hist<<<grid, threads, smem, st>>>(labels, n, k, y32,
                                                  reinterpret_cast<unsigned long long *>(counts),
                                                  err);
        GEE_CHECK_LAUNCH("k_label_hist");
    }
    k_inv_counts<<<(k + 255) / 256, 256, 0, st>>>(
        reinterpret_cast<const unsigned long long *>(counts), k, inv_nk);
    GEE_CHECK_LAUNCH("k_inv_counts");
    return GEE_OK;
}

int inv_counts(const int64_t *counts, int32_t k, double *inv_nk, cudaStream_t st) {
    k_inv_counts<<<(k + 255) / 256, 256, 0, st>>>(reinterpret_cast<const unsigned long long *>(counts), k, inv_nk);
    GEE_CHECK_LAUNCH("k_inv_counts");
    return GEE_OK;
}

// ---- build_weight_matrix (embedding.py:92-107) ------------------------------
// W materialised as an N x K CSR: row j holds 1/n_{Y_j} at column Y_j,
// unlabeled rows are empty.  index_pointers = exclusive scan of the labeled
// flags, then one thread per node writes its entry (values are inv_nk, i.e.
// 1.0 / counts, the reference's `1.0 / counts[cols]`).
int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st);
size_t scan_workspace(int64_t n);

__global__ void k_wm_flags(const int32_t *__restrict__ y32, int64_t n, unsigned *__restrict__ flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = y32[i] >= 0 ? 1u : 0u;
}

__global__ void k_wm_fill(const int32_t *__restrict__ y32, int64_t n, const double *__restrict__ inv_nk,
                          const int64_t *__restrict__ ptr, int32_t *__restrict__ cols, double *__restrict__ vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t y = y32[i];
        if (y >= 0) {
            const int64_t p = ptr[i];
            cols[p] = y;
            vals[p] = inv_nk[y];
        }
    }
}

size_t weight_matrix_workspace(int64_t n) { return (((size_t)n * 4 + 255) & ~(size_t)255) + scan_workspace(n); }

int weight_matrix(const int32_t *y32, int64_t n, const double *inv_nk, int64_t *ptr, int32_t *cols, double *vals,
                  void *ws, cudaStream_t st) {
    unsigned *flag = static_cast<unsigned *>(ws);
    void *sws = static_cast<unsigned char *>(ws) + (((size_t)n * 4 + 255) & ~(size_t)255);
    if (n == 0) {
        GEE_CHECK_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int64_t), st));
        return GEE_OK;
    }
    const unsigned grid = grid_for(n, 256, 4);
    k_wm_flags<<<grid, 256, 0, st>>>(y32, n, flag);
    GEE_CHECK_LAUNCH("k_wm_flags");
    const int rc = exclusive_scan_u32(flag, n, ptr, sws, st);
    if (rc != GEE_OK) return rc;
    k_wm_fill<<<grid, 256, 0, st>>>(y32, n, inv_nk, ptr, cols, vals);
    GEE_CHECK_LAUNCH("k_wm_fill");
    return GEE_OK;
}

int label_hist_pipeline(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts, double *inv_nk,
                        unsigned *partial, unsigned *done, int32_t *err, cudaStream_t st) {
    if (k > kHistSmemMax || n <= 0) return label_hist(labels, n, k, y32, counts, inv_nk, err, st);
    const int64_t per = n > 2048 * (int64_t)kLabelMaxBlocks ? (n + kLabelMaxBlocks - 1) / kLabelMaxBlocks : 2048;
    const unsigned nb = (unsigned)((n + per - 1) / per);
    const size_t smem = sizeof(unsigned) * (size_t)k * (k <= kLabelWarpHistK ? 32 : 1);
    k_label_multi<<<nb, 1024, smem, st>>>(labels, n, k, per, y32, partial,
                                                                 reinterpret_cast<long long *>(counts), inv_nk,
                                                                 done, err);
    GEE_CHECK_LAUNCH("k_label_hist");
    return GEE_OK;
}

}  // namespace gee
