// k_sparse.cu -- the reference's sparse-core seam on the device, for callers
// that hand in a CSR instead of an edge list:
//   gee_degree               degree_vector (sparse.py:193-196), of A or A+I
//   gee_add_identity         _kernels.add_identity_kernel (_kernels.py:169-198)
//   gee_laplacian_normalize  laplacian_normalize (sparse.py:199-226)
//   gee_validate_edges       EdgeList.__post_init__ checks (graph_io.py:58-72)
// All bit-exact with the reference.
#include "gee_common.cuh"

namespace gee {

int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st);
size_t scan_workspace(int64_t n);

// Degree of row r of A (or A+I): the reference folds the row's stored values
// left to right (np.bincount, sparse.py:196).  Three tiers, each exact:
//  * a thread per row of <= kDegShort entries folds it itself, in order;
//  * a warp per longer row: when the exactness certificate holds (every
//    addend a multiple of 2^m, sum|x| < 2^(m+52)) any order is bitwise equal,
//    so the warp reduces in parallel; otherwise lane 0 replays the fold;
//  * rows over kDegHub entries are listed and taken by a whole CTA each
//    (k_degree_hub) -- a hub row would otherwise hold one warp for the kernel.
constexpr int kDegShort = 16;
constexpr int64_t kDegHub = 4096;
constexpr int kDegU = 4;  // entries per lane loaded before any is used

__device__ __forceinline__ void degree_store(double *deg, double *scale, int64_t r, double d, int32_t *err) {
    deg[r] = d;
    if (scale) scale[r] = laplacian_scale(d, err);
}

// the exact sequential fold of row r, entries [s, e), the A+I diagonal
// merged into a stored (r, r) or inserted at its sorted position
__device__ __forceinline__ double fold_row(const int32_t *col, const double *val, int64_t r, int64_t s, int64_t e,
                                           bool diag) {
    double d = 0.0;
    bool ins = !diag;
    int64_t p = s;
    for (; p + 4 <= e; p += 4) {
        int32_t c4[4];
        double x4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            c4[j] = col[p + j];
            x4[j] = val[p + j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double x = x4[j];
            if (diag && (int64_t)c4[j] == r) {
                x = x + 1.0;
                ins = true;
            } else if (!ins && (int64_t)c4[j] > r) {
                d += 1.0;
                ins = true;
            }
            d += x;
        }
    }
    for (; p < e; ++p) {
        const int64_t c = col[p];
        double x = val[p];
        if (diag && c == r) {
            x = x + 1.0;
            ins = true;
        } else if (!ins && c > r) {
            d += 1.0;
            ins = true;
        }
        d += x;
    }
    if (!ins) d += 1.0;
    return d;
}

// skip_hubs: rows over kDegHub belong to hub CTAs (listed beforehand);
// else, with a hub list, they are appended to it for k_degree_hub
__device__ __forceinline__ void degree_rows(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                            const double *__restrict__ val, int64_t n, unsigned flags,
                                            double *__restrict__ deg, double *__restrict__ scale, int32_t *err,
                                            unsigned *__restrict__ hubs, unsigned *__restrict__ n_hubs,
                                            unsigned *__restrict__ work, bool skip_hubs, int64_t warp,
                                            int64_t nwarps) {
    const int lane = threadIdx.x & 31;
    const bool diag = (flags & GEE_DIAGONAL) != 0;
    // A warp takes 32 rows at a time, rows c, c + nc, c + 2 nc, ... of chunk c
    // (long rows cluster by id in power-law graphs); lanes fold the short
    // ones.  Chunks are grabbed from a counter when there is one, else dealt
    // round robin.
    const int64_t nc = (n + 31) / 32;
    int64_t c = warp;
    for (;;) {
        if (work) {
            unsigned t = 0;
            if (lane == 0) t = atomicAdd(work, 1u);
            c = __shfl_sync(0xffffffffu, t, 0);
        }
        if (c >= nc) break;
        const int64_t r = c + (int64_t)lane * nc;
        const int64_t r0 = c;
        int64_t s = 0, e = 0;
        if (r < n) {
            s = row_ptr[r];
            e = row_ptr[r + 1];
        }
        const int64_t L = e - s;
        if (r < n && L <= kDegShort) degree_store(deg, scale, r, fold_row(col, val, r, s, e, diag), err);
        // with a hub list, rows over kDegHub go to k_degree_hub; without one
        // (gee_degree has no workspace) the warp takes them too
        const bool hub = (hubs || skip_hubs) && L > kDegHub;
        unsigned longer = __ballot_sync(0xffffffffu, r < n && L > kDegShort && !hub);
        if (r < n && hub && !skip_hubs) hubs[atomicAdd(n_hubs, 1u)] = (unsigned)r;
        while (longer) {
            const int src = __ffs(longer) - 1;
            longer &= longer - 1;
            const int64_t rr = r0 + (int64_t)src * nc;
            const int64_t ss = __shfl_sync(0xffffffffu, s, src), ee = __shfl_sync(0xffffffffu, e, src);
            Cert ce;
            double psum = 0.0;
            bool placed = false;
            for (int64_t p0 = ss + lane; p0 < ee; p0 += 32 * kDegU) {
                double xs[kDegU];
                int32_t cs[kDegU];
#pragma unroll
                for (int j = 0; j < kDegU; ++j) {
                    const int64_t p = p0 + 32 * j;
                    xs[j] = p < ee ? val[p] : 0.0;
                    cs[j] = (diag && p < ee) ? col[p] : -1;
                }
#pragma unroll
                for (int j = 0; j < kDegU; ++j) {
                    double x = xs[j];
                    if (diag && (int64_t)cs[j] == rr) {
                        x = x + 1.0;
                        placed = true;
                    }
                    ce.add(x);  // zeros (padding included) change nothing
                    psum += x;
                }
            }
            const bool insert = diag && !__any_sync(0xffffffffu, placed);
            int mlow = warp_min(ce.mlow);
            const double sabs = warp_sum(ce.sabs) + (insert ? 1.0 : 0.0);
            if (insert) mlow = min(mlow, 0);
            const bool ok = cert_ok(mlow, sabs);
            const double tot = warp_sum(psum);
            if (lane == 0) degree_store(deg, scale, rr, ok ? tot + (insert ? 1.0 : 0.0) : fold_row(col, val, rr, ss, ee, diag), err);
        }
        if (!work) c += nwarps;
    }
}

__global__ void k_degree(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                         const double *__restrict__ val, int64_t n, unsigned flags,
                         double *__restrict__ deg, double *__restrict__ scale, int32_t *err,
                         const unsigned *guard, unsigned *__restrict__ hubs, unsigned *__restrict__ n_hubs,
                         unsigned *__restrict__ work) {
    if (guard && *guard == 0) return;  // device-side skip (unit-weight graphs use k_degree_stream)
    degree_rows(row_ptr, col, val, n, flags, deg, scale, err, hubs, n_hubs, work, false,
                ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, ((int64_t)gridDim.x * blockDim.x) >> 5);
}

// one CTA per hub row: certificate by block reductions, else thread 0 folds
// while the other warps stage the next 2048 entries in shared memory
constexpr int kHubThreads = 512, kHubStage = 2048;
__device__ __forceinline__ double fold_plain(const double *x, int lo, int hi, double d) {
    int i = lo;
    for (; i + 8 <= hi; i += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = x[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) d += v[j];
    }
    for (; i < hi; ++i) d += x[i];
    return d;
}

__device__ __forceinline__ void degree_hubs(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                            const double *__restrict__ val, unsigned flags,
                                            double *__restrict__ deg, double *__restrict__ scale, int32_t *err,
                                            const unsigned *__restrict__ hubs, const unsigned *__restrict__ n_hubs,
                                            unsigned first, unsigned step) {
    __shared__ double sv[2][kHubStage];
    __shared__ double dred[33];
    __shared__ int ired[33];
    const int tid = threadIdx.x, nt = blockDim.x;
    const bool diag = (flags & GEE_DIAGONAL) != 0;
    for (unsigned h = first; h < *n_hubs; h += step) {
        const int64_t r = hubs[h];
        const int64_t s = row_ptr[r], e = row_ptr[r + 1];
        const int64_t L = e - s;
        Cert ce;
        double psum = 0.0;
        int placed = 0;
        int kfirst = INT_MAX;  // first position whose column is >= r (where A+I's diagonal goes)
        for (int64_t p0 = s + tid; p0 < e; p0 += (int64_t)nt * kDegU) {
            double xs[kDegU];
            int32_t cs[kDegU];
#pragma unroll
            for (int j = 0; j < kDegU; ++j) {
                const int64_t p = p0 + (int64_t)nt * j;
                xs[j] = p < e ? val[p] : 0.0;
                cs[j] = (diag && p < e) ? col[p] : -1;
            }
#pragma unroll
            for (int j = 0; j < kDegU; ++j) {
                double x = xs[j];
                if (diag && (int64_t)cs[j] >= r) kfirst = min(kfirst, (int)(p0 + (int64_t)nt * j - s));
                if (diag && (int64_t)cs[j] == r) {
                    x = x + 1.0;
                    placed = 1;
                }
                ce.add(x);
                psum += x;
            }
        }
        placed = __syncthreads_or(placed);
        const bool insert = diag && !placed;
        int mlow = block_min(ce.mlow, ired);
        const double sabs = block_sum(ce.sabs, dred) + (insert ? 1.0 : 0.0);
        if (insert) mlow = min(mlow, 0);
        if (cert_ok(mlow, sabs)) {
            const double d = block_sum(psum, dred) + (insert ? 1.0 : 0.0);
            if (tid == 0) degree_store(deg, scale, r, d, err);
            continue;
        }
        // The exact fold: plain left-to-right adds with the diagonal applied at
        // position kfirst (merged into the stored value, or a 1.0 inserted
        // before it), so thread 0's loop is a pure add chain over shared
        // memory while warps 1.. stage the next kHubStage values.
        const int64_t kd = diag ? min((int64_t)block_min(kfirst, ired), L) : L + 1;
        auto stage = [&](int64_t b, int buf, int t0, int tstep) {
            const int nb = (int)(L - b < (int64_t)kHubStage ? L - b : (int64_t)kHubStage);
            for (int i = t0; i < nb; i += tstep) {
                double x = val[s + b + i];
                if (placed && b + i == kd) x = x + 1.0;
                sv[buf][i] = x;
            }
        };
        double d = 0.0;
        stage(0, 0, tid, nt);
        __syncthreads();
        for (int64_t b = 0; b < L; b += kHubStage) {
            const int half = (int)((b / kHubStage) & 1);
            const int nb = (int)(L - b < (int64_t)kHubStage ? L - b : (int64_t)kHubStage);
            if (tid >= 32) {
                if (b + kHubStage < L) stage(b + kHubStage, half ^ 1, tid - 32, nt - 32);
            } else if (tid == 0) {
                if (insert && kd >= b && kd < b + nb) {
                    d = fold_plain(sv[half], 0, (int)(kd - b), d);
                    d += 1.0;
                    d = fold_plain(sv[half], (int)(kd - b), nb, d);
                } else {
                    d = fold_plain(sv[half], 0, nb, d);
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            if (insert && kd >= L) d += 1.0;
            degree_store(deg, scale, r, d, err);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kHubThreads) k_degree_hub(const int64_t *__restrict__ row_ptr,
                                                            const int32_t *__restrict__ col,
                                                            const double *__restrict__ val, unsigned flags,
                                                            double *__restrict__ deg, double *__restrict__ scale,
                                                            int32_t *err, const unsigned *guard,
                                                            const unsigned *__restrict__ hubs,
                                                            const unsigned *__restrict__ n_hubs) {
    if (guard && *guard == 0) return;
    degree_hubs(row_ptr, col, val, flags, deg, scale, err, hubs, n_hubs, blockIdx.x, gridDim.x);
}

// rows over kDegHub entries -> hubs[], count in *n_hubs (warp-aggregated)
__global__ void k_hub_list(const int64_t *__restrict__ row_ptr, int64_t n, const unsigned *guard,
                           unsigned *__restrict__ hubs, unsigned *__restrict__ n_hubs) {
    if (guard && *guard == 0) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) & ~int64_t(31);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_round; r += stride) {
        const bool hub = r < n && row_ptr[r + 1] - row_ptr[r] > kDegHub;
        const unsigned m = __ballot_sync(0xffffffffu, hub);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        unsigned base = 0;
        if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(n_hubs, __popc(m));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (hub) hubs[base + __popc(m & lanemask_lt())] = (unsigned)r;
    }
}

// The hub rows' serial folds overlap the other rows: CTAs [0, hub_ctas) take
// the listed hubs (one CTA per hub, as k_degree_hub), the rest run the
// warp/lane tiers of k_degree over every other row.
__global__ void __launch_bounds__(kHubThreads) k_degree_fused(const int64_t *__restrict__ row_ptr,
                                                              const int32_t *__restrict__ col,
                                                              const double *__restrict__ val, int64_t n,
                                                              unsigned flags, double *__restrict__ deg,
                                                              double *__restrict__ scale, int32_t *err,
                                                              const unsigned *guard, const unsigned *__restrict__ hubs,
                                                              const unsigned *__restrict__ n_hubs,
                                                              unsigned *__restrict__ work, unsigned hub_ctas) {
    if (guard && *guard == 0) return;
    if (blockIdx.x < hub_ctas) {
        degree_hubs(row_ptr, col, val, flags, deg, scale, err, hubs, n_hubs, blockIdx.x, hub_ctas);
        return;
    }
    const int64_t b = blockIdx.x - hub_ctas, nb = gridDim.x - hub_ctas;
    degree_rows(row_ptr, col, val, n, flags, deg, scale, err, nullptr, nullptr, work, true,
                (b * blockDim.x + threadIdx.x) >> 5, (nb * blockDim.x) >> 5);
}

// hub_buf: [1 + nnz / kDegHub] words (count, then row ids) or null
static int launch_degree(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n, unsigned flags,
                         double *deg, double *scale, int32_t *err, const unsigned *guard, unsigned *hub_buf,
                         cudaStream_t st) {
    // hub_buf: [0] hub count, [1] chunk counter, [2..] hub rows
    if (!hub_buf) {
        k_degree<<<grid_for((n + 31) / 32 * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, flags, deg, scale, err,
                                                                       guard, nullptr, nullptr, nullptr);
        GEE_CHECK_LAUNCH("k_degree");
        return GEE_OK;
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(hub_buf, 0, 2 * sizeof(unsigned), st));
    k_hub_list<<<grid_for(n, 256, 8), 256, 0, st>>>(row_ptr, n, guard, hub_buf + 2, hub_buf);
    GEE_CHECK_LAUNCH("k_hub_list");
    const unsigned hub_ctas = (unsigned)num_sms();
    const unsigned rows_ctas = grid_for((n + 31) / 32 * 32, kHubThreads, 4);
    k_degree_fused<<<hub_ctas + rows_ctas, kHubThreads, 0, st>>>(row_ptr, col, val, n, flags, deg, scale, err, guard,
                                                                 hub_buf + 2, hub_buf, hub_buf + 1, hub_ctas);
    GEE_CHECK_LAUNCH("k_degree");
    return GEE_OK;
}

size_t degree_hub_words(int64_t nnz) { return 3 + (size_t)(nnz / kDegHub); }

int degree(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n, unsigned flags,
           double *deg, double *scale, int32_t *err, cudaStream_t st) {
    if (n <= 0) return GEE_OK;
    return launch_degree(row_ptr, col, val, n, flags, deg, scale, err, nullptr, nullptr, st);
}

// degree() that runs only if the device word *guard is nonzero; hub_buf
// (degree_hub_words(nnz) words of workspace) lets a CTA take each hub row
int degree_guarded(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                   unsigned flags, double *deg, double *scale, int32_t *err, const unsigned *guard,
                   unsigned *hub_buf, cudaStream_t st) {
    if (n <= 0) return GEE_OK;
    return launch_degree(row_ptr, col, val, n, flags, deg, scale, err, guard, hub_buf, st);
}

// ---- A + I ------------------------------------------------------------------
// new row length: +1 when no stored diagonal, -1 when v_rr + 1.0 == 0.0
__global__ void k_addid_count(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                              const double *__restrict__ val, int64_t n, unsigned *__restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
        int64_t s = row_ptr[r], e = row_ptr[r + 1];
        // binary search for the first column >= r (columns strictly increase)
        int64_t lo = s, hi = e;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (col[mid] < r) lo = mid + 1; else hi = mid;
        }
        int64_t L = e - s;
        if (lo < e && col[lo] == r)
            cnt[r] = (unsigned)(val[lo] + 1.0 == 0.0 ? L - 1 : L);
        else
            cnt[r] = (unsigned)(L + 1);
    }
}

__global__ void k_addid_fill(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                             const double *__restrict__ val, int64_t n,
                             const int64_t *__restrict__ out_ptr, int32_t *__restrict__ out_col,
                             double *__restrict__ out_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t s = row_ptr[r], e = row_ptr[r + 1], o = out_ptr[r];
        int64_t lo = s, hi = e;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (col[mid] < r) lo = mid + 1; else hi = mid;
        }
        const bool has = lo < e && col[lo] == r;
        const bool drop = has && val[lo] + 1.0 == 0.0;
        const int64_t ip = lo - s;  // insertion / diagonal position within the row
        for (int64_t p = s + lane; p < e; p += 32) {
            int64_t j = p - s;
            double v = val[p];
            if (j < ip) {
                out_col[o + j] = col[p];
                out_val[o + j] = v;
            } else if (j == ip && has) {
                if (!drop) {
                    out_col[o + j] = col[p];
                    out_val[o + j] = v + 1.0;
                }
            } else {
                int64_t d = has ? (drop ? j - 1 : j) : j + 1;
                out_col[o + d] = col[p];
                out_val[o + d] = v;
            }
        }
        if (!has && lane == 0) {
            out_col[o + ip] = (int32_t)r;
            out_val[o + ip] = 1.0;
        }
    }
}

size_t add_identity_workspace(int64_t n) {
    Carver cv(nullptr);
    cv.take<unsigned>((size_t)n + 1);
    cv.take<char>(scan_workspace(n));
    return cv.bytes();
}

int add_identity(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                 int64_t *out_ptr, int32_t *out_col, double *out_val, int64_t *nnz_out, void *ws,
                 size_t ws_bytes, cudaStream_t st) {
    Carver cv(ws);
    unsigned *cnt = cv.take<unsigned>((size_t)n + 1);
    void *sws = cv.take<char>(scan_workspace(n));
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    if (n > 0) {
        k_addid_count<<<grid_for(n, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, cnt);
        GEE_CHECK_LAUNCH("k_addid_count");
    }
    int rc = exclusive_scan_u32(cnt, n, out_ptr, sws, st);
    if (rc) return rc;
    if (n > 0) {
        k_addid_fill<<<grid_for(n * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, out_ptr, out_col,
                                                              out_val);
        GEE_CHECK_LAUNCH("k_addid_fill");
    }
    if (nnz_out)
        GEE_CHECK_CUDA(cudaMemcpyAsync(nnz_out, out_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    return GEE_OK;
}

// ---- D^-1/2 A D^-1/2 --------------------------------------------------------
__global__ void k_scale_from_degree(const double *__restrict__ deg, int64_t n,
                                    double *__restrict__ scale, int32_t *err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
        scale[r] = laplacian_scale(deg[r], err);
}

__device__ __forceinline__ double lap_value(double v, double sr, double sc) {
    return __dmul_rn(__dmul_rn(v, sr), sc);  // (data * scale[row]) * scale[col]
}

__global__ void k_lap_count(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const double *__restrict__ val, int64_t n, const double *__restrict__ scale,
                            unsigned *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t s = row_ptr[r], e = row_ptr[r + 1];
        const double sr = scale[r];
        unsigned c = 0;
        for (int64_t p = s + lane; p < e; p += 32) c += lap_value(val[p], sr, scale[col[p]]) != 0.0;
        c = warp_sum_u(c);
        if (lane == 0) cnt[r] = c;
    }
}

__global__ void k_lap_fill(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const double *__restrict__ val, int64_t n, const double *__restrict__ scale,
                           const int64_t *__restrict__ out_ptr, int32_t *__restrict__ out_col,
                           double *__restrict__ out_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t s = row_ptr[r], e = row_ptr[r + 1];
        const double sr = scale[r];
        int64_t o = out_ptr[r];
        for (int64_t p0 = s; p0 < e; p0 += 32) {
            int64_t p = p0 + lane;
            double v = 0.0;
            int c = 0;
            if (p < e) {
                c = col[p];
                v = lap_value(val[p], sr, scale[c]);
            }
            bool keep = p < e && v != 0.0;
            unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                int64_t d = o + __popc(m & lanemask_lt());
                out_col[d] = c;
                out_val[d] = v;
            }
            o += __popc(m);
        }
    }
}

size_t laplacian_workspace(int64_t n) {
    Carver cv(nullptr);
    cv.take<double>((size_t)n + 1);
    cv.take<unsigned>((size_t)n + 1);
    cv.take<char>(scan_workspace(n));
    return cv.bytes();
}

int laplacian_normalize(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                        const double *deg, int64_t *out_ptr, int32_t *out_col, double *out_val,
                        int64_t *nnz_out, void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    double *scale = cv.take<double>((size_t)n + 1);
    unsigned *cnt = cv.take<unsigned>((size_t)n + 1);
    void *sws = cv.take<char>(scan_workspace(n));
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    if (n > 0) {
        k_scale_from_degree<<<grid_for(n, 256, 8), 256, 0, st>>>(deg, n, scale, err);
        GEE_CHECK_LAUNCH("k_scale_from_degree");
        k_lap_count<<<grid_for(n * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, scale, cnt);
        GEE_CHECK_LAUNCH("k_lap_count");
    }
    int rc = exclusive_scan_u32(cnt, n, out_ptr, sws, st);
    if (rc) return rc;
    if (n > 0) {
        k_lap_fill<<<grid_for(n * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, scale, out_ptr,
                                                            out_col, out_val);
        GEE_CHECK_LAUNCH("k_lap_fill");
    }
    if (nnz_out)
        GEE_CHECK_CUDA(cudaMemcpyAsync(nnz_out, out_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    return GEE_OK;
}

// ---- EdgeList validation -------------------------------------------------------
__global__ void k_validate_edges(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                                 const void *__restrict__ w, int wt, int64_t E, int64_t n,
                                 int32_t *err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int bad = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        int64_t r = rows[e], c = cols[e];
        if (r < 0 || r >= n || c < 0 || c >= n) bad |= GEE_ERR_EDGE_RANGE;
        if (wt == GEE_W_F64) {
            if (!isfinite(static_cast<const double *>(w)[e])) bad |= GEE_ERR_EDGE_WEIGHT;
        } else if (wt == GEE_W_F32) {
            if (!isfinite(static_cast<const float *>(w)[e])) bad |= GEE_ERR_EDGE_WEIGHT;
        }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) raise_err(err, bad);
}

int validate_edges(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E,
                   int64_t n, int32_t *err, cudaStream_t st) {
    if (E <= 0) return GEE_OK;
    k_validate_edges<<<grid_for(E, 256, 8), 256, 0, st>>>(rows, cols, w, wt, E, n, err);
    GEE_CHECK_LAUNCH("k_validate_edges");
    return GEE_OK;
}

}  // namespace gee
