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
// left to right (np.bincount).  When the exactness certificate holds any
// order is bitwise equal, so the warp reduces in parallel; otherwise lane 0
// replays the exact sequential fold.
__global__ void k_degree(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                         const double *__restrict__ val, int64_t n, unsigned flags,
                         double *__restrict__ deg, double *__restrict__ scale, int32_t *err,
                         const unsigned *guard) {
    if (guard && *guard == 0) return;  // device-side skip (unit-weight graphs use k_degree_stream)
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool diag = (flags & GEE_DIAGONAL) != 0;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t s = row_ptr[r], e = row_ptr[r + 1];
        Cert ce;
        double psum = 0.0;
        bool placed = false;
        for (int64_t p = s + lane; p < e; p += 32) {
            double x = val[p];
            if (diag && col[p] == r) {
                x = x + 1.0;
                placed = true;
            }
            ce.add(x);
            psum += x;
        }
        const bool insert = diag && !__any_sync(0xffffffffu, placed);
        int mlow = warp_min(ce.mlow);
        double sabs = warp_sum(ce.sabs) + (insert ? 1.0 : 0.0);
        if (insert) mlow = min(mlow, 0);
        double d;
        if (cert_ok(mlow, sabs)) {
            d = warp_sum(psum) + (insert ? 1.0 : 0.0);
        } else {
            d = 0.0;
            if (lane == 0) {
                bool ins = !insert;
                for (int64_t p = s; p < e; ++p) {
                    int64_t c = col[p];
                    double x = val[p];
                    if (!ins && c > r) {
                        d += 1.0;
                        ins = true;
                    }
                    if (diag && c == r) x = x + 1.0;
                    d += x;
                }
                if (!ins) d += 1.0;
            }
        }
        if (lane == 0) {
            deg[r] = d;
            if (scale) scale[r] = laplacian_scale(d, err);
        }
    }
}

int degree(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n, unsigned flags,
           double *deg, double *scale, int32_t *err, cudaStream_t st) {
    if (n <= 0) return GEE_OK;
    k_degree<<<grid_for(n * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, flags, deg, scale, err,
                                                       nullptr);
    GEE_CHECK_LAUNCH("k_degree");
    return GEE_OK;
}

// degree() that runs only if the device word *guard is nonzero
int degree_guarded(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                   unsigned flags, double *deg, double *scale, int32_t *err, const unsigned *guard,
                   cudaStream_t st) {
    if (n <= 0) return GEE_OK;
    k_degree<<<grid_for(n * 32, 256, 8), 256, 0, st>>>(row_ptr, col, val, n, flags, deg, scale, err,
                                                       guard);
    GEE_CHECK_LAUNCH("k_degree");
    return GEE_OK;
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
