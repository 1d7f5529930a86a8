// gee_abi.cu -- the extern "C" boundary of libgee.so (declared in include/gee.h).
#include <mutex>
#include <stdio.h>
#include <string.h>

#include "gee_common.cuh"

#define GEE_VERSION "gee-b200 0.1.0 (sm_100a)"

namespace gee {

static thread_local uint64_t t_launches = 0;
static thread_local char t_last_error[256] = "";

uint64_t &launch_counter() { return t_launches; }

// ---- per-kernel timing marks (bench.py only) --------------------------------
constexpr int kMaxMarks = 4096;
struct Profile {
    bool on = false;
    int n = 0;
    cudaEvent_t ev[kMaxMarks + 1] = {};
    const char *name[kMaxMarks + 1] = {};
};
static thread_local Profile t_prof;

void profile_mark(const char *name, cudaStream_t st) {
    Profile &p = t_prof;
    if (!p.on || p.n >= kMaxMarks) return;
    if (!p.ev[p.n]) cudaEventCreate(&p.ev[p.n]);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(p.ev[p.n], st, cudaEventRecordExternal);  // a record node in the graph
    else
        cudaEventRecord(p.ev[p.n], st);
    p.name[p.n] = name;
    ++p.n;
}

int cuda_status(cudaError_t e) {
    snprintf(t_last_error, sizeof(t_last_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return GEE_E_CUDA;
}

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kSMs;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = kSMs;
        cache[dev] = v;
    }
    return cache[dev];
}

int label_hist(const int64_t *, int64_t, int32_t, int32_t *, int64_t *, double *, int32_t *, cudaStream_t);
size_t label_partial_words(int64_t n, int k);
int inv_counts(const int64_t *counts, int32_t k, double *inv_nk, cudaStream_t st);
size_t weight_matrix_workspace(int64_t n);
int weight_matrix(const int32_t *y32, int64_t n, const double *inv_nk, int64_t *ptr, int32_t *cols, double *vals,
                  void *ws, cudaStream_t st);
int label_hist_pipeline(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts, double *inv_nk,
                        unsigned *partial, unsigned *done, int32_t *err, cudaStream_t st);
size_t csr_build_workspace(int64_t E, int64_t n_rows, int64_t n_cols, int directed);
size_t csr_build_workspace_any(int64_t E, int64_t n_rows, int64_t n_cols, int directed);
bool sort_path_ok(int64_t E, int64_t n_rows, int64_t n_cols, int directed, int wt);
int set_force_buckets(int v);
int set_embed_flat_bytes(int v);
int set_embed_flat_rowmax(int v);
size_t partition_workspace(int64_t E, int world);
int shuffle_row_hist(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed, int64_t nb,
                     unsigned long long *hist, cudaStream_t st);
int shuffle_bounds(const unsigned long long *hist, int64_t nb, int64_t n, int world, int64_t *bounds,
                   cudaStream_t st);
int partition(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int directed,
              const int64_t *bounds, int world, int64_t *out_rows, int64_t *out_cols, void *out_w,
              unsigned long long *counts, void *ws, size_t ws_bytes, cudaStream_t st);
int shuffle_max_world();
int64_t shuffle_buckets(int64_t n);
int sort_csr_build(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int64_t n_rows,
                   int64_t n_cols, int directed, int force_vals, int64_t *row_ptr, int32_t *col, double *val,
                   int64_t *nnz, unsigned deg_flags, double *deg, double *scale, void *ws, size_t ws_bytes,
                   unsigned **val_mode, int32_t *err, cudaStream_t st);
int csr_build(const int64_t *, const int64_t *, const void *, int, int64_t, int64_t, int64_t, int, int,
              int64_t *, unsigned *, int32_t *, double *, int64_t *, unsigned, double *, double *, void *,
              size_t, int32_t *, cudaStream_t);
int degree(const int64_t *, const int32_t *, const double *, int64_t, unsigned, double *, double *,
           int32_t *, cudaStream_t);
size_t add_identity_workspace(int64_t n);
int add_identity(const int64_t *, const int32_t *, const double *, int64_t, int64_t *, int32_t *, double *,
                 int64_t *, void *, size_t, cudaStream_t);
size_t laplacian_workspace(int64_t n);
int laplacian_normalize(const int64_t *, const int32_t *, const double *, int64_t, const double *, int64_t *,
                        int32_t *, double *, int64_t *, void *, size_t, int32_t *, cudaStream_t);
size_t embed_workspace(int64_t n_rows, int64_t n_cols);
int embed(const int64_t *row_ptr, const unsigned *row_cnt, const int32_t *col, const double *val,
          const unsigned *val_flags, const unsigned char *row_flag, int64_t rb, int64_t re, int64_t n_cols,
          const int32_t *y32, const double *inv, const double *scale, int k, unsigned flags, double *z, int64_t ldz,
          void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st, int prepared = 0);
int embed_long_row();
void embed_scratch(void *ws, int64_t n_rows, int64_t n_cols, unsigned **ctr, unsigned **list, double2 **rec,
                   double **tab_g, signed char **tab_lab);
bool bitmap_path_ok(int wt, int64_t E, int64_t n_rows, int64_t n_cols, int directed, int k);
size_t bitmap_workspace(int64_t E, int64_t n, int directed, int k);
int bitmap_encode(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed,
                  const int64_t *labels, int k, unsigned flags, int32_t *y32, int64_t *counts, double *inv,
                  double *deg, double *scale, double *z, void *ws, size_t ws_bytes, int32_t *err,
                  cudaStream_t st);
int validate_edges(const int64_t *, const int64_t *, const void *, int, int64_t, int64_t, int32_t *,
                   cudaStream_t);
size_t bitmap_shard_workspace(int64_t n, int64_t nloc, int k);
int bitmap_shard_degrees(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int64_t row0, int64_t nloc,
                         const int64_t *labels, int k, unsigned flags, unsigned *deg_local, void *ws,
                         size_t ws_bytes, int32_t *err, cudaStream_t st);
int bitmap_shard_encode(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int64_t row0, int64_t nloc,
                        int k, unsigned flags, const unsigned *deg_all, double *z_local, void *ws, size_t ws_bytes,
                        int32_t *err, cudaStream_t st);
int bitmap_max_nodes();
bool stream_path_ok(int wt, unsigned flags, int64_t E, int64_t N, int directed, int k);
size_t stream_workspace(int64_t E, int64_t N, int directed, int k, int wt);
int stream_encode(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int64_t N, int directed,
                  const int64_t *labels, int32_t k, unsigned flags, void *z, void *ws, size_t ws_bytes,
                  int32_t *err, cudaStream_t st);
int set_stream_mode(int v);
bool stream_shard_ok(int wt, unsigned flags, int64_t e_local, int64_t N, int64_t rb, int64_t re, int k);
size_t stream_shard_workspace(int64_t e_local, int64_t N, int64_t rb, int64_t re, int k, int wt);
int stream_shard_degrees(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t e_local, int64_t N,
                         int64_t rb, int64_t re, const int64_t *labels, int32_t k, unsigned flags, double *deg_local,
                         void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st);
int stream_shard_encode(int wt, int64_t e_local, int64_t N, int64_t rb, int64_t re, int32_t k, unsigned flags,
                        const double *deg_all, void *z_local, void *ws, size_t ws_bytes, int32_t *err,
                        cudaStream_t st);
int set_stream_tile_kb(int v);
int set_stream_embed_nt(int v);

static bool index_ok(int64_t x) { return x >= 0 && x < ((int64_t)1 << 31); }
static bool wt_ok(int wt, const void *w, int64_t n_edges) {
    if (n_edges == 0) return wt == GEE_W_UNIT || wt == GEE_W_F64 || wt == GEE_W_F32;
    if (wt == GEE_W_UNIT) return true;
    return (wt == GEE_W_F64 || wt == GEE_W_F32) && w != nullptr;
}

// Pipeline workspace: everything encode needs between K1 and K4.
struct EncodeWs {
    int32_t *y32;
    int64_t *counts;
    double *inv, *deg, *scale;
    int64_t *row_ptr;
    unsigned *row_cnt;
    unsigned char *row_flag;
    int32_t *col;
    double *val;
    unsigned *label_partial;
    void *csr_ws;
    size_t csr_bytes;
    void *emb_ws;
    size_t emb_bytes;
};

static size_t carve_encode(Carver &cv, EncodeWs &w, int64_t E, int64_t n, int32_t k, int directed, int wt) {
    const int64_t M = directed ? E : 2 * E;
    w.y32 = cv.take<int32_t>((size_t)n + 1);
    w.counts = cv.take<int64_t>((size_t)k);
    w.inv = cv.take<double>((size_t)k);
    w.deg = cv.take<double>((size_t)n + 1);
    w.scale = cv.take<double>((size_t)n + 1);
    w.row_ptr = cv.take<int64_t>((size_t)n + 1);
    w.row_cnt = cv.take<unsigned>((size_t)n + 1);
    w.row_flag = cv.take<unsigned char>((size_t)n + 1);
    w.col = cv.take<int32_t>((size_t)(M > 0 ? M : 1));
    w.val = cv.take<double>((size_t)(M > 0 ? M : 1));
    w.label_partial = cv.take<unsigned>(label_partial_words(n, k));
    // every path the arguments allow (the test hooks switch paths after a plan is sized)
    w.csr_bytes = csr_build_workspace_any(E, n, n, directed);
    if (wt == GEE_W_UNIT && n >= 1 && n <= bitmap_max_nodes() && k <= 8) {
        const size_t b = bitmap_workspace(E, n, directed, k);
        if (b > w.csr_bytes) w.csr_bytes = b;
    }
    w.csr_ws = cv.take<char>(w.csr_bytes);
    w.emb_bytes = embed_workspace(n, n);
    w.emb_ws = cv.take<char>(w.emb_bytes);
    return cv.bytes();
}

}  // namespace gee

using namespace gee;

extern "C" {

const char *gee_version(void) { return GEE_VERSION; }

const char *gee_status_string(int s) {
    switch (s) {
        case GEE_OK: return "ok";
        case GEE_E_ARG: return "invalid argument";
        case GEE_E_WORKSPACE: return "workspace too small";
        case GEE_E_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

const char *gee_last_error_string(void) { return t_last_error; }

uint64_t gee_launch_count(void) { return t_launches; }
void gee_reset_launch_count(void) { t_launches = 0; }

int gee_profile_start(void *stream) {
    Profile &p = t_prof;
    p.on = true;
    p.n = 0;
    profile_mark("start", (cudaStream_t)stream);
    return GEE_OK;
}

int gee_debug_set(int key, int value) {
    if (key == GEE_DEBUG_FORCE_BUCKETS) return set_force_buckets(value);
    if (key == GEE_DEBUG_STREAM) return set_stream_mode(value);
    if (key == GEE_DEBUG_STREAM_TILE) return set_stream_tile_kb(value);
    if (key == 6) return set_stream_embed_nt(value);
    if (key == GEE_DEBUG_EMBED_FLAT_BYTES) return set_embed_flat_bytes(value);
    if (key == GEE_DEBUG_EMBED_FLAT_ROWMAX) return set_embed_flat_rowmax(value);
    return -1;
}

int gee_profile_stop(void) {
    t_prof.on = false;
    return t_prof.n;
}

int gee_profile_read(float *ms, const char **names, int cap) {
    Profile &p = t_prof;
    if (p.n < 1) return 0;
    cudaError_t e = cudaEventSynchronize(p.ev[p.n - 1]);
    if (e != cudaSuccess) return -cuda_status(e);
    int m = 0;
    for (int i = 1; i < p.n && m < cap; ++i, ++m) {
        float t = 0.f;
        e = cudaEventElapsedTime(&t, p.ev[i - 1], p.ev[i]);
        if (e != cudaSuccess) return -cuda_status(e);
        ms[m] = t;
        names[m] = p.name[i];
    }
    return m;
}

int gee_validate_edges(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t n_edges,
                       int64_t n_nodes, int32_t *err, void *stream) {
    if (n_edges < 0 || n_nodes < 0 || !wt_ok(w_type, w, n_edges) || !err) return GEE_E_ARG;
    return validate_edges(rows, cols, w, w_type, n_edges, n_nodes, err, (cudaStream_t)stream);
}

int gee_label_hist(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts, double *inv_nk,
                   int32_t *err, void *stream) {
    if (n < 0 || k < 1 || !index_ok(n) || !y32 || !counts || !inv_nk) return GEE_E_ARG;
    if (n > 0 && !labels) return GEE_E_ARG;
    return label_hist(labels, n, k, y32, counts, inv_nk, err, (cudaStream_t)stream);
}

int gee_inv_counts(const int64_t *counts, int32_t k, double *inv_nk, void *stream) {
    if (k < 1 || !counts || !inv_nk) return GEE_E_ARG;
    return inv_counts(counts, k, inv_nk, (cudaStream_t)stream);
}

int gee_weight_matrix_workspace(int64_t n, size_t *ws_bytes) {
    if (!ws_bytes || n < 0 || !index_ok(n)) return GEE_E_ARG;
    *ws_bytes = weight_matrix_workspace(n);
    return GEE_OK;
}

int gee_weight_matrix(const int32_t *y32, int64_t n, const double *inv_nk, int64_t *index_pointers,
                      int32_t *col_indices, double *data, void *ws, size_t ws_bytes, void *stream) {
    if (n < 0 || !index_ok(n) || !index_pointers || !inv_nk) return GEE_E_ARG;
    if (n > 0 && (!y32 || !col_indices || !data || !ws || ws_bytes < weight_matrix_workspace(n))) return GEE_E_ARG;
    return weight_matrix(y32, n, inv_nk, index_pointers, col_indices, data, ws, (cudaStream_t)stream);
}

int gee_csr_build_workspace(int64_t n_edges, int64_t n_rows, int64_t n_cols, int directed, size_t *ws_bytes) {
    if (!ws_bytes || n_edges < 0 || !index_ok(n_edges) || !index_ok(n_rows) || !index_ok(n_cols))
        return GEE_E_ARG;
    *ws_bytes = csr_build_workspace(n_edges, n_rows, n_cols, directed);
    return GEE_OK;
}

int gee_csr_build(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t n_edges,
                  int64_t n_rows, int64_t n_cols, int directed, int compact, int64_t *row_ptr, uint32_t *row_cnt,
                  int32_t *col, double *val, int64_t *nnz, unsigned deg_flags, double *deg, double *scale,
                  void *ws, size_t ws_bytes, int32_t *err, void *stream) {
    if (!index_ok(n_edges) || !index_ok(n_rows) || !index_ok(n_cols) || !wt_ok(w_type, w, n_edges)) return GEE_E_ARG;
    if (!row_ptr || (!compact && !row_cnt) || (n_edges > 0 && (!rows || !cols || !col || !val)))
        return GEE_E_ARG;
    if (!directed && n_rows != n_cols) return GEE_E_ARG;
    if (deg_flags && (n_rows != n_cols || !deg || ((deg_flags & GEE_LAPLACIAN) && !scale)))
        return GEE_E_ARG;
    return csr_build(rows, cols, w, w_type, n_edges, n_rows, n_cols, directed, compact, row_ptr, row_cnt, col, val,
                     nnz, deg_flags, deg, scale, ws, ws_bytes, err, (cudaStream_t)stream);
}

int gee_degree(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n, unsigned flags,
               double *deg, double *scale, int32_t *err, void *stream) {
    if (!index_ok(n) || !row_ptr || !deg) return GEE_E_ARG;
    return degree(row_ptr, col, val, n, flags, deg, scale, err, (cudaStream_t)stream);
}

int gee_add_identity_workspace(int64_t n, size_t *ws_bytes) {
    if (!ws_bytes || !index_ok(n)) return GEE_E_ARG;
    *ws_bytes = add_identity_workspace(n);
    return GEE_OK;
}

int gee_add_identity(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                     int64_t *out_row_ptr, int32_t *out_col, double *out_val, int64_t *nnz_out, void *ws,
                     size_t ws_bytes, void *stream) {
    if (!index_ok(n) || !row_ptr || !out_row_ptr) return GEE_E_ARG;
    return add_identity(row_ptr, col, val, n, out_row_ptr, out_col, out_val, nnz_out, ws, ws_bytes,
                        (cudaStream_t)stream);
}

int gee_laplacian_normalize_workspace(int64_t n, size_t *ws_bytes) {
    if (!ws_bytes || !index_ok(n)) return GEE_E_ARG;
    *ws_bytes = laplacian_workspace(n);
    return GEE_OK;
}

int gee_laplacian_normalize(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                            const double *deg, int64_t *out_row_ptr, int32_t *out_col, double *out_val,
                            int64_t *nnz_out, void *ws, size_t ws_bytes, int32_t *err, void *stream) {
    if (!index_ok(n) || !row_ptr || !deg || !out_row_ptr) return GEE_E_ARG;
    return laplacian_normalize(row_ptr, col, val, n, deg, out_row_ptr, out_col, out_val, nnz_out, ws, ws_bytes,
                               err, (cudaStream_t)stream);
}

int gee_embed_workspace(int64_t n_rows, int64_t n_cols, size_t *ws_bytes) {
    if (!ws_bytes || !index_ok(n_rows) || !index_ok(n_cols)) return GEE_E_ARG;
    *ws_bytes = embed_workspace(n_rows, n_cols);
    return GEE_OK;
}

int gee_embed(const int64_t *row_ptr, const uint32_t *row_cnt, const int32_t *col, const double *val,
              int64_t row_begin, int64_t row_end, int64_t n_cols, const int32_t *y32, const double *inv_nk,
              const double *scale, int32_t k, unsigned flags, double *z, int64_t ldz, void *ws, size_t ws_bytes,
              int32_t *err, void *stream) {
    if (k < 1 || ldz < k || row_begin < 0 || row_end < row_begin || !index_ok(row_end) || !index_ok(n_cols))
        return GEE_E_ARG;
    if (row_end > row_begin && (!row_ptr || !y32 || !inv_nk || !z)) return GEE_E_ARG;
    if ((flags & GEE_LAPLACIAN) && !scale) return GEE_E_ARG;
    return embed(row_ptr, row_cnt, col, val, nullptr, nullptr, row_begin, row_end, n_cols, y32, inv_nk, scale, k,
                 flags, z, ldz, ws, ws_bytes, err, (cudaStream_t)stream);
}

// row shard of a unit-weight graph on the bitmap path
static bool bm_shard_ok(int64_t e_local, int64_t n, int64_t rb, int64_t re, int32_t k) {
    return index_ok(e_local) && n >= 1 && n <= bitmap_max_nodes() && rb >= 0 && rb <= re && re <= n && k >= 1 &&
           k <= 8;
}

int gee_bitmap_shard_workspace(int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end, int32_t k,
                               size_t *ws_bytes) {
    if (!ws_bytes || !bm_shard_ok(e_local, n_nodes, row_begin, row_end, k)) return GEE_E_ARG;
    *ws_bytes = bitmap_shard_workspace(n_nodes, row_end - row_begin, k);
    return GEE_OK;
}

int gee_bitmap_shard_degrees(const int64_t *rows, const int64_t *cols, int64_t e_local, int64_t n_nodes,
                             int64_t row_begin, int64_t row_end, const int64_t *labels, int32_t k, unsigned flags,
                             uint32_t *deg_local, void *ws, size_t ws_bytes, int32_t *err, void *stream) {
    if (!bm_shard_ok(e_local, n_nodes, row_begin, row_end, k) || !labels || !err) return GEE_E_ARG;
    if ((e_local && (!rows || !cols)) || (row_end > row_begin && !deg_local)) return GEE_E_ARG;
    if (!ws) return GEE_E_WORKSPACE;
    return bitmap_shard_degrees(rows, cols, e_local, n_nodes, row_begin, row_end - row_begin, labels, k, flags,
                                deg_local, ws, ws_bytes, err, (cudaStream_t)stream);
}

int gee_bitmap_shard_encode(const int64_t *rows, const int64_t *cols, int64_t e_local, int64_t n_nodes,
                            int64_t row_begin, int64_t row_end, int32_t k, unsigned flags, const uint32_t *deg_all,
                            double *z_local, void *ws, size_t ws_bytes, int32_t *err, void *stream) {
    if (!bm_shard_ok(e_local, n_nodes, row_begin, row_end, k) || !err) return GEE_E_ARG;
    if ((e_local && (!rows || !cols)) || (row_end > row_begin && !z_local)) return GEE_E_ARG;
    if ((flags & GEE_LAPLACIAN) && !deg_all) return GEE_E_ARG;
    if (!ws) return GEE_E_WORKSPACE;
    return bitmap_shard_encode(rows, cols, e_local, n_nodes, row_begin, row_end - row_begin, k, flags, deg_all,
                               z_local, ws, ws_bytes, err, (cudaStream_t)stream);
}

int gee_encode_edges_workspace(int64_t n_edges, int64_t n_nodes, int32_t k, int directed, int w_type,
                               size_t *ws_bytes) {
    if (!ws_bytes || !index_ok(n_edges) || !index_ok(n_nodes) || k < 1) return GEE_E_ARG;
    Carver cv(nullptr);
    EncodeWs w;
    *ws_bytes = carve_encode(cv, w, n_edges, n_nodes, k, directed, w_type);
    const size_t sb = stream_workspace(n_edges, n_nodes, directed, k, w_type);
    if (sb > *ws_bytes) *ws_bytes = sb;
    return GEE_OK;
}

int gee_encode_edges(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t n_edges,
                     int64_t n_nodes, int directed, const int64_t *labels, int32_t k, unsigned flags, void *zv,
                     void *ws, size_t ws_bytes, int32_t *err, void *stream) {
    if (!index_ok(n_edges) || !index_ok(n_nodes) || k < 1 || !wt_ok(w_type, w, n_edges) || !zv) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const bool bitmap = !(flags & GEE_FP32) && bitmap_path_ok(w_type, n_edges, n_nodes, n_nodes, directed, k);
    if (!bitmap && stream_path_ok(w_type, flags, n_edges, n_nodes, directed, k)) {
        // non-negative weights: the bucketed stream encode (no CSR)
        if (!ws) return GEE_E_WORKSPACE;
        return stream_encode(rows, cols, w, w_type, n_edges, n_nodes, directed, labels, k, flags, zv, ws, ws_bytes,
                             err, st);
    }
    if (flags & GEE_FP32) return GEE_E_ARG;  // float32 output is produced by the stream path only
    double *z = static_cast<double *>(zv);
    Carver cv(ws);
    EncodeWs W;
    size_t need = carve_encode(cv, W, n_edges, n_nodes, k, directed, w_type);
    if (ws_bytes < need || !ws) return GEE_E_WORKSPACE;
    if (bitmap) {
        // unit weights, small node count, K <= 8: labels, an L2-resident N x N
        // adjacency bitmap and Z in three launches (no CSR, no embed pass)
        return bitmap_encode(rows, cols, n_edges, n_nodes, directed, labels, k, flags, W.y32, W.counts, W.inv,
                             W.deg, W.scale, z, W.csr_ws, W.csr_bytes, err, st);
    }
    // control words: embed counters [0..2] and the label kernel's done word [3]
    unsigned *ectr, *elist;
    double2 *erec;
    double *etg;
    signed char *etl;
    embed_scratch(W.emb_ws, n_nodes, n_nodes, &ectr, &elist, &erec, &etg, &etl);
    GEE_CHECK_CUDA(cudaMemsetAsync(ectr, 0, 8 * sizeof(unsigned), st));
    int rc = label_hist_pipeline(labels, n_nodes, k, W.y32, W.counts, W.inv, W.label_partial, ectr + 3, err, st);
    if (rc) return rc;
    const unsigned deg_flags = (flags & GEE_LAPLACIAN) ? (GEE_LAPLACIAN | (flags & GEE_DIAGONAL)) : 0u;
    const double *sc = (flags & GEE_LAPLACIAN) ? W.scale : nullptr;
    if (sort_path_ok(n_edges, n_nodes, n_nodes, directed, w_type)) {
        // compact CSR from the radix sort; values stay implicit (1.0) when the
        // graph has unit weights and no duplicate entries
        unsigned *val_mode = nullptr;
        rc = sort_csr_build(rows, cols, w, w_type, n_edges, n_nodes, n_nodes, directed, 0, W.row_ptr, W.col, W.val,
                            nullptr, deg_flags, W.deg, W.scale, W.csr_ws, W.csr_bytes, &val_mode, err, st);
        if (rc) return rc;
        return embed(W.row_ptr, nullptr, W.col, W.val, val_mode, nullptr, 0, n_nodes, n_nodes, W.y32, W.inv, sc, k,
                     flags, z, k, W.emb_ws, W.emb_bytes, err, st);
    }
    rc = csr_build(rows, cols, w, w_type, n_edges, n_nodes, n_nodes, directed, 0, W.row_ptr, W.row_cnt, W.col,
                   W.val, nullptr, deg_flags, W.deg, W.scale, W.csr_ws, W.csr_bytes, err, st);
    if (rc) return rc;
    return embed(W.row_ptr, W.row_cnt, W.col, W.val, nullptr, nullptr, 0, n_nodes, n_nodes, W.y32, W.inv, sc, k,
                 flags, z, k, W.emb_ws, W.emb_bytes, err, st);
}

}  // extern "C"

// ---- row shards through the stream encode (k_stream.cu) --------------------
extern "C" {

int gee_stream_shard_workspace(int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end, int32_t k,
                               int w_type, unsigned flags, size_t *ws_bytes) {
    if (!ws_bytes || !stream_shard_ok(w_type, flags, e_local, n_nodes, row_begin, row_end, k)) return GEE_E_ARG;
    *ws_bytes = stream_shard_workspace(e_local, n_nodes, row_begin, row_end, k, w_type);
    return GEE_OK;
}

int gee_stream_shard_degrees(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t e_local,
                             int64_t n_nodes, int64_t row_begin, int64_t row_end, const int64_t *labels, int32_t k,
                             unsigned flags, double *deg_local, void *ws, size_t ws_bytes, int32_t *err,
                             void *stream) {
    if (!stream_shard_ok(w_type, flags, e_local, n_nodes, row_begin, row_end, k) || !labels || !deg_local ||
        (e_local && (!rows || !cols || (w_type != GEE_W_UNIT && !w))))
        return GEE_E_ARG;
    return stream_shard_degrees(rows, cols, w, w_type, e_local, n_nodes, row_begin, row_end, labels, k, flags,
                                deg_local, ws, ws_bytes, err, (cudaStream_t)stream);
}

int gee_stream_shard_encode(int w_type, int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end,
                            int32_t k, unsigned flags, const double *deg_all, void *z_local, void *ws,
                            size_t ws_bytes, int32_t *err, void *stream) {
    if (!stream_shard_ok(w_type, flags, e_local, n_nodes, row_begin, row_end, k) || !z_local ||
        ((flags & GEE_LAPLACIAN) && !deg_all))
        return GEE_E_ARG;
    return stream_shard_encode(w_type, e_local, n_nodes, row_begin, row_end, k, flags, deg_all, z_local, ws,
                               ws_bytes, err, (cudaStream_t)stream);
}

}  // extern "C"

// ---- distributed CSR build: the edge shuffle (k_shuffle.cu) ----------------
int64_t gee_shuffle_buckets(int64_t n_nodes) { return n_nodes > 0 ? shuffle_buckets(n_nodes) : 0; }

int gee_shuffle_row_hist(const int64_t *rows, const int64_t *cols, int64_t n_edges, int64_t n_nodes, int directed,
                         uint64_t *hist, void *stream) {
    if (n_edges < 0 || n_nodes <= 0 || !hist || (n_edges && (!rows || !cols))) return GEE_E_ARG;
    return shuffle_row_hist(rows, cols, n_edges, n_nodes, directed, shuffle_buckets(n_nodes),
                            reinterpret_cast<unsigned long long *>(hist), (cudaStream_t)stream);
}

int gee_shuffle_bounds(const uint64_t *hist, int64_t n_nodes, int world, int64_t *bounds, void *stream) {
    if (n_nodes <= 0 || world < 1 || world > shuffle_max_world() || !hist || !bounds) return GEE_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    return shuffle_bounds(reinterpret_cast<const unsigned long long *>(hist), shuffle_buckets(n_nodes), n_nodes,
                          world, bounds, st);
}

int gee_partition_workspace(int64_t n_edges, int world, size_t *ws_bytes) {
    if (!ws_bytes || n_edges < 0 || world < 1 || world > shuffle_max_world()) return GEE_E_ARG;
    *ws_bytes = partition_workspace(n_edges, world);
    return GEE_OK;
}

int gee_partition(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t n_edges, int directed,
                  const int64_t *bounds, int world, int64_t *out_rows, int64_t *out_cols, void *out_w,
                  uint64_t *counts, void *ws, size_t ws_bytes, void *stream) {
    if (n_edges < 0 || world < 1 || world > shuffle_max_world() || !bounds || !counts) return GEE_E_ARG;
    if (w_type != GEE_W_UNIT && w_type != GEE_W_F64 && w_type != GEE_W_F32) return GEE_E_ARG;
    if (n_edges && (!rows || !cols || !out_rows || !out_cols)) return GEE_E_ARG;
    if (n_edges && w_type != GEE_W_UNIT && (!w || !out_w)) return GEE_E_ARG;
    if (!ws && partition_workspace(n_edges, world) > 0 && n_edges) return GEE_E_WORKSPACE;
    return partition(rows, cols, w, w_type, n_edges, directed, bounds, world, out_rows, out_cols, out_w,
                     reinterpret_cast<unsigned long long *>(counts), ws, ws_bytes, (cudaStream_t)stream);
}
