/*
 * gee.h -- C ABI of libgee.so, the B200 (sm_100a) sparse Graph Encoder
 * Embedding hot path (arXiv 2406.03726).
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no C++ or torch
 * types cross this boundary.  All array pointers are DEVICE pointers unless
 * a name says _host.  Every call is stream-ordered, never synchronises the
 * host, never allocates device memory (workspaces are caller-provided after
 * a *_workspace size query) and is re-entrant across streams.
 *
 * Each entry point replaces one reference interface of the `graphee` 0.1.0
 * package (paths relative to /root/reference/pkg/src/graphee):
 *
 *   gee_label_hist           LabelVector.class_counts  embedding.py:68-71
 *                            + build_weight_matrix     embedding.py:92-107
 *   gee_csr_build            EdgeList.to_csr           graph_io.py:78-92
 *                            -> _kernels.coo_to_csr    _kernels.py:39-130, :314/:321
 *   gee_degree               degree_vector             sparse.py:193-196
 *                            (of A, or of add_identity(A) sparse.py:184-190)
 *                            + the scale of laplacian_normalize sparse.py:211-215
 *   gee_add_identity         _kernels.add_identity_kernel _kernels.py:137-198, :315/:322
 *   gee_laplacian_normalize  laplacian_normalize       sparse.py:199-226
 *   gee_embed                spmm(A', build_weight_matrix(Y)).to_dense()
 *                            sparse.py:166-181 -> _kernels.spmm_kernel _kernels.py:208-307
 *                            + correlate_rows          embedding.py:134-143
 *   gee_encode_edges         encode(EdgeList.to_csr(), labels, opts)
 *                            embedding.py:110-131 (the reference's timed region,
 *                            cli.py:170-180)
 *
 * Errors.  Host-detectable argument problems return a status synchronously
 * (GEE_E_ARG, GEE_E_WORKSPACE) and launch failures return GEE_E_CUDA.
 * Data-dependent problems are detected on the device and OR-ed into the
 * caller's device word `err` as GEE_ERR_* bits; the caller reads it once
 * after synchronising and raises the reference's exception class:
 *   GEE_ERR_NEG_DEGREE  -> NumericalDomainError  (sparse.py:211-212)
 *   GEE_ERR_NONFINITE   -> NumericalDomainError  (embedding.py:137-138)
 *   GEE_ERR_LABEL       -> StructuralError       (embedding.py:45-51)
 *   GEE_ERR_EDGE_RANGE  -> StructuralError       (graph_io.py:65-70)
 *   GEE_ERR_EDGE_WEIGHT -> StructuralError       (graph_io.py:71-72)
 */
#ifndef GEE_H
#define GEE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* synchronous status codes */
#define GEE_OK 0
#define GEE_E_ARG 1
#define GEE_E_WORKSPACE 2
#define GEE_E_CUDA 3

/* device error bits (OR-ed into *err) */
#define GEE_ERR_NEG_DEGREE 1
#define GEE_ERR_NONFINITE 2
#define GEE_ERR_LABEL 4
#define GEE_ERR_EDGE_RANGE 8
#define GEE_ERR_EDGE_WEIGHT 16
#define GEE_ERR_NEG_WEIGHT 32 /* GEE_NONNEG was passed but a weight is < 0 */

/* EmbedOptions (embedding.py:74-89) as a bit set */
#define GEE_LAPLACIAN 1u
#define GEE_DIAGONAL 2u
#define GEE_CORRELATION 4u
/* Caller's assertion that every edge weight is >= 0 (the EdgeList checks it
 * at construction).  Lets gee_encode_edges take the bucketed stream path,
 * which sums in any order; a violated assertion sets GEE_ERR_NEG_WEIGHT and
 * the result must be recomputed without the flag. */
#define GEE_NONNEG 8u
/* Output Z as float32 instead of float64 (accumulation stays in f64; the
 * north_star's optional fp32 path, 1e-5 relative). */
#define GEE_FP32 16u

/* edge-weight element types */
#define GEE_W_UNIT 0 /* w == NULL: every weight is 1.0 */
#define GEE_W_F64 1
#define GEE_W_F32 2 /* promoted to f64 exactly, as EdgeList does (graph_io.py:61) */

const char *gee_version(void);
const char *gee_status_string(int status);
/* last CUDA error text seen by this thread (for GEE_E_CUDA) */
const char *gee_last_error_string(void);

/* Validate an edge list on the device: 0 <= rows,cols < n and finite
 * weights (EdgeList.__post_init__, graph_io.py:58-72). */
int gee_validate_edges(const int64_t *rows, const int64_t *cols, const void *w, int w_type,
                       int64_t n_edges, int64_t n_nodes, int32_t *err, void *stream);

/* K1: labels int64[n] in {-1..k-1} -> y32 int32[n], counts int64[k]
 * (bit-exact n_k) and inv_nk f64[k] = 1.0/n_k (0 for empty classes, which
 * are never read).  Bad labels set GEE_ERR_LABEL. */
int gee_label_hist(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts,
                   double *inv_nk, int32_t *err, void *stream);

/* inv_nk[c] = 1.0 / counts[c] (0 for empty classes): used after the class
 * histograms of row shards are all-reduced (multi-GPU, dist.py). */
int gee_inv_counts(const int64_t *counts, int32_t k, double *inv_nk, void *stream);

/* build_weight_matrix (embedding.py:92-107): W = the N x K one-hot CSR of
 * the labels, row j holding inv_nk[y32[j]] (= 1.0/n_k) at column y32[j],
 * unlabeled rows empty.  y32 / inv_nk as gee_label_hist produces them;
 * index_pointers int64[n+1], col_indices int32[n], data f64[n] (the first
 * index_pointers[n] entries are written).  Workspace from
 * gee_weight_matrix_workspace. */
int gee_weight_matrix_workspace(int64_t n, size_t *ws_bytes);
int gee_weight_matrix(const int32_t *y32, int64_t n, const double *inv_nk, int64_t *index_pointers,
                      int32_t *col_indices, double *data, void *ws, size_t ws_bytes, void *stream);

/* K2: edge list -> CSR with the reference's exact structure and values:
 * undirected lists are symmetrised in the order [originals, reversed
 * off-diagonals]; entries are ordered by (row, col); duplicates are summed
 * left to right in that stream order; exact-zero sums are dropped.
 *   capacity of col/val: n_edges (directed) or 2*n_edges (undirected)
 *   row_ptr int64[n_rows+1], *nnz (device int64) = row_ptr[n_rows]
 * deg_flags: 0, or GEE_LAPLACIAN [| GEE_DIAGONAL] to also produce, fused,
 * the degree vector of A (or A+I) and scale = 1/sqrt(deg) (0 where deg==0)
 * into deg/scale (f64[n_rows]); requires n_rows == n_cols.
 * compact = 0 leaves each row's unique entries at the start of its
 * pre-dedup slot range (row i: [slot_ptr[i], slot_ptr[i]+row_cnt[i])) and
 * only gee_embed may consume it; compact = 1 produces a standard CSR. */
int gee_csr_build_workspace(int64_t n_edges, int64_t n_rows, int64_t n_cols, int directed,
                            size_t *ws_bytes);
int gee_csr_build(const int64_t *rows, const int64_t *cols, const void *w, int w_type,
                  int64_t n_edges, int64_t n_rows, int64_t n_cols, int directed, int compact,
                  int64_t *row_ptr, uint32_t *row_cnt, int32_t *col, double *val, int64_t *nnz,
                  unsigned deg_flags, double *deg, double *scale, void *ws, size_t ws_bytes,
                  int32_t *err, void *stream);

/* K3: degree of A (flags 0) or of A+I (GEE_DIAGONAL) for a square CSR,
 * folded per row in storage order exactly as np.bincount does, plus
 * scale = 1/sqrt(deg).  deg < 0 sets GEE_ERR_NEG_DEGREE. */
int gee_degree(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
               unsigned flags, double *deg, double *scale, int32_t *err, void *stream);

/* Materialised A+I (the reference seam; the embed path fuses it instead).
 * Two phases: counts -> (caller scans nothing; *nnz_out on device) then fill.
 * out capacity nnz + n. */
int gee_add_identity(const int64_t *row_ptr, const int32_t *col, const double *val, int64_t n,
                     int64_t *out_row_ptr, int32_t *out_col, double *out_val, int64_t *nnz_out,
                     void *ws, size_t ws_bytes, void *stream);
int gee_add_identity_workspace(int64_t n, size_t *ws_bytes);

/* Materialised D^-1/2 A D^-1/2 with zero pruning (bit-exact with
 * sparse.py:217: (v*s_r)*s_c).  deg < 0 sets GEE_ERR_NEG_DEGREE. */
int gee_laplacian_normalize(const int64_t *row_ptr, const int32_t *col, const double *val,
                            int64_t n, const double *deg, int64_t *out_row_ptr,
                            int32_t *out_col, double *out_val, int64_t *nnz_out, void *ws,
                            size_t ws_bytes, int32_t *err, void *stream);
int gee_laplacian_normalize_workspace(int64_t n, size_t *ws_bytes);

/* K4: Z[r - row_begin, :] for r in [row_begin, row_end):
 *   Z[r, c] = sum over stored (r, j) with Y_j == c of a'_rj * inv_nk[c]
 * with a' = a (+1 on the diagonal under GEE_DIAGONAL, inserted if absent)
 * and, under GEE_LAPLACIAN, a' <- (a' * scale_r) * scale_j; under
 * GEE_CORRELATION each nonzero row is divided by its 2-norm (non-finite
 * rows set GEE_ERR_NONFINITE).  row_cnt may be NULL (standard CSR) or the
 * uncompacted counts from gee_csr_build(compact=0).  val may be NULL for
 * unit weights.  n_cols is the node count (length of y32 / scale).  z is
 * dense row-major with leading dimension ldz >= k. */
int gee_embed_workspace(int64_t n_rows, int64_t n_cols, size_t *ws_bytes);
int gee_embed(const int64_t *row_ptr, const uint32_t *row_cnt, const int32_t *col,
              const double *val, int64_t row_begin, int64_t row_end, int64_t n_cols,
              const int32_t *y32, const double *inv_nk, const double *scale, int32_t k,
              unsigned flags, double *z, int64_t ldz, void *ws, size_t ws_bytes, int32_t *err,
              void *stream);

/* The whole reference timed region on the device: edge list + labels ->
 * Z (N x K, f64; f32 with GEE_FP32).  One stream, no host synchronisation.
 * Paths: the L2-resident bitmap + tcgen05 product (unit weights, N <= 16384,
 * K <= 8); the bucketed stream encode (unit weights, or GEE_NONNEG: no CSR
 * is built, sums in any order, 1e-12); otherwise the exact CSR assembly
 * (radix sort or row buckets) + fused embed.  The workspace query covers
 * every path the arguments allow. */
int gee_encode_edges_workspace(int64_t n_edges, int64_t n_nodes, int32_t k, int directed,
                               int w_type, size_t *ws_bytes);
int gee_encode_edges(const int64_t *rows, const int64_t *cols, const void *w, int w_type,
                     int64_t n_edges, int64_t n_nodes, int directed, const int64_t *labels,
                     int32_t k, unsigned flags, void *z, void *ws, size_t ws_bytes,
                     int32_t *err, void *stream);

/* Row shard of a unit-weight graph (multi-GPU, dist.py; replaces the
 * per-shard share of encode() embedding.py:110-131 for graphs of at most
 * 16384 nodes and k <= 8).  The shard owns rows [row_begin, row_end); rows /
 * cols hold its e_local entries of the SYMMETRISED stream (both directions
 * of every off-diagonal undirected edge, global node ids), labels all
 * n_nodes labels (replicated).  Two phases on the same workspace:
 *   gee_bitmap_shard_degrees -> deg_local uint32[row_end - row_begin], the
 *     stream length (unit-weight degree, without the A+I 1) of each local row;
 *   the caller all-gathers them into deg_all uint32[n_nodes] (only needed
 *     under GEE_LAPLACIAN; may be NULL otherwise);
 *   gee_bitmap_shard_encode -> z_local f64[(row_end - row_begin) x k].
 * Every encode must follow its own degrees call (the first clears the
 * workspace's counters).  Entries whose row is outside the shard set
 * GEE_ERR_EDGE_RANGE and are dropped. */
int gee_bitmap_shard_workspace(int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end,
                               int32_t k, size_t *ws_bytes);
int gee_bitmap_shard_degrees(const int64_t *rows, const int64_t *cols, int64_t e_local,
                             int64_t n_nodes, int64_t row_begin, int64_t row_end,
                             const int64_t *labels, int32_t k, unsigned flags, uint32_t *deg_local,
                             void *ws, size_t ws_bytes, int32_t *err, void *stream);
int gee_bitmap_shard_encode(const int64_t *rows, const int64_t *cols, int64_t e_local,
                            int64_t n_nodes, int64_t row_begin, int64_t row_end, int32_t k,
                            unsigned flags, const uint32_t *deg_all, double *z_local, void *ws,
                            size_t ws_bytes, int32_t *err, void *stream);

/* Row shard through the bucketed stream encode (multi-GPU, dist.py; unit or
 * GEE_NONNEG weights).  The shard owns rows [row_begin, row_end); rows / cols
 * / w hold its e_local stream entries (row in the range, any column: the
 * symmetrised list's entries of those rows), labels all n_nodes labels.
 *   gee_stream_shard_degrees -> deg_local f64[row_end - row_begin]: the raw
 *     weighted degrees of the local rows (without the A+I 1); the entries stay
 *     partitioned in the workspace;
 *   the caller all-gathers them into deg_all f64[n_nodes] (Laplacian only);
 *   gee_stream_shard_encode -> z_local (f64, or f32 under GEE_FP32)
 *     [(row_end - row_begin) x k]: node table of every node, then the embed.
 * Both calls take the same arguments and workspace.  Out-of-range entries set
 * GEE_ERR_EDGE_RANGE. */
int gee_stream_shard_workspace(int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end, int32_t k,
                               int w_type, unsigned flags, size_t *ws_bytes);
int gee_stream_shard_degrees(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t e_local,
                             int64_t n_nodes, int64_t row_begin, int64_t row_end, const int64_t *labels, int32_t k,
                             unsigned flags, double *deg_local, void *ws, size_t ws_bytes, int32_t *err,
                             void *stream);
int gee_stream_shard_encode(int w_type, int64_t e_local, int64_t n_nodes, int64_t row_begin, int64_t row_end,
                            int32_t k, unsigned flags, const double *deg_all, void *z_local, void *ws,
                            size_t ws_bytes, int32_t *err, void *stream);

/* Distributed CSR build: ranks start from contiguous slices
 * of the ORIGINAL edge list (slice p = stream positions [e_p, e_{p+1}) of
 * EdgeList(rows, cols, w), graph_io.py:48-92) and shuffle the symmetrised
 * stream to the P row owners.  Replaces the host-side partition of dist.py
 * (stream_row_counts / row_ranges / local_stream).
 *   gee_shuffle_row_hist   adds this slice's stream entries per coarse row
 *     bucket into hist uint64[n_buckets] (caller zeroes it, then
 *     all-reduces it); n_buckets = gee_shuffle_buckets(n_nodes);
 *   gee_shuffle_bounds     bounds int64[world + 1]: contiguous row ranges
 *     with near-equal stream entries (bucket-granular, as dist.row_ranges);
 *   gee_partition          stable partition into 2*world send buckets laid
 *     out [half][dest]: half 0 = originals by their row, half 1 = mirrored
 *     off-diagonals (undirected) by their column, written as (col, row);
 *     every bucket keeps slice order; counts uint64[2*world] bucket sizes;
 *     out_* hold up to 2*n_edges entries; w / out_w in w_type's width.
 * Exchanging the originals region, then the mirrors region, with one
 * all-to-all each and concatenating what arrives in source-rank order gives
 * each rank its slice of the symmetrised stream in stream order. world <= 16. */
int64_t gee_shuffle_buckets(int64_t n_nodes);
int gee_shuffle_row_hist(const int64_t *rows, const int64_t *cols, int64_t n_edges, int64_t n_nodes,
                         int directed, uint64_t *hist, void *stream);
int gee_shuffle_bounds(const uint64_t *hist, int64_t n_nodes, int world, int64_t *bounds, void *stream);
int gee_partition_workspace(int64_t n_edges, int world, size_t *ws_bytes);
int gee_partition(const int64_t *rows, const int64_t *cols, const void *w, int w_type, int64_t n_edges,
                  int directed, const int64_t *bounds, int world, int64_t *out_rows, int64_t *out_cols,
                  void *out_w, uint64_t *counts, void *ws, size_t ws_bytes, void *stream);

/* On-device synthetic generators (the reference's generator
 * is sbm.py:52-155, a sequential PCG64 stream).  Counter-based: word t of
 * stream `key` is splitmix64's output mix64(key + (t+1)*0x9e3779b97f4a7c15),
 * key = mix64(seed ^ stream_id * 0x9e3779b97f4a7c15), so the C restatement
 * oracle/gee_gen.c yields identical arrays.  Thresholds are integers
 * (probability * 2^32, computed by the caller).
 *   gee_gen_rmat     edge i: word i*16+h gives levels 2h (low 32 bits) and
 *                    2h+1 (high 32); u < t1 -> (0,0), < t2 -> (0,1),
 *                    < t3 -> (1,0), else (1,1); w (may be NULL) f32
 *                    1 - (word_i(wkey) >> 40) * 2^-24.
 *   gee_gen_chunglu  rows/cols = searchsorted(cdf, (word_i >> 11) * 2^-53,
 *                    'right') clipped to n-1; w (may be NULL) f64
 *                    1 - (word_i(wkey) >> 11) * 2^-53.
 *   gee_gen_pairs    keys[i] for candidate t0+i: a = hi32(lo32 * n),
 *                    b = hi32(hi32 * n); min*n + max, or -1 when a == b.
 *   gee_gen_sbm_*    pair (i, j), i < j: edge iff (word_{i*n+j} >> 32) <
 *                    (labels_i == labels_j ? thr_in : thr_out); counts[i]
 *                    per row, then the fill at the caller's exclusive
 *                    offsets, row-major. */
int gee_gen_rmat(uint64_t key, uint64_t wkey, int scale, int64_t n_edges, uint32_t t1, uint32_t t2, uint32_t t3,
                 int64_t *rows, int64_t *cols, float *w, void *stream);
int gee_gen_chunglu(uint64_t rkey, uint64_t ckey, uint64_t wkey, const double *cdf, int64_t n_nodes,
                    int64_t n_edges, int64_t *rows, int64_t *cols, double *w, void *stream);
int gee_gen_pairs(uint64_t key, int64_t t0, int64_t count, int64_t n_nodes, int64_t *keys, void *stream);
int gee_gen_sbm_count(uint64_t key, int64_t n_nodes, const int64_t *labels, uint32_t thr_in, uint32_t thr_out,
                      int64_t *counts, void *stream);
int gee_gen_sbm_fill(uint64_t key, int64_t n_nodes, const int64_t *labels, uint32_t thr_in, uint32_t thr_out,
                     const int64_t *offsets, int64_t *rows, int64_t *cols, void *stream);

/* Device text parsers (replace graph_io.parse_edge_list /
 * parse_labels, graph_io.py:95-257).  `text` is the file's bytes in device
 * memory.  Lines end at \n, \r\n or \r; each is stripped; blank lines and
 * '#' comments are skipped; the delimiter (0 auto: comma when the first data
 * line holds one, 1 whitespace, 2 comma) splits the fields; tokens follow
 * Python's int() / float().  Errors: info[2] = (1-based line << 8 | code) of
 * the first failing line, -1 if none; the host raises ParseError(line).
 *   gee_text_count_lines   *n_breaks; parsers take n_lines = n_breaks + 1
 *   gee_parse_edges        (i, j, w) of the data lines in file order into
 *                          rows / cols / w (capacity n_lines), shifted by the
 *                          index base; fallback[slot] = 1 where the weight has
 *                          more than 19 significant digits (host converts),
 *                          slot_line (may be NULL) the file line of each slot;
 *                          info: [0] edges, [1] max index, [2] error,
 *                          [3] fallbacks, [4] first data line
 *   gee_parse_labels       per data line: node (-1 in per-line form) and
 *                          label, slot_line = its file line
 *   gee_labels_assign      pair form: values[nv] (-1 unmentioned), the
 *                          conflicting-duplicate error into *err_word */
int gee_text_workspace(int64_t nbytes, int64_t n_lines, size_t *ws_bytes);
int gee_text_count_lines(const char *text, int64_t nbytes, int64_t *n_breaks, void *ws, size_t ws_bytes,
                         void *stream);
int gee_parse_edges(const char *text, int64_t nbytes, int64_t n_lines, int delim_mode, int index_base,
                    double default_weight, int64_t n_nodes, int64_t *line_start, int64_t *rows, int64_t *cols,
                    double *w, unsigned char *fallback, int64_t *slot_line, int64_t *info, void *ws,
                    size_t ws_bytes, void *stream);
int gee_parse_labels(const char *text, int64_t nbytes, int64_t n_lines, int delim_mode, int index_base,
                     int64_t n_nodes, int64_t *line_start, int64_t *node, int64_t *lab, int64_t *slot_line,
                     int64_t *info, void *ws, size_t ws_bytes, void *stream);
int gee_labels_assign(const int64_t *node, const int64_t *lab, const int64_t *slot_line, int64_t m, int64_t nv,
                      uint64_t *first, int64_t *values, uint64_t *err_word, void *stream);

/* Launch statistics: number of kernels this thread launched through the
 * library since the last reset (for bench.py's gpu_launches). */
uint64_t gee_launch_count(void);
void gee_reset_launch_count(void);

/* Per-kernel timing for the benchmark: after gee_profile_start(stream) the
 * calling thread's launches are each followed by an event record on their
 * stream; gee_profile_stop() ends recording and returns the mark count;
 * gee_profile_read() synchronises on the last mark and returns, per launch,
 * the elapsed ms since the previous mark and the kernel name. */
int gee_profile_start(void *stream);
int gee_profile_stop(void);
int gee_profile_read(float *ms, const char **names, int cap);

/* Test hook (thread-local) selecting the CSR assembly path so parity tests
 * cover all three: GEE_DEBUG_FORCE_BUCKETS = 0 default (bitmap for small
 * unit-weight graphs, radix sort when (row, col) packs into 32 bits or the
 * graph is weighted, row buckets otherwise), 1 = row buckets, 2 = never the
 * bitmap path, 3 = as 2 with the radix sort on every 64-bit (row, col) key.
 * Returns the previous value. */
#define GEE_DEBUG_FORCE_BUCKETS 1
/* Second hook: the shared-memory budget (bytes per warp) of the embed's flat
 * row blocks for K > 8; 0 = one warp per row instead.  Default 8192. */
#define GEE_DEBUG_EMBED_FLAT_BYTES 2
/* Third hook: the longest row a flat block takes (default 256); longer rows
 * get a warp each, rows over 4096 entries a CTA each. */
#define GEE_DEBUG_EMBED_FLAT_ROWMAX 3
/* Fourth hook: the bucketed stream encode: 0 auto, 1 never (tests force the
 * CSR paths with it). */
#define GEE_DEBUG_STREAM 4
/* Fifth hook: KB of the stream encode's shared Z tile (R x K x 8 bytes;
 * default 104; tests use it to force more, smaller buckets). */
#define GEE_DEBUG_STREAM_TILE 5
int gee_debug_set(int key, int value);

#ifdef __cplusplus
}
#endif

#endif /* GEE_H */
