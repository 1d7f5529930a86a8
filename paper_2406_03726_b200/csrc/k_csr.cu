// k_csr.cu -- K2: edge list -> CSR with the reference's exact structure, and
// the fused K3 degree of A / A+I for the rows it assembles.
//
// Reference semantics (bitwise):
//   * EdgeList.to_csr (graph_io.py:78-92): undirected lists become the stream
//     [originals..., reversed off-diagonals...]; self-loops contribute once.
//   * _coo_to_csr_loops (_kernels.py:73-130): stable by (row, col); duplicate
//     runs summed LEFT TO RIGHT IN STREAM ORDER; sums equal to 0.0 dropped.
//   * degree_vector (sparse.py:193-196): per-row left fold in column order,
//     of A or of add_identity(A) (_kernels.py:169-198, diagonal merged as one
//     v+1.0 term or inserted as 1.0 at its sorted position).
//
// B200 design: stream entry e of the symmetrised list is identified by
// idx = e (original) or E + e (reversed), which orders exactly like the
// reference's concatenation.  Entries are bucketed by row (count -> scan ->
// scatter, shared-memory privatised when the row count is small), then every
// row is ordered on chip by the 64-bit key (col << 32 | idx):
//   tier S  L <= 32            warp rank-sort in registers
//   tier M  L <= kMCap         warp bitonic sort in a per-warp shared slice
//   tier D  small n_cols       CTA counting sort over the column range in
//                              shared memory (rows of ~1K entries, cfg 0/1)
//   tier B  L <= kCap          CTA bitonic sort in shared memory
//   tier X  L >  kCap          CTA stable LSD radix over the column bits in
//                              global memory (hub rows of power-law graphs)
// Tiers D and X sort by column only; equal-column runs of length >= 3 are then
// put back into idx order (a run of 2 sums commutatively, so order is moot).
// One persistent kernel drains the tiers longest-first.
#include "gee_common.cuh"

namespace gee {
#ifdef GEE_TRACE
__device__ unsigned long long g_lsd_t[512][4];
#endif

int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st);
size_t scan_workspace(int64_t n);

constexpr int kRowsThreads = 512;
constexpr int kCap = 4096;           // entries staged in shared memory per row
constexpr int kSmallRows = 16384;    // privatised row histogram (64 KB)
constexpr int kSmallCols = 12288;    // dense per-row column counting (48 KB)
constexpr int kSChunk = 64;          // tier-S rows per work grab
constexpr int kMCap = 256;           // tier-M rows: one warp, 256 x 16 B of shared memory

enum { TIER_D = 0, TIER_B = 1, TIER_X = 2, TIER_M = 3, kTiers = 4 };

__device__ __forceinline__ double load_w(const void *w, int wt, int64_t e) {
    if (wt == GEE_W_F64) return static_cast<const double *>(w)[e];
    if (wt == GEE_W_F32) return (double)static_cast<const float *>(w)[e];
    return 1.0;
}

// ---------------------------------------------------------------------------
// Pass 1: per-row counts of the symmetrised stream.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void warp_agg_add(unsigned *ctr, unsigned key, bool valid) {
    unsigned k = valid ? key : 0xffffffffu;
    unsigned peers = __match_any_sync(0xffffffffu, k);
    if (valid && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&ctr[key], __popc(peers));
}

// returns this lane's slot from a warp-aggregated atomicAdd on ctr[key]
__device__ __forceinline__ unsigned warp_agg_take(unsigned *ctr, unsigned key, bool valid) {
    unsigned k = valid ? key : 0xffffffffu;
    unsigned peers = __match_any_sync(0xffffffffu, k);
    int leader = __ffs(peers) - 1;
    unsigned base = 0;
    if (valid && (int)(threadIdx.x & 31) == leader) base = atomicAdd(&ctr[key], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(peers & lanemask_lt());
}

__global__ void k_count_global(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                               int64_t E, int directed, unsigned *__restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const unsigned r = (unsigned)rows[e], c = (unsigned)cols[e];
        atomicAdd(&cnt[r], 1u);  // RED: no return, nothing waits on it
        if (!directed && r != c) atomicAdd(&cnt[c], 1u);
    }
}

__device__ __forceinline__ void chunk_of(int64_t E, int64_t &e0, int64_t &e1) {
    e0 = (int64_t)((__int128)E * blockIdx.x / gridDim.x);
    e1 = (int64_t)((__int128)E * (blockIdx.x + 1) / gridDim.x);
}

// small row count: CTA-private histogram of its contiguous edge chunk
__global__ void k_count_part(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                             int64_t E, int directed, int n_rows, unsigned *__restrict__ part) {
    extern __shared__ unsigned sh[];
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) sh[r] = 0;
    __syncthreads();
    int64_t e0, e1;
    chunk_of(E, e0, e1);
    for (int64_t b = e0; b < e1; b += blockDim.x) {
        int64_t e = b + threadIdx.x;
        bool v = e < e1;
        unsigned r = v ? (unsigned)rows[e] : 0u, c = v ? (unsigned)cols[e] : 0u;
        warp_agg_add(sh, r, v);
        warp_agg_add(sh, c, v && !directed && r != c);
    }
    __syncthreads();
    unsigned *dst = part + (size_t)blockIdx.x * n_rows;
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x) dst[r] = sh[r];
}

// part[g][r] -> exclusive prefix over g; cnt[r] = total
__global__ void k_part_reduce(unsigned *__restrict__ part, int G, int n_rows,
                              unsigned *__restrict__ cnt) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rows) return;
    unsigned run = 0;
    for (int g = 0; g < G; ++g) {
        unsigned x = part[(size_t)g * n_rows + r];
        part[(size_t)g * n_rows + r] = run;
        run += x;
    }
    cnt[r] = run;
}

// ---------------------------------------------------------------------------
// Pass 2: scatter (key = col<<32 | idx, value = weight) into row buckets.
// ---------------------------------------------------------------------------
__global__ void k_scatter_global(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                                 const void *__restrict__ w, int wt, int64_t E, int directed,
                                 const int64_t *__restrict__ slot_ptr, unsigned *__restrict__ cursor,
                                 unsigned long long *__restrict__ key, double *__restrict__ val) {
    // kU entries per thread with every slot reservation (a returning atomic)
    // and bucket-start load in flight together: one round trip per kU entries
    constexpr int kU = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * kU;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x * kU + threadIdx.x; e0 < E; e0 += stride) {
        unsigned r[kU], c[kU], s1[kU], s2[kU];
        double wv[kU];
        int64_t p1[kU], p2[kU];
        bool v[kU], v2[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t e = e0 + (int64_t)u * blockDim.x;
            v[u] = e < E;
            r[u] = v[u] ? (unsigned)rows[e] : 0u;
            c[u] = v[u] ? (unsigned)cols[e] : 0u;
            wv[u] = v[u] ? load_w(w, wt, e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            v2[u] = v[u] && !directed && r[u] != c[u];
            s1[u] = v[u] ? atomicAdd(&cursor[r[u]], 1u) : 0u;
            s2[u] = v2[u] ? atomicAdd(&cursor[c[u]], 1u) : 0u;
            p1[u] = v[u] ? slot_ptr[r[u]] : 0;
            p2[u] = v2[u] ? slot_ptr[c[u]] : 0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t e = e0 + (int64_t)u * blockDim.x;
            if (v[u]) {
                key[p1[u] + s1[u]] = ((unsigned long long)c[u] << 32) | (unsigned long long)e;
                if (wt != GEE_W_UNIT) val[p1[u] + s1[u]] = wv[u];
            }
            if (v2[u]) {
                key[p2[u] + s2[u]] = ((unsigned long long)r[u] << 32) | (unsigned long long)(E + e);
                if (wt != GEE_W_UNIT) val[p2[u] + s2[u]] = wv[u];
            }
        }
    }
}

__global__ void k_scatter_part(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols,
                               const void *__restrict__ w, int wt, int64_t E, int directed,
                               int n_rows, const int64_t *__restrict__ slot_ptr,
                               const unsigned *__restrict__ part,
                               unsigned long long *__restrict__ key, double *__restrict__ val) {
    extern __shared__ unsigned cur[];
    const unsigned *off = part + (size_t)blockIdx.x * n_rows;
    for (int r = threadIdx.x; r < n_rows; r += blockDim.x)
        cur[r] = (unsigned)(slot_ptr[r] + off[r]);
    __syncthreads();
    int64_t e0, e1;
    chunk_of(E, e0, e1);
    for (int64_t b = e0; b < e1; b += blockDim.x) {
        int64_t e = b + threadIdx.x;
        bool v = e < e1;
        unsigned r = 0, c = 0;
        double wv = 0.0;
        if (v) {
            r = (unsigned)rows[e];
            c = (unsigned)cols[e];
            wv = load_w(w, wt, e);
        }
        unsigned p1 = warp_agg_take(cur, r, v);
        if (v) {
            key[p1] = ((unsigned long long)c << 32) | (unsigned long long)e;
            if (wt != GEE_W_UNIT) val[p1] = wv;
        }
        bool v2 = v && !directed && r != c;
        unsigned p2 = warp_agg_take(cur, c, v2);
        if (v2) {
            key[p2] = ((unsigned long long)r << 32) | (unsigned long long)(E + e);
            if (wt != GEE_W_UNIT) val[p2] = wv;
        }
    }
}

// ---------------------------------------------------------------------------
// Row classification into work lists (tier S is implicit: every row <= 32).
// ---------------------------------------------------------------------------
__global__ void k_classify(const int64_t *__restrict__ slot_ptr, int64_t n_rows, int dense_ok,
                           int64_t n_cols, unsigned *__restrict__ lists, unsigned *__restrict__ nlist) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n_rows + 31) & ~int64_t(31);
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_round; r += stride) {
        int tier = -1;
        if (r < n_rows) {
            int64_t L = slot_ptr[r + 1] - slot_ptr[r];
            if (L > 32) {
                if (dense_ok && (L * 16 >= n_cols || L > kCap))
                    tier = TIER_D;
                else if (L <= kMCap)
                    tier = TIER_M;
                else if (L <= kCap)
                    tier = TIER_B;
                else
                    tier = TIER_X;
            }
        }
        unsigned k = tier >= 0 ? (unsigned)tier : 0xffffffffu;
        unsigned peers = __match_any_sync(0xffffffffu, k);
        int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (tier >= 0 && (int)(threadIdx.x & 31) == leader) base = atomicAdd(&nlist[tier], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (tier >= 0)
            lists[(size_t)tier * n_rows + base + __popc(peers & lanemask_lt())] = (unsigned)r;
    }
}

// ---------------------------------------------------------------------------
// Row assembly (persistent kernel).
// ---------------------------------------------------------------------------
struct RowsArgs {
    const int64_t *slot_ptr;
    int64_t n_rows, n_cols;
    int colbits, idxbits;     // bits of a column index, of a stream index
    unsigned long long *key;  // scattered buckets (input)
    double *val;
    unsigned long long *key2;  // global staging / LSD ping-pong
    double *val2;
    int unit;  // unit weights: bucket values are implicit 1.0 and never stored
    const void *w;  // the input weights (tier B gathers values by stream index)
    int wt;
    int64_t E;
    int32_t *out_col;  // unique entries at slot positions
    double *out_val;
    unsigned *ucnt;
    const unsigned *lists;  // [kTiers][n_rows]
    const unsigned *nlist;  // [kTiers]
    unsigned *work;         // [5] work counters
    unsigned deg_flags;
    double *deg;
    double *scale;
    int32_t *err;
    int dense_ok;
};

// a bucket entry's value
__device__ __forceinline__ double bval(const RowsArgs &a, int64_t p) { return a.unit ? 1.0 : a.val[p]; }

struct RowsShared {
    unsigned ured[33];
    double dred[33];
    int ired[33];
    int task;
};

__device__ __forceinline__ void store_degree(const RowsArgs &a, int64_t r, double d) {
    a.deg[r] = d;
    if (a.scale) a.scale[r] = laplacian_scale(d, a.err);
}

// Finish a row whose L entries sit sorted by column in (sk, sv); when
// `fixup`, equal-column runs are still in arbitrary idx order.  Sums runs in
// stream order, drops zeros, writes the unique entries at the row's slot
// start, and folds the degree.  Whole CTA.
__device__ void finish_row(const RowsArgs &a, RowsShared &sm, int64_t r, int64_t s0, int L,
                           unsigned long long *sk, double *sv, bool fixup, int32_t *scol, double *sval) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int per = (L + nt - 1) / nt;
    const int p0 = min(L, tid * per), p1 = min(L, p0 + per);
    unsigned nkeep = 0;
    for (int p = p0; p < p1; ++p) {
        unsigned c = (unsigned)(sk[p] >> 32);
        if (p > 0 && (unsigned)(sk[p - 1] >> 32) == c) continue;
        // run end: a short linear probe, then binary search (the keys are
        // sorted by column), so a hub's run of thousands of repeats costs
        // log2(L) dependent loads instead of one per repeat
        int q = p + 1;
        while (q < L && q < p + 8 && (unsigned)(sk[q] >> 32) == c) ++q;
        if (q == p + 8 && q < L && (unsigned)(sk[q] >> 32) == c) {
            int lo = q, hi = L;  // sk[lo] has column c; find the first index with a larger column
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if ((unsigned)(sk[mid] >> 32) == c)
                    lo = mid;
                else
                    hi = mid;
            }
            q = hi;
        }
        if (fixup && q - p >= 3) {
            // the run back into idx (stream) order: Shell sort with Ciura's
            // gaps, so the long duplicate runs of power-law hubs (thousands of
            // repeats of one pair) stay O(n^1.3) for the one thread that owns them
            const int gaps[9] = {1750, 701, 301, 132, 57, 23, 10, 4, 1};
            for (int gi = 0; gi < 9; ++gi) {
                const int gap = gaps[gi];
                if (gap >= q - p) continue;
                for (int i = p + gap; i < q; ++i) {
                    const unsigned long long kk = sk[i];
                    const double vv = sv[i];
                    int j = i;
                    while (j - gap >= p && sk[j - gap] > kk) {
                        sk[j] = sk[j - gap];
                        sv[j] = sv[j - gap];
                        j -= gap;
                    }
                    sk[j] = kk;
                    sv[j] = vv;
                }
            }
        }
        double acc = sv[p];
#pragma unroll 8
        for (int i = p + 1; i < q; ++i) acc += sv[i];  // stream order; loads run ahead of the adds
        sv[p] = acc;
        nkeep += acc != 0.0;
    }
    __syncthreads();
    unsigned total;
    unsigned off = block_exclusive_scan(nkeep, sm.ured, &total);
    const bool want_deg = a.deg_flags != 0;
    const bool diag = (a.deg_flags & GEE_DIAGONAL) != 0;
    Cert cert;
    double psum = 0.0;
    int placed = 0;
    for (int p = p0; p < p1; ++p) {
        unsigned c = (unsigned)(sk[p] >> 32);
        if (p > 0 && (unsigned)(sk[p - 1] >> 32) == c) continue;
        double acc = sv[p];
        if (acc == 0.0) continue;
        a.out_col[s0 + off] = (int32_t)c;
        a.out_val[s0 + off] = acc;
        ++off;
        if (want_deg) {
            double x = acc;
            if (diag && (int64_t)c == r) {
                x = acc + 1.0;
                placed = 1;
            }
            cert.add(x);
            psum += x;
        }
    }
    if (tid == 0) a.ucnt[r] = total;
    if (!want_deg) return;
    placed = __syncthreads_or(placed);
    const bool insert = diag && !placed;
    int mlow = block_min(cert.mlow, sm.ired);
    double sabs = block_sum(cert.sabs, sm.dred) + (insert ? 1.0 : 0.0);
    if (insert) mlow = min(mlow, 0);
    if (cert_ok(mlow, sabs)) {
        double d = block_sum(psum, sm.dred) + (insert ? 1.0 : 0.0);
        if (tid == 0) store_degree(a, r, d);
    } else {
        // the sequential fold in column order (sparse.py:196): the CTA stages
        // the row's output kCap entries at a time in shared memory (scol/sval,
        // free once the outputs are written) so thread 0 folds from shared
        // memory instead of one dependent global load per entry
        double d = 0.0;
        bool ins = !insert;
        for (unsigned b = 0; b < total; b += kCap) {
            const unsigned nb = min((unsigned)kCap, total - b);
            __syncthreads();  // out_* writes visible; the previous chunk consumed
            for (unsigned i = tid; i < nb; i += nt) {
                scol[i] = a.out_col[s0 + b + i];
                sval[i] = a.out_val[s0 + b + i];
            }
            __syncthreads();
            if (tid == 0) {
                for (unsigned i = 0; i < nb; ++i) {
                    const int64_t c = scol[i];
                    double x = sval[i];
                    if (!ins && c > r) {
                        d += 1.0;
                        ins = true;
                    }
                    if (diag && c == r) x = x + 1.0;
                    d += x;
                }
            }
        }
        if (tid == 0) {
            if (!ins) d += 1.0;
            store_degree(a, r, d);
        }
    }
    __syncthreads();
}

// tier D: counting sort over the (small) column range; cnt in shared memory
__device__ void row_dense(const RowsArgs &a, RowsShared &sm, int64_t r, unsigned *cnt,
                          unsigned long long *stk, double *stv) {
    const int64_t s0 = a.slot_ptr[r];
    const int L = (int)(a.slot_ptr[r + 1] - s0);
    const int nc = (int)a.n_cols;
    const unsigned long long *key = a.key + s0;
    for (int c = threadIdx.x; c < nc; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < L; i += blockDim.x) atomicAdd(&cnt[(unsigned)(key[i] >> 32)], 1u);
    __syncthreads();
    {
        const int per = (nc + blockDim.x - 1) / blockDim.x;
        const int c0 = min(nc, (int)threadIdx.x * per), c1 = min(nc, c0 + per);
        unsigned s = 0;
        for (int c = c0; c < c1; ++c) s += cnt[c];
        unsigned run = block_exclusive_scan(s, sm.ured, nullptr);
        for (int c = c0; c < c1; ++c) {
            unsigned x = cnt[c];
            cnt[c] = run;
            run += x;
        }
    }
    __syncthreads();
    unsigned long long *sk = L <= kCap ? stk : a.key2 + s0;
    double *sv = L <= kCap ? stv : a.val2 + s0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        unsigned long long k = key[i];
        unsigned p = atomicAdd(&cnt[(unsigned)(k >> 32)], 1u);
        sk[p] = k;
        sv[p] = bval(a, s0 + i);
    }
    __syncthreads();
    finish_row(a, sm, r, s0, L, sk, sv, true, reinterpret_cast<int32_t *>(stk), stv);
}

// tier B: bitonic sort of (key, value) pairs padded to a power of two
// weight of stream entry idx (idx < E: original edge idx, else its reverse)
__device__ __forceinline__ double stream_w(const RowsArgs &a, unsigned long long idx) {
    if (a.wt == GEE_W_UNIT) return 1.0;
    const int64_t e = (int64_t)idx < a.E ? (int64_t)idx : (int64_t)idx - a.E;
    return load_w(a.w, a.wt, e);
}

// tier B: bitonic sort of the full keys (col << 32 | idx) of a row of
// 257..kCap entries, E = P/512 keys per thread in registers: partners within
// a thread are register swaps, within a warp shuffles, across warps one
// shared-memory exchange per stage.  Values are gathered after the sort from
// the weight array by stream index.
template <int E>
__device__ __forceinline__ void block_bitonic_keys(unsigned long long (&x)[E], unsigned long long *sk, int tid,
                                                   int lane) {
    constexpr int P = E * kRowsThreads;
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= kRowsThreads) {
                // partner in the same thread: element e ^ (j / 512), static indices
#pragma unroll
                for (int jj = 1; jj < E; jj <<= 1) {
                    if (j != jj * kRowsThreads) continue;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const int f = e ^ jj;
                        if (f > e) {
                            const bool asc = ((e * kRowsThreads + tid) & k) == 0;
                            const unsigned long long lo = min(x[e], x[f]), hi = max(x[e], x[f]);
                            x[e] = asc ? lo : hi;
                            x[f] = asc ? hi : lo;
                        }
                    }
                }
            } else if (j >= 32) {
                __syncthreads();  // previous readers of sk are done
#pragma unroll
                for (int e = 0; e < E; ++e) sk[e * kRowsThreads + tid] = x[e];
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = e * kRowsThreads + tid;
                    const unsigned long long y = sk[i ^ j];
                    const bool asc = (i & k) == 0, lower = (i & j) == 0;
                    x[e] = (lower == asc) ? min(x[e], y) : max(x[e], y);
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = e * kRowsThreads + tid;
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[e], j);
                    const bool asc = (i & k) == 0, lower = (i & j) == 0;
                    x[e] = (lower == asc) ? min(x[e], y) : max(x[e], y);
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) sk[e * kRowsThreads + threadIdx.x] = x[e];
    __syncthreads();
}

template <int E>
__device__ __forceinline__ void row_bitonic_e(const RowsArgs &a, int64_t s0, int L, unsigned long long *sk,
                                              double *sv) {
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * kRowsThreads + tid;
        x[e] = i < L ? a.key[s0 + i] : ~0ull;
    }
    block_bitonic_keys<E>(x, sk, tid, lane);
    for (int i = tid; i < L; i += kRowsThreads) sv[i] = stream_w(a, sk[i] & 0xffffffffull);
    __syncthreads();
}

__device__ void row_bitonic(const RowsArgs &a, RowsShared &sm, int64_t r, unsigned long long *sk,
                            double *sv) {
    const int64_t s0 = a.slot_ptr[r];
    const int L = (int)(a.slot_ptr[r + 1] - s0);
    if (L <= kRowsThreads)
        row_bitonic_e<1>(a, s0, L, sk, sv);
    else if (L <= 2 * kRowsThreads)
        row_bitonic_e<2>(a, s0, L, sk, sv);
    else if (L <= 4 * kRowsThreads)
        row_bitonic_e<4>(a, s0, L, sk, sv);
    else
        row_bitonic_e<8>(a, s0, L, sk, sv);
    finish_row(a, sm, r, s0, L, sk, sv, false, reinterpret_cast<int32_t *>(sk), sv);
}

// tier X: stable LSD radix (8-bit digits) over the column bits, one CTA per
// row, ping-ponging between the bucket and the staging arrays.
__device__ void row_lsd(const RowsArgs &a, RowsShared &sm, int64_t r, unsigned *hist, unsigned long long *stk,
                        double *stv) {
    const int64_t s0 = a.slot_ptr[r];
    const int L = (int)(a.slot_ptr[r + 1] - s0);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int chunk = (L + nw - 1) / nw;
    const int a0 = min(L, wid * chunk), a1 = min(L, a0 + chunk);
    unsigned long long *src = a.key + s0, *dst = a.key2 + s0;
    double *srcv = a.val + s0, *dstv = a.val2 + s0;
    if (a.unit) {
        for (int i = threadIdx.x; i < L; i += blockDim.x) srcv[i] = 1.0;
        __syncthreads();
    }
    // the full key (col << 32 | idx): idx digits first, then column digits,
    // so equal-column runs leave in stream order (hub rows of power-law
    // graphs carry runs of thousands of repeats; no per-run fix-up)
    const int ipasses = (a.idxbits + 7) / 8;
    const int passes = ipasses + (a.colbits + 7) / 8;
#ifdef GEE_TRACE
    const long long tl0 = clock64();
#endif
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = pass < ipasses ? 8 * pass : 32 + 8 * (pass - ipasses);
        unsigned *h = hist + wid * 256;
        for (int d = lane; d < 256; d += 32) h[d] = 0;
        __syncthreads();
        // warp-aggregated: a hub row's columns crowd a few digits, and one
        // shared atomic per distinct digit per 32 entries avoids serialising;
        // kLU chunks of keys are loaded before any is used (latency overlap)
        constexpr int kLU = 4;
        for (int b = a0; b < a1; b += 32 * kLU) {
            unsigned dd[kLU];
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const int i = b + u * 32 + lane;
                dd[u] = i < a1 ? ((unsigned)(src[i] >> shift) & 255u) : 256u + lane;
            }
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const unsigned peers = __match_any_sync(0xffffffffu, dd[u]);
                if (dd[u] < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[dd[u]], (unsigned)__popc(peers));
            }
        }
        __syncthreads();
        unsigned tot = 0;
        if (threadIdx.x < 256) {
            for (int w = 0; w < nw; ++w) {
                unsigned x = hist[w * 256 + threadIdx.x];
                hist[w * 256 + threadIdx.x] = tot;
                tot += x;
            }
        }
        unsigned base = block_exclusive_scan(threadIdx.x < 256 ? tot : 0u, sm.ured, nullptr);
        if (threadIdx.x < 256)
            for (int w = 0; w < nw; ++w) hist[w * 256 + threadIdx.x] += base;
        __syncthreads();
        for (int b = a0; b < a1; b += 32 * kLU) {
            unsigned long long kk[kLU];
            double xx[kLU];
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const int i = b + u * 32 + lane;
                kk[u] = i < a1 ? src[i] : 0ull;
                xx[u] = i < a1 ? srcv[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kLU; ++u) {
                const bool v = b + u * 32 + lane < a1;
                const unsigned d = v ? ((unsigned)(kk[u] >> shift) & 255u) : 256u + lane;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const unsigned pos = v ? h[d] + __popc(peers & lanemask_lt()) : 0u;
                __syncwarp();
                if (v) {
                    dst[pos] = kk[u];
                    dstv[pos] = xx[u];
                    if (lane == __ffs(peers) - 1) h[d] += __popc(peers);
                }
                __syncwarp();
            }
        }
        __syncthreads();
        unsigned long long *t = src;
        src = dst;
        dst = t;
        double *tv = srcv;
        srcv = dstv;
        dstv = tv;
    }
#ifdef GEE_TRACE
    const long long tf0 = clock64();
#endif
    finish_row(a, sm, r, s0, L, src, srcv, false, reinterpret_cast<int32_t *>(stk), stv);
#ifdef GEE_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 512 && L > (int)g_lsd_t[blockIdx.x][0]) {
        g_lsd_t[blockIdx.x][0] = L;
        g_lsd_t[blockIdx.x][1] = tf0 - tl0;
        g_lsd_t[blockIdx.x][2] = clock64() - tf0;
        g_lsd_t[blockIdx.x][3] = r;
    }
#endif
}

// tier S: one warp per row of <= 32 entries; rank sort by the full key
__device__ void row_small(const RowsArgs &a, int64_t r, unsigned long long *wk, double *wv) {
    const int lane = threadIdx.x & 31;
    const int64_t s0 = a.slot_ptr[r];
    const int L = (int)(a.slot_ptr[r + 1] - s0);
    unsigned long long k = ~0ull;
    double v = 0.0;
    if (lane < L) {
        k = a.key[s0 + lane];
        v = bval(a, s0 + lane);
    }
    int rank = 0;
    for (int j = 0; j < L; ++j) rank += __shfl_sync(0xffffffffu, k, j) < k;
    if (lane < L) {
        wk[rank] = k;
        wv[rank] = v;
    }
    __syncwarp();
    unsigned col = 0xffffffffu;
    double x = 0.0;
    if (lane < L) {
        col = (unsigned)(wk[lane] >> 32);
        x = wv[lane];
    }
    unsigned prev = __shfl_up_sync(0xffffffffu, col, 1);
    bool head = lane < L && (lane == 0 || prev != col);
    double acc = 0.0;
    if (head) {
        acc = x;
        for (int j = lane + 1; j < L && (unsigned)(wk[j] >> 32) == col; ++j) acc += wv[j];
    }
    bool keep = head && acc != 0.0;
    unsigned km = __ballot_sync(0xffffffffu, keep);
    if (keep) {
        int pos = __popc(km & lanemask_lt());
        a.out_col[s0 + pos] = (int32_t)col;
        a.out_val[s0 + pos] = acc;
    }
    if (lane == 0) a.ucnt[r] = __popc(km);
    if (a.deg_flags) {
        const bool diag = (a.deg_flags & GEE_DIAGONAL) != 0;
        double xm = 0.0;
        bool isd = false;
        if (keep) {
            xm = acc;
            if (diag && (int64_t)col == r) {
                xm = acc + 1.0;
                isd = true;
            }
        }
        const bool insert = diag && !__any_sync(0xffffffffu, isd);
        Cert ce;
        ce.add(xm);
        int mlow = warp_min(ce.mlow);
        double sabs = warp_sum(ce.sabs) + (insert ? 1.0 : 0.0);
        if (insert) mlow = min(mlow, 0);
        double d;
        if (cert_ok(mlow, sabs)) {
            d = warp_sum(xm) + (insert ? 1.0 : 0.0);
        } else {
            d = 0.0;
            bool ins = !insert;
            unsigned mm = km;
            while (mm) {
                int j = __ffs(mm) - 1;
                mm &= mm - 1;
                int64_t cj = (unsigned)__shfl_sync(0xffffffffu, col, j);
                double xj = __shfl_sync(0xffffffffu, xm, j);
                if (!ins && cj > r) {
                    d += 1.0;
                    ins = true;
                }
                d += xj;
            }
            if (!ins) d += 1.0;
        }
        if (lane == 0) store_degree(a, r, d);
    }
    __syncwarp();
}

// tier M: one warp per row of kMCap or fewer entries: bitonic sort of the
// full key (col << 32 | idx, so equal-column runs come out in stream order)
// in a per-warp shared slice, then the warp sums runs, drops zeros, writes the
// unique entries at the row's slot start and folds the degree.
// ascending bitonic sort of 32*E keys held striped in registers (element
// e*32 + lane in x[e]): partners across lanes by shuffles, within a lane by
// register swaps; no shared memory, no barriers
template <int E>
__device__ __forceinline__ void warp_sort_u32(unsigned (&x)[E], int lane) {
    constexpr int P = E * 32;
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int f = e ^ (j >> 5);
                    if (f > e) {
                        const bool asc = ((e * 32 + lane) & k) == 0;
                        const unsigned lo = min(x[e], x[f]), hi = max(x[e], x[f]);
                        x[e] = asc ? lo : hi;
                        x[f] = asc ? hi : lo;
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const unsigned y = __shfl_xor_sync(0xffffffffu, x[e], j);
                    const bool asc = ((e * 32 + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    x[e] = (lower == asc) ? min(x[e], y) : max(x[e], y);
                }
            }
        }
    }
}

// sort the row by (col, bucket position) in registers, then gather the full
// entries into the warp's shared slice in that order
template <int E>
__device__ __forceinline__ void row_medium_sort(const RowsArgs &a, int64_t s0, int L, unsigned long long *wk,
                                                double *wv, int lane) {
    unsigned x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * 32 + lane;
        x[e] = i < L ? ((unsigned)(a.key[s0 + i] >> 32) << 8) | (unsigned)i : 0xffffffffu;
    }
    warp_sort_u32<E>(x, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = e * 32 + lane;
        if (i < L) {
            const int pos = (int)(x[e] & 255u);
            wk[i] = a.key[s0 + pos];
            wv[i] = bval(a, s0 + pos);
        }
    }
}

// tier M: one warp per row of kMCap or fewer entries.  Columns < 2^24: a
// register bitonic sort of (col << 8 | position); equal-column runs of >= 3
// are then put back into stream order (runs of 2 sum commutatively).
// Otherwise a shared-memory bitonic sort of the full key (col << 32 | idx).
// The warp then sums runs, drops zeros, writes the unique entries at the
// row's slot start and folds the degree.
__device__ void row_medium(const RowsArgs &a, int64_t r, unsigned long long *wk, double *wv) {
    const int lane = threadIdx.x & 31;
    const int64_t s0 = a.slot_ptr[r];
    const int L = (int)(a.slot_ptr[r + 1] - s0);
    const bool regsort = a.colbits <= 24;
    if (regsort) {
        if (L <= 64)
            row_medium_sort<2>(a, s0, L, wk, wv, lane);
        else if (L <= 128)
            row_medium_sort<4>(a, s0, L, wk, wv, lane);
        else
            row_medium_sort<8>(a, s0, L, wk, wv, lane);
        __syncwarp();
    } else {
        int P = 64;
        while (P < L) P <<= 1;
        for (int i = lane; i < P; i += 32) {
            wk[i] = i < L ? a.key[s0 + i] : ~0ull;
            wv[i] = i < L ? bval(a, s0 + i) : 0.0;
        }
        __syncwarp();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < P; i += 32) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long x = wk[i], y = wk[ixj];
                        if ((x > y) == ((i & k) == 0)) {
                            wk[i] = y;
                            wk[ixj] = x;
                            const double t = wv[i];
                            wv[i] = wv[ixj];
                            wv[ixj] = t;
                        }
                    }
                }
                __syncwarp();
            }
        }
    }
    const bool want_deg = a.deg_flags != 0;
    const bool diag = (a.deg_flags & GEE_DIAGONAL) != 0;
    unsigned base = 0;
    Cert cert;
    double psum = 0.0;
    bool placed = false;
    for (int c0 = 0; c0 < L; c0 += 32) {
        const int i = c0 + lane;
        const bool v = i < L;
        const unsigned col = v ? (unsigned)(wk[i] >> 32) : 0xffffffffu;
        const bool head = v && (i == 0 || (unsigned)(wk[i - 1] >> 32) != col);
        double acc = 0.0;
        if (head) {
            int q = i + 1;
            while (q < L && (unsigned)(wk[q] >> 32) == col) ++q;
            if (regsort && q - i >= 3) {
                // a run of repeats: back into stream (idx) order
                for (int m = i + 1; m < q; ++m) {
                    const unsigned long long kk = wk[m];
                    const double vv = wv[m];
                    int j = m - 1;
                    while (j >= i && wk[j] > kk) {
                        wk[j + 1] = wk[j];
                        wv[j + 1] = wv[j];
                        --j;
                    }
                    wk[j + 1] = kk;
                    wv[j + 1] = vv;
                }
            }
            acc = wv[i];
            for (int j = i + 1; j < q; ++j) acc += wv[j];  // stream order
        }
        const bool keep = head && acc != 0.0;
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const unsigned pos = base + __popc(km & lanemask_lt());
            a.out_col[s0 + pos] = (int32_t)col;
            a.out_val[s0 + pos] = acc;
            if (want_deg) {
                double x = acc;
                if (diag && (int64_t)col == r) {
                    x = acc + 1.0;
                    placed = true;
                }
                cert.add(x);
                psum += x;
            }
        }
        base += __popc(km);
    }
    if (lane == 0) a.ucnt[r] = base;
    if (!want_deg) return;
    const bool insert = diag && !__any_sync(0xffffffffu, placed);
    int mlow = warp_min(cert.mlow);
    double sabs = warp_sum(cert.sabs) + (insert ? 1.0 : 0.0);
    if (insert) mlow = min(mlow, 0);
    if (cert_ok(mlow, sabs)) {
        const double d = warp_sum(psum) + (insert ? 1.0 : 0.0);
        if (lane == 0) store_degree(a, r, d);
    } else {
        __syncwarp();  // the warp's out_* writes visible to lane 0
        if (lane == 0) {
            double d = 0.0;
            bool ins = !insert;
            for (unsigned i = 0; i < base; ++i) {
                const int64_t c = a.out_col[s0 + i];
                double x = a.out_val[s0 + i];
                if (!ins && c > r) {
                    d += 1.0;
                    ins = true;
                }
                if (diag && c == r) x = x + 1.0;
                d += x;
            }
            if (!ins) d += 1.0;
            store_degree(a, r, d);
        }
    }
    __syncwarp();
}

#ifdef GEE_TRACE
__device__ unsigned long long g_phase_t[512][6];
__device__ unsigned long long g_rows_t[4096][3];
__device__ unsigned g_rows_n;
#define ROWS_TRACE_BEGIN() long long _t0 = clock64();
#define ROWS_TRACE_END(tier, row) \
    if (threadIdx.x == 0) { unsigned _i = atomicAdd(&g_rows_n, 1u); if (_i < 4096) { g_rows_t[_i][0] = tier; g_rows_t[_i][1] = row; g_rows_t[_i][2] = clock64() - _t0; } }
#else
#define ROWS_TRACE_BEGIN()
#define ROWS_TRACE_END(tier, row)
#endif
__global__ void __launch_bounds__(kRowsThreads, 2) k_rows(RowsArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ RowsShared sm;
    unsigned long long *stk = reinterpret_cast<unsigned long long *>(dsm);
    double *stv = reinterpret_cast<double *>(dsm + sizeof(unsigned long long) * kCap);
    unsigned *region2 = reinterpret_cast<unsigned *>(dsm + 16 * kCap);
    const int n_x = (int)a.nlist[TIER_X], n_d = (int)a.nlist[TIER_D], n_b = (int)a.nlist[TIER_B];
    const int n_m = (int)a.nlist[TIER_M];
    const unsigned *lx = a.lists + (size_t)TIER_X * a.n_rows;
    const unsigned *ld = a.lists + (size_t)TIER_D * a.n_rows;
    const unsigned *lb = a.lists + (size_t)TIER_B * a.n_rows;
#ifdef GEE_TRACE
    if (threadIdx.x == 0 && blockIdx.x < 512) g_phase_t[blockIdx.x][0] = clock64();
#define PHASE_MARK(k) if (threadIdx.x == 0 && blockIdx.x < 512) g_phase_t[blockIdx.x][k] = clock64();
#else
#define PHASE_MARK(k)
#endif
    // phase X: hub rows first (longest critical path)
    for (;;) {
        if (threadIdx.x == 0) sm.task = (int)atomicAdd(&a.work[0], 1u);
        __syncthreads();
        int t = sm.task;
        __syncthreads();
        if (t >= n_x) break;
        ROWS_TRACE_BEGIN();
        row_lsd(a, sm, lx[t], region2, stk, stv);
        ROWS_TRACE_END(2, lx[t]);
    }
    PHASE_MARK(1);
    for (;;) {
        if (threadIdx.x == 0) sm.task = (int)atomicAdd(&a.work[1], 1u);
        __syncthreads();
        int t = sm.task;
        __syncthreads();
        if (t >= n_d) break;
        row_dense(a, sm, ld[t], region2, stk, stv);
    }
    for (;;) {
        if (threadIdx.x == 0) sm.task = (int)atomicAdd(&a.work[2], 1u);
        __syncthreads();
        int t = sm.task;
        __syncthreads();
        if (t >= n_b) break;
        ROWS_TRACE_BEGIN();
        row_bitonic(a, sm, lb[t], stk, stv);
        ROWS_TRACE_END(1, lb[t]);
    }
    PHASE_MARK(2);
    // phase M: one warp per row, warps grab rows independently
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    {
        const unsigned *lm = a.lists + (size_t)TIER_M * a.n_rows;
        unsigned long long *mk = stk + wid * kMCap;
        double *mv = stv + wid * kMCap;
        // rows are grabbed kMChunk at a time: one counter shared by every
        // warp of the grid would otherwise serialise 10^5 atomics
        constexpr int kMChunk = 16;
        for (;;) {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(&a.work[4], (unsigned)kMChunk);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_m) break;
            for (int u = t; u < min(n_m, t + kMChunk); ++u) row_medium(a, lm[u], mk, mv);
        }
    }
    __syncthreads();
    PHASE_MARK(3);
    // phase S: every warp grabs its own chunks of rows (no CTA barrier per
    // chunk: row lengths vary), one warp per row, rows > 32 skipped
    unsigned long long *wk = stk + wid * 32;
    double *wv = stv + wid * 32;
    const int64_t n_chunks = (a.n_rows + kSChunk - 1) / kSChunk;
    for (;;) {
        unsigned tw = 0;
        if (lane == 0) tw = atomicAdd(&a.work[3], 1u);
        const int64_t t = __shfl_sync(0xffffffffu, tw, 0);
        if (t >= n_chunks) break;
        const int64_t r0 = t * kSChunk, r1 = min(a.n_rows, r0 + kSChunk);
        for (int64_t r = r0; r < r1; ++r) {
            int64_t L = a.slot_ptr[r + 1] - a.slot_ptr[r];
            if (L > 32) continue;
            if (L == 0) {
                if (lane == 0) {
                    a.ucnt[r] = 0;
                    if (a.deg_flags) store_degree(a, r, (a.deg_flags & GEE_DIAGONAL) ? 1.0 : 0.0);
                }
                continue;
            }
            row_small(a, r, wk, wv);
        }
    }
    PHASE_MARK(4);
    (void)nw;
}

// ---------------------------------------------------------------------------
// Optional compaction into a standard CSR (to_csr() callers).
// ---------------------------------------------------------------------------
__global__ void k_compact(const int64_t *__restrict__ slot_ptr, const unsigned *__restrict__ ucnt,
                          const int64_t *__restrict__ row_ptr, int64_t n_rows,
                          const int32_t *__restrict__ in_col, const double *__restrict__ in_val,
                          int32_t *__restrict__ out_col, double *__restrict__ out_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n_rows; r += nwarps) {
        int64_t s = slot_ptr[r], d = row_ptr[r];
        unsigned u = ucnt[r];
        for (unsigned i = lane; i < u; i += 32) {
            out_col[d + i] = in_col[s + i];
            out_val[d + i] = in_val[s + i];
        }
    }
}

__global__ void k_copy_back(const int64_t *__restrict__ nnz, const int32_t *__restrict__ in_col,
                            const double *__restrict__ in_val, int32_t *__restrict__ out_col,
                            double *__restrict__ out_val) {
    const int64_t n = *nnz;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        out_col[i] = in_col[i];
        out_val[i] = in_val[i];
    }
}

__global__ void k_copy_i64(const int64_t *__restrict__ in, int64_t n, int64_t *__restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

// ---------------------------------------------------------------------------
// Host orchestration.
// ---------------------------------------------------------------------------
struct CsrWs {
    unsigned *cnt;
    int64_t *slot_ptr;
    int64_t *tmp_ptr;
    unsigned *part;
    unsigned *lists;
    unsigned *nlist;  // [kTiers] tier counts, then the work counters
    unsigned *ucnt;
    unsigned long long *key, *key2;
    double *val, *val2;
    void *scan_ws;
    int G;
};

static int partition_ctas() { return 2 * num_sms(); }

static size_t carve_csr(Carver &cv, CsrWs &w, int64_t E, int64_t n_rows, int directed) {
    const int64_t M = directed ? E : 2 * E;
    const int64_t Mc = M > 0 ? M : 1;
    w.G = partition_ctas();
    w.cnt = cv.take<unsigned>((size_t)n_rows + 1);
    w.slot_ptr = cv.take<int64_t>((size_t)n_rows + 1);
    w.tmp_ptr = cv.take<int64_t>((size_t)n_rows + 1);
    w.part = n_rows <= kSmallRows ? cv.take<unsigned>((size_t)w.G * (size_t)(n_rows + 1)) : nullptr;
    w.lists = cv.take<unsigned>((size_t)kTiers * (size_t)(n_rows + 1));
    w.nlist = cv.take<unsigned>(16);
    w.ucnt = cv.take<unsigned>((size_t)n_rows + 1);
    w.key = cv.take<unsigned long long>((size_t)Mc);
    w.val = cv.take<double>((size_t)Mc);
    w.key2 = cv.take<unsigned long long>((size_t)Mc);
    w.val2 = cv.take<double>((size_t)Mc);
    w.scan_ws = cv.take<char>(scan_workspace(n_rows + 1));
    return cv.bytes();
}

bool sort_path_ok(int64_t E, int64_t n_rows, int64_t n_cols, int directed, int wt);
size_t sort_workspace(int64_t E, int64_t n_rows, int64_t n_cols, int directed);
int sort_csr_build(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int64_t n_rows,
                   int64_t n_cols, int directed, int force_vals, int64_t *row_ptr, int32_t *col, double *val,
                   int64_t *nnz, unsigned deg_flags, double *deg, double *scale, void *ws, size_t ws_bytes,
                   unsigned **val_mode, int32_t *err, cudaStream_t st);

// the weight type is not known here: room for whichever path csr_build picks
bool sort_fits(int64_t E, int64_t n_rows, int64_t n_cols, int directed);

// workspace for any assembly path the test hooks may select (the plan's size
// must not depend on the hook state at query time)
size_t csr_build_workspace_any(int64_t E, int64_t n_rows, int64_t n_cols, int directed) {
    size_t need = sort_fits(E, n_rows, n_cols, directed) ? sort_workspace(E, n_rows, n_cols, directed) : 0;
    Carver cv(nullptr);
    CsrWs w;
    const size_t b = carve_csr(cv, w, E, n_rows, directed);
    return need > b ? need : b;
}

size_t csr_build_workspace(int64_t E, int64_t n_rows, int64_t n_cols, int directed) {
    size_t need = 0;
    if (sort_path_ok(E, n_rows, n_cols, directed, -1)) need = sort_workspace(E, n_rows, n_cols, directed);
    if (!sort_path_ok(E, n_rows, n_cols, directed, GEE_W_UNIT)) {
        Carver cv(nullptr);
        CsrWs w;
        const size_t b = carve_csr(cv, w, E, n_rows, directed);
        need = need > b ? need : b;
    }
    return need;
}

__global__ void k_row_cnt(const int64_t *__restrict__ row_ptr, int64_t n, unsigned *__restrict__ cnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
        cnt[r] = (unsigned)(row_ptr[r + 1] - row_ptr[r]);
}

static int bit_length(int64_t x) {
    int b = 0;
    while (x > 0) {
        ++b;
        x >>= 1;
    }
    return b;
}

static size_t rows_smem(int dense_ok, int64_t n_cols) {
    size_t region2 = 16 * 256 * sizeof(unsigned);  // LSD per-warp histograms
    if (dense_ok) region2 = region2 > (size_t)n_cols * 4 ? region2 : (size_t)n_cols * 4;
    return 16 * (size_t)kCap + region2;
}

int csr_build(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E,
              int64_t n_rows, int64_t n_cols, int directed, int compact, int64_t *row_ptr,
              unsigned *row_cnt, int32_t *col, double *val, int64_t *nnz, unsigned deg_flags,
              double *deg, double *scale, void *ws, size_t ws_bytes, int32_t *err,
              cudaStream_t st) {
    if (sort_path_ok(E, n_rows, n_cols, directed, wt)) {
        // packed (row, col) keys: radix-sort path, always a compact CSR
        int rc = sort_csr_build(rows, cols, w, wt, E, n_rows, n_cols, directed, 1, row_ptr, col, val, nnz,
                                deg_flags, deg, scale, ws, ws_bytes, nullptr, err, st);
        if (rc) return rc;
        if (row_cnt && n_rows > 0) {
            k_row_cnt<<<grid_for(n_rows, 256, 8), 256, 0, st>>>(row_ptr, n_rows, row_cnt);
            GEE_CHECK_LAUNCH("k_row_cnt");
        }
        return GEE_OK;
    }
    Carver cv(ws);
    CsrWs W;
    size_t need = carve_csr(cv, W, E, n_rows, directed);
    if (ws_bytes < need) return GEE_E_WORKSPACE;
    const int threads = 512;
    const bool small_rows = n_rows <= kSmallRows;
    static PerDevice part_attr;
    if (!part_attr.done()) {
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_count_part, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kSmallRows * 4));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_scatter_part, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            kSmallRows * 4));
        part_attr.mark();
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(W.nlist, 0, 16 * sizeof(unsigned), st));
    GEE_CHECK_CUDA(cudaMemsetAsync(W.cnt, 0, sizeof(unsigned) * (size_t)(n_rows + 1), st));
    // pass 1: counts
    if (E > 0) {
        if (small_rows) {
            size_t smem = sizeof(unsigned) * (size_t)n_rows;
            k_count_part<<<W.G, threads, smem, st>>>(rows, cols, E, directed, (int)n_rows, W.part);
            GEE_CHECK_LAUNCH("k_count_part");
            k_part_reduce<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(W.part, W.G, (int)n_rows,
                                                                           W.cnt);
            GEE_CHECK_LAUNCH("k_part_reduce");
        } else {
            k_count_global<<<grid_for(E, threads, 4), threads, 0, st>>>(rows, cols, E, directed, W.cnt);
            GEE_CHECK_LAUNCH("k_count_global");
        }
    }
    int rc = exclusive_scan_u32(W.cnt, n_rows, W.slot_ptr, W.scan_ws, st);
    if (rc) return rc;
    // pass 2: scatter into row buckets
    if (E > 0) {
        if (small_rows) {
            size_t smem = sizeof(unsigned) * (size_t)n_rows;
            k_scatter_part<<<W.G, threads, smem, st>>>(rows, cols, w, wt, E, directed, (int)n_rows,
                                                       W.slot_ptr, W.part, W.key, W.val);
            GEE_CHECK_LAUNCH("k_scatter_part");
        } else {
            GEE_CHECK_CUDA(cudaMemsetAsync(W.cnt, 0, sizeof(unsigned) * (size_t)(n_rows + 1), st));
            k_scatter_global<<<grid_for(E, threads, 4), threads, 0, st>>>(
                rows, cols, w, wt, E, directed, W.slot_ptr, W.cnt, W.key, W.val);
            GEE_CHECK_LAUNCH("k_scatter_global");
        }
    }
    // classify + assemble rows
    const int dense_ok = n_cols <= kSmallCols;
    if (n_rows > 0) {
        k_classify<<<grid_for(n_rows, 256, 8), 256, 0, st>>>(W.slot_ptr, n_rows, dense_ok, n_cols,
                                                            W.lists, W.nlist);
        GEE_CHECK_LAUNCH("k_classify");
        RowsArgs a;
        a.slot_ptr = W.slot_ptr;
        a.n_rows = n_rows;
        a.n_cols = n_cols;
        a.colbits = bit_length(n_cols > 1 ? n_cols - 1 : 1);
        a.idxbits = bit_length(2 * E > 1 ? 2 * E - 1 : 1);
        a.key = W.key;
        a.val = W.val;
        a.key2 = W.key2;
        a.val2 = W.val2;
        a.unit = wt == GEE_W_UNIT;
        a.w = w;
        a.wt = wt;
        a.E = E;
        a.out_col = col;
        a.out_val = val;
        a.ucnt = compact ? W.ucnt : row_cnt;
        a.lists = W.lists;
        a.nlist = W.nlist;
        a.work = W.nlist + kTiers;
        a.deg_flags = deg_flags;
        a.deg = deg;
        a.scale = (deg_flags & GEE_LAPLACIAN) ? scale : nullptr;
        a.err = err;
        a.dense_ok = dense_ok;
        size_t smem = rows_smem(dense_ok, n_cols);
        static PerDevice attr_set;
        if (!attr_set.done()) {
            GEE_CHECK_CUDA(cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                16 * kCap + kSmallCols * 4 + 1024));
            attr_set.mark();
        }
        k_rows<<<2 * num_sms(), kRowsThreads, smem, st>>>(a);
        GEE_CHECK_LAUNCH("k_rows");
    }
    if (compact) {
        unsigned *uc = W.ucnt;
        rc = exclusive_scan_u32(uc, n_rows, row_ptr, W.scan_ws, st);
        if (rc) return rc;
        if (row_cnt) GEE_CHECK_CUDA(cudaMemcpyAsync(row_cnt, uc, sizeof(unsigned) * (size_t)n_rows,
                                                    cudaMemcpyDeviceToDevice, st));
        int32_t *tcol = reinterpret_cast<int32_t *>(W.key);
        double *tval = W.val;
        if (n_rows > 0) {
            k_compact<<<grid_for(n_rows * 32, 256, 8), 256, 0, st>>>(W.slot_ptr, uc, row_ptr, n_rows,
                                                                    col, val, tcol, tval);
            GEE_CHECK_LAUNCH("k_compact");
            const int64_t M = directed ? E : 2 * E;
            k_copy_back<<<grid_for(M > 0 ? M : 1, 256, 8), 256, 0, st>>>(row_ptr + n_rows, tcol, tval,
                                                                        col, val);
            GEE_CHECK_LAUNCH("k_copy_back");
        }
        if (nnz) GEE_CHECK_CUDA(cudaMemcpyAsync(nnz, row_ptr + n_rows, sizeof(int64_t),
                                                cudaMemcpyDeviceToDevice, st));
    } else {
        k_copy_i64<<<grid_for(n_rows + 1, 256, 8), 256, 0, st>>>(W.slot_ptr, n_rows + 1, row_ptr);
        GEE_CHECK_LAUNCH("k_copy_i64");
        if (nnz) {
            // nnz = sum of unique counts
            rc = exclusive_scan_u32(row_cnt, n_rows, W.tmp_ptr, W.scan_ws, st);
            if (rc) return rc;
            GEE_CHECK_CUDA(cudaMemcpyAsync(nnz, W.tmp_ptr + n_rows, sizeof(int64_t),
                                           cudaMemcpyDeviceToDevice, st));
        }
    }
    return GEE_OK;
}

#ifdef GEE_TRACE
extern "C" int gee_lsd_dump(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_lsd_t, sizeof(g_lsd_t)) == cudaSuccess ? 0 : -1;
}
extern "C" int gee_phase_dump(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_phase_t, sizeof(g_phase_t)) == cudaSuccess ? 0 : -1;
}
extern "C" int gee_rows_dump(unsigned long long *out, unsigned *n) {
    cudaMemcpyFromSymbol(n, g_rows_n, sizeof(unsigned));
    unsigned z = 0;
    cudaMemcpyToSymbol(g_rows_n, &z, sizeof(unsigned));
    return cudaMemcpyFromSymbol(out, g_rows_t, sizeof(g_rows_t)) == cudaSuccess ? 0 : -1;
}
#endif
}  // namespace gee
