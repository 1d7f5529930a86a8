// k_bitmap.cu -- K2 for unit-weight graphs with at most kBmMax nodes
// (configs 0/1: unweighted SBM, N = 10^4).
//
// With every weight equal to 1.0 a stored value is just the multiplicity of
// its (row, col) pair and the order duplicates are summed in is irrelevant
// (sums of ones are exact), so the CSR of a row is the sorted set of its
// distinct columns and its degree is its stream length.  Rows are grouped in
// buckets of kRB = 32; every symmetrised stream entry becomes one 32-bit word
// (row % 32) << 16 | col.
//   k_cb_count    CTA-private bucket histograms of contiguous edge chunks
//   k_cb_offsets  one CTA per bucket: each chunk's offset inside the bucket;
//                 the last CTA scans the bucket totals
//   k_cb_scatter  tiles of 1024 edges are counting-sorted by bucket in shared
//                 memory, so every bucket's fragment leaves as one coalesced
//                 burst (no scattered 2-byte stores)
//   k_cb_rows     one CTA per bucket streams its entries once (coalesced),
//                 sets the 32 rows' column bitmaps in shared memory, then
//                 emits each row's columns in order: output position o is
//                 mapped to its bitmap word by binary search over per-word
//                 popc prefixes and to its bit by a 5-step popc select, so
//                 consecutive lanes store consecutive columns.  Duplicates
//                 (bitmap bit already set) give the row multiplicities in val
//                 and a per-row flag for gee_embed.  The same pass writes the
//                 degree (stream length, +1 under A+I), the Laplacian scale,
//                 gee_embed's node records and its long-row list.
#include "gee_common.cuh"

namespace gee {

constexpr int kBmMax = 16384;  // nodes (bitmaps + prefixes: 2 x 32 x 512 words)
constexpr int kRB = 32;        // rows per bucket
constexpr int kCbThreads = 512;
constexpr int kTileEdges = 1024;  // edges per scatter tile (<= 2048 entries)
constexpr int kRowsThreads = 512;

__device__ __forceinline__ void chunk_range(int64_t E, int64_t &e0, int64_t &e1) {
    e0 = (int64_t)((__int128)E * blockIdx.x / gridDim.x);
    e1 = (int64_t)((__int128)E * (blockIdx.x + 1) / gridDim.x);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCbThreads) k_cb_count(const int64_t *__restrict__ rows,
                                                          const int64_t *__restrict__ cols, int64_t E,
                                                          int directed, int B, unsigned *__restrict__ part) {
    extern __shared__ unsigned h[];
    for (int b = threadIdx.x; b < B; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int64_t e0, e1;
    chunk_range(E, e0, e1);
    constexpr int U = 4;
    for (int64_t base = e0; base < e1; base += (int64_t)blockDim.x * U) {
        unsigned r[U], c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = base + (int64_t)u * blockDim.x + threadIdx.x;
            r[u] = e < e1 ? (unsigned)__ldcs(rows + e) : 0u;
            c[u] = e < e1 ? (unsigned)__ldcs(cols + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = base + (int64_t)u * blockDim.x + threadIdx.x;
            const bool v = e < e1;
            // originals: rows often arrive in runs -> one atomic per run
            const unsigned bk = r[u] / kRB;
            const unsigned prev = __shfl_up_sync(0xffffffffu, bk, 1);
            const bool head = v && (lane == 0 || prev != bk);
            const unsigned heads = __ballot_sync(0xffffffffu, head);
            const int nv = __popc(__ballot_sync(0xffffffffu, v));
            if (head) {
                const unsigned after = heads & ~((2u << lane) - 1u);
                const int next = after ? __ffs(after) - 1 : nv;
                atomicAdd(&h[bk], (unsigned)(next - lane));
            }
            if (!directed && v && r[u] != c[u]) atomicAdd(&h[c[u] / kRB], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < B; b += blockDim.x) part[(size_t)blockIdx.x * B + b] = h[b];
}

// one CTA per bucket: part[g][b] -> exclusive prefix over chunks g; the last
// CTA scans the bucket totals into bstart[0..B] (bstart[B] = stream length)
__global__ void __launch_bounds__(1024) k_cb_offsets(unsigned *__restrict__ part, int G, int B,
                                                     unsigned *__restrict__ btot, unsigned *__restrict__ bstart,
                                                     unsigned *__restrict__ done) {
    __shared__ unsigned red[33];
    __shared__ bool last;
    const int b = blockIdx.x;
    unsigned run = 0;
    for (int g0 = 0; g0 < G; g0 += blockDim.x) {
        const int g = g0 + threadIdx.x;
        const unsigned x = g < G ? part[(size_t)g * B + b] : 0u;
        unsigned tot;
        const unsigned ex = block_exclusive_scan(x, red, &tot);
        if (g < G) part[(size_t)g * B + b] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) btot[b] = run;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    unsigned carry = 0;
    for (int b0 = 0; b0 < B; b0 += blockDim.x) {
        const int bb = b0 + threadIdx.x;
        const unsigned x = bb < B ? __ldcg(btot + bb) : 0u;
        unsigned tot;
        const unsigned ex = block_exclusive_scan(x, red, &tot);
        if (bb < B) bstart[bb] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        bstart[B] = carry;
        *done = 0;  // re-armed for the next launch / graph replay
    }
}

__global__ void __launch_bounds__(kCbThreads) k_cb_scatter(const int64_t *__restrict__ rows,
                                                            const int64_t *__restrict__ cols, int64_t E,
                                                            int directed, int B, const unsigned *__restrict__ bstart,
                                                            const unsigned *__restrict__ part,
                                                            unsigned *__restrict__ out) {
    extern __shared__ unsigned csm[];
    unsigned *cur = csm;                   // [B] next free slot of each bucket for this CTA
    unsigned *th = cur + B;                // [B] tile histogram
    unsigned *ts = th + B;                 // [B] tile bucket starts
    unsigned *stage = ts + B;              // [2 * kTileEdges]
    unsigned short *sb = reinterpret_cast<unsigned short *>(stage + 2 * kTileEdges);  // bucket of stage[i]
    __shared__ unsigned red[33];
    __shared__ unsigned s_ntile;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        cur[b] = bstart[b] + part[(size_t)blockIdx.x * B + b];
        th[b] = 0;
    }
    __syncthreads();
    int64_t e0, e1;
    chunk_range(E, e0, e1);
    constexpr int EPT = kTileEdges / kCbThreads;  // edges per thread per tile
    for (int64_t t0 = e0; t0 < e1; t0 += kTileEdges) {
        unsigned key[2 * EPT], bk[2 * EPT], rank[2 * EPT];
        bool ok[2 * EPT];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int64_t e = t0 + (int64_t)u * blockDim.x + threadIdx.x;
            const bool v = e < e1;
            const unsigned r = v ? (unsigned)__ldcs(rows + e) : 0u;
            const unsigned c = v ? (unsigned)__ldcs(cols + e) : 0u;
            ok[2 * u] = v;
            key[2 * u] = ((r % kRB) << 16) | c;
            bk[2 * u] = r / kRB;
            ok[2 * u + 1] = v && !directed && r != c;
            key[2 * u + 1] = ((c % kRB) << 16) | r;
            bk[2 * u + 1] = c / kRB;
        }
#pragma unroll
        for (int j = 0; j < 2 * EPT; ++j)
            if (ok[j]) rank[j] = atomicAdd(&th[bk[j]], 1u);
        __syncthreads();
        unsigned tot = 0;
        for (int b0 = 0; b0 < B; b0 += blockDim.x) {
            const int b = b0 + threadIdx.x;
            const unsigned x = b < B ? th[b] : 0u;
            unsigned t;
            const unsigned ex = block_exclusive_scan(x, red, &t);
            if (b < B) ts[b] = tot + ex;
            tot += t;
        }
        if (threadIdx.x == 0) s_ntile = tot;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 2 * EPT; ++j) {
            if (ok[j]) {
                const unsigned pos = ts[bk[j]] + rank[j];
                stage[pos] = key[j];
                sb[pos] = (unsigned short)bk[j];
            }
        }
        __syncthreads();
        const unsigned nt = s_ntile;
        for (unsigned i = threadIdx.x; i < nt; i += blockDim.x) {
            const unsigned b = sb[i];
            out[cur[b] + (i - ts[b])] = stage[i];
        }
        __syncthreads();
        for (int b = threadIdx.x; b < B; b += blockDim.x) {
            cur[b] += th[b];
            th[b] = 0;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
struct CbRowsArgs {
    const unsigned *bstart;
    const unsigned *entries;
    int n, B, words;
    int64_t *slot_ptr;
    int32_t *out_col;
    double *out_val;
    unsigned *row_cnt;
    unsigned char *row_flag;
    unsigned *has_multi;
    unsigned deg_flags;
    double *deg, *scale;
    int32_t *err;
    const int32_t *y32;
    const double *inv;
    unsigned laplacian;
    double2 *rec;
    unsigned *long_list, *n_long;
    int long_row;
};

// index of the k-th (0-based) set bit of w
__device__ __forceinline__ int select_bit(unsigned w, int k) {
    int pos = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned lo = w & ((1u << s) - 1u);
        const int c = __popc(lo);
        if (k >= c) {
            k -= c;
            w >>= s;
            pos += s;
        } else {
            w = lo;
        }
    }
    return pos;
}

__global__ void __launch_bounds__(kRowsThreads) k_cb_rows(CbRowsArgs a) {
    extern __shared__ unsigned rsm[];
    const int W = a.words;
    unsigned *bm = rsm;                 // [kRB][W] column bitmaps
    unsigned *pre = bm + kRB * W;       // [kRB][W] exclusive popc prefix per word
    __shared__ unsigned dupc[kRB], uniq[kRB], slen[kRB];
    __shared__ int64_t rstart[kRB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int b = blockIdx.x;
    const int row0 = b * kRB;
    const int nrows = min(kRB, a.n - row0);
    for (int i = threadIdx.x; i < kRB * W; i += blockDim.x) bm[i] = 0u;
    if (threadIdx.x < kRB) dupc[threadIdx.x] = 0;
    __syncthreads();
    // 1. stream the bucket once (coalesced) into the bitmaps
    const unsigned s0 = a.bstart[b], s1 = a.bstart[b + 1];
    for (unsigned i = s0 + threadIdx.x; i < s1; i += 4 * blockDim.x) {
        unsigned ev[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned j = i + u * blockDim.x;
            ev[u] = j < s1 ? __ldcs(a.entries + j) : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (ev[u] == 0xffffffffu) continue;
            const unsigned rl = ev[u] >> 16, c = ev[u] & 0xffffu;
            const unsigned bit = 1u << (c & 31);
            if (atomicOr(&bm[rl * W + (c >> 5)], bit) & bit) atomicAdd(&dupc[rl], 1u);
        }
    }
    __syncthreads();
    // 2. per row: word prefixes (one warp per row), distinct count, stream length
    for (int rl = wid; rl < nrows; rl += nw) {
        const unsigned *rb = bm + rl * W;
        unsigned *rp = pre + rl * W;
        unsigned carry = 0;
        for (int w0 = 0; w0 < W; w0 += 32) {
            const int w = w0 + lane;
            const unsigned c = w < W ? __popc(rb[w]) : 0u;
            unsigned incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (w < W) rp[w] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            uniq[rl] = carry;
            slen[rl] = carry + dupc[rl];
        }
    }
    __syncthreads();
    // 3. slot pointers of the bucket's rows (stream-length prefix) + per-row outputs
    if (threadIdx.x == 0) {
        int64_t run = s0;
        for (int rl = 0; rl < nrows; ++rl) {
            rstart[rl] = run;
            run += slen[rl];
        }
        if (row0 + nrows == a.n) a.slot_ptr[a.n] = run;
    }
    __syncthreads();
    if (threadIdx.x < nrows) {
        const int rl = threadIdx.x, r = row0 + rl;
        const unsigned u = uniq[rl], L = slen[rl];
        a.slot_ptr[r] = rstart[rl];
        a.row_cnt[r] = u;
        a.row_flag[r] = dupc[rl] ? 1 : 0;
        if (dupc[rl]) atomicOr(a.has_multi, 1u);
        double sr = 1.0;
        if (a.deg_flags) {
            const double d = (double)L + ((a.deg_flags & GEE_DIAGONAL) ? 1.0 : 0.0);
            a.deg[r] = d;
            if (a.scale) {
                sr = laplacian_scale(d, a.err);
                a.scale[r] = sr;
            }
        }
        if (a.rec) {
            const int lab = a.y32[r];
            const double g = lab < 0 ? 0.0 : (a.laplacian ? sr * a.inv[lab] : a.inv[lab]);
            a.rec[r] = make_double2(__longlong_as_double((long long)(unsigned)lab), g);
        }
        if (a.long_list && (int)u > a.long_row) a.long_list[atomicAdd(a.n_long, 1u)] = (unsigned)r;
    }
    // 4. emission: consecutive lanes store consecutive columns of a row
    for (int rl = wid; rl < nrows; rl += nw) {
        const unsigned *rb = bm + rl * W;
        const unsigned *rp = pre + rl * W;
        const unsigned u = uniq[rl];
        int32_t *dst = a.out_col + rstart[rl];
        for (unsigned o = lane; o < u; o += 32) {
            int lo = 0, hi = W - 1;  // last word with prefix <= o
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (rp[mid] <= o) lo = mid; else hi = mid - 1;
            }
            dst[o] = lo * 32 + select_bit(rb[lo], (int)(o - rp[lo]));
        }
    }
    // 5. rare: rows with duplicates get their multiplicities as values
    __syncthreads();
    bool anydup = false;
    for (int rl = 0; rl < nrows; ++rl) anydup |= dupc[rl] != 0;
    if (!anydup) return;
    for (int rl = wid; rl < nrows; rl += nw)
        if (dupc[rl])
            for (unsigned o = lane; o < uniq[rl]; o += 32) a.out_val[rstart[rl] + o] = 0.0;
    __syncthreads();
    for (unsigned i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
        const unsigned ev = a.entries[i];
        const unsigned rl = ev >> 16, c = ev & 0xffffu;
        if (!dupc[rl]) continue;
        const unsigned w = c >> 5;
        const unsigned rank = pre[rl * W + w] + __popc(bm[rl * W + w] & ((1u << (c & 31)) - 1u));
        atomicAdd(&a.out_val[rstart[rl] + rank], 1.0);
    }
}

// ---------------------------------------------------------------------------
int force_path();

bool bitmap_path_ok(int wt, int64_t E, int64_t n_rows, int64_t n_cols, int directed) {
    if (force_path() != 0) return false;  // test hook: exercise the general paths
    const int64_t M = directed ? E : 2 * E;
    return wt == GEE_W_UNIT && n_rows == n_cols && n_rows >= 1 && n_rows <= kBmMax && M < ((int64_t)1 << 31);
}

struct BmWs {
    unsigned *part, *btot, *bstart, *flags, *entries;
    int G, B;
};

static void carve_bm(Carver &cv, BmWs &w, int64_t E, int64_t n, int directed) {
    const int64_t M = directed ? E : 2 * E;
    w.G = 2 * num_sms();  // two 512-thread CTAs per SM for count/scatter
    w.B = (int)((n + kRB - 1) / kRB);
    w.part = cv.take<unsigned>((size_t)w.G * (size_t)w.B);
    w.btot = cv.take<unsigned>((size_t)w.B);
    w.bstart = cv.take<unsigned>((size_t)w.B + 1);
    w.flags = cv.take<unsigned>(4);  // [0] has_multi, [2] done
    w.entries = cv.take<unsigned>((size_t)(M > 0 ? M : 1));
}

size_t bitmap_workspace(int64_t E, int64_t n, int directed) {
    Carver cv(nullptr);
    BmWs w;
    carve_bm(cv, w, E, n, directed);
    return cv.bytes();
}

// Unit-weight CSR in the slot layout: row r's distinct columns at
// [slot_ptr[r], slot_ptr[r] + row_cnt[r]); multiplicities in val only for
// rows with row_flag[r] != 0.  row_ptr receives the slot pointers.  Also
// emits the embed's node records and long-row list (rec/long_list/n_long,
// n_long zeroed by the caller) so gee_embed needs no preparation launches.
int bitmap_csr_build(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed,
                     int64_t *row_ptr, unsigned *row_cnt, unsigned char *row_flag, int32_t *col, double *val,
                     unsigned deg_flags, double *deg, double *scale, const int32_t *y32, const double *inv,
                     unsigned laplacian, double2 *rec, unsigned *long_list, unsigned *n_long, int long_row,
                     void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, E, n, directed);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    const int words = (int)((n + 31) / 32);
    const size_t rows_smem = sizeof(unsigned) * 2 * kRB * (size_t)words;
    const size_t scat_smem = sizeof(unsigned) * (3 * (size_t)W.B + 2 * kTileEdges) + sizeof(unsigned short) * 2 * kTileEdges;
    static bool attr = false;
    if (!attr) {
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_cb_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(unsigned) * 2 * kRB * (kBmMax / 32))));
        attr = true;
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(W.flags, 0, 4 * sizeof(unsigned), st));
    if (E > 0) {
        k_cb_count<<<W.G, kCbThreads, sizeof(unsigned) * (size_t)W.B, st>>>(rows, cols, E, directed, W.B, W.part);
        GEE_CHECK_LAUNCH("k_cb_count");
        k_cb_offsets<<<W.B, 512, 0, st>>>(W.part, W.G, W.B, W.btot, W.bstart, W.flags + 2);
        GEE_CHECK_LAUNCH("k_cb_offsets");
        k_cb_scatter<<<W.G, kCbThreads, scat_smem, st>>>(rows, cols, E, directed, W.B, W.bstart, W.part, W.entries);
        GEE_CHECK_LAUNCH("k_cb_scatter");
    } else {
        GEE_CHECK_CUDA(cudaMemsetAsync(W.bstart, 0, sizeof(unsigned) * (size_t)(W.B + 1), st));
    }
    CbRowsArgs a;
    a.bstart = W.bstart;
    a.entries = W.entries;
    a.n = (int)n;
    a.B = W.B;
    a.words = words;
    a.slot_ptr = row_ptr;
    a.out_col = col;
    a.out_val = val;
    a.row_cnt = row_cnt;
    a.row_flag = row_flag;
    a.has_multi = W.flags;
    a.deg_flags = deg_flags;
    a.deg = deg;
    a.scale = (deg_flags & GEE_LAPLACIAN) ? scale : nullptr;
    a.err = err;
    a.y32 = y32;
    a.inv = inv;
    a.laplacian = laplacian;
    a.rec = rec;
    a.long_list = long_list;
    a.n_long = n_long;
    a.long_row = long_row;
    k_cb_rows<<<W.B, kRowsThreads, rows_smem, st>>>(a);
    GEE_CHECK_LAUNCH("k_cb_rows");
    return GEE_OK;
}

}  // namespace gee
