// k_bitmap.cu -- K2 for unit-weight graphs with at most kBmMax nodes
// (configs 0/1: unweighted SBM, N = 10^4).
//
// With every weight equal to 1.0 a stored value is just the multiplicity of
// its (row, col) pair and the order duplicates are summed in is irrelevant
// (sums of ones are exact), so the CSR of a row is the sorted set of its
// distinct columns.  The B200 layout:
//   k_bm_count    CTA-private row histograms of contiguous edge chunks
//   k_bm_reduce   per-row totals + each chunk's offset inside every row
//   (scan)        row slot pointers
//   k_bm_scatter  each chunk writes its entries' 16-bit columns into the row
//                 buckets (2 bytes per entry: the whole bucket array is
//                 ~22 MB at cfg 1 and stays in L2, so partial-sector writes
//                 merge on chip instead of read-modify-writing HBM)
//   k_bm_rows     one warp per row: set the row's columns in a warp-private
//                 shared-memory bitmap (N bits), then emit them in column
//                 order with popc prefix sums -- no comparison sort at all.
//                 Duplicates are detected by the bitmap (atomicOr returns the
//                 old word); such rows also get their multiplicities in val
//                 and a per-row flag telling gee_embed to read them.
//   degree        the row's stream length (+1 under A+I): exact.
#include "gee_common.cuh"

namespace gee {

int exclusive_scan_u32(const unsigned *in, int64_t n, int64_t *out, void *ws, cudaStream_t st);
size_t scan_workspace(int64_t n);

constexpr int kBmMax = 16384;       // nodes (bitmap 2 KB + prefix 2 KB per warp)
constexpr int kBmThreads = 1024;
constexpr int kBmRowsThreads = 256;

// warp run-length aggregation of ctr[key] += 1 for lanes in `valid`
// (valid lanes are a prefix of the warp); returns this lane's slot
__device__ __forceinline__ unsigned rle_take(unsigned *ctr, unsigned key, bool valid, int nv, bool want_slot) {
    const int lane = threadIdx.x & 31;
    const unsigned prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = valid && (lane == 0 || prev != key);
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    unsigned base = 0;
    if (head) {
        const unsigned after = heads & ~((2u << lane) - 1u);
        const int next = after ? __ffs(after) - 1 : nv;
        base = atomicAdd(&ctr[key], (unsigned)(next - lane));
    }
    if (!want_slot) return 0;
    // my head = highest head lane <= me
    const unsigned upto = heads & (0xffffffffu >> (31 - lane));
    const int hl = upto ? 31 - __clz(upto) : 0;
    const unsigned hb = __shfl_sync(0xffffffffu, base, hl);
    return hb + (unsigned)(lane - hl);
}

__device__ __forceinline__ void chunk_range(int64_t E, int64_t &e0, int64_t &e1) {
    e0 = (int64_t)((__int128)E * blockIdx.x / gridDim.x);
    e1 = (int64_t)((__int128)E * (blockIdx.x + 1) / gridDim.x);
}

constexpr int kBmUnroll = 4;  // edges per thread per iteration (loads issued together)

__global__ void __launch_bounds__(kBmThreads) k_bm_count(const int64_t *__restrict__ rows,
                                                          const int64_t *__restrict__ cols, int64_t E,
                                                          int directed, int n, unsigned *__restrict__ part) {
    extern __shared__ unsigned h[];
    for (int r = threadIdx.x; r < n; r += blockDim.x) h[r] = 0;
    __syncthreads();
    int64_t e0, e1;
    chunk_range(E, e0, e1);
    for (int64_t b = e0; b < e1; b += (int64_t)blockDim.x * kBmUnroll) {
        unsigned r[kBmUnroll], c[kBmUnroll];
#pragma unroll
        for (int u = 0; u < kBmUnroll; ++u) {
            const int64_t e = b + (int64_t)u * blockDim.x + threadIdx.x;
            r[u] = e < e1 ? (unsigned)__ldcs(rows + e) : 0u;
            c[u] = e < e1 ? (unsigned)__ldcs(cols + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kBmUnroll; ++u) {
            const int64_t e = b + (int64_t)u * blockDim.x + threadIdx.x;
            const bool v = e < e1;
            const int nv = __popc(__ballot_sync(0xffffffffu, v));
            rle_take(h, r[u], v, nv, false);
            // reversed entries: their rows are the (random) columns
            if (!directed && v && r[u] != c[u]) atomicAdd(&h[c[u]], 1u);
        }
    }
    __syncthreads();
    unsigned *dst = part + (size_t)blockIdx.x * n;
    for (int r = threadIdx.x; r < n; r += blockDim.x) dst[r] = h[r];
}

// part[g][r] -> exclusive prefix over g (each chunk's offset inside row r);
// cnt[r] = total.  A CTA takes 32 consecutive rows: the [G x 32] tile is
// staged in shared memory with coalesced loads (consecutive threads read
// consecutive rows of one chunk), warp w scans row w across the chunks, and
// the tile is written back coalesced.  The last CTA to finish also turns cnt
// into the slot pointers (exclusive scan, n <= 16384), so no separate scan
// launches are needed.
__global__ void __launch_bounds__(1024) k_bm_reduce(unsigned *__restrict__ part, int G, int n,
                                                    unsigned *__restrict__ cnt, int64_t *__restrict__ slot_ptr,
                                                    unsigned *__restrict__ done) {
    extern __shared__ unsigned tile[];  // [G][33]
    __shared__ unsigned red[33];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = blockIdx.x * 32;
    const int nr = min(32, n - r0);
#pragma unroll 4
    for (int i = threadIdx.x; i < G * 32; i += blockDim.x) {
        const int g = i >> 5, c = i & 31;
        tile[g * 33 + c] = c < nr ? __ldcg(part + (size_t)g * n + r0 + c) : 0u;
    }
    __syncthreads();
    {
        unsigned run = 0;
        for (int g0 = 0; g0 < G; g0 += 32) {
            const int g = g0 + lane;
            const unsigned x = g < G ? tile[g * 33 + wid] : 0u;
            unsigned incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (g < G) tile[g * 33 + wid] = run + incl - x;
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0 && wid < nr) cnt[r0 + wid] = run;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * 32; i += blockDim.x) {
        const int g = i >> 5, c = i & 31;
        if (c < nr) part[(size_t)g * n + r0 + c] = tile[g * 33 + c];
    }
    // last-CTA-done: the final CTA sees every cnt[] and scans them
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int q0 = min(n, (int)threadIdx.x * per), q1 = min(n, q0 + per);
    unsigned s = 0;
    for (int r = q0; r < q1; ++r) s += __ldcg(cnt + r);
    unsigned tot;
    unsigned run = block_exclusive_scan(s, red, &tot);
    for (int r = q0; r < q1; ++r) {
        slot_ptr[r] = run;
        run += __ldcg(cnt + r);
    }
    if (threadIdx.x == 0) {
        slot_ptr[n] = tot;
        *done = 0;  // reusable by the next launch / graph replay
    }
}

__global__ void __launch_bounds__(kBmThreads) k_bm_scatter(const int64_t *__restrict__ rows,
                                                            const int64_t *__restrict__ cols, int64_t E,
                                                            int directed, int n,
                                                            const int64_t *__restrict__ slot_ptr,
                                                            const unsigned *__restrict__ part,
                                                            unsigned short *__restrict__ colbuf) {
    extern __shared__ unsigned cur[];
    const unsigned *off = part + (size_t)blockIdx.x * n;
    for (int r = threadIdx.x; r < n; r += blockDim.x) cur[r] = (unsigned)(slot_ptr[r] + off[r]);
    __syncthreads();
    int64_t e0, e1;
    chunk_range(E, e0, e1);
    for (int64_t b = e0; b < e1; b += (int64_t)blockDim.x * kBmUnroll) {
        unsigned r[kBmUnroll], c[kBmUnroll];
#pragma unroll
        for (int u = 0; u < kBmUnroll; ++u) {
            const int64_t e = b + (int64_t)u * blockDim.x + threadIdx.x;
            r[u] = e < e1 ? (unsigned)__ldcs(rows + e) : 0u;
            c[u] = e < e1 ? (unsigned)__ldcs(cols + e) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kBmUnroll; ++u) {
            const int64_t e = b + (int64_t)u * blockDim.x + threadIdx.x;
            const bool v = e < e1;
            const int nv = __popc(__ballot_sync(0xffffffffu, v));
            const unsigned p = rle_take(cur, r[u], v, nv, true);
            if (v) colbuf[p] = (unsigned short)c[u];
            if (!directed && v && r[u] != c[u]) colbuf[atomicAdd(&cur[c[u]], 1u)] = (unsigned short)r[u];
        }
    }
}

struct BmRowsArgs {
    const int64_t *slot_ptr;
    const unsigned short *colbuf;
    int n;
    int words;  // ceil(n / 32)
    int32_t *out_col;
    double *out_val;
    unsigned *row_cnt;
    unsigned char *row_flag;
    unsigned *has_multi;
    unsigned deg_flags;
    double *deg, *scale;
    int32_t *err;
    // embed inputs produced here (one pass over rows): node records and the
    // list of long rows gee_embed hands to whole CTAs
    const int32_t *y32;
    const double *inv;
    unsigned laplacian;
    double2 *rec;
    double *tab_g;          // compact node table for gee_embed's shared-memory copy
    signed char *tab_lab;
    unsigned *long_list, *n_long;
    int long_row;
};

constexpr int kBmStage = 1536;  // per-warp staging of a row's sorted columns

__global__ void __launch_bounds__(kBmRowsThreads) k_bm_rows(BmRowsArgs a) {
    extern __shared__ unsigned bsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int W = a.words;
    unsigned *bm = bsm + (size_t)wid * (2 * W + kBmStage);  // bitmap
    unsigned *pre = bm + W;                                 // exclusive popc prefix per word
    unsigned *stage = pre + W;                              // sorted columns of the row
    const int wpl = (W + 31) / 32;                          // words per lane in the emission
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < a.n; r += nwarps) {
        const int64_t s = a.slot_ptr[r];
        const int L = (int)(a.slot_ptr[r + 1] - s);
        for (int i = lane; i < W; i += 32) bm[i] = 0u;
        __syncwarp();
        // set bits with non-returning shared atomics (RED); duplicates show up
        // as fewer distinct columns than stream entries (u < L), so no
        // per-entry old-value check is needed
        for (int i0 = lane; i0 < L; i0 += 128) {
            unsigned c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + 32 * u;
                c[u] = i < L ? (unsigned)a.colbuf[s + i] : 0xffffffffu;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c[u] != 0xffffffffu) atomicOr(&bm[c[u] >> 5], 1u << (c[u] & 31));
        }
        __syncwarp();
        // emission: lane l owns words [l*wpl, (l+1)*wpl); set bits leave in
        // column order, staged in shared memory so the global write coalesces
        const int w0 = min(W, lane * wpl), w1 = min(W, w0 + wpl);
        unsigned cnt = 0;
        for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        unsigned off = incl - cnt;
        const unsigned u = __shfl_sync(0xffffffffu, incl, 31);
        const bool staged = u <= (unsigned)kBmStage;
        for (int w = w0; w < w1; ++w) {
            unsigned word = bm[w];
            pre[w] = off;
            while (word) {
                const int b = __ffs(word) - 1;
                word &= word - 1;
                if (staged)
                    stage[off] = w * 32 + b;
                else
                    a.out_col[s + off] = w * 32 + b;
                ++off;
            }
        }
        __syncwarp();
        if (staged)
            for (unsigned i = lane; i < u; i += 32) a.out_col[s + i] = (int32_t)stage[i];
        const bool multi = u < (unsigned)L;
        if (lane == 0) {
            a.row_cnt[r] = u;
            a.row_flag[r] = multi ? 1 : 0;
        }
        if (multi) {
            // multiplicities of the distinct columns (sums of ones, exact)
            __syncwarp();
            for (unsigned i = lane; i < u; i += 32) a.out_val[s + i] = 0.0;
            __syncwarp();
            for (int i = lane; i < L; i += 32) {
                const unsigned c = a.colbuf[s + i];
                const unsigned rank = pre[c >> 5] + __popc(bm[c >> 5] & ((1u << (c & 31)) - 1u));
                atomicAdd(&a.out_val[s + rank], 1.0);
            }
            if (lane == 0) atomicOr(a.has_multi, 1u);
        }
        if (lane == 0) {
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
                if (a.tab_g) {
                    a.tab_g[r] = g;
                    a.tab_lab[r] = (signed char)lab;
                }
            }
            if (a.long_list && (int)u > a.long_row) a.long_list[atomicAdd(a.n_long, 1u)] = (unsigned)r;
        }
        __syncwarp();
    }
}

int force_path();

bool bitmap_path_ok(int wt, int64_t E, int64_t n_rows, int64_t n_cols, int directed) {
    if (force_path() != 0) return false;  // test hook: exercise the general paths
    const int64_t M = directed ? E : 2 * E;
    return wt == GEE_W_UNIT && n_rows == n_cols && n_rows >= 1 && n_rows <= kBmMax && M < ((int64_t)1 << 31);
}

struct BmWs {
    unsigned *part, *cnt, *flags;
    int64_t *slot_ptr;
    unsigned short *colbuf;
    int G;
};

static void carve_bm(Carver &cv, BmWs &w, int64_t E, int64_t n, int directed) {
    const int64_t M = directed ? E : 2 * E;
    w.G = num_sms();  // one 1024-thread CTA per SM for count/scatter
    w.part = cv.take<unsigned>((size_t)w.G * (size_t)n);
    w.cnt = cv.take<unsigned>((size_t)n + 1);
    w.flags = cv.take<unsigned>(4);
    w.slot_ptr = cv.take<int64_t>((size_t)n + 1);
    w.colbuf = cv.take<unsigned short>((size_t)(M > 0 ? M : 1));
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
                     unsigned laplacian, double2 *rec, double *tab_g, signed char *tab_lab,
                     unsigned *long_list, unsigned *n_long, int long_row,
                     void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, E, n, directed);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    static bool attr = false;
    if (!attr) {
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_count, cudaFuncAttributeMaxDynamicSharedMemorySize, kBmMax * 4));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kBmMax * 4));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (kBmRowsThreads / 32) * (2 * (kBmMax / 32) + kBmStage) * 4));
        attr = true;
    }
    GEE_CHECK_CUDA(cudaMemsetAsync(W.flags, 0, 4 * sizeof(unsigned), st));
    const size_t hsm = sizeof(unsigned) * (size_t)n;
    if (E > 0) {
        k_bm_count<<<W.G, kBmThreads, hsm, st>>>(rows, cols, E, directed, (int)n, W.part);
        GEE_CHECK_LAUNCH("k_bm_count");
        k_bm_reduce<<<(unsigned)((n + 31) / 32), 1024, sizeof(unsigned) * 33 * (size_t)W.G, st>>>(
            W.part, W.G, (int)n, W.cnt, row_ptr, W.flags + 2);
        GEE_CHECK_LAUNCH("k_bm_reduce_scan");
        k_bm_scatter<<<W.G, kBmThreads, hsm, st>>>(rows, cols, E, directed, (int)n, row_ptr, W.part, W.colbuf);
        GEE_CHECK_LAUNCH("k_bm_scatter");
    } else {
        GEE_CHECK_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1), st));
    }
    BmRowsArgs a;
    a.slot_ptr = row_ptr;
    a.colbuf = W.colbuf;
    a.n = (int)n;
    a.words = (int)((n + 31) / 32);
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
    a.tab_g = tab_g;
    a.tab_lab = tab_lab;
    a.long_list = long_list;
    a.n_long = n_long;
    a.long_row = long_row;
    const size_t rsm = (size_t)(kBmRowsThreads / 32) * (2 * (size_t)a.words + kBmStage) * 4;
    k_bm_rows<<<grid_for(n * 32, kBmRowsThreads, 8), kBmRowsThreads, rsm, st>>>(a);
    GEE_CHECK_LAUNCH("k_bm_rows");
    return GEE_OK;
}

}  // namespace gee
