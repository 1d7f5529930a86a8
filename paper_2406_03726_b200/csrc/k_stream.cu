// k_stream.cu -- the bucketed stream encode: edge list -> Z without a CSR.
//
// Replaces the reference timed region encode(EdgeList(...).to_csr(), Y, opts)
// (cli.py:170-180; embedding.py:110-131) for graphs whose weights are all
// >= 0 -- the unit-weight and U(0,1] configurations of BASELINE.json.  With
// no negative weight, every degree and every Z entry is a sum of
// non-negative terms, so any summation order is within a few ulp of the
// reference's sequential folds (the 1e-12 bar), and the
// sorted, de-duplicated CSR the reference builds (_kernels.py:73-130) is not
// needed for Z: duplicates contribute the sum of their terms whether merged
// first or not, and a merged run is pruned only when it is exactly zero,
// i.e. when it contributes nothing.  (Signed weights need the reference's
// exact fold order for degrees near cancellation; they take the CSR path.
// The caller asserts non-negativity with GEE_NONNEG -- the EdgeList checks
// it at construction -- and a violation raises GEE_ERR_NEG_WEIGHT.)
//
// Stream entries are the symmetrised list of graph_io.py:82-88 (originals,
// plus the mirror of every off-diagonal edge of an undirected list).  Rows
// are grouped into BUCKETS of R = 2^lrow_bits consecutive rows, R*K*8 bytes
// of Z being one shared-memory tile; the bucket id has sub_bits bits.
//
//   k_st_hist1   8-bit MSD digit of the bucket id: shared-memory histogram
//   k_st_scan1   digit bases
//   k_st_part1   partition by that digit: each 4096-entry tile is ranked with
//                shared-memory atomics, reserves its digit runs with one global
//                atomic per digit, is reordered in shared memory and written
//                as coalesced runs: (row << 32 | col) + weight
//   k_st_hist2   bucket histogram: tiles of the digit-ordered list span few
//                digits, so a 2048-bin shared window covers them
//   k_st_scan2   bucket bases; work items = buckets cut into <= C entries
//   k_st_part2   partition into buckets (same tile scheme):
//                ((row mod R) << col_bits | col) + weight, 4 + w bytes
//   k_st_degree  per item: row degrees in shared memory (per-warp copies);
//                a bucket's last item writes d, s = 1/sqrt(d) and the node
//                record {Y_r, g_r = s_r / n_{Y_r}}; split buckets combine
//                through global f64 reductions and zero their Z rows
//   k_st_embed   per item: the R x K Z tile in shared memory; per entry one
//                16-byte node-record gather and one shared f64 add of w * g_j;
//                epilogue: + g_r on the diagonal (A+I), * s_r (Laplacian),
//                row L2 normalisation (correlation), one contiguous streaming
//                store of the tile.  Split buckets reduce into Z and their
//                last item runs the epilogue in place.
//
// Every pass is a coalesced stream; the only scattered traffic is the node
// record gather (L2-resident for skewed graphs) and global atomics at tile /
// item granularity.  No CUB, no sort library.
#include <type_traits>

#include "gee_common.cuh"

namespace gee {

int label_hist_pipeline(const int64_t *labels, int64_t n, int32_t k, int32_t *y32, int64_t *counts, double *inv_nk,
                        unsigned *partial, unsigned *done, int32_t *err, cudaStream_t st);
size_t label_partial_words(int64_t n, int k);

namespace {

constexpr int kStNT = 512;            // partition / histogram threads
constexpr int kStTile = 4096;         // entries per partition tile
constexpr int kStWin = 2048;          // shared bins of the bucket window
constexpr int kEmbNT = 512;           // embed threads (upper bound)
constexpr int kDegNT = 256;           // degree threads (8 warps, a work item each)
constexpr int kEmbWarps = kEmbNT / 32;
constexpr size_t kZTileMax = 104 * 1024;  // bytes of the R x K f64 Z tile (upper bound)
constexpr size_t kZTileDefault = 32 * 1024;  // default (A/B, profiles/r2_stream_ab.txt): several CTAs per SM hide item latency
constexpr size_t emb_stage_bytes(int nt, int u = 4) { return (size_t)2 * u * nt * 16; }  // two stages of u records per thread
int t_emb_nt = 128;  // threads of the embed CTA (the debug hook that chose 256 / 512 is retired)
constexpr unsigned kDegItem = 4096;  // entries per degree work item (one warp)
constexpr int kScanBlock = 4096;     // buckets per k_st_scan2 block (1024 threads x 4)
constexpr int kLrowMax = 9;  // at most 512 rows per bucket (per-warp degree copies: 64 KB)

int t_stream_mode = 0;  // debug hook: 0 auto, 1 never, >= 16 embed A/B variant

// debug phase trace of the embed (variant bit 16): per CTA, clock64 totals of
// [0] start-of-item wait, [1] accumulation, [2] tile barrier, [3] epilogue,
// [4] items, [5] entries
constexpr int kTraceSlots = 8;
__device__ unsigned long long g_emb_trace[4096 * kTraceSlots];
// The trace is compiled in only with -DGEE_EMBED_TRACE (make EXTRA=-DGEE_EMBED_TRACE):
// its running totals cost the embed ~8 registers it does not have (96 at 5 CTAs
// per SM; a spill of 48 bytes took configs[3]'s embed from 3.25 to 5.6 ms).
#ifdef GEE_EMBED_TRACE
#define GEE_TRACE_ON(x) (x)
#else
#define GEE_TRACE_ON(x) false
#endif
size_t t_ztile_bytes = kZTileDefault;  // debug hook: bytes of the R x K Z tile

struct StGeo {
    int64_t E, N;
    int64_t nloc;  // rows this call owns (row shard), N for a whole graph
    int directed, wt, k;
    unsigned flags;
    int lrow_bits, sub_bits, d1_bits, d2_bits, d1_shift, col_bits;
    unsigned S;   // buckets
    unsigned C;   // entries per work item
    int64_t Mcap; // entry capacity
    int64_t max_items;
    int64_t max_split;  // buckets with more than one item (> C entries)
};

__host__ __device__ __forceinline__ int bitlen64(int64_t x) {
    int b = 0;
    while (x > 0) {
        ++b;
        x >>= 1;
    }
    return b;
}

bool make_geo(StGeo &g, int64_t E, int64_t N, int directed, int wt, int k, unsigned flags, int64_t nloc = -1) {
    g.E = E;
    g.N = N;
    g.nloc = nloc < 0 ? N : nloc;
    if (g.nloc < 1) return false;
    g.directed = directed;
    g.wt = wt;
    g.k = k;
    g.flags = flags;
    const int rb = bitlen64(g.nloc - 1) > 0 ? bitlen64(g.nloc - 1) : 1;  // local row bits
    g.col_bits = bitlen64(N - 1) > 0 ? bitlen64(N - 1) : 1;
    int lr = 0;
    // row-in-bucket + column fit 31 bits: 0xffffffff is the embed's "no entry" key
    if (g.col_bits > 31) return false;
    const int lr_cap = kLrowMax < 31 - g.col_bits ? kLrowMax : 31 - g.col_bits;
    while (lr < rb && lr < lr_cap && (size_t)(2ll << lr) * (size_t)k * 8 <= t_ztile_bytes) ++lr;
    if ((size_t)(1ll << lr) * (size_t)k * 8 > t_ztile_bytes) return false;  // K too large for one row
    g.lrow_bits = lr;
    g.sub_bits = rb - lr;
    if (g.sub_bits < 1) {
        g.sub_bits = 1;
        g.lrow_bits = rb - 1 > 0 ? rb - 1 : 0;
    }
    g.d1_bits = g.sub_bits < 8 ? g.sub_bits : 8;
    g.d2_bits = g.sub_bits - g.d1_bits;
    if ((1 << g.d2_bits) > kStWin) return false;
    g.d1_shift = g.lrow_bits + g.d2_bits;
    if (g.lrow_bits + g.col_bits > 31) return false;
    g.S = (unsigned)(((g.nloc - 1) >> g.lrow_bits) + 1);
    g.Mcap = directed ? E : 2 * E;
    // work items of <= C entries, C ~ M / (16 SMs): a hub bucket (power-law
    // rows) splits over enough CTAs to finish with the rest (A/B: C / 4 took
    // configs[2]'s embed 0.41 -> 0.25 ms and configs[3]'s 3.43 -> 3.34 ms;
    // C / 16 lost again to the split-tile reductions)
    const int64_t per = g.Mcap / ((int64_t)num_sms() * 16);
    int64_t c = 4096;
    while (c < per && c < (1 << 16)) c <<= 1;
    g.C = (unsigned)c;
    g.max_items = (int64_t)g.S + g.Mcap / g.C + 1;
    g.max_split = g.Mcap / g.C + 1;
    return true;
}

struct StWs {
    unsigned *ctl;  // [0..255] hist1, [256..512] base1 (257), [520..775] cur1, [776] n_items, [777..779] work,
                    // [780] label done
    unsigned long long *keys1;
    void *w1;
    unsigned *hist2, *base2, *cur2, *item_off, *done_deg, *done_emb, *item_bucket, *split_slot;
    unsigned *ditem_off, *ditem_bucket;  // degree work items (<= kDegItem entries, a warp each)
    uint4 *item_desc;                    // embed work items {bucket, p0, p1, items of the bucket}
    unsigned *scan_part;                 // [blocks][4] partial sums of k_st_scan2a
    double *scratch;  // [max_split][R * K]: f64 partial tiles of split buckets
    uint32_t *keys2;
    void *w2;
    double *deg, *scale;
    double2 *rec;   // node record {bits of Y_r (-1 unlabeled), g_r = s_r / n_{Y_r}}
    double *zeros;  // a zeroed Z tile: source of the embed's bulk re-zeroing
    int32_t *y32;
    int64_t *counts;
    double *inv;
    unsigned *label_partial;
};
constexpr int kCtlHist1 = 0, kCtlBase1 = 256, kCtlCur1 = 520, kCtlItems = 776, kCtlWork = 777, kCtlLabel = 780,
              kCtlDItems = 781, kCtlSplit = 782, kCtlWLow = 783, kCtlWHigh = 784;
// kCtlWLow / kCtlWHigh: min over nonzero weights of the exponent of the lowest
// set bit, and max of ilogb(w) + 1 (both + kExpBias, so unsigned atomicMin/Max
// order them): every weight is a multiple of 2^low and below 2^high
constexpr int kCtlWords = 788;
constexpr int kExpBias = 4096;

size_t carve(Carver &cv, StWs &w, const StGeo &g) {
    const size_t wb = g.wt == GEE_W_F64 ? 8 : g.wt == GEE_W_F32 ? 4 : 0;
    const size_t M = (size_t)(g.Mcap > 0 ? g.Mcap : 1);
    w.ctl = cv.take<unsigned>(kCtlWords);
    w.keys1 = cv.take<unsigned long long>(M);
    w.w1 = wb ? (void *)cv.take<char>(M * wb) : nullptr;
    w.hist2 = cv.take<unsigned>((size_t)g.S + 1);
    w.base2 = cv.take<unsigned>((size_t)g.S + 1);
    w.cur2 = cv.take<unsigned>((size_t)g.S + 1);
    w.item_off = cv.take<unsigned>((size_t)g.S + 1);
    w.done_deg = cv.take<unsigned>((size_t)g.S + 1);
    w.done_emb = cv.take<unsigned>((size_t)g.S + 1);
    w.item_bucket = cv.take<unsigned>((size_t)g.max_items);
    w.split_slot = cv.take<unsigned>((size_t)g.S + 1);
    w.ditem_off = cv.take<unsigned>((size_t)g.S + 1);
    w.item_desc = cv.take<uint4>((size_t)g.max_items);
    w.ditem_bucket = cv.take<unsigned>((size_t)g.S + g.Mcap / kDegItem + 1);
    w.scan_part = cv.take<unsigned>(4 * ((size_t)g.S / kScanBlock + 2));
    w.scratch = cv.take<double>((size_t)g.max_split * ((size_t)1 << g.lrow_bits) * (size_t)g.k);
    w.keys2 = cv.take<uint32_t>(M);
    w.w2 = wb ? (void *)cv.take<char>(M * wb) : nullptr;
    w.deg = cv.take<double>((size_t)g.nloc);
    w.scale = cv.take<double>((size_t)g.N);
    w.rec = cv.take<double2>((size_t)g.N);
    w.zeros = cv.take<double>(((size_t)1 << g.lrow_bits) * (size_t)g.k + 2);
    w.y32 = cv.take<int32_t>((size_t)g.N + 1);
    w.counts = cv.take<int64_t>((size_t)g.k);
    w.inv = cv.take<double>((size_t)g.k);
    w.label_partial = cv.take<unsigned>(label_partial_words(g.N, g.k));
    return cv.bytes();
}

struct StArgs {
    const int64_t *rows, *cols;
    const void *w;
    int64_t E, N;
    int64_t row0, nloc;  // the rows [row0, row0 + nloc) this call owns
    double *deg_out;     // row-shard phase 1: raw local degrees (else nullptr)
    int directed, k;
    unsigned flags;
    int lrow_bits, d2_bits, d1_shift, col_bits;
    unsigned S, C;
    int variant;  // debug A/B (stream mode >= 16)
    int deg_copies;  // partial-sum copies per row in the degree kernel (power of two)
    unsigned long long magic;  // ceil(2^32 / K): row of a tile element by multiply-shift
    StWs ws;
    void *z;  // f64, or f32 under GEE_FP32
    int32_t *err;
};

// ---- entry helpers -----------------------------------------------------------
template <int WT>
struct WTraits;
template <>
struct WTraits<GEE_W_UNIT> {
    using T = char;  // unused
    static constexpr int bytes = 0;
};
template <>
struct WTraits<GEE_W_F32> {
    using T = float;
    static constexpr int bytes = 4;
};
template <>
struct WTraits<GEE_W_F64> {
    using T = double;
    static constexpr int bytes = 8;
};

// EdgeList validity (graph_io.py:65-72): an entry with an index outside
// [0, N) is raised and stored as a zero-weight entry so that every pass sees
// the same entry count; the row and column are repaired independently so a
// directed list's row (all the histogram reads) never changes.
__device__ __forceinline__ int64_t fix_index(int64_t x, int64_t N, bool &bad) {
    if (x < 0 || x >= N) {
        bad = true;
        return 0;
    }
    return x;
}

// A non-finite weight (graph_io.py:71-72) is raised and stored as 0.
// a row of this call's range -> its local index (out of range: raised, 0)
__device__ __forceinline__ int64_t fix_row(int64_t r, const StArgs &a, bool &bad) {
    r -= a.row0;
    if (r < 0 || r >= a.nloc) {
        bad = true;
        return 0;
    }
    return r;
}

template <int WT>
__device__ __forceinline__ void load_weight(const StArgs &a, int64_t i, typename WTraits<WT>::T &w, bool &badw,
                                            bool &neg) {
    if constexpr (WT != GEE_W_UNIT) {
        w = __ldg(reinterpret_cast<const typename WTraits<WT>::T *>(a.w) + i);
        if (!isfinite((double)w)) {
            badw = true;
            w = 0;
        } else if (w < 0) {
            neg = true;
        }
    }
}

// Exponent of the lowest set bit of |w| and an exclusive power-of-two bound
// (|w| < 2^hi), from the bits (w finite, nonzero).
__device__ __forceinline__ void weight_exponents(float w, int &lo, int &hi) {
    const unsigned b = __float_as_uint(w) & 0x7fffffffu;
    const int e = (int)(b >> 23);
    const unsigned m = b & 0x7fffffu;
    lo = e == 0 ? -150 + __ffs(m) : e - 151 + __ffs(m | 0x800000u);
    hi = e == 0 ? -126 : e - 126;
}
__device__ __forceinline__ void weight_exponents(double w, int &lo, int &hi) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(w) & 0x7fffffffffffffffull;
    const int e = (int)(b >> 52);
    const unsigned long long m = b & ((1ull << 52) - 1);
    lo = e == 0 ? -1075 + __ffsll((long long)m) : e - 1076 + __ffsll((long long)(m | (1ull << 52)));
    hi = e == 0 ? -1022 : e - 1022;
}
__device__ __forceinline__ void weight_exponents(char, int &lo, int &hi) { lo = hi = 0; }

// ---- pass H: 8-bit MSD digit histogram --------------------------------------
// Eight sub-histograms (by warp) against the contention of a skewed digit
// (R-MAT: 11% of configs[3]'s entries share digit 0); 16-byte loads of row
// pairs for directed lists.
__global__ void __launch_bounds__(kStNT) k_st_hist1(StArgs a) {
    __shared__ unsigned cnt[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kStNT) (&cnt[0][0])[i] = 0;
    __syncthreads();
    unsigned *mine = cnt[(threadIdx.x >> 5) & 7];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a.directed && (reinterpret_cast<uintptr_t>(a.rows) & 15) == 0) {
        const longlong2 *r2 = reinterpret_cast<const longlong2 *>(a.rows);
        const int64_t npair = a.E >> 1;
        for (int64_t i = t0; i < npair; i += stride) {
            const longlong2 rv = __ldcs(r2 + i);
            bool bad = false;
            const int64_t r0 = fix_row(rv.x, a, bad), r1 = fix_row(rv.y, a, bad);
            atomicAdd(mine + (unsigned)(r0 >> a.d1_shift), 1u);
            atomicAdd(mine + (unsigned)(r1 >> a.d1_shift), 1u);
        }
        if ((a.E & 1) && t0 == 0) {
            bool bad = false;
            atomicAdd(mine + (unsigned)(fix_row(__ldg(a.rows + a.E - 1), a, bad) >> a.d1_shift), 1u);
        }
    } else {
        for (int64_t i = t0; i < a.E; i += stride) {
            bool bad = false;
            int64_t r = a.directed ? fix_row(__ldg(a.rows + i), a, bad) : fix_index(__ldg(a.rows + i), a.N, bad);
            if (a.directed) {
                atomicAdd(mine + (unsigned)(r >> a.d1_shift), 1u);
            } else {
                int64_t c = fix_index(__ldg(a.cols + i), a.N, bad);
                if (bad) r = c = 0;
                atomicAdd(mine + (unsigned)(r >> a.d1_shift), 1u);
                if (r != c) atomicAdd(mine + (unsigned)(c >> a.d1_shift), 1u);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 256) {
        unsigned t = 0;
        for (int w = 0; w < 8; ++w) t += cnt[w][threadIdx.x];
        if (t) atomicAdd(a.ws.ctl + kCtlHist1 + threadIdx.x, t);
    }
}

__global__ void k_st_scan1(StArgs a) {
    // 256 digits, one warp-synchronous scan per 32
    __shared__ unsigned s[256];
    const int t = threadIdx.x;
    s[t] = a.ws.ctl[kCtlHist1 + t];
    __syncthreads();
    if (t == 0) {
        unsigned acc = 0;
        for (int d = 0; d < 256; ++d) {
            const unsigned v = s[d];
            s[d] = acc;
            acc += v;
        }
        a.ws.ctl[kCtlBase1 + 256] = acc;
    }
    __syncthreads();
    a.ws.ctl[kCtlBase1 + t] = s[t];
    a.ws.ctl[kCtlCur1 + t] = s[t];
}

// block-wide exclusive scan of cnt[0..n) in place (n <= 4 * blockDim)
template <int NT>
__device__ __forceinline__ void block_scan_bins(unsigned *cnt, int n, unsigned *red) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    constexpr int PER = 4;
    unsigned v[PER], sum = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int i = t * PER + j;
        v[j] = i < n ? cnt[i] : 0u;
        sum += v[j];
    }
    unsigned incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned x = lane < NT / 32 ? red[lane] : 0u, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < NT / 32) red[lane] = xi - x;
    }
    __syncthreads();
    unsigned run = red[wid] + incl - sum;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int i = t * PER + j;
        if (i < n) cnt[i] = run;
        run += v[j];
    }
    __syncthreads();
}

// block-wide exclusive scan of cnt[0..n) in place for n <= blockDim (one bin
// per thread: fewer live registers than block_scan_bins, whose peak made
// k_st_part1 spill its ranks and keys)
template <int NT>
__device__ __forceinline__ void block_scan_small(unsigned *cnt, int n, unsigned *red) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const unsigned v = t < n ? cnt[t] : 0u;
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) red[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned x = lane < NT / 32 ? red[lane] : 0u, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < NT / 32) red[lane] = xi - x;
    }
    __syncthreads();
    if (t < n) cnt[t] = red[wid] + incl - v;
    __syncthreads();
}

// ---- pass P1: partition by the MSD digit ------------------------------------
// Each thread owns EPT edges of the tile (8 entries: directed 8 edges, an
// undirected list 4 edges and their mirrors); all loads are issued before the
// first use so a warp has its whole tile share in flight.
template <int WT, bool DIR>
__global__ void __launch_bounds__(kStNT, 2) k_st_part1(StArgs a) {
    using WTy = typename WTraits<WT>::T;
    constexpr int EPT = DIR ? 8 : 4;
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long *skey = reinterpret_cast<unsigned long long *>(sm);
    WTy *sw = reinterpret_cast<WTy *>(sm + 8 * kStTile);
    __shared__ unsigned cnt[256], off[256], gbase[256], red[32];
    const int64_t tile_edges = (int64_t)EPT * kStNT;
    const int64_t ntiles = (a.E + tile_edges - 1) / tile_edges;
    int errbits = 0;
    int elow = INT_MAX / 2, ehigh = -INT_MAX / 2;  // weight exponent range (k_st_degree's integer mode)
    // software pipeline: the next tile's edges are loaded as soon as this
    // tile's entries sit in shared memory, and fly during the write-out
    long long r[EPT], c[EPT];
    WTy wv[EPT];
    auto load_tile = [&](int64_t tile) {
        const int64_t e0 = tile * tile_edges;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int64_t i = e0 + (int64_t)u * kStNT + threadIdx.x;
            r[u] = -2;
            if (tile < ntiles && i < a.E) {
                r[u] = __ldcs(reinterpret_cast<const long long *>(a.rows) + i);
                c[u] = __ldcs(reinterpret_cast<const long long *>(a.cols) + i);
                if constexpr (WT != GEE_W_UNIT) wv[u] = __ldcs(reinterpret_cast<const WTy *>(a.w) + i);
            }
        }
    };
    load_tile(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (threadIdx.x < 256) cnt[threadIdx.x] = 0;
        __syncthreads();
        unsigned long long key[EPT][DIR ? 1 : 2];
        unsigned rk[EPT][DIR ? 1 : 2];
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            rk[u][0] = 0xffffffffu;
            if (!DIR) rk[u][DIR ? 0 : 1] = 0xffffffffu;
            if (r[u] == -2) continue;
            bool bad = false;
            long long rr = DIR ? fix_row(r[u], a, bad) : fix_index(r[u], a.N, bad);
            long long cc = fix_index(c[u], a.N, bad);
            if constexpr (WT != GEE_W_UNIT) {
                if (!isfinite((double)wv[u])) {
                    errbits |= GEE_ERR_EDGE_WEIGHT;
                    wv[u] = 0;
                } else if (wv[u] < 0 && (a.flags & GEE_NONNEG)) {
                    errbits |= GEE_ERR_NEG_WEIGHT;
                }
                if (wv[u] != 0) {
                    int lo, hi;
                    weight_exponents(wv[u], lo, hi);
                    elow = min(elow, lo);
                    ehigh = max(ehigh, hi);
                }
            }
            if (bad) {
                // repaired exactly as k_st_hist1 counted it; the entry adds nothing
                errbits |= GEE_ERR_EDGE_RANGE;
                if constexpr (WT != GEE_W_UNIT) wv[u] = 0;
                if (!DIR) rr = cc = 0;
            }
            key[u][0] = ((unsigned long long)rr << 32) | (unsigned long long)cc;
            rk[u][0] = atomicAdd(cnt + (unsigned)(rr >> a.d1_shift), 1u);
            if constexpr (!DIR) {
                if (rr != cc) {
                    key[u][1] = ((unsigned long long)cc << 32) | (unsigned long long)rr;
                    rk[u][1] = atomicAdd(cnt + (unsigned)(cc >> a.d1_shift), 1u);
                }
            }
        }
        __syncthreads();
        // reserve each digit's run in the global digit region
        if (threadIdx.x < 256) {
            const unsigned n = cnt[threadIdx.x];
            gbase[threadIdx.x] = n ? atomicAdd(a.ws.ctl + kCtlCur1 + threadIdx.x, n) : 0u;
            off[threadIdx.x] = n;
        }
        __syncthreads();
        block_scan_small<kStNT>(off, 256, red);
        const unsigned total = off[255] + cnt[255];
        // reorder in shared memory by digit
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
#pragma unroll
            for (int h = 0; h < (DIR ? 1 : 2); ++h) {
                if (rk[u][h] == 0xffffffffu) continue;
                const unsigned d = (unsigned)((key[u][h] >> 32) >> a.d1_shift);
                const unsigned p = off[d] + rk[u][h];
                skey[p] = key[u][h];
                if constexpr (WT != GEE_W_UNIT) sw[p] = wv[u];
            }
        }
        load_tile(tile + gridDim.x);
        __syncthreads();
        // coalesced runs out
        for (unsigned t = threadIdx.x; t < total; t += kStNT) {
            const unsigned long long kk = skey[t];
            const unsigned d = (unsigned)((kk >> 32) >> a.d1_shift);
            const unsigned pos = gbase[d] + (t - off[d]);
            GEE_DASSERT(d < 256 && pos < a.ws.ctl[kCtlBase1 + d + 1] && pos >= a.ws.ctl[kCtlBase1 + d]);
            a.ws.keys1[pos] = kk;
            if constexpr (WT != GEE_W_UNIT) reinterpret_cast<WTy *>(a.ws.w1)[pos] = sw[t];
        }
        __syncthreads();
    }
    if (errbits) raise_err(a.err, errbits);
    if constexpr (WT != GEE_W_UNIT) {
        for (int o = 16; o > 0; o >>= 1) {
            elow = min(elow, __shfl_xor_sync(0xffffffffu, elow, o));
            ehigh = max(ehigh, __shfl_xor_sync(0xffffffffu, ehigh, o));
        }
        if ((threadIdx.x & 31) == 0 && ehigh > -INT_MAX / 2) {
            atomicMin(a.ws.ctl + kCtlWLow, (unsigned)(elow + kExpBias));
            atomicMax(a.ws.ctl + kCtlWHigh, (unsigned)(ehigh + kExpBias));
        }
    }
}

// ---- bucket histogram over the digit-ordered list ---------------------------
// 16384-entry tiles (four times the partition tile): a tile still lies within
// the 2048-bucket window (one digit region spans 2^d2_bits <= 1024 buckets),
// and its non-zero bins -- about one flush atomic per bucket of the region --
// amortise over four times the entries; 16-byte loads of entry pairs.
constexpr int kH2Tile = 16384;
__global__ void __launch_bounds__(kStNT) k_st_hist2(StArgs a) {
    __shared__ unsigned cnt[kStWin];
    const unsigned M = a.ws.ctl[kCtlBase1 + 256];
    const unsigned ntiles = (M + kH2Tile - 1) / kH2Tile;
    const ulonglong2 *k2 = reinterpret_cast<const ulonglong2 *>(a.ws.keys1);
    for (unsigned tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int i = threadIdx.x; i < kStWin; i += kStNT) cnt[i] = 0;
        __syncthreads();
        const unsigned p0 = tile * kH2Tile;
        const unsigned sub0 = (unsigned)((a.ws.keys1[p0] >> 32) >> a.d1_shift) << a.d2_bits;
        auto count = [&](unsigned long long key) {
            const unsigned sub = (unsigned)((key >> 32) >> a.lrow_bits);
            const unsigned rel = sub - sub0;
            if (rel < kStWin) atomicAdd(cnt + rel, 1u);
            else atomicAdd(a.ws.hist2 + sub, 1u);
        };
#pragma unroll 4
        for (int u = 0; u < kH2Tile / (2 * kStNT); ++u) {
            const unsigned p = p0 + 2 * (u * kStNT + threadIdx.x);  // even: keys1 is 256-byte aligned
            if (p + 1 < M) {
                const ulonglong2 kv = __ldcs(k2 + (p >> 1));
                count(kv.x);
                count(kv.y);
            } else if (p < M) {
                count(a.ws.keys1[p]);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kStWin; i += kStNT)
            if (cnt[i]) atomicAdd(a.ws.hist2 + sub0 + i, cnt[i]);
        __syncthreads();
    }
}

// Bucket bases, work items and split slots: a three-kernel scan over the S
// buckets (S <= 2^19).  Channels: entries, embed items (<= C entries each,
// at least one per bucket), degree items (<= kDegItem), split buckets.
__device__ __forceinline__ void bucket_channels(const StArgs &a, unsigned b, unsigned (&v)[4]) {
    const unsigned h = a.ws.hist2[b];
    const unsigned ni = h ? (h + a.C - 1) / a.C : 1u;
    v[0] = h;
    v[1] = ni;
    v[2] = h ? (h + kDegItem - 1) / kDegItem : 1u;
    v[3] = ni > 1;
}

__device__ __forceinline__ void block_scan4(unsigned (&v)[4], unsigned (&excl)[4], unsigned (&tot)[4],
                                            unsigned *red /* [4][32] */) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned inc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) inc[c] = v[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned y = __shfl_up_sync(0xffffffffu, inc[c], o);
            if (lane >= o) inc[c] += y;
        }
    __syncthreads();
    if (lane == 31)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[32 * c + wid] = inc[c];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned x = lane < nw ? red[32 * c + lane] : 0u;
            unsigned xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            red[32 * c + lane] = xi - x;
            if (lane == 31) red[128 + c] = xi;
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        excl[c] = red[32 * c + wid] + inc[c] - v[c];
        tot[c] = red[128 + c];
    }
}

__global__ void __launch_bounds__(1024) k_st_scan2a(StArgs a) {
    __shared__ unsigned red[132];
    const unsigned b0 = blockIdx.x * kScanBlock + threadIdx.x * 4;
    unsigned v[4] = {0u, 0u, 0u, 0u}, e[4], t[4];
    for (int j = 0; j < 4; ++j) {
        if (b0 + j < a.S) {
            unsigned c[4];
            bucket_channels(a, b0 + j, c);
            for (int q = 0; q < 4; ++q) v[q] += c[q];
        }
    }
    block_scan4(v, e, t, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < 4; ++q) a.ws.scan_part[4 * blockIdx.x + q] = t[q];
}

__global__ void __launch_bounds__(1024) k_st_scan2b(StArgs a, unsigned nblk) {
    __shared__ unsigned red[132];
    unsigned v[4] = {0u, 0u, 0u, 0u}, e[4], t[4];
    if (threadIdx.x < nblk)
        for (int q = 0; q < 4; ++q) v[q] = a.ws.scan_part[4 * threadIdx.x + q];
    block_scan4(v, e, t, red);
    if (threadIdx.x < nblk)
        for (int q = 0; q < 4; ++q) a.ws.scan_part[4 * threadIdx.x + q] = e[q];
    if (threadIdx.x == 0) {
        a.ws.base2[a.S] = t[0];
        a.ws.item_off[a.S] = t[1];
        a.ws.ditem_off[a.S] = t[2];
        a.ws.ctl[kCtlItems] = t[1];
        a.ws.ctl[kCtlDItems] = t[2];
        a.ws.ctl[kCtlSplit] = t[3];
    }
}

__global__ void __launch_bounds__(1024) k_st_scan2c(StArgs a) {
    __shared__ unsigned red[132];
    const unsigned b0 = blockIdx.x * kScanBlock + threadIdx.x * 4;
    unsigned c[4][4], v[4] = {0u, 0u, 0u, 0u}, e[4], t[4];
    for (int j = 0; j < 4; ++j) {
        for (int q = 0; q < 4; ++q) c[j][q] = 0;
        if (b0 + j < a.S) bucket_channels(a, b0 + j, c[j]);
        for (int q = 0; q < 4; ++q) v[q] += c[j][q];
    }
    block_scan4(v, e, t, red);
    for (int q = 0; q < 4; ++q) e[q] += a.ws.scan_part[4 * blockIdx.x + q];
    for (int j = 0; j < 4; ++j) {
        const unsigned b = b0 + j;
        if (b >= a.S) break;
        a.ws.base2[b] = e[0];
        a.ws.cur2[b] = e[0];
        a.ws.item_off[b] = e[1];
        a.ws.ditem_off[b] = e[2];
        a.ws.split_slot[b] = c[j][3] ? e[3] : 0xffffffffu;
        a.ws.done_deg[b] = 0;
        a.ws.done_emb[b] = 0;
        for (unsigned i = 0; i < c[j][1]; ++i) {
            a.ws.item_bucket[e[1] + i] = b;
            const unsigned q0 = e[0] + i * a.C;
            a.ws.item_desc[e[1] + i] = make_uint4(b, q0, min(e[0] + c[j][0], q0 + a.C), c[j][1]);
        }
        for (unsigned i = 0; i < c[j][2]; ++i) a.ws.ditem_bucket[e[2] + i] = b;
        for (int q = 0; q < 4; ++q) e[q] += c[j][q];
    }
}

// ---- pass P2: partition into buckets ----------------------------------------
template <int WT, int NT, int TILE>
__global__ void __launch_bounds__(NT, 1024 / NT) k_st_part2(StArgs a) {
    using WTy = typename WTraits<WT>::T;
    extern __shared__ __align__(16) unsigned char sm[];
    uint32_t *skey = reinterpret_cast<uint32_t *>(sm);
    WTy *sw = reinterpret_cast<WTy *>(sm + 4 * TILE);
    unsigned *cnt = reinterpret_cast<unsigned *>(sm + (4 + WTraits<WT>::bytes) * TILE);
    unsigned *off = cnt + kStWin;
    unsigned *gbase = off + kStWin;
    unsigned short *srel = reinterpret_cast<unsigned short *>(gbase + kStWin);
    __shared__ unsigned red[32];
    const unsigned M = a.ws.ctl[kCtlBase1 + 256];
    const unsigned ntiles = (M + TILE - 1) / TILE;
    const unsigned rmask = (1u << a.lrow_bits) - 1u;
    constexpr int PER = TILE / NT;
    // software pipeline: the next tile's keys and weights are loaded into
    // registers as soon as this tile's are staged in shared memory, so they
    // fly while this tile is written out
    unsigned long long kk[PER];
    WTy wv[PER];
    auto load_tile = [&](unsigned tile) {
        const unsigned p0 = tile * TILE;
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const unsigned p = p0 + u * NT + threadIdx.x;
            kk[u] = ~0ull;
            if (tile < ntiles && p < M) {
                kk[u] = __ldcs(a.ws.keys1 + p);
                if constexpr (WT != GEE_W_UNIT) wv[u] = __ldcs(reinterpret_cast<const WTy *>(a.ws.w1) + p);
            }
        }
    };
    __shared__ unsigned s_sub0;
    load_tile(blockIdx.x);
    for (unsigned tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int i = threadIdx.x; i < kStWin; i += NT) cnt[i] = 0;
        if (threadIdx.x == 0) s_sub0 = (unsigned)((kk[0] >> 32) >> a.d1_shift) << a.d2_bits;  // entry p0
        __syncthreads();
        const unsigned sub0 = s_sub0;
        uint32_t k2[PER];
        unsigned rel[PER], rk[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            rel[u] = 0xffffffffu;
            if (kk[u] != ~0ull) {
                const unsigned r = (unsigned)(kk[u] >> 32), c = (unsigned)kk[u];
                const unsigned sub = r >> a.lrow_bits;
                k2[u] = ((r & rmask) << a.col_bits) | c;
                const unsigned rl = sub - sub0;
                if (rl < kStWin) {
                    rel[u] = rl;
                    rk[u] = atomicAdd(cnt + rl, 1u);
                } else {
                    // a tile spanning more than the window (tiny buckets): direct slot
                    const unsigned pos = atomicAdd(a.ws.cur2 + sub, 1u);
                    GEE_DASSERT(sub < a.S && pos < a.ws.base2[sub + 1]);
                    a.ws.keys2[pos] = k2[u];
                    if constexpr (WT != GEE_W_UNIT) reinterpret_cast<WTy *>(a.ws.w2)[pos] = wv[u];
                }
            }
        }
        __syncthreads();
        {
            // all of this thread's reservations in flight at once
            constexpr int PB = kStWin / NT;
            unsigned cc[PB], gb[PB];
#pragma unroll
            for (int j = 0; j < PB; ++j) cc[j] = cnt[threadIdx.x + j * NT];
#pragma unroll
            for (int j = 0; j < PB; ++j)
                gb[j] = cc[j] ? atomicAdd(a.ws.cur2 + sub0 + threadIdx.x + j * NT, cc[j]) : 0u;
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                gbase[threadIdx.x + j * NT] = gb[j];
                off[threadIdx.x + j * NT] = cc[j];
            }
        }
        __syncthreads();
        block_scan_bins<NT>(off, kStWin, red);
        const unsigned total = off[kStWin - 1] + cnt[kStWin - 1];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            if (rel[u] != 0xffffffffu) {
                const unsigned p = off[rel[u]] + rk[u];
                skey[p] = k2[u];
                srel[p] = (unsigned short)rel[u];
                if constexpr (WT != GEE_W_UNIT) sw[p] = wv[u];
            }
        }
        load_tile(tile + gridDim.x);
        __syncthreads();
        // coalesced runs out
        for (unsigned t = threadIdx.x; t < total; t += NT) {
            const unsigned lo = srel[t];
            const unsigned pos = gbase[lo] + (t - off[lo]);
            GEE_DASSERT(sub0 + lo < a.S && pos >= a.ws.base2[sub0 + lo] && pos < a.ws.base2[sub0 + lo + 1]);
            a.ws.keys2[pos] = skey[t];
            if constexpr (WT != GEE_W_UNIT) reinterpret_cast<WTy *>(a.ws.w2)[pos] = sw[t];
        }
        __syncthreads();
    }
}

// ---- degrees and node records -------------------------------------------------
__device__ __forceinline__ void item_range(const StArgs &a, unsigned item, unsigned &b, unsigned &p0, unsigned &p1,
                                           unsigned &nitems) {
    b = a.ws.item_bucket[item];
    const unsigned j = item - a.ws.item_off[b];
    nitems = a.ws.item_off[b + 1] - a.ws.item_off[b];
    const unsigned s0 = a.ws.base2[b], s1 = a.ws.base2[b + 1];
    p0 = s0 + j * a.C;
    p1 = min(s1, p0 + a.C);
    if (p0 > s1) p0 = s1;
}

// node r (global id): s_r = 1/sqrt(d_r (+1 under A+I)) and its record
__device__ __forceinline__ void finish_node(const StArgs &a, int64_t r, double d) {
    double s = 1.0;
    if (a.flags & GEE_LAPLACIAN) {
        if (a.flags & GEE_DIAGONAL) d = d + 1.0;
        s = laplacian_scale(d, a.err);
    }
    a.ws.scale[r] = s;
    const int y = a.ws.y32[r];
    a.ws.rec[r] = make_double2(__longlong_as_double((long long)y), y >= 0 ? s * a.ws.inv[y] : 0.0);
}

__device__ __forceinline__ int rec_label(double2 rc) { return (int)__double_as_longlong(rc.x); }

// 16-byte global -> shared copy that bypasses L1 (cp.async.cg): the node
// record gathers of the embed land in shared memory without occupying the
// small L1 the Z tile leaves, so hundreds of them stay in flight per warp.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void *smem, const void *gmem, unsigned long long pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                     (unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int WT>
__device__ __forceinline__ double entry_w(const StArgs &a, unsigned p) {
    if constexpr (WT == GEE_W_UNIT) {
        return 1.0;
    } else {
        return (double)__ldcs(reinterpret_cast<const typename WTraits<WT>::T *>(a.ws.w2) + p);
    }
}

// Split bucket, degree side: the last of its items finalises the rows and
// clears the bucket's scratch tile for the embed items.
__device__ __forceinline__ void zero_scratch(const StArgs &a, unsigned b, int nrows, int t, int nt) {
    double *zs = a.ws.scratch + (size_t)a.ws.split_slot[b] * ((size_t)(1 << a.lrow_bits) * a.k);
    const int64_t nz = (int64_t)nrows * a.k;
    for (int64_t i = t; i < nz; i += nt) zs[i] = 0.0;
}

// Degrees and node records: a WARP per degree item (<= kDegItem entries of
// one bucket), so thousands of items are in flight per launch and no CTA
// barrier is ever taken.  Each warp keeps its bucket's R partial degrees in
// its own shared slice; a bucket with one item finalises its rows directly,
// the items of a larger bucket add into deg[] and the last one finalises
// (and clears the bucket's embed scratch tile when the embed splits it too).
template <int WT>
__global__ void __launch_bounds__(kDegNT, 5) k_st_degree(StArgs a) {  // 48 registers: a fifth CTA per SM
    extern __shared__ double wdeg[];  // [kDegNT / 32][R][copies] f64, or [kDegNT / 32][2][R] u32 (integer mode)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int R = 1 << a.lrow_bits;
    const bool lap = (a.flags & GEE_LAPLACIAN) != 0;
    const unsigned n_items = a.ws.ctl[kCtlDItems];
    const int cb = a.col_bits;
    // Integer mode: when every weight is a multiple of 2^low and the total of
    // all entries stays below 2^62 after scaling by 2^-low (unit weights;
    // configs[3]'s float32 weights are multiples of 2^-24), degrees are exact
    // 64-bit fixed-point sums kept as two native 32-bit shared atomics per
    // add (lo, and hi on a carry) -- no CAS retries on hot rows, and the
    // reference's fold bits whenever the total fits 53 bits.
    // When every scaled weight is below 2^16 (unit weights) an item's sum
    // (<= kDegItem entries) stays below 2^28, so one native non-returning
    // 32-bit reduction per add is exact.
    // When every scaled weight is below 2^32 (configs[3]'s f32 weights span
    // 25 bits), each is split into 16-bit limbs added by two non-returning
    // reductions: an item's sums of either limb stay below 2^28.
    int q = 0;
    bool imode = WT == GEE_W_UNIT, small = WT == GEE_W_UNIT, limb2 = false;
    if constexpr (WT != GEE_W_UNIT) {
        const unsigned lo = a.ws.ctl[kCtlWLow], hi = a.ws.ctl[kCtlWHigh];
        const unsigned M = a.ws.ctl[kCtlBase1 + 256];
        if (lo == 0xffffffffu) {
            imode = true;  // no nonzero weight
        } else {
            const int elow = (int)lo - kExpBias, ehigh = (int)hi - kExpBias;
            int mbits = 0;
            while ((1u << mbits) < M && mbits < 32) ++mbits;
            imode = elow > -1000 && ehigh - elow + mbits <= 62;
            q = -elow;
            small = ehigh - elow <= 16;
            limb2 = !small && ehigh - elow <= 32;
        }
    }
    const int copies = imode ? 1 : a.deg_copies;
    double *mine = wdeg + (size_t)wid * R * copies;
    unsigned *ilo = reinterpret_cast<unsigned *>(wdeg) + (size_t)wid * 2 * R, *ihi = ilo + R;
    const int cp = lane & (copies - 1);
    unsigned long long *gdeg = reinterpret_cast<unsigned long long *>(a.ws.deg);
    // x * 2^q is an integer below 2^62 with x's significant bits: the
    // multiplication by the power of two is exact (and far cheaper than ldexp)
    const double up = ldexp(1.0, q), down = ldexp(1.0, -q);
    auto to_fixed = [&](double x) -> unsigned long long { return (unsigned long long)(x * up); };
    auto iadd = [&](unsigned l, unsigned long long v) {
        if (small) {
            atomicAdd(ilo + l, (unsigned)v);  // result unused: a reduction
            return;
        }
        if (limb2) {  // v < 2^37 (a warp's sum): limbs of the item total < 2^44 stay below 2^28
            atomicAdd(ilo + l, (unsigned)v & 0xffffu);
            atomicAdd(ihi + l, (unsigned)(v >> 16));
            return;
        }
        const unsigned vlo = (unsigned)v, vhi = (unsigned)(v >> 32);
        const unsigned old = atomicAdd(ilo + l, vlo);
        const unsigned carry = (old + vlo) < old;
        if (vhi + carry) atomicAdd(ihi + l, vhi + carry);
    };
    auto ival = [&](int l) -> unsigned long long {
        return small   ? (unsigned long long)ilo[l]
               : limb2 ? ((unsigned long long)ihi[l] << 16) + ilo[l]
                       : ((unsigned long long)ihi[l] << 32) + ilo[l];
    };
    auto fdeg = [&](unsigned long long v) -> double { return (double)v * down; };
    constexpr int U = 8;
    // items claimed dynamically, a warp at a time (their sizes range from an
    // empty bucket to 4096 entries of a hub row); debug A/B: variant bit 512
    // keeps the static warp-strided assignment
    const bool dyn = !(a.variant & 512);
    auto claim = [&](unsigned prev) -> unsigned {
        if (!dyn) return prev == 0xffffffffu ? (blockIdx.x * kDegNT + threadIdx.x) >> 5 : prev + ((gridDim.x * kDegNT) >> 5);
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(a.ws.ctl + kCtlWork + 2, 1u);
        return __shfl_sync(0xffffffffu, it, 0);
    };
    for (unsigned item = claim(0xffffffffu); item < n_items; item = claim(item)) {
        const unsigned b = a.ws.ditem_bucket[item];
        const unsigned j = item - a.ws.ditem_off[b];
        const unsigned nitems = a.ws.ditem_off[b + 1] - a.ws.ditem_off[b];
        const unsigned s1 = a.ws.base2[b + 1];
        const unsigned p0 = min(s1, a.ws.base2[b] + j * kDegItem), p1 = min(s1, p0 + kDegItem);
        const int64_t r0 = (int64_t)b << a.lrow_bits;  // local row of the bucket
        const int nrows = (int)min((int64_t)R, a.nloc - r0);
        if (lap) {
            if (imode) {
                for (int l = lane; l < 2 * R; l += 32) ilo[l] = 0u;
            } else {
                for (int l = lane; l < R * copies; l += 32) mine[l] = 0.0;
            }
            __syncwarp();
            // warp-uniform trip count (the shuffles below need every lane)
            unsigned base = p0;
            for (; base + U * 32 <= p1; base += U * 32) {
                const unsigned p = base + lane;
                unsigned l[U];
                double x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) l[u] = __ldcs(a.ws.keys2 + p + u * 32) >> cb;
#pragma unroll
                for (int u = 0; u < U; ++u) x[u] = entry_w<WT>(a, p + u * 32);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    // a row-sorted input gives a warp 32 entries of one row: one
                    // shuffle reduction and a single add instead of 32 colliding adds
                    const unsigned l0 = __shfl_sync(0xffffffffu, l[u], 0);
                    const bool uni = __all_sync(0xffffffffu, l[u] == l0);
                    if (imode) {
                        unsigned long long v = to_fixed(x[u]);
                        if (uni) {
                            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                            if (lane == 0) iadd(l0, v);
                        } else {
                            iadd(l[u], v);
                        }
                    } else if (uni) {
                        const double sum = warp_sum(x[u]);
                        if (lane == 0) atomicAdd(mine + l0 * copies, sum);
                    } else {
                        atomicAdd(mine + l[u] * copies + cp, x[u]);
                    }
                }
            }
            for (unsigned p = base + lane; p < p1; p += 32) {
                const unsigned l = __ldcs(a.ws.keys2 + p) >> cb;
                GEE_DASSERT((int)l < R);
                if (imode) iadd(l, to_fixed(entry_w<WT>(a, p)));
                else atomicAdd(mine + l * copies + cp, entry_w<WT>(a, p));
            }
            __syncwarp();
            if (!imode) {
                for (int l = lane; l < R; l += 32) {
                    double d = 0.0;
                    for (int c = 0; c < copies; ++c) d += mine[l * copies + c];
                    mine[l * copies] = d;
                }
                __syncwarp();
            }
        }
        if (nitems == 1) {
            for (int l = lane; l < nrows; l += 32) {
                const double d = !lap ? 0.0 : imode ? fdeg(ival(l)) : mine[l * copies];
                if (a.deg_out) a.deg_out[r0 + l] = d;
                else finish_node(a, a.row0 + r0 + l, d);
            }
        } else {
            if (lap) {
                for (int l = lane; l < nrows; l += 32) {
                    if (imode) {
                        const unsigned long long v = ival(l);
                        if (v) atomicAdd(gdeg + r0 + l, v);
                    } else if (mine[l * copies] != 0.0) {
                        atomicAdd(a.ws.deg + r0 + l, mine[l * copies]);
                    }
                }
            }
            __threadfence();
            __syncwarp();
            unsigned last = 0;
            if (lane == 0) last = atomicAdd(a.ws.done_deg + b, 1u) == nitems - 1;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
                for (int l = lane; l < nrows; l += 32) {
                    const double d = !lap ? 0.0 : imode ? fdeg(__ldcg(gdeg + r0 + l)) : __ldcg(a.ws.deg + r0 + l);
                    if (a.deg_out) a.deg_out[r0 + l] = d;
                    else finish_node(a, a.row0 + r0 + l, d);
                }
                if (a.ws.split_slot[b] != 0xffffffffu) zero_scratch(a, b, nrows, lane, 32);
            }
        }
        __syncwarp();
    }
}

// Row-shard phase 2: the node table of every node from the all-gathered
// degrees (deg_all may be null without the Laplacian)
__global__ void k_st_nodes(StArgs a, const double *deg_all) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.N; j += (int64_t)gridDim.x * blockDim.x)
        finish_node(a, j, deg_all ? deg_all[j] : 0.0);
}

// ---- the fused embed ------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    unsigned ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// Bulk (TMA) copies between shared and global memory, no tensor map: the Z
// tile of a bucket is one contiguous run of Z, so one instruction stores it.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_store_s2g(void *g, const void *s, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the same with an L2 eviction policy (Z is written once: evict first, so the
// node records stay resident)
__device__ __forceinline__ void bulk_store_s2g_hint(void *g, const void *s, unsigned bytes, unsigned long long pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(g),
                 "r"(smem_u32(s)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_load_g2s(void *s, const void *g, unsigned bytes, unsigned long long *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(s)),
                 "l"(g), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Factor pass of the epilogue, L = 2^lgL lanes per row (L * R = NT when
// R <= NT, so every lane works): the A+I term g_r at the row's own label,
// f_r = s_r (Laplacian) times 1/||s_r z_r|| (correlation; one division per
// row -- z * (1/nrm) is within 1 ulp of the reference's z / nrm,
// embedding.py:140), then the row is scaled by f_r in place, each lane
// rescaling the V-element units it summed.  Rows start 16-byte aligned when
// K is even (V = 2: 16-byte shared loads and stores).
template <int NT, int V>
__device__ __forceinline__ void epi_rows(const StArgs &a, double *zt, const double *fac, const double2 *drec,
                                         int nrows, int lgL, int tid) {
    const int K = a.k;
    const unsigned flags = a.flags;
    const bool lap = (flags & GEE_LAPLACIAN) != 0, corr = (flags & GEE_CORRELATION) != 0;
    const int L = 1 << lgL;
    const int sub = tid & (L - 1);
    const int KU = K / V;  // units per row
    using VT = typename std::conditional<V == 2, double2, double>::type;
    const int R = 1 << a.lrow_bits;
    for (int l0 = 0; l0 < R && l0 < nrows; l0 += NT >> lgL) {  // uniform: the shuffles need whole warps
        const int l = l0 + (tid >> lgL);
        const bool live = l < nrows;
        double *row = zt + (size_t)(live ? l : 0) * K;
        VT *rv = reinterpret_cast<VT *>(row);
        const double s_r = lap && live ? fac[l] : 1.0;
        if ((flags & GEE_DIAGONAL) && live && sub == 0) {
            const double2 rc = drec[l];
            const int y = rec_label(rc);
            if (y >= 0) row[y] += rc.y;
        }
        __syncwarp();  // the diagonal term lands before the row is read
        double f = s_r;
        if (corr) {
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            if (live) {
                int c = sub;
                for (; c + 3 * L < KU; c += 4 * L) {
                    VT v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = rv[c + j * L];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if constexpr (V == 2) {
                            const double t0 = v[j].x * s_r, t1 = v[j].y * s_r;
                            s4[j] = fma(t0, t0, s4[j]);
                            s4[j] = fma(t1, t1, s4[j]);
                        } else {
                            const double t = v[j] * s_r;
                            s4[j] = fma(t, t, s4[j]);
                        }
                    }
                }
                for (; c < KU; c += L) {
                    const VT v = rv[c];
                    if constexpr (V == 2) {
                        const double t0 = v.x * s_r, t1 = v.y * s_r;
                        s4[0] = fma(t0, t0, s4[0]);
                        s4[1] = fma(t1, t1, s4[1]);
                    } else {
                        const double t = v * s_r;
                        s4[0] = fma(t, t, s4[0]);
                    }
                }
            }
            double ss = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            bool fin = true;
            if (live && !isfinite(ss)) {
                // a non-finite element, or finite ones whose squares overflow
                // (the reference raises only for the former, embedding.py:137-138)
                for (int c2 = sub; c2 < K; c2 += L) fin &= isfinite(row[c2]);
            }
            for (int o = L >> 1; o > 0; o >>= 1) {
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
                fin &= __shfl_xor_sync(0xffffffffu, (int)fin, o) != 0;
            }
            if (live) {
                if (!fin) {
                    if (sub == 0) raise_err(a.err, GEE_ERR_NONFINITE);
                } else {
                    const double nrm = __dsqrt_rn(ss);
                    if (nrm > 0.0) f = s_r * __ddiv_rn(1.0, nrm);
                }
            }
        }
        if (live && f != 1.0) {
            for (int c = sub; c < KU; c += L) {
                VT v = rv[c];
                if constexpr (V == 2) {
                    v.x *= f;
                    v.y *= f;
                } else {
                    v *= f;
                }
                rv[c] = v;
            }
        }
    }
}

// The factor pass for K even (16-byte units), free of shared-memory bank
// conflicts for any number of lanes per row.  A 16-byte shared access is served a
// quarter-warp (8 lanes) at a time, conflict-free when the 8 lanes touch 8
// different 16-byte bank groups, i.e. different (unit address mod 8).  With
// lanes (row, sub) reading unit `c = sub, sub + L, ...` of rows whose stride is
// K / 2 units (25 at configs[3]: consecutive rows are one group apart) the
// lanes (r, 1) and (r + 1, 0) met in one group: every access of the three
// passes cost two wavefronts instead of one (ncu: 7.7 per instruction, ideal
// 3.85).  Here a row is walked in blocks of 8 units; in step m of a block the
// lane reads unit 8 b + ((sub * G + c_r + m) mod 8), G = 8 / L rows per
// quarter-warp, c_r = (row-in-quarter - row * K/2) mod G: the 8 lanes of a
// quarter-warp then cover all 8 groups, and the L lanes of a row all 8 units.
template <int NT>
__device__ __forceinline__ void epi_rows_q(const StArgs &a, double *zt, const double *fac, const double2 *drec,
                                           int nrows, int lgL, int tid) {
    // 8 or more lanes per row (wide): consecutive units, conflict-free as is --
    // blocks of L units, one step each
    const bool wide = lgL >= 3;
    const int L = 1 << lgL, G = wide ? 1 : 8 >> lgL;
    const int bstep = wide ? L : 8, msk = bstep - 1;
    const int K = a.k, KU = K >> 1;
    const unsigned flags = a.flags;
    const bool lap = (flags & GEE_LAPLACIAN) != 0, corr = (flags & GEE_CORRELATION) != 0;
    const int sub = tid & (L - 1);
    const int R = 1 << a.lrow_bits;
    for (int l0 = 0; l0 < R && l0 < nrows; l0 += NT >> lgL) {  // uniform: the shuffles need whole warps
        const int l = l0 + (tid >> lgL);
        const bool live = l < nrows;
        const int lr = live ? l : 0;
        double *row = zt + (size_t)lr * K;
        double2 *rv = reinterpret_cast<double2 *>(row);
        const int rot = wide ? sub : sub * G + ((((tid >> lgL) & (G - 1)) - lr * KU) & (G - 1));
        const double s_r = lap && live ? fac[l] : 1.0;
        if ((flags & GEE_DIAGONAL) && live && sub == 0) {
            const double2 rc = drec[l];
            const int y = rec_label(rc);
            if (y >= 0) row[y] += rc.y;
        }
        __syncwarp();  // the diagonal term lands before the row is read
        double f = s_r;
        if (corr) {
            double sq0 = 0.0, sq1 = 0.0;
            if (live) {
                for (int b = 0; b < KU; b += bstep) {
                    for (int m = 0; m < G; ++m) {
                        const int u = b + ((rot + m) & msk);
                        if (u < KU) {
                            const double2 v = rv[u];
                            const double t0 = v.x * s_r, t1 = v.y * s_r;
                            sq0 = fma(t0, t0, sq0);
                            sq1 = fma(t1, t1, sq1);
                        }
                    }
                }
            }
            double ss = sq0 + sq1;
            bool fin = true;
            if (live && !isfinite(ss)) {
                // a non-finite element, or finite ones whose squares overflow
                // (the reference raises only for the former, embedding.py:137-138)
                for (int c2 = sub; c2 < K; c2 += L) fin &= isfinite(row[c2]);
            }
            for (int o = L >> 1; o > 0; o >>= 1) {
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
                fin &= __shfl_xor_sync(0xffffffffu, (int)fin, o) != 0;
            }
            if (live) {
                if (!fin) {
                    if (sub == 0) raise_err(a.err, GEE_ERR_NONFINITE);
                } else {
                    const double nrm = __dsqrt_rn(ss);
                    if (nrm > 0.0) f = s_r * __ddiv_rn(1.0, nrm);
                }
            }
        }
        if (live && f != 1.0) {
            for (int b = 0; b < KU; b += bstep) {
                for (int m = 0; m < G; ++m) {
                    const int u = b + ((rot + m) & msk);
                    if (u < KU) {
                        const double2 v = rv[u];
                        rv[u] = make_double2(v.x * f, v.y * f);
                    }
                }
            }
        }
    }
}

// The scaled tile (nrows * K elements, one contiguous run of Z at zoff) to Z:
// f64 output from a 16-byte aligned address leaves by one bulk copy issued by
// thread 0, and the tile is re-zeroed by a bulk copy from the zero page that
// completes on `zbar` (returns true: the caller waits on zbar before the next
// accumulation); otherwise the threads convert / store / zero it themselves.
template <bool OUT32, int NT>
__device__ __forceinline__ bool epi_store(const StArgs &a, double *zt, int64_t zoff, int tsz, int tid,
                                          unsigned long long *zbar, bool bulk, unsigned long long zpol) {
    if (!OUT32) {
        double *zg = reinterpret_cast<double *>(a.z) + zoff;
        if ((reinterpret_cast<uintptr_t>(zg) & 15) == 0 && !bulk) {
            double2 *z2 = reinterpret_cast<double2 *>(zt);
            double2 *g2 = reinterpret_cast<double2 *>(zg);
            for (int j = tid; j < (tsz >> 1); j += NT) {
                __stcs(g2 + j, z2[j]);
                z2[j] = make_double2(0.0, 0.0);
            }
            if ((tsz & 1) && tid == 0) {
                __stcs(zg + tsz - 1, zt[tsz - 1]);
                zt[tsz - 1] = 0.0;
            }
            return false;
        }
        if ((reinterpret_cast<uintptr_t>(zg) & 15) == 0) {
            if (tid == 0) {
                const unsigned bytes = (unsigned)(tsz & ~1) * 8u;
                if (bytes) {
                    if (a.variant & 64) bulk_store_s2g(zg, zt, bytes);  // debug A/B: no L2 hint
                    else bulk_store_s2g_hint(zg, zt, bytes, zpol);
                }
                if (tsz & 1) __stcs(zg + tsz - 1, zt[tsz - 1]);
                bulk_wait_read_all();  // the tile may be overwritten
                if (!(a.variant & 128)) bulk_load_g2s(zt, a.ws.zeros, (unsigned)((tsz + 1) & ~1) * 8u, zbar);
            }
            if (!(a.variant & 128)) return true;
            // debug A/B: re-zeroed by the threads once the bulk copy has read
            // the tile (measured 1% slower than the bulk re-zeroing)
            __syncthreads();
            double2 *z2 = reinterpret_cast<double2 *>(zt);
            for (int j = tid; j < ((tsz + 1) >> 1); j += NT) z2[j] = make_double2(0.0, 0.0);
            return false;
        }
    }
    if (OUT32 && ((reinterpret_cast<uintptr_t>(reinterpret_cast<float *>(a.z) + zoff) & 7) == 0)) {
        float2 *zg = reinterpret_cast<float2 *>(reinterpret_cast<float *>(a.z) + zoff);
        double2 *z2 = reinterpret_cast<double2 *>(zt);
        for (int j = tid; j < (tsz >> 1); j += NT) {
            const double2 v = z2[j];
            __stcs(zg + j, make_float2((float)v.x, (float)v.y));
            z2[j] = make_double2(0.0, 0.0);
        }
        if ((tsz & 1) && tid == 0) {
            __stcs(reinterpret_cast<float *>(a.z) + zoff + tsz - 1, (float)zt[tsz - 1]);
            zt[tsz - 1] = 0.0;
        }
        return false;
    }
    for (int e = tid; e < tsz; e += NT) {
        if (OUT32) __stcs(reinterpret_cast<float *>(a.z) + zoff + e, (float)zt[e]);
        else __stcs(reinterpret_cast<double *>(a.z) + zoff + e, zt[e]);
        zt[e] = 0.0;
    }
    return false;
}

// Epilogue of long rows (K even, K >= kEpiDirectK), a warp per row: the A+I
// term, the row's sum of squares from one read of the tile (16-byte units,
// consecutive lanes), the factor f_r = s_r / ||s_r z_r|| (correlation; one
// division per row, within 1 ulp of the reference's z / nrm,
// embedding.py:140), then every unit is read, zeroed and leaves as a
// streaming 16-byte store of f_r * z: 24 shared bytes per element against
// the 40 of epi_rows' in-place scaling + bulk store + bulk re-zeroing
// (configs[4]: 3.12 -> 2.69 ms).  Short rows keep the bulk path, where this
// one measured slower (configs[3]: 3.73 -> 3.99 ms).
constexpr int kEpiDirectK = 128;
template <int NT, bool OUT32>
__device__ __forceinline__ void epi_direct(const StArgs &a, double *zt, const double *fac, const double2 *drec,
                                           int64_t r0, int nrows) {
    const int K = a.k, KU = K >> 1;
    const unsigned flags = a.flags;
    const bool lap = (flags & GEE_LAPLACIAN) != 0, corr = (flags & GEE_CORRELATION) != 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int W = NT / 32;
    for (int l = wid; l < nrows; l += W) {
        double *row = zt + (size_t)l * K;
        double2 *rv = reinterpret_cast<double2 *>(row);
        const double s_r = lap ? fac[l] : 1.0;
        if ((flags & GEE_DIAGONAL) && lane == 0) {
            const double2 rc = drec[l];
            const int y = rec_label(rc);
            if (y >= 0) row[y] += rc.y;
        }
        __syncwarp();  // the diagonal term lands before the row is read
        double f = s_r;
        if (corr) {
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            int c = lane;
            for (; c + 32 < KU; c += 64) {
                const double2 p = rv[c], q = rv[c + 32];
                const double t0 = p.x * s_r, t1 = p.y * s_r, t2 = q.x * s_r, t3 = q.y * s_r;
                s4[0] = fma(t0, t0, s4[0]);
                s4[1] = fma(t1, t1, s4[1]);
                s4[2] = fma(t2, t2, s4[2]);
                s4[3] = fma(t3, t3, s4[3]);
            }
            if (c < KU) {
                const double2 p = rv[c];
                const double t0 = p.x * s_r, t1 = p.y * s_r;
                s4[0] = fma(t0, t0, s4[0]);
                s4[1] = fma(t1, t1, s4[1]);
            }
            double ss = (s4[0] + s4[1]) + (s4[2] + s4[3]);
            bool fin = true;
            if (!isfinite(ss))  // a non-finite element, or finite ones whose squares overflow
                for (int e = lane; e < K; e += 32) fin &= isfinite(row[e]);  // (the reference raises only for the former)
            ss = warp_sum(ss);
            fin = __all_sync(0xffffffffu, fin);
            if (!fin) {
                if (lane == 0) raise_err(a.err, GEE_ERR_NONFINITE);
            } else {
                const double nrm = __dsqrt_rn(ss);
                if (nrm > 0.0) f = s_r * __ddiv_rn(1.0, nrm);
            }
        }
        const int64_t g0 = (r0 + l) * K;
        for (int c = lane; c < KU; c += 32) {
            const double2 p = rv[c];
            rv[c] = make_double2(0.0, 0.0);
            if (OUT32) {
                __stcs(reinterpret_cast<float2 *>(reinterpret_cast<float *>(a.z) + g0) + c,
                       make_float2((float)(p.x * f), (float)(p.y * f)));
            } else {
                asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(reinterpret_cast<double *>(a.z) + g0 + 2 * c),
                             "d"(p.x * f), "d"(p.y * f)
                             : "memory");
            }
        }
    }
}

// The fused embed.  A CTA owns one R x K f64 Z tile in shared memory and
// pulls work items (<= C entries of one bucket) off a global counter.  The
// entries of the CTA's successive items form ONE stream of stages (U entries
// per thread); per thread the stream is a three-deep pipeline that never
// stops at an item boundary:
//   stage t     its node records (16-byte cp.async.cg gathers, L1 bypassed)
//               have landed in shared slot t&1: consumed -- one shared f64
//               add of w * g_j into the tile per entry;
//   stage t+1   records in flight (slot (t+1)&1);
//   stage t+2   keys + weights in registers (their loads in flight).
// Consuming stage t requests the records of t+2 and the keys of t+3, so when
// an item's last stage is consumed, the first stages of the items after it
// are already on their way and the epilogue (factor pass, bulk store of the
// tile, bulk re-zeroing) runs while they land.  The stage cursor reads the
// descriptors of up to three items ahead from a ring that thread 0 refills
// (one item per item consumed); an empty bucket's item has no stage, and a
// position the cursor cannot fill yet is a bubble.
template <int WT, bool OUT32, int NT, int U = 4>  // U entries per thread per stage
__global__ void __launch_bounds__(NT, (U == 1 ? 896 : U == 2 ? 768 : 640) / NT > 0 ? (U == 1 ? 896 : U == 2 ? 768 : 640) / NT : 1) k_st_embed(StArgs a) {
    constexpr int kRing = 8;   // work item descriptors {bucket, p0, p1, items of the bucket}
    constexpr int kAhead = 3;  // the cursor stays within this many items of the consumer
    extern __shared__ __align__(16) double zt[];  // [R][K], then fac[R], drec[R], the record slots
    __shared__ uint4 s_meta[kRing];
    __shared__ unsigned s_flag;
    __shared__ unsigned long long s_zbar;  // completes the bulk re-zeroing of the tile
    const int R = 1 << a.lrow_bits;
    const int K = a.k;
    double *fac = zt + (((size_t)R * K + 1) & ~(size_t)1);
    double2 *drec = reinterpret_cast<double2 *>(fac + ((R + 1) & ~1));  // [R] the rows' own records (A+I term)
    double2 *stage = drec + R;                                           // [2][U][NT]
    const unsigned n_items = a.ws.ctl[kCtlItems];
    const unsigned cmask = (1u << a.col_bits) - 1u;
    const int cb = a.col_bits;
    const unsigned step = U * NT;
    // epilogue: L = NT / R lanes per row (1..32), 16-byte units when K is even
    const int lgL = max(0, min(5, __ffs(NT) - 1 - a.lrow_bits));
    const bool kv2 = (K & 1) == 0;
    const bool bulk = (a.variant & 15) != 1;  // debug A/B: threads store the tile
    bool zpending = false;
    unsigned zphase = 0;
    // L2 policies: node records (the gather target) evict last, Z evict first
    const bool hints = !(a.variant & 64);
    const unsigned long long rpol = l2_policy_evict_last(), zpol = l2_policy_evict_first();
    // weights stay in their own type while loading (kC / xC); they are
    // converted when the stage's keys move to kA / kB (the gather has waited
    // for that load batch by then)
    using XT = typename std::conditional<WT == GEE_W_UNIT, float, typename WTraits<WT>::T>::type;
    uint32_t kA[U], kB[U], kC[U];
    XT xC[U];
    double xA[U], xB[U];  // converted when a stage's keys move out of kC
    auto loadk = [&](unsigned base, unsigned end, uint32_t(&kk)[U], XT(&x)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned p = base + u * NT + threadIdx.x;
            kk[u] = 0xffffffffu;
            if (p < end) {
                kk[u] = __ldcs(a.ws.keys2 + p);
                if constexpr (WT != GEE_W_UNIT) x[u] = __ldcs(reinterpret_cast<const XT *>(a.ws.w2) + p);
            }
        }
    };
    auto gather = [&](const uint32_t(&kk)[U], int s) {  // one commit group per call, possibly empty
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (kk[u] == 0xffffffffu) continue;
            const void *src = a.ws.rec + (kk[u] & cmask);
            if (hints) cp_async16_hint(stage + (s * U + u) * NT + threadIdx.x, src, rpol);
            else cp_async16(stage + (s * U + u) * NT + threadIdx.x, src);
        }
        cp_async_commit();
    };
    auto record = [&](int s, int u) -> double2 { return stage[(s * U + u) * NT + threadIdx.x]; };
    auto consume = [&](const uint32_t(&kk)[U], const double(&x)[U], int s) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (K <= 8 && __all_sync(0xffffffffu, kk[u] != 0xffffffffu)) {
                // few classes and a row-sorted input: every lane of the warp
                // on one row collides on K words -- reduce per class instead
                const unsigned lr0 = __shfl_sync(0xffffffffu, kk[u] >> cb, 0);
                if (__all_sync(0xffffffffu, (kk[u] >> cb) == lr0)) {
                    const double2 rc = record(s, u);
                    const int y = rec_label(rc);
                    const double v = (WT == GEE_W_UNIT ? 1.0 : x[u]) * rc.y;
                    for (int c = 0; c < K; ++c) {
                        const double t = warp_sum(y == c ? v : 0.0);
                        if ((threadIdx.x & 31) == 0 && t != 0.0) atomicAdd(zt + lr0 * K + c, t);
                    }
                    continue;
                }
            }
            if (kk[u] == 0xffffffffu) continue;
            const double2 rc = record(s, u);
            const int y = rec_label(rc);
            const double xv = WT == GEE_W_UNIT ? 1.0 : x[u];
            GEE_DASSERT((int)(kk[u] >> cb) < R && (int64_t)(kk[u] & cmask) < a.N && y < K);
            if ((a.variant & 15) == 4) {  // debug diagnostics only: plain add instead of the atomic
                if (y >= 0) zt[(kk[u] >> cb) * K + y] += xv * rc.y;
            } else if (y >= 0) {
                atomicAdd(zt + (kk[u] >> cb) * K + y, xv * rc.y);
            }
        }
    };
    auto grab = [&](unsigned n) {  // thread 0: the CTA's n-th work item into the ring
        const unsigned item = atomicAdd(a.ws.ctl + kCtlWork + 1, 1u);
        s_meta[n % kRing] = item < n_items ? a.ws.item_desc[item] : make_uint4(0xffffffffu, 0, 0, 0);
    };
    const bool direct_epi = kv2 && K >= kEpiDirectK && !(a.variant & 32) && (a.variant & 15) == 0;
    // Per-warp tile segments (short rows, R <= NT): the factor pass gives each
    // warp 32/L whole consecutive rows, i.e. one contiguous run of the tile and
    // of Z, so each warp stores its run with its own bulk copy and re-zeroes
    // it, with no CTA barrier between the factor pass and the store (the
    // re-zeroing copies of all warps complete on s_zbar, waited before the
    // next accumulation).  Debug A/B bit 2048: the whole-tile store.
    const bool seg_epi = !OUT32 && !direct_epi && kv2 && bulk && (a.variant & 15) == 0 && !(a.variant & 2048) &&
                         R <= NT && R * 32 >= NT && (reinterpret_cast<uintptr_t>(a.z) & 15) == 0;
    auto epilogue = [&](int64_t r0, int nrows) {
        if (direct_epi) {
            epi_direct<NT, OUT32>(a, zt, fac, drec, r0, nrows);
            return;  // the tile's zeroing is ordered by the item's closing barrier
        }
        if (seg_epi) {
            epi_rows_q<NT>(a, zt, fac, drec, nrows, lgL, threadIdx.x);
            fence_proxy_async_smem();  // this lane's scaled units are visible to the bulk copy
            __syncwarp();
            if ((threadIdx.x & 31) == 0) {
                const int rw = 32 >> lgL;
                const int l0 = (threadIdx.x >> 5) * rw;
                const int nr = max(0, min(rw, nrows - l0));
                if (nr > 0) {
                    const unsigned bytes = (unsigned)(nr * K) * 8u;
                    bulk_store_s2g_hint(reinterpret_cast<double *>(a.z) + (r0 + l0) * K, zt + (size_t)l0 * K, bytes, zpol);
                    bulk_wait_read_all();  // the segment may be overwritten
                    bulk_load_g2s(zt + (size_t)l0 * K, a.ws.zeros, bytes, &s_zbar);
                } else {
                    mbar_arrive(&s_zbar);
                }
            }
            zpending = true;
            return;
        }
        if ((a.variant & 15) != 2 && (a.variant & 15) != 3) {
            if (kv2) epi_rows_q<NT>(a, zt, fac, drec, nrows, lgL, threadIdx.x);
            else epi_rows<NT, 1>(a, zt, fac, drec, nrows, lgL, threadIdx.x);
        }
        fence_proxy_async_smem();  // the scaled tile is visible to the bulk copy
        __syncthreads();
        if ((a.variant & 15) == 3) {  // debug diagnostics only: the tile is zeroed, Z not written
            for (int i = threadIdx.x; i < nrows * K; i += NT) zt[i] = 0.0;
            return;
        }
        if (epi_store<OUT32, NT>(a, zt, r0 * K, nrows * K, threadIdx.x, &s_zbar, bulk, zpol)) zpending = true;
    };
    // the stage cursor (uniform across the CTA): item qi of the CTA, next entry qb
    unsigned ci = 0, qi = 0, qb = 0xffffffffu;
    auto cursor = [&](unsigned &base, unsigned &end) -> bool {
        for (;;) {
            if (qi > ci + kAhead) return false;  // descriptor not published yet: a bubble
            const uint4 d = s_meta[qi % kRing];
            if (d.x == 0xffffffffu) return false;  // no more work
            if (qb == 0xffffffffu) qb = d.y;
            if (qb < d.z) {
                base = qb;
                end = d.z;
                qb += step;
                return true;
            }
            ++qi;
            qb = 0xffffffffu;
        }
    };
    {
        double2 *z2 = reinterpret_cast<double2 *>(zt);
        for (int i = threadIdx.x; i < (R * K + 1) / 2; i += NT) z2[i] = make_double2(0.0, 0.0);
    }
    if (threadIdx.x == 0) {
        for (unsigned n = 0; n <= (unsigned)kAhead; ++n) grab(n);
        mbar_init(&s_zbar, seg_epi ? NT / 32 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // init visible to the bulk copies
    }
    __syncthreads();
    // prologue: stages 0 and 1 gathered, stage 2's keys loading
    unsigned vbits = 0;  // bit j: stream position t + j holds a stage (not a bubble)
    {
        // every load lands in kC / xC and reaches kA / kB by a register move,
        // as in the loop: a consumed operand is then never the destination of
        // an outstanding load, so its use does not wait on a scoreboard the
        // newest key loads share
        unsigned b0, e0;
        for (int j = 0; j < 3; ++j) {
            const bool ok = cursor(b0, e0);
            loadk(ok ? b0 : 0u, ok ? e0 : 0u, kC, xC);
            vbits |= ok ? 1u << j : 0u;
            if (j < 2) {
                gather(kC, j);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j == 0) {
                        kA[u] = kC[u];
                        xA[u] = WT == GEE_W_UNIT ? 1.0 : (double)xC[u];
                    } else {
                        kB[u] = kC[u];
                        xB[u] = WT == GEE_W_UNIT ? 1.0 : (double)xC[u];
                    }
                }
            }
        }
    }
    int par = 0;  // slot / register set of stream position t
    // one stream position: consume it (if it is a stage), gather t + 2 into its
    // slot, rotate the key registers, load the keys of t + 3
    const bool trace0 = GEE_TRACE_ON((a.variant & 16) && threadIdx.x == 0 && blockIdx.x < 4096);
    long long tw = 0, tc = 0, tg = 0;  // debug trace: wait / consume / refill cycles
    auto advance = [&](bool live) {
        const long long c0 = trace0 ? clock64() : 0;
        cp_async_wait<1>();
        const long long c1 = trace0 ? clock64() : 0;
        long long c2 = 0;
        unsigned b0 = 0, e0 = 0;
        if (par == 0) {
            if (live) consume(kA, xA, 0);
            if (trace0) c2 = clock64();
            gather(kC, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                kA[u] = kC[u];
                xA[u] = WT == GEE_W_UNIT ? 1.0 : (double)xC[u];
            }
        } else {
            if (live) consume(kB, xB, 1);
            if (trace0) c2 = clock64();
            gather(kC, 1);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                kB[u] = kC[u];
                xB[u] = WT == GEE_W_UNIT ? 1.0 : (double)xC[u];
            }
        }
        const bool ok = cursor(b0, e0);
        loadk(ok ? b0 : 0u, ok ? e0 : 0u, kC, xC);
        vbits = (vbits >> 1) | (ok ? 4u : 0u);
        par ^= 1;
        if (trace0) {
            const long long c3 = clock64();
            tw += c1 - c0;
            tc += c2 - c1;
            tg += c3 - c2;
        }
    };
    for (;; ++ci) {
        const uint4 d = s_meta[ci % kRing];
        const unsigned b = d.x;
        if (b == 0xffffffffu) break;
        const unsigned p0 = d.y, p1 = d.z, nitems = d.w;
        if (threadIdx.x == 0) grab(ci + kAhead + 1);  // published by the tile barrier below
        // Empty items take no stage, so the consumer passes them without a
        // cursor call and the cursor can fall behind it; its descriptors
        // would then come from ring slots already refilled with later items
        // (a stage-count mismatch: the item loop below spun forever on
        // bubbles).  Every item before ci is fully enumerated, so the cursor
        // restarts at ci.
        if (qi < ci) {
            qi = ci;
            qb = 0xffffffffu;
        }
        const int64_t r0 = (int64_t)b << a.lrow_bits;  // local row (Z row) of the bucket
        const int nrows = (int)min((int64_t)R, a.nloc - r0);
        const int tsz = nrows * K;
        // per-row data of the epilogue: asynchronous copies in a commit group
        // of their own, complete by the epilogue (every group but the newest
        // is; an item without stages waits for all) -- no load latency at
        // the start of the item
        if (a.variant & 256) {  // debug A/B: synchronous loads
            for (int l = threadIdx.x; l < nrows; l += NT) {
                if (a.flags & GEE_LAPLACIAN) fac[l] = a.ws.scale[a.row0 + r0 + l];
                if (a.flags & GEE_DIAGONAL) drec[l] = a.ws.rec[a.row0 + r0 + l];
            }
        } else {
            for (int l = threadIdx.x; l < nrows; l += NT) {
                if (a.flags & GEE_LAPLACIAN) cp_async8(fac + l, a.ws.scale + a.row0 + r0 + l);
                if (a.flags & GEE_DIAGONAL) cp_async16(drec + l, a.ws.rec + a.row0 + r0 + l);
            }
            cp_async_commit();
        }
        if (zpending) {  // the previous tile's bulk re-zeroing
            mbar_wait(&s_zbar, zphase);
            zphase ^= 1;
            zpending = false;
        }
        const bool trace = GEE_TRACE_ON((a.variant & 16) && threadIdx.x == 0 && blockIdx.x < 4096);
        const long long t1 = trace ? clock64() : 0;
        for (unsigned left = (p1 - p0 + step - 1) / step; left > 0;) {
            const bool live = vbits & 1u;
            advance(live);
            if (live) --left;
        }
        const long long t2 = trace ? clock64() : 0;
        if (p1 == p0) cp_async_wait<0>();  // the item's fac / drec copies (see above)
        else cp_async_wait<1>();
        __syncthreads();  // tile complete; the descriptor grabbed above visible; fac / drec landed
        const long long t3 = trace ? clock64() : 0;
        if (nitems == 1) {
            epilogue(r0, nrows);
        } else {
            GEE_DASSERT(a.ws.split_slot[b] < a.ws.ctl[kCtlSplit]);
            double *zs = a.ws.scratch + (size_t)a.ws.split_slot[b] * ((size_t)R * K);
            for (int i = threadIdx.x; i < tsz; i += NT) {
                const double v = zt[i];
                if (v != 0.0) {
                    atomicAdd(zs + i, v);
                    zt[i] = 0.0;
                }
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) s_flag = atomicAdd(a.ws.done_emb + b, 1u) == nitems - 1;
            __syncthreads();
            if (s_flag) {
                __threadfence();
                for (int i = threadIdx.x; i < tsz; i += NT) zt[i] = __ldcg(zs + i);
                __syncthreads();
                epilogue(r0, nrows);
            }
        }
        __syncthreads();  // tile zeroed (or its re-zeroing issued); s_flag free
        if (trace) {
            const long long t4 = clock64();
            unsigned long long *tr = g_emb_trace + (size_t)blockIdx.x * kTraceSlots;
            tr[1] += t2 - t1;
            tr[2] += t3 - t2;
            tr[3] += t4 - t3;
            tr[4] += 1;
            tr[5] += p1 - p0;
            tr[0] = tw;
            tr[6] = tc;
            tr[7] = tg;
        }
    }
    cp_async_wait<0>();
    if (zpending) mbar_wait(&s_zbar, zphase);  // no bulk copy outlives the CTA
    if (threadIdx.x == 0 || (seg_epi && (threadIdx.x & 31) == 0)) bulk_wait_all();
}

template <class T>
int set_smem(T *kern, size_t bytes) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return e == cudaSuccess ? GEE_OK : cuda_status(e);
}

template <int WT, int NT, int U>
int launch_embed(const StGeo &g, const StArgs &a, bool out32, cudaStream_t st) {
    static PerDevice attr;
    const size_t smem =
        sizeof(double) * (((size_t)1 << g.lrow_bits) * ((size_t)g.k + 3) + 4) + emb_stage_bytes(NT, U);
    const size_t smax = kZTileMax + 24 * 512 + emb_stage_bytes(NT, U);
    if (!attr.done()) {
        int rc;
        if ((rc = set_smem(k_st_embed<WT, false, NT, U>, smax))) return rc;
        if ((rc = set_smem(k_st_embed<WT, true, NT, U>, smax))) return rc;
        attr.mark();
    }
    int occ = 1;
    if (out32) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_st_embed<WT, true, NT, U>, NT, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_st_embed<WT, false, NT, U>, NT, smem);
    if (occ < 1) occ = 1;
    if (out32) k_st_embed<WT, true, NT, U><<<num_sms() * occ, NT, smem, st>>>(a);
    else k_st_embed<WT, false, NT, U><<<num_sms() * occ, NT, smem, st>>>(a);
    return GEE_OK;
}

// phase 1: partition the entries into row buckets and compute the degrees
// (node records, or the raw local degrees of a row shard)
template <int WT>
int run_phase1(const StGeo &g, StArgs &a, cudaStream_t st) {
    static PerDevice attr;
    const size_t p1_smem = (size_t)(8 + WTraits<WT>::bytes) * kStTile;
    // part2: 1024-thread CTAs over 8192-entry tiles (one per SM; bucket runs
    // twice as long as with 4096) unless the debug A/B bit 1024 asks for 512 / 4096
    const bool p2big = !(a.variant & 1024);
    const size_t p2_smem = (size_t)(4 + WTraits<WT>::bytes + 2) * (p2big ? 8192 : kStTile) + 3 * sizeof(unsigned) * kStWin;
    const size_t deg_smem = sizeof(double) * (kDegNT / 32) * ((size_t)1 << g.lrow_bits) * (size_t)a.deg_copies;
    if (!attr.done()) {
        int rc;
        if ((rc = set_smem(k_st_part1<WT, true>, p1_smem))) return rc;
        if ((rc = set_smem(k_st_part1<WT, false>, p1_smem))) return rc;
        if ((rc = set_smem(k_st_part2<WT, 1024, 8192>, (size_t)(4 + WTraits<WT>::bytes + 2) * 8192 + 3 * sizeof(unsigned) * kStWin))) return rc;
        if ((rc = set_smem(k_st_part2<WT, kStNT, kStTile>, (size_t)(4 + WTraits<WT>::bytes + 2) * kStTile + 3 * sizeof(unsigned) * kStWin))) return rc;
        if ((rc = set_smem(k_st_degree<WT>, sizeof(double) * (kDegNT / 32) * 512))) return rc;
        attr.mark();
    }
    const int sms = num_sms();
    k_st_hist1<<<sms * 4, kStNT, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_hist1");
    k_st_scan1<<<1, 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_scan1");
    if (g.directed) k_st_part1<WT, true><<<sms * 2, kStNT, p1_smem, st>>>(a);
    else k_st_part1<WT, false><<<sms * 2, kStNT, p1_smem, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_part1");
    k_st_hist2<<<sms * 4, kStNT, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_hist2");
    {
        const unsigned nblk = (g.S + kScanBlock - 1) / kScanBlock;
        k_st_scan2a<<<nblk, 1024, 0, st>>>(a);
        GEE_CHECK_LAUNCH("k_st_scan2a");
        k_st_scan2b<<<1, 1024, 0, st>>>(a, nblk);
        GEE_CHECK_LAUNCH("k_st_scan2b");
        k_st_scan2c<<<nblk, 1024, 0, st>>>(a);
        GEE_CHECK_LAUNCH("k_st_scan2c");
    }
    // as many CTAs as are resident (64 registers x 512 threads: two per SM);
    // the tiles are grid-strided, so a third CTA per SM ran as a second,
    // half-occupied wave
    if (p2big) k_st_part2<WT, 1024, 8192><<<sms, 1024, p2_smem, st>>>(a);
    else k_st_part2<WT, kStNT, kStTile><<<sms * 2, kStNT, p2_smem, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_part2");
    k_st_degree<WT><<<sms * 8, kDegNT, deg_smem, st>>>(a);
    GEE_CHECK_LAUNCH("k_st_degree");
    return GEE_OK;
}

// phase 2: the fused embed (+ the node table of a row shard from deg_all)
template <int WT>
int run_phase2(const StGeo &g, StArgs &a, const double *deg_all, bool shard, cudaStream_t st) {
    if (shard) {
        k_st_nodes<<<grid_for(g.N, 256, 8), 256, 0, st>>>(a, deg_all);
        GEE_CHECK_LAUNCH("k_st_nodes");
    }
    const bool out32 = (a.flags & GEE_FP32) != 0;
    int rc2;
    // Entries per thread and stage (U): fewer mean fewer registers and less stage
    // memory, so more resident CTAs whose epilogues and accumulations overlap --
    // U = 4: 96 registers, 5 CTAs/SM; U = 2: 80, 6 CTAs; U = 1: 72, 7 CTAs (the
    // gathers in flight per SM, 7 x 256, still cover DRAM latency at this rate).
    // Measured (profiles/r2_session3_ab.txt): configs[3] 3.17 / 3.12 / 3.52 ms,
    // configs[4] 2.71 / 2.48 / 2.40 ms, configs[2] 0.246 / 0.249 / 0.265 ms for
    // U = 4 / 2 / 1: U = 1 where buckets are small next to their tile (the
    // epilogue dominates), else U = 2.  Debug A/B bits: 16384 forces U = 4,
    // 32768 U = 1, both U = 2.
    const int force = (a.variant >> 14) & 3;
    const int u = force == 1 ? 4 : force == 2 ? 1 : force == 3 ? 2 : (g.Mcap / (int64_t)(g.S ? g.S : 1) < 768 ? 1 : 2);
    rc2 = u == 1   ? launch_embed<WT, 128, 1>(g, a, out32, st)
          : u == 2 ? launch_embed<WT, 128, 2>(g, a, out32, st)
                   : launch_embed<WT, 128, 4>(g, a, out32, st);
    if (rc2) return rc2;
    GEE_CHECK_LAUNCH("k_st_embed");
    return GEE_OK;
}

template <int WT>
int run_stream(const StGeo &g, StArgs &a, cudaStream_t st) {
    const int rc = run_phase1<WT>(g, a, st);
    return rc ? rc : run_phase2<WT>(g, a, nullptr, false, st);
}

}  // namespace

int set_stream_tile_kb(int v) {
    const int old = (int)(t_ztile_bytes >> 10);
    t_ztile_bytes = v > 0 && v <= 104 ? (size_t)v << 10 : kZTileDefault;
    return old;
}

int set_stream_embed_nt(int v) {
    const int old = t_emb_nt;
    (void)v;  // only 128-thread embed CTAs are built
    return old;
}

extern "C" int dbg_stream_trace_read(unsigned long long *out, int cap) {
    const int n = cap < 4096 * kTraceSlots ? cap : 4096 * kTraceSlots;
    if (cudaMemcpyFromSymbol(out, g_emb_trace, sizeof(unsigned long long) * (size_t)n) != cudaSuccess) return -1;
    static unsigned long long zero[4096 * kTraceSlots];
    cudaMemcpyToSymbol(g_emb_trace, zero, sizeof(zero));
    return n;
}

int set_stream_mode(int v) {
    const int old = t_stream_mode;
    t_stream_mode = v;
    return old;
}

bool stream_path_ok(int wt, unsigned flags, int64_t E, int64_t N, int directed, int k) {
    if (t_stream_mode == 1) return false;
    if (E < 1 || N < 2 || k < 1) return false;
    if (wt != GEE_W_UNIT && !(flags & GEE_NONNEG)) return false;
    if ((directed ? E : 2 * E) >= (int64_t)0xffffffffll) return false;
    StGeo g;
    return make_geo(g, E, N, directed, wt, k, flags);
}

size_t stream_workspace(int64_t E, int64_t N, int directed, int k, int wt) {
    StGeo g;
    if (!make_geo(g, E, N, directed, wt, k, 0)) return 0;
    Carver cv(nullptr);
    StWs w;
    return carve(cv, w, g);
}

static void fill_args(StArgs &a, const StGeo &g, const StWs &W, const int64_t *rows, const int64_t *cols,
                      const void *w, int64_t row0, void *z, int32_t *err) {
    a.rows = rows;
    a.cols = cols;
    a.w = w;
    a.E = g.E;
    a.N = g.N;
    a.row0 = row0;
    a.nloc = g.nloc;
    a.deg_out = nullptr;
    a.directed = g.directed;
    a.k = g.k;
    a.flags = g.flags;
    a.lrow_bits = g.lrow_bits;
    a.d2_bits = g.d2_bits;
    a.d1_shift = g.d1_shift;
    a.col_bits = g.col_bits;
    a.S = g.S;
    a.C = g.C;
    a.variant = t_stream_mode >= 16 ? t_stream_mode - 16 : 0;
    // 8 interleaved copies while the per-warp slice stays <= 4 KB (R <= 64), fewer for larger R
    a.deg_copies = g.lrow_bits <= 6 ? 8 : g.lrow_bits <= 7 ? 4 : g.lrow_bits <= 8 ? 2 : 1;  // <= 4 KB per warp
    a.magic = (0x100000000ull + (unsigned)g.k - 1) / (unsigned)g.k;
    a.ws = W;
    a.z = z;
    a.err = err;
}

static int setup(StGeo &g, StWs &W, void *ws, size_t ws_bytes, const int64_t *labels, cudaStream_t st,
                 int32_t *err) {
    Carver cv(ws);
    if (carve(cv, W, g) > ws_bytes || !ws) return GEE_E_WORKSPACE;
    GEE_CHECK_CUDA(cudaMemsetAsync(W.ctl, 0, sizeof(unsigned) * kCtlWords, st));
    GEE_CHECK_CUDA(cudaMemsetAsync(W.ctl + kCtlWLow, 0xff, sizeof(unsigned), st));
    GEE_CHECK_CUDA(cudaMemsetAsync(W.hist2, 0, sizeof(unsigned) * ((size_t)g.S + 1), st));
    GEE_CHECK_CUDA(cudaMemsetAsync(W.zeros, 0, sizeof(double) * (((size_t)1 << g.lrow_bits) * (size_t)g.k + 2), st));
    if (g.flags & GEE_LAPLACIAN) GEE_CHECK_CUDA(cudaMemsetAsync(W.deg, 0, sizeof(double) * (size_t)g.nloc, st));
    return label_hist_pipeline(labels, g.N, g.k, W.y32, W.counts, W.inv, W.label_partial, W.ctl + kCtlLabel, err, st);
}

int stream_encode(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int64_t N, int directed,
                  const int64_t *labels, int32_t k, unsigned flags, void *z, void *ws, size_t ws_bytes,
                  int32_t *err, cudaStream_t st) {
    StGeo g;
    if (!make_geo(g, E, N, directed, wt, k, flags)) return GEE_E_ARG;
    StWs W;
    int rc = setup(g, W, ws, ws_bytes, labels, st, err);
    if (rc) return rc;
    StArgs a;
    fill_args(a, g, W, rows, cols, w, 0, z, err);
    switch (wt) {
        case GEE_W_UNIT: return run_stream<GEE_W_UNIT>(g, a, st);
        case GEE_W_F32: return run_stream<GEE_W_F32>(g, a, st);
        default: return run_stream<GEE_W_F64>(g, a, st);
    }
}

// ---- row shards (multi-GPU, dist.py) ----------------------------------------------
bool stream_shard_ok(int wt, unsigned flags, int64_t e_local, int64_t N, int64_t rb, int64_t re, int k) {
    if (wt != GEE_W_UNIT && !(flags & GEE_NONNEG)) return false;
    if (e_local < 0 || e_local >= (int64_t)0xffffffffll || rb < 0 || re <= rb || re > N) return false;
    StGeo g;
    return make_geo(g, e_local, N, 1, wt, k, flags, re - rb);
}

size_t stream_shard_workspace(int64_t e_local, int64_t N, int64_t rb, int64_t re, int k, int wt) {
    StGeo g;
    if (!make_geo(g, e_local, N, 1, wt, k, 0, re - rb)) return 0;
    Carver cv(nullptr);
    StWs w;
    return carve(cv, w, g);
}

int stream_shard_degrees(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t e_local, int64_t N,
                         int64_t rb, int64_t re, const int64_t *labels, int32_t k, unsigned flags, double *deg_local,
                         void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st) {
    StGeo g;
    if (!make_geo(g, e_local, N, 1, wt, k, flags, re - rb)) return GEE_E_ARG;
    StWs W;
    int rc = setup(g, W, ws, ws_bytes, labels, st, err);
    if (rc) return rc;
    StArgs a;
    fill_args(a, g, W, rows, cols, w, rb, nullptr, err);
    a.deg_out = deg_local;
    switch (wt) {
        case GEE_W_UNIT: return run_phase1<GEE_W_UNIT>(g, a, st);
        case GEE_W_F32: return run_phase1<GEE_W_F32>(g, a, st);
        default: return run_phase1<GEE_W_F64>(g, a, st);
    }
}

int stream_shard_encode(int wt, int64_t e_local, int64_t N, int64_t rb, int64_t re, int32_t k, unsigned flags,
                        const double *deg_all, void *z_local, void *ws, size_t ws_bytes, int32_t *err,
                        cudaStream_t st) {
    StGeo g;
    if (!make_geo(g, e_local, N, 1, wt, k, flags, re - rb)) return GEE_E_ARG;
    Carver cv(ws);
    StWs W;
    if (carve(cv, W, g) > ws_bytes || !ws) return GEE_E_WORKSPACE;
    StArgs a;
    fill_args(a, g, W, nullptr, nullptr, nullptr, rb, z_local, err);
    switch (wt) {
        case GEE_W_UNIT: return run_phase2<GEE_W_UNIT>(g, a, deg_all, true, st);
        case GEE_W_F32: return run_phase2<GEE_W_F32>(g, a, deg_all, true, st);
        default: return run_phase2<GEE_W_F64>(g, a, deg_all, true, st);
    }
}

}  // namespace gee
