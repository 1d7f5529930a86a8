// k_shuffle.cu -- distributed CSR build: the device side of the edge shuffle.
//
// Input: every rank holds one contiguous slice of the ORIGINAL edge list
// (stream positions [e0, e1) of EdgeList(rows, cols, w), slices in rank
// order).  The symmetrised stream of the reference is
// [originals..., reversed off-diagonals...] (graph_io.py:82-88); rows of Z
// are owned by P contiguous row ranges.  Three device steps per rank:
//
//   k_shuffle_hist   coarse histogram of the local stream entries per row
//                    bucket (bucket of row r = floor(r * B / N)); the caller
//                    all-reduces it (equal-entry ranges)
//   k_shuffle_bounds P contiguous row ranges with near-equal stream entries
//                    from the all-reduced histogram (bucket-granular)
//   k_part_*         a stable partition of the local entries into 2P send
//                    buckets [half][dest] (half 0: originals routed by their
//                    row, half 1: mirrored off-diagonals routed by their
//                    column, written as (col, row)), each bucket in slice
//                    order: count per warp tile -> scan per bucket -> scatter
//
// The caller exchanges the originals region and then the mirrors region with
// one all-to-all each; concatenating what arrives ([originals from ranks
// 0..P-1] then [mirrors from ranks 0..P-1]) is exactly the destination's
// slice of the symmetrised stream in stream order -- the local_stream() of
// dist.py -- so duplicate sums, degrees and Z stay bitwise shard-invariant.
#include "gee_common.cuh"

namespace gee {

constexpr int kShufMaxWorld = 16;       // 2P send buckets <= 32 lanes
constexpr int kShufBuckets = 16384;     // coarse row buckets (<= N)
constexpr int kPartChunks = 64;         // 32-entry chunks per warp tile
constexpr int kPartTile = 32 * kPartChunks;

__device__ __forceinline__ int64_t shuf_bucket(int64_t r, int64_t n, int64_t nb) {
    // floor(r * nb / n) without overflow for n, nb < 2^31 * 2^14
    return (int64_t)(((unsigned __int128)r * (unsigned __int128)nb) / (unsigned __int128)n);
}

__global__ void k_shuffle_hist(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols, int64_t E,
                               int64_t n, int directed, int64_t nb, unsigned long long *__restrict__ hist) {
    extern __shared__ unsigned sh_hist[];
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) sh_hist[b] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const int64_t r = rows[e], c = cols[e];
        atomicAdd(&sh_hist[shuf_bucket(r, n, nb)], 1u);
        if (!directed && r != c) atomicAdd(&sh_hist[shuf_bucket(c, n, nb)], 1u);
    }
    __syncthreads();
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x)
        if (sh_hist[b]) atomicAdd(&hist[b], (unsigned long long)sh_hist[b]);
}

// bounds[0] = 0, bounds[P] = n; bounds[p] = first row of the first bucket at
// which the running entry count reaches total * p / P (dist.row_ranges on
// bucket granularity), kept monotone.  One thread: B <= 16384 buckets.
__global__ void k_shuffle_bounds(const unsigned long long *__restrict__ hist, int64_t nb, int64_t n, int world,
                                 int64_t *__restrict__ bounds) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned long long total = 0;
    for (int64_t b = 0; b < nb; ++b) total += hist[b];
    bounds[0] = 0;
    unsigned long long run = 0;  // entries in buckets < b
    int64_t b = 0;
    for (int p = 1; p < world; ++p) {
        const unsigned long long target = (unsigned long long)(((unsigned __int128)total * p) / world);
        while (b < nb && run < target) run += hist[b++];
        // first row of bucket b: ceil(b * n / nb)
        int64_t row = (int64_t)(((unsigned __int128)b * n + nb - 1) / nb);
        if (row < bounds[p - 1]) row = bounds[p - 1];
        if (row > n) row = n;
        bounds[p] = row;
    }
    bounds[world] = n;
}

struct PartArgs {
    const int64_t *rows, *cols;
    const void *w;
    int wt;  // GEE_W_*
    int64_t E;
    int directed;
    int world;
    const int64_t *bounds;
    int64_t n_tiles;
    unsigned *tile_cnt;     // [2P][n_tiles]
    int64_t *tile_off;      // [2P][n_tiles] exclusive, within the bucket
    unsigned long long *counts;  // [2P] bucket sizes
    int64_t *out_rows, *out_cols;
    void *out_w;
};

__device__ __forceinline__ int dest_of(const int64_t *bnd, int world, int64_t r) {
    int d = 0;
#pragma unroll 1
    for (int p = 1; p < world; ++p) d += r >= bnd[p] ? 1 : 0;
    return d;
}

// Send buckets of the entries of one 32-entry chunk: bo = the original's
// bucket (dest), bm = the mirror's bucket (P + dest) or -1.
__device__ __forceinline__ void chunk_buckets(const PartArgs &a, const int64_t *bnd, int64_t e, int64_t &r,
                                              int64_t &c, int &bo, int &bm) {
    bo = -1;
    bm = -1;
    r = 0;
    c = 0;
    if (e < a.E) {
        r = a.rows[e];
        c = a.cols[e];
        bo = dest_of(bnd, a.world, r);
        if (!a.directed && r != c) bm = a.world + dest_of(bnd, a.world, c);
    }
}

// Count of each bucket in this chunk, added into lane b's register.
__device__ __forceinline__ void add_bucket_counts(int bo, int bm, unsigned &mine) {
    const int lane = threadIdx.x & 31;
    for (int half = 0; half < 2; ++half) {
        const int b = half ? bm : bo;
        unsigned rest = __ballot_sync(0xffffffffu, b >= 0);
        while (rest) {
            const int leader = __ffs(rest) - 1;
            const int bl = __shfl_sync(0xffffffffu, b, leader);
            const unsigned m = __ballot_sync(0xffffffffu, b == bl);
            if (lane == bl) mine += __popc(m);
            rest &= ~m;
        }
    }
}

__global__ void k_part_count(PartArgs a) {
    __shared__ int64_t bnd[kShufMaxWorld + 1];
    for (int i = threadIdx.x; i <= a.world; i += blockDim.x) bnd[i] = a.bounds[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < a.n_tiles; t += warps) {
        unsigned mine = 0;
        for (int ch = 0; ch < kPartChunks; ++ch) {
            const int64_t e = t * kPartTile + ch * 32 + lane;
            if (t * kPartTile + ch * 32 >= a.E) break;
            int64_t r, c;
            int bo, bm;
            chunk_buckets(a, bnd, e, r, c, bo, bm);
            add_bucket_counts(bo, bm, mine);
        }
        if (lane < 2 * a.world) a.tile_cnt[(int64_t)lane * a.n_tiles + t] = mine;
    }
}

// one CTA per bucket: exclusive scan of its tile counts, and the bucket size
__global__ void k_part_scan(PartArgs a) {
    __shared__ unsigned long long red[33];
    const int b = blockIdx.x;
    const unsigned *cnt = a.tile_cnt + (int64_t)b * a.n_tiles;
    int64_t *off = a.tile_off + (int64_t)b * a.n_tiles;
    unsigned long long carry = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t t0 = 0; t0 < a.n_tiles; t0 += blockDim.x) {
        const int64_t t = t0 + threadIdx.x;
        const unsigned long long v = t < a.n_tiles ? cnt[t] : 0ull;
        unsigned long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) red[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned long long s = lane < nw ? red[lane] : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            if (lane < nw) red[lane] = s;
        }
        __syncthreads();
        const unsigned long long before = carry + (wid ? red[wid - 1] : 0ull) + x - v;
        if (t < a.n_tiles) off[t] = (int64_t)before;
        carry += red[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.counts[b] = carry;
}

template <typename W>
__device__ __forceinline__ void put_w(const PartArgs &a, int64_t src, int64_t dst) {
    static_cast<W *>(a.out_w)[dst] = static_cast<const W *>(a.w)[src];
}

__global__ void k_part_scatter(PartArgs a) {
    __shared__ int64_t bnd[kShufMaxWorld + 1];
    __shared__ unsigned long long base[2 * kShufMaxWorld];
    for (int i = threadIdx.x; i <= a.world; i += blockDim.x) bnd[i] = a.bounds[i];
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int b = 0; b < 2 * a.world; ++b) {
            base[b] = s;
            s += a.counts[b];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < a.n_tiles; t += warps) {
        // lane b holds the next free slot of bucket b for this tile
        int64_t next = 0;
        if (lane < 2 * a.world) next = (int64_t)base[lane] + a.tile_off[(int64_t)lane * a.n_tiles + t];
        for (int ch = 0; ch < kPartChunks; ++ch) {
            if (t * kPartTile + ch * 32 >= a.E) break;
            const int64_t e = t * kPartTile + ch * 32 + lane;
            int64_t r, c;
            int bo, bm;
            chunk_buckets(a, bnd, e, r, c, bo, bm);
            for (int half = 0; half < 2; ++half) {
                const int b = half ? bm : bo;
                // rank among this chunk's entries of the same bucket (lane order = slice order)
                const unsigned peers = __match_any_sync(0xffffffffu, b);
                const int64_t slot = __shfl_sync(0xffffffffu, next, b < 0 ? 0 : b) + __popc(peers & lanemask_lt());
                if (b >= 0) {
                    a.out_rows[slot] = half ? c : r;
                    a.out_cols[slot] = half ? r : c;
                    if (a.wt == GEE_W_F64)
                        put_w<double>(a, e, slot);
                    else if (a.wt == GEE_W_F32)
                        put_w<float>(a, e, slot);
                }
                // advance each bucket's cursor by its count in this chunk
                unsigned rest = __ballot_sync(0xffffffffu, b >= 0);
                while (rest) {
                    const int leader = __ffs(rest) - 1;
                    const int bl = __shfl_sync(0xffffffffu, b, leader);
                    const unsigned m = __ballot_sync(0xffffffffu, b == bl);
                    if (lane == bl) next += __popc(m);
                    rest &= ~m;
                }
            }
        }
    }
}

static int64_t part_tiles(int64_t E) { return (E + kPartTile - 1) / kPartTile; }

size_t partition_workspace(int64_t E, int world) {
    Carver cv(nullptr);
    const int64_t nt = part_tiles(E);
    cv.take<unsigned>((size_t)(2 * world) * nt);
    cv.take<int64_t>((size_t)(2 * world) * nt);
    return cv.bytes();
}

int shuffle_row_hist(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed,
                     int64_t nb, unsigned long long *hist, cudaStream_t st) {
    if (E <= 0) return GEE_OK;
    const size_t smem = sizeof(unsigned) * (size_t)nb;
    static PerDevice attr;
    if (!attr.done()) {
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_shuffle_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(unsigned) * kShufBuckets)));
        attr.mark();
    }
    k_shuffle_hist<<<grid_for(E, 512, 2), 512, smem, st>>>(rows, cols, E, n, directed, nb, hist);
    GEE_CHECK_LAUNCH("k_shuffle_hist");
    return GEE_OK;
}

int shuffle_bounds(const unsigned long long *hist, int64_t nb, int64_t n, int world, int64_t *bounds,
                   cudaStream_t st) {
    k_shuffle_bounds<<<1, 32, 0, st>>>(hist, nb, n, world, bounds);
    GEE_CHECK_LAUNCH("k_shuffle_bounds");
    return GEE_OK;
}

int partition(const int64_t *rows, const int64_t *cols, const void *w, int wt, int64_t E, int directed,
              const int64_t *bounds, int world, int64_t *out_rows, int64_t *out_cols, void *out_w,
              unsigned long long *counts, void *ws, size_t ws_bytes, cudaStream_t st) {
    PartArgs a;
    a.rows = rows;
    a.cols = cols;
    a.w = w;
    a.wt = wt;
    a.E = E;
    a.directed = directed;
    a.world = world;
    a.bounds = bounds;
    a.n_tiles = part_tiles(E);
    Carver cv(ws);
    a.tile_cnt = cv.take<unsigned>((size_t)(2 * world) * a.n_tiles);
    a.tile_off = cv.take<int64_t>((size_t)(2 * world) * a.n_tiles);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    a.counts = counts;
    a.out_rows = out_rows;
    a.out_cols = out_cols;
    a.out_w = out_w;
    if (E <= 0) {
        GEE_CHECK_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 2 * world, st));
        return GEE_OK;
    }
    const unsigned g = grid_for(a.n_tiles * 32, 256, 8);
    k_part_count<<<g, 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_part_count");
    k_part_scan<<<2 * world, 1024, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_part_scan");
    k_part_scatter<<<g, 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_part_scatter");
    return GEE_OK;
}

int shuffle_max_world() { return kShufMaxWorld; }
int64_t shuffle_buckets(int64_t n) { return n < kShufBuckets ? n : kShufBuckets; }

}  // namespace gee
