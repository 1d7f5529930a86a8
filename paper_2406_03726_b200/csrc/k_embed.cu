// k_embed.cu -- K4: Z = A'W with the option transforms fused in.
//
// Replaces spmm(A', build_weight_matrix(Y)).to_dense() (sparse.py:166-181,
// _kernels.py:257-307, sparse.py:87-91) plus add_identity (sparse.py:184-190),
// laplacian_normalize (sparse.py:199-226) and correlate_rows
// (embedding.py:134-143).  Per stored entry (r, j, v):
//     a'  = v (+1.0 when j == r under DIAGONAL; a missing diagonal is a
//           virtual 1.0 entry)                          _kernels.py:176-196
//     a'  = (a' * s_r) * s_j under LAPLACIAN            sparse.py:217
//     Z[r, Y_j] += a' * (1/n_{Y_j})  (Y_j >= 0)         _kernels.py:292-296
// W is never built.  Each node j is one 16-byte record {Y_j, g_j} with
// g_j = s_j * (1/n_{Y_j}) (s_j = 1 without Laplacian), so an entry costs one
// coalesced 4-byte column read plus one 16-byte gather; the term is
// (a' * s_r) * g_j, the reference's product re-associated (<= 2 ulp per term,
// far inside the 1e-12 budget).
//
// Work split: rows longer than kLongRow are taken first, one CTA per row
// (per-warp partial K-vectors combined in shared memory); every other row is
// one warp.  K <= 8 accumulates in registers (predicated adds, no dynamic
// indexing); larger K accumulates in a per-warp shared K-vector, combining
// equal-label lanes with __match_any_sync so no shared-memory fp64 atomics
// (a CAS loop on sm_100a) are ever issued.  K beyond kKTile is tiled, and
// correlation then rescales the row in a second sweep.
#include "gee_common.cuh"

namespace gee {

constexpr int kEmbedThreads = 256;
constexpr int kEmbedWarps = kEmbedThreads / 32;
constexpr int kLongRow = 4096;
constexpr int kKTile = 1024;
constexpr int kRowChunk = 32;  // rows per work grab (one warp)
// nodes whose table (9 B each) is staged in shared memory, by one 1024-thread
// CTA per SM so a single table copy serves 32 warps (with 256-thread CTAs the
// 90 KB table at N = 10^4 halved occupancy and lost to L1 record gathers)
constexpr int kTabMax = 12288;
constexpr int kTabThreads = 1024;

struct EmbedArgs {
    const int64_t *row_ptr;
    const unsigned *row_cnt;
    const int32_t *col;
    const double *val;
    int64_t row_begin, row_end;
    const double2 *rec;  // node records: x = bits of (label), y = g
    const double *scale;
    int k;
    unsigned flags;
    double *z;
    int64_t ldz;
    int32_t *err;
    const unsigned *long_list;
    const unsigned *n_long;
    unsigned *work;                // [2]
    const unsigned *val_flags;     // [2] from the sort path: both 0 => every value is 1.0
    const unsigned char *row_flag; // per row: 1 => read val for this row, 0 => values are 1.0
    const double *tab_g;           // optional compact node table (g, label) to stage on chip
    const signed char *tab_lab;
    int flat_rows;                 // > 0: phase 2 streams blocks of this many rows (K > 8)
    int flat_max;                  // longest row a block takes (longer: phase 1.5 / phase 1)
    int kp;                        // row stride of a flat block's shared tile
};

__device__ __forceinline__ void row_extent(const EmbedArgs &a, int64_t r, int64_t &s, int64_t &e) {
    s = a.row_ptr[r];
    e = a.row_cnt ? s + a.row_cnt[r] : a.row_ptr[r + 1];
}

__device__ __forceinline__ void node_rec(const EmbedArgs &a, int c, int &lab, double &g) {
    const double2 rc = __ldg(a.rec + c);
    lab = (int)(unsigned)(unsigned long long)__double_as_longlong(rc.x);
    g = rc.y;
}

// value array to use for row r (nullptr: every value is exactly 1.0)
__device__ __forceinline__ const double *row_vals(const EmbedArgs &a, int64_t r) {
    if (a.row_flag && !a.row_flag[r]) return nullptr;
    return a.val;
}

// One stored entry -> (label, contribution).  Returns false when it adds
// nothing (unlabeled column or padding).
__device__ __forceinline__ bool entry_term(const EmbedArgs &a, const double *val, int64_t r, double s_r,
                                           int64_t p, bool valid, int &lab, double &x, bool &isdiag) {
    lab = -1;
    x = 0.0;
    isdiag = false;
    if (!valid) return false;
    const int c = a.col[p];
    double v = val ? val[p] : 1.0;
    double g;
    node_rec(a, c, lab, g);
    if ((a.flags & GEE_DIAGONAL) && c == r) {
        v = v + 1.0;
        isdiag = true;
    }
    if (lab < 0) return false;
    if (a.flags & GEE_LAPLACIAN) v = v * s_r;
    x = v * g;
    return true;
}

// The virtual diagonal 1.0 of A+I for a row with no stored diagonal.
__device__ __forceinline__ bool diag_term(const EmbedArgs &a, int64_t r, double s_r, int &lab, double &x) {
    double g;
    node_rec(a, (int)r, lab, g);
    if (lab < 0) return false;
    x = ((a.flags & GEE_LAPLACIAN) ? s_r : 1.0) * g;
    return true;
}

__device__ __forceinline__ double row_scale(const EmbedArgs &a, int64_t r) {
    return (a.flags & GEE_LAPLACIAN) ? a.scale[r] : 1.0;
}

// streaming 16-byte load of column indices: read once, so keep them out of
// L1 (which holds the node-record table the gathers hit)
__device__ __forceinline__ int4 ld_stream_i4(const int32_t *p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ int ld_stream_i1(const int32_t *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------
// K <= KP <= 8: register accumulators, one warp per row.
// ---------------------------------------------------------------------------
// Node table staged in shared memory (small graphs): 9 bytes per node.
struct NodeTab {
    const double *g;
    const signed char *lab;
};

template <int KP, bool TAB>
__device__ __forceinline__ void consume(const EmbedArgs &a, const NodeTab &tab, int64_t r, double s_r, int c,
                                        double v, double (&acc)[KP], bool &found) {
    int lab;
    double g;
    if (TAB) {
        lab = tab.lab[c];
        g = tab.g[c];
    } else {
        node_rec(a, c, lab, g);
    }
    if ((a.flags & GEE_DIAGONAL) && c == r) {
        v = v + 1.0;
        found = true;
    }
    if (lab < 0) return;
    if (a.flags & GEE_LAPLACIAN) v = v * s_r;
    const double x = v * g;
#pragma unroll
    for (int q = 0; q < KP; ++q) acc[q] += (lab == q) ? x : 0.0;
}

template <int KP, bool TAB>
__device__ void row_regs(const EmbedArgs &a, const NodeTab &tab, int64_t r) {
    const int lane = threadIdx.x & 31;
    int64_t s, e;
    row_extent(a, r, s, e);
    const double s_r = row_scale(a, r);
    const double *val = row_vals(a, r);
    double acc[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) acc[q] = 0.0;
    bool found = false;
    if (TAB) {
        // node table in shared memory: lane-consecutive entries (a row's
        // columns are sorted, so one 32-lane gather spans ~32 nearby nodes and
        // hits distinct banks), 8 coalesced 128-byte loads in flight per warp
        for (int64_t p0 = s; p0 < e; p0 += 256) {
            int cc[8];
            double vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t p = p0 + 32 * u + lane;
                cc[u] = p < e ? __ldcs(a.col + p) : -1;
                vv[u] = (val && p < e) ? val[p] : 1.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cc[u] >= 0) consume<KP, TAB>(a, tab, r, s_r, cc[u], vv[u], acc, found);
        }
    } else {
    // head up to a 16-byte boundary of col, body in 16-byte vectors (4 entries
    // per lane, 256 entries per warp per iteration), scalar tail
    const int64_t a0 = min(e, (s + 3) & ~int64_t(3));
    if (s + lane < a0) consume<KP, TAB>(a, tab, r, s_r, a.col[s + lane], val ? val[s + lane] : 1.0, acc, found);
    // body: 4 x 16-byte column loads per lane in flight (512 entries per warp)
    const int64_t a1 = a0 + ((e - a0) & ~int64_t(511));
    for (int64_t p = a0 + 4 * lane; p < a1; p += 512) {
        int4 cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cc[u] = ld_stream_i4(a.col + p + 128 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double v[4] = {1.0, 1.0, 1.0, 1.0};
            if (val) {
                const double2 *vp = reinterpret_cast<const double2 *>(val + p + 128 * u);
                const double2 x0 = __ldg(vp), x1 = __ldg(vp + 1);
                v[0] = x0.x; v[1] = x0.y; v[2] = x1.x; v[3] = x1.y;
            }
            consume<KP, TAB>(a, tab, r, s_r, cc[u].x, v[0], acc, found);
            consume<KP, TAB>(a, tab, r, s_r, cc[u].y, v[1], acc, found);
            consume<KP, TAB>(a, tab, r, s_r, cc[u].z, v[2], acc, found);
            consume<KP, TAB>(a, tab, r, s_r, cc[u].w, v[3], acc, found);
        }
    }
    // remaining whole vectors, then the scalar tail
    const int64_t a2 = a1 + ((e - a1) & ~int64_t(3));
    for (int64_t p = a1 + 4 * lane; p < a2; p += 128) {
        const int4 c4 = ld_stream_i4(a.col + p);
        double v[4] = {1.0, 1.0, 1.0, 1.0};
        if (val) {
            const double2 *vp = reinterpret_cast<const double2 *>(val + p);
            const double2 x0 = __ldg(vp), x1 = __ldg(vp + 1);
            v[0] = x0.x; v[1] = x0.y; v[2] = x1.x; v[3] = x1.y;
        }
        consume<KP, TAB>(a, tab, r, s_r, c4.x, v[0], acc, found);
        consume<KP, TAB>(a, tab, r, s_r, c4.y, v[1], acc, found);
        consume<KP, TAB>(a, tab, r, s_r, c4.z, v[2], acc, found);
        consume<KP, TAB>(a, tab, r, s_r, c4.w, v[3], acc, found);
    }
    for (int64_t p = a2 + lane; p < e; p += 32) consume<KP, TAB>(a, tab, r, s_r, a.col[p], val ? val[p] : 1.0, acc, found);
    }
    if (a.flags & GEE_DIAGONAL) {
        found = __any_sync(0xffffffffu, found);
        int lb;
        double xd;
        if (!found && lane == 0 && diag_term(a, r, s_r, lb, xd)) {
#pragma unroll
            for (int q = 0; q < KP; ++q) acc[q] += (lb == q) ? xd : 0.0;
        }
    }
#pragma unroll
    for (int q = 0; q < KP; ++q) acc[q] = warp_sum(acc[q]);
    if (a.flags & GEE_CORRELATION) {
        double ss = 0.0;
        bool fin = true;
#pragma unroll
        for (int q = 0; q < KP; ++q) {
            if (q < a.k) {
                ss += acc[q] * acc[q];
                fin &= isfinite(acc[q]);
            }
        }
        if (!fin) {
            if (lane == 0) raise_err(a.err, GEE_ERR_NONFINITE);
        } else {
            double nrm = __dsqrt_rn(ss);
            if (nrm > 0.0) {
#pragma unroll
                for (int q = 0; q < KP; ++q) acc[q] = __ddiv_rn(acc[q], nrm);
            }
        }
    }
    double mine = 0.0;
#pragma unroll
    for (int q = 0; q < KP; ++q) mine = (lane == q) ? acc[q] : mine;
    if (lane < a.k) a.z[(r - a.row_begin) * a.ldz + lane] = mine;
}

// ---------------------------------------------------------------------------
// General K: per-warp shared K-tile.  Entries of this lane are
// p = s + lane + 32*(warp_off + j*warp_stride) (strided so a CTA can split
// a long row over its warps).
// ---------------------------------------------------------------------------
__device__ void accumulate_tile(const EmbedArgs &a, const double *val, int64_t r, double s_r, int64_t s,
                                int64_t e, int warp_off, int warp_stride, double *zs, double *xs, int t0, int kt,
                                bool &found) {
    const int lane = threadIdx.x & 31;
    for (int64_t p0 = s + (int64_t)warp_off * 32; p0 < e; p0 += (int64_t)warp_stride * 32) {
        int64_t p = p0 + lane;
        int lab;
        double x;
        bool isd;
        bool ok = entry_term(a, val, r, s_r, p, p < e, lab, x, isd);
        found |= isd;
        ok = ok && lab >= t0 && lab < t0 + kt;
        unsigned key = ok ? (unsigned)lab : 0x80000000u + lane;
        unsigned peers = __match_any_sync(0xffffffffu, key);
        xs[lane] = x;
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) {
            double sum = 0.0;
            unsigned m = peers;
            while (m) {
                int l = __ffs(m) - 1;
                m &= m - 1;
                sum += xs[l];
            }
            zs[lab - t0] += sum;
        }
        __syncwarp();
    }
}

// one warp, one row, K > 8
__device__ void row_smem(const EmbedArgs &a, int64_t r, double *zs, double *xs) {
    const int lane = threadIdx.x & 31;
    int64_t s, e;
    row_extent(a, r, s, e);
    const double s_r = row_scale(a, r);
    const double *val = row_vals(a, r);
    double *zrow = a.z + (r - a.row_begin) * a.ldz;
    const bool corr = (a.flags & GEE_CORRELATION) != 0;
    if (e == s) {
        // empty row (common in power-law graphs): zeros, plus A+I's diagonal
        // term x = s_r * g_r at the row's own label (x / |x| under correlation)
        int lb = -1;
        double xd = 0.0;
        if (a.flags & GEE_DIAGONAL) {
            if (!diag_term(a, r, s_r, lb, xd)) lb = -1;
        }
        if (lb >= 0 && corr) {
            if (!isfinite(xd)) {
                if (lane == 0) raise_err(a.err, GEE_ERR_NONFINITE);
            } else {
                const double nrm = __dsqrt_rn(xd * xd);
                if (nrm > 0.0) xd = xd * __ddiv_rn(1.0, nrm);
            }
        }
        for (int c = lane; c < a.k; c += 32) zrow[c] = c == lb ? xd : 0.0;
        return;
    }
    const int ntiles = (a.k + kKTile - 1) / kKTile;
    bool found = false;
    double ss = 0.0;
    bool fin = true;
    for (int t = 0; t < ntiles; ++t) {
        const int t0 = t * kKTile, kt = min(kKTile, a.k - t0);
        for (int c = lane; c < kt; c += 32) zs[c] = 0.0;
        __syncwarp();
        accumulate_tile(a, val, r, s_r, s, e, 0, 1, zs, xs, t0, kt, found);
        if (a.flags & GEE_DIAGONAL) {
            bool f = __any_sync(0xffffffffu, found);
            int lb;
            double xd;
            if (!f && lane == 0 && diag_term(a, r, s_r, lb, xd) && lb >= t0 && lb < t0 + kt) zs[lb - t0] += xd;
            __syncwarp();
        }
        for (int c = lane; c < kt; c += 32) {
            double v = zs[c];
            ss += v * v;
            fin &= isfinite(v);
        }
        if (!corr || ntiles > 1) {
            for (int c = lane; c < kt; c += 32) zrow[t0 + c] = zs[c];
        }
        __syncwarp();
    }
    if (!corr) return;
    ss = warp_sum(ss);
    fin = __all_sync(0xffffffffu, fin);
    if (!fin) {
        if (lane == 0) raise_err(a.err, GEE_ERR_NONFINITE);
        if (ntiles == 1)
            for (int c = lane; c < a.k; c += 32) zrow[c] = zs[c];
        return;
    }
    const double nrm = __dsqrt_rn(ss);
    if (ntiles == 1) {
        // one division per row; z * (1/nrm) is within 1 ulp of z / nrm
        // (embedding.py:140 divides; Z's bar is 1e-12 relative)
        const double rn = nrm > 0.0 ? __ddiv_rn(1.0, nrm) : 1.0;
        for (int c = lane; c < a.k; c += 32) zrow[c] = zs[c] * rn;
    } else if (nrm > 0.0) {
        const double rn = __ddiv_rn(1.0, nrm);
        for (int c = lane; c < a.k; c += 32) zrow[c] = zrow[c] * rn;
    }
    __syncwarp();
}

// one CTA, one long row (any K): warps accumulate strided slices into their
// own K-tile, then the tiles are summed.
__device__ void row_long(const EmbedArgs &a, int64_t r, double *zsm, double *xsm, double *dred) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int kt_max = min(a.k, kKTile);
    double *zs = zsm + wid * kt_max;
    double *xs = xsm + wid * 32;
    int64_t s, e;
    row_extent(a, r, s, e);
    const double s_r = row_scale(a, r);
    const double *val = row_vals(a, r);
    double *zrow = a.z + (r - a.row_begin) * a.ldz;
    const bool corr = (a.flags & GEE_CORRELATION) != 0;
    const int ntiles = (a.k + kKTile - 1) / kKTile;
    bool found = false;
    double ss = 0.0;
    int fin = 1;
    for (int t = 0; t < ntiles; ++t) {
        const int t0 = t * kKTile, kt = min(kKTile, a.k - t0);
        for (int c = lane; c < kt; c += 32) zs[c] = 0.0;
        __syncwarp();
        accumulate_tile(a, val, r, s_r, s, e, wid, (int)(blockDim.x >> 5), zs, xs, t0, kt, found);
        const int f = __syncthreads_or(found ? 1 : 0);
        // combine warp tiles into warp 0's tile (column c read from every warp,
        // written only to warp 0's copy by the thread owning c)
        for (int c = threadIdx.x; c < kt; c += blockDim.x) {
            double v = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += zsm[w * kt_max + c];
            zsm[c] = v;
        }
        __syncthreads();
        if ((a.flags & GEE_DIAGONAL) && !f && threadIdx.x == 0) {
            int lb;
            double xd;
            if (diag_term(a, r, s_r, lb, xd) && lb >= t0 && lb < t0 + kt) zsm[lb - t0] += xd;
        }
        __syncthreads();
        for (int c = threadIdx.x; c < kt; c += blockDim.x) {
            double v = zsm[c];
            ss += v * v;
            fin &= isfinite(v) ? 1 : 0;
            if (!corr || ntiles > 1) zrow[t0 + c] = v;
        }
        __syncthreads();
    }
    if (!corr) return;
    ss = block_sum(ss, dred);
    fin = __syncthreads_and(fin);
    if (!fin) {
        if (threadIdx.x == 0) raise_err(a.err, GEE_ERR_NONFINITE);
        if (ntiles == 1)
            for (int c = threadIdx.x; c < a.k; c += blockDim.x) zrow[c] = zsm[c];
        __syncthreads();
        return;
    }
    const double nrm = __dsqrt_rn(ss);
    if (ntiles == 1) {
        const double rn = nrm > 0.0 ? __ddiv_rn(1.0, nrm) : 1.0;
        for (int c = threadIdx.x; c < a.k; c += blockDim.x) zrow[c] = zsm[c] * rn;
    } else if (nrm > 0.0) {
        const double rn = __ddiv_rn(1.0, nrm);
        for (int c = threadIdx.x; c < a.k; c += blockDim.x) zrow[c] = zrow[c] * rn;
    }
    __syncthreads();
}


// ---------------------------------------------------------------------------
// K > 8, rows up to kLongRow: a warp takes R = a.flat_rows consecutive rows
// and streams their entries as ONE lane-consecutive sequence (entry f of the
// block belongs to the row whose prefix brackets f), accumulating into an
// R x K shared tile.  The per-row fixed costs of a warp-per-row walk (extent
// loads, a K-vector clear and sweep, a partial-sector Z row) are shared by R
// rows: extents, scales and flags of the block arrive in one round trip,
// every iteration has 32*U column loads and then 32*U node-record gathers in
// flight, and the block's R x K slice of Z is written as one contiguous run.
// Rows longer than kLongRow are left to phase 1 (their Z rows are skipped).
// ---------------------------------------------------------------------------
constexpr int kFlatU = 4;

// One flat block: rows r0 .. r0+nr-1 (a lone listed row when nr == 1 and
// rmax == kLongRow); rows longer than rmax are left to their own phase and
// their Z rows are not written.
__device__ void flat_block(const EmbedArgs &a, int64_t r0, int nr, int rmax, double *zs, double *xs) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int K = a.k, Kp = a.kp;
    const bool lap = (a.flags & GEE_LAPLACIAN) != 0, dia = (a.flags & GEE_DIAGONAL) != 0;
    const bool corr = (a.flags & GEE_CORRELATION) != 0;
    int64_t st = 0;
    int cnt = 0, uv = 0, dlab = -1;
    bool excl = false;
    double sr = 1.0, dg = 0.0;
    if (lane < nr) {
        const int64_t r = r0 + lane;
        int64_t s, e;
        row_extent(a, r, s, e);
        st = s;
        excl = e - s > rmax;
        cnt = excl ? 0 : (int)(e - s);
        if (lap) sr = a.scale[r];
        uv = (a.val != nullptr && !(a.row_flag && !a.row_flag[r])) ? 1 : 0;
        if (dia) node_rec(a, (int)r, dlab, dg);
    }
    const unsigned exmask = __ballot_sync(full, excl);
    int inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(full, inc, o);
        if (lane >= o) inc += y;
    }
    const int pre = lane < nr ? inc - cnt : INT_MAX;
    const int T = __shfl_sync(full, inc, 31);
    {
        // the tile is 16-byte aligned with an even stride (wst): clear pairs
        double2 *z2 = reinterpret_cast<double2 *>(zs);
        for (int q = lane; 2 * q < nr * Kp; q += 32) z2[q] = make_double2(0.0, 0.0);
    }
    __syncwarp();
    unsigned dmask = 0;
    for (int f0 = 0; f0 < T; f0 += 32 * kFlatU) {
        int ri[kFlatU], cc[kFlatU];
        double vv[kFlatU];
#pragma unroll
        for (int u = 0; u < kFlatU; ++u) {
            const int f = f0 + 32 * u + lane;
            int lo = 0;
            if (nr > 1) {
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int pm = __shfl_sync(full, pre, lo + step);
                    if (pm <= f) lo += step;
                }
            }
            ri[u] = lo;
            const int64_t p = __shfl_sync(full, st, lo) + (f - __shfl_sync(full, pre, lo));
            const int use_v = __shfl_sync(full, uv, lo);
            const bool ok = f < T;
            cc[u] = ok ? ld_stream_i1(a.col + p) : -1;
            vv[u] = (ok && use_v) ? a.val[p] : 1.0;
        }
        int lab[kFlatU];
        double g[kFlatU];
#pragma unroll
        for (int u = 0; u < kFlatU; ++u) {
            lab[u] = -1;
            g[u] = 0.0;
            if (cc[u] >= 0) node_rec(a, cc[u], lab[u], g[u]);
        }
#pragma unroll
        for (int u = 0; u < kFlatU; ++u) {
            const double s_i = __shfl_sync(full, sr, ri[u]);
            double v = vv[u];
            if (dia && cc[u] >= 0 && (int64_t)cc[u] == r0 + ri[u]) {
                v = v + 1.0;
                dmask |= 1u << ri[u];
            }
            const bool ok = cc[u] >= 0 && lab[u] >= 0;
            const double x = (lap ? v * s_i : v) * g[u];
            const unsigned key = ok ? (unsigned)(ri[u] * Kp + lab[u]) : 0x80000000u + lane;
            const unsigned peers = __match_any_sync(full, key);
            xs[lane] = x;
            __syncwarp();
            if (ok && lane == __ffs(peers) - 1) {
                double sum = 0.0;
                unsigned m = peers;
                while (m) {
                    const int l = __ffs(m) - 1;
                    m &= m - 1;
                    sum += xs[l];
                }
                zs[key] += sum;
            }
            __syncwarp();
        }
    }
    // A+I: the virtual 1.0 of rows without a stored diagonal
    if (dia) {
        dmask = __reduce_or_sync(full, dmask);
        if (lane < nr && !excl && !((dmask >> lane) & 1u) && dlab >= 0) zs[lane * Kp + dlab] += (lap ? sr : 1.0) * dg;
        __syncwarp();
    }
    // correlation: L lanes per row (L = the largest power of two with
    // L * nr <= 32) fold every L-th column, an L-lane butterfly gives every
    // one of them the norm, and they rescale their columns in place
    double rn = 1.0;
    if (corr) {
        int L = 32;
        while (L > 1 && L * nr > 32) L >>= 1;
        const int i = lane / L, j = lane - i * L;
        double ss = 0.0;
        double *zi = zs + i * Kp;
        if (nr == 1 && !(K & 1)) {
            // one row: 16-byte shared loads, two independent accumulators
            const double2 *z2 = reinterpret_cast<const double2 *>(zs);
            double s1 = 0.0;
            for (int q = lane; 2 * q < K; q += 32) {
                const double2 v = z2[q];
                ss = fma(v.x, v.x, ss);
                s1 = fma(v.y, v.y, s1);
            }
            ss += s1;
        } else if (i < nr) {
            for (int q = j; q < K; q += L) ss = fma(zi[q], zi[q], ss);
        }
        for (int o = 1; o < L; o <<= 1) ss += __shfl_xor_sync(full, ss, o);
        const bool live = i < nr && !((exmask >> i) & 1u);
        int fin = 1;
        if (live && !isfinite(ss)) {
            // inf/nan in the row, or a norm beyond the double range
            // (embedding.py:137-138 checks the entries themselves)
            for (int q = j; q < K; q += L) fin &= isfinite(zi[q]) ? 1 : 0;
        }
        for (int o = 1; o < L; o <<= 1) fin &= __shfl_xor_sync(full, fin, o);
        if (live) {
            if (!fin) {
                if (j == 0) raise_err(a.err, GEE_ERR_NONFINITE);
            } else {
                // one division per row; z * (1/nrm) is within 1 ulp of
                // z / nrm (embedding.py:140 divides; Z's bar is 1e-12)
                const double nrm = __dsqrt_rn(ss);
                if (nrm > 0.0) {
                    rn = __ddiv_rn(1.0, nrm);
                    // one row per block: the copy below applies rn instead
                    if (nr > 1)
                        for (int q = j; q < K; q += L) zi[q] *= rn;
                }
            }
        }
        __syncwarp();
    }
    // the block's Z rows: one contiguous copy when the tile is dense and no
    // row belongs to another phase, else row by row (others' rows skipped)
    double *zb = a.z + (r0 - a.row_begin) * a.ldz;
    if (nr == 1) {
        rn = __shfl_sync(full, rn, 0);
        if (!exmask) {
            if (!(K & 1) && !(a.ldz & 1) && !(reinterpret_cast<uintptr_t>(a.z) & 15)) {
                const double2 *z2 = reinterpret_cast<const double2 *>(zs);
                double2 *o2 = reinterpret_cast<double2 *>(zb);
                for (int q = lane; 2 * q < K; q += 32) {
                    const double2 v = z2[q];
                    __stcs(o2 + q, make_double2(v.x * rn, v.y * rn));
                }
            } else {
                for (int q = lane; q < K; q += 32) __stcs(zb + q, zs[q] * rn);
            }
        }
    } else if (exmask == 0 && Kp == K && a.ldz == K) {
        const int n = nr * K;
        int e = lane;
        for (; e + 96 < n; e += 128) {
            const double v0 = zs[e], v1 = zs[e + 32], v2 = zs[e + 64], v3 = zs[e + 96];
            __stcs(zb + e, v0);
            __stcs(zb + e + 32, v1);
            __stcs(zb + e + 64, v2);
            __stcs(zb + e + 96, v3);
        }
        for (; e < n; e += 32) __stcs(zb + e, zs[e]);
    } else {
        for (int i = 0; i < nr; ++i, zb += a.ldz) {
            if ((exmask >> i) & 1u) continue;
            const double *zi = zs + i * Kp;
            for (int q = lane; q < K; q += 32) __stcs(zb + q, zi[q]);
        }
    }
    __syncwarp();
}

// phase 1.5: rows of (flat_max, kLongRow] entries, one warp each (listed from
// the back of the long-row list); phase 2: blocks of R consecutive rows
__device__ void rows_flat(const EmbedArgs &a, double *zs, double *xs) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned n_med = a.n_long[5];
    const int64_t n_rows = a.row_end - a.row_begin;
    for (;;) {
        unsigned tw = 0;
        if (lane == 0) tw = atomicAdd(&a.work[3], 1u);
        tw = __shfl_sync(full, tw, 0);
        if (tw >= n_med) break;
        flat_block(a, (int64_t)a.long_list[n_rows - 1 - tw], 1, kLongRow, zs, xs);
    }
    const int R = a.flat_rows;
    const int64_t n_chunks = (n_rows + R - 1) / R;
    unsigned tw = 0;
    if (lane == 0) tw = atomicAdd(&a.work[1], 1u);
    int64_t t = __shfl_sync(full, tw, 0);
    while (t < n_chunks) {
        // the next block's id is fetched now: its round trip overlaps this block
        if (lane == 0) tw = atomicAdd(&a.work[1], 1u);
        const int64_t r0 = a.row_begin + t * R;
        flat_block(a, r0, (int)min((int64_t)R, a.row_end - r0), a.flat_max, zs, xs);
        t = __shfl_sync(full, tw, 0);
    }
}

template <int KP, bool TAB, int NT, bool FLAT = false>
__global__ void __launch_bounds__(NT, FLAT ? 3 : 65536 / (NT * 64)) k_embed(EmbedArgs a, int n_tab) {
    constexpr int kWarps = NT / 32;
    // values implicit (all exactly 1.0) when the sort path says so: skip the val stream
    if (a.val_flags && a.val_flags[0] == 0 && a.val_flags[1] == 0) a.val = nullptr;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ double dred[33];
    __shared__ int task;
    const int kt_max = min(a.k, kKTile);
    // per-warp tile: a K-vector (kt_max) or a flat block (flat_rows x kp)
    const int wst = FLAT ? (max(kt_max, a.flat_rows * a.kp) + 1) & ~1 : kt_max;
    double *zsm = reinterpret_cast<double *>(dsm);    // [warps][wst]
    double *xsm = zsm + (size_t)kWarps * wst;     // [warps][32]
    const int wid = threadIdx.x >> 5;
    NodeTab tab{nullptr, nullptr};
    if (TAB) {
        // stage the node table on chip: g (8 B) and the label (1 B) per node
        double *tg = xsm + (size_t)kWarps * 32;
        signed char *tl = reinterpret_cast<signed char *>(tg + ((n_tab + 1) & ~1));  // 16-B aligned
        if (a.tab_g) {
            // compact 9-byte/node source (written by the bitmap row pass):
            // 16-byte loads, 4 in flight per thread, so staging is not a
            // chain of dependent L2 round trips
            const int n2 = n_tab / 2;
            const double2 *src = reinterpret_cast<const double2 *>(a.tab_g);
            double2 *dst = reinterpret_cast<double2 *>(tg);
            for (int j0 = threadIdx.x; j0 < n2; j0 += 4 * blockDim.x) {
                double2 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + u * blockDim.x;
                    if (j < n2) v[u] = __ldcg(src + j);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + u * blockDim.x;
                    if (j < n2) dst[j] = v[u];
                }
            }
            if ((n_tab & 1) && threadIdx.x == 0) tg[n_tab - 1] = __ldcg(a.tab_g + n_tab - 1);
            const int n16 = n_tab / 16;
            const int4 *lsrc = reinterpret_cast<const int4 *>(a.tab_lab);
            int4 *ldst = reinterpret_cast<int4 *>(tl);
            for (int j = threadIdx.x; j < n16; j += blockDim.x) ldst[j] = __ldcg(lsrc + j);
            for (int j = n16 * 16 + threadIdx.x; j < n_tab; j += blockDim.x) tl[j] = a.tab_lab[j];
        } else {
            for (int j = threadIdx.x; j < n_tab; j += blockDim.x) {
                const double2 rc = __ldg(a.rec + j);
                tg[j] = rc.y;
                tl[j] = (signed char)(int)(unsigned)(unsigned long long)__double_as_longlong(rc.x);
            }
        }
        tab.g = tg;
        tab.lab = tl;
        __syncthreads();
    }
    // phase 1: long rows, one CTA each
    const unsigned n_long = *a.n_long;
    for (;;) {
        if (threadIdx.x == 0) task = (int)atomicAdd(&a.work[0], 1u);
        __syncthreads();
        int t = task;
        __syncthreads();
        if (t >= (int)n_long) break;
        row_long(a, a.long_list[t], zsm, xsm, dred);
    }
    // phase 2: every warp grabs its own chunks of rows, one warp per row (no
    // CTA-wide barrier: row lengths vary, so a barrier per chunk would idle
    // the warps that drew short rows)
    if (FLAT) {
        rows_flat(a, zsm + (size_t)wid * wst, xsm + wid * 32);
        return;
    }
    const int64_t n_rows = a.row_end - a.row_begin;
    const int64_t n_chunks = (n_rows + kRowChunk - 1) / kRowChunk;
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned tw = 0;
        if (lane == 0) tw = atomicAdd(&a.work[1], 1u);
        const int64_t t = __shfl_sync(0xffffffffu, tw, 0);
        if (t >= n_chunks) break;
        // chunk t = rows t, t + n_chunks, t + 2 n_chunks, ...: long rows
        // cluster in id ranges of power-law graphs, a strided chunk spreads
        // them over many warps
        for (int64_t r = a.row_begin + t; r < a.row_end; r += n_chunks) {
            int64_t s, e;
            row_extent(a, r, s, e);
            if (e - s > kLongRow) continue;
            if (KP > 0)
                row_regs<(KP > 0 ? KP : 1), TAB>(a, tab, r);
            else
                row_smem(a, r, zsm + wid * wst, xsm + wid * 32);
        }
    }
}

__global__ void k_embed_classify(const int64_t *__restrict__ row_ptr, const unsigned *__restrict__ row_cnt,
                                 int64_t rb, int64_t re, int64_t flat_max, unsigned *__restrict__ list,
                                 unsigned *__restrict__ ctr) {
    // long rows (> kLongRow) listed from the front (count ctr[0]); with flat
    // blocks, medium rows (flat_max, kLongRow] from the back (count ctr[5])
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n = re - rb;
    const int64_t n_round = (n + 31) & ~int64_t(31);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        bool lng = false, med = false;
        int64_t r = rb + i;
        if (i < n) {
            int64_t L = row_cnt ? (int64_t)row_cnt[r] : row_ptr[r + 1] - row_ptr[r];
            lng = L > kLongRow;
            med = !lng && L > flat_max;
        }
        unsigned m = __ballot_sync(0xffffffffu, lng);
        if (m) {
            int leader = __ffs(m) - 1;
            unsigned base = 0;
            if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(ctr, __popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (lng) list[base + __popc(m & lanemask_lt())] = (unsigned)r;
        }
        m = __ballot_sync(0xffffffffu, med);
        if (m) {
            int leader = __ffs(m) - 1;
            unsigned base = 0;
            if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(ctr + 5, __popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (med) list[n - 1 - (base + __popc(m & lanemask_lt()))] = (unsigned)r;
        }
    }
}

// node records {label bits, g = s_j / n_{Y_j}}; label -1 for unlabeled nodes
__global__ void k_node_rec(const int32_t *__restrict__ y32, const double *__restrict__ inv,
                           const double *__restrict__ scale, int64_t n, double2 *__restrict__ rec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const int lab = y32[j];
        double g = 0.0;
        if (lab >= 0) g = scale ? scale[j] * inv[lab] : inv[lab];
        rec[j] = make_double2(__longlong_as_double((long long)(unsigned)lab), g);
    }
}

// Embed workspace: [4] counters (n_long, work0, work1), the long-row list and
// the node-record table.  A CSR builder that already knows row lengths and
// degrees (the bitmap path) fills them itself and calls embed(prepared=1).
struct EmbedScratch {
    unsigned *ctr, *list;
    double2 *rec;
    double *tab_g;
    signed char *tab_lab;
};

static EmbedScratch carve_embed(Carver &cv, int64_t n_rows, int64_t n_cols) {
    EmbedScratch s;
    s.ctr = cv.take<unsigned>(8);
    s.list = cv.take<unsigned>((size_t)n_rows + 1);
    s.rec = cv.take<double2>((size_t)n_cols + 1);
    const bool small = n_cols <= kTabMax;
    s.tab_g = cv.take<double>(small ? (size_t)n_cols + 1 : 0);
    s.tab_lab = cv.take<signed char>(small ? (size_t)n_cols + 1 : 0);
    return s;
}

size_t embed_workspace(int64_t n_rows, int64_t n_cols) {
    Carver cv(nullptr);
    carve_embed(cv, n_rows, n_cols);
    return cv.bytes();
}

int embed_long_row() { return kLongRow; }

// shared-memory budget of one warp's flat block (bytes); 0 disables the flat
// phase 2 (test hook GEE_DEBUG_EMBED_FLAT_BYTES)
static thread_local int t_flat_bytes = 8192;
constexpr int kFlatBytesMax = 24576;

int set_embed_flat_bytes(int v) {
    const int old = t_flat_bytes;
    t_flat_bytes = v < 0 ? 0 : (v > kFlatBytesMax ? kFlatBytesMax : v);
    return old;
}

// longest row a flat block takes; longer rows get a warp (or, beyond
// kLongRow, a CTA) of their own (test hook GEE_DEBUG_EMBED_FLAT_ROWMAX)
static thread_local int t_flat_max = 256;

int set_embed_flat_rowmax(int v) {
    const int old = t_flat_max;
    t_flat_max = v < 1 ? 1 : (v > kLongRow ? kLongRow : v);
    return old;
}

void embed_scratch(void *ws, int64_t n_rows, int64_t n_cols, unsigned **ctr, unsigned **list, double2 **rec,
                   double **tab_g, signed char **tab_lab) {
    Carver cv(ws);
    EmbedScratch s = carve_embed(cv, n_rows, n_cols);
    *ctr = s.ctr;
    *list = s.list;
    *rec = s.rec;
    *tab_g = n_cols <= kTabMax ? s.tab_g : nullptr;
    *tab_lab = n_cols <= kTabMax ? s.tab_lab : nullptr;
}

int embed(const int64_t *row_ptr, const unsigned *row_cnt, const int32_t *col, const double *val,
          const unsigned *val_flags, const unsigned char *row_flag, int64_t rb, int64_t re, int64_t n_cols,
          const int32_t *y32, const double *inv, const double *scale, int k, unsigned flags, double *z, int64_t ldz,
          void *ws, size_t ws_bytes, int32_t *err, cudaStream_t st, int prepared) {
    const int64_t n = re - rb;
    Carver cv(ws);
    EmbedScratch sc = carve_embed(cv, n, n_cols);
    unsigned *ctr = sc.ctr, *list = sc.list;
    double2 *rec = sc.rec;
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    if (n <= 0) return GEE_OK;
    EmbedArgs a;
    // K > 8: flat blocks of R rows (R x kp doubles within the warp budget)
    a.kp = k < 32 ? (k | 1) : k;
    a.flat_rows = 0;
    a.flat_max = kLongRow;
    if (k > 8 && k <= kKTile) {
        // a power of two, so the correlation's lanes-per-row split uses every lane
        const int r = t_flat_bytes / (8 * a.kp);
        a.flat_rows = r >= 16 ? 16 : r >= 8 ? 8 : r >= 4 ? 4 : r >= 2 ? 2 : r;
        if (a.flat_rows > 0) a.flat_max = t_flat_max;
    }
    if (!prepared) {
        GEE_CHECK_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(unsigned), st));
        k_node_rec<<<grid_for(n_cols, 256, 8), 256, 0, st>>>(y32, inv, (flags & GEE_LAPLACIAN) ? scale : nullptr,
                                                              n_cols, rec);
        GEE_CHECK_LAUNCH("k_node_rec");
        k_embed_classify<<<grid_for(n, 256, 8), 256, 0, st>>>(row_ptr, row_cnt, rb, re, a.flat_max, list, ctr);
        GEE_CHECK_LAUNCH("k_embed_classify");
    }
    a.row_ptr = row_ptr;
    a.row_cnt = row_cnt;
    a.col = col;
    a.val = val;
    a.row_begin = rb;
    a.row_end = re;
    a.rec = rec;
    a.scale = scale;
    a.k = k;
    a.flags = flags;
    a.z = z;
    a.ldz = ldz;
    a.err = err;
    a.long_list = list;
    a.n_long = ctr;
    a.work = ctr + 1;
    a.val_flags = val_flags;
    a.row_flag = row_flag;
    // prepared by the bitmap row pass: the compact table is valid
    a.tab_g = (prepared && n_cols <= kTabMax) ? sc.tab_g : nullptr;
    a.tab_lab = (prepared && n_cols <= kTabMax) ? sc.tab_lab : nullptr;
    const int kt_max = k < kKTile ? k : kKTile;
    const int wst = a.flat_rows > 0 ? ((kt_max > a.flat_rows * a.kp ? kt_max : a.flat_rows * a.kp) + 1) & ~1 : kt_max;
    // small graphs with K <= 8: node table (9 B/node) staged in shared memory
    // by one 1024-thread CTA per SM (one table copy serves 32 warps)
    const bool tab = k <= 8 && n_cols <= kTabMax;
    const int nt = tab ? kTabThreads : kEmbedThreads;
    const size_t base_smem = sizeof(double) * (size_t)(nt / 32) * ((size_t)wst + 32);
    const size_t smem = base_smem + (tab ? 9 * (size_t)n_cols + 32 : 0);
    static PerDevice attr;
    if (!attr.done()) {
        size_t mx = sizeof(double) * (size_t)kEmbedWarps * ((size_t)kFlatBytesMax / 8 + 32);
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<0, false, kEmbedThreads>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<0, false, kEmbedThreads, true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
        const int tmx = (int)(sizeof(double) * (kTabThreads / 32) * (8 + 32) + 9 * kTabMax + 32);
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<1, true, kTabThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<2, true, kTabThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<4, true, kTabThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_embed<8, true, kTabThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, tmx));
        attr.mark();
    }
    int occ = 0;
    const unsigned grid_cap = (unsigned)num_sms() * 8;
    unsigned grid;
    const int n_tab = tab ? (int)n_cols : 0;
#define GEE_LAUNCH_EMBED(KP, TB, NT, ...)                                                                    \
    do {                                                                                                     \
        GEE_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_embed<KP, TB, NT, ##__VA_ARGS__>, \
                                                                     NT, smem));                             \
        grid = (unsigned)num_sms() * (unsigned)(occ > 0 ? occ : 1);                                          \
        if (grid > grid_cap) grid = grid_cap;                                                                \
        k_embed<KP, TB, NT, ##__VA_ARGS__><<<grid, NT, smem, st>>>(a, n_tab);                                \
    } while (0)
    if (k <= 1) {
        if (tab) GEE_LAUNCH_EMBED(1, true, kTabThreads); else GEE_LAUNCH_EMBED(1, false, kEmbedThreads);
    } else if (k <= 2) {
        if (tab) GEE_LAUNCH_EMBED(2, true, kTabThreads); else GEE_LAUNCH_EMBED(2, false, kEmbedThreads);
    } else if (k <= 4) {
        if (tab) GEE_LAUNCH_EMBED(4, true, kTabThreads); else GEE_LAUNCH_EMBED(4, false, kEmbedThreads);
    } else if (k <= 8) {
        if (tab) GEE_LAUNCH_EMBED(8, true, kTabThreads); else GEE_LAUNCH_EMBED(8, false, kEmbedThreads);
    } else if (a.flat_rows > 0) {
        GEE_LAUNCH_EMBED(0, false, kEmbedThreads, true);
    } else {
        GEE_LAUNCH_EMBED(0, false, kEmbedThreads);
    }
#undef GEE_LAUNCH_EMBED
    (void)nt;
    GEE_CHECK_LAUNCH("k_embed");
    return GEE_OK;
}

}  // namespace gee
