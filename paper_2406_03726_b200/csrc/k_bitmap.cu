// k_bitmap.cu -- the whole encode for unit-weight graphs with at most
// kBmMax nodes and K <= 8 classes (configs 0/1: unweighted SBM, N = 10^4).
//
// With every weight equal to 1.0 a stored value is the multiplicity of its
// (row, col) pair, and the order duplicates are summed in is irrelevant (sums
// of ones are exact).  When no pair repeats, the CSR row of r is the set of
// its columns, its degree is the set size and
//     Z[r, q] = s_r * (1/n_q) * sum_{c in row r, Y_c = q} s_c   (+ the A+I diagonal),
// a product of the 0/1 adjacency matrix S with the N x K matrix X[c, q] =
// s_c [Y_c = q].  The encode needs only the N x N adjacency bitmap -- Np^2/8
// bytes, 13 MB at N = 10^4 -- which stays resident in the 126 MB L2; the CSR
// itself is never materialised (gee_encode_edges returns Z only).  The
// bitmap is stored as 128 x 128-bit tiles (see bm_index).  Four kernels, each
// launched with programmatic dependent launch behind the previous one:
//   k_bm_set   the labels (validated, y32, class histogram) and one read of the
//              int64 edge list, a pair of entries per lane (16-byte loads):
//              each entry sets bit (r, c) of U with a global reduction
//              (RED.OR, no return).  Runs of entries on the same bitmap word
//              (a row-major list) OR-combine first, in the lane and then by a
//              segmented warp scan, so a sorted list costs about one
//              reduction per touched word.
//   k_bm_sym   undirected lists: S = U | U^T in place, one CTA per pair of
//              128 x 128 tiles, 32 x 32 transposes by warp shuffles; row
//              popcounts u_r, popc(U) (= E exactly when no pair repeats in the
//              list) and pairs present in both directions (U & U^T off the
//              diagonal, the other way a pair repeats in the stream).
//              (Directed lists: k_bm_scan, one warp per row, instead.)
//   k_bm_table thread per node: d_r = u_r (+1 under A+I), s_r = d_r^-1/2, and
//              X^T's column r as 7 base-256 digits of s_r * 2^55 in the rows
//              of class Y_r, stored as the GEMM's shared-memory B tiles.
//   k_bm_gemm  S x X on the 5th-generation tensor cores (tcgen05.mma
//              kind::i8, u8 x u8 -> s32): A = S's bits expanded to bytes and
//              written straight into TMEM (tcgen05.st), B = the X^T tile
//              bulk-copied into shared memory; persistent stream-K over
//              (128-row tile, 256-column K step).  Integer accumulation is
//              exact, so sum_c S_rc s_c is known to 2^-55 per term whatever
//              the order; stream-K partials are integer too.  The epilogue
//              recombines the digits in f64 and applies 1/n_q, the diagonal,
//              s_r and the correlation.
// Rare path (some pair repeats): k_bm_gemm first recomputes the stream
// lengths by atomics, the node table and, for rows with repeats, per-class
// sums of g = s_c/n_q over every stream entry, in grid-wide phases (all CTAs
// are co-resident: cooperative launch); those rows take their sums from there.
#include <algorithm>

#include "gee_common.cuh"

namespace gee {

#ifdef GEE_TRACE
__device__ unsigned long long g_trace[10][64];
__device__ unsigned long long g_trace_end[160];
__device__ unsigned long long g_trace_cta[160][12];  // entry, setup done, last MMA issued, epilogue done, seg0 acc ready, seg0 published, first step expanded
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
}
#define TRACE(slot, i) \
    do {               \
        if (blockIdx.x == 0 && (i) < 64) g_trace[slot][i] = gtime(); \
    } while (0)
// kernel spans: [k][0] first CTA start, [k][1] first dependency wait passed, [k][2] last CTA end
__device__ unsigned long long g_kspan[8][3];
#define KSPAN(k, j)                                                              \
    do {                                                                         \
        if (threadIdx.x == 0) {                                                  \
            if ((j) < 2) atomicMin(&g_kspan[k][j], gtime());                     \
            else atomicMax(&g_kspan[k][j], gtime());                             \
        }                                                                        \
    } while (0)
#else
#define KSPAN(k, j) \
    do {            \
    } while (0)
#define TRACE(slot, i) \
    do {               \
    } while (0)
#endif

constexpr int kBmMax = 16384;   // nodes: bitmap Np^2/8 <= 32 MB (L2-resident)
constexpr int kBlk = 256;       // the bitmap's side is padded to a multiple of 256
constexpr int kSetThreads = 512;
constexpr int kKMax = 8;        // classes
constexpr int kPopParts = 64;   // spread counters for popc(U)
constexpr int kDig = 7;         // base-256 digits of s * 2^55
constexpr int kTM = 128;        // GEMM rows per tile (TMEM lanes)
constexpr int kTK = 256;        // GEMM columns per K step (two 128-byte swizzle atoms)

struct BmArgs {
    int n, Wp, Np;            // nodes, bitmap words per row (multiple of 8), Wp*32
    // Rows held here: [row0, row0 + nloc), bitmap rows Nlp (a multiple of
    // 128).  The single-GPU encode holds every row (row0 = 0, nloc = n,
    // Nlp = Np); a row shard (multi-GPU, bitmap_shard_*) holds its range
    // and reads the degrees of every node from deg_all.  ucnt, len, zacc, z
    // and the bitmap are indexed by local row r - row0; labels, the node
    // table and X^T by global node.
    int row0, nloc, Nlp;
    int shard;
    const unsigned *deg_all;  // [n] shard encode: stream lengths of every row (NULL without Laplacian)
    int64_t E;
    int directed;
    unsigned *bm;             // [Np][Wp]
    unsigned *ucnt;           // [nloc] distinct columns per row
    unsigned *len;            // [nloc] stream lengths (rare path)
    unsigned *cnt;            // [kKMax] class histogram
    unsigned *mdone;          // [Nlp/128] K steps accumulated per GEMM row tile
    unsigned *flags;          // [0] pair in both directions, [1] rare-path barrier, [3] table barrier
    unsigned *upop;           // [kPopParts * 32] popc(U) partial sums, 128 B apart
    unsigned char *xt;        // [NB][Np] X^T digits (K-major B operand)
    int nbx;                  // NB: X columns (kDig * K padded to 16/32/64)
    int32_t *cpart;           // [grid][2][128][NB] stream-K partial sums (slab per CTA segment)
    double *zacc;             // [nloc][kKMax] rare path class sums
    const int64_t *labels;
    int32_t *y32;
    int64_t *counts;
    double *inv;
    double *deg, *scale;
    double *tab_g;
    signed char *tab_lab;
    unsigned flags_opts;      // GEE_LAPLACIAN | GEE_DIAGONAL | GEE_CORRELATION
    double *z;
    int k;
    int32_t *err;
};

// programmatic dependent launch: a kernel launched with the PDL attribute
// may start while its predecessor drains; it waits here before touching the
// predecessor's outputs, and the predecessor lets it launch once its CTAs
// have written everything
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned lanemask_le() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
    return m;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_gpu(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// The bitmap is stored in 128 x 128-bit tiles (2 KB, row-major inside: a
// row's 4 words are 16 contiguous bytes), tile (R, K) at (R * Wp/4 + K) * 2 KB,
// so one GEMM K step of a 128-row tile is one contiguous bulk copy.
__device__ __forceinline__ unsigned bm_index(const BmArgs &a, unsigned r, unsigned w) {
    return (((r >> 7) * (unsigned)(a.Wp >> 2) + (w >> 2)) << 9) + ((r & 127u) << 2) + (w & 3u);
}

// X^T is stored as the K-step tiles of the GEMM's B operand, each exactly its
// shared-memory image (NB rows x 128 B, 128-byte swizzle: 16-byte chunk c of
// row j at chunk c ^ (j & 7), 8-row groups 1 KB apart)
__device__ __forceinline__ size_t xt_index(const BmArgs &a, int j, int c) {
    const int ks = c >> 7, cin = c & 127;
    return (size_t)ks * a.nbx * 128 + (j >> 3) * 1024 + (j & 7) * 128 + ((((cin >> 4) ^ (j & 7))) << 4) + (cin & 15);
}

// 32 x 32 bit transpose across a warp: out(lane i) bit j = in(lane j) bit i
__device__ __forceinline__ unsigned transpose32(unsigned x, int lane) {
    const unsigned m16 = 0x0000ffffu, m8 = 0x00ff00ffu, m4 = 0x0f0f0f0fu, m2 = 0x33333333u, m1 = 0x55555555u;
#define GEE_TSTAGE(J, M)                                                           \
    {                                                                              \
        const unsigned y = __shfl_xor_sync(0xffffffffu, x, J);                     \
        x = (lane & J) ? ((x & ~M) | ((y >> J) & M)) : ((x & M) | ((y & M) << J)); \
    }
    GEE_TSTAGE(16, m16)
    GEE_TSTAGE(8, m8)
    GEE_TSTAGE(4, m4)
    GEE_TSTAGE(2, m2)
    GEE_TSTAGE(1, m1)
#undef GEE_TSTAGE
    return x;
}

// NQ independent 32 x 32 transposes, stage-major
template <int NQ>
__device__ __forceinline__ void transpose32_n(unsigned (&x)[NQ], int lane) {
    // byte-granular stages: one byte permute each (lane-dependent selector)
    {
        const unsigned sel = (lane & 16) ? 0x3276u : 0x5410u;
        unsigned y[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) y[q] = __shfl_xor_sync(0xffffffffu, x[q], 16);
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q] = __byte_perm(x[q], y[q], sel);
    }
    {
        const unsigned sel = (lane & 8) ? 0x3715u : 0x6240u;
        unsigned y[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) y[q] = __shfl_xor_sync(0xffffffffu, x[q], 8);
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q] = __byte_perm(x[q], y[q], sel);
    }
#pragma unroll
    for (int J = 4; J >= 1; J >>= 1) {
        const unsigned M = J == 4 ? 0x0f0f0f0fu : J == 2 ? 0x33333333u : 0x55555555u;
        unsigned y[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) y[q] = __shfl_xor_sync(0xffffffffu, x[q], J);
        const bool hi = (lane & J) != 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q] = hi ? ((x[q] & ~M) | ((y[q] >> J) & M)) : ((x[q] & M) | ((y[q] & M) << J));
    }
}

// node-table entry of row r from its stream length L (k_bm_sym / k_bm_scan /
// the rare path); y32 and the histogram are complete when this runs
__device__ __forceinline__ void node_entry(const BmArgs &a, int r, unsigned L, int lab, unsigned nk) {
    double sr = 1.0;
    if (a.flags_opts & GEE_LAPLACIAN) {
        const double d = (double)L + ((a.flags_opts & GEE_DIAGONAL) ? 1.0 : 0.0);
        a.deg[r] = d;
        sr = laplacian_scale(d, a.err);
        a.scale[r] = sr;
    }
    double g = 0.0;
    if (lab >= 0) {
        const double inv = __ddiv_rn(1.0, (double)nk);  // 1/n_k (embedding.py:106)
        g = (a.flags_opts & GEE_LAPLACIAN) ? sr * inv : inv;
        // X[r, lab] = s_r as 7 base-256 digits of floor(s_r * 2^55) (s_r <= 1)
        const unsigned long long T = __double2ull_rz(sr * 0x1p55);
#pragma unroll
        for (int d = 0; d < kDig; ++d) a.xt[xt_index(a, lab * kDig + d, r)] = (unsigned char)(T >> (8 * d));
    }
    a.tab_g[r] = g;
    a.tab_lab[r] = (signed char)lab;
}

__device__ __forceinline__ void node_entry(const BmArgs &a, int r, unsigned L) {
    const int lab = __ldcg(a.y32 + r);
    node_entry(a, r, L, lab, lab >= 0 ? __ldcg(a.cnt + lab) : 0u);
}

// class counts and 1/n_k as the reference's LabelVector / W (run once)
__device__ __forceinline__ void write_counts(const BmArgs &a, int t) {
    if (t < a.k) {
        const unsigned m = __ldcg(a.cnt + t);
        a.counts[t] = (int64_t)m;
        a.inv[t] = m ? __ddiv_rn(1.0, (double)m) : 0.0;
    }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSetThreads) k_bm_set(const int64_t *__restrict__ rows,
                                                        const int64_t *__restrict__ cols, BmArgs a) {
    __shared__ unsigned sh_hist[kKMax];
    const int lane = threadIdx.x & 31;
    KSPAN(0, 0);
    // k_bm_sym may be scheduled as this grid drains; it waits for its completion
    pdl_trigger();
    // labels: int64 -> int32 (-1 = unlabeled), validated, histogrammed
    if (threadIdx.x < kKMax) sh_hist[threadIdx.x] = 0;
    __syncthreads();
    for (int base = blockIdx.x * blockDim.x; base < a.n; base += gridDim.x * blockDim.x) {
        const int i = base + threadIdx.x;
        int lab = -1;
        if (i < a.n) {
            int64_t v = a.labels[i];
            if (v < -1 || v >= a.k) {
                raise_err(a.err, GEE_ERR_LABEL);
                v = -1;
            }
            lab = (int)v;
            a.y32[i] = lab;
        }
        for (int q = 0; q < a.k; ++q) {
            const unsigned c = __popc(__ballot_sync(0xffffffffu, lab == q));
            if (lane == 0 && c) atomicAdd(&sh_hist[q], c);
        }
    }
    __syncthreads();
    if (threadIdx.x < a.k && sh_hist[threadIdx.x]) atomicAdd(&a.cnt[threadIdx.x], sh_hist[threadIdx.x]);

    // Each lane takes a pair of consecutive stream entries (16-byte loads of
    // rows and cols), so a warp covers 64 consecutive entries.  Runs of
    // entries on the same bitmap word OR-combine: inside the pair, then across
    // lanes with one segmented scan over the lanes' last runs; each run issues
    // one reduction (RED.OR, no return value).  A sorted list costs about one
    // reduction per touched word.
    constexpr unsigned INV = 0xffffffffu;
    const int64_t E = a.E;
    const unsigned le = lanemask_le();
    const bool vec = (((uintptr_t)rows | (uintptr_t)cols) & 15) == 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    // this lane's pair at e (row INV = past the end); only the low 32 bits of
    // the int64 indices are used (n <= kBmMax)
    auto fetch = [&](int64_t e, unsigned &r0, unsigned &r1, unsigned &c0, unsigned &c1) {
        r0 = r1 = INV;
        c0 = c1 = 0;
        if (vec && e + 1 < E) {
            const longlong2 rv = __ldcs(reinterpret_cast<const longlong2 *>(rows + e));
            const longlong2 cv = __ldcs(reinterpret_cast<const longlong2 *>(cols + e));
            r0 = (unsigned)rv.x, r1 = (unsigned)rv.y, c0 = (unsigned)cv.x, c1 = (unsigned)cv.y;
        } else {
            if (e < E) r0 = (unsigned)rows[e], c0 = (unsigned)cols[e];
            if (e + 1 < E) r1 = (unsigned)rows[e + 1], c1 = (unsigned)cols[e + 1];
        }
    };
    // global row -> local bitmap row; an entry outside this bitmap's rows or
    // columns is an edge-range error, dropped (EdgeList validates first)
    auto localise = [&](unsigned &r0, unsigned &r1, unsigned &c0, unsigned &c1) {
        const unsigned nl = (unsigned)a.nloc, nc = (unsigned)a.n;
        if (r0 != INV) {
            r0 -= (unsigned)a.row0;
            if (r0 >= nl || c0 >= nc) {
                raise_err(a.err, GEE_ERR_EDGE_RANGE);
                r0 = INV;
            }
        }
        if (r1 != INV) {
            r1 -= (unsigned)a.row0;
            if (r1 >= nl || c1 >= nc) {
                raise_err(a.err, GEE_ERR_EDGE_RANGE);
                r1 = INV;
            }
        }
        if (r0 == INV) r0 = r1, c0 = c1, r1 = INV;  // an empty first slot only ends the list
    };
    int64_t base = (int64_t)blockIdx.x * blockDim.x * 2;
    unsigned r0, r1, c0, c1;
    fetch(base + threadIdx.x * 2, r0, r1, c0, c1);
    // software-pipelined: the next pair is in flight while this one is scanned
    for (; base < E; base += stride) {
        unsigned nr0, nr1, nc0, nc1;
        fetch(base + stride + threadIdx.x * 2, nr0, nr1, nc0, nc1);
        localise(r0, r1, c0, c1);
        const unsigned k0 = r0 != INV ? bm_index(a, r0, c0 >> 5) : INV;
        const unsigned k1 = r1 != INV ? bm_index(a, r1, c1 >> 5) : INV;
        const unsigned b0 = r0 != INV ? 1u << (c0 & 31) : 0u;
        const unsigned b1 = r1 != INV ? 1u << (c1 & 31) : 0u;
        const bool two = k1 != INV && k1 != k0;  // two distinct runs in this pair
        const unsigned kf = k0, kl = k1 == INV ? k0 : k1;
        const unsigned bf = two ? b0 : (b0 | b1);
        const unsigned bl = two ? b1 : (b0 | b1);
        const unsigned kl_prev = __shfl_up_sync(0xffffffffu, kl, 1);
        const unsigned kf_next = __shfl_down_sync(0xffffffffu, kf, 1);
        // the first run continues the previous lane's last run
        const bool cont = lane > 0 && kf != INV && kl_prev == kf;
        const bool head = !(cont && !two);
        const int start = 31 - __clz(__ballot_sync(0xffffffffu, head) & le);
        unsigned incl = bl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane - o >= start) incl |= y;
        }
        const unsigned prev = __shfl_up_sync(0xffffffffu, incl, 1);
#ifndef GEE_NORED  // timing experiment only: no bitmap reductions
        if (two) atomicOr(&a.bm[kf], bf | (cont ? prev : 0u));
        const bool tail = lane == 31 || kf_next != kl;
        if (tail && kl != INV) atomicOr(&a.bm[kl], incl);
#else
        if (two && kf == 0x7fffffffu) a.bm[0] = bf | prev | incl;
#endif
        r0 = nr0, r1 = nr1, c0 = nc0, c1 = nc1;
    }
    KSPAN(0, 2);
}

// S = U | U^T for the block pair (BI, BJ), BI <= BJ, in place.  Blocks are
// the bitmap's 128 x 128-bit tiles, so each side is one contiguous 2 KB tile
// (thread t = tile row t, one 16-byte load and store per side).
constexpr int kSB = 128;
__global__ void __launch_bounds__(kSB) k_bm_sym(BmArgs a) {
    constexpr int kW = kSB / 32;  // words per tile row
    __shared__ unsigned sat[kSB][kW + 1], sbt[kSB][kW + 1];
    __shared__ unsigned red[kSB / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // linear index -> (BI, BJ) on the upper triangle
    const unsigned x = blockIdx.x;
    unsigned bj = (unsigned)((sqrtf(8.0f * x + 1.0f) - 1.0f) * 0.5f);
    KSPAN(1, 0);
    pdl_wait();
    KSPAN(1, 1);
    // k_bm_table may be scheduled as this grid drains (it reads only k_bm_set's
    // outputs before waiting for this grid)
    pdl_trigger();
    while ((bj + 1) * (bj + 2) / 2 <= x) ++bj;
    while (bj * (bj + 1) / 2 > x) --bj;
    const unsigned bi = x - bj * (bj + 1) / 2;
    const int ra = bi * kSB + t, rb = bj * kSB + t;
    uint4 *pa = reinterpret_cast<uint4 *>(a.bm + bm_index(a, ra, bj * kW));
    uint4 *pb = reinterpret_cast<uint4 *>(a.bm + bm_index(a, rb, bi * kW));
    const bool same = bi == bj;
    const uint4 av4 = __ldcg(pa);
    const uint4 bv4 = same ? av4 : __ldcg(pb);
    unsigned av[kW] = {av4.x, av4.y, av4.z, av4.w}, bv[kW] = {bv4.x, bv4.y, bv4.z, bv4.w};
    // sub-tile (w, q) transposes into row q*32+lane, word w of its mirror;
    // 8 independent transposes, stage-major so the shuffles overlap
    unsigned pu = 0;  // popc of the U words read here (each U word is read once)
    {
        unsigned xx[2 * kW];
#pragma unroll
        for (int q = 0; q < kW; ++q) {
            pu += __popc(av[q]) + (same ? 0u : __popc(bv[q]));
            xx[q] = av[q];
            xx[kW + q] = bv[q];
        }
        // an all-zero 32 x 128 slice transposes to zeros (one side of every
        // pair is empty for a triangular list): skip its shuffles
        const bool az = !__any_sync(0xffffffffu, (av[0] | av[1] | av[2] | av[3]) != 0u);
        const bool bz = !__any_sync(0xffffffffu, (bv[0] | bv[1] | bv[2] | bv[3]) != 0u);
        if (!az && !bz) {
            transpose32_n<2 * kW>(xx, lane);
        } else if (!az) {
            transpose32_n<kW>(*reinterpret_cast<unsigned(*)[kW]>(&xx[0]), lane);
        } else if (!bz) {
            transpose32_n<kW>(*reinterpret_cast<unsigned(*)[kW]>(&xx[kW]), lane);
        }
#pragma unroll
        for (int q = 0; q < kW; ++q) {
            sat[q * 32 + lane][w] = xx[q];
            sbt[q * 32 + lane][w] = xx[kW + q];
        }
    }
    pu = warp_sum_u(pu);
    if (lane == 0) red[w] = pu;
    __syncthreads();
    unsigned mut = 0, ca = 0, cb = 0;
    unsigned sv[kW], uv[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) {
        const unsigned tb = sbt[t][q], ta = sat[t][q];
        sv[q] = av[q] | tb;
        uv[q] = bv[q] | ta;
        unsigned m = av[q] & tb;
        if (same && q == w) m &= ~(1u << lane);  // the diagonal is its own mirror
        mut |= m;
        ca += __popc(sv[q]);
        cb += __popc(uv[q]);
    }
    *pa = make_uint4(sv[0], sv[1], sv[2], sv[3]);
    if (!same) *pb = make_uint4(uv[0], uv[1], uv[2], uv[3]);
    if (t == 0) {
        unsigned tot = 0;
#pragma unroll
        for (int i = 0; i < kSB / 32; ++i) tot += red[i];
        if (tot) atomicAdd(a.upop + (blockIdx.x % kPopParts) * 32, tot);  // spread: one address serialises
    }
    // rows >= n are padding and stay empty
    if (ca) atomicAdd(&a.ucnt[ra], ca);
    if (cb && !same) atomicAdd(&a.ucnt[rb], cb);
    if (__syncthreads_or(mut != 0) && t == 0) a.flags[0] = 1u;
    KSPAN(1, 2);
}

// node table from the distinct counts: d_r, s_r, X^T digits, g_r (thread per row)
__global__ void __launch_bounds__(256) k_bm_table(BmArgs a) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    // labels and class sizes are k_bm_set's (complete when this grid is
    // launched): loaded while the distinct counts are still being finished
    int lab = -1;
    unsigned nk = 0;
    if (r < a.n) {
        lab = __ldcg(a.y32 + r);
        if (lab >= 0) nk = __ldcg(a.cnt + lab);
    }
    if (blockIdx.x == 0) write_counts(a, threadIdx.x);
    KSPAN(2, 0);
    // k_bm_gemm may be scheduled now: it sets up TMEM and its barriers, then
    // waits for this grid (and so for k_bm_sym) before reading anything
    pdl_trigger();
    pdl_wait();
    KSPAN(2, 1);
    if (r < a.n) {
        // a shard without the Laplacian needs no degrees (s_r = 1)
        const unsigned L = !a.shard ? __ldcg(a.ucnt + r) : a.deg_all ? __ldcg(a.deg_all + r) : 0u;
        node_entry(a, r, L, lab, nk);
    }
    KSPAN(2, 2);
}

// directed lists: one warp per row, 8 rows per CTA
__global__ void __launch_bounds__(256) k_bm_scan(BmArgs a) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    pdl_wait();
    if (r >= a.nloc) return;
    unsigned u = 0;
    for (int i = lane; i < a.Wp / 4; i += 32) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(a.bm + bm_index(a, r, 4 * i)));
        u += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    u = warp_sum_u(u);
    if (lane == 0) {
        a.ucnt[r] = u;
        if (u) atomicAdd(a.upop + (blockIdx.x % kPopParts) * 32, u);  // popc(U): S = U for directed lists
    }
}

// Does some pair repeat in the stream?  popc(U) = E exactly when none does
// (undirected lists: and no pair is present in both directions).  Every
// thread of the CTA gets the answer.
__device__ __forceinline__ bool block_repeats(const BmArgs &a) {
    __shared__ unsigned s_rep;
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) TRACE(7, 3);
        // every load issued before any is used: one round trip
        const unsigned mut = threadIdx.x == 0 ? __ldcg(a.flags) : 0u;
        unsigned long long tot = 0;
        for (int i = threadIdx.x; i < kPopParts; i += 32) tot += __ldcg(a.upop + i * 32);
        if (threadIdx.x == 0) TRACE(7, 4);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (threadIdx.x == 0) s_rep = mut != 0 || (int64_t)tot != a.E;
        if (threadIdx.x == 0) TRACE(7, 5);
    }
    __syncthreads();
    return s_rep != 0;
}

// Row shard, after k_bm_scan: when some pair repeats, the exact stream
// lengths of the local rows (their degrees) and zeroed class sums.
__global__ void __launch_bounds__(256) k_bm_len(const int64_t *__restrict__ rows, BmArgs a) {
    pdl_wait();
    if (!block_repeats(a)) return;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < (int64_t)a.nloc * kKMax; i += nth) a.zacc[i] = 0.0;
    for (int64_t e = tid; e < a.E; e += nth) {
        const unsigned r = (unsigned)rows[e] - (unsigned)a.row0;
        if (r < (unsigned)a.nloc) atomicAdd(&a.len[r], 1u);
    }
}

// Row shard: the local rows' degrees (stream lengths) for the all-gather
__global__ void __launch_bounds__(256) k_bm_deg(BmArgs a, unsigned *__restrict__ deg_local) {
    pdl_wait();
    const bool rep = block_repeats(a);
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < a.nloc) deg_local[r] = rep ? __ldcg(a.len + r) : __ldcg(a.ucnt + r);
}

// ---------------------------------------------------------------------------
// rare path
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_gpu(ctr) < target) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
}

// rare path phases 1-3 (all CTAs of k_bm_gemm; co-resident)
__device__ void repeat_phases(const int64_t *__restrict__ rows, const int64_t *__restrict__ cols, const BmArgs &a) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    if (a.shard) {
        // a row shard's lengths, zeroed sums (k_bm_len) and node table (from
        // the all-gathered degrees) are ready: only the class sums of the
        // local rows with repeats, over the local (directed) stream
        for (int64_t e = tid; e < a.E; e += nth) {
            const unsigned r = (unsigned)rows[e] - (unsigned)a.row0, c = (unsigned)cols[e];
            if (r < (unsigned)a.nloc && __ldcg(a.len + r) != __ldcg(a.ucnt + r)) {
                const int lab = __ldcg(a.tab_lab + c);
                if (lab >= 0) atomicAdd(&a.zacc[(size_t)r * kKMax + lab], __ldcg(a.tab_g + c));
            }
        }
        grid_barrier(a.flags + 1, gridDim.x);
        return;
    }
    const bool und = !a.directed;
    // 1: exact stream lengths
    for (int64_t i = tid; i < (int64_t)a.n * kKMax; i += nth) a.zacc[i] = 0.0;
    for (int64_t e = tid; e < a.E; e += nth) {
        const unsigned r = (unsigned)rows[e], c = (unsigned)cols[e];
        atomicAdd(&a.len[r], 1u);
        if (und && r != c) atomicAdd(&a.len[c], 1u);
    }
    grid_barrier(a.flags + 1, gridDim.x);
    // 2: node table from the stream lengths
    for (int64_t r = tid; r < a.n; r += nth) node_entry(a, (int)r, __ldcg(a.len + r));
    asm volatile("fence.proxy.async.global;" ::: "memory");
    grid_barrier(a.flags + 1, 2 * gridDim.x);
    // 3: per-class sums of g over every stream entry of rows with repeats
    for (int64_t e = tid; e < a.E; e += nth) {
        const unsigned r = (unsigned)rows[e], c = (unsigned)cols[e];
        if (__ldcg(a.len + r) != __ldcg(a.ucnt + r)) {
            const int lab = __ldcg(a.tab_lab + c);
            if (lab >= 0) atomicAdd(&a.zacc[(size_t)r * kKMax + lab], __ldcg(a.tab_g + c));
        }
        if (und && r != c && __ldcg(a.len + c) != __ldcg(a.ucnt + c)) {
            const int lab = __ldcg(a.tab_lab + r);
            if (lab >= 0) atomicAdd(&a.zacc[(size_t)c * kKMax + lab], __ldcg(a.tab_g + r));
        }
    }
    grid_barrier(a.flags + 1, 3 * gridDim.x);
}

// ---------------------------------------------------------------------------
// k_bm_gemm: tcgen05 helpers (inline PTX, sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "GEE_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra GEE_DONE;\n\t"
        "bra GEE_WAIT;\n"
        "GEE_DONE:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// a waiter off the critical path: back off between polls so the spinning
// warp does not take issue slots from the producers
__device__ __forceinline__ void mbar_wait_idle(uint32_t bar, uint32_t parity, unsigned ns) {
    uint32_t ok = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
    }
}

// K-major operand, 128-byte swizzle: 8-row core groups 1024 B apart
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;             // leading byte offset (unused: K fits one swizzle row)
    d |= (uint64_t)(1024 >> 4) << 32;   // stride byte offset
    d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;             // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

// A from TMEM (K-major, row = lane), B from shared memory
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

// two bitmap words (64 columns of a row) -> 16 TMEM columns of bytes 0/1
__device__ __forceinline__ void tmem_st_word2(uint32_t taddr, unsigned x, unsigned y) {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = ((x >> (4 * i)) & 0xFu) * 0x00204081u & 0x01010101u;
        v[8 + i] = ((y >> (4 * i)) & 0xFu) * 0x00204081u & 0x01010101u;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
        "elect.sync rx|px, %1;\n\t"
        "@px mov.s32 %0, 1;\n\t}"
        : "+r"(pred)
        : "r"(0xffffffffu));
    return pred != 0;
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// 8 bits of a word -> 8 bytes of 0/1 (two u32): nibble * 0x00204081 puts
// bit i of the nibble at bit 8i, no carries
__device__ __forceinline__ uint4 expand16(unsigned w) {
    uint4 o;
    o.x = ((w & 0xFu) * 0x00204081u) & 0x01010101u;
    o.y = (((w >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
    o.z = (((w >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
    o.w = (((w >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
    return o;
}

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// 2^e for a normal exponent, exactly
__device__ __forceinline__ double pow2i(int e) {
    return __longlong_as_double((long long)(1023 + e) << 52);
}

// Z row epilogue (one thread per row): per-class sums v_q of s_c (digits
// recombined, or the rare path's f64 sums of g), then 1/n_q, diagonal, s_r,
// correlation
template <int NB>
__device__ __forceinline__ void gemm_epilogue(const BmArgs &a, int r, const int32_t (&C)[NB], bool rep,
                                              const double (&inv)[kKMax], double sr, int lab) {
    double acc[kKMax];
    const bool lap = (a.flags_opts & GEE_LAPLACIAN) != 0;
    if (rep) {
#pragma unroll
        for (int q = 0; q < kKMax; ++q) acc[q] = q < a.k ? __ldcg(a.zacc + (size_t)r * kKMax + q) : 0.0;
    } else {
#pragma unroll
        for (int q = 0; q < kKMax; ++q) {
            double v = 0.0;
            if (q * kDig + kDig <= NB && q < a.k) {
                // sum_c s_c * 2^55 = lo + hi * 2^32 exactly in integers (digit
                // sums < 2^23: lo < 2^48, hi < 2^40), one rounding to f64
                const int32_t *D = C + q * kDig;
                const long long lo = (long long)D[0] + ((long long)D[1] << 8) + ((long long)D[2] << 16) +
                                     ((long long)D[3] << 24);
                const long long hi = (long long)D[4] + ((long long)D[5] << 8) + ((long long)D[6] << 16);
                v = fma((double)hi, pow2i(32 - 55), (double)lo * pow2i(-55)) * inv[q];
            }
            acc[q] = v;
        }
    }
    if (a.flags_opts & GEE_DIAGONAL) {
        // A+I: the diagonal gains 1.0 whether or not (r, r) is stored
#pragma unroll
        for (int q = 0; q < kKMax; ++q)
            if (q == lab) acc[q] += sr * inv[q];
    }
    if (lap) {
#pragma unroll
        for (int q = 0; q < kKMax; ++q) acc[q] *= sr;
    }
    if (a.flags_opts & GEE_CORRELATION) {
        double ss = 0.0;
        bool fin = true;
#pragma unroll
        for (int q = 0; q < kKMax; ++q) {
            if (q < a.k) {
                ss += acc[q] * acc[q];
                fin &= isfinite(acc[q]);
            }
        }
        if (!fin) {
            raise_err(a.err, GEE_ERR_NONFINITE);
        } else {
            const double nrm = __dsqrt_rn(ss);
            if (nrm > 0.0) {
                const double rn = __ddiv_rn(1.0, nrm);  // within 1 ulp of acc / nrm
#pragma unroll
                for (int q = 0; q < kKMax; ++q) acc[q] *= rn;
            }
        }
    }
    double *zr = a.z + (int64_t)r * a.k;
#pragma unroll
    for (int q = 0; q < kKMax; ++q)
        if (q < a.k) zr[q] = acc[q];
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// 1-D bulk copy global -> shared (async proxy), completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }



// k_bm_gemm geometry
constexpr int kACols = kTK / 4;  // TMEM columns per A stage (128 rows x 256 bytes, 4 bytes per column)
template <int NB>
constexpr int chains() { return 2; }                    // independent accumulators per buffer
template <int NB>
constexpr int a_stages() { return (512 - 4 * NB) / kACols; }  // TMEM A stages after 2 x 2 accumulators
template <int NB>
constexpr int rr_stages() { return a_stages<NB>(); }  // ring stage s = A stage s: one release per K step
constexpr int kGemmNT = 448;    // warps 0-7 expand, 8-11 epilogue, 12 MMA, 13 bulk copies
constexpr int kExp = 128;       // expander threads per K step (thread = tile row)
constexpr int kWMma = 12, kWTma = 13;

template <int NB>
constexpr size_t gemm_smem() {
    return 1024 + (size_t)rr_stages<NB>() * (kTM * 32 + NB * kTK) + 8 * (2 * a_stages<NB>() + 2 * rr_stages<NB>() + 4) +
           16;
}

// Stream-K over the flattened (row tile, K step) space: CTA b takes steps
// [b*T/G, (b+1)*T/G), T = tiles * KT, so every CTA does the same number of K
// steps; the steps of one row tile form a segment whose integer partial sums
// are added to Cacc, and the CTA completing a tile's KT steps runs its
// epilogue.  Warp 13 bulk-copies each step's two 2 KB bitmap tiles and B
// tile (kRR stages ahead); warps 0-7 (two threads per tile row, one per
// 128-column half) expand the bits to bytes straight into the TMEM A stage;
// warp 12 issues the MMAs into one of two TMEM accumulators (segment parity);
// warps 8-11 drain the accumulators.
template <int NB>
__global__ void __launch_bounds__(kGemmNT, 1) k_bm_gemm(const int64_t *__restrict__ rows,
                                                        const int64_t *__restrict__ cols, BmArgs a) {
    extern __shared__ unsigned char sm_raw[];
    constexpr int kRR = rr_stages<NB>();
    constexpr int kRB = kTM * 32;    // 4 KB: two consecutive 2 KB bitmap tiles
    constexpr int kBB = NB * kTK;    // two consecutive X^T tiles
    constexpr int kChains = chains<NB>();
    constexpr int kAS = a_stages<NB>();
    constexpr int kAccCols = 2 * kChains * NB;  // two accumulator buffers, then the A stages
    constexpr int kTmemCols = 512;
    static_assert(kAccCols + kAS * kACols <= kTmemCols, "TMEM budget");
    unsigned char *sm = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *sB = sm;
    unsigned char *sR = sB + kRR * kBB;
    uint64_t *full = reinterpret_cast<uint64_t *>(sR + kRR * kRB);
    uint64_t *aempty = full + kAS;
    uint64_t *rfull = aempty + kAS;
    uint64_t *rempty = rfull + kRR;
    uint64_t *accfull = rempty + kRR;
    uint64_t *accempty = accfull + 2;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(accempty + 2);

    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) TRACE(7, 0);
#ifdef GEE_TRACE
    if (t == 0) g_trace_cta[blockIdx.x][0] = gtime();
#endif
    KSPAN(3, 0);
    // Launched while k_bm_table runs (PDL): k_bm_sym's outputs (bitmap, counts,
    // flags) are complete, the node table is not until pdl_wait().
    if (w == kWMma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        for (int s = 0; s < kAS; ++s) {
            mbar_init(smem_u32(full + s), kExp);
            mbar_init(smem_u32(aempty + s), 1);
        }
        for (int s = 0; s < kRR; ++s) {
            mbar_init(smem_u32(rfull + s), 1);
            mbar_init(smem_u32(rempty + s), kExp + 1);  // expanders read the bitmap tiles, the MMA the B tile
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(accfull + s), 1);
            mbar_init(smem_u32(accempty + s), kTM);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    if (t == 0) TRACE(7, 2);
#ifdef GEE_TRACE
    if (t == 0) g_trace_cta[blockIdx.x][1] = gtime();
#endif

    const int KT = a.Np / kTK;
    const int64_t total = (int64_t)(a.Nlp / kTM) * KT;
    const int s0 = (int)((int64_t)blockIdx.x * total / gridDim.x);
    const int s1 = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
    const int nsteps = s1 - s0;
    const int pre = min(nsteps, kRR);

    // Launched (PDL) while k_bm_table runs, possibly before k_bm_sym is
    // done: TMEM and the barriers are set up by now; after pdl_wait() the
    // bitmap, counts and node table are complete.  The first kRR bitmap tiles
    // go out at once; the repeat check (one round trip) overlaps them, and
    // the X^T tiles follow it (the rare path rewrites X^T).
    pdl_wait();
#ifdef GEE_TRACE
    if (t == 0) atomicMin(&g_kspan[3][1], gtime());
#endif
    if (w == kWTma && lane == 0) {
        for (int i = 0; i < pre; ++i) {
            const int g = s0 + i, m = g / KT, ks = g % KT;
            const uint32_t bar = smem_u32(rfull + i);
            mbar_expect_tx(bar, kRB + kBB);
            bulk_g2s(smem_u32(sR + i * kRB), a.bm + ((size_t)(m * KT + ks) << 10), kRB, bar);
        }
    }
    const bool rep = block_repeats(a);
    if (rep) repeat_phases(rows, cols, a);
    if (t == 0) TRACE(7, 1);

    if (w == kWTma) {
        // ---- bulk copies
        if (lane == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            for (int i = 0; i < pre; ++i) {
                const int ks = (s0 + i) % KT;
                bulk_g2s(smem_u32(sB + i * kBB), a.xt + (size_t)ks * kBB, kBB, smem_u32(rfull + i));
            }
#pragma unroll 1
            for (int i = pre; i < nsteps; ++i) {
                const int rs = i % kRR, g = s0 + i, m = g / KT, ks = g % KT;
                mbar_wait_idle(smem_u32(rempty + rs), ((i / kRR) - 1) & 1, 32);
                const uint32_t bar = smem_u32(rfull + rs);
                TRACE(0, i);
                mbar_expect_tx(bar, kRB + kBB);
                bulk_g2s(smem_u32(sR + rs * kRB), a.bm + ((size_t)(m * KT + ks) << 10), kRB, bar);
                bulk_g2s(smem_u32(sB + rs * kBB), a.xt + (size_t)ks * kBB, kBB, bar);
            }
        }
        __syncwarp();
    } else if (w < 8) {
        // ---- bit -> byte expansion, thread = tile row.  Two groups (warps
        // 0-3, 4-7) take alternate K steps, so one group's TMEM stores are in
        // flight while the other waits for its own to land; a warp reaches
        // only TMEM lanes 32(w%4)..32(w%4)+31
        const int rl = t & 127, grp = t >> 7;
#pragma unroll 1
        for (int i = grp; i < nsteps; i += 2) {
            const int rs = i % kRR, as = i % kAS;
            mbar_wait(smem_u32(rfull + rs), (i / kRR) & 1);
            const uint4 w0 = lds128(smem_u32(sR + rs * kRB + rl * 16));
            const uint4 w1 = lds128(smem_u32(sR + rs * kRB + kTM * 16 + rl * 16));
            mbar_arrive(smem_u32(rempty + rs));
            // A stage as is free: the ring refilled stage rs (= as) only after
            // the MMAs of step i - kAS, which read it, had completed
            // row rl of the A stage = TMEM lane rl: column 8m + i holds the
            // bytes of bits 4i..4i+3 of word m (K-major, 4 bytes per column)
            const uint32_t ta = tmem + ((uint32_t)((w & 3) * 32) << 16) + kAccCols + as * kACols;
            tmem_st_word2(ta + 0, w0.x, w0.y);
            tmem_st_word2(ta + 16, w0.z, w0.w);
            tmem_st_word2(ta + 32, w1.x, w1.y);
            tmem_st_word2(ta + 48, w1.z, w1.w);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(smem_u32(full + as));
            if ((rl & 31) == 0) TRACE(1 + (rl >> 5), i);
#ifdef GEE_TRACE
            if (i == 0 && t == 0) g_trace_cta[blockIdx.x][6] = gtime();
#endif
        }
    } else if (w == kWMma) {
        // ---- MMA issue: the whole warp runs the loop (warp-uniform operands
        // stay in uniform registers); one elected lane issues
        const bool leader = elect_one();
        const uint32_t idesc = (2u << 4) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
        int seg = 0;
#pragma unroll 1
        for (int i = 0; i < nsteps; ++i) {
            const int ks = (s0 + i) % KT;
            const bool first = i == 0 || ks == 0, last = i == nsteps - 1 || ks == KT - 1;
            const int buf = seg & 1;
            if (first && seg >= 2) mbar_wait(smem_u32(accempty + buf), ((seg >> 1) - 1) & 1);
            const int as = i % kAS, rs = i % kRR;
            mbar_wait(smem_u32(full + as), (i / kAS) & 1);  // expanders passed rfull[rs] first
            if (leader) TRACE(8, i);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t ta = tmem + kAccCols + as * kACols;
            const uint64_t bd = sdesc_sw128(smem_u32(sB + rs * kBB));
            if (leader) {
#pragma unroll
                for (int k = 0; k < kTK / 32; ++k)
                    mma_i8_ts(tmem + (buf * kChains + (k % kChains)) * NB, ta + 8 * k,
                              bd + (k >> 2) * (NB * 128 >> 4) + 2 * (k & 3), idesc, !first || k >= kChains);
                mma_commit(smem_u32(rempty + rs));  // bitmap, B and A stage all free
                if (last) mma_commit(smem_u32(accfull + buf));
            }
            __syncwarp();
            if (last) ++seg;
        }
#ifdef GEE_TRACE
        if (lane == 0) g_trace_cta[blockIdx.x][2] = gtime();
#endif
    } else {
        // ---- epilogue: warp 4 + e reads TMEM lanes 32e..32e+31 (= tile rows)
        const int e = w - 8;  // TMEM lane quarter w % 4
        {
            // Touch the pages the tail will use (partial slabs of this CTA and
            // its neighbours, the stream-K counters, this CTA's Z rows) while
            // waiting for the first accumulator: their address translations
            // are then cached when the epilogue is on the critical path.
            const int tt = t - 32 * 8;
            const int nb = (int)gridDim.x;
            const int bb = min(max((int)blockIdx.x + (tt % 5) - 2, 0), nb - 1);
            const char *p0 = reinterpret_cast<const char *>(a.cpart + (size_t)bb * 2 * kTM * NB) + (tt / 5) * 4096;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p0));
            const int m0 = s0 / KT, m1 = (s1 - 1) / KT;
            const int rr = min((tt & 1 ? m1 : m0) * kTM + (tt >> 1), a.n - 1);
            if (nsteps > 0 && rr >= 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.z + (size_t)rr * a.k));
            if (tt == 0 && nsteps > 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.mdone + m0));
        }
        double inv[kKMax];
#pragma unroll
        for (int q = 0; q < kKMax; ++q) inv[q] = q < a.k ? __ldcg(a.inv + q) : 0.0;
        const bool lap = (a.flags_opts & GEE_LAPLACIAN) != 0;
        int seg = 0;
#pragma unroll 1
        for (int i = 0; i < nsteps; ++seg) {
            const int g = s0 + i, m = g / KT;
            const int seglen = min(nsteps - i, KT - g % KT);
            const int buf = seg & 1;
            const int r = m * kTM + e * 32 + lane;  // local row
            const bool live = r < a.nloc;
            // the row's epilogue inputs, loaded while the MMAs run
            const int rlab = live ? __ldcg(a.y32 + a.row0 + r) : -1;
            const double rsc = (lap && live) ? __ldcg(a.scale + a.row0 + r) : 1.0;
            mbar_wait_idle(smem_u32(accfull + buf), (seg >> 1) & 1, 32);
#ifdef GEE_TRACE
            if (seg == 0 && e == 0 && lane == 0) g_trace_cta[blockIdx.x][4] = gtime();
            if (e == 0 && lane == 0) g_trace_cta[blockIdx.x][11] = gtime();
#endif
            if (e == 0 && lane == 0) TRACE(9, seg);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            int32_t C[NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) C[j] = 0;
            {
                uint32_t v[kChains][NB];
#pragma unroll
                for (int ch = 0; ch < kChains; ++ch)
#pragma unroll
                    for (int c0 = 0; c0 < NB; c0 += 16)
                        tmem_ld16(tmem + ((uint32_t)(e * 32) << 16) + (buf * kChains + ch) * NB + c0,
                                  *reinterpret_cast<uint32_t(*)[16]>(&v[ch][c0]));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int ch = 0; ch < kChains; ++ch)
#pragma unroll
                    for (int j = 0; j < NB; ++j) C[j] += (int32_t)v[ch][j];
            }
            if (e == 0 && lane == 0) TRACE(9, 16 + 8 * seg);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(smem_u32(accempty + buf));
            const int sidx = m - s0 / KT;  // this CTA's segment index (0 or 1)
            // Tile m's finisher is the CTA holding its first K step (its segment
            // of m ends last in time: it is that CTA's final segment, while the
            // partners' segments of m are mostly their first).  Partners store
            // their partial sums and bump ready[m]; the finisher never waits on
            // its own store, it only polls ready[m] and reads the partners' slabs.
            const bool fin = g % KT == 0;
            // the CTAs whose step ranges meet tile m (32-bit: T <= 128 * 64)
            const unsigned G = gridDim.x, T = (unsigned)total;
            const unsigned lo = (unsigned)m * KT, hi = lo + KT;
            if (!fin) {
                int4 *dst = reinterpret_cast<int4 *>(a.cpart + (((size_t)blockIdx.x * 2 + sidx) * kTM + e * 32 + lane) * NB);
#pragma unroll
                for (int j = 0; j < NB / 4; ++j) dst[j] = make_int4(C[4 * j], C[4 * j + 1], C[4 * j + 2], C[4 * j + 3]);
                // the barrier orders the 128 threads' stores before one
                // gpu-scope release (cumulative), which publishes the slab
                epi_bar();
                if (e == 0 && lane == 0) red_release_gpu(&a.mdone[m], 1u);
#ifdef GEE_TRACE
                if (seg == 0 && e == 0 && lane == 0) g_trace_cta[blockIdx.x][5] = gtime();
#endif
            } else if (seglen < KT && live) {
                // partners: participating CTAs other than this one
                unsigned b = lo * G / T;
                while (b > 0 && b * T / G > lo) --b;
                while ((b + 1) * T / G <= lo) ++b;
                unsigned npart = 0;
                for (unsigned bb = b; bb < G && bb * T / G < hi; ++bb) {
                    const unsigned bs0 = bb * T / G, bs1 = (bb + 1) * T / G;
                    if (bb != blockIdx.x && bs1 != bs0 && bs1 > lo) ++npart;
                }
                while (ld_acquire_gpu(a.mdone + m) < npart) {
                }
#ifdef GEE_TRACE
                if (e == 0 && lane == 0) g_trace_cta[blockIdx.x][8] = gtime();
#endif
                for (; b < G && b * T / G < hi; ++b) {
                    const unsigned bs0 = b * T / G, bs1 = (b + 1) * T / G;
                    if (b == blockIdx.x || bs1 == bs0 || bs1 <= lo) continue;  // self, idle CTAs
                    const int bsi = m - (int)(bs0 / KT);
                    const int4 *src = reinterpret_cast<const int4 *>(
                        a.cpart + (((size_t)b * 2 + bsi) * kTM + e * 32 + lane) * NB);
#pragma unroll
                    for (int j = 0; j < NB / 4; ++j) {
                        const int4 v = src[j];  // after the acquire: L1 holds no stale copy
                        C[4 * j] += v.x, C[4 * j + 1] += v.y, C[4 * j + 2] += v.z, C[4 * j + 3] += v.w;
                    }
                }
            }
            if (fin && live) {
                if (e == 0 && lane == 0) TRACE(9, 19 + 8 * seg);
#ifdef GEE_TRACE
                if (e == 0 && lane == 0) g_trace_cta[blockIdx.x][9] = gtime();
#endif
                const bool rrep = rep && __ldcg(a.len + r) != __ldcg(a.ucnt + r);
                gemm_epilogue<NB>(a, r, C, rrep, inv, rsc, rlab);
                if (e == 0 && lane == 0) TRACE(9, 20 + 8 * seg);
#ifdef GEE_TRACE
                if (e == 0 && lane == 0) g_trace_cta[blockIdx.x][10] = gtime();
#endif
            }
            if (e == 0 && lane == 0) TRACE(9, 8 + seg);
            i += seglen;
        }
#ifdef GEE_TRACE
        if (e == 0 && lane == 0) g_trace_cta[blockIdx.x][3] = gtime();
#endif
    }
    if (t == 0) TRACE(5, 0);
#ifdef GEE_TRACE
    if (t == 256) g_trace_end[blockIdx.x] = gtime();
#endif
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    KSPAN(3, 2);
    if (w == kWMma) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

// ---------------------------------------------------------------------------
int force_path();

int bitmap_max_nodes() { return kBmMax; }

// unit weights, square, at most kBmMax nodes, K <= 8
bool bitmap_path_ok(int wt, int64_t E, int64_t n_rows, int64_t n_cols, int directed, int k) {
    if (force_path() != 0) return false;  // test hook: exercise the general paths
    const int64_t M = directed ? E : 2 * E;
    return wt == GEE_W_UNIT && n_rows == n_cols && n_rows >= 1 && n_rows <= kBmMax && k >= 1 && k <= kKMax &&
           M < ((int64_t)1 << 31);
}

static int nb_cols(int k) {
    const int need = k * kDig;
    return need <= 16 ? 16 : need <= 32 ? 32 : 64;
}

struct BmWs {
    unsigned *bm, *ucnt, *len, *cnt, *mdone, *flags, *upop;
    unsigned char *xt;
    int32_t *cacc;
    double *zacc, *tab_g;
    signed char *tab_lab;
    int Wp, Np, Nlp, nbx;
    size_t clear_bytes;
    // row shards only: the label outputs and node tables of every node
    int32_t *y32;
    int64_t *counts;
    double *inv, *deg, *scale;
};

// nloc rows of an n-node graph (the single-GPU encode: nloc = n)
static void carve_bm(Carver &cv, BmWs &w, int64_t n, int64_t nloc, int k, bool shard) {
    const int64_t np = (n + kBlk - 1) / kBlk * kBlk;
    const int64_t nlp = shard ? std::max<int64_t>(kTM, (nloc + kTM - 1) / kTM * kTM) : np;
    w.Wp = (int)(np / 32);
    w.Np = (int)np;
    w.Nlp = (int)nlp;
    w.nbx = nb_cols(k);
    // bitmap, counters, flags and X^T are contiguous: one memset clears them
    const size_t bmw = (size_t)nlp * w.Wp;
    const size_t words =
        (bmw + 2 * (size_t)nloc + kKMax + (size_t)(nlp / kTM) + 4 + 32 * kPopParts + 3) & ~size_t(3);
    const size_t xbytes = (size_t)w.nbx * (size_t)np;
    w.clear_bytes = 4 * words + xbytes;
    unsigned char *base = cv.take<unsigned char>(w.clear_bytes);
    w.bm = reinterpret_cast<unsigned *>(base);
    w.ucnt = w.bm ? w.bm + bmw : nullptr;
    w.len = w.bm ? w.ucnt + nloc : nullptr;
    w.cnt = w.bm ? w.len + nloc : nullptr;
    w.mdone = w.bm ? w.cnt + kKMax : nullptr;
    w.flags = w.bm ? w.mdone + nlp / kTM : nullptr;
    w.upop = w.bm ? w.flags + 4 : nullptr;
    w.xt = base ? base + 4 * words : nullptr;
    w.cacc = cv.take<int32_t>((size_t)num_sms() * 2 * kTM * w.nbx);
    w.zacc = cv.take<double>((size_t)std::max<int64_t>(nloc, 1) * kKMax);
    w.tab_g = cv.take<double>((size_t)n + 2);
    w.tab_lab = cv.take<signed char>((size_t)n + 16);
    w.y32 = nullptr;
    w.counts = nullptr;
    w.inv = w.deg = w.scale = nullptr;
    if (shard) {
        w.y32 = cv.take<int32_t>((size_t)n);
        w.counts = cv.take<int64_t>(kKMax);
        w.inv = cv.take<double>(kKMax);
        w.deg = cv.take<double>((size_t)n);
        w.scale = cv.take<double>((size_t)n);
    }
}

size_t bitmap_workspace(int64_t E, int64_t n, int directed, int k) {
    (void)E;
    (void)directed;
    Carver cv(nullptr);
    BmWs w;
    carve_bm(cv, w, n, n, k, false);
    return cv.bytes();
}

// launch with the programmatic-dependent-launch attribute (and optionally
// cooperative); its kernel calls pdl_wait() before reading its inputs
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              bool coop, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int NB>
static int launch_gemm(const BmArgs &a, const int64_t *rows, const int64_t *cols, cudaStream_t st) {
    static PerDevice attr;
    if (!attr.done()) {
        GEE_CHECK_CUDA(cudaFuncSetAttribute(k_bm_gemm<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)gemm_smem<NB>()));
        attr.mark();
    }
    // persistent stream-K grid, one CTA per SM; cooperative so the rare
    // path's grid barrier is safe (a launch error, never a hang)
    GEE_CHECK_CUDA(launch_pdl(k_bm_gemm<NB>, dim3((unsigned)num_sms()), dim3(kGemmNT), gemm_smem<NB>(), st, true, rows,
                              cols, a));
    GEE_CHECK_LAUNCH("k_bm_gemm");
    return GEE_OK;
}

// The fused encode for unit-weight graphs, labels included.  Outputs: y32,
// counts, 1/n_k, Z (n x k) and, under the Laplacian, deg / scale.  The CSR
// is not materialised.
int bitmap_encode(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int directed,
                  const int64_t *labels, int k, unsigned flags, int32_t *y32, int64_t *counts, double *inv,
                  double *deg, double *scale, double *z, void *ws, size_t ws_bytes, int32_t *err,
                  cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, n, n, k, false);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    BmArgs a;
    a.n = (int)n;
    a.Wp = W.Wp;
    a.Np = W.Np;
    a.row0 = 0;
    a.nloc = (int)n;
    a.Nlp = W.Nlp;
    a.shard = 0;
    a.deg_all = nullptr;
    a.E = E;
    a.directed = directed;
    a.bm = W.bm;
    a.ucnt = W.ucnt;
    a.len = W.len;
    a.cnt = W.cnt;
    a.mdone = W.mdone;
    a.flags = W.flags;
    a.upop = W.upop;
    a.xt = W.xt;
    a.nbx = W.nbx;
    a.cpart = W.cacc;
    a.zacc = W.zacc;
    a.labels = labels;
    a.y32 = y32;
    a.counts = counts;
    a.inv = inv;
    a.deg = deg;
    a.scale = scale;
    a.tab_g = W.tab_g;
    a.tab_lab = W.tab_lab;
    a.flags_opts = flags;
    a.z = z;
    a.k = k;
    a.err = err;
    GEE_CHECK_CUDA(cudaMemsetAsync(W.bm, 0, W.clear_bytes, st));
    profile_mark("memset(bitmap)", st);  // its own line in the bench breakdown (not a kernel of ours)
    k_bm_set<<<(unsigned)num_sms() * 4, kSetThreads, 0, st>>>(rows, cols, a);
    GEE_CHECK_LAUNCH("k_bm_set");
    if (!directed) {
        const unsigned nt = (unsigned)(W.Np / kSB);
        GEE_CHECK_CUDA(launch_pdl(k_bm_sym, dim3(nt * (nt + 1) / 2), dim3(kSB), 0, st, false, a));
        GEE_CHECK_LAUNCH("k_bm_sym");
    } else {
        GEE_CHECK_CUDA(launch_pdl(k_bm_scan, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, st, false, a));
        GEE_CHECK_LAUNCH("k_bm_scan");
    }
    GEE_CHECK_CUDA(launch_pdl(k_bm_table, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, false, a));
    GEE_CHECK_LAUNCH("k_bm_table");
    if (W.nbx == 16) return launch_gemm<16>(a, rows, cols, st);
    if (W.nbx == 32) return launch_gemm<32>(a, rows, cols, st);
    return launch_gemm<64>(a, rows, cols, st);
}

// ---------------------------------------------------------------------------
// Row shards (multi-GPU, dist.py): rank p holds rows [row0, row0 + nloc) and
// their entries of the symmetrised stream (a directed list, global ids).
// Phase 1 (bitmap_shard_degrees): labels of every node, the local bitmap
// rows, their popcounts and -- when a pair repeats -- exact stream lengths;
// returns the local rows' degrees.  The caller all-gathers them (NCCL).
// Phase 2 (bitmap_shard_encode): the node table of every node from the
// gathered degrees, then the GEMM over the local row tiles -> Z's local rows.
// Both phases take the same workspace, untouched in between.
static BmArgs shard_args(const BmWs &W, int64_t E, int64_t n, int64_t row0, int64_t nloc, int k, unsigned flags,
                         int32_t *err) {
    BmArgs a = {};
    a.n = (int)n;
    a.Wp = W.Wp;
    a.Np = W.Np;
    a.row0 = (int)row0;
    a.nloc = (int)nloc;
    a.Nlp = W.Nlp;
    a.shard = 1;
    a.deg_all = nullptr;
    a.E = E;
    a.directed = 1;  // the local stream holds both directions explicitly
    a.bm = W.bm;
    a.ucnt = W.ucnt;
    a.len = W.len;
    a.cnt = W.cnt;
    a.mdone = W.mdone;
    a.flags = W.flags;
    a.upop = W.upop;
    a.xt = W.xt;
    a.nbx = W.nbx;
    a.cpart = W.cacc;
    a.zacc = W.zacc;
    a.labels = nullptr;
    a.y32 = W.y32;
    a.counts = W.counts;
    a.inv = W.inv;
    a.deg = W.deg;
    a.scale = W.scale;
    a.tab_g = W.tab_g;
    a.tab_lab = W.tab_lab;
    a.flags_opts = flags;
    a.z = nullptr;
    a.k = k;
    a.err = err;
    return a;
}

size_t bitmap_shard_workspace(int64_t n, int64_t nloc, int k) {
    Carver cv(nullptr);
    BmWs w;
    carve_bm(cv, w, n, nloc, k, true);
    return cv.bytes();
}

int bitmap_shard_degrees(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int64_t row0, int64_t nloc,
                         const int64_t *labels, int k, unsigned flags, unsigned *deg_local, void *ws,
                         size_t ws_bytes, int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, n, nloc, k, true);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    BmArgs a = shard_args(W, E, n, row0, nloc, k, flags, err);
    a.labels = labels;
    GEE_CHECK_CUDA(cudaMemsetAsync(W.bm, 0, W.clear_bytes, st));
    profile_mark("memset(bitmap)", st);  // its own line in the bench breakdown (not a kernel of ours)
    k_bm_set<<<(unsigned)num_sms() * 4, kSetThreads, 0, st>>>(rows, cols, a);
    GEE_CHECK_LAUNCH("k_bm_set");
    const unsigned nb = (unsigned)std::max<int64_t>(1, (nloc + 7) / 8);
    GEE_CHECK_CUDA(launch_pdl(k_bm_scan, dim3(nb), dim3(256), 0, st, false, a));
    GEE_CHECK_LAUNCH("k_bm_scan");
    GEE_CHECK_CUDA(launch_pdl(k_bm_len, dim3((unsigned)num_sms() * 2), dim3(256), 0, st, false, rows, a));
    GEE_CHECK_LAUNCH("k_bm_len");
    GEE_CHECK_CUDA(launch_pdl(k_bm_deg, dim3((unsigned)std::max<int64_t>(1, (nloc + 255) / 256)), dim3(256), 0, st,
                              false, a, deg_local));
    GEE_CHECK_LAUNCH("k_bm_deg");
    return GEE_OK;
}

int bitmap_shard_encode(const int64_t *rows, const int64_t *cols, int64_t E, int64_t n, int64_t row0, int64_t nloc,
                        int k, unsigned flags, const unsigned *deg_all, double *z_local, void *ws, size_t ws_bytes,
                        int32_t *err, cudaStream_t st) {
    Carver cv(ws);
    BmWs W;
    carve_bm(cv, W, n, nloc, k, true);
    if (ws_bytes < cv.bytes()) return GEE_E_WORKSPACE;
    BmArgs a = shard_args(W, E, n, row0, nloc, k, flags, err);
    a.deg_all = (flags & GEE_LAPLACIAN) ? deg_all : nullptr;
    a.z = z_local;
    // plain launch: the predecessor is the degree all-gather
    k_bm_table<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
    GEE_CHECK_LAUNCH("k_bm_table");
    if (W.nbx == 16) return launch_gemm<16>(a, rows, cols, st);
    if (W.nbx == 32) return launch_gemm<32>(a, rows, cols, st);
    return launch_gemm<64>(a, rows, cols, st);
}

#ifdef GEE_TRACE
extern "C" int gee_kspan(unsigned long long *out, int reset) {
    if (reset) {
        unsigned long long init[8][3];
        for (int k = 0; k < 8; ++k) init[k][0] = init[k][1] = ~0ull, init[k][2] = 0;
        return cudaMemcpyToSymbol(g_kspan, init, sizeof(init)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(out, g_kspan, sizeof(g_kspan)) == cudaSuccess ? 0 : -1;
}

extern "C" int gee_trace_dump(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess &&
                   cudaMemcpyFromSymbol(out + 640, g_trace_end, sizeof(g_trace_end)) == cudaSuccess &&
                   cudaMemcpyFromSymbol(out + 800, g_trace_cta, sizeof(g_trace_cta)) == cudaSuccess
               ? 0
               : -1;
}
#endif
}  // namespace gee
